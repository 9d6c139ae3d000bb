// common.cuh -- error handling, device buffers and small device helpers shared
// by the libtgraph translation units.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "tgraph.h"

namespace tg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define TG_CK(call)                                                                     \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      ::tg::fail(TG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e) + " @" +  \
                              __FILE__ + ":" + std::to_string(__LINE__));               \
  } while (0)

#define TG_REQUIRE(cond, code, msg) \
  do {                              \
    if (!(cond)) ::tg::fail((code), (msg)); \
  } while (0)

// Owning device allocation (cudaMalloc), move-only.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) {
      cudaError_t e = cudaMalloc(&p, count * sizeof(T));
      if (e != cudaSuccess) {
        p = nullptr;
        n = 0;
        cudaGetLastError();
        fail(e == cudaErrorMemoryAllocation ? TG_ECAPACITY : TG_ECUDA,
             "cudaMalloc(" + std::to_string(count * sizeof(T)) + " B): " + cudaGetErrorString(e));
      }
    }
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
  T* get() const { return p; }
};

constexpr uint32_t kRemote = 0x80000000u;  // col entry flag: payload is an outbox slot
constexpr uint32_t kInf = 0xFFFFFFFFu;

__device__ __forceinline__ bool bit_test(const uint32_t* bm, uint32_t i) {
  return (bm[i >> 5] >> (i & 31)) & 1u;
}
__device__ __forceinline__ void bit_set_atomic(uint32_t* bm, uint32_t i) {
  atomicOr(&bm[i >> 5], 1u << (i & 31));
}

// L2 eviction-priority hints (createpolicy + .L2::cache_hint): gathered hot
// state is loaded evict_last, single-use streams evict_first, so the 126 MB L2
// keeps the hub prefix of the gathered arrays.
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(p) : "f"(1.0f));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, %1;" : "=l"(p) : "f"(1.0f));
  return p;
}
__device__ __forceinline__ float ld_f32_hint(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_u32_hint(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
// L1 placement variants: no_allocate for single-use data, evict_last for hubs
__device__ __forceinline__ float ld_f32_hot(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::evict_last.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_f32_cold(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
// coherent (not .nc) load with an L2 policy: data other threads update with
// atomics in the same kernel (SSSP distances)
__device__ __forceinline__ uint32_t ld_u32_hint_coh(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_f64_hint_coh(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint16_t ld_u16_hint(const uint16_t* p, uint64_t pol) {
  uint16_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_u32_stream(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_f32_hint(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 64u) {
  uint64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

__host__ __device__ __forceinline__ uint64_t words_for(uint64_t bits) { return (bits + 31) / 32; }

}  // namespace tg
