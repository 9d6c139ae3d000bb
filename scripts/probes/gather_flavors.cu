// Load-flavor probe (round 2, session 3).  PageRank's class pulls read ~1.4
// L2 sectors per L1-missing 4-byte gather (ncu: lts__t_sectors_srcunit_tex_op_read
// vs l1tex sectors).  Which load flavor fetches exactly one sector per miss,
// and does it gather faster?  Random 4 B gathers (hashed indices, U = 8 in
// flight per thread) over a 16 MB (L2-resident) and a 1 GB region with:
//   0 ld.global.nc.L2::cache_hint (evict_last)  -- PageRank's hot gathers
//   1 ld.global.nc
//   2 ld.global (.ca)
//   3 ld.global.cg (L2 only)
//   4 ld.global.nc.L1::no_allocate
//   5 ld.global.cs
// Measurement tool, not product code.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

template <int F>
__device__ __forceinline__ float ld(const float* p, uint64_t pol) {
  float v;
  if constexpr (F == 0) asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  else if constexpr (F == 1) asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if constexpr (F == 2) asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if constexpr (F == 3) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if constexpr (F == 4) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else asm volatile("ld.global.cs.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

template <int F>
__global__ void k_gather(const float* __restrict__ a, uint32_t mask, uint32_t per, float* out) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(pol) : "f"(1.0f));
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  float s = 0.f;
  for (uint32_t i = 0; i < per; i += 8) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ld<F>(a + (hash32(t * 0x9E3779B9u + i + k) & mask), pol);
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  if (s == 12345.f) out[0] = s;
}

int main() {
  const uint64_t maxn = 1ull << 28;  // 1 GB of floats
  float *a, *o;
  cudaMalloc(&a, maxn * 4);
  cudaMalloc(&o, 4);
  cudaMemset(a, 0, maxn * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 148 * 8, threads = 256;
  const uint32_t per = 512;
  const double loads = (double)blocks * threads * per;
  printf("# region_MB flavor G_loads/s   (0 nc+L2hint 1 nc 2 ca 3 cg 4 nc.L1::no_allocate 5 cs)\n");
  for (int lg : {24, 30}) {
    const uint32_t mask = (uint32_t)((1ull << (lg - 2)) - 1);
    for (int f = 0; f < 6; ++f) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        switch (f) {
          case 0: k_gather<0><<<blocks, threads>>>(a, mask, per, o); break;
          case 1: k_gather<1><<<blocks, threads>>>(a, mask, per, o); break;
          case 2: k_gather<2><<<blocks, threads>>>(a, mask, per, o); break;
          case 3: k_gather<3><<<blocks, threads>>>(a, mask, per, o); break;
          case 4: k_gather<4><<<blocks, threads>>>(a, mask, per, o); break;
          default: k_gather<5><<<blocks, threads>>>(a, mask, per, o); break;
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("%8.0f %d %10.1f\n", (double)(1ull << lg) / (1 << 20), f, loads / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
