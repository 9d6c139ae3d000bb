// L2 random-gather ceiling, second version (round 2).  The round-1 probe
// formed each index with a 64-bit modulo (% n) -- ~100 integer instructions per
// load -- so its 230 G loads/s plateau might be the probe's ALU, not the L2.
// Here the region is a power of two (index = hash & mask, a few instructions),
// and a second mode reads the indices from a streamed array exactly like
// PageRank's in_col (coalesced 4-byte index stream + dependent 4-byte gather).
// Reports G gathers/s per region size.  Measurement tool, not product code.
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

template <int U>
__global__ void k_hash(const float* __restrict__ a, uint32_t mask, uint32_t per_thread, float* out,
                       uint64_t pol_last) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  float s = 0.f;
  for (uint32_t i = 0; i < per_thread; i += U) {
    float v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t idx = hash32(t * 0x9E3779B9u + i + k) & mask;
      asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v[k]) : "l"(a + idx), "l"(pol_last));
    }
#pragma unroll
    for (int k = 0; k < U; ++k) s += v[k];
  }
  if (s == 12345.f) out[0] = s;
}

// index stream (coalesced, evict_first) + gather (evict_last): PageRank's pattern
__global__ void k_stream(const float* __restrict__ a, const uint32_t* __restrict__ idx, uint64_t n,
                         float* out, uint64_t pol_last, uint64_t pol_first) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  float s = 0.f;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint32_t c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(c[k]) : "l"(idx + i + k * stride), "l"(pol_first));
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v[k]) : "l"(a + c[k]), "l"(pol_last));
    s += v[0] + v[1] + v[2] + v[3];
  }
  if (s == 12345.f) out[0] = s;
}

__global__ void k_fill_idx(uint32_t* idx, uint64_t n, uint32_t mask) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    idx[i] = hash32((uint32_t)i * 0x9E3779B9u + 7u) & mask;
}

__global__ void k_pols(uint64_t* p) {
  uint64_t a, b;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(a) : "f"(1.0f));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, %1;" : "=l"(b) : "f"(1.0f));
  p[0] = a;
  p[1] = b;
}

int main() {
  const uint64_t maxn = 1ull << 29;  // 2 GB of floats
  float *a, *o;
  uint32_t* idx;
  uint64_t* pols;
  const uint64_t nidx = 1ull << 30;  // 4 GB index stream (1 G gathers)
  cudaMalloc(&a, maxn * 4);
  cudaMalloc(&o, 4);
  cudaMalloc(&idx, nidx * 4);
  cudaMalloc(&pols, 16);
  cudaMemset(a, 0, maxn * 4);
  k_pols<<<1, 1>>>(pols);
  uint64_t hp[2];
  cudaMemcpy(hp, pols, 16, cudaMemcpyDeviceToHost);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 148 * 8, threads = 256;
  const uint32_t per = 1024;
  const double loads = (double)blocks * threads * per;
  printf("# region_MB  hash_U4_Gloads/s  hash_U8_Gloads/s  stream+gather_Ggathers/s\n");
  for (int lg = 22; lg <= 31; ++lg) {  // region = 2^lg bytes: 4 MB .. 2 GB
    const uint32_t mask = (uint32_t)((1ull << (lg - 2)) - 1);
    float r[3];
    for (int m = 0; m < 3; ++m) {
      if (m == 2) {
        k_fill_idx<<<4096, 256>>>(idx, nidx, mask);
        cudaDeviceSynchronize();
      }
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (m == 0) k_hash<4><<<blocks, threads>>>(a, mask, per, o, hp[0]);
        else if (m == 1) k_hash<8><<<blocks, threads>>>(a, mask, per, o, hp[0]);
        else k_stream<<<blocks, threads>>>(a, idx, nidx, o, hp[0], hp[1]);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      r[m] = (m == 2 ? (double)nidx : loads) / (ms * 1e-3) / 1e9;
    }
    printf("%8.0f %12.1f %12.1f %12.1f\n", (double)(1ull << lg) / (1 << 20), r[0], r[1], r[2]);
  }
  return 0;
}
