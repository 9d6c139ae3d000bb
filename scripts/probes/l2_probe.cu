// L2 effective-capacity probe for 4-byte random gathers (PageRank's contrib[]
// access pattern).  For a region of X MB, every thread issues random 4-byte
// loads (counter hash) into the region; reports G loads/s.  The knee of the
// curve is the capacity the gather sees.  Measurement tool, not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull; x ^= x >> 31;
  return x;
}
template <int POL>
__global__ void k_gather(const float* __restrict__ a, uint64_t n, uint64_t per_thread, float* out) {
  uint64_t pol;
  if (POL == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(pol) : "f"(1.0f));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, %1;" : "=l"(pol) : "f"(1.0f));
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  float s = 0.f;
  for (uint64_t i = 0; i < per_thread; i += 4) {
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t idx = mix64(t * 0x9E3779B97F4A7C15ull + i + k) % n;
      asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v[k]) : "l"(a + idx), "l"(pol));
    }
    s += v[0] + v[1] + v[2] + v[3];
  }
  if (s == 12345.f) out[0] = s;
}

int main() {
  const uint64_t maxn = (1ull << 30) / 4 * 2;  // 2 GB
  float* a; float* o;
  cudaMalloc(&a, maxn * 4); cudaMalloc(&o, 4);
  cudaMemset(a, 0, maxn * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 8, threads = 256;
  const uint64_t per = 512;
  const double loads = (double)blocks * threads * per;
  int mbs[] = {4, 8, 16, 24, 32, 40, 48, 56, 64, 72, 80, 96, 112, 128, 160, 256, 1024, 2048};
  printf("# region_MB  Gloads/s(evict_normal)  Gloads/s(evict_last)\n");
  for (int mb : mbs) {
    const uint64_t n = (uint64_t)mb * (1 << 20) / 4;
    float r[2];
    for (int pol = 0; pol < 2; ++pol) {
      for (int rep = 0; rep < 2; ++rep) {  // second rep is timed (warm L2)
        cudaEventRecord(e0);
        if (pol) k_gather<1><<<blocks, threads>>>(a, n, per, o);
        else k_gather<0><<<blocks, threads>>>(a, n, per, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      r[pol] = loads / (ms * 1e-3) / 1e9;
    }
    printf("%6d %10.1f %10.1f\n", mb, r[0], r[1]);
  }
  return 0;
}
