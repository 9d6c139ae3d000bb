// Random-reduction throughput probe: RED.ADD.F64 / RED.ADD.F32 / RED.ADD.U32 /
// RED.MIN.U32 to uniformly random addresses of a region (and to a skewed
// distribution: index = hash^3 scaled, most hits near 0, like hub targets).
// G ops/s per op and region.  Measurement tool, not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull; x ^= x >> 31;
  return x;
}
__device__ __forceinline__ uint64_t pick(uint64_t h, uint64_t n, bool skew) {
  if (!skew) return h % n;
  const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
  return (uint64_t)(u * u * u * u * (double)n);  // density ~ x^(-3/4): hub-heavy
}
template <int OP>
__global__ void k_red(void* a, uint64_t n, uint64_t per, bool skew) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (uint64_t i = 0; i < per; ++i) {
    const uint64_t idx = pick(mix64(t * 0x9E3779B97F4A7C15ull + i), n, skew);
    if (OP == 0) atomicAdd((double*)a + idx, 1.0);
    else if (OP == 1) atomicAdd((float*)a + idx, 1.0f);
    else if (OP == 2) atomicAdd((unsigned*)a + idx, 1u);
    else atomicMin((unsigned*)a + idx, (unsigned)i);
  }
}
int main() {
  void* a; cudaMalloc(&a, 1ull << 31); cudaMemset(a, 0, 1ull << 31);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 8, threads = 256; const uint64_t per = 256;
  const double ops = (double)blocks * threads * per;
  const char* names[] = {"red.add.f64", "red.add.f32", "red.add.u32", "red.min.u32"};
  const uint64_t mbs[] = {8, 64, 1024};
  printf("# op  region_MB  uniform_Gops  skewed_Gops\n");
  for (int op = 0; op < 4; ++op)
    for (uint64_t mb : mbs) {
      const uint64_t n = mb * (1 << 20) / (op == 0 ? 8 : 4);
      float r[2];
      for (int sk = 0; sk < 2; ++sk) {
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0);
          if (op == 0) k_red<0><<<blocks, threads>>>(a, n, per, sk);
          else if (op == 1) k_red<1><<<blocks, threads>>>(a, n, per, sk);
          else if (op == 2) k_red<2><<<blocks, threads>>>(a, n, per, sk);
          else k_red<3><<<blocks, threads>>>(a, n, per, sk);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        r[sk] = ops / (ms * 1e-3) / 1e9;
      }
      printf("%s %6llu %8.1f %8.1f\n", names[op], (unsigned long long)mb, r[0], r[1]);
    }
  return 0;
}
