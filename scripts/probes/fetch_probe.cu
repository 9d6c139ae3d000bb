// DRAM bytes per random 4-byte miss (round 2, session 3).  gather_flavors.cu
// found that a random 4 B gather that misses L2 moves ~117 B of DRAM (the L2
// misses ~3.75 sectors per load, i.e. fills whole 128 B lines) whatever the
// load flavor.  Which allocation / limit gives sector-sized (32 B) fills?
//   A cudaMalloc (default)
//   B cudaMalloc + cudaLimitMaxL2FetchGranularity = 32
//   C cuMemCreate, compressionType = CU_MEM_ALLOCATION_COMP_NONE
//   D cuMemCreate, compressionType = CU_MEM_ALLOCATION_COMP_GENERIC (if granted)
// Each: random 4 B gathers over 1 GB (U = 8 per thread), G loads/s; run under
// ncu for dram__bytes_read per load.  Measurement tool, not product code.
#include <cuda.h>
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

__global__ void k_gather(const float* __restrict__ a, uint32_t mask, uint32_t per, float* out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  float s = 0.f;
  for (uint32_t i = 0; i < per; i += 8) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(a + (hash32(t * 0x9E3779B9u + i + k) & mask));
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  if (s == 12345.f) out[0] = s;
}

static float run(const float* a, uint32_t mask, float* o) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_gather<<<148 * 8, 256>>>(a, mask, 512, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

static CUdeviceptr vmm_alloc(size_t bytes, unsigned char comp, bool* granted) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  prop.allocFlags.compressionType = comp;
  size_t gran = 0;
  cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  bytes = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  if (cuMemCreate(&h, bytes, &prop, 0) != CUDA_SUCCESS) return 0;
  CUmemAllocationProp got = {};
  cuMemGetAllocationPropertiesFromHandle(&got, h);
  *granted = got.allocFlags.compressionType == comp;
  CUdeviceptr p = 0;
  cuMemAddressReserve(&p, bytes, 0, 0, 0);
  cuMemMap(p, bytes, 0, h, 0);
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cuMemSetAccess(p, bytes, &acc, 1);
  cudaMemset((void*)p, 0, bytes);
  return p;
}

int main() {
  cudaFree(0);
  const size_t bytes = 1ull << 30;
  const uint32_t mask = (uint32_t)(bytes / 4 - 1);
  const double loads = 148.0 * 8 * 256 * 512;
  float *a, *o;
  cudaMalloc(&a, bytes);
  cudaMalloc(&o, 4);
  cudaMemset(a, 0, bytes);
  size_t g = 0;
  cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
  printf("# default MaxL2FetchGranularity %zu\n", g);
  printf("A cudaMalloc                 %.1f G loads/s\n", loads / (run(a, mask, o) * 1e-3) / 1e9);
  cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32);
  cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
  printf("B cudaMalloc + fetch gran %zu  %.1f G loads/s\n", g, loads / (run(a, mask, o) * 1e-3) / 1e9);
  cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 64);
  bool gr = false;
  CUdeviceptr c = vmm_alloc(bytes, CU_MEM_ALLOCATION_COMP_NONE, &gr);
  if (c) printf("C cuMemCreate COMP_NONE (granted %d) %.1f G loads/s\n", gr, loads / (run((const float*)c, mask, o) * 1e-3) / 1e9);
  CUdeviceptr d = vmm_alloc(bytes, CU_MEM_ALLOCATION_COMP_GENERIC, &gr);
  if (d) printf("D cuMemCreate COMP_GENERIC (granted %d) %.1f G loads/s\n", gr, loads / (run((const float*)d, mask, o) * 1e-3) / 1e9);
  int comp = 0;
  cuDeviceGetAttribute(&comp, CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, 0);
  printf("# generic compression supported: %d\n", comp);
  return 0;
}
