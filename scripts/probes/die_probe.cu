// Two-die L2 probe (round 2).  Question: does each die's L2 cache the lines its
// own SMs read (so data read by every SM occupies both halves, ~63 MB usable
// for a shared gather set), or is the 126 MB L2 one cache?
//  1. SM -> die map: after an L2 flush, the SM `ref` pointer-chases a 2 MB
//     region (it now sits in ref's L2); then each SM s in turn chases the same
//     region and times it.  Same-die SMs hit; other-die SMs see a longer latency.
//  2. Gather rate over a 2R MB region: (A) every SM gathers uniformly from the
//     whole region; (B) the SMs of die 0 gather only from the first half and
//     those of die 1 only from the second; (C) split by SM-id parity instead
//     (not die-aligned).  If the L2 halves cache their own SMs' reads, (B) keeps
//     the L2 hit rate of an R MB region while (A) and (C) see 2R MB.
// Measurement tool, not product code.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// one CTA per SM (big dynamic smem); the CTA on SM `who` chases `steps` links
__global__ void k_chase(const uint32_t* chain, uint32_t start, int steps, uint32_t who,
                        unsigned long long* out_cycles, uint32_t* sink) {
  extern __shared__ uint8_t pad[];
  if (threadIdx.x != 0 || smid() != who) return;
  uint32_t i = start;
  const long long t0 = clock64();
  for (int k = 0; k < steps; ++k) i = ld_cg(chain + (size_t)i * 32);  // one 128 B line per link
  const long long t1 = clock64();
  out_cycles[0] = (unsigned long long)(t1 - t0);
  sink[0] = i + pad[0];
}

__global__ void k_flush(uint32_t* buf, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) buf[i] += 1;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// mode 0: whole region; 1: die half (die_of[smid]); 2: smid parity half
__global__ void k_gather(const float* a, uint32_t half_mask, const uint8_t* die_of, int mode,
                         uint32_t per_thread, float* out, uint64_t pol) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t sm = smid();
  uint32_t base = 0, mask = 2 * half_mask + 1;
  if (mode == 1) {
    base = die_of[sm] ? half_mask + 1 : 0;
    mask = half_mask;
  } else if (mode == 2) {
    base = (sm & 1) ? half_mask + 1 : 0;
    mask = half_mask;
  }
  float s = 0.f;
  for (uint32_t i = 0; i < per_thread; i += 4) {
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t idx = base + (hash32(t * 0x9E3779B9u + i + k) & mask);
      asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v[k]) : "l"(a + idx), "l"(pol));
    }
    s += v[0] + v[1] + v[2] + v[3];
  }
  if (s == 12345.f) out[0] = s;
}

__global__ void k_pol(uint64_t* p) {
  uint64_t a;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(a) : "f"(1.0f));
  p[0] = a;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_chase, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // chain: 2 MB = 16384 lines, a random cycle
  const uint32_t L = 16384;
  std::vector<uint32_t> perm(L);
  std::iota(perm.begin(), perm.end(), 0u);
  std::shuffle(perm.begin(), perm.end(), std::mt19937(7));
  std::vector<uint32_t> h((size_t)L * 32, 0);
  for (uint32_t k = 0; k < L; ++k) h[(size_t)perm[k] * 32] = perm[(k + 1) % L];
  uint32_t *chain, *flush, *sink;
  unsigned long long* cyc;
  const size_t nflush = (size_t)1 << 27;  // 512 MB
  cudaMalloc(&chain, h.size() * 4);
  cudaMalloc(&flush, nflush * 4);
  cudaMalloc(&sink, 4);
  cudaMalloc(&cyc, 8);
  cudaMemcpy(chain, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(flush, 0, nflush * 4);
  const int steps = 4096;
  std::vector<double> lat(nsm);
  for (int ref = 0; ref < 2; ++ref) {
    const uint32_t refsm = ref == 0 ? 0 : nsm - 1;
    for (int s = 0; s < nsm; ++s) {
      k_flush<<<nsm * 8, 256>>>(flush, nflush);
      k_chase<<<nsm, 32, smem>>>(chain, perm[0], L, refsm, cyc, sink);  // warm ref's L2
      k_chase<<<nsm, 32, smem>>>(chain, perm[0], steps, (uint32_t)s, cyc, sink);
      unsigned long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      lat[s] = (double)c / steps;
    }
    printf("# ref SM %u: cycles per chased line, by SM id\n", refsm);
    for (int s = 0; s < nsm; ++s) printf("%d:%.0f%c", s, lat[s], (s % 12 == 11) ? '\n' : ' ');
    printf("\n");
  }
  // die map from the last pass (ref = last SM): threshold halfway between min and max
  const double lo = *std::min_element(lat.begin(), lat.end()),
               hi = *std::max_element(lat.begin(), lat.end());
  std::vector<uint8_t> die(nsm);
  int n1 = 0;
  for (int s = 0; s < nsm; ++s) {
    die[s] = lat[s] > (lo + hi) / 2 ? 1 : 0;  // 0 = same die as the last SM
    n1 += die[s];
  }
  printf("# die map: %d SMs with the last SM, %d on the other die (lat %.0f .. %.0f)\n", nsm - n1,
         n1, lo, hi);
  for (int s = 0; s < nsm; ++s) printf("%d", die[s]);
  printf("\n");
  uint8_t* d_die;
  cudaMalloc(&d_die, nsm);
  cudaMemcpy(d_die, die.data(), nsm, cudaMemcpyHostToDevice);
  float *a, *o;
  uint64_t* pol;
  cudaMalloc(&a, (size_t)1 << 30);
  cudaMalloc(&o, 4);
  cudaMalloc(&pol, 8);
  cudaMemset(a, 0, (size_t)1 << 30);
  k_pol<<<1, 1>>>(pol);
  uint64_t hp;
  cudaMemcpy(&hp, pol, 8, cudaMemcpyDeviceToHost);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = nsm * 8, threads = 256;
  const uint32_t per = 2048;
  printf("# halfMB  whole_Gl/s  die_split_Gl/s  parity_split_Gl/s\n");
  for (int lg = 24; lg <= 28; ++lg) {  // half region 16 .. 256 MB of floats... 2^lg bytes
    const uint32_t half_mask = (uint32_t)((1ull << (lg - 2)) - 1);
    double r[3];
    for (int m = 0; m < 3; ++m) {
      float ms = 0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_gather<<<blocks, threads>>>(a, half_mask, d_die, m, per, o, hp);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      r[m] = (double)blocks * threads * per / (ms * 1e-3) / 1e9;
    }
    printf("%8.0f %10.1f %10.1f %10.1f\n", (double)(1ull << lg) / (1 << 20), r[0], r[1], r[2]);
  }
  // also 48 MB halves (96 MB total)
  return 0;
}
