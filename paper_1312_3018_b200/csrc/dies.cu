// dies.cu -- the SM -> die map of a two-die GPU, measured at run time.
//
// B200 is two dies; each die's half of the L2 caches the lines its own SMs
// read (scripts/probes/die_probe.cu, profiles/r02_die_probe.txt).  Which SM
// ids sit on which die depends on the part (yield), so it is measured: after an
// L2 flush the reference SM pointer-chases a small region, pulling it into its
// die's L2; then every SM in turn chases the same region.  SMs of the same die
// hit (~290 cycles per line on B200), the others do not (~480).  Used by the
// PageRank die split (pagerank.cu).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <numeric>
#include <random>

#include "engine.cuh"

namespace tg {

namespace {

__device__ __forceinline__ uint32_t sm_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// one CTA per SM (the dynamic shared memory allows no second one); only the
// CTA on SM `who` chases `steps` links of the chain (one 128-byte line each)
__global__ void k_die_chase(const uint32_t* chain, uint32_t start, int steps, uint32_t who,
                            unsigned long long* cycles, uint32_t* sink) {
  extern __shared__ uint8_t pad[];
  if (threadIdx.x != 0 || sm_id() != who) return;
  uint32_t i = start;
  const long long t0 = clock64();
  for (int k = 0; k < steps; ++k) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(chain + (size_t)i * 32));
    i = v;
  }
  const long long t1 = clock64();
  if (cycles) cycles[who] = (unsigned long long)(t1 - t0);
  sink[0] = i + pad[0];
}

__global__ void k_die_flush(uint32_t* buf, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) buf[i] += 1u;
}

void measure(int device, DieMap& m) {
  int nsm = 0, smem = 0;
  TG_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  TG_CK(cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  m.nsm = nsm;
  if (nsm < 4) return;
  smem -= 1024;  // one CTA per SM
  TG_CK(cudaFuncSetAttribute(k_die_chase, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const uint32_t L = 4096;  // 512 KB chain
  std::vector<uint32_t> perm(L), h((size_t)L * 32, 0u);
  std::iota(perm.begin(), perm.end(), 0u);
  std::shuffle(perm.begin(), perm.end(), std::mt19937(12345));
  for (uint32_t k = 0; k < L; ++k) h[(size_t)perm[k] * 32] = perm[(k + 1) % L];
  const size_t nflush = (size_t)64 << 20;  // 256 MB of u32: twice the L2
  DevBuf<uint32_t> chain(h.size()), flush(nflush), sink(1);
  DevBuf<unsigned long long> cyc(nsm);
  cudaStream_t s;
  TG_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  TG_CK(cudaMemcpyAsync(chain.get(), h.data(), h.size() * 4, cudaMemcpyHostToDevice, s));
  TG_CK(cudaMemsetAsync(flush.get(), 0, nflush * 4, s));
  TG_CK(cudaMemsetAsync(cyc.get(), 0, nsm * 8, s));
  const int steps = 1024;
  const uint32_t ref = 0;
  for (int sm = 0; sm < nsm; ++sm) {
    k_die_flush<<<nsm * 4, 256, 0, s>>>(flush.get(), nflush);
    k_die_chase<<<nsm, 32, smem, s>>>(chain.get(), perm[0], (int)L, ref, nullptr, sink.get());
    k_die_chase<<<nsm, 32, smem, s>>>(chain.get(), perm[0], steps, (uint32_t)sm, cyc.get(),
                                      sink.get());
  }
  TG_CK(cudaGetLastError());
  std::vector<unsigned long long> c(nsm);
  TG_CK(cudaMemcpyAsync(c.data(), cyc.get(), nsm * 8, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaStreamSynchronize(s));
  TG_CK(cudaStreamDestroy(s));
  std::vector<double> lat(nsm);
  const bool dbg = std::getenv("TG_DIE_DEBUG") != nullptr;
  for (int i = 0; i < nsm; ++i) {
    if (dbg) std::fprintf(stderr, "[tg dies] sm %d cycles %llu\n", i, c[i]);
    if (!c[i]) return;  // an SM never ran its probe: no map
    lat[i] = (double)c[i] / steps;
  }
  // cut at the largest gap of the sorted latencies
  std::vector<double> srt(lat);
  std::sort(srt.begin(), srt.end());
  double cut = srt.back() + 1, gap = 0;
  for (int i = 1; i < nsm; ++i)
    if (srt[i] - srt[i - 1] > gap) {
      gap = srt[i] - srt[i - 1];
      cut = 0.5 * (srt[i] + srt[i - 1]);
    }
  m.h_die_of.assign(nsm, 0);
  double s0 = 0, s1 = 0;
  for (int i = 0; i < nsm; ++i) {
    m.h_die_of[i] = lat[i] > cut ? 1 : 0;
    m.n[m.h_die_of[i]]++;
    (m.h_die_of[i] ? s1 : s0) += lat[i];
  }
  if (!m.n[0] || !m.n[1]) return;
  m.lat_near = s0 / m.n[0];
  m.lat_far = s1 / m.n[1];
  // two clear clusters, neither tiny (a one-die part shows one cluster)
  m.ok = m.lat_far > 1.3 * m.lat_near && std::min(m.n[0], m.n[1]) * 5 >= nsm;
  if (dbg)
    std::fprintf(stderr, "[tg dies] n0 %d n1 %d near %.0f far %.0f ok %d\n", m.n[0], m.n[1],
                 m.lat_near, m.lat_far, (int)m.ok);
  if (m.ok) {
    m.die_of.alloc(nsm);
    TG_CK(cudaMemcpy(m.die_of.get(), m.h_die_of.data(), nsm, cudaMemcpyHostToDevice));
  }
}

}  // namespace

const DieMap& die_map(int device) {
  static std::mutex mu;
  static DieMap maps[64];
  static bool done[64] = {};
  std::lock_guard<std::mutex> g(mu);
  TG_REQUIRE(device >= 0 && device < 64, TG_EINVAL, "die_map: device id");
  if (!done[device]) {
    int cur = 0;
    TG_CK(cudaGetDevice(&cur));
    TG_CK(cudaSetDevice(device));
    measure(device, maps[device]);
    TG_CK(cudaSetDevice(cur));
    done[device] = true;
  }
  return maps[device];
}

}  // namespace tg
