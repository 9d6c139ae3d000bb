// HBM home-die probe (round 2).  Question: does a DRAM miss cost more when the
// line's memory sits on the other die than the SM that loads it, and at what
// address granularity do lines alternate between the dies' HBM stacks?  If the
// home of a line is learnable, a gather kernel can send each source's loads
// from SMs of its home die (PageRank die split by home instead of a hash).
//  1. SM -> die map as in die_probe.cu (pointer chase after an L2 flush).
//  2. For address sets (consecutive 128 B lines; 4 KB stride; 2 MB stride) of a
//     1 GB buffer: after an L2 flush, one thread on SM a (die 0) loads each
//     address once (ld.global.cg, dependent chain) and times every load; then
//     the same from SM b (die 1).  Lines homed near a are fast from a and slow
//     from b, and the reverse.
// Measurement tool, not product code.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long clk() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
  return t;
}

__global__ void k_chase(const uint32_t* chain, uint32_t start, int steps, uint32_t who,
                        unsigned long long* out_cycles, uint32_t* sink) {
  extern __shared__ uint8_t pad[];
  if (threadIdx.x != 0 || smid() != who) return;
  uint32_t i = start;
  const long long t0 = clock64();
  for (int k = 0; k < steps; ++k) i = ld_cg(chain + (size_t)i * 32);
  const long long t1 = clock64();
  out_cycles[0] = (unsigned long long)(t1 - t0);
  sink[0] = i + pad[0];
}

__global__ void k_flush(uint32_t* buf, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) buf[i] += 1;
}

// one CTA per SM; the CTA on SM `who` times, for each of n pages, a dependent
// chain of kL first-touch loads to distinct 128 B lines of that 4 KB page
// (cycles per load; a single clock pair per chain, so scheduling skew of the
// clock reads is amortized over kL loads)
constexpr int kL = 8;
__global__ void k_lat(const uint32_t* buf, const uint64_t* pages, int n, uint32_t who,
                      uint32_t* lat, uint32_t* sink) {
  extern __shared__ uint64_t s_pg[];  // page offsets staged in shared memory
  if (threadIdx.x != 0 || smid() != who) return;
  for (int k = 0; k < n; ++k) s_pg[k] = pages[k];
  uint32_t v = 0;
  for (int k = 0; k < n; ++k) {
    const uint32_t* p = buf + s_pg[k] * 1024;  // 4 KB page = 1024 words
    const long long t0 = clk();
#pragma unroll
    for (int j = 0; j < kL; ++j) v = ld_cg(p + ((j * 5 + 3) % 32) * 32 + v);
    s_pg[k] = v;  // consume the chain's last value before the second clock read
    const long long t1 = clk();
    lat[k] = (uint32_t)((t1 - t0) / kL);
  }
  sink[0] = v;
}

static void ck(cudaError_t e, const char* w) {
  if (e != cudaSuccess) {
    std::fprintf(stderr, "%s: %s\n", w, cudaGetErrorString(e));
    std::exit(1);
  }
}

int main() {
  int nsm = 0;
  ck(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0), "attr");
  const size_t smem = 160 * 1024;  // one CTA per SM
  ck(cudaFuncSetAttribute(k_chase, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "a1");
  ck(cudaFuncSetAttribute(k_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "a2");
  const size_t flushN = (512ull << 20) / 4;
  uint32_t *flush, *chain, *sink, *buf, *lat;
  unsigned long long* cyc;
  uint64_t* offs;
  ck(cudaMalloc(&flush, flushN * 4), "m");
  const uint32_t links = (2u << 20) / 128;
  ck(cudaMalloc(&chain, (size_t)links * 128), "m");
  ck(cudaMalloc(&sink, 64), "m");
  ck(cudaMalloc(&cyc, 64), "m");
  const size_t bufN = (1ull << 30) / 4;
  ck(cudaMalloc(&buf, bufN * 4), "m");
  ck(cudaMemset(buf, 0, bufN * 4), "ms");
  const int maxn = 8192;
  ck(cudaMalloc(&offs, maxn * 8), "m");
  ck(cudaMalloc(&lat, maxn * 4), "m");
  {  // random single cycle over the 2 MB chain
    std::vector<uint32_t> perm(links), h((size_t)links * 32, 0);
    for (uint32_t i = 0; i < links; ++i) perm[i] = i;
    uint64_t s = 12345;
    for (uint32_t i = links - 1; i > 0; --i) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      std::swap(perm[i], perm[(s >> 33) % (i + 1)]);
    }
    for (uint32_t i = 0; i < links; ++i) h[(size_t)perm[i] * 32] = perm[(i + 1) % links];
    ck(cudaMemcpy(chain, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "cp");
  }
  auto flushL2 = [&] { k_flush<<<nsm * 4, 512>>>(flush, flushN); };
  // 1. die map relative to SM 0
  std::vector<double> cpl(nsm);
  for (int s = 0; s < nsm; ++s) {
    flushL2();
    k_chase<<<nsm, 32, smem>>>(chain, 0, links, 0, cyc, sink);
    k_chase<<<nsm, 32, smem>>>(chain, 0, links, (uint32_t)s, cyc, sink);
    ck(cudaDeviceSynchronize(), "chase");
    unsigned long long c = 0;
    ck(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost), "c");
    cpl[s] = (double)c / links;
  }
  std::vector<double> srt = cpl;
  std::sort(srt.begin(), srt.end());
  const double mid = 0.5 * (srt.front() + srt.back());
  int a = 0, b = -1;
  for (int s = 0; s < nsm; ++s)
    if (cpl[s] > mid) { b = s; break; }
  std::printf("# die map: SM 0 near %.0f cycles, far %.0f; SM a=%d (die of SM 0), SM b=%d (other die)\n",
              srt.front(), srt.back(), a, b);
  if (b < 0) return 1;
  // 2. per-page latency from SM a and SM b: (A) the first 16384 4 KB pages (64 MB)
  //    of buffer 1; (B) the same of a second 1 GB buffer; (C) every 512th page
  //    (2 MB stride) over buffer 1's 1 GB
  uint32_t* buf2;
  ck(cudaMalloc(&buf2, bufN * 4), "m");
  ck(cudaMemset(buf2, 0, bufN * 4), "ms");
  struct Set { const char* name; const uint32_t* base; uint64_t page_stride; int n; };
  const Set sets[] = {{"buf1_pages", buf, 1, 16384}, {"buf2_pages", buf2, 1, 16384},
                      {"buf1_2MB", buf, 512, 512}};
  std::printf("# buf1 %p buf2 %p\n", (void*)buf, (void*)buf2);
  ck(cudaFuncSetAttribute(k_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8), "a3");
  ck(cudaFree(offs), "f");
  ck(cudaMalloc(&offs, 16384 * 8), "m");
  ck(cudaFree(lat), "f");
  ck(cudaMalloc(&lat, 16384 * 4), "m");
  for (const Set& st : sets) {
    std::vector<uint64_t> h(st.n);
    for (int k = 0; k < st.n; ++k) h[k] = (uint64_t)k * st.page_stride;
    std::vector<uint32_t> la(st.n), lb(st.n);
    for (int who : {a, b}) {
      for (int c0 = 0; c0 < st.n; c0 += 2048) {  // chunks: every chain starts after a flush-free
        const int c = std::min(2048, st.n - c0);  // run of first touches (one flush per chunk)
        ck(cudaMemcpy(offs, h.data() + c0, c * 8, cudaMemcpyHostToDevice), "cp");
        flushL2();
        k_lat<<<nsm, 32, 16384 * 8>>>(st.base, offs, c, (uint32_t)who, lat, sink);
        ck(cudaDeviceSynchronize(), "lat");
        ck(cudaMemcpy((who == a ? la.data() : lb.data()) + c0, lat, c * 4, cudaMemcpyDeviceToHost), "c");
      }
    }
    std::printf("== set %s (page stride %llu x 4 KB, n %d): k lat_a lat_b\n", st.name,
                (unsigned long long)st.page_stride, st.n);
    for (int k = 0; k < st.n; ++k) std::printf("%d %u %u\n", k, la[k], lb[k]);
  }
  return 0;
}
