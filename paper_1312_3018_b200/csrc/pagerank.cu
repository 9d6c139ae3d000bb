// pagerank.cu -- pull PageRank over BSP rounds (Fig. 14;
// readings A1-A8 in DESIGN.md).  Iteration t on partition p, everything in
// local-id order (out-degree order: the gathered side of a pull is the source,
// so the hottest contributions -- the hubs -- are a compact prefix):
//   pull    : sum_e contrib[in_col[e]] over the row's in-edges from LOCAL
//             sources, accumulated in fp64 (contrib = rank/outdeg stored fp32,
//             the paper's 4-byte rank).  Rows [Vp, Vp+S) are outbox
//             slots: their sums are this partition's source-reduced partial
//             sums for remote vertices ("the 'rank' sum in PageRank").
//             Three row classes by in-degree: a CTA per row (>= 2048), a warp
//             per row (32..2047, from build-time row lists), a thread per row.
//   P == 1  : fused finalize: rank = (1-d)/V + d*sum, next contrib = rank/outdeg.
//   P > 1   : outbox partial sums -> owners' inboxes (full buffer),
//             scatter-add into acc, then finalize.  Fused (default): the pull
//             kernel stores each outbox row's sum straight into the owner's
//             inbox slot (RemoteOut; NVLink peer stores across processes),
//             double-buffered by round parity, so the communication phase is
//             one arrival barrier per round and no copy.
// No vote: a fixed number of rounds.
#include <cstdlib>

#include "frontier.cuh"

namespace tg {

namespace {

constexpr unsigned kCtaThreads = 256;

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// sum of contrib[in_col[i]] for i = i0, i0+step, ... < e; four independent
// column loads then four independent gathers per iteration (memory-level
// parallelism for the dependent load chain), fp64 accumulation.
// Sources are in out-degree order, so ids below `hot` are the hubs that most
// in-edges gather from: they are loaded evict_last; the cold tail and the
// streamed in_col are evict_first, so they do not push the hub lines out of L2.
// L1 placement (kL1, TG_PR_L1 A/B): 0 = L1 default for everything (L2 hints
// only); 1 = the streamed in_col bypasses L1 (L1::no_allocate); 2 = 1 + cold
// gathers (c >= hot) bypass L1 too, so L1 keeps hub contributions; 3 = 2 +
// the hottest sources (c < l1hot) are L1::evict_last.
template <int kL1>
__device__ __forceinline__ float gather_one(const float* __restrict__ contrib, uint32_t c,
                                            uint32_t hot, uint64_t keep, uint64_t stream,
                                            uint32_t l1hot) {
  if constexpr (kL1 >= 2) {
    if (c >= hot) return ld_f32_cold(contrib + c, stream);
    if constexpr (kL1 >= 3) {
      if (c < l1hot) return ld_f32_hot(contrib + c, keep);
    }
    return ld_f32_hint(contrib + c, keep);
  } else {
    return ld_f32_hint(contrib + c, c < hot ? keep : stream);
  }
}

template <int kL1>
__device__ __forceinline__ double gather_sum(const uint32_t* __restrict__ in_col,
                                             const float* __restrict__ contrib, uint64_t i,
                                             uint64_t e, uint32_t step, uint32_t hot,
                                             uint32_t l1hot) {
  const uint64_t keep = l2_evict_last(), stream = l2_evict_first();
  auto col = [&](uint64_t j) {
    if constexpr (kL1 >= 1) return ld_u32_stream(in_col + j, stream);
    else return ld_u32_hint(in_col + j, stream);
  };
  auto gather_one = [&](const float* __restrict__ cb, uint32_t c, uint32_t h, uint64_t k,
                        uint64_t st) { return tg::gather_one<kL1>(cb, c, h, k, st, l1hot); };
  double s0 = 0.0, s1 = 0.0;
  for (; i + 3ull * step < e; i += 4ull * step) {
    const uint32_t c0 = col(i), c1 = col(i + step);
    const uint32_t c2 = col(i + 2ull * step);
    const uint32_t c3 = col(i + 3ull * step);
    const float f0 = gather_one(contrib, c0, hot, keep, stream);
    const float f1 = gather_one(contrib, c1, hot, keep, stream);
    const float f2 = gather_one(contrib, c2, hot, keep, stream);
    const float f3 = gather_one(contrib, c3, hot, keep, stream);
    s0 += (double)f0 + (double)f1;
    s1 += (double)f2 + (double)f3;
  }
  for (; i < e; i += step)
    s0 += (double)gather_one(contrib, col(i), hot, keep, stream);
  return s0 + s1;
}

struct PullOut {
  bool fused;
  uint64_t Vp;
  double base, d;
  double* acc;             // !fused: local rows
  double* obox;            // outbox partial sums (row Vp + slot)
  float* rank;             // fused
  float* contrib_next;     // fused
  const uint32_t* outdeg;  // fused
  uint32_t hot;            // sources [0, hot) are gathered evict_last
  uint32_t l1hot;          // kL1 3: sources [0, l1hot) L1::evict_last
  RemoteOut rout;          // remote: outbox sums go straight into the owner's inbox ...
  bool remote;
  int parity;              // ... double-buffered by round parity (arena slot = 2 x f64)
  __device__ __forceinline__ void put(uint64_t r, double sum) const {
    if (r < Vp) {
      if (fused) {
        const double rk = base + d * sum;
        const uint64_t stream = l2_evict_first();
        st_f32_hint(rank + r, (float)rk, stream);
        const uint32_t od = outdeg[r];
        // next round's contributions: hubs stay evict_last like their gathers
        st_f32_hint(contrib_next + r, od ? (float)(rk / (double)od) : 0.0f,
                    r < hot ? l2_evict_last() : stream);
      } else {
        acc[r] = sum;
      }
    } else if (remote) {
      reinterpret_cast<double*>(rout.slot<double2>((uint32_t)(r - Vp)))[parity] = sum;
    } else {
      obox[r - Vp] = sum;
    }
  }
};

// one CTA per listed row (in-degree >= kPrCta)
template <int kL1>
__global__ void __launch_bounds__(kCtaThreads) k_pull_cta(const uint64_t* in_off,
                                                          const uint32_t* in_col,
                                                          const float* contrib,
                                                          const uint32_t* rows, PullOut o) {
  __shared__ double s_part[kCtaThreads / 32];
  const uint64_t r = rows[blockIdx.x];
  const uint64_t b = in_off[r], e = in_off[r + 1];
  double sum = gather_sum<kL1>(in_col, contrib, b + threadIdx.x, e, kCtaThreads, o.hot, o.l1hot);
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kCtaThreads / 32 ? s_part[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) o.put(r, v);
  }
}

// one warp per listed row (32 <= in-degree < kPrCta)
template <int kL1>
__global__ void __launch_bounds__(256) k_pull_warp(const uint64_t* in_off, const uint32_t* in_col,
                                                   const float* contrib, const uint32_t* rows,
                                                   uint64_t n, PullOut o) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t k = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; k < n; k += nwarps) {
    const uint64_t r = rows[k];
    const uint64_t b = in_off[r], e = in_off[r + 1];
    double sum = gather_sum<kL1>(in_col, contrib, b + lane, e, 32, o.hot, o.l1hot);
    sum = warp_sum(sum);
    if (lane == 0) o.put(r, sum);
  }
}

// one thread per row of [r0, r1) with in-degree < 32 (incl. 0); others skipped
template <int kL1>
__global__ void __launch_bounds__(256) k_pull_thread(const uint64_t* in_off, const uint32_t* in_col,
                                                     const float* contrib, uint64_t r0, uint64_t r1,
                                                     PullOut o) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = r0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < r1; r += stride) {
    const uint64_t b = in_off[r], e = in_off[r + 1];
    if (e - b >= 32) continue;
    o.put(r, gather_sum<kL1>(in_col, contrib, b, e, 1, o.hot, o.l1hot));
  }
}

// rows with in-degree < 32, a warp per 32 consecutive rows (TG_PR_SEG=1): the
// warp walks the rows' concatenated in-edges 32 at a time (in_col reads
// coalesced, where a thread per row makes 32 lanes read 32 separate rows) and
// sums each row's contributions with a segmented shuffle scan (fp64), the
// row's lane collecting its segment's partial at the end of every 32-edge chunk.
// Rows of in-degree >= 32 are left to the CTA / warp classes.
__global__ void __launch_bounds__(256) k_pull_seg(const uint64_t* in_off, const uint32_t* in_col,
                                                  const float* contrib, uint64_t R, PullOut o) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lowm = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t keep = l2_evict_last(), stream = l2_evict_first();
  for (uint64_t r0 = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * 32; r0 < R;
       r0 += nwarps * 32) {
    const uint64_t r = r0 + lane;
    uint64_t b = 0, e = 0;
    if (r < R) {
      b = in_off[r];
      e = in_off[r + 1];
    }
    const bool mine = r < R && e - b < 32;
    const uint32_t len = mine ? (uint32_t)(e - b) : 0u;
    uint32_t incl = len;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, k);
      if (lane >= (uint32_t)k) incl += y;
    }
    const uint32_t T = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = incl - len;
    const uint64_t basev = b - excl;  // in_col index of flattened position i of my row = basev + i
    const uint32_t lmask = __ballot_sync(0xffffffffu, len > 0);
    const uint32_t owner_of = __fns(lmask, 0, (int)lane + 1);  // lane of non-empty row #lane
    double acc = 0.0;
    uint32_t s0 = 0;
    for (uint32_t c0 = 0; c0 < T; c0 += 32) {
      const uint32_t flag = (len > 0 && excl > c0 && excl < c0 + 32) ? (1u << (excl - c0)) : 0u;
      const uint32_t starts = __reduce_or_sync(0xffffffffu, flag);
      const uint32_t s = s0 + __popc(starts & lowm);
      const uint32_t idx = c0 + lane;
      const uint32_t ow = __shfl_sync(0xffffffffu, owner_of, s & 31);
      const uint64_t bs = __shfl_sync(0xffffffffu, basev, ow & 31);
      double val = 0.0;
      if (idx < T) {
        const uint32_t c = ld_u32_hint(in_col + bs + idx, stream);
        val = (double)ld_f32_hint(contrib + c, c < o.hot ? keep : stream);
      }
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {
        const double vo = __shfl_up_sync(0xffffffffu, val, k);
        const uint32_t so = __shfl_up_sync(0xffffffffu, s, k);
        if (lane >= (uint32_t)k && so == s) val += vo;
      }
      int tail = -1;
      if (len > 0) {
        const uint32_t st = excl > c0 ? excl : c0;
        const uint32_t en = (excl + len) < (c0 + 32) ? (excl + len) : (c0 + 32);
        if (st < en) tail = (int)(en - 1 - c0);
      }
      const double got = __shfl_sync(0xffffffffu, val, tail < 0 ? 0 : tail);
      if (tail >= 0) acc += got;
      const uint32_t sl = __shfl_sync(0xffffffffu, s, 31);
      const uint32_t nb = __reduce_or_sync(0xffffffffu, (len > 0 && excl == c0 + 32) ? 1u : 0u);
      s0 = sl + nb;
    }
    if (mine) o.put(r, acc);
  }
}

__global__ void k_pr_init(const uint32_t* outdeg, uint64_t Vp, double r0, float* contrib, float* rank) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < Vp; i += stride) {
    const uint32_t od = outdeg[i];
    contrib[i] = od ? (float)(r0 / (double)od) : 0.0f;
    rank[i] = (float)r0;
  }
}

// msg[j * stride] is inbox entry j (stride 2 for the fused double buffer)
__global__ void k_pr_scatter(const double* msg, uint32_t mstride, const uint32_t* lid, uint64_t I,
                             double* acc) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < I; j += stride) {
    const uint32_t r = lid[j];
    if (r != kInf) atomicAdd(&acc[r], msg[j * mstride]);
  }
}

__global__ void k_pr_finalize(const double* acc, const uint32_t* outdeg, uint64_t Vp, double base,
                              double d, float* rank, float* contrib_next) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < Vp; i += stride) {
    const double rk = base + d * acc[i];
    rank[i] = (float)rk;
    const uint32_t od = outdeg[i];
    contrib_next[i] = od ? (float)(rk / (double)od) : 0.0f;
  }
}

// The three row classes touch disjoint rows and read only the previous
// round's contributions, so with `concurrent` they run on fork/join side
// streams: the long hub rows of k_pull_cta overlap the other classes instead
// of leaving the GPU to their tail.
// the in-CSR a pull walks: the push layout (rows [0, Vp + S)) or the
// ghost-pull layout (rows [0, Vp), ghost sources at Vp + g)
struct PullCsr {
  const uint64_t* off;
  const uint32_t* col;
  const uint32_t* cta;
  uint64_t n_cta;
  const uint32_t* warp;
  uint64_t n_warp;
  uint64_t R;
};
PullCsr push_csr(const Part& p) {
  return {p.in_off.get(), p.in_col.get(), p.pr_cta.get(), p.n_cta, p.pr_warp.get(), p.n_warp,
          p.Vp + p.S};
}
PullCsr ghost_csr(const Part& p) {
  const PRGhost& g = p.gh;
  return {g.off.get(), g.col.get(), g.cta.get(), g.n_cta, g.warp.get(), g.n_warp, p.Vp};
}

// ghost-pull: p's published contributions -> q's ghost slots (Vq + gh_off[p] + k)
__global__ void k_publish(const uint32_t* lid, uint64_t n, const float* src, float* dst) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += stride)
    dst[k] = src[lid[k]];
}

// one barrier per round across processes: the peers' ghost slots of buffer
// `buf` were last read by their pull two rounds ago, which precedes their
// previous publish and that round's barrier
void publish(Engine& eng, int buf) {
  for (auto& pp : eng.parts) {
    Part& p = *pp;
    for (int q = 0; q < eng.P; ++q) {
      const uint64_t n = q == p.id ? 0 : p.gh.pub_off[q + 1] - p.gh.pub_off[q];
      if (!n) continue;
      k_publish<<<grid_for(n, 256), 256, 0, eng.stream>>>(p.gh.pub_lid.get() + p.gh.pub_off[q], n,
                                                           p.pr.contrib[buf].get(),
                                                           p.gh.pub_dst[buf][q]);
      eng.launches++;
      eng.comm_bytes += n * sizeof(float);
    }
  }
  TG_CK(cudaGetLastError());
  fused_arrival(eng);  // processes: published values land before any pull reads them
}

template <int kL1>
void launch_pull_l1(Engine& eng, const PullCsr& c, const float* contrib, const PullOut& o,
                    bool concurrent) {
  cudaStream_t s = eng.stream, s_cta = s, s_warp = s;
  if (concurrent) {
    eng.fork();
    s_cta = eng.side[0];
    s_warp = eng.side[1];
  }
  const uint64_t R = c.R;
  if (c.n_cta) {
    k_pull_cta<kL1><<<(unsigned)c.n_cta, kCtaThreads, 0, s_cta>>>(c.off, c.col, contrib, c.cta, o);
    eng.launches++;
  }
  if (c.n_warp) {
    k_pull_warp<kL1><<<grid_for(c.n_warp * 32, 256, 148u * 16u), 256, 0, s_warp>>>(
        c.off, c.col, contrib, c.warp, c.n_warp, o);
    eng.launches++;
  }
  if (R) {
    const char* seg = std::getenv("TG_PR_SEG");
    if (seg && seg[0] == '1')
      k_pull_seg<<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, R, o);
    else
      k_pull_thread<kL1><<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, 0, R, o);
    eng.launches++;
  }
  if (concurrent) eng.join();
  TG_CK(cudaGetLastError());
}

void launch_pull(Engine& eng, const PullCsr& c, const float* contrib, const PullOut& o,
                 bool concurrent, int l1) {
  switch (l1) {
    case 1: launch_pull_l1<1>(eng, c, contrib, o, concurrent); break;
    case 2: launch_pull_l1<2>(eng, c, contrib, o, concurrent); break;
    case 3: launch_pull_l1<3>(eng, c, contrib, o, concurrent); break;
    default: launch_pull_l1<0>(eng, c, contrib, o, concurrent);
  }
}

void* send_obox(Part& p) { return p.pr.obox.get(); }
void* recv_ibox(Part& p) { return p.arena_fwd.get(); }

}  // namespace

void run_pagerank(Engine& eng, int iters, double d, float* out, int mem, tg_stats* st) {
  TG_REQUIRE(iters >= 1, TG_EINVAL, "tg_pagerank: iterations must be >= 1");
  TG_REQUIRE(eng.has_in, TG_EINVAL, "tg_pagerank: engine built without the in-CSR");
  TG_REQUIRE(out != nullptr || (eng.multi() && eng.rank != 0), TG_EINVAL,
             "tg_pagerank: NULL output");
  cudaStream_t s = eng.stream;
  // ghost-pull (TG_PR_PULL, single process, P > 1): outside the timed region
  const bool ghost = eng.pr_comm == TG_PR_PULL && eng.P > 1;
  if (ghost) build_pr_ghost(eng);
  for (auto& pp : eng.parts) {
    Part& p = *pp;
    PRState& r = p.pr;
    const uint64_t Vn = std::max<uint64_t>(p.Vp, 1);
    const uint64_t Cn = std::max<uint64_t>(p.Vp + (ghost ? p.gh.G : 0), 1);  // + ghost slots
    if (r.contrib[0].n < Cn) {
      r.contrib[0].alloc(Cn);
      r.contrib[1].alloc(Cn);
    }
    if (r.rank.n < Vn) {
      r.rank.alloc(Vn);
      if (eng.P > 1) {
        r.acc.alloc(Vn);
        r.obox.alloc(std::max<uint64_t>(p.S, 1));
      }
    }
  }
  eng.launches = 0;
  eng.comm_bytes = 0;
  const double base = (1.0 - d) / (double)eng.V, r0 = 1.0 / (double)eng.V;
  // hub prefix kept in L2 (evict_last): default 16M sources = 64 MB of fp32
  // contributions, half of the 126 MB L2 (TG_PR_HOT overrides; RMAT-28 sweep
  // in profiles/r01_pr_hot_sweep.txt: 0 -> 28.2, 16M -> 20.35, all -> 21.0 ms)
  uint32_t hot = 16u << 20;
  if (const char* h = std::getenv("TG_PR_HOT")) hot = (uint32_t)std::strtoul(h, nullptr, 10);
  // L1 placement variant (gather_one) and its L1-hot prefix (TG_PR_L1, TG_PR_L1HOT)
  int l1 = 0;
  if (const char* v = std::getenv("TG_PR_L1")) l1 = std::atoi(v);
  uint32_t l1hot = 32768;
  if (const char* v = std::getenv("TG_PR_L1HOT")) l1hot = (uint32_t)std::strtoul(v, nullptr, 10);
  // row classes on fork/join streams (TG_PR_CONCURRENT=0: one stream)
  const bool concurrent =
      !(std::getenv("TG_PR_CONCURRENT") && std::getenv("TG_PR_CONCURRENT")[0] == '0');
  time_begin(eng);
  for (auto& pp : eng.parts) {
    Part& p = *pp;
    if (!p.Vp) continue;
    k_pr_init<<<grid_for(p.Vp, 256), 256, 0, s>>>(p.outdeg.get(), p.Vp, r0, p.pr.contrib[0].get(),
                                                  p.pr.rank.get());
    eng.launches++;
  }
  if (ghost) publish(eng, 0);
  int cur = 0;
  for (int it = 0; it < iters; ++it) {
    eng.prof_begin(TG_K_PR_PULL);
    for (auto& pp : eng.parts) {
      Part& p = *pp;
      PRState& r = p.pr;
      // P == 1 and ghost-pull: every in-edge is in the row, finalize in the pull
      PullOut o{eng.P == 1 || ghost, p.Vp, base, d, r.acc.get(), r.obox.get(), r.rank.get(),
                r.contrib[cur ^ 1].get(), p.outdeg.get(), hot, l1hot, p.rout(), eng.fused, it & 1};
      if (eng.P == 1) eng.l2_window(r.contrib[cur].get(), p.Vp * sizeof(float));  // opt-in
      launch_pull(eng, ghost ? ghost_csr(p) : push_csr(p), r.contrib[cur].get(), o, concurrent, l1);
    }
    eng.prof_end(TG_K_PR_PULL);
    if (ghost) {  // communication: contributions of boundary sources -> peers' ghosts
      eng.prof_begin(TG_K_EXCHANGE);
      if (it + 1 < iters) publish(eng, cur ^ 1);
      eng.prof_end(TG_K_EXCHANGE);
    }
    // pull: in_col 4 + contrib gather 4 per edge; in_off 8 + outdeg 4 + rank 4 +
    // next contrib 4 per row
    eng.prof_bytes(TG_K_PR_PULL, 8.0 * eng.E + 20.0 * eng.V);
    if (eng.P > 1 && !ghost) {
      eng.prof_begin(TG_K_EXCHANGE);
      // fused: the pull wrote this round's sums into the owners' arenas (buffer
      // it & 1); one barrier per round orders them before the scatters, and the
      // next round writes the other buffer, whose readers finished before that
      // barrier (their scatter precedes their pull in stream order)
      if (eng.fused) {
        fused_arrival(eng);
        for (auto& pp : eng.parts) eng.comm_bytes += pp->S * 8;
      } else {
        exchange(eng, send_obox, recv_ibox, 8, false);
      }
      for (auto& pp : eng.parts) {
        Part& p = *pp;
        PRState& r = p.pr;
        if (p.I) {
          const double* msg = reinterpret_cast<const double*>(p.arena_fwd.get());
          k_pr_scatter<<<grid_for(p.I, 256), 256, 0, s>>>(eng.fused ? msg + (it & 1) : msg,
                                                          eng.fused ? 2u : 1u, p.ibox_lid.get(),
                                                          p.I, r.acc.get());
          eng.launches++;
        }
        if (p.Vp) {
          k_pr_finalize<<<grid_for(p.Vp, 256), 256, 0, s>>>(r.acc.get(), p.outdeg.get(), p.Vp, base,
                                                            d, r.rank.get(),
                                                            r.contrib[cur ^ 1].get());
          eng.launches++;
        }
        TG_CK(cudaGetLastError());
      }
      eng.prof_end(TG_K_EXCHANGE);
    }
    cur ^= 1;
  }
  const double ms = time_end(eng);
  eng.l2_window(nullptr, 0);
  if (st) {
    st->device_ms = ms;
    st->supersteps = (uint64_t)iters;
    st->relaxations = eng.E * (uint64_t)iters;
    st->traversed_edges = eng.E * (uint64_t)iters;
    // per iteration: 8 B per edge (in_col + contrib gather) + 20 B per vertex
    // (in_off 8, outdeg 4, rank 4, contrib 4) -- DESIGN.md "Roofline"
    st->algorithmic_bytes = (8 * eng.E + 20 * eng.V) * (uint64_t)iters;
    st->comm_bytes = eng.comm_bytes;
    st->launches = eng.launches;
  }
  collect(eng, [](Part& p) -> const void* { return p.pr.rank.get(); }, sizeof(float), out, mem);
}

}  // namespace tg
