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
#include <cstdio>
#include <cstdlib>

#include <cub/cub.cuh>

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
// Shared-memory replica of the hub prefix contrib[0, k) (TG_PR_REP A/B): a
// gather of a source below k is an LDS instead of an L2 request.
struct Rep {
  const float* s;
  uint32_t k;
};

// kL1 == 9: TIMING PROBE ONLY (wrong results): gathers of sources in
// [c_xlo, c_xhi) are skipped, to measure what a source range costs
// (TG_PR_L1=9, TG_PR_XLO / TG_PR_XHI; scripts/sweep_pr.py).
__constant__ uint32_t c_xlo, c_xhi;

template <int kL1, bool kRep = false>
__device__ __forceinline__ float gather_one(const float* __restrict__ contrib, uint32_t c,
                                            uint32_t hot, uint64_t keep, uint64_t stream,
                                            uint32_t l1hot, Rep rep = {nullptr, 0}) {
  if constexpr (kRep) {
    if (c < rep.k) return rep.s[c];
  }
  if constexpr (kL1 == 8) {  // A/B: no L2 policy hints at all
    return __ldg(contrib + c);
  } else if constexpr (kL1 == 9) {
    if (c >= c_xlo && c < c_xhi) return 0.0f;
    return ld_f32_hint(contrib + c, c < hot ? keep : stream);
  } else if constexpr (kL1 >= 2) {
    if (c >= hot) return ld_f32_cold(contrib + c, stream);
    if constexpr (kL1 >= 3) {
      if (c < l1hot) return ld_f32_hot(contrib + c, keep);
    }
    return ld_f32_hint(contrib + c, keep);
  } else {
    return ld_f32_hint(contrib + c, c < hot ? keep : stream);
  }
}

template <int kL1, bool kRep = false>
__device__ __forceinline__ double gather_sum(const uint32_t* __restrict__ in_col,
                                             const float* __restrict__ contrib, uint64_t i,
                                             uint64_t e, uint32_t step, uint32_t hot,
                                             uint32_t l1hot, Rep rep = {nullptr, 0}) {
  const uint64_t keep = l2_evict_last(), stream = l2_evict_first();
  auto col = [&](uint64_t j) {
    if constexpr (kL1 == 8) return __ldg(in_col + j);
    else if constexpr (kL1 >= 1 && kL1 <= 3) return ld_u32_stream(in_col + j, stream);
    else return ld_u32_hint(in_col + j, stream);
  };
  auto gather_one = [&](const float* __restrict__ cb, uint32_t c, uint32_t h, uint64_t k,
                        uint64_t st) { return tg::gather_one<kL1, kRep>(cb, c, h, k, st, l1hot, rep); };
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

// Predicated batches (TG_PR_PRED): U column loads, then U gathers, per lane and
// iteration, every one predicated on the row end -- no remainder loop.  The
// plain gather_sum issues a row's last < 4 x step entries one load at a time
// (a warp-class row of ~214 entries: one 128-entry batch, then three
// serialized 32-entry steps, each a full memory round trip); here a row of up
// to U x step entries is one round trip of column loads and one of gathers.
template <int U>
__device__ __forceinline__ double gather_sum_pred(const uint32_t* __restrict__ in_col,
                                                  const float* __restrict__ contrib, uint64_t i,
                                                  uint64_t e, uint32_t step, uint32_t hot) {
  const uint64_t keep = l2_evict_last(), stream = l2_evict_first();
  double s0 = 0.0, s1 = 0.0;
  for (; i < e; i += (uint64_t)U * step) {
    uint32_t c[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint64_t j = i + (uint64_t)k * step;
      c[k] = j < e ? ld_u32_hint(in_col + j, stream) : kInf;
    }
    float f[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      f[k] = c[k] != kInf ? ld_f32_hint(contrib + c[k], c[k] < hot ? keep : stream) : 0.0f;
#pragma unroll
    for (int k = 0; k < U; k += 2) {
      s0 += (double)f[k];
      if (k + 1 < U) s1 += (double)f[k + 1];
    }
  }
  return s0 + s1;
}

// Lean predicated batches (kP < 0 in the class kernels, TG_PR_PRED negative
// U): the lane's column pointer advances by a compile-time STEP, so the U
// column loads of a batch are one base register + immediate offsets; each
// batch's U contributions are summed in fp32 (U <= 8 terms: relative error
// <= 7 x 2^-24 of the batch) and the batch total accumulated in fp64 (reading
// A7: fp64 accumulation across the row), which replaces U fp32->fp64
// conversions + U DADDs by U FADDs + 1 conversion + 1 DADD.
// kUni (warp / CTA rows, TG_PR_UNIPOL): one L2 policy per warp and batch --
// the load's policy operand is a uniform register, so a per-lane policy costs
// a select + two register moves per gather; a row's entries ascend, so the
// batch is all-hot when its largest column (one REDUX) is below `hot`.
template <int U, int STEP, bool kUni = false>
__device__ __forceinline__ double gather_sum_lean(const uint32_t* __restrict__ in_col,
                                                  const float* __restrict__ contrib, uint64_t i,
                                                  uint64_t e, uint32_t hot) {
  const uint64_t keep = l2_evict_last(), stream = l2_evict_first();
  double s = 0.0;
  const uint32_t* pc = in_col + i;
  for (; i < e; i += (uint64_t)U * STEP, pc += U * STEP) {
    const uint64_t left = e - i;  // > 0
    uint32_t c[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      c[k] = (uint64_t)k * STEP < left ? ld_u32_hint(pc + k * STEP, stream) : kInf;
    float f = 0.0f;
    if constexpr (kUni) {
      uint32_t mx = 0;
#pragma unroll
      for (int k = 0; k < U; ++k) mx = (c[k] != kInf && c[k] > mx) ? c[k] : mx;
      const uint64_t pol = __reduce_max_sync(__activemask(), mx) < hot ? keep : stream;
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (c[k] != kInf) f += ld_f32_hint(contrib + c[k], pol);
    } else {
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (c[k] != kInf) f += ld_f32_hint(contrib + c[k], c[k] < hot ? keep : stream);
    }
    s += (double)f;
  }
  return s;
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
  int npol;                // next contributions of rows < hot: 0 evict_last, 1 normal, 2 evict_first
  const uint32_t* hot_len; // PRCold: row r gathers only its first hot_len[r] in-edges ...
  const float* csum;       // ... and adds the cold partial sum csum[r] (nullptr: off)
  RemoteOut rout;          // remote: outbox sums go straight into the owner's inbox ...
  bool remote;
  int parity;              // ... double-buffered by round parity (arena slot = 2 x f64)
  // fused: rows >= nz_end have out-degree 0 (ids in out-degree order), so no
  // pull ever gathers their contribution: neither outdeg nor the next
  // contribution is touched for them (0: every row writes it)
  uint64_t nz_end = 0;
  // fused: rank is the output only after the last round; earlier rounds keep
  // it in registers for the next contribution (false: no rank store)
  bool rank_out = true;
  // fused, non-final rounds: rows >= rows_end (the sinks, out-degree 0) have
  // neither a rank to store nor a contribution anyone gathers -- they are not
  // pulled at all (0: every row is)
  uint64_t rows_end = 0;
  // fused, last round: no next round gathers a contribution (false: none stored)
  bool contrib_out = true;
  __device__ __forceinline__ uint64_t row_end(uint64_t r, uint64_t b, uint64_t e) const {
    return hot_len ? b + hot_len[r] : e;
  }
  __device__ __forceinline__ void put(uint64_t r, double sum) const {
    if (csum) sum += (double)csum[r];
    if (r < Vp) {
      if (fused) {
        const double rk = base + d * sum;
        const uint64_t stream = l2_evict_first();
        if (rank_out) st_f32_hint(rank + r, (float)rk, stream);
        if ((nz_end && r >= nz_end) || !contrib_out) return;
        const uint32_t od = outdeg[r];
        // next round's contributions: hubs stay evict_last like their gathers
        const float cn = od ? (float)(rk / (double)od) : 0.0f;
        if (npol == 1 && r < hot) contrib_next[r] = cn;
        else st_f32_hint(contrib_next + r, cn, (npol == 0 && r < hot) ? l2_evict_last() : stream);
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
// Hub split (PRHub): hlen / hsum non-null -> the row's first hlen[k] in-edges
// (sources < K) were summed by k_pull_hub into hsum[k]; start after them.
template <int kL1, int kP = 0>
__global__ void __launch_bounds__(kCtaThreads) k_pull_cta(const uint64_t* in_off,
                                                          const uint32_t* in_col,
                                                          const float* contrib,
                                                          const uint32_t* rows, PullOut o,
                                                          const uint32_t* hlen,
                                                          const double* hsum) {
  __shared__ double s_part[kCtaThreads / 32];
  const uint64_t r = rows[blockIdx.x];
  if (o.rows_end && r >= o.rows_end) return;  // a sink in a non-final round
  const uint64_t b0 = in_off[r];
  const uint64_t b = b0 + (hlen ? hlen[blockIdx.x] : 0u), e = o.row_end(r, b0, in_off[r + 1]);
  double sum;
  if constexpr (kP < -100) sum = gather_sum_lean<-kP - 100, kCtaThreads, true>(in_col, contrib, b + threadIdx.x, e, o.hot);
  else if constexpr (kP < 0) sum = gather_sum_lean<-kP, kCtaThreads>(in_col, contrib, b + threadIdx.x, e, o.hot);
  else if constexpr (kP > 0) sum = gather_sum_pred<kP>(in_col, contrib, b + threadIdx.x, e, kCtaThreads, o.hot);
  else sum = gather_sum<kL1>(in_col, contrib, b + threadIdx.x, e, kCtaThreads, o.hot, o.l1hot);
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kCtaThreads / 32 ? s_part[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) o.put(r, v + (hsum ? hsum[blockIdx.x] : 0.0));
  }
}

// one warp per listed row (32 <= in-degree < kPrCta)
// kRep: 1024-thread CTAs holding the shared-memory replica of contrib[0, rep_k)
template <bool kRep>
__device__ __forceinline__ Rep load_rep(const float* contrib, uint32_t k) {
  if constexpr (kRep) {
    extern __shared__ float s_rep[];
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) s_rep[i] = contrib[i];
    __syncthreads();
    return {s_rep, k};
  } else {
    return {nullptr, 0};
  }
}

template <int kL1, bool kRep = false, int kP = 0>
__global__ void __launch_bounds__(kRep ? 1024 : 256) k_pull_warp(const uint64_t* in_off, const uint32_t* in_col,
                                                   const float* contrib, const uint32_t* rows,
                                                   uint64_t n, PullOut o, uint32_t rep_k,
                                                   const uint32_t* hlen, const double* hsum) {
  const Rep rep = load_rep<kRep>(contrib, rep_k);
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t k = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; k < n; k += nwarps) {
    const uint64_t r = rows[k];
    if (o.rows_end && r >= o.rows_end) continue;  // a sink in a non-final round
    const uint64_t b0 = in_off[r];
    const uint64_t b = b0 + (hlen ? hlen[k] : 0u), e = o.row_end(r, b0, in_off[r + 1]);
    double sum;
    if constexpr (kP < -100) sum = gather_sum_lean<-kP - 100, 32, true>(in_col, contrib, b + lane, e, o.hot);
    else if constexpr (kP < 0) sum = gather_sum_lean<-kP, 32>(in_col, contrib, b + lane, e, o.hot);
    else if constexpr (kP > 0) sum = gather_sum_pred<kP>(in_col, contrib, b + lane, e, 32, o.hot);
    else sum = gather_sum<kL1, kRep>(in_col, contrib, b + lane, e, 32, o.hot, o.l1hot, rep);
    sum = warp_sum(sum);
    if (lane == 0) o.put(r, sum + (hsum ? hsum[k] : 0.0));
  }
}

// one thread per row of [r0, r1) with in-degree < 32 (incl. 0); others skipped
template <int kL1, bool kRep = false, int kP = 0>
__global__ void __launch_bounds__(kRep ? 1024 : 256) k_pull_thread(const uint64_t* in_off, const uint32_t* in_col,
                                                     const float* contrib, uint64_t r0, uint64_t r1,
                                                     PullOut o, uint32_t rep_k = 0) {
  const Rep rep = load_rep<kRep>(contrib, rep_k);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = r0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < r1; r += stride) {
    const uint64_t b = in_off[r], e = in_off[r + 1];
    if (e - b >= 32) continue;
    if constexpr (kP < 0) o.put(r, gather_sum_lean<-kP, 1>(in_col, contrib, b, o.row_end(r, b, e), o.hot));
    else if constexpr (kP > 0) o.put(r, gather_sum_pred<kP>(in_col, contrib, b, o.row_end(r, b, e), 1, o.hot));
    else o.put(r, gather_sum<kL1, kRep>(in_col, contrib, b, o.row_end(r, b, e), 1, o.hot, o.l1hot, rep));
  }
}

// Software-pipelined class pulls (TG_PR_PIPE=1): the row-setup chain (list
// entry -> in_off -> in_col -> gathers) is cut by issuing the next row's
// offsets (and, for the warp class, the list entry two rows ahead) before the
// current row's gathers, so a warp's gathers no longer wait on its own setup.
template <int kL1>
__global__ void __launch_bounds__(256) k_pull_warp_pipe(const uint64_t* in_off,
                                                        const uint32_t* in_col,
                                                        const float* contrib, const uint32_t* rows,
                                                        uint64_t n, PullOut o) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t k0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  uint32_t rA = k0 < n ? rows[k0] : 0u;
  uint32_t rB = k0 + nwarps < n ? rows[k0 + nwarps] : 0u;
  uint64_t bA = 0, eA = 0;
  if (k0 < n) {
    bA = in_off[rA];
    eA = in_off[rA + 1];
  }
  for (uint64_t k = k0; k < n; k += nwarps) {
    const uint64_t kC = k + 2 * nwarps;
    const uint32_t rC = kC < n ? rows[kC] : 0u;
    uint64_t bB = 0, eB = 0;
    if (k + nwarps < n) {
      bB = in_off[rB];
      eB = in_off[rB + 1];
    }
    double sum = gather_sum<kL1>(in_col, contrib, bA + lane, eA, 32, o.hot, o.l1hot);
    sum = warp_sum(sum);
    if (lane == 0) o.put(rA, sum);
    rA = rB;
    bA = bB;
    eA = eB;
    rB = rC;
  }
}

template <int kL1>
__global__ void __launch_bounds__(256) k_pull_thread_pipe(const uint64_t* in_off,
                                                          const uint32_t* in_col,
                                                          const float* contrib, uint64_t r0,
                                                          uint64_t r1, PullOut o) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t r = r0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t b = 0, e = 0;
  if (r < r1) {
    b = in_off[r];
    e = in_off[r + 1];
  }
  for (; r < r1; r += stride) {
    const uint64_t rn = r + stride;
    uint64_t bn = 0, en = 0;
    if (rn < r1) {
      bn = in_off[rn];
      en = in_off[rn + 1];
    }
    if (e - b < 32) o.put(r, gather_sum<kL1>(in_col, contrib, b, e, 1, o.hot, o.l1hot));
    b = bn;
    e = en;
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

// ---------------------------------------------------------------- hub split
constexpr uint32_t kHubThreads = 1024;
constexpr uint32_t kHubChunk = 4096;  // hub entries per task (CTA-class rows split)

// The hub pass: one 1024-thread CTA per SM holds contrib[0, K) in shared
// memory (rep[K] = 0 pads); a warp takes 32 tasks at a time (coalesced task
// reads), and sums them four at a time: 4 independent coalesced u16 column
// loads, 4 LDS gathers, then the rest of any task longer than 32, a warp sum
// per task, and one fp64 atomicAdd per task into its row's hub sum (a CTA-class
// row is several tasks).
__global__ void __launch_bounds__(kHubThreads, 1)
    k_pull_hub(const uint64_t* __restrict__ t_off, const uint32_t* __restrict__ t_len,
               const uint32_t* __restrict__ t_k, uint64_t ntask,
               const uint16_t* __restrict__ hcol, const float* __restrict__ contrib, uint32_t K,
               double* hsum) {
  extern __shared__ float rep[];
  for (uint32_t i = threadIdx.x; i < K; i += blockDim.x) rep[i] = contrib[i];
  if (threadIdx.x == 0) rep[K] = 0.0f;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t stream = l2_evict_first();
  for (uint64_t base = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * 32; base < ntask;
       base += nwarps * 32) {
    const uint64_t my = base + lane;
    uint64_t o = 0;
    uint32_t n = 0, k = 0;
    if (my < ntask) {
      o = t_off[my];
      n = t_len[my];
      k = t_k[my];
    }
    double mine = 0.0;
    const uint32_t cnt = ntask - base < 32 ? (uint32_t)(ntask - base) : 32u;
    for (uint32_t j = 0; j < cnt; j += 4) {
      uint64_t oj[4];
      uint32_t nj[4], ej[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        oj[t] = __shfl_sync(kFull, o, (j + t) & 31);
        nj[t] = __shfl_sync(kFull, n, (j + t) & 31);
        if (j + t >= cnt) nj[t] = 0;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t)
        ej[t] = lane < nj[t] ? (uint32_t)ld_u16_hint(hcol + oj[t] + lane, stream) : K;
      double sj[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) sj[t] = (double)rep[ej[t]];
#pragma unroll
      for (int t = 0; t < 4; ++t)
        for (uint32_t i = lane + 32; i < nj[t]; i += 32)
          sj[t] += (double)rep[ld_u16_hint(hcol + oj[t] + i, stream)];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double v = warp_sum(sj[t]);
        if (lane == j + t) mine = v;
      }
    }
    if (my < ntask) atomicAdd(&hsum[k], mine);
  }
}

// list row k (CTA-class rows, then warp-class rows) -> hub-prefix length (the
// row is ascending, so it is the lower bound of K), entries, tasks
__global__ void k_hub_len(const uint64_t* off, const uint32_t* col, const uint32_t* cta,
                          uint64_t n_cta, const uint32_t* warp, uint64_t n_list, uint32_t K,
                          uint32_t* hlen, uint64_t* h64, uint64_t* tcnt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n_list; k += stride) {
    const uint64_t r = k < n_cta ? cta[k] : warp[k - n_cta];
    uint64_t lo = off[r], hi = off[r + 1];
    const uint64_t b = lo;
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if (col[m] < K) lo = m + 1;
      else hi = m;
    }
    const uint64_t h = lo - b;
    hlen[k] = (uint32_t)h;
    h64[k] = h;
    tcnt[k] = (h + kHubChunk - 1) / kHubChunk;
  }
}

// a warp per list row: copy its hub prefix (u16) and write its tasks
__global__ void k_hub_fill(const uint64_t* off, const uint32_t* col, const uint32_t* cta,
                           uint64_t n_cta, const uint32_t* warp, uint64_t n_list,
                           const uint64_t* hoff, const uint64_t* toff, uint16_t* hcol,
                           uint64_t* t_off, uint32_t* t_len, uint32_t* t_k) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t k = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; k < n_list;
       k += nwarps) {
    const uint64_t r = k < n_cta ? cta[k] : warp[k - n_cta];
    const uint64_t b = off[r], h0 = hoff[k], h = hoff[k + 1] - h0;
    for (uint64_t i = lane; i < h; i += 32) hcol[h0 + i] = (uint16_t)col[b + i];
    const uint64_t t0 = toff[k], nt = toff[k + 1] - t0;
    for (uint64_t j = lane; j < nt; j += 32) {
      t_off[t0 + j] = h0 + j * kHubChunk;
      t_len[t0 + j] = (uint32_t)(h - j * kHubChunk < kHubChunk ? h - j * kHubChunk : kHubChunk);
      t_k[t0 + j] = (uint32_t)k;
    }
  }
}

void scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  size_t tmp = 0;
  TG_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int64_t)n, s));
  DevBuf<uint8_t> t(tmp ? tmp : 1);
  TG_CK(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, (int64_t)n, s));
}

// rows with in-degree < 32, a warp per group of 32 consecutive rows
// (TG_PR_GROUP=1): when every row of the group is short, their in-edges are one
// contiguous range of in_col, walked 128 at a time -- each lane loads 4 columns
// (coalesced) and gathers their contributions into a per-warp shared-memory
// window -- and each row's lane then sums its own entries of the window
// (LDS, fp64).  No per-lane row loops over global memory (a thread per row
// diverges to the group's longest row and reads in_col one lane at a time);
// the rank / contribution writes stay coalesced.  Groups holding a row of
// in-degree >= 32 (left to the warp / CTA classes) take the thread-per-row path.
constexpr int kGroupWin = 128;
template <int kL1>
__global__ void __launch_bounds__(256) k_pull_group(const uint64_t* in_off, const uint32_t* in_col,
                                                    const float* contrib, uint64_t R, PullOut o) {
  __shared__ float s_win[256 / 32][kGroupWin];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* win = s_win[w];
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t keep = l2_evict_last(), stream = l2_evict_first();
  for (uint64_t r0 = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * 32; r0 < R;
       r0 += nwarps * 32) {
    const uint64_t r = r0 + lane;
    const uint64_t rr = r < R ? r : R;
    const uint64_t b = in_off[rr], e = r < R ? in_off[r + 1] : b;
    const bool small = e - b < 32;
    if (__all_sync(kFull, small)) {
      const uint64_t base = __shfl_sync(kFull, b, 0);
      const uint32_t T = (uint32_t)(__shfl_sync(kFull, e, 31) - base);
      const uint32_t lo = (uint32_t)(b - base), hi = (uint32_t)(e - base);
      double acc = 0.0;
      for (uint32_t c0 = 0; c0 < T; c0 += kGroupWin) {
        uint32_t cc[kGroupWin / 32];
#pragma unroll
        for (int k = 0; k < kGroupWin / 32; ++k) {
          const uint32_t idx = c0 + k * 32 + lane;
          cc[k] = idx < T ? ld_u32_hint(in_col + base + idx, stream) : 0u;
        }
#pragma unroll
        for (int k = 0; k < kGroupWin / 32; ++k) {
          const uint32_t idx = c0 + k * 32 + lane;
          float v = 0.0f;
          if (idx < T) v = ld_f32_hint(contrib + cc[k], cc[k] < o.hot ? keep : stream);
          win[k * 32 + lane] = v;
        }
        __syncwarp();
        const uint32_t a0 = lo > c0 ? lo : c0;
        const uint32_t a1 = hi < c0 + kGroupWin ? hi : c0 + kGroupWin;
        for (uint32_t k = a0; k < a1; ++k) acc += (double)win[k - c0];
        __syncwarp();
      }
      if (r < R) o.put(r, acc);
    } else if (r < R && small) {
      o.put(r, gather_sum<kL1>(in_col, contrib, b, e, 1, o.hot, o.l1hot));
    }
  }
}

// r_0 = 1/|V| as the first round's contributions, for rows [0, n) -- rows past
// nz_end have out-degree 0 and nothing gathers them (n = nz_end when the sink
// trims are on).  rank needs no initial value: the last round stores every row.
__global__ void k_pr_init(const uint32_t* outdeg, uint64_t n, double r0, float* contrib) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t od = outdeg[i];
    contrib[i] = od ? (float)(r0 / (double)od) : 0.0f;
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

// Hub split layout for the in-CSR `c` (outside the timed region; rebuilt when
// the layout or K changes).  K = 0 or no class rows: disabled.
void build_pr_hub(PRHub& h, const PullCsr& c, uint64_t Vp, uint32_t K, cudaStream_t s) {
  K = (uint32_t)std::min<uint64_t>(K, Vp);
  if (h.built_for == c.col && h.K == K) return;
  h = PRHub{};
  h.K = K;
  h.built_for = c.col;
  h.n_list = c.n_cta + c.n_warp;
  if (!K || !h.n_list) return;
  const uint64_t n = h.n_list;
  h.hlen.alloc(n);
  DevBuf<uint64_t> h64(n + 1), tc(n + 1), hoff(n + 1), toff(n + 1);
  TG_CK(cudaMemsetAsync(h64.get() + n, 0, 8, s));
  TG_CK(cudaMemsetAsync(tc.get() + n, 0, 8, s));
  k_hub_len<<<grid_for(n, 256), 256, 0, s>>>(c.off, c.col, c.cta, c.n_cta, c.warp, n, K,
                                             h.hlen.get(), h64.get(), tc.get());
  scan_u64(h64.get(), hoff.get(), n + 1, s);
  scan_u64(tc.get(), toff.get(), n + 1, s);
  uint64_t tot[2];
  TG_CK(cudaMemcpyAsync(&tot[0], hoff.get() + n, 8, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaMemcpyAsync(&tot[1], toff.get() + n, 8, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaStreamSynchronize(s));
  h.H = tot[0];
  h.ntask = tot[1];
  TG_REQUIRE(h.ntask < (1ull << 32), TG_ECAPACITY, "pagerank hub split: too many tasks");
  h.col.alloc(std::max<uint64_t>(h.H, 1));
  h.t_off.alloc(std::max<uint64_t>(h.ntask, 1));
  h.t_len.alloc(std::max<uint64_t>(h.ntask, 1));
  h.t_k.alloc(std::max<uint64_t>(h.ntask, 1));
  h.hsum.alloc(n);
  k_hub_fill<<<grid_for(n * 32, 256), 256, 0, s>>>(c.off, c.col, c.cta, c.n_cta, c.warp, n,
                                                   hoff.get(), toff.get(), h.col.get(),
                                                   h.t_off.get(), h.t_len.get(), h.t_k.get());
  TG_CK(cudaGetLastError());
  TG_CK(cudaStreamSynchronize(s));
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
                    bool concurrent, PRHub* hub) {
  cudaStream_t s = eng.stream, s_cta = s, s_warp = s;
  // hub pass first: the class pulls of the CTA / warp rows add its sums
  const uint32_t* hl = nullptr;
  const double* hs = nullptr;
  if (hub && hub->K && hub->ntask && !o.hot_len) {
    const size_t smem = ((size_t)hub->K + 1) * sizeof(float);
    TG_CK(cudaFuncSetAttribute(k_pull_hub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TG_CK(cudaMemsetAsync(hub->hsum.get(), 0, hub->n_list * sizeof(double), s));
    k_pull_hub<<<148, kHubThreads, smem, s>>>(hub->t_off.get(), hub->t_len.get(), hub->t_k.get(),
                                              hub->ntask, hub->col.get(), contrib, hub->K,
                                              hub->hsum.get());
    eng.launches++;
    hl = hub->hlen.get();
    hs = hub->hsum.get();
  }
  if (concurrent) {
    eng.fork();
    s_cta = eng.side[0];
    s_warp = eng.side[1];
  }
  const uint64_t R = o.rows_end ? std::min<uint64_t>(c.R, o.rows_end) : c.R;
  // batches per class (TG_PR_PRED=Ucta,Uwarp,Uthread): U > 0 predicated batches
  // (gather_sum_pred), U < 0 lean batches of -U (gather_sum_lean), 0 the plain
  // loop.  Default -8,-8,-4: RMAT-28 19.2 -> 18.2 ms per round
  // (profiles/r02_pr_lean_ab.txt)
  int pu[3] = {-8, -8, -4};
  if (kL1 != 0 || hl) pu[0] = pu[1] = pu[2] = 0;
  else if (const char* v = std::getenv("TG_PR_PRED"))
    std::sscanf(v, "%d,%d,%d", &pu[0], &pu[1], &pu[2]);
  if (c.n_cta) {
    if (pu[0] == -108)
      k_pull_cta<kL1, -108><<<(unsigned)c.n_cta, kCtaThreads, 0, s_cta>>>(c.off, c.col, contrib, c.cta, o, hl, hs);
    else if (pu[0] == -16)
      k_pull_cta<kL1, -16><<<(unsigned)c.n_cta, kCtaThreads, 0, s_cta>>>(c.off, c.col, contrib, c.cta, o, hl, hs);
    else if (pu[0] == -8)
      k_pull_cta<kL1, -8><<<(unsigned)c.n_cta, kCtaThreads, 0, s_cta>>>(c.off, c.col, contrib, c.cta, o, hl, hs);
    else if (pu[0] == -4)
      k_pull_cta<kL1, -4><<<(unsigned)c.n_cta, kCtaThreads, 0, s_cta>>>(c.off, c.col, contrib, c.cta, o, hl, hs);
    else if (pu[0] == 2)
      k_pull_cta<kL1, 2><<<(unsigned)c.n_cta, kCtaThreads, 0, s_cta>>>(c.off, c.col, contrib, c.cta, o, hl, hs);
    else if (pu[0] == 4)
      k_pull_cta<kL1, 4><<<(unsigned)c.n_cta, kCtaThreads, 0, s_cta>>>(c.off, c.col, contrib, c.cta, o, hl, hs);
    else
      k_pull_cta<kL1><<<(unsigned)c.n_cta, kCtaThreads, 0, s_cta>>>(c.off, c.col, contrib, c.cta, o,
                                                                    hl, hs);
    eng.launches++;
  }
  // TG_PR_REP=k (A/B): warp / thread classes (TG_PR_REP_CLASSES bits 2 / 4) in
  // 1024-thread CTAs, TG_PR_REP_CTAS per SM, each with a shared-memory replica
  // of contrib[0, k)
  uint32_t rep_k = 0, rep_cls = 6, rep_ctas = 2;
  if (const char* v = std::getenv("TG_PR_REP")) rep_k = (uint32_t)std::strtoul(v, nullptr, 10);
  if (const char* v = std::getenv("TG_PR_REP_CLASSES")) rep_cls = (uint32_t)std::atoi(v);
  if (const char* v = std::getenv("TG_PR_REP_CTAS")) rep_ctas = (uint32_t)std::atoi(v);
  const size_t rep_bytes = (size_t)rep_k * sizeof(float);
  if (rep_k) {
    TG_CK(cudaFuncSetAttribute(k_pull_warp<kL1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)rep_bytes));
    TG_CK(cudaFuncSetAttribute(k_pull_thread<kL1, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rep_bytes));
  }
  const char* pipe_env = std::getenv("TG_PR_PIPE");
  // bit 1 warp class, bit 2 thread class; the cold-tail split (o.hot_len) runs
  // the default class kernels only
  const int pipe = pipe_env && !o.hot_len ? std::atoi(pipe_env) : 0;
  if (o.hot_len) rep_k = 0;
  if (c.n_warp && (pipe & 1) && !hl) {
    k_pull_warp_pipe<kL1><<<grid_for(c.n_warp * 32, 256, 148u * 16u), 256, 0, s_warp>>>(
        c.off, c.col, contrib, c.warp, c.n_warp, o);
    eng.launches++;
  } else if (c.n_warp && (pu[1] == 4 || pu[1] == 8 || pu[1] == 6 || pu[1] == -4 || pu[1] == -8 ||
                           pu[1] == -6 || pu[1] == -108)) {
    const unsigned g = grid_for(c.n_warp * 32, 256, 148u * 16u);
    if (pu[1] == -108)
      k_pull_warp<kL1, false, -108><<<g, 256, 0, s_warp>>>(c.off, c.col, contrib, c.warp, c.n_warp, o, 0u, nullptr, nullptr);
    else if (pu[1] == -6)
      k_pull_warp<kL1, false, -6><<<g, 256, 0, s_warp>>>(c.off, c.col, contrib, c.warp, c.n_warp, o, 0u, nullptr, nullptr);
    else if (pu[1] == -4)
      k_pull_warp<kL1, false, -4><<<g, 256, 0, s_warp>>>(c.off, c.col, contrib, c.warp, c.n_warp, o, 0u, nullptr, nullptr);
    else if (pu[1] == -8)
      k_pull_warp<kL1, false, -8><<<g, 256, 0, s_warp>>>(c.off, c.col, contrib, c.warp, c.n_warp, o, 0u, nullptr, nullptr);
    else if (pu[1] == 4)
      k_pull_warp<kL1, false, 4><<<g, 256, 0, s_warp>>>(c.off, c.col, contrib, c.warp, c.n_warp, o, 0u, nullptr, nullptr);
    else if (pu[1] == 6)
      k_pull_warp<kL1, false, 6><<<g, 256, 0, s_warp>>>(c.off, c.col, contrib, c.warp, c.n_warp, o, 0u, nullptr, nullptr);
    else
      k_pull_warp<kL1, false, 8><<<g, 256, 0, s_warp>>>(c.off, c.col, contrib, c.warp, c.n_warp, o, 0u, nullptr, nullptr);
    eng.launches++;
  } else if (c.n_warp) {
    if (rep_k && (rep_cls & 2))
      k_pull_warp<kL1, true><<<148u * rep_ctas, 1024, rep_bytes, s_warp>>>(
          c.off, c.col, contrib, c.warp, c.n_warp, o, rep_k, hl ? hl + c.n_cta : nullptr,
          hs ? hs + c.n_cta : nullptr);
    else
      k_pull_warp<kL1><<<grid_for(c.n_warp * 32, 256, 148u * 16u), 256, 0, s_warp>>>(
          c.off, c.col, contrib, c.warp, c.n_warp, o, 0u, hl ? hl + c.n_cta : nullptr,
          hs ? hs + c.n_cta : nullptr);
    eng.launches++;
  }
  if (R) {
    const char* seg = o.hot_len ? nullptr : std::getenv("TG_PR_SEG");
    const char* grp = o.hot_len ? nullptr : std::getenv("TG_PR_GROUP");
    if (seg && seg[0] == '1')
      k_pull_seg<<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, R, o);
    else if (pu[2] == 2 || pu[2] == 4 || pu[2] == -4 || pu[2] == -8 || pu[2] == -2) {
      if (pu[2] == -8)
        k_pull_thread<kL1, false, -8><<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, 0, R, o);
      else if (pu[2] == -2)
        k_pull_thread<kL1, false, -2><<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, 0, R, o);
      else if (pu[2] == -4)
        k_pull_thread<kL1, false, -4><<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, 0, R, o);
      else if (pu[2] == 2)
        k_pull_thread<kL1, false, 2><<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, 0, R, o);
      else
        k_pull_thread<kL1, false, 4><<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, 0, R, o);
    } else if (pipe & 2)
      k_pull_thread_pipe<kL1><<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, 0,
                                                                          R, o);
    else if (grp && grp[0] == '1')
      k_pull_group<kL1><<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, R, o);
    else if (rep_k && (rep_cls & 4))
      k_pull_thread<kL1, true><<<148u * rep_ctas, 1024, rep_bytes, s>>>(c.off, c.col, contrib, 0, R,
                                                                       o, rep_k);
    else
      k_pull_thread<kL1><<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(c.off, c.col, contrib, 0, R, o);
    eng.launches++;
  }
  if (concurrent) eng.join();
  TG_CK(cudaGetLastError());
}

void launch_pull(Engine& eng, const PullCsr& c, const float* contrib, const PullOut& o,
                 bool concurrent, int l1, PRHub* hub) {
  switch (l1) {
    case 1: launch_pull_l1<1>(eng, c, contrib, o, concurrent, hub); break;
    case 2: launch_pull_l1<2>(eng, c, contrib, o, concurrent, hub); break;
    case 3: launch_pull_l1<3>(eng, c, contrib, o, concurrent, hub); break;
    case 8: launch_pull_l1<8>(eng, c, contrib, o, concurrent, hub); break;
    case 9: {
      uint32_t lo = 0, hi = 0;
      if (const char* v = std::getenv("TG_PR_XLO")) lo = (uint32_t)std::strtoul(v, nullptr, 10);
      if (const char* v = std::getenv("TG_PR_XHI")) hi = (uint32_t)std::strtoul(v, nullptr, 10);
      TG_CK(cudaMemcpyToSymbolAsync(c_xlo, &lo, 4, 0, cudaMemcpyHostToDevice, eng.stream));
      TG_CK(cudaMemcpyToSymbolAsync(c_xhi, &hi, 4, 0, cudaMemcpyHostToDevice, eng.stream));
      launch_pull_l1<9>(eng, c, contrib, o, concurrent, hub);
      break;
    }
    default: launch_pull_l1<0>(eng, c, contrib, o, concurrent, hub);
  }
}

// ---------------------------------------------------------------- die split
constexpr uint32_t kSplitChunk = 2048;  // rows with more half-edges are cut into chunks
constexpr unsigned kSplitGrab = 8;      // tasks a warp takes from its die's queue at once

__host__ __device__ __forceinline__ uint32_t line_hash(uint32_t l) {
  l ^= l >> 16;
  l *= 0x7feb352du;
  l ^= l >> 15;
  l *= 0x846ca68bu;
  l ^= l >> 16;
  return l;
}
// the die whose SMs gather source u: by its 128-byte line of contributions
__device__ __forceinline__ int src_die(uint32_t u, uint32_t thresh) {
  return line_hash(u >> 5) >= thresh ? 1 : 0;
}

__global__ void k_split_count(const uint64_t* off, const uint32_t* col, uint64_t R, uint32_t thresh,
                              uint64_t* c0, uint64_t* c1) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R; r += stride) {
    uint64_t n1 = 0;
    const uint64_t b = off[r], e = off[r + 1];
    for (uint64_t i = b; i < e; ++i) n1 += src_die(col[i], thresh);
    c0[r] = (e - b) - n1;
    c1[r] = n1;
  }
}

__global__ void k_split_fill(const uint64_t* off, const uint32_t* col, uint64_t R, uint32_t thresh,
                             const uint64_t* o0, const uint64_t* o1, uint32_t* d0, uint32_t* d1) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R; r += stride) {
    uint64_t j0 = o0[r], j1 = o1[r];
    for (uint64_t i = off[r], e = off[r + 1]; i < e; ++i) {
      const uint32_t u = col[i];
      if (src_die(u, thresh)) d1[j1++] = u;
      else d0[j0++] = u;
    }
  }
}

// per row of one half: warp-row flag, chunked-row flag, chunk count
__global__ void k_split_class(const uint64_t* off, uint64_t R, uint64_t* wf, uint64_t* cf,
                              uint64_t* cn) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R; r += stride) {
    const uint64_t n = off[r + 1] - off[r];
    wf[r] = n >= 32 && n < kSplitChunk;
    cf[r] = n >= kSplitChunk;
    cn[r] = n >= kSplitChunk ? (n + kSplitChunk - 1) / kSplitChunk : 0;
  }
}

__global__ void k_split_lists(const uint64_t* off, uint64_t R, const uint64_t* wp, const uint64_t* cp,
                              const uint64_t* np, uint32_t* wrow, uint32_t* c_list, uint32_t* c_row,
                              uint32_t* c_k, uint32_t* c_len, uint64_t* c_start) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R; r += stride) {
    const uint64_t b = off[r], n = off[r + 1] - b;
    if (n >= 32 && n < kSplitChunk) wrow[wp[r]] = (uint32_t)r;
    if (n >= kSplitChunk) {
      const uint64_t k = cp[r];
      c_list[k] = (uint32_t)r;
      for (uint64_t j = 0, t = np[r]; j * kSplitChunk < n; ++j, ++t) {
        c_row[t] = (uint32_t)r;
        c_k[t] = (uint32_t)k;
        c_start[t] = b + j * kSplitChunk;
        c_len[t] = (uint32_t)(n - j * kSplitChunk < kSplitChunk ? n - j * kSplitChunk : kSplitChunk);
      }
    }
  }
}

struct SplitArgs {
  const uint64_t* off[2];
  const uint32_t* col[2];
  const uint32_t* wrow[2];
  const uint32_t* c_k[2];
  const uint32_t* c_len[2];
  const uint64_t* c_start[2];
  uint64_t n_w[2], n_c[2];
  double* cacc[2];
  float* psum[2];
  uint64_t R, nT;
  unsigned long long* qnext;
  const uint8_t* die_of;
  uint32_t hot;
};

__device__ __forceinline__ uint32_t sm_id_pr() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// Persistent warps; each serves the task queue of its own SM's die first
// (chunks of the long rows, then warp rows, then blocks of 32 short rows, one
// lane per row), then helps the other die's queue once its own is empty.
__global__ void __launch_bounds__(256) k_pr_split(SplitArgs a, const float* __restrict__ contrib) {
  const uint32_t lane = threadIdx.x & 31;
  const int mine = a.die_of[sm_id_pr()];
  for (int pass = 0; pass < 2; ++pass) {
    const int d = pass ? mine ^ 1 : mine;
    const uint64_t nc = a.n_c[d], nw = a.n_w[d], nt = nc + nw + a.nT;
    const uint64_t* off = a.off[d];
    const uint32_t* col = a.col[d];
    for (;;) {
      unsigned long long t0 = 0;
      if (lane == 0) t0 = atomicAdd(&a.qnext[d], (unsigned long long)kSplitGrab);
      t0 = __shfl_sync(kFull, t0, 0);
      if (t0 >= nt) break;
      const uint64_t t1 = t0 + kSplitGrab < nt ? t0 + kSplitGrab : nt;
      for (uint64_t t = t0; t < t1; ++t) {
        if (t < nc) {
          const uint64_t b = a.c_start[d][t];
          double sum = gather_sum<0>(col, contrib, b + lane, b + a.c_len[d][t], 32, a.hot, 0);
          sum = warp_sum(sum);
          if (lane == 0) atomicAdd(&a.cacc[d][a.c_k[d][t]], sum);
        } else if (t < nc + nw) {
          const uint32_t r = a.wrow[d][t - nc];
          const uint64_t b = off[r], e = off[r + 1];
          double sum = gather_sum<0>(col, contrib, b + lane, e, 32, a.hot, 0);
          sum = warp_sum(sum);
          if (lane == 0) a.psum[d][r] = (float)sum;
        } else {
          const uint64_t r = (t - nc - nw) * 32 + lane;
          if (r < a.R) {
            const uint64_t b = off[r], e = off[r + 1];
            if (e - b < 32) a.psum[d][r] = (float)gather_sum<0>(col, contrib, b, e, 1, a.hot, 0);
          }
        }
      }
    }
  }
}

__global__ void k_split_cfix(const uint32_t* c_list, const double* cacc, uint64_t n, float* psum) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += stride)
    psum[c_list[k]] = (float)cacc[k];
}

__global__ void k_split_finalize(const float* __restrict__ p0, const float* __restrict__ p1,
                                 uint64_t R, PullOut o) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R; r += stride)
    o.put(r, (double)p0[r] + (double)p1[r]);
}

// Die-split layout of the in-CSR `c` (outside the timed region).  Needs a
// measured two-die map and room for a second copy of the in-CSR; else off.
void build_pr_split(Engine& eng, PRSplit& sp, const PullCsr& c, cudaStream_t s) {
  if (sp.built && sp.built_for == c.col) return;
  sp = PRSplit{};
  sp.built = true;
  sp.built_for = c.col;
  const DieMap& dm = die_map(eng.device);
  const uint64_t R = c.R;
  if (!dm.ok || !R) return;
  uint64_t Ein = 0;
  TG_CK(cudaMemcpyAsync(&Ein, c.off + R, 8, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaStreamSynchronize(s));
  // room: the split in-CSR (4 B per edge + 2 x 8 B per row) + psum + build scratch
  size_t fr = 0, tot = 0;
  TG_CK(cudaMemGetInfo(&fr, &tot));
  const uint64_t need = Ein * 4 + R * (16 + 8 + 5 * 8) + (1ull << 30);
  if (need > fr) return;
  sp.R = R;
  sp.thresh = (uint32_t)(((uint64_t)dm.n[0] << 32) / (uint64_t)dm.nsm);
  {
    DevBuf<uint64_t> c0(R + 1), c1(R + 1);
    TG_CK(cudaMemsetAsync(c0.get() + R, 0, 8, s));
    TG_CK(cudaMemsetAsync(c1.get() + R, 0, 8, s));
    k_split_count<<<grid_for(R, 256), 256, 0, s>>>(c.off, c.col, R, sp.thresh, c0.get(), c1.get());
    sp.off[0].alloc(R + 1);
    sp.off[1].alloc(R + 1);
    scan_u64(c0.get(), sp.off[0].get(), R + 1, s);
    scan_u64(c1.get(), sp.off[1].get(), R + 1, s);
  }
  uint64_t n0 = 0, n1 = 0;
  TG_CK(cudaMemcpyAsync(&n0, sp.off[0].get() + R, 8, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaMemcpyAsync(&n1, sp.off[1].get() + R, 8, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaStreamSynchronize(s));
  sp.col[0].alloc(std::max<uint64_t>(n0, 1));
  sp.col[1].alloc(std::max<uint64_t>(n1, 1));
  k_split_fill<<<grid_for(R, 256), 256, 0, s>>>(c.off, c.col, R, sp.thresh, sp.off[0].get(),
                                                sp.off[1].get(), sp.col[0].get(), sp.col[1].get());
  for (int d = 0; d < 2; ++d) {
    DevBuf<uint64_t> wf(R + 1), cf(R + 1), cn(R + 1), wp(R + 1), cp(R + 1), np(R + 1);
    TG_CK(cudaMemsetAsync(wf.get() + R, 0, 8, s));
    TG_CK(cudaMemsetAsync(cf.get() + R, 0, 8, s));
    TG_CK(cudaMemsetAsync(cn.get() + R, 0, 8, s));
    k_split_class<<<grid_for(R, 256), 256, 0, s>>>(sp.off[d].get(), R, wf.get(), cf.get(), cn.get());
    scan_u64(wf.get(), wp.get(), R + 1, s);
    scan_u64(cf.get(), cp.get(), R + 1, s);
    scan_u64(cn.get(), np.get(), R + 1, s);
    uint64_t cnt[3];
    TG_CK(cudaMemcpyAsync(&cnt[0], wp.get() + R, 8, cudaMemcpyDeviceToHost, s));
    TG_CK(cudaMemcpyAsync(&cnt[1], cp.get() + R, 8, cudaMemcpyDeviceToHost, s));
    TG_CK(cudaMemcpyAsync(&cnt[2], np.get() + R, 8, cudaMemcpyDeviceToHost, s));
    TG_CK(cudaStreamSynchronize(s));
    sp.n_w[d] = cnt[0];
    sp.n_ck[d] = cnt[1];
    sp.n_c[d] = cnt[2];
    sp.wrow[d].alloc(std::max<uint64_t>(cnt[0], 1));
    sp.c_list[d].alloc(std::max<uint64_t>(cnt[1], 1));
    sp.cacc[d].alloc(std::max<uint64_t>(cnt[1], 1));
    sp.c_row[d].alloc(std::max<uint64_t>(cnt[2], 1));
    sp.c_k[d].alloc(std::max<uint64_t>(cnt[2], 1));
    sp.c_len[d].alloc(std::max<uint64_t>(cnt[2], 1));
    sp.c_start[d].alloc(std::max<uint64_t>(cnt[2], 1));
    k_split_lists<<<grid_for(R, 256), 256, 0, s>>>(sp.off[d].get(), R, wp.get(), cp.get(), np.get(),
                                                   sp.wrow[d].get(), sp.c_list[d].get(),
                                                   sp.c_row[d].get(), sp.c_k[d].get(),
                                                   sp.c_len[d].get(), sp.c_start[d].get());
    sp.psum[d].alloc(R);
  }
  sp.qnext.alloc(2);
  TG_CK(cudaGetLastError());
  TG_CK(cudaStreamSynchronize(s));
  sp.on = true;
}

void launch_split(Engine& eng, PRSplit& sp, const float* contrib, const PullOut& o) {
  cudaStream_t s = eng.stream;
  const DieMap& dm = die_map(eng.device);
  SplitArgs a{};
  for (int d = 0; d < 2; ++d) {
    a.off[d] = sp.off[d].get();
    a.col[d] = sp.col[d].get();
    a.wrow[d] = sp.wrow[d].get();
    a.c_k[d] = sp.c_k[d].get();
    a.c_len[d] = sp.c_len[d].get();
    a.c_start[d] = sp.c_start[d].get();
    a.n_w[d] = sp.n_w[d];
    a.n_c[d] = sp.n_c[d];
    a.cacc[d] = sp.cacc[d].get();
    a.psum[d] = sp.psum[d].get();
    if (sp.n_ck[d]) TG_CK(cudaMemsetAsync(sp.cacc[d].get(), 0, sp.n_ck[d] * 8, s));
  }
  a.R = sp.R;
  a.nT = (sp.R + 31) / 32;
  a.qnext = sp.qnext.get();
  a.die_of = dm.die_of.get();
  a.hot = o.hot;
  TG_CK(cudaMemsetAsync(sp.qnext.get(), 0, 16, s));
  static int per_sm = 0;
  if (!per_sm) {
    TG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pr_split, 256, 0));
    if (per_sm < 1) per_sm = 1;
  }
  k_pr_split<<<(unsigned)(dm.nsm * per_sm), 256, 0, s>>>(a, contrib);
  eng.launches++;
  for (int d = 0; d < 2; ++d)
    if (sp.n_ck[d]) {
      k_split_cfix<<<grid_for(sp.n_ck[d], 256), 256, 0, s>>>(sp.c_list[d].get(), sp.cacc[d].get(),
                                                             sp.n_ck[d], sp.psum[d].get());
      eng.launches++;
    }
  k_split_finalize<<<grid_for(sp.R, 256), 256, 0, s>>>(sp.psum[0].get(), sp.psum[1].get(), sp.R, o);
  eng.launches++;
  TG_CK(cudaGetLastError());
}

// ---------------------------------------------------------------- cold tail
// phase A: a thread per cold source, its contribution into the slot of each
// of its out-edges (slots grouped by target bin, in source order within a bin)
__global__ void k_cold_bin(const uint64_t* __restrict__ row_off, uint64_t T, uint64_t nz_end,
                           uint64_t e0, const uint32_t* __restrict__ pos,
                           const float* __restrict__ contrib, float* binval) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t stream = l2_evict_first();
  for (uint64_t u = T + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nz_end; u += stride) {
    const float v = ld_f32_hint(contrib + u, stream);
    for (uint64_t e = row_off[u], e1 = row_off[u + 1]; e < e1; ++e)
      binval[ld_u32_hint(pos + (e - e0), stream)] = v;
  }
}

// phase B: a CTA per bin sums its slots into 2^kb shared-memory accumulators
// (fp32: a row's cold part is a few small terms) and writes the rows' sums
constexpr unsigned kColdThreads = 1024;
__global__ void __launch_bounds__(kColdThreads) k_cold_acc(const uint64_t* __restrict__ bin_off,
                                                           const uint16_t* __restrict__ binv,
                                                           const float* __restrict__ binval,
                                                           int kb, uint64_t R, float* csum) {
  extern __shared__ float acc[];
  const uint32_t Bz = 1u << kb;
  for (uint32_t j = threadIdx.x; j < Bz; j += blockDim.x) acc[j] = 0.0f;
  __syncthreads();
  const uint64_t stream = l2_evict_first();
  const uint64_t s0 = bin_off[blockIdx.x], s1 = bin_off[blockIdx.x + 1];
  uint64_t i = s0 + threadIdx.x;
  constexpr int U = 8;
  for (; i + (U - 1) * (uint64_t)blockDim.x < s1; i += U * (uint64_t)blockDim.x) {
    uint32_t t[U];
    float v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      t[k] = ld_u16_hint(binv + i + k * blockDim.x, stream);
      v[k] = ld_f32_hint(binval + i + k * blockDim.x, stream);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) atomicAdd(&acc[t[k]], v[k]);
  }
  for (; i < s1; i += blockDim.x) atomicAdd(&acc[ld_u16_hint(binv + i, stream)], ld_f32_hint(binval + i, stream));
  __syncthreads();
  const uint64_t r0 = (uint64_t)blockIdx.x << kb;
  for (uint32_t j = threadIdx.x; j < Bz && r0 + j < R; j += blockDim.x) csum[r0 + j] = acc[j];
}

__global__ void k_cold_keys(const uint32_t* col, uint64_t e0, uint64_t n, int kb, uint32_t* key,
                            uint32_t* idx, unsigned long long* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t t = col[e0 + i];
    if (t & kRemote) *bad = 1ull;
    key[i] = t >> kb;
    idx[i] = (uint32_t)i;
  }
}

__global__ void k_cold_slots(const uint32_t* skey, const uint32_t* sidx, const uint32_t* col,
                             uint64_t e0, uint64_t n, int kb, uint32_t* pos, uint16_t* binv) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t e = sidx[i];
    pos[e] = (uint32_t)i;
    binv[i] = (uint16_t)(col[e0 + e] & ((1u << kb) - 1u));
  }
}

// bin_off[b] = first sorted slot with key >= b
__global__ void k_cold_binoff(const uint32_t* skey, uint64_t n, uint64_t nbins, uint64_t* bin_off) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b <= nbins; b += stride) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if (skey[m] < b) lo = m + 1;
      else hi = m;
    }
    bin_off[b] = lo;
  }
}

__global__ void k_cold_hotlen(const uint64_t* off, const uint32_t* col, uint64_t R, uint32_t T,
                              uint32_t* hot_len) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R; r += stride) {
    uint64_t lo = off[r], hi = off[r + 1];
    const uint64_t b = lo;
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if (col[m] < T) lo = m + 1;
      else hi = m;
    }
    hot_len[r] = (uint32_t)(lo - b);
  }
}

// Cold-tail layout (outside the timed region).  Needs one partition with its
// out-CSR, and memory for the slots + sort scratch; else stays off.
void build_pr_cold(Engine& eng, Part& p, PRCold& c, uint32_t T, int kb, cudaStream_t s) {
  if (c.built_for == p.in_col.get() && c.T == T && c.kb == kb) return;
  c = PRCold{};
  c.T = T;
  c.kb = kb;
  c.built_for = p.in_col.get();
  if (eng.P != 1 || eng.in_only || !p.row_off.get() || T >= p.nz_end || kb < 8 || kb > 16) return;
  uint64_t h[2];
  TG_CK(cudaMemcpyAsync(&h[0], p.row_off.get() + T, 8, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaMemcpyAsync(&h[1], p.row_off.get() + p.nz_end, 8, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaStreamSynchronize(s));
  c.e0 = h[0];
  c.n = h[1] - h[0];
  const uint64_t R = p.Vp;
  if (!c.n || c.n >= (1ull << 32)) return;
  size_t fr = 0, tot = 0;
  TG_CK(cudaMemGetInfo(&fr, &tot));
  if (c.n * 30 + R * 8 + (1ull << 30) > fr) return;
  c.nbins = (R + (1ull << kb) - 1) >> kb;
  {
    DevBuf<uint32_t> key(c.n), idx(c.n), skey(c.n), sidx(c.n);
    DevBuf<unsigned long long> bad(1);
    TG_CK(cudaMemsetAsync(bad.get(), 0, 8, s));
    k_cold_keys<<<grid_for(c.n, 256), 256, 0, s>>>(p.col.get(), c.e0, c.n, kb, key.get(), idx.get(),
                                                   bad.get());
    int bits = 1;
    while ((1ull << bits) < c.nbins) ++bits;
    size_t tmp = 0;
    TG_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.get(), skey.get(), idx.get(), sidx.get(),
                                          (int64_t)c.n, 0, bits, s));
    DevBuf<uint8_t> t(tmp ? tmp : 1);
    TG_CK(cub::DeviceRadixSort::SortPairs(t.get(), tmp, key.get(), skey.get(), idx.get(), sidx.get(),
                                          (int64_t)c.n, 0, bits, s));
    c.pos.alloc(c.n);
    c.binv.alloc(c.n);
    c.bin_off.alloc(c.nbins + 1);
    k_cold_slots<<<grid_for(c.n, 256), 256, 0, s>>>(skey.get(), sidx.get(), p.col.get(), c.e0, c.n,
                                                    kb, c.pos.get(), c.binv.get());
    k_cold_binoff<<<grid_for(c.nbins + 1, 256), 256, 0, s>>>(skey.get(), c.n, c.nbins,
                                                             c.bin_off.get());
    unsigned long long hb = 0;
    TG_CK(cudaMemcpyAsync(&hb, bad.get(), 8, cudaMemcpyDeviceToHost, s));
    TG_CK(cudaStreamSynchronize(s));
    if (hb) {  // remote targets: not a single-partition layout
      c = PRCold{};
      c.built_for = p.in_col.get();
      return;
    }
  }
  c.binval.alloc(c.n);
  c.hot_len.alloc(R);
  c.csum.alloc(R);
  k_cold_hotlen<<<grid_for(R, 256), 256, 0, s>>>(p.in_off.get(), p.in_col.get(), R, T,
                                                 c.hot_len.get());
  TG_CK(cudaGetLastError());
  TG_CK(cudaStreamSynchronize(s));
  c.on = true;
}

void launch_cold(Engine& eng, Part& p, PRCold& c, const float* contrib) {
  cudaStream_t s = eng.stream;
  k_cold_bin<<<grid_for(p.nz_end - c.T, 256, 148u * 16u), 256, 0, s>>>(
      p.row_off.get(), c.T, p.nz_end, c.e0, c.pos.get(), contrib, c.binval.get());
  const size_t smem = ((size_t)1 << c.kb) * sizeof(float);
  TG_CK(cudaFuncSetAttribute(k_cold_acc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_cold_acc<<<(unsigned)c.nbins, kColdThreads, smem, s>>>(c.bin_off.get(), c.binv.get(),
                                                          c.binval.get(), c.kb, p.Vp, c.csum.get());
  eng.launches += 2;
  TG_CK(cudaGetLastError());
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
  // L2 policy of the next round's hub contributions (TG_PR_NEXTPOL)
  int npol = 0;
  if (const char* v = std::getenv("TG_PR_NEXTPOL")) npol = std::atoi(v);
  // row classes on fork/join streams (TG_PR_CONCURRENT=0: one stream)
  const bool concurrent =
      !(std::getenv("TG_PR_CONCURRENT") && std::getenv("TG_PR_CONCURRENT")[0] == '0');
  // rows of out-degree 0 skip their (never gathered) next contribution
  // (TG_PR_NZSKIP=0: every row writes it)
  const bool nzskip = !(std::getenv("TG_PR_NZSKIP") && std::getenv("TG_PR_NZSKIP")[0] == '0');
  // rank stored by the last round only (TG_PR_RANKLAST=0: every round)
  const bool ranklast = !(std::getenv("TG_PR_RANKLAST") && std::getenv("TG_PR_RANKLAST")[0] == '0');
  // non-final rounds do not pull the sinks' rows (TG_PR_SINKSKIP=0: they do)
  const bool sinkskip = !(std::getenv("TG_PR_SINKSKIP") && std::getenv("TG_PR_SINKSKIP")[0] == '0');
  // hub split (PRHub): K hub sources in shared memory (TG_PR_HUB, 0 = off)
  uint32_t hubk = 0;
  if (const char* v = std::getenv("TG_PR_HUB")) hubk = (uint32_t)std::strtoul(v, nullptr, 10);
  if (hubk)
    for (auto& pp : eng.parts) {
      Part& p = *pp;
      build_pr_hub(p.pr.hub, ghost ? ghost_csr(p) : push_csr(p), p.Vp, hubk, s);
    }
  // die split (PRSplit): TG_PR_SPLIT=1 (A/B)
  bool split = false;
  if (const char* v = std::getenv("TG_PR_SPLIT")) split = v[0] == '1';
  if (split)
    for (auto& pp : eng.parts) {
      Part& p = *pp;
      build_pr_split(eng, p.pr.split, ghost ? ghost_csr(p) : push_csr(p), s);
    }
  // cold-tail propagation blocking (PRCold): sources >= TG_PR_COLD (0 = off),
  // target bins of 2^TG_PR_COLD_KB rows
  uint32_t coldT = 0;
  int coldkb = 15;
  if (const char* v = std::getenv("TG_PR_COLD")) coldT = (uint32_t)std::strtoul(v, nullptr, 10);
  if (const char* v = std::getenv("TG_PR_COLD_KB")) coldkb = std::atoi(v);
  bool cold = false;
  if (coldT && !ghost && !split && eng.P == 1) {
    Part& p0 = *eng.parts[0];
    build_pr_cold(eng, p0, p0.pr.cold, coldT, coldkb, s);
    cold = p0.pr.cold.on;
  }

  // rows (and their in-edges) a non-final round does not pull: the sinks
  const bool sinks_idle = sinkskip && nzskip && ranklast && (eng.P == 1 || ghost) && iters > 1;
  uint64_t skip_rows = 0, skip_edges = 0;
  if (sinks_idle) {
    for (auto& pp : eng.parts) {
      Part& p = *pp;
      const PullCsr c = ghost ? ghost_csr(p) : push_csr(p);
      if (p.pr.sinks_for != c.off) {
        uint64_t h[2] = {0, 0};
        if (p.nz_end < p.Vp) {
          TG_CK(cudaMemcpyAsync(&h[0], c.off + std::max<uint64_t>(p.nz_end, 1), 8,
                                cudaMemcpyDeviceToHost, s));
          TG_CK(cudaMemcpyAsync(&h[1], c.off + p.Vp, 8, cudaMemcpyDeviceToHost, s));
          TG_CK(cudaStreamSynchronize(s));
        }
        p.pr.sink_rows = p.Vp - std::min<uint64_t>(std::max<uint64_t>(p.nz_end, 1), p.Vp);
        p.pr.sink_edges = h[1] - h[0];
        p.pr.sinks_for = c.off;
      }
      skip_rows += p.pr.sink_rows;
      skip_edges += p.pr.sink_edges;
    }
    uint64_t x[2] = {skip_rows, skip_edges};
    comm_allreduce(eng, x, 2, 0);
    skip_rows = x[0];
    skip_edges = x[1];
  }
  time_begin(eng);
  eng.each_part([&](Part& p) {
    cudaStream_t s = eng.stream;
    if (!p.Vp) return;
    const uint64_t n = nzskip ? std::min<uint64_t>(p.nz_end, p.Vp) : p.Vp;
    if (n) k_pr_init<<<grid_for(n, 256), 256, 0, s>>>(p.outdeg.get(), n, r0, p.pr.contrib[0].get());
    eng.launches++;
  });
  if (ghost) publish(eng, 0);
  int cur = 0;
  for (int it = 0; it < iters; ++it) {
    eng.prof_begin(TG_K_PR_PULL);
    eng.each_part([&](Part& p) {
      cudaStream_t s = eng.stream;
      PRState& r = p.pr;
      // P == 1 and ghost-pull: every in-edge is in the row, finalize in the pull
      PullOut o{eng.P == 1 || ghost, p.Vp, base, d, r.acc.get(), r.obox.get(), r.rank.get(),
                r.contrib[cur ^ 1].get(), p.outdeg.get(), hot, l1hot, npol,
                cold ? r.cold.hot_len.get() : nullptr, cold ? r.cold.csum.get() : nullptr,
                p.rout(), eng.fused, it & 1};
      if (nzskip) o.nz_end = p.nz_end;
      if (ranklast) o.rank_out = it + 1 == iters;
      if (ranklast && !ghost) o.contrib_out = it + 1 < iters;  // ghost: published after the pull
      if (sinkskip && nzskip && !o.rank_out && o.fused) o.rows_end = std::max<uint64_t>(p.nz_end, 1);
      if (cold) launch_cold(eng, p, r.cold, r.contrib[cur].get());
      if (eng.P == 1) eng.l2_window(r.contrib[cur].get(), p.Vp * sizeof(float));  // opt-in
      if (split && r.split.on)
        launch_split(eng, r.split, r.contrib[cur].get(), o);
      else
        launch_pull(eng, ghost ? ghost_csr(p) : push_csr(p), r.contrib[cur].get(), o, concurrent,
                    l1, hubk ? &r.hub : nullptr);
    });
    eng.prof_end(TG_K_PR_PULL);
    if (ghost) {  // communication: contributions of boundary sources -> peers' ghosts
      eng.prof_begin(TG_K_EXCHANGE);
      if (it + 1 < iters) publish(eng, cur ^ 1);
      eng.prof_end(TG_K_EXCHANGE);
    }
    // pull: in_col 4 + contrib gather 4 per edge; in_off 8 + outdeg 4 + rank 4 +
    // next contrib 4 per row
    {  // the units this round pulled (non-final rounds skip the sinks' rows)
      const bool skipped = sinks_idle && it + 1 < iters;
      eng.prof_bytes(TG_K_PR_PULL, 8.0 * (eng.E - (skipped ? skip_edges : 0)) +
                                       20.0 * (eng.V - (skipped ? skip_rows : 0)));
    }
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
      eng.each_part([&](Part& p) {
        cudaStream_t s = eng.stream;
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
      });
      eng.prof_end(TG_K_EXCHANGE);
    }
    cur ^= 1;
  }
  const double ms = time_end(eng);
  eng.l2_window(nullptr, 0);
  if (st) {
    st->device_ms = ms;
    st->supersteps = (uint64_t)iters;
    // edges and rows pulled: the non-final rounds skip the sinks' rows (their
    // in-edges, ~0.8 % of E on RMAT, are not counted as traversed)
    const uint64_t rounds_skip = sinks_idle ? (uint64_t)iters - 1 : 0;
    st->relaxations = eng.E * (uint64_t)iters - skip_edges * rounds_skip;
    st->traversed_edges = st->relaxations;
    // per pulled edge 8 B (in_col + contrib gather) + 20 B per pulled row
    // (in_off 8, outdeg 4, rank 4, contrib 4) -- DESIGN.md "Roofline"
    st->algorithmic_bytes = st->relaxations * 8 + (eng.V * (uint64_t)iters - skip_rows * rounds_skip) * 20;
    st->comm_bytes = eng.comm_bytes;
    st->launches = eng.launches;
  }
  collect(eng, [](Part& p) -> const void* { return p.pr.rank.get(); }, sizeof(float), out, mem);
}

}  // namespace tg
