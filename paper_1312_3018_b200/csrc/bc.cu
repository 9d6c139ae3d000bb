// bc.cu -- Brandes betweenness centrality as two BSP cycles per source
// (Fig. 18; readings A9-A14).
//
// Forward cycle, superstep L (frontier = level-L bitmap F[L]):
//   edge (v,t): t unvisited -> sigma[t] += sigma[v] (fp64 atomic add, Fig. 18
//   line 12) and t joins F[L+1] (lines 7-9).  Remote t: the partial sigma is
//   summed into t's outbox slot unless the slot was sent at an earlier level
//   (then t is known to be at level <= L); sigma messages are pushed, the owner
//   adds those that reach a still-unvisited vertex.  Level bitmaps F[0..maxL]
//   are kept for the backward cycle.
// Backward cycle, L = maxL .. 1 (pull):
//   c[w] = (1 + delta[w]) / sigma[w] for w in F[L+1]; owners publish c of their
//   boundary vertices to the referencing partitions (ghosts);
//   delta[v] = sigma[v] * sum_{(v,w), w in F[L+1]} c[w]     (Fig. 18 lines 22-30
//   with the "1 +" of Brandes' recurrence restored, reading A9);
//   bc[v] += delta[v]; the source (level 0) is never updated (line 34).
// The backward sum uses the tile kernel in reduce mode: per-row sums in shared
// memory, rows that span tiles accumulate with fp64 atomics.
// Fused exchange (Engine::fused, default): forward sigma partial sums are
// RED.ADD straight into the owner's inbox slot; backward, owners store c of
// their boundary vertices straight into the referencing partitions' ghost
// slots (arena_rev, double-buffered by level parity).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "frontier.cuh"

namespace tg {

namespace {

struct BcFwdOp {
  using Aux = double;
  static constexpr bool kReduce = false, kFilter = false;
  const uint32_t* col;
  const uint32_t* visited;
  uint32_t* next;
  double* sigma;
  const uint32_t* omark;
  uint32_t* onew;
  double* osigma;
  RemoteOut rout;  // fused: sigma partial sums RED.ADD straight into the owner's inbox slot
  bool fused;
  __device__ __forceinline__ Aux aux(uint32_t v) const { return sigma[v]; }
  // split walker (frontier.cuh): column, then the target's state words, then
  // the sigma reductions
  static constexpr bool kSplit = true;
  static constexpr int kUnroll = 2;
  struct Pre {
    uint32_t t;
  };
  struct St {
    uint32_t a, b;  // local: visited / next word; remote: sent-before / sent-now word
  };
  __device__ __forceinline__ Pre pre(uint64_t e) const { return {__ldcs(col + e)}; }
  __device__ __forceinline__ St st(const Pre& p) const {
    if (p.t & kRemote) {
      const uint32_t s = p.t & ~kRemote;
      return {omark[s >> 5], onew[s >> 5]};
    }
    return {__ldg(visited + (p.t >> 5)), next[p.t >> 5]};
  }
  __device__ __forceinline__ void fin(const Aux& sv, const Pre& p, const St& q) const {
    const uint32_t t = p.t;
    if (t & kRemote) {
      const uint32_t s = t & ~kRemote, m = 1u << (s & 31);
      if (!(q.a & m)) {
        atomicAdd(fused ? rout.slot<double>(s) : &osigma[s], sv);
        if (!(q.b & m)) atomicOr(&onew[s >> 5], m);
      }
    } else {
      const uint32_t m = 1u << (t & 31);
      if (!(q.a & m)) {
        atomicAdd(&sigma[t], sv);
        if (!(q.b & m)) atomicOr(&next[t >> 5], m);
      }
    }
  }
};

struct BcBwdOp {
  using Aux = Empty;
  static constexpr bool kReduce = true, kFilter = false;
  const uint32_t* col;
  const uint32_t* succ;  // F[L+1]
  const double* c;
  const double* ghost;  // owners' c of boundary targets (arena_rev; stride 2 when fused)
  uint32_t gstride;
  double* dsum;
  __device__ __forceinline__ Aux aux(uint32_t) const { return {}; }
  __device__ __forceinline__ double edge_val(uint64_t e) const {
    const uint32_t t = __ldcs(col + e);
    if (t & kRemote) return ghost[(uint64_t)(t & ~kRemote) * gstride];
    return bit_test(succ, t) ? c[t] : 0.0;
  }
  __device__ __forceinline__ void vertex_done(uint32_t v, double acc, bool whole) const {
    if (whole) dsum[v] = acc;
    else atomicAdd(&dsum[v], acc);
  }
};

// Pull forward superstep for dense levels (direction optimization): every
// unvisited v sums sigma over its in-neighbours in F[L]; a non-zero sum puts v
// in F[L+1].  No atomics: the warp owns its word of F[L+1] and each lane its
// sigma[v].  Same sigma as the push form (integer-valued fp64 sums are exact).
// P > 1: the ghost in-CSR; a source u >= Vp is ghost u - Vp whose owner
// published sigma (0 when not in F[L]) into gsig.
__global__ void __launch_bounds__(256) k_bc_pull(const uint64_t* in_off, const uint32_t* in_col,
                                                 const uint32_t* F, const uint32_t* visited,
                                                 double* sigma, uint32_t* next, uint64_t Vp,
                                                 unsigned long long* edges, const double* gsig) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t nwords = words_for(Vp);
  unsigned long long cnt = 0;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < nwords; w += nwarps) {
    const uint32_t vis = visited[w];
    const uint64_t v = w * 32 + lane;
    const bool cand = v < Vp && !((vis >> lane) & 1u);
    if (!__ballot_sync(0xffffffffu, cand)) continue;
    double s = 0.0;
    if (cand) {
      const uint64_t b = in_off[v], e = in_off[v + 1];
      cnt += e - b;
      for (uint64_t i = b; i < e; ++i) {
        const uint32_t u = __ldg(in_col + i);
        if (gsig && u >= Vp) s += gsig[u - Vp];
        else if ((__ldg(F + (u >> 5)) >> (u & 31)) & 1u) s += sigma[u];
      }
      if (s > 0.0) sigma[v] = s;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, s > 0.0);
    if (lane == 0 && m) next[w] = m;
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  if (lane == 0 && cnt) atomicAdd(edges, cnt);
}

// Pull-sigma by in-degree class (the PageRank row classes of the in-CSR): the
// thread-per-vertex k_bc_pull walks a hub row's in-edges serially in one
// thread; here rows of in-degree >= 2048 get a CTA, 32..2047 a warp (lanes
// stride the row: coalesced in_col, independent gathers), < 32 a thread.
// Visited rows are skipped; a non-zero sum sets sigma[v] and v's F[L+1] bit.
struct PullSigma {
  const uint64_t* in_off;
  const uint32_t* in_col;
  const uint32_t* F;        // F[L]
  const uint32_t* visited;
  const uint32_t* has_in;   // rows with an in-edge
  double* sigma;
  uint32_t* next;           // F[L+1]
  unsigned long long* edges;
  const double* gsig;       // P > 1: ghost sources u >= Vp (sigma, 0 if not in F[L])
  uint32_t Vp;
  __device__ __forceinline__ bool skip(uint64_t v) const {
    return bit_test(visited, (uint32_t)v) || !bit_test(has_in, (uint32_t)v);
  }
  __device__ __forceinline__ double val(uint32_t u) const {
    if (gsig && u >= Vp) return gsig[u - Vp];
    return bit_test(F, u) ? sigma[u] : 0.0;
  }
  __device__ __forceinline__ double sum(uint64_t i, uint64_t e, uint32_t step) const {
    double s0 = 0.0, s1 = 0.0;
    if (gsig) {
      for (; i + step < e; i += 2ull * step) {
        const uint32_t u0 = __ldg(in_col + i), u1 = __ldg(in_col + i + step);
        s0 += val(u0);
        s1 += val(u1);
      }
      if (i < e) s0 += val(__ldg(in_col + i));
      return s0 + s1;
    }
    for (; i + step < e; i += 2ull * step) {
      const uint32_t u0 = __ldg(in_col + i), u1 = __ldg(in_col + i + step);
      const uint32_t w0 = __ldg(F + (u0 >> 5)), w1 = __ldg(F + (u1 >> 5));
      if ((w0 >> (u0 & 31)) & 1u) s0 += sigma[u0];
      if ((w1 >> (u1 & 31)) & 1u) s1 += sigma[u1];
    }
    if (i < e) {
      const uint32_t u = __ldg(in_col + i);
      if (bit_test(F, u)) s0 += sigma[u];
    }
    return s0 + s1;
  }
  __device__ __forceinline__ void put(uint64_t v, double x) const {
    if (x > 0.0) {
      sigma[v] = x;
      atomicOr(&next[v >> 5], 1u << (v & 31));
    }
  }
};

__global__ void __launch_bounds__(256) k_bc_pull_cta(PullSigma o, const uint32_t* rows) {
  __shared__ double s_part[8];
  const uint64_t v = rows[blockIdx.x];
  if (o.skip(v)) return;  // uniform over the CTA
  const uint64_t b = o.in_off[v], e = o.in_off[v + 1];
  double x = o.sum(b + threadIdx.x, e, 256);
  for (int k = 16; k; k >>= 1) x += __shfl_xor_sync(0xffffffffu, x, k);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += s_part[k];
    o.put(v, t);
    atomicAdd(o.edges, (unsigned long long)(e - b));
  }
}

__global__ void __launch_bounds__(256) k_bc_pull_warp(PullSigma o, const uint32_t* rows, uint64_t n) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long cnt = 0;
  for (uint64_t k = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; k < n; k += nw) {
    const uint64_t v = rows[k];
    if (o.skip(v)) continue;  // uniform over the warp
    const uint64_t b = o.in_off[v], e = o.in_off[v + 1];
    double x = o.sum(b + lane, e, 32);
    for (int m = 16; m; m >>= 1) x += __shfl_xor_sync(0xffffffffu, x, m);
    if (lane == 0) {
      o.put(v, x);
      cnt += e - b;
    }
  }
  if (lane == 0 && cnt) atomicAdd(o.edges, cnt);
}

__global__ void __launch_bounds__(256) k_bc_pull_thread(PullSigma o, uint64_t Vp) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long cnt = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < Vp; v += stride) {
    if (o.skip(v)) continue;  // visited bitmap first: sparse levels skip the offsets
    const uint64_t b = o.in_off[v], e = o.in_off[v + 1];
    if (e - b >= 32) continue;
    o.put(v, o.sum(b, e, 1));
    cnt += e - b;
  }
  for (int m = 16; m; m >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, m);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(o.edges, cnt);
}

// Backward pull by out-degree class: for v in F[L], dsum[v] = sum over its
// out-edges (v, t) with t in F[L+1] of c[t] (remote t: the owner's published c
// in the ghost slot).  Local ids are in out-degree order, so the classes are
// id ranges: [0, n_big) a CTA per row, [n_big, n_mid) a warp, the rest a
// thread; rows not in F[L] are skipped.  Replaces the reduce-mode tile walker
// (segmented fp64 shuffles per 32 edges) on the dense backward levels.
struct PullDelta {
  const uint64_t* row_off;
  const uint32_t* col;
  const uint32_t* FL;    // F[L]
  const uint32_t* succ;  // F[L+1]
  const double* c;
  const double* ghost;
  uint32_t gstride;
  double* dsum;
  unsigned long long* edges;
  __device__ __forceinline__ double val(uint32_t t) const {
    if (t & kRemote) return ghost[(uint64_t)(t & ~kRemote) * gstride];
    return bit_test(succ, t) ? c[t] : 0.0;
  }
  __device__ __forceinline__ double sum(uint64_t i, uint64_t e, uint32_t step) const {
    double s0 = 0.0, s1 = 0.0;
    for (; i + step < e; i += 2ull * step) {
      const uint32_t t0 = __ldcs(col + i), t1 = __ldcs(col + i + step);
      s0 += val(t0);
      s1 += val(t1);
    }
    if (i < e) s0 += val(__ldcs(col + i));
    return s0 + s1;
  }
};

__global__ void __launch_bounds__(256) k_bc_bwd_cta(PullDelta o, uint64_t n) {
  __shared__ double s_part[8];
  for (uint64_t v = blockIdx.x; v < n; v += gridDim.x) {
    if (!bit_test(o.FL, (uint32_t)v)) continue;  // uniform over the CTA
    const uint64_t b = o.row_off[v], e = o.row_off[v + 1];
    double x = o.sum(b + threadIdx.x, e, 256);
    for (int k = 16; k; k >>= 1) x += __shfl_xor_sync(0xffffffffu, x, k);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int k = 0; k < 8; ++k) t += s_part[k];
      o.dsum[v] = t;
      atomicAdd(o.edges, (unsigned long long)(e - b));
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_bc_bwd_warp(PullDelta o, uint64_t r0, uint64_t r1) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long cnt = 0;
  for (uint64_t v = r0 + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5); v < r1; v += nw) {
    if (!bit_test(o.FL, (uint32_t)v)) continue;  // uniform over the warp
    const uint64_t b = o.row_off[v], e = o.row_off[v + 1];
    double x = o.sum(b + lane, e, 32);
    for (int m = 16; m; m >>= 1) x += __shfl_xor_sync(0xffffffffu, x, m);
    if (lane == 0) {
      o.dsum[v] = x;
      cnt += e - b;
    }
  }
  if (lane == 0 && cnt) atomicAdd(o.edges, cnt);
}

__global__ void __launch_bounds__(256) k_bc_bwd_thread(PullDelta o, uint64_t r0, uint64_t r1) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long cnt = 0;
  for (uint64_t v = r0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < r1; v += stride) {
    if (!bit_test(o.FL, (uint32_t)v)) continue;
    const uint64_t b = o.row_off[v], e = o.row_off[v + 1];
    o.dsum[v] = o.sum(b, e, 1);
    cnt += e - b;
  }
  for (int m = 16; m; m >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, m);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(o.edges, cnt);
}

// first local id with out-degree < deg (ids sorted by out-degree descending)
__global__ void k_first_below(const uint64_t* row_off, uint64_t n, uint32_t deg, uint64_t* out) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (row_off[mid + 1] - row_off[mid] >= deg) lo = mid + 1;
    else hi = mid;
  }
  *out = lo;
}

void degree_classes(Engine& eng, Part& p) {
  BCState& b = p.bcs;
  if (b.classes) return;
  DevBuf<uint64_t> d(2);
  k_first_below<<<1, 1, 0, eng.stream>>>(p.row_off.get(), p.nz_end, 2048, d.get());
  k_first_below<<<1, 1, 0, eng.stream>>>(p.row_off.get(), p.nz_end, 32, d.get() + 1);
  TG_CK(cudaGetLastError());
  uint64_t h[2];
  TG_CK(cudaMemcpyAsync(h, d.get(), 16, cudaMemcpyDeviceToHost, eng.stream));
  TG_CK(cudaStreamSynchronize(eng.stream));
  b.n_big = h[0];
  b.n_mid = h[1];
  b.classes = true;
}

// Backward push over the in-CSR (direction-optimized backward level): for each
// w in F[L+1] (Aux = c[w]) and in-edge (v, w) with v in F[L]: dsum[v] += c[w].
struct BcBwdPushOp {
  using Aux = double;
  static constexpr bool kReduce = false, kFilter = false;
  const uint32_t* in_col;
  const uint32_t* FL;
  const double* c;
  double* dsum;
  // row w < Vp: local w in F[L+1]; row Vp + s (P > 1): outbox slot s, whose
  // owner published c of its vertex into ghost slot s (0 if not in F[L+1])
  __device__ __forceinline__ Aux aux(uint32_t w) const {
    return w < Vp ? c[w] : ghost[(uint64_t)(w - Vp) * gstride];
  }
  static constexpr bool kSplit = true;
  static constexpr int kUnroll = 2;  // in_col, then the F[L] word, then the add
  struct Pre {
    uint32_t v;
  };
  struct St {
    uint32_t word;
  };
  __device__ __forceinline__ Pre pre(uint64_t e) const { return {__ldcs(in_col + e)}; }
  __device__ __forceinline__ St st(const Pre& p) const { return {FL[p.v >> 5]}; }
  // Hub targets [0, priv) accumulate in a per-CTA shared-memory copy of dsum,
  // flushed once per CTA: contended global RED.ADD.F64 on a few hot addresses
  // runs at 11-31 G/s vs ~185 G/s spread out (profiles/r01_atomic_probe.txt),
  // and the backward push's targets are mostly hubs (ids are in out-degree order).
  // Privatized targets are [hub, hub + priv): the hottest ones, [0, hub), are
  // not pushed at all -- their dsum comes from a pull over their out-rows
  // (k_bc_bwd_cta over [0, hub) before the push), which costs their out-degree
  // in coalesced reads instead of ~that many RED.ADDs serialized on one address.
  uint32_t priv;
  static constexpr bool kBlockHooks = true;
  size_t smem_bytes() const { return (size_t)priv * sizeof(double); }
  __device__ __forceinline__ void block_begin() const {
    extern __shared__ double s_dsum[];
    for (uint32_t i = threadIdx.x; i < priv; i += blockDim.x) s_dsum[i] = 0.0;
    __syncthreads();
  }
  __device__ __forceinline__ void block_end() const {
    extern __shared__ double s_dsum[];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < priv; i += blockDim.x)
      if (s_dsum[i] != 0.0) atomicAdd(&dsum[hub + i], s_dsum[i]);
  }
  uint32_t Vp;
  const double* ghost;
  uint32_t gstride;
  uint32_t hub;  // sources [0, hub) are pulled, not pushed
  __device__ __forceinline__ void fin(const Aux& cw, const Pre& p, const St& q) const {
    if (p.v < hub || !((q.word >> (p.v & 31)) & 1u)) return;
    const uint32_t k = p.v - hub;
    if (k < priv) {
      extern __shared__ double s_dsum[];
      atomicAdd(&s_dsum[k], cw);
    } else {
      atomicAdd(&dsum[p.v], cw);
    }
  }
};

// P > 1 backward push: active rows of the whole in-CSR [0, Vp + S) = F[L+1]
// for the local rows, ghost c != 0 for the outbox rows (thread per row, one
// ballot per word)
__global__ void k_bc_ext(const uint32_t* F, uint64_t Vp, const double* ghost, uint32_t gstride,
                         uint64_t R, uint32_t* ext) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t n = (R + 31) / 32 * 32;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += stride) {
    bool b = false;
    if (r < Vp) b = bit_test(F, (uint32_t)r);
    else if (r < R) b = ghost[(r - Vp) * gstride] != 0.0;
    const uint32_t m = __ballot_sync(0xffffffffu, b);
    if ((threadIdx.x & 31) == 0) ext[r >> 5] = m;
  }
}

__global__ void k_bc_seed(uint32_t* bm, uint32_t i, double* sigma) {
  bm[i >> 5] |= 1u << (i & 31);
  sigma[i] = 1.0;
}

__global__ void k_bc_scatter(const double* msg, const uint32_t* lid, uint64_t I, const uint32_t* visited,
                             double* sigma, uint32_t* next) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < I; j += stride) {
    const double m = msg[j];
    if (!(m > 0.0)) continue;
    const uint32_t v = lid[j];
    if (bit_test(visited, v)) continue;
    atomicAdd(&sigma[v], m);
    bit_set_atomic(next, v);
  }
}

__global__ void k_or_clear(uint32_t* mark, uint32_t* nw, uint64_t words) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words; i += stride) {
    const uint32_t x = nw[i];
    if (x) {
      mark[i] |= x;
      nw[i] = 0;
    }
  }
}

// owner side of the backward pull: c of boundary vertices in F[L+1], else 0
// fused (pack == nullptr): stored straight into the referencing partition's
// ghost slot (RemoteOut over the inbox, arena_rev double-buffered by parity)
__global__ void k_bc_pack(const uint32_t* lid, uint64_t I, const uint32_t* succ, const double* c,
                          double* pack, RemoteOut rin, int parity) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < I; j += stride) {
    const uint32_t v = lid[j];
    const double x = (v != kInf && bit_test(succ, v)) ? c[v] : 0.0;
    if (pack) pack[j] = x;
    else reinterpret_cast<double*>(rin.slot<double2>((uint32_t)j))[parity] = x;
  }
}

// delta, bc and c for the vertices of level L.  A warp loads 32 consecutive
// bitmap words (coalesced), then visits only the non-zero ones, one lane per
// vertex of the word: sparse levels cost one pass over the bitmap, dense ones
// touch sigma / dsum / bc / c in 32-vertex runs.
__global__ void k_bc_level(const uint32_t* F, uint64_t Vp, uint64_t nz_end, const double* sigma,
                           const double* dsum, double* bc, double* c, unsigned long long* inexact) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t nwords = words_for(Vp);
  for (uint64_t w0 = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * 32; w0 < nwords;
       w0 += nwarps * 32) {
    const uint32_t mine = (w0 + lane < nwords) ? F[w0 + lane] : 0u;
    uint32_t nz = __ballot_sync(0xffffffffu, mine != 0u);
    while (nz) {
      const int j = __ffs(nz) - 1;
      nz &= nz - 1;
      const uint32_t x = __shfl_sync(0xffffffffu, mine, j);
      if (!((x >> lane) & 1u)) continue;
      const uint64_t v = (w0 + j) * 32 + lane;
      const double sv = sigma[v];
      // reading A11: path counts are exact fp64 integers only below 2^53
      if (sv >= 9007199254740992.0) atomicOr(inexact, 1ull);
      const double delta = v < nz_end ? sv * dsum[v] : 0.0;
      bc[v] += delta;
      c[v] = (1.0 + delta) / sv;
    }
  }
}

void* send_osigma(Part& p) { return p.bcs.obox_sigma.get(); }
void* recv_isigma(Part& p) { return p.arena_fwd.get(); }
void* send_pack(Part& p) { return p.bcs.ibox_pack.get(); }
void* recv_ghost(Part& p) { return p.arena_rev.get(); }

// Level bitmaps F[L] are allocated ahead of use (kLevelReserve up front, then
// kLevelReserve more whenever a source reaches past them): cudaMalloc
// synchronizes the device, so growing one level at a time inside a run put an
// allocation (and a stall) in the timed region of every source deeper than
// all earlier ones.
constexpr size_t kLevelReserve = 16;

void reserve_levels(Part& p, size_t L) {
  BCState& b = p.bcs;
  if (b.level_bm.size() > L) return;
  const uint64_t nw = std::max<uint64_t>(words_for(p.Vp), 1);
  const size_t want = (L / kLevelReserve + 1) * kLevelReserve;
  while (b.level_bm.size() < want) b.level_bm.emplace_back(nw);
}

uint32_t* level_bitmap(Part& p, size_t L) {
  reserve_levels(p, L);
  return p.bcs.level_bm[L].get();
}

}  // namespace

void run_bc(Engine& eng, const uint64_t* sources, int k, double* out, int mem, tg_stats* st) {
  TG_REQUIRE(k >= 0 && (k == 0 || sources), TG_EINVAL, "tg_bc: bad source list");
  TG_REQUIRE(out != nullptr || (eng.multi() && eng.rank != 0), TG_EINVAL, "tg_bc: NULL output");
  for (int i = 0; i < k; ++i) TG_REQUIRE(sources[i] < eng.V, TG_EINVAL, "tg_bc: source >= V");
  ensure_frontier_state(eng);
  // outside the timed region: level bitmaps, out-degree class bounds
  for (auto& pp : eng.parts) {
    reserve_levels(*pp, 0);
    degree_classes(eng, *pp);
  }
  // pull-sigma at P > 1 reads remote in-neighbours through the ghost in-CSR
  if (eng.P > 1 && eng.has_in && direction_policy(eng).mode != 1) build_pr_ghost(eng);
  // backward pull by out-degree class (TG_BC_BWD_CLASSES=0: reduce-mode walker)
  const bool bwd_classes =
      !(std::getenv("TG_BC_BWD_CLASSES") && std::getenv("TG_BC_BWD_CLASSES")[0] == '0');
  cudaStream_t s = eng.stream;
  for (auto& pp : eng.parts) {
    Part& p = *pp;
    BCState& b = p.bcs;
    const uint64_t Vn = std::max<uint64_t>(p.Vp, 1);
    if (b.sigma.n < Vn) {
      b.sigma.alloc(Vn);
      b.dsum.alloc(Vn);
      b.c.alloc(Vn);
      b.bc.alloc(Vn);
    }
    if (eng.P > 1 && b.obox_sigma.n < std::max<uint64_t>(p.S, 1)) {
      b.obox_sigma.alloc(std::max<uint64_t>(p.S, 1));
      b.ibox_pack.alloc(std::max<uint64_t>(p.I, 1));
    }
    TG_CK(cudaMemsetAsync(b.bc.get(), 0, Vn * 8, s));
    TG_CK(cudaMemsetAsync(p.fs.counters.get() + 4, 0, 8, s));  // sigma >= 2^53 flag
  }
  eng.launches = 0;
  eng.comm_bytes = 0;
  double total_ms = 0;
  const DirectionPolicy dir = direction_policy(eng);
  // hub targets privatized per CTA in the backward push (TG_BC_PRIV, 0 = off)
  // pull-sigma by in-degree class (TG_BC_PULL_CLASSES=0: thread per vertex)
  const bool pull_classes =
      !(std::getenv("TG_BC_PULL_CLASSES") && std::getenv("TG_BC_PULL_CLASSES")[0] == '0');
  uint32_t bc_priv = 512;  // RMAT-28 sweep: profiles/r01_bc_priv_sweep.txt
  if (const char* e = std::getenv("TG_BC_PRIV")) bc_priv = (uint32_t)std::strtoul(e, nullptr, 10);
  // backward push: the top `bc_hub` local ids (highest out-degree) are pulled
  // instead (TG_BC_HUBPULL)
  uint32_t bc_hub = 0;  // A/B: profiles/r02_bc_hubpull_ab.txt (a CTA per hub row serializes 2M-edge rows)
  if (const char* e = std::getenv("TG_BC_HUBPULL")) bc_hub = (uint32_t)std::strtoul(e, nullptr, 10);
  uint64_t supersteps = 0, traversed = 0, bytes = 0, bm_bytes = 0, relax = 0;
  for (auto& pp : eng.parts) bm_bytes += words_for(pp->Vp) * 4;
  for (int si = 0; si < k; ++si) {
    int ps;
    uint32_t ls;
    eng.locate(sources[si], &ps, &ls);
    if (eng.P == 1) eng.l2_window(eng.parts[0]->bcs.sigma.get(), eng.parts[0]->Vp * 8);
    time_begin(eng);
    // the init advance below accumulates F[0]'s count and degree sums into the
    // vote counters: start them from zero (they hold the previous run's values)
    reset_vote(eng);
    // ---------------- forward cycle ----------------
    eng.each_part([&](Part& p) {
      cudaStream_t s = eng.stream;
      FrontierState& f = p.fs;
      BCState& b = p.bcs;
      const uint64_t nw = words_for(p.Vp);
      TG_CK(cudaMemsetAsync(b.sigma.get(), 0, p.Vp * 8, s));
      TG_CK(cudaMemsetAsync(b.dsum.get(), 0, p.Vp * 8, s));
      TG_CK(cudaMemsetAsync(f.visited.get(), 0, nw * 4, s));
      uint32_t* F0 = level_bitmap(p, 0);
      TG_CK(cudaMemsetAsync(F0, 0, nw * 4, s));
      if (p.S) {
        TG_CK(cudaMemsetAsync(f.obox_mark.get(), 0, p.S / 8, s));
        TG_CK(cudaMemsetAsync(f.obox_new.get(), 0, p.S / 8, s));
        TG_CK(cudaMemsetAsync(b.obox_sigma.get(), 0, p.S * 8, s));
      }
      // fused: inbox sigma sums start at 0 (peers write only after the vote below)
      if (eng.fused && p.I) TG_CK(cudaMemsetAsync(p.arena_fwd.get(), 0, p.I * 8, s));
      if (p.id == ps) {
        k_bc_seed<<<1, 1, 0, s>>>(F0, ls, b.sigma.get());
        eng.launches++;
      }
      launch_advance(eng, p, p.ts, F0, nullptr, f.visited.get(), nullptr, 0, f.counters.get(),
                     f.counters.get() + 2, f.counters.get() + 3);
    });
    uint32_t maxL = 0;
    uint64_t reached = 1;
    std::vector<uint64_t> lvl_count{1};  // |F[L]|
    const Vote v0 = read_vote(eng);
    uint64_t mf = v0.degsum, explored = mf;
    std::vector<uint64_t> lvl_out{v0.degsum}, lvl_in{v0.indegsum};  // degree sums of F[L]
    bool was_pull = false;
    for (uint32_t L = 0;; ++L) {
      reset_vote(eng);
      const bool pull = dir.bottom_up(eng, lvl_count[L], mf, eng.E - std::min(explored, eng.E),
                                      was_pull, dir.bc_alpha);
      was_pull = pull;
      if (pull && eng.P > 1) {
        // sigma of every published source in F[L] (0 otherwise) -> peers' ghosts
        eng.prof_begin(TG_K_EXCHANGE);
        eng.each_part([&](Part& p) {
          publish_frontier_sigma(eng, p, p.bcs.level_bm[L].get(), p.bcs.sigma.get());
        });
        fused_arrival(eng);
        eng.prof_end(TG_K_EXCHANGE);
      }
      eng.each_part([&](Part& p) {
        cudaStream_t s = eng.stream;
        FrontierState& f = p.fs;
        BCState& b = p.bcs;
        uint32_t* next = level_bitmap(p, L + 1);
        TG_CK(cudaMemsetAsync(next, 0, words_for(p.Vp) * 4, s));
        launch_compact(eng, p.ts);
        // class kernels when the unexplored edges (~ the pull's work) are a
        // large share; otherwise the per-word kernel's cheaper full scan wins
        const bool dense = (eng.E - std::min(explored, eng.E)) * 16 > eng.E;
        const bool gh = eng.P > 1;  // ghost in-CSR (remote in-neighbours)
        if (pull && pull_classes && dense) {
          // rows by in-degree class on fork/join streams (disjoint rows)
          PullSigma o{gh ? p.gh.off.get() : p.in_off.get(), gh ? p.gh.col.get() : p.in_col.get(),
                      b.level_bm[L].get(), f.visited.get(), gh ? p.gh.nz.get() : p.in_nz.get(),
                      b.sigma.get(), next, f.counters.get() + 1,
                      gh ? p.gh.sigma.get() : nullptr, (uint32_t)p.Vp};
          const uint64_t n_cta = gh ? p.gh.n_cta : p.n_cta, n_warp = gh ? p.gh.n_warp : p.n_warp;
          eng.prof_begin(TG_K_BCF_EXPAND);
          eng.fork();
          if (n_cta) {
            k_bc_pull_cta<<<(unsigned)n_cta, 256, 0, eng.side[0]>>>(
                o, gh ? p.gh.cta.get() : p.pr_cta.get());
            eng.launches++;
          }
          if (n_warp) {
            k_bc_pull_warp<<<grid_for(n_warp * 32, 256, 148u * 16u), 256, 0, eng.side[1]>>>(
                o, gh ? p.gh.warp.get() : p.pr_warp.get(), n_warp);
            eng.launches++;
          }
          k_bc_pull_thread<<<grid_for(p.Vp, 256, 148u * 16u), 256, 0, s>>>(o, p.Vp);
          eng.launches++;
          eng.join();
          eng.prof_end(TG_K_BCF_EXPAND);
          TG_CK(cudaGetLastError());
        } else if (pull) {
          eng.prof_begin(TG_K_BCF_EXPAND);
          k_bc_pull<<<grid_for(words_for(p.Vp) * 32, 256, 148u * 16u), 256, 0, s>>>(
              gh ? p.gh.off.get() : p.in_off.get(), gh ? p.gh.col.get() : p.in_col.get(),
              b.level_bm[L].get(), f.visited.get(), b.sigma.get(), next, p.Vp,
              f.counters.get() + 1, gh ? p.gh.sigma.get() : nullptr);
          eng.prof_end(TG_K_BCF_EXPAND);
          TG_CK(cudaGetLastError());
          eng.launches++;
        } else {
          BcFwdOp op{p.col.get(), f.visited.get(), next, b.sigma.get(), f.obox_mark.get(),
                     f.obox_new.get(), b.obox_sigma.get(), p.rout(), eng.fused};
          launch_expand(eng, p, p.ts, b.level_bm[L].get(), op, TG_K_BCF_EXPAND,
                        f.counters.get() + 1);
        }
      });
      supersteps++;
      if (eng.P > 1 && !pull) {  // a pull step only sets owned vertices: no messages
        eng.prof_begin(TG_K_EXCHANGE);
        if (eng.fused) {
          fused_arrival(eng);
          for (auto& pp : eng.parts) eng.comm_bytes += pp->S * 8;
        } else {
          exchange(eng, send_osigma, recv_isigma, 8, false);
        }
        eng.each_part([&](Part& p) {
          cudaStream_t s = eng.stream;
          FrontierState& f = p.fs;
          BCState& b = p.bcs;
          if (p.S) {
            k_or_clear<<<grid_for(p.S / 32, 256), 256, 0, s>>>(f.obox_mark.get(), f.obox_new.get(),
                                                               p.S / 32);
            if (!eng.fused) TG_CK(cudaMemsetAsync(b.obox_sigma.get(), 0, p.S * 8, s));
            eng.launches++;
          }
          if (p.I) {
            k_bc_scatter<<<grid_for(p.I, 256), 256, 0, s>>>(
                reinterpret_cast<const double*>(p.arena_fwd.get()), p.ibox_lid.get(), p.I,
                                                            f.visited.get(), b.sigma.get(),
                                                            b.level_bm[L + 1].get());
            eng.launches++;
            // fused: consumed; zero for the next superstep (peers write after the vote)
            if (eng.fused) TG_CK(cudaMemsetAsync(p.arena_fwd.get(), 0, p.I * 8, s));
          }
          TG_CK(cudaGetLastError());
        });
        eng.prof_end(TG_K_EXCHANGE);
      }
      eng.each_part([&](Part& p) {
        cudaStream_t s = eng.stream;
        FrontierState& f = p.fs;
        launch_advance(eng, p, p.ts, p.bcs.level_bm[L + 1].get(), nullptr, f.visited.get(), nullptr,
                       0, f.counters.get(), f.counters.get() + 2, f.counters.get() + 3);
      });
      const Vote v = read_vote(eng);
      relax += v.edges;
      mf = v.degsum;
      explored += mf;
      lvl_out.push_back(v.degsum);
      lvl_in.push_back(v.indegsum);
      if (dir.trace)
        std::fprintf(stderr, "[tg bc] L=%u %s frontier=%llu edges=%llu next=%llu ms=%.3f\n", L,
                     pull ? "pull" : "push", (unsigned long long)lvl_count[L],
                     (unsigned long long)v.edges, (unsigned long long)v.count, dir.lap(s));
      // push: col 4 per edge; offsets 16 + sigma[v] 8 per frontier vertex;
      // sigma[t] 8 per newly reached vertex; 3 bitmap passes.  pull: in_col 4
      // per examined in-edge; in-offsets 16 per unvisited vertex; sigma 8 per
      // newly reached vertex; 3 bitmap passes
      if (pull)
        eng.prof_bytes(TG_K_BCF_EXPAND, 4.0 * v.edges + 16.0 * (eng.V - reached) + 8.0 * v.count +
                                            3.0 * bm_bytes);
      else
        eng.prof_bytes(TG_K_BCF_EXPAND,
                       4.0 * v.edges + 24.0 * lvl_count[L] + 8.0 * v.count + 3.0 * bm_bytes);
      reached += v.count;
      lvl_count.push_back(v.count);
      if (v.count == 0) {
        maxL = L;  // F[L+1] is empty
        break;
      }
      TG_REQUIRE(L <= eng.V, TG_EINTERNAL, "tg_bc: superstep bound exceeded");
    }
    // ---------------- backward cycle ----------------
    if (eng.P == 1) eng.l2_window(eng.parts[0]->bcs.c.get(), eng.parts[0]->Vp * 8);
    reset_vote(eng);  // counters[1] accumulates the backward edges
    for (uint32_t L = maxL; L >= 1; --L) {
      if (L < maxL) {
        if (eng.P > 1) {
          eng.each_part([&](Part& p) {
            cudaStream_t s = eng.stream;
            if (!p.I) return;
            k_bc_pack<<<grid_for(p.I, 256), 256, 0, s>>>(
                p.ibox_lid.get(), p.I, p.bcs.level_bm[L + 1].get(), p.bcs.c.get(),
                eng.fused ? nullptr : p.bcs.ibox_pack.get(), p.rin(), (int)(L & 1));
            eng.launches++;
          });
          TG_CK(cudaGetLastError());
          // fused: the owners stored c into the referencing partitions' ghost
          // slots (buffer L & 1); one arrival barrier, and the next level writes
          // the other buffer, whose readers finished before this barrier
          if (eng.fused) {
            fused_arrival(eng);
            for (auto& pp : eng.parts) eng.comm_bytes += pp->I * 8;
          } else {
            exchange(eng, send_pack, recv_ghost, 8, true);
          }
        }
        // direction per level: pull over the out-edges of F[L] (cost ~ their
        // count) or push c[w] over the in-edges of F[L+1] (fp64 atomics, ~2x
        // per edge) -- whichever touches fewer edges
        // (P > 1: over every in-CSR row -- the outbox rows carry the edges into
        // remote successors, whose c the owners just published into the ghosts)
        const bool push = dir.mode != 1 && pull_ready(eng) &&
                          (eng.P == 1 ? eng.parts[0]->in_ntiles > 0 : true) &&
                          (dir.mode == 2 || 2 * lvl_in[L + 1] < lvl_out[L]);
        eng.each_part([&](Part& p) {
          cudaStream_t s = eng.stream;
          const uint32_t hub = push ? (uint32_t)std::min<uint64_t>(bc_hub, p.nz_end) : 0u;
          if (hub) {  // hub rows of F[L]: pull over their out-edges (CTA per row)
            const double* ghost = reinterpret_cast<const double*>(p.arena_rev.get());
            PullDelta o{p.row_off.get(), p.col.get(), p.bcs.level_bm[L].get(),
                        p.bcs.level_bm[L + 1].get(), p.bcs.c.get(),
                        eng.fused ? ghost + (L & 1) : ghost, eng.fused ? 2u : 1u,
                        p.bcs.dsum.get(), p.fs.counters.get() + 1};
            eng.prof_begin(TG_K_BCB_EXPAND);
            k_bc_bwd_cta<<<grid_for(hub, 1, 148u * 8u), 256, 0, s>>>(o, hub);
            eng.prof_end(TG_K_BCB_EXPAND);
            TG_CK(cudaGetLastError());
            eng.launches++;
          }
          const uint32_t priv = (uint32_t)std::min<uint64_t>(bc_priv, p.Vp - std::min<uint64_t>(hub, p.Vp));
          if (push && eng.P > 1) {
            if (!p.in_all_ntiles) return;
            const uint64_t R = p.Vp + p.S;
            if (p.bcs.ext.n < words_for(R)) p.bcs.ext.alloc(words_for(R));
            const double* ghost = reinterpret_cast<const double*>(p.arena_rev.get());
            const double* gh = eng.fused ? ghost + (L & 1) : ghost;
            const uint32_t gs = eng.fused ? 2u : 1u;
            k_bc_ext<<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(p.bcs.level_bm[L + 1].get(), p.Vp,
                                                                 gh, gs, R, p.bcs.ext.get());
            TG_CK(cudaGetLastError());
            eng.launches++;
            launch_mark_tiles(eng, in_all_tiles(p), R, p.bcs.ext.get(), p.ts_in);
            launch_compact(eng, p.ts_in);
            BcBwdPushOp op{p.in_col.get(), p.bcs.level_bm[L].get(), p.bcs.c.get(), p.bcs.dsum.get(),
                           priv, (uint32_t)p.Vp, gh, gs, hub};
            launch_expand_on(eng, in_all_tiles(p), p.ts_in, p.bcs.ext.get(), op, TG_K_BCB_EXPAND,
                             p.fs.counters.get() + 1);
          } else if (push) {
            launch_mark_tiles(eng, in_tiles(p), p.Vp, p.bcs.level_bm[L + 1].get(), p.ts_in);
            launch_compact(eng, p.ts_in);
            BcBwdPushOp op{p.in_col.get(), p.bcs.level_bm[L].get(), p.bcs.c.get(), p.bcs.dsum.get(),
                           priv, (uint32_t)p.Vp, nullptr, 1u, hub};
            launch_expand_on(eng, in_tiles(p), p.ts_in, p.bcs.level_bm[L + 1].get(), op,
                             TG_K_BCB_EXPAND, p.fs.counters.get() + 1);
          } else if (bwd_classes && lvl_out[L] * 16 > eng.E) {
            // dense level (F[L]'s out-edges > |E|/16): class kernels; sparse
            // levels keep the tile walker, which only visits active tiles
            if (!p.nz_end) return;
            const double* ghost = reinterpret_cast<const double*>(p.arena_rev.get());
            PullDelta o{p.row_off.get(), p.col.get(), p.bcs.level_bm[L].get(),
                        p.bcs.level_bm[L + 1].get(), p.bcs.c.get(),
                        eng.fused ? ghost + (L & 1) : ghost, eng.fused ? 2u : 1u,
                        p.bcs.dsum.get(), p.fs.counters.get() + 1};
            const uint64_t nb = p.bcs.n_big, nm = p.bcs.n_mid;
            eng.prof_begin(TG_K_BCB_EXPAND);
            eng.fork();
            if (nb) {
              k_bc_bwd_cta<<<grid_for(nb, 1, 148u * 8u), 256, 0, eng.side[0]>>>(o, nb);
              eng.launches++;
            }
            if (nm > nb) {
              k_bc_bwd_warp<<<grid_for((nm - nb) * 32, 256, 148u * 16u), 256, 0, eng.side[1]>>>(
                  o, nb, nm);
              eng.launches++;
            }
            if (p.nz_end > nm) {
              k_bc_bwd_thread<<<grid_for(p.nz_end - nm, 256, 148u * 16u), 256, 0, s>>>(o, nm,
                                                                                      p.nz_end);
              eng.launches++;
            }
            eng.join();
            eng.prof_end(TG_K_BCB_EXPAND);
            TG_CK(cudaGetLastError());
          } else {
            if (!p.ntiles) return;
            launch_mark_tiles(eng, out_tiles(p), p.Vp, p.bcs.level_bm[L].get(), p.ts);
            launch_compact(eng, p.ts);
            const double* ghost = reinterpret_cast<const double*>(p.arena_rev.get());
            BcBwdOp op{p.col.get(), p.bcs.level_bm[L + 1].get(), p.bcs.c.get(),
                       eng.fused ? ghost + (L & 1) : ghost, eng.fused ? 2u : 1u,
                       p.bcs.dsum.get()};
            launch_expand(eng, p, p.ts, p.bcs.level_bm[L].get(), op, TG_K_BCB_EXPAND,
                          p.fs.counters.get() + 1);
          }
        });
        if (dir.trace)
          std::fprintf(stderr, "[tg bc-bwd] L=%u %s out(F[L])=%llu in(F[L+1])=%llu ms=%.3f\n", L,
                       push ? "push" : "pull", (unsigned long long)lvl_out[L],
                       (unsigned long long)lvl_in[L + 1], dir.lap(s));
        // backward expand: c 8 per successor (read once); offsets 16 + dsum 8
        // per level-L vertex; level + successor bitmaps (+ 4 B per edge below)
        eng.prof_bytes(TG_K_BCB_EXPAND,
                       8.0 * lvl_count[L + 1] + 24.0 * lvl_count[L] + 2.0 * bm_bytes);
        supersteps++;
      }
      eng.each_part([&](Part& p) {
        cudaStream_t s = eng.stream;
        if (!p.Vp) return;
        k_bc_level<<<grid_for(words_for(p.Vp), 256, 148u * 16u), 256, 0, s>>>(
            p.bcs.level_bm[L].get(), p.Vp, p.nz_end, p.bcs.sigma.get(), p.bcs.dsum.get(),
            p.bcs.bc.get(), p.bcs.c.get(), p.fs.counters.get() + 4);
        TG_CK(cudaGetLastError());
        eng.launches++;
      });
    }
    total_ms += time_end(eng);
    eng.l2_window(nullptr, 0);
    const uint64_t bwd_edges = read_vote(eng).edges;
    relax += bwd_edges;
    eng.prof_bytes(TG_K_BCB_EXPAND, 4.0 * bwd_edges);
    // every reached vertex is in exactly one level: the levels' exact out-degree
    // sums give the reached out-degree total without another pass
    const uint64_t nreached = reached;
    uint64_t tr = 0;
    for (const uint64_t x : lvl_out) tr += x;
    traversed += 2 * tr;
    // forward: col 4 + visited probe 4 + sigma RMW 8 per edge; backward: col 4 +
    // successor probe 4 + c gather 8 per edge; per reached vertex offsets 16 x2,
    // sigma/dsum/bc/c 32
    bytes += 32 * tr + 64 * nreached;
  }
  TG_REQUIRE(read_counts(eng, 4) == 0, TG_EINTERNAL,
             "tg_bc: a shortest-path count reached 2^53 (no longer exact in fp64, reading A11)");
  if (st) {
    st->device_ms = total_ms;
    st->supersteps = supersteps;
    st->relaxations = relax;
    st->traversed_edges = traversed;
    st->algorithmic_bytes = bytes;
    st->comm_bytes = eng.comm_bytes;
    st->launches = eng.launches;
  }
  collect(eng, [](Part& p) -> const void* { return p.bcs.bc.get(); }, sizeof(double), out, mem);
}

}  // namespace tg
