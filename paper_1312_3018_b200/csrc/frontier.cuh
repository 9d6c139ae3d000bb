// frontier.cuh -- the load-balanced frontier machinery shared by BFS, SSSP and
// both BC phases (the compute phase of PAPER.md:200-208, Figs. 11/18/20).
//
// A superstep over partition p runs three kernels:
//   k_tile_compact : tile bitmap -> list of active edge tiles;
//   k_warp_expand  : persistent warps, one active tile at a time.  A tile is
//                    kTile consecutive edges of the out-CSR; the warp walks the
//                    rows the tile touches 32 at a time ("windows"): one
//                    broadcast load of the frontier word + a ballot gives the
//                    active rows, their tile-clipped lengths are prefix-summed
//                    with shuffles, and the flattened edges are processed 32 per
//                    step (consecutive edges -> coalesced column reads), lanes
//                    mapped to rows with one OR-reduce + popc + shuffle.  No
//                    shared memory, no block barriers.  Hubs span many tiles,
//                    so the work per warp is bounded by kTile edges whatever the
//                    degree skew (replaces the paper's thread-per-vertex kernel,
//                    P:857-867, and Kepler-era virtual warps);
//   k_advance      : next-frontier bitmap -> per-vertex state writes, visited,
//                    vote count and the tile bitmap of the next superstep.
#pragma once

#include <chrono>
#include <cstdlib>
#include <type_traits>

#include "engine.cuh"

namespace tg {

struct Empty {};
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

__device__ __forceinline__ Empty shfl_aux(Empty x, int) { return x; }
__device__ __forceinline__ uint32_t shfl_aux(uint32_t x, int l) { return __shfl_sync(kFull, x, l); }
__device__ __forceinline__ double shfl_aux(double x, int l) { return __shfl_sync(kFull, x, l); }

struct TileArgs {
  const uint64_t* row_off;
  const uint32_t* tile_vf;
  const uint32_t* tile_vl;
  const uint32_t* tile_list;
  const unsigned long long* tile_count;
  uint64_t Ep;
  const uint32_t* frontier;  // bitmap of active rows
  unsigned long long* edges; // += edges processed (one atomic per warp)
};

constexpr unsigned kExpandThreads = 256;

// Split (pipelined) edge ops: an Op with kSplit = true provides
//   Pre pre(uint64_t e)            -- the streamed loads of edge e (col, weight)
//   St  st(const Pre&)             -- the dependent gathers (target state words)
//   void fin(const Aux&, const Pre&, const St&)  -- compare + reductions
// and the walker runs U consecutive 32-edge steps per batch: U column loads in
// flight, then U gathers, then the reductions (memory-level parallelism for the
// latency-bound walk: ncu shows long-scoreboard stalls dominating).
// Block hooks: an Op with kBlockHooks = true owns `smem_bytes()` of dynamic
// shared memory per CTA and gets block_begin() before the first tile and
// block_end() after the last (e.g. per-CTA privatized accumulators of hub
// targets, flushed once per CTA).
template <class Op, class = void>
struct has_block_hooks {
  static constexpr bool value = false;
};
template <class Op>
struct has_block_hooks<Op, std::void_t<decltype(Op::kBlockHooks)>> {
  static constexpr bool value = Op::kBlockHooks;
};
template <class Op>
size_t smem_of(const Op& op) {
  if constexpr (has_block_hooks<Op>::value) return op.smem_bytes();
  else return 0;
}

template <class Op, class = void>
struct is_split {
  static constexpr bool value = false;
};
template <class Op>
struct is_split<Op, std::void_t<decltype(Op::kSplit)>> {
  static constexpr bool value = Op::kSplit;
};

// Persistent warps over the active tiles.  Op provides
//   using Aux; static constexpr bool kReduce, kFilter;
//   bool keep(uint32_t v, const Aux&) const; void defer(uint32_t v) const;  (kFilter)
//   Aux aux(uint32_t v) const;                                 // per active row
//   void edge(const Aux&, uint64_t e) const;                   (!kReduce)
//   double edge_val(uint64_t e) const;                         (kReduce)
//   void vertex_done(uint32_t v, double sum, bool whole_row) const;  (kReduce)
// Row-offset staging (north star: "shared-memory or TMA staging of row
// offsets"; kStage = 1): while a warp walks tile k, one lane has already
// issued a bulk async copy (cp.async.bulk, the TMA engine's 1-D form,
// completing on a per-warp mbarrier) of tile k+1's row offsets
// row_off[vf..vl+1] into a shared-memory double buffer, so the window loop
// reads its offsets from shared memory instead of waiting on global loads.
// Tiles spanning more than kStageRows rows fall back to global reads.
constexpr int kStageRows = 128;
struct StageSlot {
  uint64_t base;  // first staged row (even: 16-byte aligned source)
  bool on;
};
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// lane 0: arm the barrier with the byte count, then the bulk copy completes it
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <class Op, int U, int MB = 0, int kStage = 0>  // MB 0: no min-blocks bound
__global__ void __launch_bounds__(kExpandThreads, MB) k_warp_expand(TileArgs a, Op op) {
  using Aux = typename Op::Aux;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lowm = lane == 31 ? kFull : ((2u << lane) - 1u);
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned long long ntl = *a.tile_count;
  unsigned long long edges = 0;
  if constexpr (has_block_hooks<Op>::value) op.block_begin();
  __shared__ __align__(16) uint64_t s_ro[kStage ? kExpandThreads / 32 : 1][2][kStageRows + 2];
  __shared__ __align__(8) uint64_t s_bar[kStage ? kExpandThreads / 32 : 1][2];
  const uint32_t wib = kStage ? threadIdx.x >> 5 : 0;
  // two staging slots (scalars, not arrays: no local-memory indexing)
  StageSlot sl0{0, false}, sl1{0, false};
  uint32_t ph0 = 0, ph1 = 0;
  int buf = 0;
  // stage tile list entry `it` into buffer b (all lanes agree on the slot)
  auto stage = [&](uint64_t it, int b) {
    StageSlot st{0, false};
    if (it < ntl) {
      const uint32_t t = a.tile_list[it];
      const uint32_t vf = a.tile_vf[t], vl = a.tile_vl[t];
      const uint64_t base = vf & ~1u;
      const uint64_t n = ((uint64_t)vl + 2 - base + 1) & ~1ull;  // even count: 16-byte multiple
      if (n <= (uint64_t)kStageRows + 2) {
        st = {base, true};
        __syncwarp();  // every lane is done reading this buffer (previous tile)
        if (lane == 0)
          bulk_load(&s_ro[wib][b][0], a.row_off + base, (uint32_t)(n * 8), &s_bar[wib][b]);
      }
    }
    if (b) sl1 = st;
    else sl0 = st;
  };
  const uint64_t it0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  if constexpr (kStage != 0) {
    if (lane == 0) {
      mbar_init(&s_bar[wib][0]);
      mbar_init(&s_bar[wib][1]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    stage(it0, 0);
  }
  for (uint64_t it = it0; it < ntl; it += nwarps) {
    const uint32_t t = a.tile_list[it];
    const uint32_t vf = a.tile_vf[t], vl = a.tile_vl[t];
    const uint64_t e_lo = (uint64_t)t * kTile;
    const uint64_t e_hi = min(e_lo + (uint64_t)kTile, a.Ep);
    const uint64_t* ro = a.row_off;  // row offsets: global, or the staged window
    int64_t ro_shift = 0;
    if constexpr (kStage != 0) {
      stage(it + nwarps, buf ^ 1);  // the next tile's offsets, in flight during this one
      const StageSlot cs = buf ? sl1 : sl0;
      if (cs.on) {
        mbar_wait(&s_bar[wib][buf], buf ? ph1 : ph0);
        if (buf) ph1 ^= 1u;
        else ph0 ^= 1u;
        ro = &s_ro[wib][buf][0];
        ro_shift = (int64_t)cs.base;
      }
      buf ^= 1;
    }
    // the tile's frontier words, 32 windows per coalesced load: only windows
    // with an active row are walked (a sparse frontier spread over the id range
    // leaves most of a low-degree tile's ~16 windows empty)
    for (uint32_t wb = vf >> 5; wb <= (vl >> 5); wb += 32) {
      const uint32_t xw = wb + lane <= (vl >> 5) ? a.frontier[wb + lane] : 0u;
      uint32_t wmask = __ballot_sync(kFull, xw != 0u);
      while (wmask) {
      const uint32_t kw = (uint32_t)__ffs(wmask) - 1u;
      wmask &= wmask - 1u;
      const uint32_t wv = (wb + kw) << 5;
      const uint32_t x = __shfl_sync(kFull, xw, (int)kw);
      const uint32_t v = wv + lane;
      const bool act = ((x >> lane) & 1u) && v >= vf && v <= vl;
      if (!__ballot_sync(kFull, act)) continue;
      uint32_t len = 0;
      uint64_t b = 0;
      bool whole = false;
      Aux aux{};
      if (act) {
        aux = op.aux(v);
        if constexpr (Op::kFilter) {
          // scheduling filter (near-far SSSP): a deferred row stays active
          if (!op.keep(v, aux)) {
            op.defer(v);
            aux = Aux{};
          } else {
            const uint64_t rb = ro[v - ro_shift], re = ro[v + 1 - ro_shift];
            b = rb > e_lo ? rb : e_lo;
            const uint64_t en = re < e_hi ? re : e_hi;
            len = (uint32_t)(en - b);
            whole = (b == rb) && (en == re);
          }
        } else {
          const uint64_t rb = ro[v - ro_shift], re = ro[v + 1 - ro_shift];
          b = rb > e_lo ? rb : e_lo;
          const uint64_t en = re < e_hi ? re : e_hi;
          len = (uint32_t)(en - b);
          whole = (b == rb) && (en == re);
        }
      }
      const uint32_t incl = warp_incl_scan(len);
      const uint32_t T = __shfl_sync(kFull, incl, 31);
      const uint32_t excl = incl - len;
      const uint64_t basev = b - excl;  // edge of flattened index i in my row = basev + i
      const uint32_t lmask = __ballot_sync(kFull, len > 0);
      const uint32_t owner_of = __fns(lmask, 0, (int)lane + 1);  // lane of segment #lane
      double acc = 0.0;
      uint32_t s0 = 0;
      if constexpr (!Op::kReduce && is_split<Op>::value) {
        for (uint32_t c0 = 0; c0 < T; c0 += 32u * U) {
          Aux ax[U];
          uint64_t ee[U];
          bool ok[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t cc = c0 + 32u * u;
            const uint32_t flag = (len > 0 && excl > cc && excl < cc + 32) ? (1u << (excl - cc)) : 0u;
            const uint32_t starts = __reduce_or_sync(kFull, flag);
            const uint32_t s = s0 + __popc(starts & lowm);
            const uint32_t idx = cc + lane;
            ok[u] = idx < T;
            const uint32_t ow = __shfl_sync(kFull, owner_of, s & 31);
            ee[u] = __shfl_sync(kFull, basev, ow & 31) + idx;
            ax[u] = shfl_aux(aux, ow & 31);
            const uint32_t sl = __shfl_sync(kFull, s, 31);
            const uint32_t nb = __reduce_or_sync(kFull, (len > 0 && excl == cc + 32) ? 1u : 0u);
            s0 = sl + nb;
          }
          typename Op::Pre pr[U];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (ok[u]) pr[u] = op.pre(ee[u]);
          typename Op::St st[U];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (ok[u]) st[u] = op.st(pr[u]);
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (ok[u]) op.fin(ax[u], pr[u], st[u]);
        }
        edges += T;
        continue;
      }
      for (uint32_t c0 = 0; c0 < T; c0 += 32) {
        const uint32_t flag = (len > 0 && excl > c0 && excl < c0 + 32) ? (1u << (excl - c0)) : 0u;
        const uint32_t starts = __reduce_or_sync(kFull, flag);
        const uint32_t s = s0 + __popc(starts & lowm);
        const uint32_t idx = c0 + lane;
        const bool valid = idx < T;
        const uint32_t ow = __shfl_sync(kFull, owner_of, s & 31);
        const uint64_t bs = __shfl_sync(kFull, basev, ow & 31);
        if constexpr (!Op::kReduce) {
          if constexpr (!is_split<Op>::value) {  // split ops never reach this loop
            const Aux ax = shfl_aux(aux, ow & 31);
            if (valid) op.edge(ax, bs + idx);
          }
        } else {
          double val = valid ? op.edge_val(bs + idx) : 0.0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double vo = __shfl_up_sync(kFull, val, o);
            const uint32_t so = __shfl_up_sync(kFull, s, o);
            if (lane >= (uint32_t)o && so == s) val += vo;
          }
          int tail = -1;
          if (len > 0) {
            const uint32_t st = excl > c0 ? excl : c0;
            const uint32_t en = (excl + len) < (c0 + 32) ? (excl + len) : (c0 + 32);
            if (st < en) tail = (int)(en - 1 - c0);
          }
          const double got = __shfl_sync(kFull, val, tail < 0 ? 0 : tail);
          if (tail >= 0) acc += got;
        }
        const uint32_t sl = __shfl_sync(kFull, s, 31);
        const uint32_t nb = __reduce_or_sync(kFull, (len > 0 && excl == c0 + 32) ? 1u : 0u);
        s0 = sl + nb;
      }
      if constexpr (Op::kReduce) {
        if (len > 0) op.vertex_done(v, acc, whole);
      }
      edges += T;
      }  // windows with an active row
    }
  }
  if constexpr (kStage != 0) {  // drain a copy still in flight (issued past the last tile)
    if (buf ? sl1.on : sl0.on) mbar_wait(&s_bar[wib][buf], buf ? ph1 : ph0);
  }
  if (a.edges && lane == 0 && edges) atomicAdd(a.edges, edges);
  if constexpr (has_block_hooks<Op>::value) op.block_end();
}

// tile bitmap -> list (clears the bitmap)
__global__ void k_tile_compact(uint32_t* tile_bm, uint64_t nwords, uint32_t* list,
                               unsigned long long* count);

// next bitmap -> state; see frontier.cu
__global__ void k_advance(uint32_t* next, uint32_t* cur_old, uint32_t* visited, uint32_t* vals,
                          uint32_t level_val, uint64_t Vp, const uint64_t* row_off,
                          uint32_t* tile_bm, unsigned long long* count,
                          unsigned long long* degsum, const uint64_t* in_off,
                          unsigned long long* indegsum, const uint32_t* minvals,
                          unsigned long long* minout);

// mark the tiles touched by the rows set in `bm`
__global__ void k_mark_tiles(const uint32_t* bm, uint64_t Vp, const uint64_t* row_off,
                             uint32_t* tile_bm);

// set bit i of bm and (optionally) vals[i] = val
__global__ void k_seed(uint32_t* bm, uint32_t i, uint32_t* vals, uint32_t val);

// the pull directions need the ghost in-CSR when P > 1 (built outside the
// timed region, collective across processes)
inline bool pull_ready(const Engine& eng) {
  if (!eng.has_in) return false;
  for (auto& pp : eng.parts)
    if (eng.P > 1 && !pp->gh.built) return false;
  return true;
}

// Direction optimization (Beamer et al. 2013, cited at
// PAPER.md:767): switch top-down -> bottom-up when the frontier's out-edges m_f
// exceed (edges not yet explored m_u) / alpha, and back when the frontier holds
// fewer than V/beta vertices.  Engines with an in-CSR (P > 1: once the ghost
// in-CSR is built, pull_ready).
// Env overrides: TG_DIRECTION=top|bottom|auto, TG_BU_ALPHA (BFS, 14),
// TG_BC_ALPHA (BC pull-sigma, 2), TG_BU_BETA (24), TG_TRACE=1.
struct DirectionPolicy {
  int mode = 0;  // 0 auto, 1 top-down only, 2 always bottom-up
  double alpha = 14.0, bc_alpha = 2.0, beta = 24.0;
  bool trace = false;  // one stderr line per superstep
  // trace only: ms since the previous lap (synchronizes the stream)
  mutable std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  double lap(cudaStream_t s) const {
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(now - last).count();
    last = now;
    return ms;
  }
  bool bottom_up(const Engine& eng, uint64_t nf, uint64_t mf, uint64_t mu, bool was_bu,
                 double a) const {
    if (!pull_ready(eng) || mode == 1) return false;
    if (mode == 2) return true;
    if (was_bu) return (double)nf * beta > (double)eng.V;
    return (double)mf * a > (double)mu;
  }
};
DirectionPolicy direction_policy(const Engine& eng);

// Direction optimization across partitions: before a bottom-up BFS / pull-
// sigma superstep every partition publishes, for each source on its publish
// lists (PRGhost), its frontier bit (and sigma) into the peers' ghost slots;
// the pulls then read local sources from F and ghost v = Vp + g from
// gh.bits / gh.sigma.  One launch per partition covers every peer.  Across
// processes the stores go to CUDA-IPC-mapped peer memory; the caller runs the
// arrival barrier before any peer pulls.
void publish_frontier_bits(Engine& eng, Part& p, const uint32_t* F);
void publish_frontier_sigma(Engine& eng, Part& p, const uint32_t* F, const double* sigma);

// A CSR with its edge tiles: the out-CSR, or the in-CSR restricted to the
// local rows [0, Vp).
struct CsrTiles {
  const uint64_t* row_off;
  const uint32_t* vf;
  const uint32_t* vl;
  uint64_t ntiles, E;
};
inline CsrTiles out_tiles(const Part& p) {
  return {p.row_off.get(), p.tile_vf.get(), p.tile_vl.get(), p.ntiles, p.Ep};
}
inline CsrTiles in_tiles(const Part& p) {
  return {p.in_off.get(), p.in_tile_vf.get(), p.in_tile_vl.get(), p.in_ntiles, p.in_E_local};
}
// every in-CSR row [0, Vp + S): local rows, then the outbox rows (P > 1)
inline CsrTiles in_all_tiles(const Part& p) {
  return {p.in_off.get(), p.in_all_vf.get(), p.in_all_vl.get(), p.in_all_ntiles, p.Ep};
}

template <class Op>
void launch_expand_on(Engine& eng, const CsrTiles& c, TileSched& ts, const uint32_t* frontier,
                      const Op& op, int kid, unsigned long long* edges);

// launch helpers (frontier.cu)
void launch_compact(Engine& eng, TileSched& ts);
// degsum (nullable) += out-degree sum of the new frontier; indegsum (nullable)
// += its in-degree sum (needs the in-CSR)
void launch_advance(Engine& eng, Part& p, TileSched& ts, uint32_t* next, uint32_t* cur_old,
                    uint32_t* visited, uint32_t* vals, uint32_t level_val,
                    unsigned long long* count, unsigned long long* degsum = nullptr,
                    unsigned long long* indegsum = nullptr, const uint32_t* minvals = nullptr,
                    unsigned long long* minout = nullptr);
void launch_mark_tiles(Engine& eng, const CsrTiles& c, uint64_t Vp, const uint32_t* bm,
                       TileSched& ts);
unsigned expand_grid();

template <class Op>
void launch_expand(Engine& eng, Part& p, TileSched& ts, const uint32_t* frontier, const Op& op,
                   int kid, unsigned long long* edges) {
  launch_expand_on(eng, out_tiles(p), ts, frontier, op, kid, edges);
}

template <class Op, int U, int MB = 0, int S = 0>
void launch_walker_s(Engine& eng, const TileArgs& a, const Op& op) {
  // persistent grid = exactly the resident CTAs (static tile striding assumes residency)
  static int per_sm = 0;
  static size_t per_sm_smem = ~(size_t)0;
  const size_t smem = smem_of(op);
  if (!per_sm || smem != per_sm_smem) {
    if (smem > 48 * 1024)
      TG_CK(cudaFuncSetAttribute(k_warp_expand<Op, U, MB, S>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_warp_expand<Op, U, MB, S>,
                                                        kExpandThreads, smem));
    if (per_sm < 1) per_sm = 1;
    per_sm_smem = smem;
  }
  k_warp_expand<Op, U, MB, S><<<expand_grid() / 8u * (unsigned)per_sm, kExpandThreads, smem,
                                eng.stream>>>(a, op);
}
// TG_STAGE_ROWOFF=1: the row-offset staging variant (kStage = 1)
bool stage_rowoff();
template <class Op, int U, int MB = 0>
void launch_walker(Engine& eng, const TileArgs& a, const Op& op) {
  if (stage_rowoff()) launch_walker_s<Op, U, MB, 1>(eng, a, op);
  else launch_walker_s<Op, U, MB, 0>(eng, a, op);
}

template <class Op>
void launch_expand_on(Engine& eng, const CsrTiles& c, TileSched& ts, const uint32_t* frontier,
                      const Op& op, int kid, unsigned long long* edges) {
  if (!c.ntiles) return;
  TileArgs a{c.row_off, c.vf, c.vl, ts.list.get(), ts.count.get(), c.E, frontier, edges};
  eng.prof_begin(kid);
  if constexpr (is_split<Op>::value) {
    // 32-edge steps per batch of the split walker: Op::kUnroll (RMAT-28 sweep,
    // profiles/r01_walker_unroll.txt), TG_UNROLL=1|2|4|8 overrides
    static int unroll = 0;
    if (!unroll) {
      const char* u = std::getenv("TG_UNROLL");
      unroll = u ? std::atoi(u) : Op::kUnroll;
    }
    // TG_WALK_MINB (experiment): __launch_bounds__ min blocks 5 / 6 caps the
    // registers (48 / 40) for more resident warps
    static int minb = -1;
    if (minb < 0) {
      const char* m = std::getenv("TG_WALK_MINB");
      minb = m ? std::atoi(m) : 0;
    }
    if (minb == 5 && unroll == 4) launch_walker<Op, 4, 5>(eng, a, op);
    else if (minb == 6 && unroll == 4) launch_walker<Op, 4, 6>(eng, a, op);
    else if (minb == 5 && unroll == 2) launch_walker<Op, 2, 5>(eng, a, op);
    else if (unroll == 1) launch_walker<Op, 1>(eng, a, op);
    else if (unroll == 3) launch_walker<Op, 3>(eng, a, op);
    else if (unroll == 4) launch_walker<Op, 4>(eng, a, op);
    else if (unroll == 8) launch_walker<Op, 8>(eng, a, op);
    else launch_walker<Op, 2>(eng, a, op);
  } else {
    launch_walker<Op, 1>(eng, a, op);
  }
  eng.prof_end(kid);
  TG_CK(cudaGetLastError());
  eng.launches++;
}

}  // namespace tg
