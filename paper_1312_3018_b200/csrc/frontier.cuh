// frontier.cuh -- the load-balanced frontier machinery shared by BFS, SSSP and
// both BC phases (the compute phase of PAPER.md:200-208, Figs. 11/18/20).
//
// A superstep over partition p runs three kernels:
//   k_tile_compact : tile bitmap -> list of active edge tiles;
//   k_tile_expand  : one persistent CTA loop over the active tiles.  A tile is
//                    kTile consecutive edges of the out-CSR; its CTA finds the
//                    frontier vertices among the rows it touches (bitmap words
//                    + popc), clips their rows to the tile, prefix-sums the
//                    clipped lengths in shared memory and walks the flattened
//                    edge list warp by warp (32 consecutive edges per step, so
//                    column reads are coalesced), mapping lanes to rows with one
//                    ballot-style OR-reduce + popc per step.  Hubs simply span
//                    many tiles, so the work per CTA is bounded by kTile edges
//                    whatever the degree skew (replaces the paper's
//                    thread-per-vertex kernel, and virtual warps);
//   k_advance      : next-frontier bitmap -> per-vertex state writes, visited,
//                    vote count and the tile bitmap of the next superstep.
#pragma once

#include "engine.cuh"

namespace tg {

struct Empty {};

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Block exclusive scan for blockDim.x == NT (multiple of 32, <= 1024).
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* s_warp, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t incl = warp_incl_scan(x);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < NT / 32 ? s_warp[lane] : 0u;
    const uint32_t vi = warp_incl_scan(v);
    if (lane < NT / 32) s_warp[lane] = vi - v;
    if (lane == NT / 32 - 1) s_warp[NT / 32] = vi;
  }
  __syncthreads();
  const uint32_t r = s_warp[warp] + incl - x;
  *total = s_warp[NT / 32];
  return r;
}

struct TileArgs {
  const uint64_t* row_off;
  const uint32_t* tile_vf;
  const uint32_t* tile_vl;
  const uint32_t* tile_list;
  const unsigned long long* tile_count;
  uint64_t Ep;
  const uint32_t* frontier;  // bitmap of active rows
  unsigned long long* edges; // += edges processed (one atomic per tile)
};

template <class Op>
struct TileSmem {
  uint32_t act[kTile];
  int32_t base[kTile];
  uint32_t pre[kTile + 1];
  typename Op::Aux aux[kTile];
  double acc[Op::kReduce ? kTile : 1];
  uint32_t word[72];
  uint32_t woff[72];
  uint32_t scan[kTileThreads / 32 + 1];
  uint32_t A;
};

// Persistent CTA loop over the active tiles.  Op provides
//   using Aux; static constexpr bool kReduce;
//   Aux aux(uint32_t v) const;                       // per active vertex
//   void edge(uint32_t v, const Aux&, uint64_t e) const;          (!kReduce)
//   double edge_val(uint32_t v, const Aux&, uint64_t e) const;     (kReduce)
//   void vertex_done(uint32_t v, const Aux&, double acc, bool whole_row) const;
template <class Op>
__global__ void __launch_bounds__(kTileThreads) k_tile_expand(TileArgs a, Op op) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem<Op>& S = *reinterpret_cast<TileSmem<Op>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long ntl = *a.tile_count;
  for (unsigned long long it = blockIdx.x; it < ntl; it += gridDim.x) {
    const uint32_t t = a.tile_list[it];
    const uint32_t vf = a.tile_vf[t], vl = a.tile_vl[t];
    const uint64_t e_lo = (uint64_t)t * kTile;
    const uint64_t e_hi = min(e_lo + (uint64_t)kTile, a.Ep);
    const uint32_t w0 = vf >> 5, nw = (vl >> 5) - w0 + 1;  // <= 65
    const uint32_t nv = vl - vf + 1;                        // <= kTile
    // 1. masked frontier words of the rows [vf, vl] and their popc offsets
    if (warp == 0) {
      uint32_t wv[3], cnt = 0;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const uint32_t i = 3 * lane + j;
        uint32_t x = 0;
        if (i < nw) {
          x = a.frontier[w0 + i];
          if (i == 0) x &= ~0u << (vf & 31);
          if (i == nw - 1) x &= ((vl & 31) == 31) ? ~0u : ((2u << (vl & 31)) - 1u);
        }
        wv[j] = x;
        cnt += __popc(x);
      }
      const uint32_t incl = warp_incl_scan(cnt);
      uint32_t ex = incl - cnt;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const uint32_t i = 3 * lane + j;
        if (i < nw) {
          S.word[i] = wv[j];
          S.woff[i] = ex;
          ex += __popc(wv[j]);
        }
      }
      if (lane == 31) S.A = incl;
    }
    __syncthreads();
    const uint32_t A = S.A;
    if (A == 0) {
      __syncthreads();
      continue;
    }
    // 2. compaction of the active rows (in row order)
    for (uint32_t j = tid; j < nv; j += kTileThreads) {
      const uint32_t v = vf + j, i = (v >> 5) - w0, x = S.word[i], b = v & 31;
      if ((x >> b) & 1u) S.act[S.woff[i] + __popc(x & ((1u << b) - 1u))] = v;
    }
    __syncthreads();
    // 3. clipped row ranges, per-vertex aux, exclusive prefix of lengths (blocked: 4 per thread)
    uint32_t len[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t k = 4 * tid + q;
      len[q] = 0;
      if (k < A) {
        const uint32_t v = S.act[k];
        const uint64_t rb = a.row_off[v], re = a.row_off[v + 1];
        const uint64_t b = rb > e_lo ? rb : e_lo, en = re < e_hi ? re : e_hi;
        len[q] = (uint32_t)(en - b);
        S.base[k] = (int32_t)(b - e_lo);
        S.aux[k] = op.aux(v);
        if (Op::kReduce) S.acc[k] = 0.0;
      }
      sum += len[q];
    }
    uint32_t W;
    uint32_t ex = block_excl_scan<kTileThreads>(sum, S.scan, &W);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t k = 4 * tid + q;
      if (k < A) {
        S.pre[k] = ex;
        S.base[k] -= (int32_t)ex;
        ex += len[q];
      }
    }
    if (tid == 0) {
      S.pre[A] = W;
      if (a.edges) atomicAdd(a.edges, (unsigned long long)W);
    }
    __syncthreads();
    // 4. warp w walks flattened edges [j0, j1) in 32-edge steps
    {
      constexpr uint32_t NW = kTileThreads / 32;
      const uint32_t per = ((W + NW - 1) / NW + 31) & ~31u;
      const uint32_t j0 = warp * per, j1 = min(j0 + per, W);
      if (j0 < j1) {
        // k_a = largest k with pre[k] <= j0
        uint32_t lo = 0, hi = A - 1;
        while (lo < hi) {
          const uint32_t m = (lo + hi + 1) >> 1;
          if (S.pre[m] <= j0) lo = m;
          else hi = m - 1;
        }
        uint32_t ka = lo;
        for (uint32_t c0 = j0; c0 < j1; c0 += 32) {
          const uint32_t kc = ka + 1 + lane;
          const uint32_t bnd = kc < A ? S.pre[kc] - c0 : 0xFFFFFFFFu;
          const uint32_t flag = (bnd >= 1 && bnd < 32) ? (1u << bnd) : 0u;
          const uint32_t mask = __reduce_or_sync(0xffffffffu, flag);
          const uint32_t lowm = lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u);
          const uint32_t k = ka + __popc(mask & lowm);
          const uint32_t idx = c0 + lane;
          const bool valid = idx < j1;
          if constexpr (!Op::kReduce) {
            if (valid) op.edge(S.act[k], S.aux[k], e_lo + (uint64_t)(S.base[k] + (int32_t)idx));
          } else {
            double val = valid ? op.edge_val(S.act[k], S.aux[k],
                                             e_lo + (uint64_t)(S.base[k] + (int32_t)idx))
                               : 0.0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const double vo = __shfl_up_sync(0xffffffffu, val, o);
              const uint32_t ko = __shfl_up_sync(0xffffffffu, k, o);
              if (lane >= o && ko == k) val += vo;
            }
            const uint32_t kn = __shfl_down_sync(0xffffffffu, k, 1);
            const bool tail = (lane == 31) || (kn != k) || (idx + 1 >= j1);
            if (valid && tail) atomicAdd(&S.acc[k], val);
          }
          uint32_t kl = __shfl_sync(0xffffffffu, k, 31);
          if (kl + 1 < A && S.pre[kl + 1] <= c0 + 32) kl++;
          ka = kl;
        }
      }
    }
    __syncthreads();
    if constexpr (Op::kReduce) {
      for (uint32_t k = tid; k < A; k += kTileThreads) {
        const uint32_t v = S.act[k];
        const uint32_t L = S.pre[k + 1] - S.pre[k];
        const bool whole = (a.row_off[v + 1] - a.row_off[v]) == L;
        op.vertex_done(v, S.aux[k], S.acc[k], whole);
      }
      __syncthreads();
    }
  }
}

// tile bitmap -> list (clears the bitmap)
__global__ void k_tile_compact(uint32_t* tile_bm, uint64_t nwords, uint32_t* list,
                               unsigned long long* count);

// next bitmap -> state; see frontier.cu
__global__ void k_advance(uint32_t* next, uint32_t* cur_old, uint32_t* visited, uint32_t* vals,
                          uint32_t level_val, uint64_t Vp, const uint64_t* row_off,
                          uint32_t* tile_bm, unsigned long long* count,
                          unsigned long long* degsum);

// mark the tiles touched by the rows set in `bm`
__global__ void k_mark_tiles(const uint32_t* bm, uint64_t Vp, const uint64_t* row_off,
                             uint32_t* tile_bm);

// set bit i of bm and (optionally) vals[i] = val
__global__ void k_seed(uint32_t* bm, uint32_t i, uint32_t* vals, uint32_t val);

// launch helpers (frontier.cu)
void launch_compact(Engine& eng, TileSched& ts);
void launch_advance(Engine& eng, Part& p, TileSched& ts, uint32_t* next, uint32_t* cur_old,
                    uint32_t* visited, uint32_t* vals, uint32_t level_val,
                    unsigned long long* count, unsigned long long* degsum = nullptr);
unsigned expand_grid();

template <class Op>
void launch_expand(Engine& eng, Part& p, TileSched& ts, const uint32_t* frontier, const Op& op,
                   int kid, unsigned long long* edges) {
  if (!p.ntiles) return;
  TileArgs a{p.row_off.get(), p.tile_vf.get(), p.tile_vl.get(), ts.list.get(), ts.count.get(),
             p.Ep, frontier, edges};
  const size_t smem = sizeof(TileSmem<Op>);
  static bool configured = false;
  if (!configured) {
    TG_CK(cudaFuncSetAttribute(k_tile_expand<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
    configured = true;
  }
  eng.prof_begin(kid);
  k_tile_expand<Op><<<expand_grid(), kTileThreads, smem, eng.stream>>>(a, op);
  eng.prof_end(kid);
  TG_CK(cudaGetLastError());
  eng.launches++;
}

}  // namespace tg
