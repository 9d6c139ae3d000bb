// frontier.cu -- tile scheduling and frontier advance kernels (see frontier.cuh).
#include <cstdlib>
#include <cstring>

#include "frontier.cuh"

namespace tg {

__global__ void k_tile_compact(uint32_t* tile_bm, uint64_t nwords, uint32_t* list,
                               unsigned long long* count) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  // each warp handles 32 consecutive words per step (one per lane)
  for (uint64_t base = gw * 32; base < nwords; base += nwarps * 32) {
    const uint64_t w = base + lane;
    uint32_t x = 0;
    if (w < nwords) {
      x = tile_bm[w];
      if (x) tile_bm[w] = 0;
    }
    const uint32_t c = __popc(x);
    const uint32_t incl = warp_incl_scan(c);
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    if (!tot) continue;
    unsigned long long b = 0;
    if (lane == 31) b = atomicAdd(count, (unsigned long long)tot);
    b = __shfl_sync(0xffffffffu, b, 31);
    uint32_t pos = (uint32_t)(b + incl - c);
    while (x) {
      const int bit = __ffs(x) - 1;
      x &= x - 1;
      list[pos++] = (uint32_t)(w * 32 + bit);
    }
  }
}

// set the tile bits of edges [row_off[r0], row_off[r1]) -- one atomicOr per
// 32 tiles
__device__ __forceinline__ void mark_tile_range(const uint64_t* row_off, uint64_t r0, uint64_t r1,
                                                uint32_t* tile_bm) {
  const uint64_t lo = row_off[r0], hi = row_off[r1];
  if (hi <= lo) return;
  const uint64_t t0 = lo / kTile, t1 = (hi - 1) / kTile;
  for (uint64_t t = t0; t <= t1;) {
    const uint64_t wbase = t & ~31ull;
    const uint64_t last = (t1 < wbase + 31) ? t1 : wbase + 31;
    const uint32_t hi_mask = (last - wbase == 31) ? 0xFFFFFFFFu : ((2u << (last - wbase)) - 1u);
    const uint32_t mask = hi_mask & (0xFFFFFFFFu << (t - wbase));
    atomicOr(&tile_bm[wbase >> 5], mask);
    t = wbase + 32;
  }
}

__device__ __forceinline__ void block_add(unsigned long long* dst, unsigned long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// One thread per bitmap word.
__global__ void k_advance(uint32_t* next, uint32_t* cur_old, uint32_t* visited, uint32_t* vals,
                          uint32_t level_val, uint64_t Vp, const uint64_t* row_off,
                          uint32_t* tile_bm, unsigned long long* count,
                          unsigned long long* degsum, const uint64_t* in_off,
                          unsigned long long* indegsum, const uint32_t* minvals,
                          unsigned long long* minout) {
  const uint64_t nwords = words_for(Vp);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long cnt = 0, dsum = 0, isum = 0, mn = ~0ull;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    uint32_t x = next[w];
    if (cur_old) cur_old[w] = 0;
    if (!x) continue;
    cnt += __popc(x);
    if (visited) visited[w] |= x;
    const uint64_t v0 = w * 32;
    const uint64_t v1 = (v0 + 32 < Vp) ? v0 + 32 : Vp;
    if (degsum) {  // exact out-degree sum of the new frontier (direction choice)
      if (x == 0xFFFFFFFFu) {
        dsum += row_off[v1] - row_off[v0];
      } else {
        uint32_t y = x;
        while (y) {
          const int b = __ffs(y) - 1;
          y &= y - 1;
          dsum += row_off[v0 + b + 1] - row_off[v0 + b];
        }
      }
    }
    if (minout) {  // smallest value over the new frontier (near-far SSSP)
      uint32_t y = x;
      while (y) {
        const int b = __ffs(y) - 1;
        y &= y - 1;
        const unsigned long long m = minvals[v0 + b];
        mn = m < mn ? m : mn;
      }
    }
    if (indegsum) {  // exact in-degree sum (BC backward direction choice)
      if (x == 0xFFFFFFFFu) {
        isum += in_off[v1] - in_off[v0];
      } else {
        uint32_t y = x;
        while (y) {
          const int b = __ffs(y) - 1;
          y &= y - 1;
          isum += in_off[v0 + b + 1] - in_off[v0 + b];
        }
      }
    }
    if (vals) {
      if (x == 0xFFFFFFFFu && v0 + 32 <= Vp) {
        uint4* p = reinterpret_cast<uint4*>(vals + v0);
        const uint4 q = make_uint4(level_val, level_val, level_val, level_val);
#pragma unroll
        for (int i = 0; i < 8; ++i) p[i] = q;
      } else {
        while (x) {
          const int b = __ffs(x) - 1;
          x &= x - 1;
          vals[v0 + b] = level_val;
        }
      }
    }
    mark_tile_range(row_off, v0, v1, tile_bm);
  }
  block_add(count, cnt);
  if (degsum) block_add(degsum, dsum);
  if (indegsum) block_add(indegsum, isum);
  if (minout) {
    for (int o = 16; o; o >>= 1) {
      const unsigned long long y = __shfl_down_sync(0xffffffffu, mn, o);
      mn = y < mn ? y : mn;
    }
    if ((threadIdx.x & 31) == 0 && mn != ~0ull) atomicMin(minout, mn);
  }
}

__global__ void k_mark_tiles(const uint32_t* bm, uint64_t Vp, const uint64_t* row_off,
                             uint32_t* tile_bm) {
  const uint64_t nwords = words_for(Vp);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    if (!bm[w]) continue;
    const uint64_t v0 = w * 32, v1 = (v0 + 32 < Vp) ? v0 + 32 : Vp;
    mark_tile_range(row_off, v0, v1, tile_bm);
  }
}

__global__ void k_seed(uint32_t* bm, uint32_t i, uint32_t* vals, uint32_t val) {
  bm[i >> 5] |= 1u << (i & 31);
  if (vals) vals[i] = val;
}

// warp per 32 published entries of one peer segment: ballot of the frontier
// bits -> one word of the peer's ghost bitmap (segments are 32-aligned there)
__global__ void k_pub_bits(const uint32_t* pub_lid, const uint64_t* pub_off, int P, int me,
                           const uint32_t* F, uint32_t* const* dst) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    const uint64_t o = pub_off[q], n = pub_off[q + 1] - o;
    for (uint64_t w = gw; w * 32 < n; w += nwarps) {
      const uint64_t k = w * 32 + lane;
      const bool b = k < n && bit_test(F, pub_lid[o + k]);
      const uint32_t m = __ballot_sync(0xffffffffu, b);
      if (lane == 0) dst[q][w] = m;
    }
  }
}

__global__ void k_pub_sigma(const uint32_t* pub_lid, const uint64_t* pub_off, int P, int me,
                            const uint32_t* F, const double* sigma, double* const* dst) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    const uint64_t o = pub_off[q], n = pub_off[q + 1] - o;
    for (uint64_t k = t; k < n; k += stride) {
      const uint32_t u = pub_lid[o + k];
      dst[q][k] = bit_test(F, u) ? sigma[u] : 0.0;
    }
  }
}

void publish_frontier_bits(Engine& eng, Part& p, const uint32_t* F) {
  const PRGhost& g = p.gh;
  const uint64_t n = g.pub_off.empty() ? 0 : g.pub_off[eng.P];
  if (!n) return;
  k_pub_bits<<<grid_for(n, 256, 148u * 16u), 256, 0, eng.stream>>>(
      g.pub_lid.get(), g.d_pub_off.get(), eng.P, p.id, F, g.d_bits_dst.get());
  TG_CK(cudaGetLastError());
  eng.launches++;
  eng.comm_bytes += n / 8;
}

void publish_frontier_sigma(Engine& eng, Part& p, const uint32_t* F, const double* sigma) {
  const PRGhost& g = p.gh;
  const uint64_t n = g.pub_off.empty() ? 0 : g.pub_off[eng.P];
  if (!n) return;
  k_pub_sigma<<<grid_for(n, 256, 148u * 16u), 256, 0, eng.stream>>>(
      g.pub_lid.get(), g.d_pub_off.get(), eng.P, p.id, F, sigma, g.d_sigma_dst.get());
  TG_CK(cudaGetLastError());
  eng.launches++;
  eng.comm_bytes += n * 8;
}

void TileSched::ensure(uint64_t ntiles) {
  const uint64_t nw = words_for(ntiles);
  if (list.n >= std::max<uint64_t>(ntiles, 1) && bm.n >= std::max<uint64_t>(nw, 1)) return;
  bm.alloc(std::max<uint64_t>(nw, 1));
  list.alloc(std::max<uint64_t>(ntiles, 1));
  count.alloc(1);
  nwords = nw;
  TG_CK(cudaMemset(bm.get(), 0, bm.bytes()));
}

DirectionPolicy direction_policy(const Engine&) {
  DirectionPolicy d;
  if (const char* m = std::getenv("TG_DIRECTION")) {
    if (!std::strcmp(m, "top")) d.mode = 1;
    else if (!std::strcmp(m, "bottom")) d.mode = 2;
  }
  if (const char* t = std::getenv("TG_TRACE")) d.trace = t[0] == '1';
  if (const char* v = std::getenv("TG_BU_ALPHA")) d.alpha = std::atof(v);
  if (const char* v = std::getenv("TG_BC_ALPHA")) d.bc_alpha = std::atof(v);
  if (const char* v = std::getenv("TG_BU_BETA")) d.beta = std::atof(v);
  return d;
}

bool stage_rowoff() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("TG_STAGE_ROWOFF");
    on = e && e[0] == '1';
  }
  return on != 0;
}

static int g_num_sms = 0;
unsigned expand_grid() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return (unsigned)g_num_sms * 8u;  // persistent: 8 resident CTAs of 256 threads per SM
}

void launch_compact(Engine& eng, TileSched& ts) {
  TG_CK(cudaMemsetAsync(ts.count.get(), 0, sizeof(unsigned long long), eng.stream));
  if (!ts.nwords) return;
  const unsigned blocks = grid_for(ts.nwords, 256, 148u * 8u);
  eng.prof_begin(TG_K_COMPACT);
  k_tile_compact<<<blocks, 256, 0, eng.stream>>>(ts.bm.get(), ts.nwords, ts.list.get(),
                                                 ts.count.get());
  eng.prof_end(TG_K_COMPACT);
  eng.prof_bytes(TG_K_COMPACT, 4.0 * ts.nwords);
  TG_CK(cudaGetLastError());
  eng.launches++;
}

void launch_mark_tiles(Engine& eng, const CsrTiles& c, uint64_t Vp, const uint32_t* bm,
                       TileSched& ts) {
  if (!c.ntiles || !Vp) return;
  k_mark_tiles<<<grid_for(words_for(Vp), 256, 148u * 16u), 256, 0, eng.stream>>>(
      bm, Vp, c.row_off, ts.bm.get());
  TG_CK(cudaGetLastError());
  eng.launches++;
}

void launch_advance(Engine& eng, Part& p, TileSched& ts, uint32_t* next, uint32_t* cur_old,
                    uint32_t* visited, uint32_t* vals, uint32_t level_val,
                    unsigned long long* count, unsigned long long* degsum,
                    unsigned long long* indegsum, const uint32_t* minvals,
                    unsigned long long* minout) {
  if (!p.Vp) return;
  const uint64_t nwords = words_for(p.Vp);
  const unsigned blocks = grid_for(nwords, 256, 148u * 16u);
  eng.prof_begin(TG_K_ADVANCE);
  k_advance<<<blocks, 256, 0, eng.stream>>>(next, cur_old, visited, vals, level_val, p.Vp,
                                            p.row_off.get(), ts.bm.get(), count, degsum,
                                            // P > 1: the ghost in-CSR counts remote in-edges too
                                            p.gh.built ? p.gh.off.get() : p.in_off.get(),
                                            p.has_in ? indegsum : nullptr,
                                            minvals, minvals ? minout : nullptr);
  eng.prof_end(TG_K_ADVANCE);
  // next read + cur_old clear + visited RMW, one pass each
  eng.prof_bytes(TG_K_ADVANCE, 4.0 * nwords * (1 + (cur_old ? 1 : 0) + (visited ? 2 : 0)));
  TG_CK(cudaGetLastError());
  eng.launches++;
}

}  // namespace tg
