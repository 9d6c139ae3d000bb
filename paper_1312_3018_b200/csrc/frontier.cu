// frontier.cu -- tile scheduling and frontier advance kernels (see frontier.cuh).
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

__device__ __forceinline__ void mark_tile_range(const uint64_t* row_off, uint64_t r0, uint64_t r1,
                                                uint32_t* tile_bm, int lane) {
  const uint64_t lo = row_off[r0], hi = row_off[r1];
  if (hi <= lo) return;
  const uint64_t t0 = lo / kTile, t1 = (hi - 1) / kTile;
  for (uint64_t t = t0 + lane; t <= t1; t += 32) atomicOr(&tile_bm[t >> 5], 1u << (t & 31));
}

// One warp per bitmap word; lane = bit.
__global__ void k_advance(uint32_t* next, uint32_t* cur_old, uint32_t* visited, uint32_t* vals,
                          uint32_t level_val, uint64_t Vp, const uint64_t* row_off,
                          uint32_t* tile_bm, unsigned long long* count,
                          unsigned long long* degsum) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t nwords = words_for(Vp);
  unsigned long long cnt = 0, dsum = 0;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += nwarps) {
    const uint32_t x = next[w];
    if (lane == 0 && cur_old) cur_old[w] = 0;
    if (!x) continue;
    const uint64_t v = w * 32 + lane;
    const bool set = (x >> lane) & 1u;
    if (vals && set) vals[v] = level_val;
    if (degsum) {
      unsigned long long dg = set ? row_off[v + 1] - row_off[v] : 0ull;
      for (int o = 16; o; o >>= 1) dg += __shfl_down_sync(0xffffffffu, dg, o);
      if (lane == 0) dsum += dg;
    }
    if (lane == 0) {
      if (visited) visited[w] |= x;
      cnt += __popc(x);
    }
    const uint64_t r1 = (w * 32 + 32 < Vp) ? w * 32 + 32 : Vp;
    mark_tile_range(row_off, w * 32, r1, tile_bm, lane);
  }
  if (lane == 0 && cnt) atomicAdd(count, cnt);
  if (lane == 0 && dsum) atomicAdd(degsum, dsum);
}

__global__ void k_mark_tiles(const uint32_t* bm, uint64_t Vp, const uint64_t* row_off,
                             uint32_t* tile_bm) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t nwords = words_for(Vp);
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += nwarps) {
    if (!bm[w]) continue;
    const uint64_t r1 = (w * 32 + 32 < Vp) ? w * 32 + 32 : Vp;
    mark_tile_range(row_off, w * 32, r1, tile_bm, lane);
  }
}

__global__ void k_seed(uint32_t* bm, uint32_t i, uint32_t* vals, uint32_t val) {
  bm[i >> 5] |= 1u << (i & 31);
  if (vals) vals[i] = val;
}

void TileSched::ensure(const Part& p) {
  const uint64_t nw = words_for(p.ntiles);
  if (list.n >= std::max<uint64_t>(p.ntiles, 1) && bm.n >= std::max<uint64_t>(nw, 1)) return;
  bm.alloc(std::max<uint64_t>(nw, 1));
  list.alloc(std::max<uint64_t>(p.ntiles, 1));
  count.alloc(1);
  nwords = nw;
  TG_CK(cudaMemset(bm.get(), 0, bm.bytes()));
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

void launch_advance(Engine& eng, Part& p, TileSched& ts, uint32_t* next, uint32_t* cur_old,
                    uint32_t* visited, uint32_t* vals, uint32_t level_val,
                    unsigned long long* count, unsigned long long* degsum) {
  if (!p.Vp) return;
  const uint64_t nwords = words_for(p.Vp);
  const unsigned blocks = grid_for(nwords * 32, 256, 148u * 16u);
  eng.prof_begin(TG_K_ADVANCE);
  k_advance<<<blocks, 256, 0, eng.stream>>>(next, cur_old, visited, vals, level_val, p.Vp,
                                            p.row_off.get(), ts.bm.get(), count, degsum);
  eng.prof_end(TG_K_ADVANCE);
  // next read + cur_old clear + visited RMW, one pass each
  eng.prof_bytes(TG_K_ADVANCE, 4.0 * nwords * (1 + (cur_old ? 1 : 0) + (visited ? 2 : 0)));
  TG_CK(cudaGetLastError());
  eng.launches++;
}

}  // namespace tg
