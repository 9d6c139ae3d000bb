// build.cu -- device-side CSR builder and degree-aware partitioner (untimed
// pre-processing).  Steps:
//   1. out-degrees of the edge stream (generated on the device from
//      inputs/tg_inputs.h, or uploaded);
//   2. degree order: stable radix sort of ~outdeg -> order[i], rank_of[g]
//      (§6.2 sorts by degree; ties by id, reading A23);
//   3. per partition p (serpentine deal of the order): local/remote row degrees,
//      the distinct remote targets (outbox slots, source-side reduction of
//      PAPER.md:168-182), out-CSR with local-before-remote rows and
//      kRemote|slot payloads for boundary edges, edge tiles;
//   4. optional PageRank in-CSR (rows sorted by in-degree; outbox rows appended);
//   5. inboxes = peers' outbox segments (symmetry).
// CUB is used for the V-sized sorts/scans of this untimed build only; no
// library code runs inside a timed algorithm.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "engine.cuh"
#include "tg_inputs.h"

namespace tg {

namespace {

struct EdgeGen {
  const uint32_t *src, *dst, *w;
  bool gen;
  tgin_rmat r;
  uint64_t wseed;
  __device__ __forceinline__ void get(uint64_t k, uint32_t& s, uint32_t& d) const {
    if (gen) {
      tgin_rmat_edge_g(&r, k, &s, &d);
    } else {
      s = src[k];
      d = dst[k];
    }
  }
  __device__ __forceinline__ uint32_t weight(uint64_t k) const {
    return gen ? tgin_weight(wseed, k) : (w ? w[k] : 1u);
  }
};

__device__ __forceinline__ void block_add_u64(unsigned long long* dst, unsigned long long v) {
  // warp reduce then one atomic per warp
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

__global__ void k_outdeg(EdgeGen g, uint64_t E, uint64_t V, uint32_t* outdeg,
                         unsigned long long* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < E; k += stride) {
    uint32_t s, d;
    g.get(k, s, d);
    if (s >= V || d >= V) {
      atomicAdd(bad, 1ull);
      continue;
    }
    atomicAdd(&outdeg[s], 1u);
  }
}

__global__ void k_neg_iota(const uint32_t* outdeg, uint64_t V, uint32_t* keys, uint32_t* vals) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V; v += stride) {
    keys[v] = ~outdeg[v];
    vals[v] = (uint32_t)v;
  }
}

__global__ void k_inverse(const uint32_t* order, uint64_t V, uint32_t* rank_of) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < V; i += stride)
    rank_of[order[i]] = (uint32_t)i;
}

__global__ void k_global_of(const uint32_t* order, uint64_t Vp, int p, int P, const uint32_t* outdeg,
                            uint32_t* global_of, unsigned long long* nz) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long cnt = 0;
  for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < Vp; l += stride) {
    const uint32_t g = order[undeal((uint32_t)l, p, P)];
    global_of[l] = g;
    cnt += outdeg[g] > 0;
  }
  block_add_u64(nz, cnt);
}

__global__ void k_gather_deg(const uint32_t* gof, const uint32_t* od, uint64_t n, uint32_t* o) {
  const uint64_t st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < n; l += st) o[l] = od[gof[l]];
}

// local / remote row degrees of partition p
__global__ void k_count(EdgeGen g, uint64_t E, const uint32_t* rank_of, int P, int p,
                        uint32_t* nloc, uint32_t* nrem, unsigned long long* nremote) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long cnt = 0;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < E; k += stride) {
    uint32_t s, d, ls, ld;
    int ps, pd;
    g.get(k, s, d);
    deal(rank_of[s], P, &ps, &ls);
    if (ps != p) continue;
    deal(rank_of[d], P, &pd, &ld);
    if (pd == p) {
      atomicAdd(&nloc[ls], 1u);
    } else {
      atomicAdd(&nrem[ls], 1u);
      cnt++;
    }
  }
  block_add_u64(nremote, cnt);
}

__global__ void k_collect_keys(EdgeGen g, uint64_t E, const uint32_t* rank_of, int P, int p,
                               unsigned long long* keys, unsigned long long* counter) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < E; k += stride) {
    uint32_t s, d, ls, ld;
    int ps, pd;
    g.get(k, s, d);
    deal(rank_of[s], P, &ps, &ls);
    if (ps != p) continue;
    deal(rank_of[d], P, &pd, &ld);
    if (pd == p) continue;
    keys[atomicAdd(counter, 1ull)] = ((unsigned long long)pd << 32) | ld;
  }
}

__global__ void k_deg64(const uint32_t* nloc, const uint32_t* nrem, uint64_t Vp, uint64_t* deg) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l <= Vp; l += stride)
    deg[l] = l < Vp ? (uint64_t)nloc[l] + (nrem ? nrem[l] : 0u) : 0ull;
}

__global__ void k_seg_count(const unsigned long long* ukeys, uint64_t n, unsigned long long* cnt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += stride)
    atomicAdd(&cnt[ukeys[u] >> 32], 1ull);
}

__global__ void k_place_slots(const unsigned long long* ukeys, uint64_t n, const uint64_t* ustart,
                              const uint64_t* poff, uint32_t* obox_rid) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += stride) {
    const unsigned long long key = ukeys[u];
    const uint32_t q = (uint32_t)(key >> 32);
    obox_rid[poff[q] + (u - ustart[q])] = (uint32_t)key;
  }
}

__device__ __forceinline__ uint64_t lower_bound_u64(const unsigned long long* a, uint64_t n,
                                                    unsigned long long x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t m = (lo + hi) >> 1;
    if (a[m] < x) lo = m + 1;
    else hi = m;
  }
  return lo;
}

__global__ void k_fill(EdgeGen g, uint64_t E, const uint32_t* rank_of, int P, int p,
                       const uint64_t* row_off, const uint32_t* nloc, uint32_t* cur_loc,
                       uint32_t* cur_rem, uint32_t* col, uint32_t* w, bool weighted,
                       const unsigned long long* ukeys, uint64_t nukeys, const uint64_t* ustart,
                       const uint64_t* poff) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < E; k += stride) {
    uint32_t s, d, ls, ld;
    int ps, pd;
    g.get(k, s, d);
    deal(rank_of[s], P, &ps, &ls);
    if (ps != p) continue;
    deal(rank_of[d], P, &pd, &ld);
    uint64_t pos;
    uint32_t val;
    if (pd == p) {
      pos = row_off[ls] + atomicAdd(&cur_loc[ls], 1u);
      val = ld;
    } else {
      pos = row_off[ls] + nloc[ls] + atomicAdd(&cur_rem[ls], 1u);
      const unsigned long long key = ((unsigned long long)pd << 32) | ld;
      const uint64_t u = lower_bound_u64(ukeys, nukeys, key);
      val = kRemote | (uint32_t)(poff[pd] + (u - ustart[pd]));
    }
    col[pos] = val;
    if (weighted) w[pos] = g.weight(k);
  }
}

__device__ __forceinline__ uint32_t row_of_edge(const uint64_t* row_off, uint64_t lo, uint64_t hi,
                                                uint64_t e) {
  // largest v in [lo, hi] with row_off[v] <= e
  while (lo < hi) {
    const uint64_t m = (lo + hi + 1) >> 1;
    if (row_off[m] <= e) lo = m;
    else hi = m - 1;
  }
  return (uint32_t)lo;
}

__global__ void k_tiles(const uint64_t* row_off, uint64_t Vp, uint64_t Ep, uint64_t ntiles,
                        uint32_t* vf, uint32_t* vl) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntiles; t += stride) {
    const uint64_t e0 = t * kTile;
    const uint64_t e1 = min(e0 + kTile, Ep) - 1;
    vf[t] = row_of_edge(row_off, 0, Vp - 1, e0);
    vl[t] = row_of_edge(row_off, 0, Vp - 1, e1);
  }
}

// ---- PageRank in-CSR ----
// Each thread walks edges via the tile metadata to find its source row.
__global__ void k_in_count(const uint64_t* row_off, const uint32_t* col, uint64_t Ep, uint64_t Vp,
                           const uint32_t* vf, const uint32_t* vl, uint32_t* indeg) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < Ep; e += stride) {
    const uint32_t t = col[e];
    const uint64_t r = (t & kRemote) ? Vp + (t & ~kRemote) : t;
    atomicAdd(&indeg[r], 1u);
  }
}

// in-degree -> u64 degrees for the scan + degree-class row lists (PageRank)
__global__ void k_in_deg64(const uint32_t* indeg, uint64_t n, uint64_t* deg64) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n; i += stride)
    deg64[i] = i < n ? indeg[i] : 0ull;
}

__global__ void k_class_list(const uint32_t* indeg, uint64_t n, uint32_t lo, uint32_t hi,
                             uint32_t* list, unsigned long long* count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t d = indeg[i];
    if (d >= lo && d < hi) list[atomicAdd(count, 1ull)] = (uint32_t)i;
  }
}

// in-CSR fill: row = local target (or Vp + outbox slot), entry = local source
__global__ void k_in_fill(const uint64_t* row_off, const uint32_t* col, uint64_t Ep, uint64_t Vp,
                          const uint32_t* vf, const uint32_t* vl, const uint64_t* in_off,
                          uint32_t* cursor, uint32_t* in_col) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < Ep; e += stride) {
    const uint64_t tile = e / kTile;
    const uint32_t l = row_of_edge(row_off, vf[tile], vl[tile], e);
    const uint32_t t = col[e];
    const uint64_t r = (t & kRemote) ? Vp + (t & ~kRemote) : t;
    const uint64_t pos = in_off[r] + atomicAdd(&cursor[r], 1u);
    in_col[pos] = l;
  }
}

// In-only single-partition engines (build_in_csr = 2, P = 1): the in-CSR is
// filled straight from the edge stream (local id = degree position), so the
// out-CSR's column array never exists -- RMAT-30's two CSRs (2 x 69 GB of
// columns) would not fit one B200 together.
__global__ void k_in_count_gen(EdgeGen g, uint64_t E, const uint32_t* rank_of, uint32_t* indeg) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < E; k += stride) {
    uint32_t sv, dv;
    g.get(k, sv, dv);
    atomicAdd(&indeg[rank_of[dv]], 1u);
  }
}
__global__ void k_in_fill_gen(EdgeGen g, uint64_t E, const uint32_t* rank_of, const uint64_t* in_off,
                              uint32_t* cursor, uint32_t* in_col) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < E; k += stride) {
    uint32_t sv, dv;
    g.get(k, sv, dv);
    const uint32_t r = rank_of[dv];
    in_col[in_off[r] + atomicAdd(&cursor[r], 1u)] = rank_of[sv];
  }
}

__global__ void k_outdeg_local(const uint64_t* row_off, uint64_t Vp, uint32_t* outdeg) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < Vp; i += stride)
    outdeg[i] = (uint32_t)(row_off[i + 1] - row_off[i]);
}

// ---- TG_PART_RANDOM (the "naive random-based" partitioning of P:178) ----
__global__ void k_iota(uint64_t V, uint32_t* ids) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V; v += stride)
    ids[v] = (uint32_t)v;
}
__global__ void k_part_keys(uint64_t V, uint32_t pseed, uint32_t* keys, uint32_t* vals) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V; v += stride) {
    keys[v] = tgin_part_key(pseed, v);
    vals[v] = (uint32_t)v;
  }
}
// perm = vertices in (key, id) order; composite key of v = (partition << 32) |
// ~outdeg, so a stable sort groups partitions and orders each by degree desc,
// id asc (values start in id order)
__global__ void k_part_composite(const uint32_t* perm, uint64_t V, int P, const uint32_t* outdeg,
                                 unsigned long long* key) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < V; i += stride) {
    int p;
    uint32_t l;
    deal(i, P, &p, &l);
    const uint32_t v = perm[i];
    key[v] = ((unsigned long long)p << 32) | (unsigned long long)(~outdeg[v]);
  }
}
// sorted[start_p + l] = the vertex with local id l in p -> order position undeal(l, p)
__global__ void k_part_order(const uint32_t* sorted, const unsigned long long* skey, uint64_t V, int P,
                             const uint64_t* start, uint32_t* order) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < V; i += stride) {
    const int p = (int)(skey[i] >> 32);
    order[undeal((uint32_t)(i - start[p]), p, P)] = sorted[i];
  }
}

template <typename T>
T d2h(const T* p, cudaStream_t s) {
  T v;
  TG_CK(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s));
  TG_CK(cudaStreamSynchronize(s));
  return v;
}

constexpr unsigned kB = 256;
inline unsigned G(uint64_t n) { return grid_for(n, kB, 148u * 32u); }

// Sort (keys, vals) pairs of u32 by key with CUB; results in *_out.
void sort_pairs_u32(const uint32_t* kin, uint32_t* kout, const uint32_t* vin, uint32_t* vout,
                    uint64_t n, cudaStream_t s) {
  TG_REQUIRE(n < (1ull << 31), TG_ECAPACITY, "sort: more than 2^31 items");
  size_t tmp = 0;
  TG_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0, 32, s));
  DevBuf<uint8_t> t(tmp ? tmp : 1);
  TG_CK(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kin, kout, vin, vout, (int)n, 0, 32, s));
}

void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  TG_REQUIRE(n < (1ull << 31), TG_ECAPACITY, "scan: more than 2^31 items");
  size_t tmp = 0;
  TG_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, s));
  DevBuf<uint8_t> t(tmp ? tmp : 1);
  TG_CK(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, (int)n, s));
}

constexpr uint32_t kPrCta = 2048;  // in-degree at/above which a PageRank row gets a whole CTA

// first row r with row_off[r] >= target (chunk split points for the row sort)
__global__ void k_split_rows(const uint64_t* row_off, uint64_t nrows, uint64_t step, uint64_t nsplit,
                             uint64_t* out) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k > nsplit) return;
  const uint64_t target = k * step;
  uint64_t lo = 0, hi = nrows;
  while (lo < hi) {
    const uint64_t m = (lo + hi) >> 1;
    if (row_off[m] < target) lo = m + 1;
    else hi = m;
  }
  out[k] = k == nsplit ? nrows : lo;
}

__global__ void k_rel_offsets(const uint64_t* row_off, uint64_t r0, uint64_t n, uint32_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t base = row_off[r0];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n; i += stride)
    out[i] = (uint32_t)(row_off[r0 + i] - base);
}

// Sort the entries of every CSR row ascending (values travel with their keys).
// Local targets (< kRemote) therefore stay before remote ones, and the
// lanes of a warp that gather neighbour state touch ascending addresses.
void sort_rows(const uint64_t* row_off, uint64_t nrows, uint32_t* keys, uint32_t* vals,
               cudaStream_t s) {
  if (!nrows) return;
  uint64_t E = 0;
  TG_CK(cudaMemcpyAsync(&E, row_off + nrows, 8, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaStreamSynchronize(s));
  if (E < 2) return;
  const uint64_t step = 1ull << 30;
  const uint64_t nsplit = (E + step - 1) / step;
  DevBuf<uint64_t> splits(nsplit + 1);
  k_split_rows<<<(unsigned)((nsplit + 256) / 256), 256, 0, s>>>(row_off, nrows, step, nsplit,
                                                                 splits.get());
  TG_CK(cudaGetLastError());
  std::vector<uint64_t> hs(nsplit + 1);
  TG_CK(cudaMemcpyAsync(hs.data(), splits.get(), (nsplit + 1) * 8, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaStreamSynchronize(s));
  hs[0] = 0;
  std::vector<uint64_t> ho(2);
  for (uint64_t c = 0; c < nsplit; ++c) {
    const uint64_t r0 = hs[c], r1 = std::max(hs[c + 1], r0);
    if (r1 <= r0) continue;
    uint64_t e0, e1;
    TG_CK(cudaMemcpyAsync(&e0, row_off + r0, 8, cudaMemcpyDeviceToHost, s));
    TG_CK(cudaMemcpyAsync(&e1, row_off + r1, 8, cudaMemcpyDeviceToHost, s));
    TG_CK(cudaStreamSynchronize(s));
    const uint64_t n = e1 - e0, nseg = r1 - r0;
    if (n < 2) continue;
    TG_REQUIRE(n < (1ull << 31) && nseg < (1ull << 31), TG_ECAPACITY, "row sort chunk too large");
    DevBuf<uint32_t> off(nseg + 1), kout(n), vout(vals ? n : 0);
    k_rel_offsets<<<G(nseg + 1), kB, 0, s>>>(row_off, r0, nseg, off.get());
    TG_CK(cudaGetLastError());
    size_t tmp = 0;
    if (vals) {
      TG_CK(cub::DeviceSegmentedSort::SortPairs(nullptr, tmp, keys + e0, kout.get(), vals + e0,
                                                vout.get(), (int)n, (int)nseg, off.get(),
                                                off.get() + 1, s));
      DevBuf<uint8_t> t(tmp ? tmp : 1);
      TG_CK(cub::DeviceSegmentedSort::SortPairs(t.get(), tmp, keys + e0, kout.get(), vals + e0,
                                                vout.get(), (int)n, (int)nseg, off.get(),
                                                off.get() + 1, s));
      TG_CK(cudaMemcpyAsync(vals + e0, vout.get(), n * 4, cudaMemcpyDeviceToDevice, s));
    } else {
      TG_CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, keys + e0, kout.get(), (int)n,
                                               (int)nseg, off.get(), off.get() + 1, s));
      DevBuf<uint8_t> t(tmp ? tmp : 1);
      TG_CK(cub::DeviceSegmentedSort::SortKeys(t.get(), tmp, keys + e0, kout.get(), (int)n,
                                               (int)nseg, off.get(), off.get() + 1, s));
    }
    TG_CK(cudaMemcpyAsync(keys + e0, kout.get(), n * 4, cudaMemcpyDeviceToDevice, s));
    TG_CK(cudaStreamSynchronize(s));
  }
}

__global__ void k_u32_to_u8(const uint32_t* in, uint64_t n, uint8_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (uint8_t)in[i];
}

// bitmap of the local rows with at least one in-edge (thread per word)
__global__ void k_has_in(const uint64_t* in_off, uint64_t Vp, uint32_t* bm) {
  const uint64_t nw = words_for(Vp);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += stride) {
    uint32_t x = 0;
    const uint64_t v0 = w * 32, v1 = v0 + 32 < Vp ? v0 + 32 : Vp;
    for (uint64_t v = v0; v < v1; ++v)
      if (in_off[v + 1] > in_off[v]) x |= 1u << (v - v0);
    bm[w] = x;
  }
}

void build_part(Engine& eng, Part& pt, const EdgeGen& g, const uint32_t* order,
                const uint32_t* outdeg) {
  cudaStream_t s = eng.stream;
  const int P = eng.P, p = pt.id;
  const uint64_t Vp = pt.Vp;
  DevBuf<unsigned long long> cnt(8);
  TG_CK(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s));

  pt.global_of.alloc(std::max<uint64_t>(Vp, 1));
  k_global_of<<<G(Vp), kB, 0, s>>>(order, Vp, p, P, outdeg, pt.global_of.get(), cnt.get() + 0);
  TG_CK(cudaGetLastError());
  pt.nz_end = d2h(cnt.get() + 0, s);

  DevBuf<uint32_t> nloc(std::max<uint64_t>(Vp, 1)), nrem;
  TG_CK(cudaMemsetAsync(nloc.get(), 0, nloc.bytes(), s));
  uint64_t nremote = 0;
  if (P > 1) {
    nrem.alloc(std::max<uint64_t>(Vp, 1));
    TG_CK(cudaMemsetAsync(nrem.get(), 0, nrem.bytes(), s));
    k_count<<<G(eng.E), kB, 0, s>>>(g, eng.E, eng.rank_of.get(), P, p, nloc.get(), nrem.get(),
                                    cnt.get() + 1);
    TG_CK(cudaGetLastError());
    nremote = d2h(cnt.get() + 1, s);
  } else {
    // single partition: every edge is local, row degree = out-degree
    k_gather_deg<<<G(Vp), kB, 0, s>>>(pt.global_of.get(), outdeg, Vp, nloc.get());
    TG_CK(cudaGetLastError());
  }

  // row offsets
  {
    DevBuf<uint64_t> deg(Vp + 1);
    k_deg64<<<G(Vp + 1), kB, 0, s>>>(nloc.get(), P > 1 ? nrem.get() : nullptr, Vp, deg.get());
    TG_CK(cudaGetLastError());
    pt.row_off.alloc(Vp + 1);
    exclusive_scan_u64(deg.get(), pt.row_off.get(), Vp + 1, s);
  }
  pt.Ep = d2h(pt.row_off.get() + Vp, s);
  pt.Ep_local = pt.Ep - nremote;

  // outbox slots: distinct (q, remote local id), sorted
  DevBuf<unsigned long long> ukeys;
  std::vector<uint64_t> ustart(P + 1, 0);
  pt.obox_off.assign(P + 1, 0);
  DevBuf<uint64_t> d_ustart(P + 1), d_poff(P + 1);
  if (nremote) {
    DevBuf<unsigned long long> keys(nremote), keys2(nremote);
    TG_CK(cudaMemsetAsync(cnt.get() + 2, 0, sizeof(unsigned long long), s));
    k_collect_keys<<<G(eng.E), kB, 0, s>>>(g, eng.E, eng.rank_of.get(), P, p, keys.get(),
                                           cnt.get() + 2);
    TG_CK(cudaGetLastError());
    // 64-bit item counts throughout (CUB 2.8): no 2^31 cap on boundary edges
    size_t tmp = 0;
    TG_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.get(), keys2.get(), (int64_t)nremote, 0,
                                         64, s));
    {
      DevBuf<uint8_t> t(tmp ? tmp : 1);
      TG_CK(cub::DeviceRadixSort::SortKeys(t.get(), tmp, keys.get(), keys2.get(), (int64_t)nremote, 0,
                                           64, s));
    }
    // unique into keys (reuse buffer)
    DevBuf<unsigned long long> nsel(1);
    tmp = 0;
    TG_CK(cub::DeviceSelect::Unique(nullptr, tmp, keys2.get(), keys.get(), nsel.get(),
                                    (int64_t)nremote, s));
    {
      DevBuf<uint8_t> t(tmp ? tmp : 1);
      TG_CK(cub::DeviceSelect::Unique(t.get(), tmp, keys2.get(), keys.get(), nsel.get(),
                                      (int64_t)nremote, s));
    }
    pt.S_real = d2h(nsel.get(), s);
    ukeys.alloc(pt.S_real);
    TG_CK(cudaMemcpyAsync(ukeys.get(), keys.get(), pt.S_real * 8, cudaMemcpyDeviceToDevice, s));
    DevBuf<unsigned long long> seg(P);
    TG_CK(cudaMemsetAsync(seg.get(), 0, seg.bytes(), s));
    k_seg_count<<<G(pt.S_real), kB, 0, s>>>(ukeys.get(), pt.S_real, seg.get());
    TG_CK(cudaGetLastError());
    std::vector<unsigned long long> hseg(P);
    TG_CK(cudaMemcpyAsync(hseg.data(), seg.get(), P * 8, cudaMemcpyDeviceToHost, s));
    TG_CK(cudaStreamSynchronize(s));
    pt.seg_real.assign(hseg.begin(), hseg.end());
    for (int q = 0; q < P; ++q) {
      ustart[q + 1] = ustart[q] + hseg[q];
      pt.obox_off[q + 1] = pt.obox_off[q] + ((hseg[q] + 31) / 32) * 32;
    }
  }
  pt.S = pt.obox_off[P];
  // an out-CSR entry is kRemote | slot: slots must stay below 2^31
  TG_REQUIRE(pt.S < (1ull << 31), TG_ECAPACITY, "more than 2^31 outbox slots in a partition");
  TG_CK(cudaMemcpyAsync(d_ustart.get(), ustart.data(), (P + 1) * 8, cudaMemcpyHostToDevice, s));
  TG_CK(cudaMemcpyAsync(d_poff.get(), pt.obox_off.data(), (P + 1) * 8, cudaMemcpyHostToDevice, s));
  pt.obox_rid.alloc(std::max<uint64_t>(pt.S, 1));
  TG_CK(cudaMemsetAsync(pt.obox_rid.get(), 0xFF, pt.obox_rid.bytes(), s));
  if (pt.S_real) {
    k_place_slots<<<G(pt.S_real), kB, 0, s>>>(ukeys.get(), pt.S_real, d_ustart.get(), d_poff.get(),
                                               pt.obox_rid.get());
    TG_CK(cudaGetLastError());
  }

  // out-CSR fill (skipped by a single-partition in-only engine: stream_in)
  const bool stream_in = eng.in_only && P == 1 && eng.has_in;
  if (!stream_in) {
  pt.col.alloc(std::max<uint64_t>(pt.Ep, 1));
  if (eng.weighted) pt.w.alloc(std::max<uint64_t>(pt.Ep, 1));
  {
    DevBuf<uint32_t> cur_loc(std::max<uint64_t>(Vp, 1)), cur_rem(std::max<uint64_t>(Vp, 1));
    TG_CK(cudaMemsetAsync(cur_loc.get(), 0, cur_loc.bytes(), s));
    TG_CK(cudaMemsetAsync(cur_rem.get(), 0, cur_rem.bytes(), s));
    k_fill<<<G(eng.E), kB, 0, s>>>(g, eng.E, eng.rank_of.get(), P, p, pt.row_off.get(), nloc.get(),
                                   cur_loc.get(), cur_rem.get(), pt.col.get(), pt.w.get(),
                                   eng.weighted, ukeys.get(), pt.S_real, d_ustart.get(),
                                   d_poff.get());
    TG_CK(cudaGetLastError());
  }
  nloc.release();
  nrem.release();
  ukeys.release();
  sort_rows(pt.row_off.get(), Vp, pt.col.get(), eng.weighted ? pt.w.get() : nullptr, s);
  // weights that fit a byte (RMAT weights are in [1, 63], reading A17) are
  // kept as u8: SSSP streams 1 B instead of 4 B of weight per relaxation
  if (eng.weighted && pt.Ep) {
    DevBuf<uint32_t> mx(1);
    size_t tmp = 0;
    TG_CK(cub::DeviceReduce::Max(nullptr, tmp, pt.w.get(), mx.get(), (int64_t)pt.Ep, s));
    DevBuf<uint8_t> t(tmp ? tmp : 1);
    TG_CK(cub::DeviceReduce::Max(t.get(), tmp, pt.w.get(), mx.get(), (int64_t)pt.Ep, s));
    uint32_t hmax = 0;
    TG_CK(cudaMemcpyAsync(&hmax, mx.get(), 4, cudaMemcpyDeviceToHost, s));
    TG_CK(cudaStreamSynchronize(s));
    if (hmax < 256 && !(std::getenv("TG_W32") && std::getenv("TG_W32")[0] == '1')) {
      pt.w8.alloc(pt.Ep);
      k_u32_to_u8<<<G(pt.Ep), kB, 0, s>>>(pt.w.get(), pt.Ep, pt.w8.get());
      TG_CK(cudaGetLastError());
      TG_CK(cudaStreamSynchronize(s));
      pt.w.release();
    }
  }

  }  // !stream_in
  nloc.release();

  // tiles
  pt.ntiles = stream_in ? 0 : (pt.Ep + kTile - 1) / kTile;
  pt.tile_vf.alloc(std::max<uint64_t>(pt.ntiles, 1));
  pt.tile_vl.alloc(std::max<uint64_t>(pt.ntiles, 1));
  if (pt.ntiles) {
    k_tiles<<<G(pt.ntiles), kB, 0, s>>>(pt.row_off.get(), Vp, pt.Ep, pt.ntiles, pt.tile_vf.get(),
                                        pt.tile_vl.get());
    TG_CK(cudaGetLastError());
  }

  // PageRank in-CSR
  if (eng.has_in) {
    pt.has_in = true;
    const uint64_t R = Vp + pt.S;
    DevBuf<uint32_t> indeg(std::max<uint64_t>(R, 1));
    TG_CK(cudaMemsetAsync(indeg.get(), 0, indeg.bytes(), s));
    if (pt.Ep && stream_in) {
      k_in_count_gen<<<G(eng.E), kB, 0, s>>>(g, eng.E, eng.rank_of.get(), indeg.get());
      TG_CK(cudaGetLastError());
    } else if (pt.Ep) {
      k_in_count<<<G(pt.Ep), kB, 0, s>>>(pt.row_off.get(), pt.col.get(), pt.Ep, Vp,
                                         pt.tile_vf.get(), pt.tile_vl.get(), indeg.get());
      TG_CK(cudaGetLastError());
    }
    // rows stay in local-id order (out-degree order: the gathered side of a
    // pull is the source, so hubs -- the hot sources -- are a compact prefix)
    DevBuf<uint64_t> deg64(R + 1);
    k_in_deg64<<<G(R + 1), kB, 0, s>>>(indeg.get(), R, deg64.get());
    TG_CK(cudaGetLastError());
    pt.in_off.alloc(R + 1);
    exclusive_scan_u64(deg64.get(), pt.in_off.get(), R + 1, s);
    deg64.release();
    // degree-class row lists for the PageRank pull (CTA / warp classes)
    {
      DevBuf<unsigned long long> cnt2(2);
      TG_CK(cudaMemsetAsync(cnt2.get(), 0, 16, s));
      DevBuf<uint32_t> lc(std::max<uint64_t>(R, 1)), lw(std::max<uint64_t>(R, 1));
      k_class_list<<<G(R), kB, 0, s>>>(indeg.get(), R, kPrCta, 0xFFFFFFFFu, lc.get(), cnt2.get());
      k_class_list<<<G(R), kB, 0, s>>>(indeg.get(), R, 32u, kPrCta, lw.get(), cnt2.get() + 1);
      TG_CK(cudaGetLastError());
      unsigned long long hc[2];
      TG_CK(cudaMemcpyAsync(hc, cnt2.get(), 16, cudaMemcpyDeviceToHost, s));
      TG_CK(cudaStreamSynchronize(s));
      pt.n_cta = hc[0];
      pt.n_warp = hc[1];
      pt.pr_cta.alloc(std::max<uint64_t>(pt.n_cta, 1));
      pt.pr_warp.alloc(std::max<uint64_t>(pt.n_warp, 1));
      auto sort_list = [&](DevBuf<uint32_t>& src, DevBuf<uint32_t>& dst, uint64_t n) {
        if (!n) return;
        size_t tmp = 0;
        TG_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, src.get(), dst.get(), (int)n, 0, 32, s));
        DevBuf<uint8_t> t(tmp ? tmp : 1);
        TG_CK(cub::DeviceRadixSort::SortKeys(t.get(), tmp, src.get(), dst.get(), (int)n, 0, 32, s));
      };
      sort_list(lc, pt.pr_cta, pt.n_cta);   // ascending row ids: coalesced output writes
      sort_list(lw, pt.pr_warp, pt.n_warp);
    }
    pt.in_col.alloc(std::max<uint64_t>(pt.Ep, 1));
    TG_CK(cudaMemsetAsync(indeg.get(), 0, indeg.bytes(), s));  // reuse as cursor
    if (pt.Ep && stream_in) {
      k_in_fill_gen<<<G(eng.E), kB, 0, s>>>(g, eng.E, eng.rank_of.get(), pt.in_off.get(),
                                            indeg.get(), pt.in_col.get());
      TG_CK(cudaGetLastError());
    } else if (pt.Ep) {
      k_in_fill<<<G(pt.Ep), kB, 0, s>>>(pt.row_off.get(), pt.col.get(), pt.Ep, Vp, pt.tile_vf.get(),
                                        pt.tile_vl.get(), pt.in_off.get(), indeg.get(),
                                        pt.in_col.get());
      TG_CK(cudaGetLastError());
    }
    indeg.release();
    sort_rows(pt.in_off.get(), R, pt.in_col.get(), nullptr, s);
    // edge tiles over the local rows of the in-CSR (BC backward push)
    pt.in_nz.alloc(std::max<uint64_t>(words_for(Vp), 1));
    if (Vp) {
      k_has_in<<<G(words_for(Vp)), kB, 0, s>>>(pt.in_off.get(), Vp, pt.in_nz.get());
      TG_CK(cudaGetLastError());
    }
    pt.in_E_local = Vp ? d2h(pt.in_off.get() + Vp, s) : 0;
    pt.in_ntiles = (pt.in_E_local + kTile - 1) / kTile;
    pt.in_tile_vf.alloc(std::max<uint64_t>(pt.in_ntiles, 1));
    pt.in_tile_vl.alloc(std::max<uint64_t>(pt.in_ntiles, 1));
    if (pt.in_ntiles) {
      k_tiles<<<G(pt.in_ntiles), kB, 0, s>>>(pt.in_off.get(), Vp, pt.in_E_local, pt.in_ntiles,
                                             pt.in_tile_vf.get(), pt.in_tile_vl.get());
      TG_CK(cudaGetLastError());
    }
    if (P > 1 && pt.Ep && R) {
      pt.in_all_ntiles = (pt.Ep + kTile - 1) / kTile;
      pt.in_all_vf.alloc(pt.in_all_ntiles);
      pt.in_all_vl.alloc(pt.in_all_ntiles);
      k_tiles<<<G(pt.in_all_ntiles), kB, 0, s>>>(pt.in_off.get(), R, pt.Ep, pt.in_all_ntiles,
                                                 pt.in_all_vf.get(), pt.in_all_vl.get());
      TG_CK(cudaGetLastError());
    }
    pt.outdeg.alloc(std::max<uint64_t>(Vp, 1));
    k_outdeg_local<<<G(Vp), kB, 0, s>>>(pt.row_off.get(), Vp, pt.outdeg.get());
    TG_CK(cudaGetLastError());
  }
  TG_CK(cudaStreamSynchronize(s));
}

// boundary in-edges of partition q: key (source partition, local id in q)
__global__ void k_in_keys(EdgeGen g, uint64_t E, const uint32_t* rank_of, int P, int q,
                          unsigned long long* keys, unsigned long long* counter) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long cnt = 0;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < E; k += stride) {
    uint32_t s, d, ls, ld;
    int ps, pd;
    g.get(k, s, d);
    deal(rank_of[d], P, &pd, &ld);
    if (pd != q) continue;
    deal(rank_of[s], P, &ps, &ls);
    if (ps == q) continue;
    if (keys) keys[atomicAdd(counter, 1ull)] = ((unsigned long long)ps << 32) | ld;
    else cnt++;
  }
  if (!keys) block_add_u64(counter, cnt);
}

// Inbox of partition q: for every peer p, the distinct local ids of
// q's vertices that p's edges reach, ascending, padded to 32 -- computed from
// the edge stream on q's side, so it equals p's outbox segment for q by
// construction (same set, same order, same padding) without any exchange.
void build_inbox(Engine& eng, Part& pt, const EdgeGen& g) {
  cudaStream_t s = eng.stream;
  const int P = eng.P;
  pt.ibox_off.assign(P + 1, 0);
  pt.iseg_real.assign(P, 0);
  DevBuf<unsigned long long> cnt(1);
  uint64_t n = 0;
  if (P > 1) {
    TG_CK(cudaMemsetAsync(cnt.get(), 0, 8, s));
    k_in_keys<<<G(eng.E), kB, 0, s>>>(g, eng.E, eng.rank_of.get(), P, pt.id, nullptr, cnt.get());
    TG_CK(cudaGetLastError());
    n = d2h(cnt.get(), s);
  }
  DevBuf<unsigned long long> ukeys;
  uint64_t nu = 0;
  std::vector<uint64_t> ustart(P + 1, 0);
  if (n) {
    DevBuf<unsigned long long> keys(n), keys2(n);
    TG_CK(cudaMemsetAsync(cnt.get(), 0, 8, s));
    k_in_keys<<<G(eng.E), kB, 0, s>>>(g, eng.E, eng.rank_of.get(), P, pt.id, keys.get(), cnt.get());
    TG_CK(cudaGetLastError());
    size_t tmp = 0;
    TG_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.get(), keys2.get(), (int64_t)n, 0, 64, s));
    {
      DevBuf<uint8_t> t(tmp ? tmp : 1);
      TG_CK(cub::DeviceRadixSort::SortKeys(t.get(), tmp, keys.get(), keys2.get(), (int64_t)n, 0, 64, s));
    }
    DevBuf<unsigned long long> nsel(1);
    tmp = 0;
    TG_CK(cub::DeviceSelect::Unique(nullptr, tmp, keys2.get(), keys.get(), nsel.get(), (int64_t)n, s));
    {
      DevBuf<uint8_t> t(tmp ? tmp : 1);
      TG_CK(cub::DeviceSelect::Unique(t.get(), tmp, keys2.get(), keys.get(), nsel.get(), (int64_t)n, s));
    }
    nu = d2h(nsel.get(), s);
    ukeys.alloc(nu);
    TG_CK(cudaMemcpyAsync(ukeys.get(), keys.get(), nu * 8, cudaMemcpyDeviceToDevice, s));
    DevBuf<unsigned long long> seg(P);
    TG_CK(cudaMemsetAsync(seg.get(), 0, seg.bytes(), s));
    k_seg_count<<<G(nu), kB, 0, s>>>(ukeys.get(), nu, seg.get());
    TG_CK(cudaGetLastError());
    std::vector<unsigned long long> hseg(P);
    TG_CK(cudaMemcpyAsync(hseg.data(), seg.get(), P * 8, cudaMemcpyDeviceToHost, s));
    TG_CK(cudaStreamSynchronize(s));
    for (int p = 0; p < P; ++p) {
      pt.iseg_real[p] = hseg[p];
      ustart[p + 1] = ustart[p] + hseg[p];
      pt.ibox_off[p + 1] = pt.ibox_off[p] + ((hseg[p] + 31) / 32) * 32;
    }
  }
  pt.I = pt.ibox_off[P];
  pt.I_real = nu;
  pt.ibox_lid.alloc(std::max<uint64_t>(pt.I, 1));
  TG_CK(cudaMemsetAsync(pt.ibox_lid.get(), 0xFF, pt.ibox_lid.bytes(), s));
  if (nu) {
    DevBuf<uint64_t> d_ustart(P + 1), d_poff(P + 1);
    TG_CK(cudaMemcpyAsync(d_ustart.get(), ustart.data(), (P + 1) * 8, cudaMemcpyHostToDevice, s));
    TG_CK(cudaMemcpyAsync(d_poff.get(), pt.ibox_off.data(), (P + 1) * 8, cudaMemcpyHostToDevice, s));
    k_place_slots<<<G(nu), kB, 0, s>>>(ukeys.get(), nu, d_ustart.get(), d_poff.get(),
                                        pt.ibox_lid.get());
    TG_CK(cudaGetLastError());
    TG_CK(cudaStreamSynchronize(s));
  }
}

// Fused-exchange self-test across processes: every rank adds / ORs / mins /
// fp64-adds into each peer's probe words (its staging buffer) and stores its
// rank into a per-sender word, through the same CUDA-IPC mappings the compute
// kernels use; after a barrier each rank checks what landed in its own words.
// The native-atomics attribute says peer atomics are supported; this proves
// they (and plain peer stores) arrive, before the fused transport is trusted.
__global__ void k_peer_probe(uint8_t* const* peer_stage, int world, int me) {
  const int q = threadIdx.x;
  if (q >= world || q == me) return;
  unsigned long long* w = reinterpret_cast<unsigned long long*>(peer_stage[q]);
  atomicAdd(&w[0], 1ull);
  atomicOr(reinterpret_cast<unsigned int*>(&w[1]), 1u << (me & 31));
  atomicMin(reinterpret_cast<unsigned int*>(&w[2]), (unsigned)me);
  atomicAdd(reinterpret_cast<double*>(&w[3]), 0.5);
  w[4 + me] = 1000ull + (unsigned long long)me;
}

// What every partition needs to know about every other: arena / staging /
// global_of pointers and the outbox / inbox offset tables.  One process: the
// local parts.  Several: exchanged with the host allgather, device pointers
// mapped with CUDA IPC (peer access over NVLink between GPUs).
struct PeerMeta {
  cudaIpcMemHandle_t h_fwd, h_rev, h_stage, h_gof;
  char pci[32];  // PCI bus id of the rank's GPU (device ordinals are per process)
  uint64_t Vp;
  uint64_t obox_off[TG_MAX_PARTITIONS + 1];
  uint64_t ibox_off[TG_MAX_PARTITIONS + 1];
};

void map_remote_peers(Engine& eng);

void setup_peers(Engine& eng) {
  eng.peers.assign(eng.P, PeerView{});
  auto fill_local = [&](PeerView& v, Part& p) {
    v.arena_fwd = p.arena_fwd.get();
    v.arena_rev = p.arena_rev.get();
    v.staging = p.staging.get();
    v.global_of = p.global_of.get();
    v.Vp = p.Vp;
    v.obox_off = p.obox_off;
    v.ibox_off = p.ibox_off;
  };
  for (auto& pt : eng.parts) fill_local(eng.peers[pt->id], *pt);
  if (eng.multi()) map_remote_peers(eng);
  // symmetry: p's outbox segment for q has the size of q's inbox from p
  for (auto& pt : eng.parts)
    for (int q = 0; q < eng.P; ++q) {
      if (q == pt->id) continue;
      const uint64_t a = pt->obox_off[q + 1] - pt->obox_off[q];
      const uint64_t b = eng.peers[q].ibox_off[pt->id + 1] - eng.peers[q].ibox_off[pt->id];
      TG_REQUIRE(a == b, TG_EINTERNAL, "outbox/inbox symmetry violated");
    }
  // fused-exchange tables: slot s of p's segment for q -> q's arena index of it
  for (auto& pt : eng.parts) {
    Part& p = *pt;
    std::vector<uint8_t> owner(std::max<uint64_t>(p.S / 32, 1), 0);
    std::vector<uint8_t*> arena(eng.P, nullptr);
    std::vector<int64_t> delta(eng.P, 0);
    for (int q = 0; q < eng.P; ++q) {
      for (uint64_t w = p.obox_off[q] / 32; w < p.obox_off[q + 1] / 32; ++w) owner[w] = (uint8_t)q;
      if (q == p.id) continue;
      arena[q] = eng.peers[q].arena_fwd;
      delta[q] = (int64_t)eng.peers[q].ibox_off[p.id] - (int64_t)p.obox_off[q];
      TG_REQUIRE(delta[q] % 32 == 0, TG_EINTERNAL, "unaligned inbox segment");
    }
    p.rmt_owner.alloc(owner.size());
    p.rmt_arena.alloc(eng.P);
    p.rmt_delta.alloc(eng.P);
    TG_CK(cudaMemcpy(p.rmt_owner.get(), owner.data(), owner.size(), cudaMemcpyHostToDevice));
    TG_CK(cudaMemcpy(p.rmt_arena.get(), arena.data(), eng.P * sizeof(uint8_t*), cudaMemcpyHostToDevice));
    TG_CK(cudaMemcpy(p.rmt_delta.get(), delta.data(), eng.P * sizeof(int64_t), cudaMemcpyHostToDevice));
    // reverse: inbox entry j of segment p' -> p''s arena_rev at its outbox index
    std::vector<uint8_t> iowner(std::max<uint64_t>(p.I / 32, 1), 0);
    std::vector<uint8_t*> iarena(eng.P, nullptr);
    std::vector<int64_t> idelta(eng.P, 0);
    for (int q = 0; q < eng.P; ++q) {
      for (uint64_t w = p.ibox_off[q] / 32; w < p.ibox_off[q + 1] / 32; ++w) iowner[w] = (uint8_t)q;
      if (q == p.id) continue;
      iarena[q] = eng.peers[q].arena_rev;
      idelta[q] = (int64_t)eng.peers[q].obox_off[p.id] - (int64_t)p.ibox_off[q];
    }
    p.rin_owner.alloc(iowner.size());
    p.rin_arena.alloc(eng.P);
    p.rin_delta.alloc(eng.P);
    TG_CK(cudaMemcpy(p.rin_owner.get(), iowner.data(), iowner.size(), cudaMemcpyHostToDevice));
    TG_CK(cudaMemcpy(p.rin_arena.get(), iarena.data(), eng.P * sizeof(uint8_t*), cudaMemcpyHostToDevice));
    TG_CK(cudaMemcpy(p.rin_delta.get(), idelta.data(), eng.P * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  if (const char* f = std::getenv("TG_FUSED_EXCHANGE")) eng.fused = f[0] != '0' && eng.peer_atomics;
  // the tables above were copied from pageable host memory on the legacy
  // stream: make sure they landed before any engine-stream kernel reads them
  TG_CK(cudaDeviceSynchronize());
}

void map_remote_peers(Engine& eng) {
  Part& me = *eng.parts[0];
  PeerMeta mine{};
  TG_CK(cudaIpcGetMemHandle(&mine.h_fwd, me.arena_fwd.get()));
  TG_CK(cudaIpcGetMemHandle(&mine.h_rev, me.arena_rev.get()));
  TG_CK(cudaIpcGetMemHandle(&mine.h_stage, me.staging.get()));
  TG_CK(cudaIpcGetMemHandle(&mine.h_gof, me.global_of.get()));
  mine.Vp = me.Vp;
  TG_CK(cudaDeviceGetPCIBusId(mine.pci, sizeof(mine.pci), eng.device));
  for (int q = 0; q <= eng.P; ++q) {
    mine.obox_off[q] = me.obox_off[q];
    mine.ibox_off[q] = me.ibox_off[q];
  }
  std::vector<PeerMeta> all(eng.world);
  TG_REQUIRE(eng.comm.allgather(eng.comm.ctx, &mine, all.data(), sizeof(PeerMeta)) == 0, TG_ENCCL,
             "tg_comm.allgather failed");
  for (int q = 0; q < eng.world; ++q) {
    if (q == eng.rank) continue;
    PeerView& v = eng.peers[q];
    void* p = nullptr;
    auto open = [&](const cudaIpcMemHandle_t& h) {
      void* ptr = nullptr;
      TG_CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      v.opened.push_back(ptr);
      return ptr;
    };
    (void)p;
    v.arena_fwd = static_cast<uint8_t*>(open(all[q].h_fwd));
    v.arena_rev = static_cast<uint8_t*>(open(all[q].h_rev));
    v.staging = static_cast<uint8_t*>(open(all[q].h_stage));
    v.global_of = static_cast<uint32_t*>(open(all[q].h_gof));
    v.Vp = all[q].Vp;
    v.obox_off.assign(all[q].obox_off, all[q].obox_off + eng.P + 1);
    v.ibox_off.assign(all[q].ibox_off, all[q].ibox_off + eng.P + 1);
  }
  // The fused exchange issues reductions (atomicOr / atomicMin / fp64 add) on
  // peer memory: that needs native peer atomics between every pair of GPUs
  // (NVLink / NVSwitch).  Otherwise every rank falls back to the copy
  // transport (agreed with a min-allreduce: SPMD).
  uint64_t ok = 1;
  for (int q = 0; q < eng.world; ++q) {
    if (q == eng.rank) continue;
    int pd = -1;
    if (cudaDeviceGetByPCIBusId(&pd, all[q].pci) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      continue;
    }
    if (pd == eng.device) continue;  // same GPU (ranks sharing a device)
    int atom = 0;
    if (cudaDeviceGetP2PAttribute(&atom, cudaDevP2PAttrNativeAtomicSupported, eng.device, pd) !=
            cudaSuccess ||
        !atom) {
      cudaGetLastError();
      ok = 0;
    }
  }
  TG_REQUIRE(eng.comm.allreduce_u64(eng.comm.ctx, &ok, 1, 1) == 0, TG_ENCCL,
             "tg_comm.allreduce_u64 failed");
  // self-test of peer atomics + stores through the IPC mappings (staging is
  // >= 8 B per vertex; the probe needs 4 + world words, so only when every
  // rank has that many vertices -- otherwise the attribute alone decides)
  uint64_t room = me.Vp >= (uint64_t)(4 + eng.world) ? 1 : 0;
  comm_allreduce(eng, &room, 1, 1);
  if (ok && room && !(std::getenv("TG_PEER_PROBE") && std::getenv("TG_PEER_PROBE")[0] == '0')) {
    std::vector<unsigned long long> init(4 + eng.world, 0);
    init[2] = 0xFFFFFFFFull;
    // stream-ordered and drained before the barrier: a plain cudaMemcpy from
    // pageable memory may still be in flight when it returns, and would then
    // overwrite a peer's early probe writes
    cudaStream_t s = eng.stream;
    TG_CK(cudaMemcpyAsync(me.staging.get(), init.data(), init.size() * 8, cudaMemcpyHostToDevice, s));
    TG_CK(cudaStreamSynchronize(s));
    comm_barrier(eng);
    std::vector<uint8_t*> st(eng.world, nullptr);
    for (int q = 0; q < eng.world; ++q) st[q] = eng.peers[q].staging;
    DevBuf<uint8_t*> d_st(eng.world);
    TG_CK(cudaMemcpy(d_st.get(), st.data(), eng.world * sizeof(uint8_t*), cudaMemcpyHostToDevice));
    k_peer_probe<<<1, 64, 0, s>>>(d_st.get(), eng.world, eng.rank);
    TG_CK(cudaGetLastError());
    TG_CK(cudaStreamSynchronize(s));
    comm_barrier(eng);
    std::vector<unsigned long long> got(4 + eng.world);
    TG_CK(cudaMemcpy(got.data(), me.staging.get(), got.size() * 8, cudaMemcpyDeviceToHost));
    uint32_t want_or = 0;
    unsigned want_min = 0xFFFFFFFFu;
    for (int q = 0; q < eng.world; ++q)
      if (q != eng.rank) {
        want_or |= 1u << (q & 31);
        want_min = std::min<unsigned>(want_min, (unsigned)q);
      }
    double fsum;
    std::memcpy(&fsum, &got[3], 8);
    bool good = got[0] == (unsigned long long)(eng.world - 1) && (uint32_t)got[1] == want_or &&
                (uint32_t)got[2] == want_min && fsum == 0.5 * (eng.world - 1);
    for (int q = 0; q < eng.world; ++q)
      if (q != eng.rank) good = good && got[4 + q] == 1000ull + (unsigned long long)q;
    ok = good ? 1 : 0;
    comm_allreduce(eng, &ok, 1, 1);
    eng.peer_probe_passed = ok != 0;
  }
  eng.peer_atomics = ok != 0;
  if (!eng.peer_atomics) eng.fused = false;
}

// ---- ghost-pull PageRank layout (build_pr_ghost) --------------------------
// p's inbox entry j from q <-> q's outbox slot s: j = ibox_base + s.
// Per slot s of Q's segment for p: the row v = lid[s] of p gets one entry per
// source of Q's outbox row Vq + s.
__global__ void k_gh_count(const uint64_t* q_in_off, uint64_t qVp, uint64_t s0, uint64_t s1,
                           const uint32_t* lid_by_slot, uint32_t* cnt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = s0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < s1; s += stride) {
    const uint32_t v = lid_by_slot[s];
    if (v == kInf) continue;
    const uint64_t n = q_in_off[qVp + s + 1] - q_in_off[qVp + s];
    if (n) atomicAdd(&cnt[v], (uint32_t)n);
  }
}
__global__ void k_gh_local(const uint64_t* in_off, const uint32_t* in_col, uint64_t Vp,
                           const uint64_t* off, uint32_t* col, uint32_t* cursor) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < Vp; v += stride) {
    const uint64_t b = in_off[v], e = in_off[v + 1], o = off[v];
    for (uint64_t i = b; i < e; ++i) col[o + (i - b)] = in_col[i];
    cursor[v] = (uint32_t)(e - b);
  }
}
__global__ void k_gh_fill(const uint64_t* q_in_off, const uint32_t* q_in_col, uint64_t qVp,
                          uint64_t s0, uint64_t s1, const uint32_t* lid_by_slot,
                          const uint32_t* pub, uint64_t npub, uint32_t ghost_base,
                          const uint64_t* off, uint32_t* col, uint32_t* cursor) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = s0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < s1; s += stride) {
    const uint32_t v = lid_by_slot[s];
    if (v == kInf) continue;
    for (uint64_t i = q_in_off[qVp + s], e = q_in_off[qVp + s + 1]; i < e; ++i) {
      const uint32_t u = q_in_col[i];
      uint64_t lo = 0, hi = npub;  // position of u in Q's publish list for p
      while (lo < hi) {
        const uint64_t m = (lo + hi) >> 1;
        if (pub[m] < u) lo = m + 1;
        else hi = m;
      }
      col[off[v] + atomicAdd(&cursor[v], 1u)] = ghost_base + (uint32_t)lo;
    }
  }
}
__global__ void k_deg_sum(const uint64_t* in_off, const uint32_t* cnt, uint64_t Vp, uint64_t* deg64,
                          uint32_t* deg32) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= Vp; v += stride) {
    const uint64_t d = v < Vp ? (in_off[v + 1] - in_off[v]) + cnt[v] : 0;
    deg64[v] = d;
    if (v < Vp) deg32[v] = (uint32_t)(d < 0xFFFFFFFFull ? d : 0xFFFFFFFFull);
  }
}

}  // namespace

void build_engine(Engine& eng, const EdgeInput& in) {
  auto t0 = std::chrono::steady_clock::now();
  cudaStream_t s = eng.stream;
  EdgeGen g{};
  g.src = in.src;
  g.dst = in.dst;
  g.w = in.w;
  g.gen = in.generated;
  g.r = tgin_make_rmat(in.scale, in.a, in.b, in.c, in.seed, in.scramble);
  g.wseed = in.wseed;
  const uint64_t V = eng.V;

  DevBuf<uint32_t> outdeg(V);
  DevBuf<unsigned long long> bad(1);
  TG_CK(cudaMemsetAsync(outdeg.get(), 0, outdeg.bytes(), s));
  TG_CK(cudaMemsetAsync(bad.get(), 0, bad.bytes(), s));
  if (eng.E) {
    k_outdeg<<<G(eng.E), kB, 0, s>>>(g, eng.E, V, outdeg.get(), bad.get());
    TG_CK(cudaGetLastError());
  }
  TG_REQUIRE(d2h(bad.get(), s) == 0, TG_EINVAL, "edge endpoint id >= V");

  // order[i] = the vertex dealt from position i (deal(i) -> (partition, local id))
  DevBuf<uint32_t> order(V);
  if (eng.strategy == TG_PART_RANDOM && eng.P > 1) {
    TG_REQUIRE(V < (1ull << 31), TG_ECAPACITY, "sort: more than 2^31 items");
    DevBuf<uint32_t> perm(V);
    {
      DevBuf<uint32_t> keys(V), keys_out(V), vals(V);
      k_part_keys<<<G(V), kB, 0, s>>>(V, eng.part_seed, keys.get(), vals.get());
      TG_CK(cudaGetLastError());
      sort_pairs_u32(keys.get(), keys_out.get(), vals.get(), perm.get(), V, s);
    }
    DevBuf<unsigned long long> key(V), key_out(V);
    DevBuf<uint32_t> ids(V), sorted(V);
    k_part_composite<<<G(V), kB, 0, s>>>(perm.get(), V, eng.P, outdeg.get(), key.get());
    k_iota<<<G(V), kB, 0, s>>>(V, ids.get());
    TG_CK(cudaGetLastError());
    size_t tmp = 0;
    TG_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.get(), key_out.get(), ids.get(),
                                          sorted.get(), (int)V, 0, 64, s));
    {
      DevBuf<uint8_t> t(tmp ? tmp : 1);
      TG_CK(cub::DeviceRadixSort::SortPairs(t.get(), tmp, key.get(), key_out.get(), ids.get(),
                                            sorted.get(), (int)V, 0, 64, s));
    }
    std::vector<uint64_t> start(eng.P + 1, 0);
    for (int p = 0; p < eng.P; ++p) start[p + 1] = start[p] + part_size(V, p, eng.P);
    DevBuf<uint64_t> d_start(eng.P + 1);
    TG_CK(cudaMemcpyAsync(d_start.get(), start.data(), (eng.P + 1) * 8, cudaMemcpyHostToDevice, s));
    k_part_order<<<G(V), kB, 0, s>>>(sorted.get(), key_out.get(), V, eng.P, d_start.get(),
                                     order.get());
    TG_CK(cudaGetLastError());
    TG_CK(cudaStreamSynchronize(s));
  } else {
    DevBuf<uint32_t> keys(V), keys_out(V), vals(V);
    k_neg_iota<<<G(V), kB, 0, s>>>(outdeg.get(), V, keys.get(), vals.get());
    TG_CK(cudaGetLastError());
    sort_pairs_u32(keys.get(), keys_out.get(), vals.get(), order.get(), V, s);
  }
  eng.rank_of.alloc(V);
  k_inverse<<<G(V), kB, 0, s>>>(order.get(), V, eng.rank_of.get());
  TG_CK(cudaGetLastError());

  // hosted partitions: all P in one process, or partition `rank` of `world`
  eng.parts.clear();
  for (int p = 0; p < eng.P; ++p) {
    if (eng.multi() && p != eng.rank) continue;
    auto pt = std::make_unique<Part>();
    pt->id = p;
    pt->Vp = part_size(V, p, eng.P);
    eng.parts.push_back(std::move(pt));
  }
  for (auto& pt : eng.parts) {
    build_part(eng, *pt, g, order.get(), outdeg.get());
    if (pt->seg_real.empty()) pt->seg_real.assign(eng.P, 0);
    build_inbox(eng, *pt, g);
    // receive arenas + collection staging (8 bytes per slot / vertex)
    pt->arena_fwd.alloc(std::max<uint64_t>(pt->I, 1) * 16);  // 2 x 8 B: double-buffered PR sums
    pt->arena_rev.alloc(std::max<uint64_t>(pt->S, 1) * 16);  // 2 x 8 B: double-buffered BC ghosts
    pt->staging.alloc(std::max<uint64_t>(pt->Vp, 1) * 8);
    // PageRank-only engine: its pull needs the in-CSR and outdeg only; drop
    // this partition's out-CSR before the next partition is built, so the peak
    // is the in-CSRs plus ONE out-CSR (RMAT-30 in 8 partitions on one GPU)
    if (eng.in_only) {
      TG_CK(cudaStreamSynchronize(s));
      pt->col.release();
      pt->w.release();
      pt->w8.release();
      pt->tile_vf.release();
      pt->tile_vl.release();
      pt->in_all_vf.release();
      pt->in_all_vl.release();
      pt->ntiles = pt->in_all_ntiles = 0;
    }
  }
  TG_CK(cudaStreamSynchronize(s));
  setup_peers(eng);
  eng.build_ms = (uint64_t)std::chrono::duration_cast<std::chrono::milliseconds>(
                     std::chrono::steady_clock::now() - t0)
                     .count();
}

void build_pr_ghost(Engine& eng) {
  TG_REQUIRE(eng.has_in, TG_EINVAL, "ghost-pull PageRank needs the in-CSR");
  bool all = true;
  for (auto& pp : eng.parts) all = all && pp->gh.built;
  if (all) return;
  cudaStream_t s = eng.stream;
  const int P = eng.P;
  // 1. publish lists of the hosted partitions: distinct sources of p's outbox
  //    rows for q, ascending
  for (auto& pp : eng.parts) {
    Part& p = *pp;
    PRGhost& g = p.gh;
    g.pub_off.assign(P + 1, 0);
    std::vector<DevBuf<uint32_t>> seg(P);
    std::vector<uint64_t> cnt(P, 0);
    for (int q = 0; q < P; ++q) {
      if (q == p.id || p.obox_off[q + 1] == p.obox_off[q]) continue;
      const uint64_t e0 = d2h(p.in_off.get() + p.Vp + p.obox_off[q], s);
      const uint64_t e1 = d2h(p.in_off.get() + p.Vp + p.obox_off[q + 1], s);
      const uint64_t n = e1 - e0;
      if (!n) continue;
      DevBuf<uint32_t> sorted(n);
      seg[q].alloc(n);
      size_t tmp = 0;
      TG_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, p.in_col.get() + e0, sorted.get(), (int64_t)n, 0,
                                           32, s));
      DevBuf<uint8_t> t1(tmp ? tmp : 1);
      TG_CK(cub::DeviceRadixSort::SortKeys(t1.get(), tmp, p.in_col.get() + e0, sorted.get(), (int64_t)n,
                                           0, 32, s));
      DevBuf<unsigned long long> nsel(1);
      tmp = 0;
      TG_CK(cub::DeviceSelect::Unique(nullptr, tmp, sorted.get(), seg[q].get(), nsel.get(), (int64_t)n, s));
      DevBuf<uint8_t> t2(tmp ? tmp : 1);
      TG_CK(cub::DeviceSelect::Unique(t2.get(), tmp, sorted.get(), seg[q].get(), nsel.get(), (int64_t)n, s));
      cnt[q] = d2h(nsel.get(), s);
    }
    for (int q = 0; q < P; ++q) g.pub_off[q + 1] = g.pub_off[q] + cnt[q];
    g.pub_lid.alloc(std::max<uint64_t>(g.pub_off[P], 1));
    for (int q = 0; q < P; ++q)
      if (cnt[q])
        TG_CK(cudaMemcpyAsync(g.pub_lid.get() + g.pub_off[q], seg[q].get(), cnt[q] * 4,
                              cudaMemcpyDeviceToDevice, s));
    TG_CK(cudaStreamSynchronize(s));
  }
  // 2. a view of every partition: hosted ones directly, the others through
  //    CUDA IPC (their in-CSR and publish list, read by the fill kernels below)
  struct View {
    uint64_t Vp = 0;
    std::vector<uint64_t> obox_off, pub_off;
    const uint64_t* in_off = nullptr;
    const uint32_t* in_col = nullptr;
    const uint32_t* pub_lid = nullptr;
  };
  std::vector<View> view(P);
  std::vector<void*> build_maps;
  for (auto& pp : eng.parts)
    view[pp->id] = {pp->Vp, pp->obox_off, pp->gh.pub_off, pp->in_off.get(), pp->in_col.get(),
                    pp->gh.pub_lid.get()};
  struct Meta {
    cudaIpcMemHandle_t h_off, h_col, h_pub;
    uint64_t Vp;
    uint64_t obox_off[TG_MAX_PARTITIONS + 1], pub_off[TG_MAX_PARTITIONS + 1];
  };
  if (eng.multi()) {
    Part& me = *eng.parts[0];
    Meta mine{};
    TG_CK(cudaIpcGetMemHandle(&mine.h_off, me.in_off.get()));
    TG_CK(cudaIpcGetMemHandle(&mine.h_col, me.in_col.get()));
    TG_CK(cudaIpcGetMemHandle(&mine.h_pub, me.gh.pub_lid.get()));
    mine.Vp = me.Vp;
    for (int q = 0; q <= P; ++q) {
      mine.obox_off[q] = me.obox_off[q];
      mine.pub_off[q] = me.gh.pub_off[q];
    }
    std::vector<Meta> all(eng.world);
    TG_REQUIRE(eng.comm.allgather(eng.comm.ctx, &mine, all.data(), sizeof(Meta)) == 0, TG_ENCCL,
               "tg_comm.allgather failed");
    for (int q = 0; q < eng.world; ++q) {
      if (q == eng.rank) continue;
      auto open = [&](const cudaIpcMemHandle_t& h) {
        void* ptr = nullptr;
        TG_CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        build_maps.push_back(ptr);
        return ptr;
      };
      View& v = view[q];
      v.Vp = all[q].Vp;
      v.obox_off.assign(all[q].obox_off, all[q].obox_off + P + 1);
      v.pub_off.assign(all[q].pub_off, all[q].pub_off + P + 1);
      v.in_off = static_cast<const uint64_t*>(open(all[q].h_off));
      v.in_col = static_cast<const uint32_t*>(open(all[q].h_col));
      v.pub_lid = static_cast<const uint32_t*>(open(all[q].h_pub));
    }
  }
  // size of r's publish list for q = q's ghost segment of r (padded to 32
  // slots: frontier bits are published as whole words)
  auto pubsz = [&](int r, int q) -> uint64_t {
    return r == q ? 0 : (view[r].pub_off[q + 1] - view[r].pub_off[q] + 31) / 32 * 32;
  };
  auto pubn = [&](int r, int q) -> uint64_t {  // unpadded
    return r == q ? 0 : view[r].pub_off[q + 1] - view[r].pub_off[q];
  };
  auto gh_off_of = [&](int q, int r) -> uint64_t {  // q's ghost offset of r
    uint64_t o = 0;
    for (int x = 0; x < r; ++x) o += pubsz(x, q);
    return o;
  };
  // 3. ghost in-CSR of the hosted partitions: local entries + one ghost entry
  //    per remote in-edge (u in q, v in p), from q's outbox rows for p
  for (auto& pp : eng.parts) {
    Part& p = *pp;
    PRGhost& g = p.gh;
    g.gh_off.assign(P + 1, 0);
    for (int q = 0; q < P; ++q) g.gh_off[q + 1] = g.gh_off[q] + pubsz(q, p.id);
    g.G = g.gh_off[P];
    TG_REQUIRE(p.Vp + g.G < (1ull << 31), TG_ECAPACITY, "ghost index space exceeds 2^31");
    const uint64_t Vp = p.Vp;
    DevBuf<uint32_t> cnt(std::max<uint64_t>(Vp, 1)), deg32(std::max<uint64_t>(Vp, 1));
    TG_CK(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s));
    for (int q = 0; q < P; ++q) {
      if (q == p.id) continue;
      const View& Q = view[q];
      const uint64_t s0 = Q.obox_off[p.id], s1 = Q.obox_off[p.id + 1];
      if (s1 == s0) continue;
      const uint32_t* lid_by_slot = p.ibox_lid.get() + p.ibox_off[q] - s0;
      k_gh_count<<<G(s1 - s0), kB, 0, s>>>(Q.in_off, Q.Vp, s0, s1, lid_by_slot, cnt.get());
    }
    DevBuf<uint64_t> deg64(Vp + 1);
    k_deg_sum<<<G(Vp + 1), kB, 0, s>>>(p.in_off.get(), cnt.get(), Vp, deg64.get(), deg32.get());
    TG_CK(cudaGetLastError());
    g.off.alloc(Vp + 1);
    exclusive_scan_u64(deg64.get(), g.off.get(), Vp + 1, s);
    const uint64_t n = d2h(g.off.get() + Vp, s);
    g.col.alloc(std::max<uint64_t>(n, 1));
    if (Vp) {
      k_gh_local<<<G(Vp), kB, 0, s>>>(p.in_off.get(), p.in_col.get(), Vp, g.off.get(), g.col.get(),
                                      cnt.get());  // cnt becomes the fill cursor
      TG_CK(cudaGetLastError());
    }
    for (int q = 0; q < P; ++q) {
      if (q == p.id) continue;
      const View& Q = view[q];
      const uint64_t s0 = Q.obox_off[p.id], s1 = Q.obox_off[p.id + 1];
      if (s1 == s0) continue;
      const uint32_t* lid_by_slot = p.ibox_lid.get() + p.ibox_off[q] - s0;
      k_gh_fill<<<G(s1 - s0), kB, 0, s>>>(Q.in_off, Q.in_col, Q.Vp, s0, s1, lid_by_slot,
                                          Q.pub_lid + Q.pub_off[p.id], pubn(q, p.id),
                                          (uint32_t)(Vp + g.gh_off[q]), g.off.get(), g.col.get(),
                                          cnt.get());
      TG_CK(cudaGetLastError());
    }
    sort_rows(g.off.get(), Vp, g.col.get(), nullptr, s);
    g.nz.alloc(std::max<uint64_t>(words_for(Vp), 1));
    if (Vp) {
      k_has_in<<<G(words_for(Vp)), kB, 0, s>>>(g.off.get(), Vp, g.nz.get());
      TG_CK(cudaGetLastError());
    }
    g.bits.alloc(std::max<uint64_t>(words_for(g.G), 1));
    g.sigma.alloc(std::max<uint64_t>(g.G, 1));
    TG_CK(cudaMemsetAsync(g.bits.get(), 0, g.bits.bytes(), s));
    TG_CK(cudaMemsetAsync(g.sigma.get(), 0, g.sigma.bytes(), s));
    // row classes of the ghost in-CSR
    DevBuf<unsigned long long> c2(2);
    TG_CK(cudaMemsetAsync(c2.get(), 0, 16, s));
    DevBuf<uint32_t> lc(std::max<uint64_t>(Vp, 1)), lw(std::max<uint64_t>(Vp, 1));
    k_class_list<<<G(Vp), kB, 0, s>>>(deg32.get(), Vp, kPrCta, 0xFFFFFFFFu, lc.get(), c2.get());
    k_class_list<<<G(Vp), kB, 0, s>>>(deg32.get(), Vp, 32u, kPrCta, lw.get(), c2.get() + 1);
    TG_CK(cudaGetLastError());
    unsigned long long hc[2];
    TG_CK(cudaMemcpyAsync(hc, c2.get(), 16, cudaMemcpyDeviceToHost, s));
    TG_CK(cudaStreamSynchronize(s));
    g.n_cta = hc[0];
    g.n_warp = hc[1];
    g.cta.alloc(std::max<uint64_t>(g.n_cta, 1));
    g.warp.alloc(std::max<uint64_t>(g.n_warp, 1));
    auto sort_list = [&](DevBuf<uint32_t>& src, DevBuf<uint32_t>& dst, uint64_t m) {
      if (!m) return;
      size_t tmp = 0;
      TG_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, src.get(), dst.get(), (int)m, 0, 32, s));
      DevBuf<uint8_t> t(tmp ? tmp : 1);
      TG_CK(cub::DeviceRadixSort::SortKeys(t.get(), tmp, src.get(), dst.get(), (int)m, 0, 32, s));
    };
    sort_list(lc, g.cta, g.n_cta);
    sort_list(lw, g.warp, g.n_warp);
    TG_CK(cudaStreamSynchronize(s));
    // contribution buffers [local | ghost slots]
    const uint64_t Cn = std::max<uint64_t>(Vp + g.G, 1);
    for (int b2 = 0; b2 < 2; ++b2)
      if (p.pr.contrib[b2].n < Cn) p.pr.contrib[b2].alloc(Cn);
  }
  for (void* ptr : build_maps) cudaIpcCloseMemHandle(ptr);
  // 4. publish destinations: q's contribution buffer + Vq + q's ghost offset of p
  std::vector<float*> base[2];
  base[0].assign(P, nullptr);
  base[1].assign(P, nullptr);
  for (auto& pp : eng.parts)
    for (int b2 = 0; b2 < 2; ++b2) base[b2][pp->id] = pp->pr.contrib[b2].get();
  std::vector<uint32_t*> gbits(P, nullptr);
  std::vector<double*> gsig(P, nullptr);
  for (auto& pp : eng.parts) {
    gbits[pp->id] = pp->gh.bits.get();
    gsig[pp->id] = pp->gh.sigma.get();
  }
  if (eng.multi()) {
    Part& me = *eng.parts[0];
    struct CMeta {
      cudaIpcMemHandle_t h[2], hb, hs;
    } mine{};
    for (int b2 = 0; b2 < 2; ++b2) TG_CK(cudaIpcGetMemHandle(&mine.h[b2], me.pr.contrib[b2].get()));
    TG_CK(cudaIpcGetMemHandle(&mine.hb, me.gh.bits.get()));
    TG_CK(cudaIpcGetMemHandle(&mine.hs, me.gh.sigma.get()));
    std::vector<CMeta> all(eng.world);
    TG_REQUIRE(eng.comm.allgather(eng.comm.ctx, &mine, all.data(), sizeof(CMeta)) == 0, TG_ENCCL,
               "tg_comm.allgather failed");
    for (int q = 0; q < eng.world; ++q) {
      if (q == eng.rank) continue;
      auto open = [&](const cudaIpcMemHandle_t& h) {
        void* ptr = nullptr;
        TG_CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        eng.peers[q].opened.push_back(ptr);  // closed with the engine
        return ptr;
      };
      for (int b2 = 0; b2 < 2; ++b2) base[b2][q] = static_cast<float*>(open(all[q].h[b2]));
      gbits[q] = static_cast<uint32_t*>(open(all[q].hb));
      gsig[q] = static_cast<double*>(open(all[q].hs));
    }
  }
  for (auto& pp : eng.parts) {
    PRGhost& g = pp->gh;
    for (int b2 = 0; b2 < 2; ++b2) {
      g.pub_dst[b2].assign(P, nullptr);
      for (int q = 0; q < P; ++q)
        if (q != pp->id) g.pub_dst[b2][q] = base[b2][q] + view[q].Vp + gh_off_of(q, pp->id);
    }
    std::vector<uint32_t*> bd(P, nullptr);
    std::vector<double*> sd(P, nullptr);
    for (int q = 0; q < P; ++q)
      if (q != pp->id) {
        const uint64_t go = gh_off_of(q, pp->id);  // multiple of 32
        bd[q] = gbits[q] + go / 32;
        sd[q] = gsig[q] + go;
      }
    g.d_pub_off.alloc(P + 1);
    g.d_bits_dst.alloc(P);
    g.d_sigma_dst.alloc(P);
    TG_CK(cudaMemcpy(g.d_pub_off.get(), g.pub_off.data(), (P + 1) * 8, cudaMemcpyHostToDevice));
    TG_CK(cudaMemcpy(g.d_bits_dst.get(), bd.data(), P * sizeof(uint32_t*), cudaMemcpyHostToDevice));
    TG_CK(cudaMemcpy(g.d_sigma_dst.get(), sd.data(), P * sizeof(double*), cudaMemcpyHostToDevice));
    g.built = true;
  }
  TG_CK(cudaStreamSynchronize(s));
  comm_barrier(eng);  // every rank's ghost buffers are zeroed before anyone publishes
}
}  // namespace tg
