// bfs.cu -- level-synchronous BFS over BSP supersteps (Fig. 11;
// Appendix 1).  Per superstep L and partition p:
//   compute : every edge (v,t) of a level-L vertex v: local t not yet visited ->
//             set t in the next-frontier bitmap (the visited test of Fig. 11
//             lines 6-7; the bitmap is the paper's "summary data structure",
//             P:316).  Remote t -> test-and-set its outbox slot's "ever sent"
//             bit; a first visit sets the slot's bit in this superstep's
//             outbox bitmap (the reduction of P:830-833: one message per remote
//             vertex, ever).
//   communicate: outbox bitmaps -> peers' inbox bitmaps (1 bit per slot: the
//             "compression" P:292 allows; same result as the paper's full
//             level buffer under min-combine).
//   scatter : inbox bit set and owner vertex unvisited -> next bit
//             (totem_engine_scatter_inbox_min).
//   advance : next bitmap -> level[v] = L+1, visited |= next, vote count
//             (termination when every partition's count is 0).
#include "frontier.cuh"

namespace tg {

namespace {

struct BfsOp {
  using Aux = Empty;
  static constexpr bool kReduce = false;
  const uint32_t* col;
  const uint32_t* visited;
  uint32_t* next;
  uint32_t* omark;
  uint32_t* onew;
  __device__ __forceinline__ Aux aux(uint32_t) const { return {}; }
  __device__ __forceinline__ void edge(const Aux&, uint64_t e) const {
    const uint32_t t = __ldcs(col + e);
    if (t & kRemote) {
      const uint32_t s = t & ~kRemote, m = 1u << (s & 31);
      if (!(omark[s >> 5] & m)) {
        const uint32_t old = atomicOr(&omark[s >> 5], m);
        if (!(old & m)) atomicOr(&onew[s >> 5], m);
      }
    } else {
      const uint32_t m = 1u << (t & 31);
      if (!(__ldg(visited + (t >> 5)) & m) && !(next[t >> 5] & m)) atomicOr(&next[t >> 5], m);
    }
  }
};

__global__ void k_bfs_scatter(const uint32_t* ibits, const uint32_t* lid, uint64_t I,
                              const uint32_t* visited, uint32_t* next) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < I; j += stride) {
    if (!((ibits[j >> 5] >> (j & 31)) & 1u)) continue;
    const uint32_t v = lid[j];
    if (!bit_test(visited, v)) bit_set_atomic(next, v);
  }
}

void* send_onew(Part& p) { return p.fs.obox_new.get(); }
void* recv_ibits(Part& p) { return p.fs.ibox_bits.get(); }

}  // namespace

void run_bfs(Engine& eng, uint64_t source, uint32_t* out, int mem, tg_stats* st) {
  TG_REQUIRE(out != nullptr, TG_EINVAL, "tg_bfs: NULL levels");
  int ps;
  uint32_t ls;
  eng.locate(source, &ps, &ls);
  ensure_frontier_state(eng);
  eng.launches = 0;
  eng.comm_bytes = 0;
  cudaStream_t s = eng.stream;
  uint64_t bm_bytes = 0;  // one pass over every partition's vertex bitmap
  for (auto& pp : eng.parts) bm_bytes += words_for(pp->Vp) * 4;
  if (eng.P == 1) eng.l2_window(eng.parts[0]->fs.visited.get(), words_for(eng.parts[0]->Vp) * 4);
  time_begin(eng);
  reset_vote(eng);
  for (auto& pp : eng.parts) {
    Part& p = *pp;
    FrontierState& f = p.fs;
    const uint64_t nw = words_for(p.Vp);
    TG_CK(cudaMemsetAsync(f.vals.get(), 0xFF, p.Vp * 4, s));
    TG_CK(cudaMemsetAsync(f.cur.get(), 0, nw * 4, s));
    TG_CK(cudaMemsetAsync(f.next.get(), 0, nw * 4, s));
    TG_CK(cudaMemsetAsync(f.visited.get(), 0, nw * 4, s));
    if (p.S) {
      TG_CK(cudaMemsetAsync(f.obox_mark.get(), 0, p.S / 8, s));
      TG_CK(cudaMemsetAsync(f.obox_new.get(), 0, p.S / 8, s));
    }
    if (p.id == ps) {
      k_seed<<<1, 1, 0, s>>>(f.next.get(), ls, nullptr, 0);
      eng.launches++;
    }
    launch_advance(eng, p, p.ts, f.next.get(), f.cur.get(), f.visited.get(), f.vals.get(), 0,
                   f.counters.get());
    std::swap(f.cur, f.next);
  }
  uint64_t supersteps = 0, frontier = 1, edges_total = 0;
  for (uint32_t L = 0;; ++L) {
    reset_vote(eng);
    for (auto& pp : eng.parts) {
      Part& p = *pp;
      FrontierState& f = p.fs;
      launch_compact(eng, p.ts);
      BfsOp op{p.col.get(), f.visited.get(), f.next.get(), f.obox_mark.get(), f.obox_new.get()};
      launch_expand(eng, p, p.ts, f.cur.get(), op, TG_K_BFS_EXPAND, f.counters.get() + 1);
    }
    supersteps++;
    if (eng.P > 1) {
      eng.prof_begin(TG_K_EXCHANGE);
      exchange(eng, send_onew, recv_ibits, 0, false);
      for (auto& pp : eng.parts) {
        Part& p = *pp;
        if (p.S) TG_CK(cudaMemsetAsync(p.fs.obox_new.get(), 0, p.S / 8, s));
        if (p.I) {
          k_bfs_scatter<<<grid_for(p.I, 256), 256, 0, s>>>(p.fs.ibox_bits.get(), p.ibox_lid.get(),
                                                           p.I, p.fs.visited.get(),
                                                           p.fs.next.get());
          TG_CK(cudaGetLastError());
          eng.launches++;
        }
      }
      eng.prof_end(TG_K_EXCHANGE);
    }
    for (auto& pp : eng.parts) {
      Part& p = *pp;
      FrontierState& f = p.fs;
      launch_advance(eng, p, p.ts, f.next.get(), f.cur.get(), f.visited.get(), f.vals.get(), L + 1,
                     f.counters.get());
      std::swap(f.cur, f.next);
    }
    const Vote v = read_vote(eng);
    // expand: 4 B col per edge, 16 B row offsets per frontier vertex, frontier +
    // visited + next bitmaps one pass each
    eng.prof_bytes(TG_K_BFS_EXPAND, 4.0 * v.edges + 16.0 * frontier + 3.0 * bm_bytes);
    edges_total += v.edges;
    frontier = v.count;
    if (v.count == 0) break;  // termination vote
    TG_REQUIRE(supersteps <= eng.V + 1, TG_EINTERNAL, "tg_bfs: superstep bound exceeded");
  }
  const double ms = time_end(eng);
  eng.l2_window(nullptr, 0);
  if (st) {
    st->device_ms = ms;
    st->supersteps = supersteps;
    uint64_t nreached = 0;
    st->traversed_edges = reached_outdeg_u32(eng, &nreached);
    TG_REQUIRE(st->traversed_edges == edges_total, TG_EINTERNAL,
               "tg_bfs: expanded edges != sum of reached out-degrees");
    // 4 B per traversed edge (col), 16 B row offsets + 4 B level write per
    // reached vertex, three bitmap passes (frontier, next, visited) per superstep.
    st->algorithmic_bytes = 4 * st->traversed_edges + 20 * nreached + 3 * bm_bytes * (supersteps + 1);
    st->comm_bytes = eng.comm_bytes;
    st->launches = eng.launches;
  }
  collect_u32(eng, out, mem);
}

}  // namespace tg
