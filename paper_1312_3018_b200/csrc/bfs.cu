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
//             level buffer under min-combine).  Fused (default, Engine::fused):
//             the first-time mark is an atomicOr straight into the owner's
//             inbox bitmap (RemoteOut; peer memory across processes), so the
//             phase is only the arrival barrier.
//   scatter : inbox bit set and owner vertex unvisited -> next bit
//             (totem_engine_scatter_inbox_min).
//   advance : next bitmap -> level[v] = L+1, visited |= next, vote count
//             (termination when every partition's count is 0).
#include <cstdio>

#include "frontier.cuh"

namespace tg {

namespace {

struct BfsOp {
  using Aux = Empty;
  static constexpr bool kReduce = false, kFilter = false;
  const uint32_t* col;
  const uint32_t* visited;
  uint32_t* next;
  uint32_t* omark;
  uint32_t* onew;
  RemoteOut rout;  // fused: first-time remote marks go straight to the owner's inbox bits
  bool fused;
  __device__ __forceinline__ Aux aux(uint32_t) const { return {}; }
  // split walker (frontier.cuh): column, then the target's state words, then
  // the test-and-set reductions
  static constexpr bool kSplit = true;
  static constexpr int kUnroll = 2;
  struct Pre {
    uint32_t t;
  };
  struct St {
    uint32_t a, b;  // local: visited / next word; remote: "ever sent" word
  };
  __device__ __forceinline__ Pre pre(uint64_t e) const { return {__ldcs(col + e)}; }
  __device__ __forceinline__ St st(const Pre& p) const {
    if (p.t & kRemote) return {omark[(p.t & ~kRemote) >> 5], 0u};
    return {__ldg(visited + (p.t >> 5)), next[p.t >> 5]};
  }
  __device__ __forceinline__ void fin(const Aux&, const Pre& p, const St& q) const {
    const uint32_t t = p.t;
    if (t & kRemote) {
      const uint32_t s = t & ~kRemote, m = 1u << (s & 31);
      if (!(q.a & m)) {
        const uint32_t old = atomicOr(&omark[s >> 5], m);
        if (!(old & m)) atomicOr(fused ? rout.word(s) : &onew[s >> 5], m);
      }
    } else {
      const uint32_t m = 1u << (t & 31);
      if (!(q.a & m) && !(q.b & m)) atomicOr(&next[t >> 5], m);
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

// Bottom-up superstep (direction-optimizing BFS):
// every unvisited vertex scans its in-edges until it finds a parent in the
// current frontier.  One warp per visited-bitmap word, one lane per vertex; the
// warp owns its word of `next`, so no atomics.  Same levels as top-down.
// P > 1: the pull walks the ghost in-CSR (PRGhost): a source u >= Vp is ghost
// u - Vp, whose frontier bit its owner published into gbits.
template <bool kGhost>
__global__ void __launch_bounds__(256) k_bfs_bottom_up(const uint64_t* in_off,
                                                       const uint32_t* in_col, const uint32_t* cur,
                                                       const uint32_t* visited,
                                                       const uint32_t* has_in, uint32_t* next,
                                                       uint64_t Vp, unsigned long long* edges,
                                                       const uint32_t* gbits) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t nwords = words_for(Vp);
  unsigned long long cnt = 0;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < nwords; w += nwarps) {
    // candidates: unvisited vertices with an in-edge (no offset reads for the
    // ~half of RMAT vertices that have none)
    const uint32_t open = ~visited[w] & has_in[w];
    const uint64_t v = w * 32 + lane;
    const bool cand = v < Vp && ((open >> lane) & 1u);
    if (!__ballot_sync(0xffffffffu, cand)) continue;
    bool found = false;
    if (cand) {
      const uint64_t b = in_off[v], e = in_off[v + 1];
      for (uint64_t i = b; i < e; ++i) {
        const uint32_t u = __ldg(in_col + i);
        cnt++;
        bool in_f;
        if (kGhost && u >= Vp) {
          const uint32_t g = u - (uint32_t)Vp;
          in_f = (__ldg(gbits + (g >> 5)) >> (g & 31)) & 1u;
        } else {
          in_f = (__ldg(cur + (u >> 5)) >> (u & 31)) & 1u;
        }
        if (in_f) {
          found = true;
          break;
        }
      }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, found);
    if (lane == 0 && m) next[w] = m;
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  if (lane == 0 && cnt) atomicAdd(edges, cnt);
}

void* send_onew(Part& p) { return p.fs.obox_new.get(); }
void* recv_ibits(Part& p) { return p.arena_fwd.get(); }

}  // namespace

void run_bfs(Engine& eng, uint64_t source, uint32_t* out, int mem, tg_stats* st) {
  TG_REQUIRE(out != nullptr || (eng.multi() && eng.rank != 0), TG_EINVAL, "tg_bfs: NULL levels");
  int ps;
  uint32_t ls;
  eng.locate(source, &ps, &ls);
  ensure_frontier_state(eng);
  eng.launches = 0;
  eng.comm_bytes = 0;
  uint64_t visited_total = 1;
  uint64_t bm_bytes = 0;  // one pass over every partition's vertex bitmap
  for (auto& pp : eng.parts) bm_bytes += words_for(pp->Vp) * 4;
  if (eng.P == 1) eng.l2_window(eng.parts[0]->fs.visited.get(), words_for(eng.parts[0]->Vp) * 4);
  // bottom-up steps at P > 1 pull over the ghost in-CSR: built once, outside
  // the timed region (collective across processes)
  if (eng.P > 1 && eng.has_in && direction_policy(eng).mode != 1) build_pr_ghost(eng);
  time_begin(eng);
  reset_vote(eng);
  eng.each_part([&](Part& p) {
    cudaStream_t s = eng.stream;
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
    if (eng.fused && p.I) TG_CK(cudaMemsetAsync(p.arena_fwd.get(), 0, p.I / 8, s));
    if (p.id == ps) {
      k_seed<<<1, 1, 0, s>>>(f.next.get(), ls, nullptr, 0);
      eng.launches++;
    }
    launch_advance(eng, p, p.ts, f.next.get(), f.cur.get(), f.visited.get(), f.vals.get(), 0,
                   f.counters.get(), f.counters.get() + 2);
    std::swap(f.cur, f.next);
  });
  // fused: every inbox bitmap is clear before any peer writes into it (the vote
  // below synchronizes the ranks when direction optimization reads it; the
  // barrier covers the forced top-down mode)
  if (eng.fused && eng.multi()) fused_arrival(eng);
  const DirectionPolicy dir = direction_policy(eng);
  uint64_t supersteps = 0, frontier = 1, edges_total = 0, bu_steps = 0;
  uint64_t mf = dir.mode == 1 ? 0 : read_vote(eng).degsum;  // out-edges of the frontier
  uint64_t explored = mf;
  bool was_bu = false;
  for (uint32_t L = 0;; ++L) {
    reset_vote(eng);
    const bool bottom_up =
        dir.bottom_up(eng, frontier, mf, eng.E - std::min(explored, eng.E), was_bu, dir.alpha);
    was_bu = bottom_up;
    if (bottom_up && eng.P > 1) {
      // the frontier bits of every published source -> the peers' ghost bits
      eng.prof_begin(TG_K_EXCHANGE);
      eng.each_part([&](Part& p) { publish_frontier_bits(eng, p, p.fs.cur.get()); });
      fused_arrival(eng);
      eng.prof_end(TG_K_EXCHANGE);
    }
    eng.each_part([&](Part& p) {
      cudaStream_t s = eng.stream;
      FrontierState& f = p.fs;
      launch_compact(eng, p.ts);  // drains the tile marks even when unused
      if (bottom_up) {
        eng.prof_begin(TG_K_BFS_EXPAND);
        const unsigned grid = grid_for(words_for(p.Vp) * 32, 256, 148u * 16u);
        if (eng.P > 1)
          k_bfs_bottom_up<true><<<grid, 256, 0, s>>>(p.gh.off.get(), p.gh.col.get(), f.cur.get(),
                                                    f.visited.get(), p.gh.nz.get(), f.next.get(),
                                                    p.Vp, f.counters.get() + 1, p.gh.bits.get());
        else
          k_bfs_bottom_up<false><<<grid, 256, 0, s>>>(p.in_off.get(), p.in_col.get(), f.cur.get(),
                                                     f.visited.get(), p.in_nz.get(), f.next.get(),
                                                     p.Vp, f.counters.get() + 1, nullptr);
        eng.prof_end(TG_K_BFS_EXPAND);
        TG_CK(cudaGetLastError());
        eng.launches++;
      } else {
        BfsOp op{p.col.get(), f.visited.get(), f.next.get(), f.obox_mark.get(), f.obox_new.get(),
                 p.rout(), eng.fused};
        launch_expand(eng, p, p.ts, f.cur.get(), op, TG_K_BFS_EXPAND, f.counters.get() + 1);
      }
    });
    bu_steps += bottom_up;
    supersteps++;
    if (eng.P > 1 && !bottom_up) {  // a bottom-up step only sets owned vertices: no messages
      eng.prof_begin(TG_K_EXCHANGE);
      if (eng.fused) {
        fused_arrival(eng);
        for (auto& pp : eng.parts) eng.comm_bytes += pp->S / 8;  // bitmap capacity written into
      } else {
        exchange(eng, send_onew, recv_ibits, 0, false);
      }
      eng.each_part([&](Part& p) {
        cudaStream_t s = eng.stream;
        if (p.S && !eng.fused) TG_CK(cudaMemsetAsync(p.fs.obox_new.get(), 0, p.S / 8, s));
        if (p.I) {
          k_bfs_scatter<<<grid_for(p.I, 256), 256, 0, s>>>(
              reinterpret_cast<const uint32_t*>(p.arena_fwd.get()), p.ibox_lid.get(),
                                                           p.I, p.fs.visited.get(),
                                                           p.fs.next.get());
          TG_CK(cudaGetLastError());
          eng.launches++;
          // fused: the inbox bits are consumed; clear them for the next superstep
          // (peers write again only after the vote below has synchronized)
          if (eng.fused) TG_CK(cudaMemsetAsync(p.arena_fwd.get(), 0, p.I / 8, s));
        }
      });
      eng.prof_end(TG_K_EXCHANGE);
    }
    eng.each_part([&](Part& p) {
      FrontierState& f = p.fs;
      launch_advance(eng, p, p.ts, f.next.get(), f.cur.get(), f.visited.get(), f.vals.get(), L + 1,
                     f.counters.get(), dir.mode == 1 ? nullptr : f.counters.get() + 2);
      std::swap(f.cur, f.next);
    });
    const Vote v = read_vote(eng);
    mf = v.degsum;
    explored += mf;
    // top-down: 4 B col per edge, 16 B row offsets per frontier vertex, frontier +
    // visited + next bitmaps one pass each; bottom-up: 4 B in_col per examined
    // in-edge, 16 B in-offsets per unvisited vertex
    if (bottom_up)
      eng.prof_bytes(TG_K_BFS_EXPAND, 4.0 * v.edges + 16.0 * (eng.V - visited_total) + 3.0 * bm_bytes);
    else
      eng.prof_bytes(TG_K_BFS_EXPAND, 4.0 * v.edges + 16.0 * frontier + 3.0 * bm_bytes);
    visited_total += v.count;
    if (dir.trace)
      std::fprintf(stderr, "[tg bfs] L=%u %s frontier=%llu edges=%llu next=%llu next_mf=%llu ms=%.3f\n",
                   L, bottom_up ? "bottom-up" : "top-down", (unsigned long long)frontier,
                   (unsigned long long)v.edges, (unsigned long long)v.count,
                   (unsigned long long)v.degsum, dir.lap(eng.stream));
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
    st->relaxations = edges_total;
    uint64_t nreached = 0;
    if (dir.mode != 1) {  // the frontiers' exact out-degree sums cover every reached vertex once
      st->traversed_edges = explored;
      nreached = visited_total;
    } else {
      st->traversed_edges = reached_outdeg_u32(eng, &nreached);
    }
    TG_REQUIRE(bu_steps || st->traversed_edges == edges_total, TG_EINTERNAL,
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
