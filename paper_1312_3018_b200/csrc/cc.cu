// cc.cu -- connected components by minimum-label propagation over BSP
// supersteps ("minimum 'label' in a connected components
// algorithm" -- a source-reducible combiner; P:316 / §9.4; Table 5 note:
// CC operates on the UNDIRECTED graph).  Reading A29: the
// engine's directed multigraph is read as undirected (weak components), each
// directed edge standing for both directions; label[v] = the smallest GLOBAL
// id in v's component.
//
// The paper materialises the symmetrised graph (Table 5 doubles CC's edges);
// here the out-CSR and the in-CSR the engine already holds ARE the two
// directions, so nothing is duplicated.  Per superstep and partition, with the
// active set = vertices whose label dropped in the previous superstep (all
// vertices at the start, labels = own global ids):
//   push      : out-CSR, active u -> every target t: label[t] = min(label[t],
//               label[u]) (RED.MIN), t active on improvement; remote t: min
//               into its outbox slot (the min-combiner of P:182);
//   reverse   : in-CSR (local rows), active v -> every local source u of an
//               in-edge (u, v): label[u] = min(label[u], label[v]);
//   communicate (P > 1): forward -- outbox label minima to the owners' inboxes;
//               reverse -- each owner publishes the label of every boundary
//               vertex that was active (else INF) into the referencing
//               partitions' slots (the pull path of BC), which lower
//               the local sources of that slot's in-CSR row;
//   advance   : next-active bitmap -> vote; stop when no label moved.
// Fused exchange (Engine::fused, default): the push kernel RED.MINs outbox
// improvements straight into the owners' inbox slots, and the owners' pack
// kernel stores the published labels straight into the referencing
// partitions' ghost slots; the communication phase is the arrival barrier.
// Labels only decrease and every label is the id of a vertex in the same
// component, so any interleaving reaches the same fixed point: the minimum.
#include <cstdio>

#include "frontier.cuh"

namespace tg {

namespace {

struct CcPushOp {  // out-CSR
  using Aux = uint32_t;
  static constexpr bool kReduce = false, kFilter = false;
  const uint32_t* col;
  uint32_t* label;
  uint32_t* next;
  uint32_t* obox;
  RemoteOut rout;  // fused: improvements of the local outbox minimum also go
  bool fused;      // straight to the owner's inbox slot (RED.MIN, running minimum)
  __device__ __forceinline__ Aux aux(uint32_t v) const { return label[v]; }
  // split walker (frontier.cuh): column, then the target's label (or outbox
  // minimum), then the min-reductions
  static constexpr bool kSplit = true;
  static constexpr int kUnroll = 4;
  struct Pre {
    uint32_t t;
  };
  struct St {
    uint32_t cur;
  };
  __device__ __forceinline__ Pre pre(uint64_t e) const { return {__ldcs(col + e)}; }
  __device__ __forceinline__ St st(const Pre& p) const {
    return {(p.t & kRemote) ? obox[p.t & ~kRemote] : label[p.t]};
  }
  __device__ __forceinline__ void fin(const Aux& l, const Pre& p, const St& q) const {
    if (!(l < q.cur)) return;
    const uint32_t t = p.t;
    if (t & kRemote) {
      const uint32_t s = t & ~kRemote;
      atomicMin(&obox[s], l);
      if (fused) atomicMin(rout.slot<uint32_t>(s), l);
    } else {
      atomicMin(&label[t], l);
      atomicOr(&next[t >> 5], 1u << (t & 31));
    }
  }
};

struct CcRevOp {  // in-CSR local rows: v active, entries = local sources u
  using Aux = uint32_t;
  static constexpr bool kReduce = false, kFilter = false;
  const uint32_t* in_col;
  uint32_t* label;
  uint32_t* next;
  __device__ __forceinline__ Aux aux(uint32_t v) const { return label[v]; }
  static constexpr bool kSplit = true;  // in_col, then the source's label, then the min
  static constexpr int kUnroll = 4;
  struct Pre {
    uint32_t u;
  };
  struct St {
    uint32_t cur;
  };
  __device__ __forceinline__ Pre pre(uint64_t e) const { return {__ldcs(in_col + e)}; }
  __device__ __forceinline__ St st(const Pre& p) const { return {label[p.u]}; }
  __device__ __forceinline__ void fin(const Aux& l, const Pre& p, const St& q) const {
    if (l < q.cur) {
      atomicMin(&label[p.u], l);
      atomicOr(&next[p.u >> 5], 1u << (p.u & 31));
    }
  }
};

// Referencing side of the reverse exchange as a walker over the outbox rows of
// the in-CSR (rows Vp + s, tiles over every in-CSR row): a slot whose owner
// published a label (ghost != INF) is an active row with Aux = that label, and
// lowers the row's local sources.  Replaces a warp per slot, which left 31
// lanes idle on the typical 1-2-entry outbox row and visited every slot.
struct CcGhostOp {
  using Aux = uint32_t;
  static constexpr bool kReduce = false, kFilter = false;
  const uint32_t* in_col;
  uint32_t* label;
  uint32_t* next;
  const uint32_t* ghost;  // [S] published labels (INF = none)
  uint32_t Vp;
  __device__ __forceinline__ Aux aux(uint32_t r) const { return r >= Vp ? ghost[r - Vp] : kInf; }
  static constexpr bool kSplit = true;
  static constexpr int kUnroll = 4;
  struct Pre {
    uint32_t u;
  };
  struct St {
    uint32_t cur;
  };
  __device__ __forceinline__ Pre pre(uint64_t e) const { return {__ldcs(in_col + e)}; }
  __device__ __forceinline__ St st(const Pre& p) const { return {label[p.u]}; }
  __device__ __forceinline__ void fin(const Aux& l, const Pre& p, const St& q) const {
    if (l < q.cur) {
      atomicMin(&label[p.u], l);
      atomicOr(&next[p.u >> 5], 1u << (p.u & 31));
    }
  }
};

// active rows of the whole in-CSR [0, Vp + S) for CcGhostOp: outbox rows
// whose ghost holds a label (thread per row, one ballot per word)
__global__ void k_cc_ext(const uint32_t* ghost, uint64_t Vp, uint64_t R, uint32_t* ext) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t n = (R + 31) / 32 * 32;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += stride) {
    const bool b = r >= Vp && r < R && ghost[r - Vp] != kInf;
    const uint32_t m = __ballot_sync(0xffffffffu, b);
    if ((threadIdx.x & 31) == 0) ext[r >> 5] = m;
  }
}

// labels = global ids; every vertex active (next = all ones over [0, Vp))
__global__ void k_cc_init(const uint32_t* global_of, uint64_t Vp, uint32_t* label, uint32_t* next) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < Vp; v += stride) {
    label[v] = global_of[v];
    if ((v & 31) == 0) {
      const uint64_t left = Vp - v;
      next[v >> 5] = left >= 32 ? 0xFFFFFFFFu : ((1u << left) - 1u);
    }
  }
}

// owner side of the forward exchange: min-combine received labels
__global__ void k_cc_scatter(const uint32_t* msg, const uint32_t* lid, uint64_t I, uint32_t* label,
                             uint32_t* next) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < I; j += stride) {
    const uint32_t m = msg[j];
    if (m == kInf) continue;
    const uint32_t v = lid[j];
    if (v != kInf && m < label[v]) {
      const uint32_t old = atomicMin(&label[v], m);
      if (m < old) bit_set_atomic(next, v);
    }
  }
}

// owner side of the reverse exchange: label of each active boundary vertex
// (fused, pack == nullptr: stored straight into the referencing partitions'
// ghost slots through the reverse RemoteOut)
__global__ void k_cc_pack(const uint32_t* lid, uint64_t I, const uint32_t* active,
                          const uint32_t* label, uint32_t* pack, RemoteOut rin) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < I; j += stride) {
    const uint32_t v = lid[j];
    const uint32_t x = (v != kInf && bit_test(active, v)) ? label[v] : kInf;
    if (pack) pack[j] = x;
    else *rin.slot<uint32_t>((uint32_t)j) = x;
  }
}

// referencing side: a slot whose vertex published a label lowers the local
// sources of the slot's in-CSR row Vp + s (one warp per slot)
__global__ void k_cc_ghost(const uint32_t* ghost, uint64_t S, uint64_t Vp, const uint64_t* in_off,
                           const uint32_t* in_col, uint32_t* label, uint32_t* next,
                           unsigned long long* edges) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long cnt = 0;
  for (uint64_t s = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; s < S; s += nwarps) {
    const uint32_t g = ghost[s];
    if (g == kInf) continue;
    const uint64_t b = in_off[Vp + s], e = in_off[Vp + s + 1];
    cnt += e - b;
    for (uint64_t i = b + lane; i < e; i += 32) {
      const uint32_t u = in_col[i];
      if (g < label[u]) {
        atomicMin(&label[u], g);
        atomicOr(&next[u >> 5], 1u << (u & 31));
      }
    }
  }
  if (lane == 0 && cnt) atomicAdd(edges, cnt);
}

void* send_obox(Part& p) { return p.fs.obox_u32.get(); }
void* recv_ibox(Part& p) { return p.arena_fwd.get(); }
void* send_pack(Part& p) { return p.fs.ibox_u32.get(); }
void* recv_ghost(Part& p) { return p.arena_rev.get(); }

}  // namespace

void run_cc(Engine& eng, uint32_t* out, int mem, tg_stats* st) {
  TG_REQUIRE(out != nullptr || (eng.multi() && eng.rank != 0), TG_EINVAL, "tg_cc: NULL labels");
  TG_REQUIRE(eng.has_in, TG_EINVAL, "tg_cc: engine built without the in-CSR (build_in_csr)");
  ensure_frontier_state(eng);
  for (auto& pp : eng.parts)
    if (eng.P > 1 && pp->fs.ibox_u32.n < std::max<uint64_t>(pp->I, 1))
      pp->fs.ibox_u32.alloc(std::max<uint64_t>(pp->I, 1));
  eng.launches = 0;
  eng.comm_bytes = 0;
  cudaStream_t s = eng.stream;
  const DirectionPolicy tclock;  // trace laps only
  const bool trace = direction_policy(eng).trace;
  uint64_t bm_bytes = 0;
  for (auto& pp : eng.parts) bm_bytes += words_for(pp->Vp) * 4;
  // TG_CC_GHOST_WARP=1: the round-1 warp-per-slot ghost pass (A/B)
  const bool ghost_warp = std::getenv("TG_CC_GHOST_WARP") && std::getenv("TG_CC_GHOST_WARP")[0] == '1';
  time_begin(eng);
  eng.each_part([&](Part& p) {
    cudaStream_t s = eng.stream;
    FrontierState& f = p.fs;
    const uint64_t nw = words_for(p.Vp);
    TG_CK(cudaMemsetAsync(f.counters.get(), 0, 64, s));
    TG_CK(cudaMemsetAsync(f.cur.get(), 0, nw * 4, s));
    TG_CK(cudaMemsetAsync(f.next.get(), 0, nw * 4, s));
    if (p.S) TG_CK(cudaMemsetAsync(f.obox_u32.get(), 0xFF, p.S * 4, s));
    if (eng.fused && p.I) TG_CK(cudaMemsetAsync(p.arena_fwd.get(), 0xFF, p.I * 4, s));
    if (p.Vp) {
      k_cc_init<<<grid_for(p.Vp, 256), 256, 0, s>>>(p.global_of.get(), p.Vp, f.vals.get(), f.next.get());
      TG_CK(cudaGetLastError());
      eng.launches++;
    }
    launch_advance(eng, p, p.ts, f.next.get(), f.cur.get(), nullptr, nullptr, 0, f.counters.get());
    std::swap(f.cur, f.next);
  });
  if (eng.fused && eng.multi()) fused_arrival(eng);  // inboxes at INF before any peer writes
  uint64_t supersteps = 0, frontier = eng.V, processed = 0, activations = eng.V;
  for (;;) {
    reset_vote(eng);
    eng.each_part([&](Part& p) {
      cudaStream_t s = eng.stream;
      FrontierState& f = p.fs;
      launch_compact(eng, p.ts);
      CcPushOp op{p.col.get(), f.vals.get(), f.next.get(), f.obox_u32.get(), p.rout(), eng.fused};
      launch_expand(eng, p, p.ts, f.cur.get(), op, TG_K_CC_EXPAND, f.counters.get() + 1);
      if (p.in_ntiles) {
        launch_mark_tiles(eng, in_tiles(p), p.Vp, f.cur.get(), p.ts_in);
        launch_compact(eng, p.ts_in);
        CcRevOp rop{p.in_col.get(), f.vals.get(), f.next.get()};
        launch_expand_on(eng, in_tiles(p), p.ts_in, f.cur.get(), rop, TG_K_CC_EXPAND,
                         f.counters.get() + 1);
      }
    });
    supersteps++;
    if (eng.P > 1) {
      eng.prof_begin(TG_K_EXCHANGE);
      eng.each_part([&](Part& p) {
        cudaStream_t s = eng.stream;
        if (!p.I) return;
        k_cc_pack<<<grid_for(p.I, 256), 256, 0, s>>>(p.ibox_lid.get(), p.I, p.fs.cur.get(),
                                                     p.fs.vals.get(),
                                                     eng.fused ? nullptr : p.fs.ibox_u32.get(),
                                                     p.rin());
        eng.launches++;
      });
      TG_CK(cudaGetLastError());
      // fused: forward minima and reverse ghost labels are already in the
      // receivers' arenas; readers finish before the vote, writers start after it
      if (eng.fused) {
        fused_arrival(eng);
        for (auto& pp : eng.parts) eng.comm_bytes += (pp->S + pp->I) * 4;
      } else {
        exchange(eng, send_obox, recv_ibox, 4, false);
        exchange(eng, send_pack, recv_ghost, 4, true);
      }
      eng.each_part([&](Part& p) {
        cudaStream_t s = eng.stream;
        FrontierState& f = p.fs;
        if (p.I) {
          k_cc_scatter<<<grid_for(p.I, 256), 256, 0, s>>>(
              reinterpret_cast<const uint32_t*>(p.arena_fwd.get()), p.ibox_lid.get(), p.I,
              f.vals.get(), f.next.get());
          eng.launches++;
        }
        TG_CK(cudaGetLastError());
      });
      eng.prof_end(TG_K_EXCHANGE);
      // reverse direction, referencing side: published labels lower the local
      // sources of the outbox rows (compute on the received ghosts)
      eng.each_part([&](Part& p) {
        cudaStream_t s = eng.stream;
        FrontierState& f = p.fs;
        if (p.S && p.in_all_ntiles && !ghost_warp) {
          const uint64_t R = p.Vp + p.S;
          if (p.bcs.ext.n < words_for(R)) p.bcs.ext.alloc(words_for(R));
          const uint32_t* gh = reinterpret_cast<const uint32_t*>(p.arena_rev.get());
          k_cc_ext<<<grid_for(R, 256, 148u * 16u), 256, 0, s>>>(gh, p.Vp, R, p.bcs.ext.get());
          TG_CK(cudaGetLastError());
          eng.launches++;
          launch_mark_tiles(eng, in_all_tiles(p), R, p.bcs.ext.get(), p.ts_in);
          launch_compact(eng, p.ts_in);
          CcGhostOp gop{p.in_col.get(), f.vals.get(), f.next.get(), gh, (uint32_t)p.Vp};
          launch_expand_on(eng, in_all_tiles(p), p.ts_in, p.bcs.ext.get(), gop, TG_K_CC_EXPAND,
                           f.counters.get() + 1);
        } else if (p.S) {
          k_cc_ghost<<<grid_for(p.S * 32, 256, 148u * 16u), 256, 0, s>>>(
              reinterpret_cast<const uint32_t*>(p.arena_rev.get()), p.S, p.Vp, p.in_off.get(),
              p.in_col.get(), f.vals.get(), f.next.get(), f.counters.get() + 1);
          eng.launches++;
        }
        TG_CK(cudaGetLastError());
      });
    }
    eng.each_part([&](Part& p) {
      cudaStream_t s = eng.stream;
      FrontierState& f = p.fs;
      launch_advance(eng, p, p.ts, f.next.get(), f.cur.get(), nullptr, nullptr, 0, f.counters.get());
      std::swap(f.cur, f.next);
    });
    const Vote v = read_vote(eng);
    // both directions: col/in_col 4 + label[target] 4 per edge; offsets 16 +
    // label 4 per active vertex (each CSR); active + next bitmaps per pass
    eng.prof_bytes(TG_K_CC_EXPAND, 8.0 * v.edges + 40.0 * frontier + 3.0 * bm_bytes);
    if (trace)
      std::fprintf(stderr, "[tg cc] step=%llu active=%llu edges=%llu next=%llu ms=%.3f\n",
                   (unsigned long long)supersteps, (unsigned long long)frontier,
                   (unsigned long long)v.edges, (unsigned long long)v.count, tclock.lap(s));
    processed += v.edges;
    frontier = v.count;
    activations += v.count;
    if (v.count == 0) break;  // termination vote
    TG_REQUIRE(supersteps <= eng.V + 1, TG_EINTERNAL, "tg_cc: superstep bound exceeded");
  }
  const double ms = time_end(eng);
  if (st) {
    st->device_ms = ms;
    st->supersteps = supersteps;
    st->relaxations = processed;
    st->traversed_edges = eng.E;  // every input edge, once (undirected reading A29)
    st->algorithmic_bytes = 8 * processed + 40 * activations + 3 * bm_bytes * supersteps;
    st->comm_bytes = eng.comm_bytes;
    st->launches = eng.launches;
  }
  collect_u32(eng, out, mem);
}

}  // namespace tg
