// sssp.cu -- Bellman-Ford SSSP over BSP supersteps (Fig. 20).
// Per superstep and partition:
//   compute : every edge (v,t,w) of an active v: nd = dist[v] + w; local t:
//             atomicMin(dist[t], nd) and activate t on improvement (Fig. 20
//             lines 7-12); remote t: atomicMin into its outbox slot (the
//             min-combiner of P:182).  nd is formed in 64 bits; a value that
//             does not fit u32 raises the overflow flag (TG_EINTERNAL).
//   communicate: the full outbox value array (full buffer every
//             superstep; min-combine makes re-sending idempotent).  Fused
//             (default): the local outbox minimum filters, and each improvement
//             is also a RED.MIN straight into the owner's inbox slot
//             (RemoteOut), which then holds the running minimum; the phase is
//             only the arrival barrier.
//   scatter : dist[v] = min(dist[v], msg), activate on improvement.
//   advance : next-active bitmap -> vote count + the smallest active distance.
//
// Degree-aware near-far schedule (reading A19b): an active vertex of
// out-degree >= hub_deg (128) is relaxed in a superstep only if dist[v] <
// min_active_dist + Delta (1); otherwise it stays active for a later
// superstep (after Davidson et al. 2014, the GPU SSSP work the paper cites at
// P:649).  Rows below hub_deg always relax.  Any schedule of Bellman-Ford
// relaxations reaches the same fixed point, so distances are identical; the
// schedule only removes redundant relaxations of hubs (RMAT-28: 62 GB instead
// of 92 GB, profiles/r01_sssp_hub_sweep.txt).  TG_SSSP_DELTA=0 gives plain
// Bellman-Ford; TG_SSSP_HUB_DEG=0 makes every row wait (plain near-far).
#include <cstdio>
#include <cstdlib>

#include "frontier.cuh"

namespace tg {

namespace {

template <class W>  // weight storage: uint8_t when every weight < 256, else uint32_t
struct SsspOp {
  using Aux = uint32_t;
  static constexpr bool kReduce = false, kFilter = true;
  const uint32_t* col;
  const W* w;
  uint32_t* dist;
  uint32_t* next;
  uint32_t* obox;
  unsigned long long* overflow;
  RemoteOut rout;    // fused: improvements of the local outbox minimum are forwarded
  bool fused;        // as RED.MIN straight into the owner's inbox slot
  uint32_t thresh;   // relax rows with dist < thresh now, defer the others ...
  uint32_t hub_end;  // ... but only rows v < hub_end (the high-degree prefix)
  // dense superstep: the next frontier is derived afterwards from the distances
  // that dropped (k_mark_dropped), so a relaxation issues one reduction (the
  // RED.MIN) instead of two -- the L2 request rate is what bounds this walk
  bool mark;
  // local ids >= nz_end have out-degree 0: a sink whose distance drops has
  // nothing to relax, so it is not activated (its distance is still set)
  uint32_t nz_end;
  __device__ __forceinline__ Aux aux(uint32_t v) const { return dist[v]; }
  __device__ __forceinline__ bool keep(uint32_t v, const Aux& dv) const {
    return v >= hub_end || dv < thresh;
  }
  __device__ __forceinline__ void defer(uint32_t v) const { bit_set_atomic(next, v); }
  // split walker (frontier.cuh): column + weight, then the target's current
  // distance (or outbox minimum), then the relaxation
  static constexpr bool kSplit = true;
  static constexpr int kUnroll = 4;
  struct Pre {
    uint32_t t, w;
  };
  struct St {
    uint32_t cur;
  };
  __device__ __forceinline__ Pre pre(uint64_t e) const {
    return {__ldcs(col + e), (uint32_t)__ldcs(w + e)};
  }
  __device__ __forceinline__ St st(const Pre& p) const {
    return {(p.t & kRemote) ? obox[p.t & ~kRemote] : dist[p.t]};
  }
  __device__ __forceinline__ void fin(const Aux& dv, const Pre& p, const St& q) const {
    const uint64_t nd64 = (uint64_t)dv + p.w;
    if (nd64 >= (uint64_t)kInf) {
      *overflow = 1ull;
      return;
    }
    const uint32_t nd = (uint32_t)nd64, t = p.t;
    if (!(nd < q.cur)) return;
    if (t & kRemote) {
      const uint32_t s = t & ~kRemote;
      atomicMin(&obox[s], nd);
      if (fused) atomicMin(rout.slot<uint32_t>(s), nd);
    } else {
      // nd < dist[t] as read means t's distance drops in this superstep (to nd
      // or below: values only decrease and stale reads are only ever higher),
      // so t is active next superstep.  Both updates are fire-and-forget
      // reductions (RED.MIN / RED.OR): no round trip on the critical path.
      atomicMin(&dist[t], nd);
      if (mark && t < nz_end) atomicOr(&next[t >> 5], 1u << (t & 31));
    }
  }
};

// dense superstep epilogue: next |= {v : dist[v] < prev[v]} (one ballot per word)
__global__ void k_mark_dropped(const uint32_t* __restrict__ dist, const uint32_t* __restrict__ prev,
                               uint64_t Vp, uint32_t* next) {
  const uint64_t n = (Vp + 31) / 32 * 32;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    const bool d = v < Vp && __ldcs(dist + v) < __ldcs(prev + v);
    const uint32_t m = __ballot_sync(0xffffffffu, d);
    if ((threadIdx.x & 31) == 0 && m) next[v >> 5] |= m;
  }
}

__global__ void k_sssp_scatter(const uint32_t* msg, const uint32_t* lid, uint64_t I, uint32_t* dist,
                               uint32_t* next) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < I; j += stride) {
    const uint32_t m = msg[j];
    if (m == kInf) continue;
    const uint32_t v = lid[j];
    if (m < dist[v]) {
      const uint32_t old = atomicMin(&dist[v], m);
      if (m < old) bit_set_atomic(next, v);
    }
  }
}

// Dense supersteps by out-degree class (TG_SSSP_CLASS_DIV): when the frontier's
// out-edges exceed E / div, the superstep relaxes the active rows with three
// kernels over the out-degree classes -- local ids are in out-degree order, so
// the classes are id ranges: [0, n_big) a CTA per row, [n_big, n_mid) a warp
// per row (a warp takes a frontier word and walks its active rows), the rest a
// thread per row -- instead of the tile walker, whose per-window scan and
// shuffles cost more than the load balance they buy once most tiles are busy.
// Same relaxation, filter and counters as SsspOp.
template <class W>
struct Relax {
  const uint64_t* row_off;
  const uint32_t* col;
  const W* w;
  uint32_t* dist;
  uint32_t* next;
  uint32_t* obox;
  unsigned long long* overflow;
  RemoteOut rout;
  bool fused;
  uint32_t thresh, hub_end;
  const uint32_t* cur;
  unsigned long long* edges;
  __device__ __forceinline__ bool keep(uint32_t v, uint32_t dv) const {
    return v >= hub_end || dv < thresh;
  }
  __device__ __forceinline__ uint32_t target(uint32_t t) const {
    return (t & kRemote) ? obox[t & ~kRemote] : dist[t];
  }
  __device__ __forceinline__ void relax(uint32_t dv, uint32_t t, uint32_t wt, uint32_t cd) const {
    const uint64_t nd64 = (uint64_t)dv + wt;
    if (nd64 >= (uint64_t)kInf) {
      *overflow = 1ull;
      return;
    }
    const uint32_t nd = (uint32_t)nd64;
    if (!(nd < cd)) return;
    if (t & kRemote) {
      const uint32_t sl = t & ~kRemote;
      atomicMin(&obox[sl], nd);
      if (fused) atomicMin(rout.slot<uint32_t>(sl), nd);
    } else {
      atomicMin(&dist[t], nd);
      atomicOr(&next[t >> 5], 1u << (t & 31));
    }
  }
  // edges [i, e) of a row with distance dv, stride `step`, 4 in flight
  __device__ __forceinline__ void row(uint32_t dv, uint64_t i, uint64_t e, uint32_t step) const {
    for (; i + 3ull * step < e; i += 4ull * step) {
      uint32_t t[4], wt[4], cd[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        t[k] = __ldcs(col + i + k * step);
        wt[k] = (uint32_t)__ldcs(w + i + k * step);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) cd[k] = target(t[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) relax(dv, t[k], wt[k], cd[k]);
    }
    for (; i < e; i += step) {
      const uint32_t t = __ldcs(col + i);
      relax(dv, t, (uint32_t)__ldcs(w + i), target(t));
    }
  }
};

__device__ __forceinline__ void add_edges(unsigned long long* ctr, unsigned long long n) {
#pragma unroll
  for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(ctr, n);
}

template <class W>
__global__ void __launch_bounds__(256) k_sssp_cls_cta(Relax<W> r, uint64_t n_big) {
  __shared__ uint32_t s_dv;
  __shared__ int s_go;
  unsigned long long ed = 0;
  for (uint64_t v = blockIdx.x; v < n_big; v += gridDim.x) {
    if (!((r.cur[v >> 5] >> (v & 31)) & 1u)) continue;  // block-uniform
    if (threadIdx.x == 0) {
      const uint32_t dv = r.dist[v];
      s_dv = dv;
      s_go = r.keep((uint32_t)v, dv);
      if (!s_go) bit_set_atomic(r.next, (uint32_t)v);
    }
    __syncthreads();
    const uint32_t dv = s_dv;
    const int go = s_go;
    __syncthreads();
    if (!go) continue;
    const uint64_t b = r.row_off[v], e = r.row_off[v + 1];
    r.row(dv, b + threadIdx.x, e, blockDim.x);
    if (threadIdx.x == 0) ed += e - b;
  }
  add_edges(r.edges, ed);
}

template <class W>
__global__ void __launch_bounds__(256) k_sssp_cls_warp(Relax<W> r, uint64_t v0, uint64_t v1) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long ed = 0;
  for (uint64_t wd = (v0 >> 5) + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
       wd * 32 < v1; wd += nwarps) {
    uint32_t x = r.cur[wd];
    const uint64_t base = wd * 32;
    if (base < v0) x &= ~0u << (v0 - base);
    if (base + 32 > v1) x &= (v1 - base >= 32) ? ~0u : ((1u << (v1 - base)) - 1u);
    while (x) {
      const uint32_t v = (uint32_t)base + (uint32_t)(__ffs(x) - 1);
      x &= x - 1;
      const uint32_t dv = r.dist[v];
      if (!r.keep(v, dv)) {
        if (lane == 0) bit_set_atomic(r.next, v);
        continue;
      }
      const uint64_t b = r.row_off[v], e = r.row_off[v + 1];
      r.row(dv, b + lane, e, 32);
      if (lane == 0) ed += e - b;
    }
  }
  add_edges(r.edges, ed);
}

template <class W>
__global__ void __launch_bounds__(256) k_sssp_cls_thread(Relax<W> r, uint64_t v0, uint64_t v1) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long ed = 0;
  for (uint64_t v = (v0 & ~31ull) + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
       v < ((v1 + 31) & ~31ull); v += stride) {
    const uint32_t x = r.cur[v >> 5];
    if (!x) continue;  // warp-uniform: one word per warp
    if (v < v0 || v >= v1 || !((x >> (v & 31)) & 1u)) continue;
    const uint32_t dv = r.dist[v];
    if (!r.keep((uint32_t)v, dv)) {
      bit_set_atomic(r.next, (uint32_t)v);
      continue;
    }
    const uint64_t b = r.row_off[v], e = r.row_off[v + 1];
    r.row(dv, b, e, 1);
    ed += e - b;
  }
  add_edges(r.edges, ed);
}

__global__ void k_first_below_u64(const uint64_t* row_off, uint64_t n, uint32_t deg, uint64_t* out) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (row_off[mid + 1] - row_off[mid] >= deg) lo = mid + 1;
    else hi = mid;
  }
  *out = lo;
}

void out_classes(Engine& eng, Part& p) {
  FrontierState& f = p.fs;
  if (f.cls) return;
  DevBuf<uint64_t> d(2);
  k_first_below_u64<<<1, 1, 0, eng.stream>>>(p.row_off.get(), p.nz_end, 2048, d.get());
  k_first_below_u64<<<1, 1, 0, eng.stream>>>(p.row_off.get(), p.nz_end, 32, d.get() + 1);
  TG_CK(cudaGetLastError());
  uint64_t h[2];
  TG_CK(cudaMemcpyAsync(h, d.get(), 16, cudaMemcpyDeviceToHost, eng.stream));
  TG_CK(cudaStreamSynchronize(eng.stream));
  f.n_big = h[0];
  f.n_mid = h[1];
  f.cls = true;
}

template <class W>
void launch_classes(Engine& eng, Part& p, const W* w, uint32_t thresh, uint32_t hubs) {
  FrontierState& f = p.fs;
  cudaStream_t s = eng.stream;
  Relax<W> r{p.row_off.get(), p.col.get(), w, f.vals.get(), f.next.get(), f.obox_u32.get(),
             f.counters.get() + 4, p.rout(), eng.fused, thresh, hubs, f.cur.get(),
             f.counters.get() + 1};
  eng.prof_begin(TG_K_SSSP_EXPAND);
  if (f.n_big) {
    k_sssp_cls_cta<W><<<(unsigned)std::min<uint64_t>(f.n_big, 148u * 64u), 256, 0, s>>>(r, f.n_big);
    eng.launches++;
  }
  if (f.n_mid > f.n_big) {
    k_sssp_cls_warp<W><<<grid_for((f.n_mid - f.n_big), 256, 148u * 16u), 256, 0, s>>>(r, f.n_big,
                                                                                        f.n_mid);
    eng.launches++;
  }
  if (p.nz_end > f.n_mid) {
    k_sssp_cls_thread<W><<<grid_for(p.nz_end - f.n_mid, 256, 148u * 16u), 256, 0, s>>>(r, f.n_mid,
                                                                                         p.nz_end);
    eng.launches++;
  }
  eng.prof_end(TG_K_SSSP_EXPAND);
  TG_CK(cudaGetLastError());
}

void* send_obox(Part& p) { return p.fs.obox_u32.get(); }
void* recv_ibox(Part& p) { return p.arena_fwd.get(); }

uint32_t env_u32(const char* name, uint32_t dflt) {
  if (const char* d = std::getenv(name)) return (uint32_t)std::strtoul(d, nullptr, 10);
  return dflt;
}

// Binary search over the degree-sorted rows: first local id whose out-degree
// is below `deg` (ids are sorted by out-degree descending, build.cu).
__global__ void k_hub_end(const uint64_t* __restrict__ row_off, uint64_t n, uint32_t deg,
                          uint32_t* __restrict__ out) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (row_off[mid + 1] - row_off[mid] >= deg) lo = mid + 1;
    else hi = mid;
  }
  *out = (uint32_t)lo;
}

uint32_t hub_end(Engine& eng, Part& p, uint32_t deg) {
  if (deg == 0) return 0;  // no row is held back by degree
  if (p.hub_deg != deg) {
    DevBuf<uint32_t> d(1);
    k_hub_end<<<1, 1, 0, eng.stream>>>(p.row_off.get(), p.nz_end, deg, d.get());
    TG_CK(cudaGetLastError());
    TG_CK(cudaMemcpyAsync(&p.hub_end, d.get(), 4, cudaMemcpyDeviceToHost, eng.stream));
    TG_CK(cudaStreamSynchronize(eng.stream));
    p.hub_deg = deg;
  }
  return p.hub_end;
}

}  // namespace

void run_sssp(Engine& eng, uint64_t source, uint32_t* out, int mem, tg_stats* st) {
  TG_REQUIRE(out != nullptr || (eng.multi() && eng.rank != 0), TG_EINVAL, "tg_sssp: NULL dist");
  TG_REQUIRE(eng.weighted, TG_EINVAL, "tg_sssp: engine was built without edge weights");
  int ps;
  uint32_t ls;
  eng.locate(source, &ps, &ls);
  ensure_frontier_state(eng);
  eng.launches = 0;
  eng.comm_bytes = 0;
  cudaStream_t s = eng.stream;
  // Near-far (A19b): with delta > 0 a row waits while its distance
  // is >= min + delta, but only rows of out-degree >= hub_deg wait (hub_deg 0:
  // every row).  Rows below it are cheap and relax Bellman-Ford style.
  // Defaults from the RMAT-28 sweep (profiles/r01_sssp_hub_sweep.txt):
  // delta 1 / hub_deg 128 relaxes 1.5x fewer edges than plain Bellman-Ford.
  const uint32_t delta = env_u32("TG_SSSP_DELTA", 1);
  const uint32_t hub_deg = env_u32("TG_SSSP_HUB_DEG", 128);
  // dense supersteps (more than V / dense_div active vertices) mark the next
  // frontier by comparing distances afterwards instead of RED.OR per
  // improvement (TG_SSSP_DENSE_DIV, 0 = never)
  const uint32_t dense_div = env_u32("TG_SSSP_DENSE_DIV", 0);  // A/B: profiles/r02_sssp_dense_ab.txt
  // class kernels when the frontier's out-edges exceed E / class_div (0 = never)
  const uint32_t class_div = env_u32("TG_SSSP_CLASS_DIV", 0);
  if (class_div)
    for (auto& pp : eng.parts) out_classes(eng, *pp);
  if (dense_div)
    for (auto& pp : eng.parts)
      if (pp->fs.prev.n < std::max<uint64_t>(pp->Vp, 1)) pp->fs.prev.alloc(std::max<uint64_t>(pp->Vp, 1));
  std::vector<uint32_t> hubs(eng.parts.size(), 0);
  if (delta)
    for (size_t i = 0; i < eng.parts.size(); ++i) hubs[i] = hub_end(eng, *eng.parts[i], hub_deg);
  const bool trace = std::getenv("TG_TRACE") && std::getenv("TG_TRACE")[0] == '1';
  const DirectionPolicy tclock;  // trace lap clock only
  // sinks (out-degree 0) are not activated when their distance drops
  // (TG_SSSP_SINKS=1: they are, the round-2 behaviour)
  const bool sink_idle = !(std::getenv("TG_SSSP_SINKS") && std::getenv("TG_SSSP_SINKS")[0] == '1');
  uint64_t bm_bytes = 0;
  for (auto& pp : eng.parts) bm_bytes += words_for(pp->Vp) * 4;
  if (eng.P == 1) eng.l2_window(eng.parts[0]->fs.vals.get(), eng.parts[0]->Vp * 4);
  time_begin(eng);
  for (auto& pp : eng.parts) TG_CK(cudaMemsetAsync(pp->fs.counters.get(), 0, 64, s));
  eng.each_part([&](Part& p) {
    cudaStream_t s = eng.stream;
    FrontierState& f = p.fs;
    const uint64_t nw = words_for(p.Vp);
    TG_CK(cudaMemsetAsync(f.vals.get(), 0xFF, p.Vp * 4, s));
    TG_CK(cudaMemsetAsync(f.cur.get(), 0, nw * 4, s));
    TG_CK(cudaMemsetAsync(f.next.get(), 0, nw * 4, s));
    if (p.S) TG_CK(cudaMemsetAsync(f.obox_u32.get(), 0xFF, p.S * 4, s));
    if (eng.fused && p.I) TG_CK(cudaMemsetAsync(p.arena_fwd.get(), 0xFF, p.I * 4, s));
    if (p.id == ps) {
      k_seed<<<1, 1, 0, s>>>(f.next.get(), ls, f.vals.get(), 0);
      eng.launches++;
    }
    launch_advance(eng, p, p.ts, f.next.get(), f.cur.get(), nullptr, nullptr, 0, f.counters.get());
    std::swap(f.cur, f.next);
  });
  if (eng.fused && eng.multi()) fused_arrival(eng);  // inboxes at INF before any peer writes
  uint64_t supersteps = 0, frontier = 1, relax = 0, activations = 1;
  uint64_t mind = 0;  // smallest tentative distance among the active vertices
  uint64_t fr_out = 0;  // out-degree sum of the active vertices (class_div)
  for (;;) {
    reset_vote(eng);
    TG_CK(cudaMemset2DAsync(eng.ctr_all.get() + 5, 64, 0xFF, 8, eng.parts.size(), s));
    const uint64_t th = delta ? mind + delta : (uint64_t)kInf;
    const uint32_t thresh = th >= (uint64_t)kInf ? kInf : (uint32_t)th;
    const bool dense = dense_div && frontier * dense_div > eng.V;
    const bool cls_step = class_div && fr_out * class_div > eng.E;
    eng.each_part([&](Part& p, size_t i) {
      cudaStream_t s = eng.stream;
      FrontierState& f = p.fs;
      if (cls_step) {
        if (p.w8.get()) launch_classes(eng, p, p.w8.get(), thresh, hub_deg ? hubs[i] : kInf);
        else launch_classes(eng, p, p.w.get(), thresh, hub_deg ? hubs[i] : kInf);
        return;
      }
      launch_compact(eng, p.ts);
      if (dense && p.Vp)
        TG_CK(cudaMemcpyAsync(f.prev.get(), f.vals.get(), p.Vp * 4, cudaMemcpyDeviceToDevice, s));
      if (p.w8.get()) {
        SsspOp<uint8_t> op{p.col.get(), p.w8.get(), f.vals.get(), f.next.get(), f.obox_u32.get(),
                           f.counters.get() + 4, p.rout(), eng.fused, thresh,
                           hub_deg ? hubs[i] : kInf, !dense, sink_idle ? (uint32_t)p.nz_end : ~0u};
        launch_expand(eng, p, p.ts, f.cur.get(), op, TG_K_SSSP_EXPAND, f.counters.get() + 1);
      } else {
        SsspOp<uint32_t> op{p.col.get(), p.w.get(), f.vals.get(), f.next.get(), f.obox_u32.get(),
                            f.counters.get() + 4, p.rout(), eng.fused, thresh,
                            hub_deg ? hubs[i] : kInf, !dense, sink_idle ? (uint32_t)p.nz_end : ~0u};
        launch_expand(eng, p, p.ts, f.cur.get(), op, TG_K_SSSP_EXPAND, f.counters.get() + 1);
      }
      if (dense && p.Vp) {
        eng.prof_begin(TG_K_SSSP_EXPAND);
        k_mark_dropped<<<grid_for(p.Vp, 256, 148u * 16u), 256, 0, s>>>(f.vals.get(), f.prev.get(),
                                                                      p.Vp, f.next.get());
        eng.prof_end(TG_K_SSSP_EXPAND);
        TG_CK(cudaGetLastError());
        eng.launches++;
      }
    });
    supersteps++;
    if (eng.P > 1) {
      eng.prof_begin(TG_K_EXCHANGE);
      if (eng.fused) {
        fused_arrival(eng);
        for (auto& pp : eng.parts) eng.comm_bytes += pp->S * 4;
      } else {
        exchange(eng, send_obox, recv_ibox, 4, false);
      }
      eng.each_part([&](Part& p) {
        if (!p.I) return;
        k_sssp_scatter<<<grid_for(p.I, 256), 256, 0, eng.stream>>>(
            reinterpret_cast<const uint32_t*>(p.arena_fwd.get()), p.ibox_lid.get(), p.I,
                                                          p.fs.vals.get(), p.fs.next.get());
        TG_CK(cudaGetLastError());
        eng.launches++;
      });
      eng.prof_end(TG_K_EXCHANGE);
    }
    eng.each_part([&](Part& p) {
      FrontierState& f = p.fs;
      launch_advance(eng, p, p.ts, f.next.get(), f.cur.get(), nullptr, nullptr, 0, f.counters.get(),
                     class_div ? f.counters.get() + 2 : nullptr, nullptr, f.vals.get(),
                     f.counters.get() + 5);
      std::swap(f.cur, f.next);
    });
    const Vote v = read_vote(eng);
    // relaxation: col 4 + w 4 + dist[t] 4 per edge; offsets 16 + dist[v] 4 per
    // relaxed vertex; active + next bitmaps one pass each
    eng.prof_bytes(TG_K_SSSP_EXPAND, 12.0 * v.edges + 20.0 * frontier + 2.0 * bm_bytes);
    if (trace)
      std::fprintf(stderr, "[tg sssp] step=%llu thresh=%u active=%llu edges=%llu next=%llu min=%llu ms=%.3f\n",
                   (unsigned long long)supersteps, thresh, (unsigned long long)frontier,
                   (unsigned long long)v.edges, (unsigned long long)v.count,
                   (unsigned long long)v.minval, tclock.lap(s));
    relax += v.edges;
    frontier = v.count;
    activations += v.count;
    mind = v.minval;
    fr_out = v.degsum;
    if (v.count == 0) break;
    TG_REQUIRE(supersteps <= 4 * eng.V + 64, TG_EINTERNAL, "tg_sssp: superstep bound exceeded");
  }
  const double ms = time_end(eng);
  eng.l2_window(nullptr, 0);
  TG_REQUIRE(read_counts(eng, 4) == 0, TG_EINTERNAL, "tg_sssp: distance overflows uint32");
  if (st) {
    uint64_t nreached = 0;
    st->device_ms = ms;
    st->supersteps = supersteps;
    st->relaxations = relax;
    st->traversed_edges = reached_outdeg_u32(eng, &nreached);
    st->algorithmic_bytes = 12 * relax + 20 * activations + 2 * bm_bytes * supersteps;
    st->comm_bytes = eng.comm_bytes;
    st->launches = eng.launches;
  }
  collect_u32(eng, out, mem);
}

}  // namespace tg
