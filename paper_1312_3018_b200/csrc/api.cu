// api.cu -- the extern "C" boundary (include/tgraph.h) plus engine-wide helpers:
// message exchange between partitions, result collection, statistics.
#include <chrono>
#include <cstring>
#include <functional>
#include <string>

#include "frontier.cuh"

namespace tg {

static thread_local std::string g_last_error;

Engine::~Engine() {
  if (stream) cudaStreamSynchronize(stream);
  for (auto& pv : peers)
    for (void* ptr : pv.opened) cudaIpcCloseMemHandle(ptr);
  peers.clear();
  parts.clear();
  rank_of.release();
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (h_counts) cudaFreeHost(h_counts);
  for (auto& p : pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : ev_pool) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (side[i]) cudaStreamDestroy(side[i]);
    if (join_ev[i]) cudaEventDestroy(join_ev[i]);
  }
  if (fork_ev) cudaEventDestroy(fork_ev);
  for (auto ps : pstream) cudaStreamDestroy(ps);
  for (auto e : pjoin) cudaEventDestroy(e);
  if (pfork) cudaEventDestroy(pfork);
  if (copy_stream) cudaStreamSynchronize(copy_stream);
  for (int i = 0; i < 2; ++i)
    if (stage_free[i]) cudaEventDestroy(stage_free[i]);
  if (chunk_ev) cudaEventDestroy(chunk_ev);
  for (auto e : ticket_ev)
    if (e) cudaEventDestroy(e);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (prof_open) cudaEventDestroy(prof_open);
  if (stream) cudaStreamDestroy(stream);
}

template <typename T>
static uint64_t b(const DevBuf<T>& d) {
  return d.bytes();
}

uint64_t Engine::device_bytes() const {
  uint64_t t = b(rank_of) + b(scratch) + b(stage2[0]) + b(stage2[1]);
  for (auto& pp : parts) {
    const Part& p = *pp;
    t += b(p.row_off) + b(p.col) + b(p.w) + b(p.w8) + b(p.global_of) + b(p.tile_vf) + b(p.tile_vl) +
         b(p.obox_rid) + b(p.ibox_lid) + b(p.in_off) + b(p.in_col) + b(p.outdeg) + b(p.in_nz) + b(p.pr_cta) +
         b(p.pr_warp) + b(p.in_tile_vf) + b(p.in_tile_vl) + b(p.in_all_vf) + b(p.in_all_vl) + b(p.arena_fwd) + b(p.arena_rev) +
         b(p.staging);
  }
  return t;
}

namespace {
__global__ void k_to_host(const unsigned long long* src, int n, int stride, int off,
                          unsigned long long* dst) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[(size_t)i * stride + off];
}
__global__ void k_to_host_u32(const uint32_t* src, unsigned long long* dst) { dst[0] = src[0]; }
}  // namespace

const volatile unsigned long long* to_host(Engine& eng, const unsigned long long* src, int n,
                                           int stride, int off) {
  k_to_host<<<1, 64, 0, eng.stream>>>(src, n, stride, off, eng.d_counts);
  TG_CK(cudaGetLastError());
  TG_CK(cudaStreamSynchronize(eng.stream));
  return eng.h_counts;
}

void Engine::locate(uint64_t g, int* p, uint32_t* l) const {
  TG_REQUIRE(g < V, TG_EINVAL, "source vertex " + std::to_string(g) + " >= V");
  // the position is read through the mapped scratch (a kernel store), not a
  // DMA copy that could queue behind an asynchronous result copy
  k_to_host_u32<<<1, 1, 0, stream>>>(rank_of.get() + g, d_counts);
  TG_CK(cudaGetLastError());
  TG_CK(cudaStreamSynchronize(stream));
  const uint32_t i = (uint32_t)((const volatile unsigned long long*)h_counts)[0];
  deal(i, P, p, l);
}

void ensure_frontier_state(Engine& eng) {
  if (!eng.ctr_all.n) {
    eng.ctr_all.alloc(8 * std::max<size_t>(eng.parts.size(), 1));
    TG_CK(cudaMemset(eng.ctr_all.get(), 0, eng.ctr_all.bytes()));
    for (size_t i = 0; i < eng.parts.size(); ++i) eng.parts[i]->fs.counters = {eng.ctr_all.get() + 8 * i, 8};
  }
  for (auto& pp : eng.parts) {
    Part& p = *pp;
    FrontierState& f = p.fs;
    const uint64_t nw = std::max<uint64_t>(words_for(p.Vp), 1);
    if (f.cur.n >= nw && f.counters.n) continue;
    f.cur.alloc(nw);
    f.next.alloc(nw);
    f.visited.alloc(nw);
    f.vals.alloc(std::max<uint64_t>(p.Vp, 1));
    const uint64_t sw = std::max<uint64_t>(p.S / 32, 1), iw = std::max<uint64_t>(p.I / 32, 1);
    f.obox_mark.alloc(sw);
    f.obox_new.alloc(sw);
    f.obox_u32.alloc(std::max<uint64_t>(p.S, 1));
    (void)iw;
    p.ts.ensure(p.ntiles);
    if (p.in_ntiles || p.in_all_ntiles) p.ts_in.ensure(std::max(p.in_ntiles, p.in_all_ntiles));
  }
}

// ops[i]: 0 sum, 1 min.  The shared-memory collective when the engine has
// one (one round trip for mixed ops), else one callback per op kind.
static void comm_allreduce_mixed(Engine& eng, uint64_t* data, int n, const int* ops) {
  if (!eng.multi()) return;
  if (eng.hc) {
    TG_REQUIRE(eng.hc->allreduce(data, n, ops), TG_ENCCL,
               "host collective: a peer process did not arrive within 600 s");
    return;
  }
  for (int op = 0; op < 2; ++op) {
    uint64_t tmp[16];
    int idx[16], m = 0;
    for (int i = 0; i < n; ++i)
      if (ops[i] == op) {
        idx[m] = i;
        tmp[m++] = data[i];
      }
    if (!m) continue;
    TG_REQUIRE(eng.comm.allreduce_u64(eng.comm.ctx, tmp, m, op) == 0, TG_ENCCL,
               "tg_comm.allreduce_u64 failed");
    for (int j = 0; j < m; ++j) data[idx[j]] = tmp[j];
  }
}

void comm_allreduce(Engine& eng, uint64_t* data, int n, int op) {
  if (!eng.multi()) return;
  TG_REQUIRE(n >= 0 && n <= 16, TG_EINTERNAL, "comm_allreduce: n > 16");
  int ops[16];
  for (int i = 0; i < n; ++i) ops[i] = op;
  comm_allreduce_mixed(eng, data, n, ops);
}

void comm_barrier(Engine& eng) {
  if (!eng.multi()) return;
  uint64_t x = 0;
  comm_allreduce(eng, &x, 1, 0);
}

void exchange(Engine& eng, BufOf send, BufOf recv, size_t elem, bool reverse) {
  // The communication phase.  Segments are symmetric by
  // construction, so each (p, q) pair is one copy straight into the peer's
  // receive arena: a device-to-device copy in one process, a peer (NVLink /
  // NVSwitch) copy into the CUDA-IPC-mapped arena of another process.
  // push: p's outbox segment for q -> q.arena_fwd at q's inbox offset of p.
  // pull: p's inbox segment from q (packed owner state) -> q.arena_rev at q's
  //       outbox offset for p.
  (void)recv;
  if (eng.multi()) {  // receivers must be done with the previous messages
    TG_CK(cudaStreamSynchronize(eng.stream));
    comm_barrier(eng);
  }
  for (auto& pp : eng.parts) {
    Part& p = *pp;
    for (int q = 0; q < eng.P; ++q) {
      if (q == p.id) continue;
      const PeerView& peer = eng.peers[q];
      uint64_t src_off, n, dst_off;
      uint8_t* dst;
      if (!reverse) {
        src_off = p.obox_off[q];
        n = p.obox_off[q + 1] - src_off;
        dst_off = peer.ibox_off[p.id];
        dst = peer.arena_fwd;
      } else {
        src_off = p.ibox_off[q];
        n = p.ibox_off[q + 1] - src_off;
        dst_off = peer.obox_off[p.id];
        dst = peer.arena_rev;
      }
      if (!n) continue;
      const uint64_t bytes = elem ? n * elem : n / 8;
      const uint64_t so = elem ? src_off * elem : src_off / 8;
      const uint64_t ro = elem ? dst_off * elem : dst_off / 8;
      const uint8_t* src = static_cast<const uint8_t*>(send(p));
      TG_CK(cudaMemcpyAsync(dst + ro, src + so, bytes, cudaMemcpyDefault, eng.stream));
      eng.comm_bytes += bytes;
    }
  }
  if (eng.multi()) {  // everyone's messages have landed before anyone scatters
    TG_CK(cudaStreamSynchronize(eng.stream));
    comm_barrier(eng);
  }
}

void fused_arrival(Engine& eng) {
  // the compute kernels' stores / reductions into peer arenas are complete and
  // visible once their stream has drained; the barrier orders every rank's
  // writes before every rank's scatter (one process: stream order suffices)
  if (!eng.multi()) return;
  TG_CK(cudaStreamSynchronize(eng.stream));
  comm_barrier(eng);
}

void fused_reset(Engine& eng, int byte, size_t elem) {
  for (auto& pp : eng.parts)
    if (pp->I) TG_CK(cudaMemsetAsync(pp->arena_fwd.get(), byte, elem ? pp->I * elem : pp->I / 8, eng.stream));
  if (eng.multi()) {
    TG_CK(cudaStreamSynchronize(eng.stream));
    comm_barrier(eng);
  }
}

unsigned long long read_counts(Engine& eng, int idx) {
  const int P = (int)eng.parts.size();
  const volatile unsigned long long* h = to_host(eng, eng.ctr_all.get(), P, 8, idx);
  uint64_t t = 0;
  for (int i = 0; i < P; ++i) t += h[i];
  comm_allreduce(eng, &t, 1, 0);
  return t;
}

Vote read_vote(Engine& eng) {
  const int P = (int)eng.parts.size();
  // the superstep's kernels drain first; vote_ms counts only the vote itself
  // (counter read + cross-process reduction)
  TG_CK(cudaStreamSynchronize(eng.stream));
  const auto t0 = std::chrono::steady_clock::now();
  // the partitions' counters land in mapped host memory by a kernel store
  // (the paper's host-resident vote flag)
  const volatile unsigned long long* h = to_host(eng, eng.ctr_all.get(), 8 * P);
  Vote v;
  v.minval = ~0ull;
  for (int i = 0; i < P; ++i) {
    v.count += h[8 * i];
    v.edges += h[8 * i + 1];
    v.degsum += h[8 * i + 2];
    v.indegsum += h[8 * i + 3];
    const unsigned long long mn = h[8 * i + 5];
    v.minval = std::min<unsigned long long>(v.minval, mn);
  }
  if (eng.multi()) {  // the global vote: sums + the minimum, one reduction
    uint64_t x[5] = {v.count, v.edges, v.degsum, v.indegsum, v.minval};
    static const int ops[5] = {0, 0, 0, 0, 1};
    comm_allreduce_mixed(eng, x, 5, ops);
    v.count = x[0];
    v.edges = x[1];
    v.degsum = x[2];
    v.indegsum = x[3];
    v.minval = x[4];
  }
  eng.vote_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return v;
}

void reset_vote(Engine& eng) {
  TG_CK(cudaMemset2DAsync(eng.ctr_all.get(), 64, 0, 32, eng.parts.size(), eng.stream));
}

void time_begin(Engine& eng) { TG_CK(cudaEventRecord(eng.ev0, eng.stream)); }
double time_end(Engine& eng) {
  TG_CK(cudaEventRecord(eng.ev1, eng.stream));
  TG_CK(cudaEventSynchronize(eng.ev1));
  float ms = 0;
  TG_CK(cudaEventElapsedTime(&ms, eng.ev0, eng.ev1));
  eng.prof_flush();
  return (double)ms;
}

void Engine::l2_window(const void* p, size_t bytes) {
  if (!l2_enabled || !l2_persist || !l2_max_window) return;
  cudaStreamAttrValue v{};
  if (p && bytes) {
    // the hottest prefix only (hubs first), sized to the set-aside: hitRatio 1
    size_t win = bytes < l2_max_window ? bytes : l2_max_window;
    win = win < l2_persist ? win : l2_persist;
    v.accessPolicyWindow.base_ptr = const_cast<void*>(p);
    v.accessPolicyWindow.num_bytes = win;
    v.accessPolicyWindow.hitRatio = 1.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  } else {
    v.accessPolicyWindow.num_bytes = 0;
  }
  TG_CK(cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &v));
  if (!(p && bytes)) TG_CK(cudaCtxResetPersistingL2Cache());
}

static cudaEvent_t pool_get(Engine& eng) {
  if (!eng.ev_pool.empty()) {
    cudaEvent_t e = eng.ev_pool.back();
    eng.ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  TG_CK(cudaEventCreate(&e));
  return e;
}

void Engine::fork() {
  if (!fork_ev) {
    TG_CK(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      TG_CK(cudaStreamCreateWithFlags(&side[i], cudaStreamNonBlocking));
      TG_CK(cudaEventCreateWithFlags(&join_ev[i], cudaEventDisableTiming));
    }
  }
  TG_CK(cudaEventRecord(fork_ev, stream));
  for (int i = 0; i < 2; ++i) TG_CK(cudaStreamWaitEvent(side[i], fork_ev, 0));
}

bool Engine::part_streams_on() {
  if (part_streams < 0) {
    const char* v = std::getenv("TG_PART_STREAMS");
    part_streams = (v && v[0] == '0') ? 0 : 1;
    if (part_streams && parts.size() > 1) {
      TG_CK(cudaEventCreateWithFlags(&pfork, cudaEventDisableTiming));
      pstream.resize(parts.size());
      pjoin.resize(parts.size());
      for (size_t i = 0; i < parts.size(); ++i) {
        TG_CK(cudaStreamCreateWithFlags(&pstream[i], cudaStreamNonBlocking));
        TG_CK(cudaEventCreateWithFlags(&pjoin[i], cudaEventDisableTiming));
      }
    }
  }
  return part_streams == 1;
}

void Engine::join() {
  for (int i = 0; i < 2; ++i) {
    TG_CK(cudaEventRecord(join_ev[i], side[i]));
    TG_CK(cudaStreamWaitEvent(stream, join_ev[i], 0));
  }
}

void Engine::prof_begin(int kid) {
  if (!prof) return;
  prof_open = pool_get(*this);
  prof_open_kid = kid;
  TG_CK(cudaEventRecord(prof_open, stream));
}

void Engine::prof_end(int kid) {
  if (!prof || !prof_open || prof_open_kid != kid) return;
  cudaEvent_t b = pool_get(*this);
  TG_CK(cudaEventRecord(b, stream));
  pending.push_back({kid, prof_open, b});
  prof_open = nullptr;
  prof_open_kid = -1;
}

void Engine::prof_flush() {
  if (pending.empty()) return;
  TG_CK(cudaStreamSynchronize(stream));
  for (auto& p : pending) {
    float ms = 0;
    TG_CK(cudaEventElapsedTime(&ms, p.a, p.b));
    kstat[p.kid].launches++;
    kstat[p.kid].ms += ms;
    ev_pool.push_back(p.a);
    ev_pool.push_back(p.b);
  }
  pending.clear();
}

namespace {

__global__ void k_reached_u32(const uint32_t* vals, const uint64_t* row_off, uint64_t Vp,
                              unsigned long long* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long s = 0, n = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < Vp; v += stride)
    if (vals[v] != kInf) {
      s += row_off[v + 1] - row_off[v];
      n++;
    }
  for (int o = 16; o; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    n += __shfl_down_sync(0xffffffffu, n, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (s) atomicAdd(&out[0], s);
    if (n) atomicAdd(&out[1], n);
  }
}

__global__ void k_reached_bm(const uint32_t* bm, const uint64_t* row_off, uint64_t Vp,
                             unsigned long long* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long s = 0, n = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < Vp; v += stride)
    if ((bm[v >> 5] >> (v & 31)) & 1u) {
      s += row_off[v + 1] - row_off[v];
      n++;
    }
  for (int o = 16; o; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    n += __shfl_down_sync(0xffffffffu, n, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (s) atomicAdd(&out[0], s);
    if (n) atomicAdd(&out[1], n);
  }
}

template <typename T>
__global__ void k_scatter_global(const T* vals, const uint32_t* global_of, uint64_t Vp, T* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < Vp; i += stride)
    out[global_of[i]] = vals[i];
}

void scatter_global(Engine& eng, const void* vals, const uint32_t* gof, uint64_t n, size_t elem,
                    void* out) {
  if (!n) return;
  if (elem == 4)
    k_scatter_global<uint32_t><<<grid_for(n, 256), 256, 0, eng.stream>>>(
        static_cast<const uint32_t*>(vals), gof, n, static_cast<uint32_t*>(out));
  else
    k_scatter_global<unsigned long long><<<grid_for(n, 256), 256, 0, eng.stream>>>(
        static_cast<const unsigned long long*>(vals), gof, n, static_cast<unsigned long long*>(out));
  TG_CK(cudaGetLastError());
}

// Single-process collection as a gather: out[g] = vals_p[l] with (p, l) =
// deal(rank_of[g]) -- coalesced writes in global order, so the output can be
// produced chunk by chunk and each chunk's host copy overlaps the next gather.
struct PartVals {
  const void* v[TG_MAX_PARTITIONS];
  int P;
};

template <typename T>
__global__ void k_gather_global(PartVals pv, const uint32_t* rank_of, uint64_t g0, uint64_t g1,
                                T* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t g = g0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < g1; g += stride) {
    int p;
    uint32_t l;
    deal(rank_of[g], pv.P, &p, &l);
    out[g] = static_cast<const T*>(pv.v[p])[l];
  }
}

void gather_global(Engine& eng, const PartVals& pv, size_t elem, uint64_t g0, uint64_t g1, void* out,
                   cudaStream_t s) {
  if (g1 <= g0) return;
  const unsigned grid = grid_for(g1 - g0, 256);
  if (elem == 4)
    k_gather_global<uint32_t><<<grid, 256, 0, s>>>(pv, eng.rank_of.get(), g0, g1,
                                                    static_cast<uint32_t*>(out));
  else
    k_gather_global<unsigned long long><<<grid, 256, 0, s>>>(
        pv, eng.rank_of.get(), g0, g1, static_cast<unsigned long long*>(out));
  TG_CK(cudaGetLastError());
}

uint64_t reached(Engine& eng, bool bitmap, uint64_t* nreached) {
  // persistent accumulator: a per-call cudaMalloc / cudaFree would synchronize
  // the whole device (including result copies in flight on copy_stream)
  if (!eng.reach_acc.n) eng.reach_acc.alloc(2);
  DevBuf<unsigned long long>& acc = eng.reach_acc;
  TG_CK(cudaMemsetAsync(acc.get(), 0, 16, eng.stream));
  for (auto& pp : eng.parts) {
    Part& p = *pp;
    if (!p.Vp) continue;
    if (bitmap)
      k_reached_bm<<<grid_for(p.Vp, 256), 256, 0, eng.stream>>>(p.fs.visited.get(), p.row_off.get(),
                                                                p.Vp, acc.get());
    else
      k_reached_u32<<<grid_for(p.Vp, 256), 256, 0, eng.stream>>>(p.fs.vals.get(), p.row_off.get(),
                                                                 p.Vp, acc.get());
  }
  TG_CK(cudaGetLastError());
  const volatile unsigned long long* hv = to_host(eng, acc.get(), 2);
  uint64_t h[2] = {hv[0], hv[1]};
  comm_allreduce(eng, h, 2, 0);
  if (nreached) *nreached = h[1];
  return h[0];
}

}  // namespace

uint64_t reached_outdeg_u32(Engine& eng, uint64_t* nreached) { return reached(eng, false, nreached); }
uint64_t reached_outdeg_bitmap(Engine& eng, uint64_t* nreached) { return reached(eng, true, nreached); }

void collect(Engine& eng, ValsOf vals, size_t elem, void* out, int mem) {
  const bool root = !eng.multi() || eng.rank == 0;
  TG_REQUIRE(out != nullptr || !root, TG_EINVAL, "NULL output array");
  cudaStream_t s = eng.stream;
  void* dout = out;
  if (root && mem == TG_MEM_HOST) {  // device staging for the host copy, kept across calls
    // sized for the widest result (8 B) on first use: no re-allocation (a
    // device-wide synchronizing cudaMalloc) when a wider result follows
    if (eng.scratch.bytes() < eng.V * elem) eng.scratch.alloc(eng.V * 8);
    dout = eng.scratch.get();
  }
  // TG_COLLECT: 0 scatter + one copy, 1 gather + one copy, 2 gather chunks
  // with overlapped copies
  int mode = 2;
  if (const char* c = std::getenv("TG_COLLECT")) mode = std::atoi(c);
  if (!eng.multi() && mode == 0) {
    for (auto& pp : eng.parts) scatter_global(eng, vals(*pp), pp->global_of.get(), pp->Vp, elem, dout);
  } else if (!eng.multi()) {
    PartVals pv{};
    pv.P = eng.P;
    for (auto& pp : eng.parts) pv.v[pp->id] = vals(*pp);
    if (mem == TG_MEM_HOST && eng.async_collect) {
      // gather chunks into a staging buffer on the engine stream; copy_stream
      // moves each chunk to the host as soon as it is gathered and keeps going
      // while the caller's next algorithm runs (tg_engine_sync completes it)
      if (!eng.copy_stream) {
        TG_CK(cudaStreamCreateWithFlags(&eng.copy_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) TG_CK(cudaEventCreateWithFlags(&eng.stage_free[i], cudaEventDisableTiming));
        TG_CK(cudaEventCreateWithFlags(&eng.chunk_ev, cudaEventDisableTiming));
      }
      const int k = eng.stage_next;
      eng.stage_next ^= 1;
      if (eng.stage2[k].bytes() < eng.V * elem) eng.stage2[k].alloc(eng.V * 8);
      uint8_t* st = eng.stage2[k].get();
      TG_CK(cudaStreamWaitEvent(s, eng.stage_free[k], 0));  // its previous copy is done
      const uint64_t chunk = 1ull << 25;
      for (uint64_t g0 = 0; g0 < eng.V; g0 += chunk) {
        const uint64_t g1 = std::min<uint64_t>(eng.V, g0 + chunk);
        gather_global(eng, pv, elem, g0, g1, st, s);
        TG_CK(cudaEventRecord(eng.chunk_ev, s));
        TG_CK(cudaStreamWaitEvent(eng.copy_stream, eng.chunk_ev, 0));
        TG_CK(cudaMemcpyAsync(static_cast<uint8_t*>(out) + g0 * elem, st + g0 * elem,
                              (g1 - g0) * elem, cudaMemcpyDeviceToHost, eng.copy_stream));
      }
      TG_CK(cudaEventRecord(eng.stage_free[k], eng.copy_stream));
      const uint64_t t = ++eng.collect_seq;
      cudaEvent_t& te = eng.ticket_ev[t % Engine::kTickets];
      if (!te) TG_CK(cudaEventCreateWithFlags(&te, cudaEventDisableTiming));
      else TG_CK(cudaEventSynchronize(te));  // ticket t - kTickets is complete
      TG_CK(cudaEventRecord(te, eng.copy_stream));
      return;
    }
    if (mem == TG_MEM_HOST && mode == 2) {
      // chunked: gather chunk k on the engine stream, copy it to the host on a
      // side stream while chunk k+1 is gathered
      const uint64_t chunk = 1ull << 25;
      eng.fork();  // side streams start after the algorithm's last kernel
      for (uint64_t g0 = 0; g0 < eng.V; g0 += chunk) {
        const uint64_t g1 = std::min<uint64_t>(eng.V, g0 + chunk);
        gather_global(eng, pv, elem, g0, g1, dout, s);
        TG_CK(cudaEventRecord(eng.fork_ev, s));
        TG_CK(cudaStreamWaitEvent(eng.side[0], eng.fork_ev, 0));
        TG_CK(cudaMemcpyAsync(static_cast<uint8_t*>(out) + g0 * elem,
                              static_cast<uint8_t*>(dout) + g0 * elem, (g1 - g0) * elem,
                              cudaMemcpyDeviceToHost, eng.side[0]));
      }
      eng.join();
      TG_CK(cudaStreamSynchronize(s));
      return;
    }
    gather_global(eng, pv, elem, 0, eng.V, dout, s);
  } else {
    // stage my values, then rank 0 scatters every rank's staging (IPC-mapped)
    Part& me = *eng.parts[0];
    if (me.Vp)
      TG_CK(cudaMemcpyAsync(me.staging.get(), vals(me), me.Vp * elem, cudaMemcpyDeviceToDevice, s));
    TG_CK(cudaStreamSynchronize(s));
    comm_barrier(eng);
    if (root)
      for (int q = 0; q < eng.P; ++q)
        scatter_global(eng, eng.peers[q].staging, eng.peers[q].global_of, eng.peers[q].Vp, elem,
                       dout);
    TG_CK(cudaStreamSynchronize(s));
    comm_barrier(eng);
  }
  if (root && mem == TG_MEM_HOST)
    TG_CK(cudaMemcpyAsync(out, dout, eng.V * elem, cudaMemcpyDeviceToHost, s));
  TG_CK(cudaStreamSynchronize(s));
}

void collect_u32(Engine& eng, uint32_t* out, int mem) {
  collect(eng, [](Part& p) -> const void* { return p.fs.vals.get(); }, 4, out, mem);
}

int guard(const std::function<void()>& f) {
  try {
    f();
    g_last_error.clear();
    return TG_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return TG_ECAPACITY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TG_EINTERNAL;
  } catch (...) {
    g_last_error = "unknown error";
    return TG_EINTERNAL;
  }
}

static void init_engine(Engine& eng, const tg_attr* attr) {
  TG_REQUIRE(attr != nullptr, TG_EINVAL, "NULL attr");
  TG_REQUIRE(attr->num_partitions >= 1, TG_EINVAL, "num_partitions must be >= 1");
  TG_REQUIRE(attr->num_partitions <= TG_MAX_PARTITIONS, TG_ECAPACITY,
             "num_partitions > TG_MAX_PARTITIONS");
  TG_REQUIRE(attr->strategy == TG_PART_DEGREE || attr->strategy == TG_PART_RANDOM, TG_EINVAL,
             "tg_attr.strategy: unknown partitioning strategy");
  eng.strategy = attr->strategy;
  eng.part_seed = (uint32_t)attr->part_seed;
  const int world = attr->world < 1 ? 1 : attr->world;
  TG_REQUIRE(world <= TG_MAX_PARTITIONS, TG_ECAPACITY, "world > TG_MAX_PARTITIONS");
  if (world > 1) {
    TG_REQUIRE(attr->num_partitions == 1, TG_EINVAL,
               "multi-process engines host exactly one partition per process");
    TG_REQUIRE(attr->rank >= 0 && attr->rank < world, TG_EINVAL, "rank outside [0, world)");
    TG_REQUIRE(attr->comm && attr->comm->allgather && attr->comm->allreduce_u64, TG_EINVAL,
               "world > 1 requires tg_attr.comm with allgather and allreduce_u64");
    eng.comm = *attr->comm;
  }
  if (world > 1 && !(std::getenv("TG_HOSTCOMM") && std::getenv("TG_HOSTCOMM")[0] == '0')) {
    Engine* e = &eng;
    e->rank = attr->rank;
    e->world = world;
    eng.hc = HostComm::create(
        attr->rank, world,
        [e](const void* send, void* recv, uint64_t bytes) {
          TG_REQUIRE(e->comm.allgather(e->comm.ctx, send, recv, bytes) == 0, TG_ENCCL,
                     "tg_comm.allgather failed");
        },
        [e]() {
          uint64_t x = 0;
          TG_REQUIRE(e->comm.allreduce_u64(e->comm.ctx, &x, 1, 0) == 0, TG_ENCCL,
                     "tg_comm.allreduce_u64 failed");
        });
  }
  eng.rank = world > 1 ? attr->rank : 0;
  eng.world = world;
  int ndev = 0;
  TG_CK(cudaGetDeviceCount(&ndev));
  TG_REQUIRE(attr->device >= 0 && attr->device < ndev, TG_EINVAL, "bad CUDA device ordinal");
  eng.device = attr->device;
  TG_CK(cudaSetDevice(eng.device));
  eng.P = world > 1 ? world : attr->num_partitions;
  eng.weighted = attr->weighted != 0;
  TG_REQUIRE(attr->build_in_csr >= 0 && attr->build_in_csr <= 2, TG_EINVAL,
             "tg_attr.build_in_csr must be 0, 1 or 2");
  eng.has_in = attr->build_in_csr != 0;
  eng.in_only = attr->build_in_csr == 2;
  TG_REQUIRE(!eng.in_only || attr->world <= 1, TG_EINVAL,
             "build_in_csr = 2 (in-CSR only) is single-process");
  TG_CK(cudaStreamCreateWithFlags(&eng.stream, cudaStreamNonBlocking));
  TG_CK(cudaEventCreate(&eng.ev0));
  TG_CK(cudaEventCreate(&eng.ev1));
  TG_CK(cudaHostAlloc(&eng.h_counts, sizeof(unsigned long long) * TG_MAX_PARTITIONS * 8,
                      cudaHostAllocMapped | cudaHostAllocPortable));
  TG_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&eng.d_counts), eng.h_counts, 0));
  // L2 set-aside for persisting accesses: measured slower on RMAT-28 (the
  // set-aside starves the rest of the working set), so opt-in only
  // (TG_L2_WINDOW=1).
  const char* on = std::getenv("TG_L2_WINDOW");
  eng.l2_enabled = on && on[0] == '1';
  int maxp = 0, maxw = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, eng.device);
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, eng.device);
  if (eng.l2_enabled && maxp > 0 && maxw > 0) {
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp) == cudaSuccess) {
      eng.l2_persist = (size_t)maxp;
      eng.l2_max_window = (size_t)maxw;
    } else {
      cudaGetLastError();
    }
  }
}

// SPMD check: every rank must run an algorithm with the same
// exchange transport and PageRank communication, or their barrier counts
// and message layouts disagree.  One small reduction per algorithm call.
static void agree_settings(Engine& eng) {
  if (!eng.multi()) return;
  uint64_t x[2] = {eng.fused ? 1ull : 0ull, (uint64_t)eng.pr_comm};
  comm_allreduce(eng, x, 2, 0);
  const uint64_t w = (uint64_t)eng.world;
  TG_REQUIRE((x[0] == 0 || x[0] == w) && (x[1] == 0 || x[1] == w), TG_EINVAL,
             "ranks disagree on the exchange transport or the PageRank communication "
             "(tg_engine_set_exchange / tg_engine_set_pagerank_comm must be called on every rank)");
}

// compute / exchange split of one call from the kernel ledger (profiling on)
struct RunLedger {
  Engine& eng;
  double ms0[TG_K_COUNT];
  explicit RunLedger(Engine& e) : eng(e) {
    eng.prof_flush();
    for (int k = 0; k < TG_K_COUNT; ++k) ms0[k] = eng.kstat[k].ms;
    eng.vote_ms = 0;
  }
  void fill(tg_stats* st) {
    eng.prof_flush();
    st->vote_ms = eng.vote_ms;
    if (!eng.prof) return;
    for (int k = 0; k < TG_K_COUNT; ++k) {
      const double d = eng.kstat[k].ms - ms0[k];
      if (k == TG_K_EXCHANGE) st->exchange_ms += d;
      else st->compute_ms += d;
    }
  }
};

}  // namespace tg

using namespace tg;

extern "C" {

const char* tg_version(void) { return "tgraph 0.1 (sm_100a)"; }
const char* tg_last_error(void) { return g_last_error.c_str(); }

int tg_engine_create_edges(uint64_t V, uint64_t E, const uint32_t* src, const uint32_t* dst,
                           const uint32_t* w, int mem, const tg_attr* attr, tg_engine** out) {
  return guard([&] {
    TG_REQUIRE(out != nullptr, TG_EINVAL, "NULL out");
    *out = nullptr;
    TG_REQUIRE(V >= 1 && V < (1ull << 31), TG_EINVAL, "V must be in [1, 2^31)");
    TG_REQUIRE(E == 0 || (src && dst), TG_EINVAL, "NULL edge arrays");
    TG_REQUIRE(mem == TG_MEM_HOST || mem == TG_MEM_DEVICE, TG_EINVAL, "bad mem kind");
    auto eng = std::make_unique<Engine>();
    init_engine(*eng, attr);
    TG_REQUIRE(!eng->weighted || w != nullptr || E == 0, TG_EINVAL,
               "attr.weighted set but no weight array given");
    eng->V = V;
    eng->E = E;
    DevBuf<uint32_t> ds, dd, dw;
    EdgeInput in;
    in.generated = false;
    if (mem == TG_MEM_HOST && E) {
      ds.alloc(E);
      dd.alloc(E);
      TG_CK(cudaMemcpy(ds.get(), src, E * 4, cudaMemcpyHostToDevice));
      TG_CK(cudaMemcpy(dd.get(), dst, E * 4, cudaMemcpyHostToDevice));
      if (w && eng->weighted) {
        dw.alloc(E);
        TG_CK(cudaMemcpy(dw.get(), w, E * 4, cudaMemcpyHostToDevice));
      }
      in.src = ds.get();
      in.dst = dd.get();
      in.w = dw.get();
    } else {
      in.src = src;
      in.dst = dst;
      in.w = eng->weighted ? w : nullptr;
    }
    build_engine(*eng, in);
    *out = reinterpret_cast<tg_engine*>(eng.release());
  });
}

int tg_engine_create_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                          int scramble, uint64_t wseed, const tg_attr* attr, tg_engine** out) {
  return guard([&] {
    TG_REQUIRE(out != nullptr, TG_EINVAL, "NULL out");
    *out = nullptr;
    TG_REQUIRE(scale >= 1 && scale <= 31, TG_EINVAL, "scale must be in [1, 31]");
    TG_REQUIRE(edge_factor >= 1, TG_EINVAL, "edge_factor must be >= 1");
    TG_REQUIRE(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0 + 1e-12, TG_EINVAL,
               "RMAT probabilities: need a, b, c >= 0 and a + b + c <= 1");
    auto eng = std::make_unique<Engine>();
    init_engine(*eng, attr);
    eng->V = 1ull << scale;
    eng->E = (uint64_t)edge_factor << scale;
    EdgeInput in;
    in.generated = true;
    in.scale = scale;
    in.a = a;
    in.b = b;
    in.c = c;
    in.seed = seed;
    in.wseed = wseed;
    in.scramble = scramble;
    build_engine(*eng, in);
    *out = reinterpret_cast<tg_engine*>(eng.release());
  });
}

int tg_partition_size(uint64_t V, int p, int P, uint64_t* Vp) {
  return guard([&] {
    TG_REQUIRE(Vp != nullptr, TG_EINVAL, "NULL output");
    TG_REQUIRE(P >= 1 && P <= TG_MAX_PARTITIONS, TG_EINVAL, "P outside [1, TG_MAX_PARTITIONS]");
    TG_REQUIRE(p >= 0 && p < P, TG_EINVAL, "p outside [0, P)");
    *Vp = part_size(V, p, P);
  });
}

void tg_engine_free(tg_engine* e) {
  if (!e) return;
  Engine* eng = reinterpret_cast<Engine*>(e);
  cudaSetDevice(eng->device);
  delete eng;
}

int tg_engine_info(const tg_engine* e, tg_info* info) {
  return guard([&] {
    TG_REQUIRE(e && info, TG_EINVAL, "NULL argument");
    const Engine* eng = reinterpret_cast<const Engine*>(e);
    info->V = eng->V;
    info->E = eng->E;
    info->num_partitions = eng->P;
    info->weighted = eng->weighted;
    info->has_in_csr = eng->has_in;
    info->device_bytes = eng->device_bytes();
    info->build_ms = eng->build_ms;
    info->device = eng->device;
    info->strategy = eng->strategy;
    info->exchange = eng->fused ? TG_EXCHANGE_FUSED : TG_EXCHANGE_COPY;
    info->pr_comm = eng->pr_comm;
    info->peer_probe = eng->peer_probe_passed ? 1 : 0;
  });
}

int tg_engine_partition_info(const tg_engine* e, int p, tg_part_info* info, uint64_t* slots_to) {
  return guard([&] {
    TG_REQUIRE(e && info, TG_EINVAL, "NULL argument");
    const Engine* eng = reinterpret_cast<const Engine*>(e);
    TG_REQUIRE(p >= 0 && p < eng->P, TG_EINVAL, "partition index out of range");
    const Part* found = nullptr;
    for (auto& pp : eng->parts)
      if (pp->id == p) found = pp.get();
    TG_REQUIRE(found != nullptr, TG_EINVAL, "partition is hosted by another process");
    const Part& pt = *found;
    info->Vp = pt.Vp;
    info->Ep = pt.Ep;
    info->Ep_local = pt.Ep_local;
    info->outbox_slots = pt.S_real;
    info->inbox_slots = pt.I_real;
    if (slots_to)
      for (int q = 0; q < eng->P; ++q) slots_to[q] = q < (int)pt.seg_real.size() ? pt.seg_real[q] : 0;
  });
}

// Every algorithm call: stats always computed (a NULL `stats` gets a local
// one, so multi-process ranks run the same collectives whatever they pass),
// the ranks' transport settings checked equal (SPMD), and the phase split
// filled from the kernel ledger and the vote timer.
#define TG_RUN(body)                                                     \
  return guard([&] {                                                     \
    TG_REQUIRE(e != nullptr, TG_EINVAL, "NULL engine");                  \
    Engine& eng = *reinterpret_cast<Engine*>(e);                         \
    TG_REQUIRE(mem == TG_MEM_HOST || mem == TG_MEM_DEVICE, TG_EINVAL, "bad mem kind"); \
    TG_CK(cudaSetDevice(eng.device));                                    \
    tg_stats local_st;                                                   \
    tg_stats* st = user_st ? user_st : &local_st;                        \
    std::memset(st, 0, sizeof(*st));                                     \
    agree_settings(eng);                                                 \
    RunLedger led(eng);                                                  \
    body;                                                                \
    led.fill(st);                                                        \
  })

// NULL outputs are rejected inside run_* except on non-root ranks of a
// multi-process engine (results are written on rank 0 only).
int tg_bfs(tg_engine* e, uint64_t source, uint32_t* levels, int mem, tg_stats* user_st) {
  TG_RUN({
    TG_REQUIRE(!eng.in_only, TG_EINVAL, "engine holds the in-CSR only (build_in_csr = 2): PageRank only");
    run_bfs(eng, source, levels, mem, st);
  });
}

int tg_sssp(tg_engine* e, uint64_t source, uint32_t* dist, int mem, tg_stats* user_st) {
  TG_RUN({
    TG_REQUIRE(!eng.in_only, TG_EINVAL, "engine holds the in-CSR only (build_in_csr = 2): PageRank only");
    run_sssp(eng, source, dist, mem, st);
  });
}

int tg_cc(tg_engine* e, uint32_t* labels, int mem, tg_stats* user_st) {
  TG_RUN({
    TG_REQUIRE(!eng.in_only, TG_EINVAL, "engine holds the in-CSR only (build_in_csr = 2): PageRank only");
    run_cc(eng, labels, mem, st);
  });
}

int tg_pagerank(tg_engine* e, int iterations, double damping, float* rank, int mem,
                tg_stats* user_st) {
  TG_RUN({ run_pagerank(eng, iterations, damping, rank, mem, st); });
}

int tg_bc(tg_engine* e, const uint64_t* sources, int k, double* bc, int mem, tg_stats* user_st) {
  TG_RUN({
    TG_REQUIRE(!eng.in_only, TG_EINVAL, "engine holds the in-CSR only (build_in_csr = 2): PageRank only");
    run_bc(eng, sources, k, bc, mem, st);
  });
}

int tg_engine_set_profiling(tg_engine* e, int on) {
  return guard([&] {
    TG_REQUIRE(e != nullptr, TG_EINVAL, "NULL engine");
    Engine& eng = *reinterpret_cast<Engine*>(e);
    TG_CK(cudaSetDevice(eng.device));
    eng.prof_flush();
    eng.prof = on != 0;
    for (auto& k : eng.kstat) k = tg_kernel_stat{};
  });
}

int tg_engine_set_exchange(tg_engine* e, int mode) {
  return guard([&] {
    TG_REQUIRE(e != nullptr, TG_EINVAL, "NULL engine");
    TG_REQUIRE(mode == TG_EXCHANGE_COPY || mode == TG_EXCHANGE_FUSED, TG_EINVAL,
               "tg_engine_set_exchange: unknown mode");
    Engine& eng = *reinterpret_cast<Engine*>(e);
    TG_REQUIRE(mode == TG_EXCHANGE_COPY || eng.peer_atomics, TG_EINVAL,
               "tg_engine_set_exchange: FUSED needs native peer atomics between the ranks' GPUs");
    eng.fused = mode == TG_EXCHANGE_FUSED;
  });
}

int tg_engine_set_async_collect(tg_engine* e, int on) {
  return guard([&] {
    TG_REQUIRE(e != nullptr, TG_EINVAL, "NULL engine");
    Engine& eng = *reinterpret_cast<Engine*>(e);
    TG_CK(cudaSetDevice(eng.device));
    if (eng.copy_stream) TG_CK(cudaStreamSynchronize(eng.copy_stream));
    eng.async_collect = on != 0 && !eng.multi();
  });
}

int tg_engine_sync(tg_engine* e) {
  return guard([&] {
    TG_REQUIRE(e != nullptr, TG_EINVAL, "NULL engine");
    Engine& eng = *reinterpret_cast<Engine*>(e);
    TG_CK(cudaSetDevice(eng.device));
    if (eng.copy_stream) TG_CK(cudaStreamSynchronize(eng.copy_stream));
    TG_CK(cudaStreamSynchronize(eng.stream));
  });
}

int tg_engine_last_ticket(const tg_engine* e, uint64_t* ticket) {
  return guard([&] {
    TG_REQUIRE(e != nullptr && ticket != nullptr, TG_EINVAL, "NULL engine or ticket");
    *ticket = reinterpret_cast<const Engine*>(e)->collect_seq;
  });
}

int tg_engine_wait_ticket(tg_engine* e, uint64_t ticket) {
  return guard([&] {
    TG_REQUIRE(e != nullptr, TG_EINVAL, "NULL engine");
    Engine& eng = *reinterpret_cast<Engine*>(e);
    TG_REQUIRE(ticket <= eng.collect_seq, TG_EINVAL, "tg_engine_wait_ticket: ticket not issued");
    if (ticket == 0 || ticket + Engine::kTickets <= eng.collect_seq) return;  // complete
    TG_CK(cudaSetDevice(eng.device));
    TG_CK(cudaEventSynchronize(eng.ticket_ev[ticket % Engine::kTickets]));
  });
}

int tg_device_die_map(int device, uint8_t* die_of, int cap, int* nsm, int* ok) {
  return guard([&] {
    TG_REQUIRE(nsm != nullptr && ok != nullptr, TG_EINVAL, "tg_device_die_map: NULL output");
    int nd = 0;
    TG_CK(cudaGetDeviceCount(&nd));
    TG_REQUIRE(device >= 0 && device < nd, TG_EINVAL, "tg_device_die_map: bad device");
    const DieMap& m = die_map(device);
    *nsm = m.nsm;
    *ok = m.ok ? 1 : 0;
    if (die_of)
      for (int i = 0; i < cap && i < (int)m.h_die_of.size(); ++i) die_of[i] = m.h_die_of[i];
  });
}

int tg_engine_set_pagerank_comm(tg_engine* e, int mode) {
  return guard([&] {
    TG_REQUIRE(e != nullptr, TG_EINVAL, "NULL engine");
    TG_REQUIRE(mode == TG_PR_PUSH || mode == TG_PR_PULL, TG_EINVAL,
               "tg_engine_set_pagerank_comm: unknown mode");
    reinterpret_cast<Engine*>(e)->pr_comm = mode;
  });
}

int tg_engine_kernel_stat(const tg_engine* e, int kid, tg_kernel_stat* out) {
  return guard([&] {
    TG_REQUIRE(e && out, TG_EINVAL, "NULL argument");
    TG_REQUIRE(kid >= 0 && kid < TG_K_COUNT, TG_EINVAL, "kernel id out of range");
    *out = reinterpret_cast<const Engine*>(e)->kstat[kid];
  });
}

int tg_hostcomm_create(const tg_comm* comm, int rank, int world, tg_hostcomm** out) {
  return guard([&] {
    TG_REQUIRE(out != nullptr, TG_EINVAL, "NULL out");
    *out = nullptr;
    TG_REQUIRE(comm && comm->allgather && comm->allreduce_u64, TG_EINVAL, "bad tg_comm");
    TG_REQUIRE(world >= 2 && world <= TG_MAX_PARTITIONS && rank >= 0 && rank < world, TG_EINVAL,
               "rank / world out of range");
    const tg_comm c = *comm;
    auto hc = HostComm::create(
        rank, world,
        [c](const void* send, void* recv, uint64_t bytes) {
          TG_REQUIRE(c.allgather(c.ctx, send, recv, bytes) == 0, TG_ENCCL, "tg_comm.allgather failed");
        },
        [c]() {
          uint64_t x = 0;
          TG_REQUIRE(c.allreduce_u64(c.ctx, &x, 1, 0) == 0, TG_ENCCL, "tg_comm.allreduce_u64 failed");
        });
    TG_REQUIRE(hc != nullptr, TG_ENCCL, "a rank could not map the shared-memory segment");
    *out = reinterpret_cast<tg_hostcomm*>(hc.release());
  });
}

int tg_hostcomm_allreduce_u64(tg_hostcomm* h, uint64_t* data, int n, const int* ops) {
  return guard([&] {
    TG_REQUIRE(h && (n == 0 || (data && ops)), TG_EINVAL, "NULL argument");
    TG_REQUIRE(n >= 0 && n <= 16, TG_EINVAL, "n must be in [0, 16]");
    for (int i = 0; i < n; ++i) TG_REQUIRE(ops[i] == 0 || ops[i] == 1, TG_EINVAL, "op must be 0 or 1");
    TG_REQUIRE(reinterpret_cast<HostComm*>(h)->allreduce(data, n, ops), TG_ENCCL,
               "host collective: a peer process did not arrive within 600 s");
  });
}

void tg_hostcomm_free(tg_hostcomm* h) { delete reinterpret_cast<HostComm*>(h); }

const char* tg_kernel_name(int kid) {
  static const char* names[TG_K_COUNT] = {"bfs_expand",  "sssp_expand", "bc_fwd_expand",
                                          "bc_bwd_expand", "pr_pull",   "advance",
                                          "tile_compact", "exchange_scatter", "cc_expand"};
  return (kid >= 0 && kid < TG_K_COUNT) ? names[kid] : "?";
}

}  // extern "C"
