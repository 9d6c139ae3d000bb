// engine.cuh -- device-resident partitioned graph and per-algorithm state.
//
// Layout (§4.3.1-4.3.2):
//   * every partition p owns Vp vertices with dense local ids 0..Vp-1 ordered by
//     out-degree descending (so degree classes are contiguous id ranges and
//     zero-degree vertices form the tail [nz_end, Vp));
//   * out-CSR row_off (u64) / col (u32): per row the LOCAL targets first, then
//     the remote ones; a remote entry is kRemote | outbox slot (the
//     paper's partition-tagged E entry pointing into the outbox);
//   * outbox: one slot per distinct (p, remote vertex) pair -- the source-side
//     reduction of P:168-182 is structural.  Slots are grouped by owner q,
//     sorted by the owner's local id, each segment padded to a multiple of 32
//     so bitmap words never straddle two peers;
//   * inbox of q from p = p's outbox segment for q (symmetric): only the
//     message arrays move between partitions;
//   * edge tiles: the edge array is cut into tiles of kTile edges; tile t knows
//     the first/last row it touches, so a frontier kernel is load balanced over
//     edges whatever the degree skew (hubs span many tiles);
//   * in-CSR (PageRank pull, bottom-up BFS, pull-sigma BC): rows [0,Vp) are
//     local vertices in local-id order, rows [Vp,Vp+S) are outbox slots (their
//     PageRank sums are the partition's partial-sum messages); entries are the
//     local ids of the sources, each row sorted ascending.
#pragma once

#include <exception>
#include <memory>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "hostcomm.h"

namespace tg {

constexpr uint32_t kTile = 1024;  // edges per frontier tile (one warp task)

// Degree-aware serpentine deal (reading A23): order position i -> (part, local).
__host__ __device__ __forceinline__ void deal(uint64_t i, int P, int* p, uint32_t* l) {
  const uint64_t r = i / (uint64_t)P, j = i % (uint64_t)P;
  *p = (int)((r & 1) ? (uint64_t)P - 1 - j : j);
  *l = (uint32_t)r;
}
__host__ __device__ __forceinline__ uint64_t undeal(uint32_t l, int p, int P) {
  const uint64_t j = (l & 1) ? (uint64_t)(P - 1 - p) : (uint64_t)p;
  return (uint64_t)l * (uint64_t)P + j;
}
inline uint64_t part_size(uint64_t V, int p, int P) {
  const uint64_t R = V / (uint64_t)P, rem = V % (uint64_t)P;
  if (!rem) return R;
  const uint64_t j = (R & 1) ? (uint64_t)(P - 1 - p) : (uint64_t)p;
  return R + (j < rem ? 1 : 0);
}

// Per-partition tile scheduling scratch (frontier.cu)
struct Part;
struct TileSched {
  DevBuf<uint32_t> bm;    // bitmap over tiles
  DevBuf<uint32_t> list;  // compacted active tiles
  DevBuf<unsigned long long> count;
  uint64_t nwords = 0;
  void ensure(uint64_t ntiles);
};

// Fused exchange (the fusion candidates of SURVEY 8(e)): the
// compute kernel writes a boundary message straight into the owner's receive
// arena -- a local pointer for partitions of one process, a CUDA-IPC-mapped
// peer pointer (NVLink / NVSwitch stores and reductions) across processes --
// instead of staging it in an outbox that the communication phase then copies.
// p's outbox slot s (segment of owner q) lands at q's inbox index of p, which
// is s + delta[q]; both offsets are multiples of 32, so bitmap words map whole.
struct RemoteOut {
  const uint8_t* owner = nullptr;   // [S/32] owner partition of each 32-slot word
  uint8_t* const* arena = nullptr;  // [P] owners' arena_fwd (arena_rev for rin())
  const int64_t* delta = nullptr;   // [P] inbox index at q minus outbox index at p
  template <class T>
  __device__ __forceinline__ T* slot(uint32_t s) const {
    const int q = owner[s >> 5];
    return reinterpret_cast<T*>(arena[q]) + ((int64_t)s + delta[q]);
  }
  __device__ __forceinline__ uint32_t* word(uint32_t s) const {
    const int q = owner[s >> 5];
    return reinterpret_cast<uint32_t*>(arena[q]) + (((int64_t)s + delta[q]) >> 5);
  }
};

// PageRank hub split (pagerank.cu, TG_PR_HUB): the in-edges of the CTA- and
// warp-class rows whose source is one of the K hubs (local ids [0, K): the
// out-degree order puts them first) are summed by a separate pass from a
// shared-memory replica of contrib[0, K) -- an LDS instead of a random L2
// request -- and the class pulls start each of those rows after its hub prefix.
struct PRHub {
  uint32_t K = 0;
  const uint32_t* built_for = nullptr;  // the in-CSR column array it was built from
  uint64_t n_list = 0;                  // CTA-class rows, then warp-class rows
  uint64_t ntask = 0, H = 0;            // tasks (<= kHubChunk hub entries each), entries
  DevBuf<uint32_t> hlen;                // [n_list] hub-prefix length of each list row
  DevBuf<uint16_t> col;                 // [H] hub source ids, list-row order
  DevBuf<uint64_t> t_off;               // [ntask] first entry of the task in col
  DevBuf<uint32_t> t_len, t_k;          // [ntask] entries, list row
  DevBuf<double> hsum;                  // [n_list] hub part of each list row's sum
};

// The two dies of a B200 each cache in their half of the L2 the lines their own
// SMs read (profiles/r02_die_probe.txt: a 128 MB gather region runs at 118 G
// loads/s when every SM reads all of it, 282 G/s when each die's SMs read only
// their own 64 MB half).  DieMap is the SM -> die map measured at run time
// (dies.cu): pointer-chase latency from every SM to lines the reference SM just
// pulled into its L2.
struct DieMap {
  bool ok = false;            // two clear latency clusters were found
  int nsm = 0, n[2] = {0, 0};
  double lat_near = 0, lat_far = 0;  // cycles per chased line
  DevBuf<uint8_t> die_of;     // [nsm] die of each SM id (device)
  std::vector<uint8_t> h_die_of;
};
const DieMap& die_map(int device);  // measured once per device, cached

// PageRank die split (pagerank.cu): the in-edges of every row are split by the
// die that gathers their source -- source u belongs to die d(u), a hash of its
// 128-byte line weighted by the dies' SM counts -- into two CSRs.  The SMs of
// die d pull only over CSR d, so each die's L2 caches only its half of the hot
// contributions; a finalize pass adds the two partial sums of every row.
struct PRSplit {
  bool built = false, on = false;
  const uint32_t* built_for = nullptr;  // in-CSR column array it was built from
  uint32_t thresh = 0;                  // d(u) = hash(u >> 5) >= thresh
  uint64_t R = 0;
  DevBuf<uint64_t> off[2];              // [R + 1]
  DevBuf<uint32_t> col[2];              // sources of die d, each row ascending
  DevBuf<uint32_t> wrow[2];             // rows with 32 <= half-degree < kSplitChunk
  uint64_t n_w[2] = {0, 0};
  DevBuf<uint32_t> c_row[2], c_k[2], c_len[2];  // chunks of the rows >= kSplitChunk
  DevBuf<uint64_t> c_start[2];
  DevBuf<uint32_t> c_list[2];           // those rows (k -> row)
  uint64_t n_c[2] = {0, 0}, n_ck[2] = {0, 0};  // chunks, chunked rows
  DevBuf<double> cacc[2];               // [n_ck] chunked-row sums (atomics)
  DevBuf<float> psum[2];                // [R] partial sum of every row per die
  DevBuf<unsigned long long> qnext;     // [2] task queues' next index
};

// PageRank cold-tail propagation blocking (pagerank.cu, TG_PR_COLD=T): the
// in-edges from the cold sources (local ids >= T: out-degree order puts them
// last, past the L2-resident hub prefix) are not gathered by the pull.  Phase
// A walks the cold sources in order and writes each contribution into a slot
// per out-edge, the slots grouped by target bin (2^kb rows) -- random L2
// gathers that miss to HBM become writes that L2 merges into whole lines;
// phase B sums each bin's slots into a shared-memory accumulator and writes
// the rows' cold partial sums, which the pull adds.  Single partition.
struct PRCold {
  bool on = false;
  uint32_t T = 0;
  int kb = 15;
  const uint32_t* built_for = nullptr;
  uint64_t e0 = 0, n = 0;       // cold out-edges: out-CSR [e0, e0 + n), sources [T, nz_end)
  uint64_t nbins = 0;
  DevBuf<uint32_t> pos;         // [n] slot of cold out-edge e0 + i
  DevBuf<uint16_t> binv;        // [n] target row within its bin, per slot
  DevBuf<float> binval;         // [n] contribution per slot (phase A)
  DevBuf<uint64_t> bin_off;     // [nbins + 1]
  DevBuf<uint32_t> hot_len;     // [R] in-edges of row r from sources < T (a prefix: rows ascend)
  DevBuf<float> csum;           // [R] cold partial sum of row r (phase B)
};

struct PRState {  // PageRank (local-id order)
  DevBuf<float> contrib[2];
  DevBuf<float> rank;
  DevBuf<double> acc;
  DevBuf<double> obox;  // partial sums per outbox slot (send)
  PRHub hub;
  PRSplit split;
  PRCold cold;
  // sink rows (local ids >= nz_end, out-degree 0) and their in-edges in the
  // pull CSR it was counted for (rows a non-final round does not pull)
  const uint64_t* sinks_for = nullptr;
  uint64_t sink_rows = 0, sink_edges = 0;
};

// Ghost-pull PageRank (TOTEM_COMM_PULL):
// instead of pushing per-target partial sums, every partition publishes the
// contributions of its sources that have out-edges into a peer, into ghost
// slots appended to the peer's contribution array, and each partition pulls
// over a ghost-indexed in-CSR (local sources < Vp, ghost g at Vp + g).
// Built on first use from the push layout (across processes through CUDA-IPC
// views of the peers' in-CSR and publish lists).
struct PRGhost {
  bool built = false;
  uint64_t G = 0;                          // ghost slots of this partition
  std::vector<uint64_t> pub_off, gh_off;   // P+1 each: publish segments / ghost segments
  DevBuf<uint32_t> pub_lid;                // local ids published to each peer, ascending
  DevBuf<uint64_t> off;                    // Vp + 1
  DevBuf<uint32_t> col;                    // local id, or Vp + ghost index
  DevBuf<uint32_t> cta, warp;              // row classes (in-degree >= 2048 / 32..2047)
  uint64_t n_cta = 0, n_warp = 0;
  // publish destinations per buffer and peer: q's contribution array (local
  // pointer, or CUDA-IPC-mapped across processes) + Vq + q's ghost offset of p
  std::vector<float*> pub_dst[2];
  // Direction optimization across partitions (SURVEY NEXT-1 at P > 1): the
  // same publish lists carry frontier bits (bottom-up BFS) and frontier sigma
  // (pull-sigma BC) into the peers' ghost slots.  Ghost segments are padded to
  // 32 slots, so a warp publishes whole bitmap words with plain stores.
  DevBuf<uint32_t> nz;        // bitmap over [0, Vp): ghost-CSR in-degree > 0
  DevBuf<uint32_t> bits;      // words_for(G): frontier bit of every ghost (receive)
  DevBuf<double> sigma;       // G: frontier sigma of every ghost, 0 if not in F (receive)
  DevBuf<uint64_t> d_pub_off; // P + 1 (device copy of pub_off)
  DevBuf<uint32_t*> d_bits_dst;  // [P] q's bits + q's ghost offset of p / 32
  DevBuf<double*> d_sigma_dst;   // [P] q's sigma + q's ghost offset of p
};

struct FrontierState {  // BFS / SSSP / BC-forward (messages arrive in Part::arena_fwd)
  DevBuf<uint32_t> cur, next, visited;            // bitmaps over local ids
  DevBuf<uint32_t> vals;                          // BFS level or SSSP dist (u32, Vp)
  DevBuf<uint32_t> prev;                          // SSSP dense steps: dist before the step
  DevBuf<uint32_t> obox_mark, obox_new;           // bitmaps over outbox slots
  DevBuf<uint32_t> obox_u32;                      // SSSP / CC min-combined values
  DevBuf<uint32_t> ibox_u32;                      // CC: owner-packed labels (reverse send)
  // out-degree class bounds of the local ids (ids in out-degree order): [0,
  // n_big) >= 2048, [n_big, n_mid) >= 32 (SSSP dense supersteps; lazily)
  bool cls = false;
  uint64_t n_big = 0, n_mid = 0;
  // see Vote: 8 counters per partition, a view into Engine::ctr_all (all
  // partitions contiguous, 64 B apart: one strided memset / copy per vote)
  struct {
    unsigned long long* p = nullptr;
    size_t n = 0;
    unsigned long long* get() const { return p; }
  } counters;
};

struct BCState {
  DevBuf<double> sigma, dsum, c, bc;
  DevBuf<double> obox_sigma;              // forward partial sigma sums (send)
  DevBuf<double> ibox_pack;               // backward pull: owner-packed c (send)
  std::vector<DevBuf<uint32_t>> level_bm; // frontier bitmap per level
  DevBuf<uint32_t> ext;                   // P > 1 backward push: rows [0, Vp + S) active
  // out-degree class bounds of the local ids (ids are in out-degree order):
  // [0, n_big) >= 2048, [n_big, n_mid) >= 32; computed once (backward pull)
  bool classes = false;
  uint64_t n_big = 0, n_mid = 0;
};

struct Part {
  int id = 0;
  uint64_t Vp = 0, Ep = 0, Ep_local = 0;
  uint64_t nz_end = 0;  // local ids >= nz_end have out-degree 0
  uint32_t hub_deg = 0, hub_end = 0;  // cached: first local id with out-degree < hub_deg
  DevBuf<uint64_t> row_off;
  DevBuf<uint32_t> col, w, global_of;
  DevBuf<uint8_t> w8;  // weights as bytes when every weight < 256 (then w is released)
  // tiles
  uint64_t ntiles = 0;
  DevBuf<uint32_t> tile_vf, tile_vl;  // first / last row touched by tile t
  // outbox / inbox (padded segments)
  std::vector<uint64_t> obox_off, ibox_off;  // P+1 each (host)
  uint64_t S = 0, I = 0;                     // padded totals
  uint64_t S_real = 0, I_real = 0;
  DevBuf<uint32_t> obox_rid;  // owner's local id per slot (kInf = padding)
  DevBuf<uint32_t> ibox_lid;  // local id per inbox entry (kInf = padding)
  // PageRank in-CSR
  bool has_in = false;
  DevBuf<uint64_t> in_off;          // Vp + S + 1
  DevBuf<uint32_t> in_col;          // in-order position of the local source
  DevBuf<uint32_t> outdeg;          // out-degree per local id (Vp)
  DevBuf<uint32_t> in_nz;           // bitmap over [0, Vp): in-degree > 0 (pull candidates)
  uint64_t in_E_local = 0;          // in-edges of the local rows [0, Vp)
  uint64_t in_ntiles = 0;           // edge tiles of the in-CSR local rows
  DevBuf<uint32_t> in_tile_vf, in_tile_vl;
  // P > 1: edge tiles over every in-CSR row [0, Vp + S) (local rows + outbox
  // rows), for the BC backward push across partitions
  uint64_t in_all_ntiles = 0;
  DevBuf<uint32_t> in_all_vf, in_all_vl;
  DevBuf<uint32_t> pr_cta, pr_warp; // in-CSR rows with in-degree >= 2048 / in [32, 2048)
  uint64_t n_cta = 0, n_warp = 0;
  std::vector<uint64_t> seg_real;  // real (unpadded) outbox slots per peer
  std::vector<uint64_t> iseg_real; // real (unpadded) inbox entries per peer
  // Receive arenas (cudaMalloc'd, CUDA-IPC exportable): peers copy their
  // outbox segments into arena_fwd at this partition's inbox offsets (push),
  // owners copy packed inbox segments into arena_rev at this partition's
  // outbox offsets (pull).  8 bytes per slot covers every message type.
  DevBuf<uint8_t> arena_fwd, arena_rev;
  DevBuf<uint8_t> staging;  // result collection (multi-process): Vp x 8 bytes
  // fused-exchange tables (RemoteOut), built once the peers are known
  DevBuf<uint8_t> rmt_owner;
  DevBuf<uint8_t*> rmt_arena;
  DevBuf<int64_t> rmt_delta;
  RemoteOut rout() const { return {rmt_owner.get(), rmt_arena.get(), rmt_delta.get()}; }
  // reverse direction (pull messages, BC backward): this partition's inbox
  // entry j (segment of peer p) -> p's arena_rev at p's outbox index of it
  DevBuf<uint8_t> rin_owner;
  DevBuf<uint8_t*> rin_arena;
  DevBuf<int64_t> rin_delta;
  RemoteOut rin() const { return {rin_owner.get(), rin_arena.get(), rin_delta.get()}; }
  // algorithm state (lazily allocated)
  PRGhost gh;       // ghost-pull PageRank layout (lazy)
  TileSched ts;     // tiles of the out-CSR
  TileSched ts_in;  // tiles of the in-CSR (BC backward push)
  FrontierState fs;
  PRState pr;
  BCState bcs;
};

// What a partition exposes to the others (local pointers in one process,
// CUDA-IPC-mapped peer pointers across processes).
struct PeerView {
  uint8_t* arena_fwd = nullptr;
  uint8_t* arena_rev = nullptr;
  uint8_t* staging = nullptr;
  uint32_t* global_of = nullptr;
  uint64_t Vp = 0;
  std::vector<uint64_t> obox_off, ibox_off;  // P+1 each
  std::vector<void*> opened;                 // IPC mappings to close
};

struct Engine {
  int device = 0;
  int P = 1;          // total partitions (world when multi-process)
  int rank = 0, world = 1;
  tg_comm comm{};
  // node-local shared-memory collective (hostcomm.cu): the per-superstep vote
  // and barriers of multi-process engines; nullptr -> the tg_comm callbacks
  std::unique_ptr<HostComm> hc;
  bool multi() const { return world > 1; }
  int strategy = TG_PART_DEGREE;
  uint32_t part_seed = 0;
  double vote_ms = 0;  // host time of the votes of the current run (tg_stats.vote_ms)
  // boundary messages written by the compute kernels into the owners' arenas
  // (RemoteOut) for BFS, SSSP, PageRank and BC; TG_FUSED_EXCHANGE=0 selects
  // the outbox + copy communication phase instead
  bool fused = true;
  bool peer_atomics = true;  // every peer GPU supports native atomics on its memory
  bool peer_probe_passed = false;  // the setup self-test of peer atomics / stores ran and passed
  int pr_comm = 0;           // TG_PR_PUSH (partial sums) or TG_PR_PULL (ghost contributions)
  std::vector<PeerView> peers;  // indexed by partition id (all P)
  uint64_t V = 0, E = 0;
  bool weighted = false, has_in = false;
  // tg_attr.build_in_csr == 2: the out-CSR is released after the build (only
  // the pull PageRank runs; graphs whose two CSRs do not fit one GPU, C5)
  bool in_only = false;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // fork/join side streams (independent kernels of one phase run concurrently,
  // so one kernel's tail overlaps the next one's work); created on first use
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaEvent_t fork_ev = nullptr, join_ev[2] = {nullptr, nullptr};
  void fork();   // side streams wait for the main stream's work so far
  void join();   // the main stream waits for the side streams' work
  // Per-partition streams (one process holding several partitions of one GPU):
  // each_part(f) runs f(p) for every local partition with `stream` switched to
  // p's own stream, forked from and joined back into the main stream, so the
  // partitions' kernels of one phase overlap -- as P GPUs' would -- instead of
  // queueing one partition behind another (launch tails and small grids).
  // The phases keep their order: each call is one fork ... join.
  // TG_PART_STREAMS=0: one stream (the round-2 behaviour).
  std::vector<cudaStream_t> pstream;
  std::vector<cudaEvent_t> pjoin;
  cudaEvent_t pfork = nullptr;
  int part_streams = -1;  // resolved on first use
  bool part_streams_on();
  template <class F>
  void each_part(F&& f) {
    auto call = [&](size_t i) {
      if constexpr (std::is_invocable_v<F&, Part&, size_t>) f(*parts[i], i);
      else f(*parts[i]);
    };
    if (parts.size() <= 1 || !part_streams_on()) {
      for (size_t i = 0; i < parts.size(); ++i) call(i);
      return;
    }
    TG_CK(cudaEventRecord(pfork, stream));
    cudaStream_t const main = stream;
    // an exception in f leaves through here: restore the main stream and drain
    // the partition streams, so no work is left running unjoined
    struct Restore {
      Engine& e;
      cudaStream_t m;
      int unwinding;
      ~Restore() {
        e.stream = m;
        if (std::uncaught_exceptions() > unwinding)
          for (cudaStream_t ps : e.pstream) cudaStreamSynchronize(ps);
      }
    } restore{*this, main, std::uncaught_exceptions()};
    for (size_t i = 0; i < parts.size(); ++i) {
      TG_CK(cudaStreamWaitEvent(pstream[i], pfork, 0));
      stream = pstream[i];
      call(i);
      TG_CK(cudaEventRecord(pjoin[i], pstream[i]));
    }
    stream = main;
    for (size_t i = 0; i < parts.size(); ++i) TG_CK(cudaStreamWaitEvent(main, pjoin[i], 0));
  }
  DevBuf<uint32_t> rank_of;  // global id -> degree-order position
  DevBuf<uint8_t> scratch;   // device staging of host-bound results (V x 8 max)
  // Asynchronous host collection (tg_engine_set_async_collect): results bound
  // for host memory are gathered into one of two device staging buffers on
  // the engine stream, then copied to the host on copy_stream while the next
  // algorithm already computes; tg_engine_sync waits for the copies.  A
  // staging buffer is reused only after its previous copy finished (event).
  DevBuf<unsigned long long> reach_acc;  // reached-vertex statistics (api.cu reached)
  DevBuf<unsigned long long> ctr_all;    // vote counters of every hosted partition (8 each)
  bool async_collect = false;
  cudaStream_t copy_stream = nullptr;
  DevBuf<uint8_t> stage2[2];
  cudaEvent_t stage_free[2] = {nullptr, nullptr};
  cudaEvent_t chunk_ev = nullptr;
  int stage_next = 0;
  // collection tickets (tg_engine_last_ticket / tg_engine_wait_ticket): the
  // n-th asynchronous host collection records ticket_ev[n % kTickets] on
  // copy_stream after its last copy; a slot is reused only once its previous
  // event completed, so every ticket <= collect_seq - kTickets is complete
  static constexpr int kTickets = 16;
  uint64_t collect_seq = 0;
  cudaEvent_t ticket_ev[kTickets] = {};
  std::vector<std::unique_ptr<Part>> parts;
  uint64_t build_ms = 0;
  uint64_t launches = 0;     // kernels launched by the current run
  uint64_t comm_bytes = 0;   // message bytes exchanged by the current run
  unsigned long long* h_counts = nullptr;  // pinned, MAPPED host scratch (TG_MAX_PARTITIONS * 8)
  unsigned long long* d_counts = nullptr;  // its device alias: small results (votes, source
                                           // placement, statistics) are written there by a
                                           // kernel, not read back with a DMA copy, so they never
                                           // queue behind a result copy on the copy engines
  // kernel ledger (tg_engine_set_profiling)
  bool prof = false;
  tg_kernel_stat kstat[TG_K_COUNT] = {};
  struct Pending {
    int kid;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t prof_open = nullptr;
  int prof_open_kid = -1;
  void prof_begin(int kid);             // no-op unless prof
  void prof_end(int kid);
  void prof_bytes(int kid, double bytes) { if (prof) kstat[kid].algorithmic_bytes += bytes; }
  void prof_flush();                    // sync + accumulate pending pairs
  // L2 residency control: the hot prefix of the array a kernel gathers from
  // (degree-sorted ids put hubs first) is marked persisting in the 126 MB L2.
  size_t l2_persist = 0, l2_max_window = 0;
  bool l2_enabled = true;
  void l2_window(const void* p, size_t bytes);  // bytes == 0 clears the window
  ~Engine();
  uint64_t device_bytes() const;
  // global id -> (partition, local id); one 4-byte D2H read
  void locate(uint64_t g, int* p, uint32_t* l) const;
};

// Implemented in build.cu
struct EdgeInput {
  bool generated = false;
  const uint32_t *src = nullptr, *dst = nullptr, *w = nullptr;  // device pointers
  int scale = 0;
  double a = 0, b = 0, c = 0;
  uint64_t seed = 0, wseed = 0;
  int scramble = 1;
};
void build_engine(Engine& eng, const EdgeInput& in);
// ghost-pull PageRank layout of every hosted partition (collective across
// processes; idempotent); also sizes PRState::contrib to Vp + G
void build_pr_ghost(Engine& eng);

// Implemented per algorithm TU
void run_bfs(Engine& eng, uint64_t source, uint32_t* out, int mem, tg_stats* st);
void run_sssp(Engine& eng, uint64_t source, uint32_t* out, int mem, tg_stats* st);
void run_pagerank(Engine& eng, int iters, double d, float* out, int mem, tg_stats* st);
void run_bc(Engine& eng, const uint64_t* sources, int k, double* out, int mem, tg_stats* st);
void run_cc(Engine& eng, uint32_t* out, int mem, tg_stats* st);

// Helpers shared by the algorithm TUs (api.cu)
// Message exchange between partitions (the communication phase).
// forward (push): p's outbox segment for q -> q's inbox segment from p.
// reverse (pull): q's inbox segment from p -> p's outbox segment for q.
// send/recv return the base pointer of the per-partition array; elem = bytes
// per slot, or 0 for a bitmap (one bit per slot, segments are 32-aligned).
using BufOf = void* (*)(Part&);
void exchange(Engine& eng, BufOf send, BufOf recv, size_t elem, bool reverse);
// Communication phase of a fused exchange: the messages were written by the
// compute kernels; make them visible to their owners before anyone scatters
// (stream sync + barrier across processes; nothing to do in one process).
void fused_arrival(Engine& eng);
// Reset every hosted partition's forward arena to a byte value (before the
// first superstep of an algorithm that accumulates into it); across processes
// a barrier follows, so no peer writes into an arena being reset.
void fused_reset(Engine& eng, int byte, size_t elem);
// sum of out-degrees over reached vertices (vals != INF, or visited bits);
// *nreached (nullable) receives the number of reached vertices
uint64_t reached_outdeg_u32(Engine& eng, uint64_t* nreached = nullptr);
uint64_t reached_outdeg_bitmap(Engine& eng, uint64_t* nreached = nullptr);
void collect_u32(Engine& eng, uint32_t* out, int mem);  // fs.vals -> out[global]
// Per-vertex results in global order.  vals(p) = the hosted partition's array
// (Vp elements of `elem` bytes, local-id order).  Multi-process: gathered on
// rank 0 through the peers' IPC-mapped staging buffers; other ranks' `out`
// may be NULL.
using ValsOf = const void* (*)(Part&);
void collect(Engine& eng, ValsOf vals, size_t elem, void* out, int mem);
// host collectives (no-ops when world == 1)
void comm_allreduce(Engine& eng, uint64_t* data, int n, int op);  // op 0 sum, 1 min
void comm_barrier(Engine& eng);
void ensure_frontier_state(Engine& eng);
// copy n u64 words (src[i * stride + off]) into the mapped host scratch with a
// kernel on the engine stream, wait for the stream, return the host view
const volatile unsigned long long* to_host(Engine& eng, const unsigned long long* src, int n,
                                           int stride = 1, int off = 0);
// read the per-partition counters[idx] (one sync) and return their sum
unsigned long long read_counts(Engine& eng, int idx);
// counters layout: [0] new-frontier count (advance), [1] edges processed by the
// superstep's expand, [2] out-degree sum of the new frontier, [3] its in-degree
// sum, [4] error flags, [5] minimum value over the new frontier (SSSP: the
// smallest tentative distance).  One sync for all partitions.
struct Vote {
  unsigned long long count = 0, edges = 0, degsum = 0, indegsum = 0, minval = ~0ull;
};
Vote read_vote(Engine& eng);
// zero counters[0..1] of every partition (start of a superstep)
void reset_vote(Engine& eng);
void time_begin(Engine& eng);
double time_end(Engine& eng);  // ms since time_begin (CUDA events)

}  // namespace tg
