/*
 * tgraph.h -- C ABI of the B200-native BSP graph superstep library (libtgraph.so).
 *
 * The library implements the data-parallel hot path of TOTEM (Gharaibeh et al.,
 * arXiv 1312.3018; "P:n" below = /root/reference/PAPER.md line n): the BSP
 * superstep over a partitioned CSR graph (§4.1) -- a compute phase per
 * partition (BFS frontier expansion, PageRank pull-sum, SSSP relaxation, Brandes
 * BC forward/backward) followed by a communication phase in which each
 * partition's source-reduced boundary-edge outbox is delivered to the owner
 * partition's inbox (§4.3.2) -- and the termination vote.
 *
 * The calling sequence follows the paper's statement of the problem (Appendix 1,
 * P:955-971): load an edge list into CSR and partition it (tg_engine_create_*,
 * P:958-964 graph_initialize + totem_init), run an algorithm with its source or
 * iteration count, read back per-vertex state in global vertex order
 * (totem_engine_collect).
 *
 * Conventions (all functions):
 *   - extern "C", plain pointers and sizes, no C++/torch types.
 *   - Return an int status (tg_status); never throw, never abort.  On a non-zero
 *     return tg_last_error() gives a thread-local message.
 *   - Vertex ids are uint32 values in [0, V), V <= 2^31; edge counts uint64.
 *   - Caller arrays are never retained after a call returns (the library copies
 *     what it needs).  Output arrays are caller-allocated, length V, indexed by
 *     GLOBAL vertex id, in host or device memory as `mem` says.
 *   - An engine is not re-entrant: one call at a time per engine.
 */
#ifndef TGRAPH_H
#define TGRAPH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TG_OK = 0,
  TG_EINVAL = 2,     /* bad argument: source >= V, id >= V, iterations < 1, a+b+c > 1,
                        SSSP on an engine built without weights, NULL output, ...    */
  TG_ECAPACITY = 3,  /* too many partitions / vertices, or does not fit device memory */
  TG_EIO = 4,        /* reserved for file I/O */
  TG_EINTERNAL = 5,  /* internal invariant violated (e.g. SSSP distance overflows u32) */
  TG_ECUDA = 6,      /* CUDA runtime error (message carries cudaGetErrorString)         */
  TG_ENCCL = 7,      /* NCCL error / NCCL transport unavailable                          */
} tg_status;

/* Where a caller array lives. */
typedef enum { TG_MEM_HOST = 0, TG_MEM_DEVICE = 1 } tg_mem;

/* 0xFFFFFFFF: "unreached" for BFS levels and SSSP distances (reading A16). */
#define TG_INF32 0xFFFFFFFFu
#define TG_MAX_PARTITIONS 64

const char* tg_version(void);
/* Message for the last non-OK return on this thread ("" if none). */
const char* tg_last_error(void);

typedef struct tg_engine tg_engine;

/* Host-side communicator for multi-process engines (one process per GPU).
 * The library moves boundary messages itself (CUDA IPC-mapped peer memory:
 * NVLink/NVSwitch peer copies between GPUs); it only needs these two host
 * collectives for metadata, the per-superstep vote and barriers.
 * Both are collective over all `world` processes and must return 0 on success.
 *   allgather(ctx, send, recv, bytes): recv[r*bytes .. (r+1)*bytes) = rank r's send.
 *   allreduce_u64(ctx, data, n, op): in place, op 0 = sum, 1 = min. */
typedef struct {
  void* ctx;
  int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes);
  int (*allreduce_u64)(void* ctx, uint64_t* data, int n, int op);
} tg_comm;

/* The library's node-local host collective (the per-superstep termination
 * vote of P:208 and App. 1, whose shared `finished` flag lives in
 * host memory): a POSIX shared-memory segment mapped by the `world` processes
 * of one node.  Multi-process engines create one internally; these entry
 * points expose the same object for tests and tools.
 *   tg_hostcomm_create: collective over the ranks of `comm` (allgather of the
 *     segment name + one barrier).  TG_ENCCL if a rank could not map it.
 *   tg_hostcomm_allreduce_u64: in place over n <= 16 values; ops[i] 0 = sum
 *     (mod 2^64), 1 = min.  Collective, same n and ops on every rank.
 *     TG_ENCCL if a peer does not arrive within 600 s; TG_EINVAL for bad n.
 * The segment's name is unlinked once every rank has mapped it. */
typedef struct tg_hostcomm tg_hostcomm;
int tg_hostcomm_create(const tg_comm* comm, int rank, int world, tg_hostcomm** out);
int tg_hostcomm_allreduce_u64(tg_hostcomm* h, uint64_t* data, int n, const int* ops);
void tg_hostcomm_free(tg_hostcomm* h);

/* Engine attributes (the paper's totem_attr_t, re-aimed at GPUs).
 *   num_partitions: logical partitions hosted on this process's device, >= 1
 *       (world == 1 only).  Vertices are dealt to partitions by the
 *       degree-aware serpentine rule (reading A23; §6.2):
 *       order by out-degree desc, id asc; position i -> round r = i/P,
 *       j = i%P, partition (r even ? j : P-1-j), local id r.  P > 1 on one
 *       device exercises the full outbox/inbox machinery in one process.
 *   device: CUDA device ordinal.
 *   weighted: 1 to keep per-edge SSSP weights (required by tg_sssp).
 *   build_in_csr: 1 to build the in-edge CSR used by tg_pagerank (pull);
 *       2 = in-CSR only: the out-CSR is released after the build, so only
 *       tg_pagerank runs (the others return TG_EINVAL) -- for a graph whose
 *       two CSRs do not fit one device (RMAT-30 PageRank on one B200);
 *       single-process engines only.
 *   rank, world: multi-process engine (world > 1): this process hosts
 *       partition `rank` of `world` (num_partitions must be 1); every process
 *       makes the same calls in the same order (SPMD), results are written on
 *       rank 0 only (other ranks may pass NULL outputs).
 *   comm: required when world > 1 (copied; must outlive the engine).  Used
 *       at setup (IPC handle exchange) and, where a node-local shared-memory
 *       segment cannot be created, for the per-superstep vote; normally the
 *       per-superstep vote and arrival barrier run in the library's own
 *       shared-memory collective (no callback on the per-superstep path).
 *   strategy: how vertices are dealt to partitions (§6.2
 *       lists HIGH / LOW / RAND; Fig. 4 compares against "naive
 *       random-based" partitioning):
 *       TG_PART_DEGREE (0, default): degree-aware serpentine deal above;
 *       TG_PART_RANDOM (1): partition of v = serpentine deal of v's position in
 *       a seeded pseudo-random order (tg_inputs.h mix64 of (part_seed, v);
 *       equal vertex counts, degree-blind).  Under both strategies local ids
 *       inside a partition are in out-degree order (desc, id asc).
 *   part_seed: seed of TG_PART_RANDOM (ignored otherwise).
 * TG_EINVAL for an unknown strategy. */
enum { TG_PART_DEGREE = 0, TG_PART_RANDOM = 1 };
typedef struct {
  int num_partitions;
  int device;
  int weighted;
  int build_in_csr;
  int rank;
  int world;
  const tg_comm* comm;
  int strategy;
  int part_seed;
} tg_attr;

/* Build an engine from an explicit directed edge list (duplicates and
 * self-loops kept).  src/dst/w have length E and live in `mem`; w may be NULL
 * (unweighted).  Every id must be < V (else TG_EINVAL).  V in [1, 2^31). */
int tg_engine_create_edges(uint64_t V, uint64_t E, const uint32_t* src, const uint32_t* dst,
                           const uint32_t* w, int mem, const tg_attr* attr, tg_engine** out);

/* Build an engine from the RMAT stream of inputs/tg_inputs.h, generated on the
 * device (Table 2: (A,B,C)=(0.57,0.19,0.19), degree 16).  E =
 * edge_factor * 2^scale; weights drawn from wseed when attr->weighted.
 * TG_EINVAL if a+b+c > 1, scale outside [1,31] or edge_factor < 1. */
int tg_engine_create_rmat(int scale, int edge_factor, double a, double b, double c,
                          uint64_t seed, int scramble, uint64_t wseed, const tg_attr* attr,
                          tg_engine** out);

void tg_engine_free(tg_engine* eng);

/* ---- host graphs and input generation ------------------------------------
 * The load step of the paper's calling sequence (graph_initialize) as a
 * library-owned host edge list that tg_engine_create partitions and uploads.
 * Edge order is kept as given (the engine sorts each CSR row itself). */
typedef struct tg_graph tg_graph;

/* Copy an explicit directed edge list (host arrays of length E; w nullable =
 * unweighted).  TG_EINVAL if an id is >= V or V is outside [1, 2^31). */
int tg_graph_from_edges(uint64_t V, uint64_t E, const uint32_t* src, const uint32_t* dst,
                        const uint32_t* w, tg_graph** out);

/* Text edge list (the paper's loader is artifact plumbing):
 * one edge per line, "src dst" or, with weighted = 1, "src dst weight";
 * blank lines and lines starting with '#' are skipped; a comment "# nodes: N"
 * fixes V (otherwise V = 1 + max id).  directed = 0 stores every edge in both
 * directions.  Errors: TG_EIO if the file cannot be read; TG_EINVAL for a
 * malformed line, a negative or missing weight, or an id >= the declared V --
 * the message names the line number. */
int tg_graph_load_edge_list(const char* path, int directed, int weighted, tg_graph** out);

int tg_graph_info(const tg_graph* g, uint64_t* V, uint64_t* E, int* weighted);
/* Copy the edges out (host arrays of length E; w ignored when NULL or when the
 * graph is unweighted). */
int tg_graph_edges(const tg_graph* g, uint32_t* src, uint32_t* dst, uint32_t* w);
void tg_graph_free(tg_graph* g);

/* Partition + upload a host graph (same attributes and rules as
 * tg_engine_create_edges; attr->weighted requires a weighted graph). */
int tg_engine_create(const tg_graph* g, const tg_attr* attr, tg_engine** out);

/* Edges [first, first+count) of the RMAT stream tg_engine_create_rmat builds
 * from (inputs/tg_inputs.h: counter-based, so any slice is independent),
 * generated on the calling thread's current CUDA device into src/dst (and the
 * SSSP weights 1 + mix64(wseed*phi + k) mod 63 into w when w != NULL), arrays
 * of length count in `mem`.  (a, b, c) = (0.25, 0.25, 0.25) is the UNIFORM
 * graph (every endpoint bit independent and fair).  TG_EINVAL as
 * tg_engine_create_rmat, or if first + count > edge_factor * 2^scale. */
int tg_rmat_edges(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                  int scramble, uint64_t wseed, uint64_t first, uint64_t count, uint32_t* src,
                  uint32_t* dst, uint32_t* w, int mem);

/* |V_p| of partition p of P under the degree-serpentine deal (host only; no
 * device needed): rounds r = i / P deal positions j = i % P to partition
 * (r even ? j : P-1-j).  TG_EINVAL if P < 1, P > TG_MAX_PARTITIONS or p out of
 * range. */
int tg_partition_size(uint64_t V, int p, int P, uint64_t* Vp);

typedef struct {
  uint64_t V, E;
  int num_partitions;
  int weighted, has_in_csr;
  uint64_t device_bytes;     /* bytes of device memory held by the engine */
  uint64_t build_ms;         /* wall time of the build, milliseconds       */
  int device;                /* CUDA device ordinal of this process's partition(s) */
  int strategy;              /* TG_PART_DEGREE / TG_PART_RANDOM                */
  int exchange;              /* current TG_EXCHANGE_* transport                */
  int pr_comm;               /* current TG_PR_* PageRank communication         */
  int peer_probe;            /* multi-process: 1 if the setup self-test of peer atomics and
                                stores through the CUDA-IPC mappings ran and passed (the
                                fused transport is only kept when it passes)         */
} tg_info;
int tg_engine_info(const tg_engine* eng, tg_info* info);

/* Per-partition layout (§4.3.1-4.3.2).  slots_to[q] (length P,
 * nullable) = outbox entries of p destined to q = distinct remote vertices of q
 * referenced from p (source-side reduction, §3.4). */
typedef struct {
  uint64_t Vp, Ep;           /* owned vertices, owned out-edges             */
  uint64_t Ep_local;         /* out-edges whose target is owned by p        */
  uint64_t outbox_slots;     /* |V_o| of P:267                              */
  uint64_t inbox_slots;      /* |V_i| of P:265                              */
} tg_part_info;
int tg_engine_partition_info(const tg_engine* eng, int p, tg_part_info* info, uint64_t* slots_to);

/* Run statistics.  device_ms: CUDA-event time on the engine stream from state
 * initialisation to the final vote (the paper's timed scope; result
 * collection excluded).  traversed_edges: the paper's TEPS numerator:
 * BFS/SSSP = sum of out-degrees of reached vertices; BC = 2x that per source;
 * PageRank = |E| x iterations.  supersteps: BSP rounds executed.
 * algorithmic_bytes: DESIGN.md §Roofline count for the run.  comm_bytes:
 * inbox/outbox message bytes moved between partitions.  launches: kernels.
 * relaxations: edges the compute kernels examined (SSSP: every relaxation,
 * repeats included, so relaxations / traversed_edges is Bellman-Ford's
 * redundancy; BFS/BC: out-edges expanded plus in-edges scanned bottom-up;
 * PageRank: |E| x iterations).
 * The phase split of SURVEY 8(d) (compute / exchange / vote):
 *   exchange_ms: communication phase (arrival or copies + scatter), summed
 *     CUDA-event intervals -- filled only while the kernel ledger is on
 *     (tg_engine_set_profiling), else 0;
 *   compute_ms: the compute kernels' ledger time (same condition);
 *   vote_ms: host wall time of the termination votes after the stream has
 *     drained (device->host read of the counters + the cross-process
 *     reduction), always filled. */
typedef struct {
  double device_ms;
  uint64_t supersteps;
  uint64_t traversed_edges;
  uint64_t algorithmic_bytes;
  uint64_t comm_bytes;
  uint64_t launches;
  uint64_t relaxations;
  double compute_ms, exchange_ms, vote_ms;
} tg_stats;

/* Level-synchronous BFS (Fig. 11; App. 1).  levels[v] =
 * hop distance from source, TG_INF32 if unreached.  stats nullable. */
int tg_bfs(tg_engine* eng, uint64_t source, uint32_t* levels, int mem, tg_stats* stats);

/* Bellman-Ford SSSP over BSP (Fig. 20).  dist[v] = minimum weight sum,
 * TG_INF32 if unreached.  TG_EINVAL if the engine has no weights, TG_EINTERNAL
 * if a distance overflows uint32. */
int tg_sssp(tg_engine* eng, uint64_t source, uint32_t* dist, int mem, tg_stats* stats);

/* Pull PageRank, `iterations` Jacobi rounds (Fig. 14, readings A1-A8):
 * r_0 = 1/V; r_{t+1}[v] = (1-d)/V + d * sum_{(u,v)} r_t[u]/outdeg(u).
 * rank is float32 (4-byte rank).  TG_EINVAL if iterations < 1 or the
 * engine was built without the in-CSR. */
int tg_pagerank(tg_engine* eng, int iterations, double damping, float* rank, int mem,
                tg_stats* stats);

/* Brandes betweenness centrality over k sources (Fig. 18; readings
 * A9-A14): bc[v] = sum over sources s != v of delta_s(v), fp64, unnormalised,
 * directed.  sources: host array of k global ids.  bc overwritten. */
int tg_bc(tg_engine* eng, const uint64_t* sources, int k, double* bc, int mem, tg_stats* stats);

/* Connected components by minimum-label propagation ("minimum 'label' in
 * a connected components algorithm"; CC operates on undirected graphs;
 * reading A29): the engine's directed edges are read as undirected, and
 * labels[v] = the smallest global vertex id of v's (weakly) connected
 * component.  Needs the in-CSR (attr.build_in_csr), else TG_EINVAL.
 * traversed_edges = |E| (each input edge once). */
int tg_cc(tg_engine* eng, uint32_t* labels, int mem, tg_stats* stats);

/* ---- kernel ledger (measurement) --------------------------------------------
 * With profiling on, the library brackets each hot kernel launch with CUDA
 * events on the engine stream (the stream the kernel runs on) and accumulates,
 * per kernel id: launches, summed event time and the ALGORITHMIC bytes the
 * launch had to move (per-edge and per-vertex figures x
 * the edges / vertices that launch processed).  Off by default. */
typedef enum {
  TG_K_BFS_EXPAND = 0,   /* BFS frontier expansion (edge tiles)           */
  TG_K_SSSP_EXPAND = 1,  /* SSSP relaxation (edge tiles)                  */
  TG_K_BCF_EXPAND = 2,   /* BC forward: BFS + sigma (edge tiles)          */
  TG_K_BCB_EXPAND = 3,   /* BC backward: dependency pull (edge tiles)     */
  TG_K_PR_PULL = 4,      /* PageRank pull-sum, all degree classes, 1 iter */
  TG_K_ADVANCE = 5,      /* frontier advance / vote count                 */
  TG_K_COMPACT = 6,      /* active-tile compaction                        */
  TG_K_EXCHANGE = 7,     /* inter-partition message exchange + scatter    */
  TG_K_CC_EXPAND = 8,    /* CC label push, out- and in-CSR (edge tiles)   */
  TG_K_COUNT = 9
} tg_kernel_id;

typedef struct {
  uint64_t launches;
  double ms;                 /* summed CUDA-event time                        */
  double algorithmic_bytes;  /* summed algorithmic bytes of those launches    */
} tg_kernel_stat;

int tg_engine_set_profiling(tg_engine* eng, int on);   /* also resets the ledger */

/* Communication-phase transport of the boundary messages (PAPER.md:207 and
 * P:256 §4.3.2 "the communication phase"; SURVEY 8(e) fusion candidates).
 *   TG_EXCHANGE_FUSED (default): BFS, SSSP, PageRank, BC and CC kernels write
 *     each boundary message straight into the receiving partition's arena
 *     (same-process pointer, or a CUDA-IPC-mapped peer pointer: NVLink stores
 *     and reductions between GPUs); the phase is an arrival barrier only.
 *   TG_EXCHANGE_COPY: messages are staged in the outbox and copied segment by
 *     segment into the owners' arenas (the paper's outbox -> inbox transfer).
 * Results are identical in both modes.  Engines
 * spanning processes: every rank must select the same mode before its next
 * algorithm call (SPMD).  TG_EINVAL for NULL, an unknown mode, or FUSED on a
 * multi-process engine whose GPUs lack native peer atomics (such an engine
 * starts in COPY mode).
 * The environment variable TG_FUSED_EXCHANGE=0 sets the default to COPY. */
enum { TG_EXCHANGE_COPY = 0, TG_EXCHANGE_FUSED = 1 };
int tg_engine_set_exchange(tg_engine* eng, int mode);

/* PageRank communication (PAPER.md:182 vs P:945-946; reading A8).
 *   TG_PR_PUSH (default): each partition sums its sources' contributions per
 *     remote target (outbox row of the in-CSR) and sends one partial sum per
 *     target; the owner adds them (source-side reduction).
 *   TG_PR_PULL: TOTEM_COMM_PULL -- each partition publishes the contribution
 *     of every source with an out-edge into a peer, into ghost slots appended
 *     to that peer's contribution array, and pulls over a ghost-indexed in-CSR
 *     (built on the first PULL run, outside the timed region; across
 *     processes the publish stores go to CUDA-IPC-mapped peer buffers and the
 *     build is collective: every rank must select the same mode, SPMD).
 * Results equal up to fp64 summation order (1e-5 relative per vertex).
 * TG_EINVAL for NULL or an unknown mode. */
enum { TG_PR_PUSH = 0, TG_PR_PULL = 1 };
int tg_engine_set_pagerank_comm(tg_engine* eng, int mode);

/* The SM -> die map of a two-die GPU (B200: each die's half of the L2 caches
 * the lines its own SMs read), measured once per device by a pointer-chase
 * latency probe (dies.cu) and cached.  PageRank's die split (pagerank.cu)
 * uses it to give each die's SMs their own half of the gathered sources.
 * die_of (host, cap entries, may be NULL) receives die 0 / 1 per SM id;
 * *nsm the SM count; *ok = 1 if two clear latency clusters were found (0: a
 * one-die part or an unclear probe -> no die split).  TG_EINVAL for a bad
 * device or NULL nsm / ok. */
int tg_device_die_map(int device, uint8_t* die_of, int cap, int* nsm, int* ok);

/* Asynchronous result collection into HOST memory (single-process engines;
 * the collection step of P:902-913, outside the paper's timed scope).  With
 * on = 1, an algorithm call that writes a host output array returns once its
 * results are gathered on the device: the device->host copy proceeds on a
 * copy stream, overlapping the caller's next algorithm call, and the host
 * array is complete only after tg_engine_sync.  Device outputs, stats and
 * errors are unaffected.  The caller must not free or read a host output
 * before tg_engine_sync.  on = 0 (default): outputs are complete on return.
 * TG_EINVAL for NULL; ignored (stays synchronous) on multi-process engines. */
int tg_engine_set_async_collect(tg_engine* eng, int on);
/* Wait for every pending result copy (and the engine's stream). */
int tg_engine_sync(tg_engine* eng);
/* Finer-grained completion of asynchronous host collections: every algorithm
 * call whose output went to host memory under async collect gets the next
 * ticket (1, 2, ...); tg_engine_last_ticket returns the latest (0 if none)
 * and tg_engine_wait_ticket(t) returns once collection t and every earlier
 * one is complete in host memory (ticket 0: returns at once).  A caller can
 * so keep two output sets in flight -- wait for call k's ticket while call
 * k+1 computes (double buffering).  TG_EINVAL for NULL or a ticket not yet
 * issued. */
int tg_engine_last_ticket(const tg_engine* eng, uint64_t* ticket);
int tg_engine_wait_ticket(tg_engine* eng, uint64_t ticket);
int tg_engine_kernel_stat(const tg_engine* eng, int kernel_id, tg_kernel_stat* out);
const char* tg_kernel_name(int kernel_id);

#ifdef __cplusplus
}
#endif
#endif /* TGRAPH_H */
