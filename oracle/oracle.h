/*
 * oracle.h -- plain, slow, single-threaded CPU ORACLE for the TOTEM BSP hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library.  The CUDA product path (paper_1312_3018_b200/) never links,
 * imports or executes it, and shares no code with it except the seeded input
 * generator inputs/tg_inputs.h (no method arithmetic there).
 *
 * Every function states the definition it writes out (a plain definition, so
 * these are NOT the paper's parallel BSP kernels: BFS is a FIFO queue, SSSP is
 * Dijkstra, PageRank is the Jacobi recurrence, BC is Brandes' queue+stack).
 * "P:n" = /root/reference/PAPER.md line n.  Integers use uint64 internally,
 * floating point is fp64.
 *
 * Pins (tests/test_oracle.py): exhaustive / brute force / closed forms for
 * every function; see DESIGN.md "Oracle pins".  Parity pinned for all
 * functions below except the graph generator itself (no "correct RMAT"
 * exists beyond its parameters -- "parity unpinned" for tg_inputs.h, which is
 * shared input, not an oracle).
 *
 * Return codes: 0 ok, 2 invalid argument, 3 out of memory, 5 internal
 * (e.g. SSSP distance exceeds uint32).
 */
#ifndef TG_ORACLE_H
#define TG_ORACLE_H
#include <stdint.h>

#define ORACLE_INF32 0xFFFFFFFFu

/* CSR of a directed multigraph (§4.3.1: arrays V and E), built by a
 * stable counting sort of the edge list by source: the edges of vertex v are
 * col[row_off[v] .. row_off[v+1]) in input order.  w/wout nullable. */
int oracle_csr(uint64_t V, uint64_t E, const uint32_t* src, const uint32_t* dst,
               const uint32_t* w, uint64_t* row_off, uint32_t* col, uint32_t* wout);

/* BFS levels (Fig. 11): level[v] = minimum number of edges
 * on a directed path s->v, ORACLE_INF32 if none.  FIFO queue. */
int oracle_bfs(uint64_t V, const uint64_t* row_off, const uint32_t* col, uint64_t s,
               uint32_t* level);

/* SSSP distances (Fig. 20): dist[v] = minimum sum of weights over
 * directed s->v paths, ORACLE_INF32 if unreachable.  Dijkstra with an indexed
 * binary heap over uint64 keys; returns 5 if a distance does not fit uint32. */
int oracle_sssp(uint64_t V, const uint64_t* row_off, const uint32_t* col, const uint32_t* w,
                uint64_t s, uint32_t* dist);

/* PageRank, T Jacobi iterations (Fig. 14; readings A1-A7):
 *   r_0[v] = 1/|V|;  c_t[u] = r_t[u]/outdeg(u) (0 if outdeg(u) = 0)
 *   r_{t+1}[v] = (1-d)/|V| + d * sum_{(u,v) in E} c_t[u]   (multiplicity counted) */
int oracle_pagerank(uint64_t V, const uint64_t* row_off, const uint32_t* col, int T, double d,
                    double* rank);

/* Betweenness centrality over a source list (Fig. 18; Brandes 2001,
 * readings A9-A12): bc[v] = sum_{s in S, s != v} delta_s(v),
 *   delta_s(v) = sum_{(v,w) in E, d(w) = d(v)+1} sigma(v)/sigma(w) * (1 + delta_s(w)),
 * sigma counting shortest paths as edge sequences (parallel edges distinct).
 * Unnormalised, directed.  bc is overwritten. */
int oracle_bc(uint64_t V, const uint64_t* row_off, const uint32_t* col, const uint64_t* sources,
              int k, double* bc);

/* Connected components of the graph read as UNDIRECTED ("minimum 'label'
 * in a connected components algorithm"; Table 5 note: CC "operates on
 * undirected graphs"): label[v] = the smallest vertex id in
 * v's weakly connected component.  Union-find (union by smaller root id, path
 * halving) over every edge, then each vertex takes its root, which is the
 * minimum of its set by construction.  Not the paper's label propagation. */
int oracle_cc(uint64_t V, const uint64_t* row_off, const uint32_t* col, uint32_t* label);
/* Streaming form: parent[] (length V, initialised parent[v] = v by the caller)
 * absorbs edge chunks; oracle_cc_finish writes the labels. */
int oracle_cc_edges(uint64_t V, uint32_t* parent, uint64_t n, const uint32_t* src,
                    const uint32_t* dst);
int oracle_cc_finish(uint64_t V, uint32_t* parent, uint32_t* label);

/* Degree-aware partition (reading A23; §6.2 degree centrality):
 * vertices ordered by out-degree descending, ties by id ascending, dealt in
 * serpentine order over P partitions: order position i, round r = i / P,
 * j = i % P, part = (r even ? j : P-1-j), local id = r. */
int oracle_partition(uint64_t V, const uint64_t* row_off, int P, uint32_t* part, uint32_t* local);

/* The "naive random-based" partitioning the paper compares against
 * (§3.4, Fig. 4; RAND of P:427): vertices ordered by a random key
 * (key[v], ties by id), position i dealt serpentine as above (equal vertex
 * counts, degree-blind); inside each partition the local ids follow out-degree
 * desc, id asc (the same local order as the degree-aware rule).  key[] is the
 * seeded draw of inputs/tg_inputs.h (tgin_part_key), passed in. */
int oracle_partition_random(uint64_t V, const uint64_t* row_off, int P, const uint32_t* key,
                            uint32_t* part, uint32_t* local);

/* Boundary statistics (§3.4): beta_raw = cross-partition
 * edges / |E|; beta_reduced = distinct (part(src), dst) pairs with
 * part(dst) != part(src), / |E|.  slots (nullable, P*P, row-major [p][q]):
 * number of distinct remote targets in q referenced from p = outbox size p->q. */
int oracle_beta(uint64_t V, uint64_t E, const uint32_t* src, const uint32_t* dst,
                const uint32_t* part, int P, double* beta_raw, double* beta_reduced,
                uint64_t* slots);

/* BFS certificate: returns 0 iff level[] equals the BFS distances from s
 * (level[s]=0; every edge from a reached u has level[v] <= level[u]+1; every
 * reached v != s has an in-edge from u with level[u] = level[v]-1; no edge
 * from a reached vertex enters an unreached one).  *bad = first offender. */
int oracle_bfs_certify(uint64_t V, const uint64_t* row_off, const uint32_t* col, uint64_t s,
                       const uint32_t* level, uint64_t* bad);

/* SSSP certificate (weights >= 1): dist[s]=0, no edge relaxable, every
 * reached v != s has a tight in-edge, unreached have no in-edge from reached. */
int oracle_sssp_certify(uint64_t V, const uint64_t* row_off, const uint32_t* col,
                        const uint32_t* w, uint64_t s, const uint32_t* dist, uint64_t* bad);

/* ---- streaming certificates for graphs too large for an in-memory CSR ------
 * (the full-size RMAT-28 checks in the bench launch configuration).  The edge
 * stream is regenerated by the caller in chunks (inputs/tg_inputs.h); each
 * call folds one chunk.  These loops are the definitions above written over an
 * edge list instead of a CSR; they are OpenMP-parallel over the chunk (the
 * only parallel code in the oracle) because 2^32 edges must be checked.
 * tight: caller-zeroed bitmap of V bits (uint64 words).  Returns the number
 * of violating edges in *bad (added). */
int oracle_outdeg_edges(uint64_t V, uint64_t n, const uint32_t* src, uint32_t* outdeg);
/* BFS: for every edge (u,v) with level[u] reached: level[v] <= level[u]+1;
 * level[v] == level[u]+1 marks v tight. */
int oracle_bfs_cert_edges(uint64_t V, const uint32_t* level, uint64_t n, const uint32_t* src,
                          const uint32_t* dst, uint64_t* tight, uint64_t* bad);
/* SSSP: for every edge (u,v,w) with dist[u] reached: dist[v] <= dist[u]+w;
 * equality marks v tight. */
int oracle_sssp_cert_edges(uint64_t V, const uint32_t* dist, uint64_t n, const uint32_t* src,
                           const uint32_t* dst, const uint32_t* w, uint64_t* tight, uint64_t* bad);
/* Finish either certificate: val[s] == 0 and every reached v != s is tight.
 * Returns 0 iff the certificate holds; *bad = first offender. */
int oracle_cert_finish(uint64_t V, uint64_t s, const uint32_t* val, const uint64_t* tight,
                       uint64_t* bad);
/* PageRank one-round recurrence on a vertex sample: for edges (u,v) with v in
 * the sample (mask bit set), acc[slot[v]] += r_prev[u] / outdeg[u]. */
int oracle_pr_sample_edges(uint64_t V, uint64_t n, const uint32_t* src, const uint32_t* dst,
                           const uint64_t* mask, const uint32_t* slot, const float* r_prev,
                           const uint32_t* outdeg, double* acc);

#endif
