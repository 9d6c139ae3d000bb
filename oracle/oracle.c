/*
 * oracle.c -- see oracle.h.  TEST INFRASTRUCTURE ONLY (tests/, smoke(),
 * bench.py cpu_baseline / --impl reference).  Single-threaded, plain C99.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

#define OK 0
#define EINVAL_ 2
#define ENOMEM_ 3
#define EINTERNAL_ 5

int oracle_csr(uint64_t V, uint64_t E, const uint32_t* src, const uint32_t* dst,
               const uint32_t* w, uint64_t* row_off, uint32_t* col, uint32_t* wout) {
  if (!row_off || (E && (!src || !dst || !col))) return EINVAL_;
  for (uint64_t e = 0; e < E; ++e)
    if (src[e] >= V || dst[e] >= V) return EINVAL_;
  memset(row_off, 0, (V + 1) * sizeof(uint64_t));
  for (uint64_t e = 0; e < E; ++e) row_off[src[e] + 1]++;
  for (uint64_t v = 0; v < V; ++v) row_off[v + 1] += row_off[v];
  uint64_t* cur = (uint64_t*)malloc((V + 1) * sizeof(uint64_t));
  if (!cur) return ENOMEM_;
  memcpy(cur, row_off, (V + 1) * sizeof(uint64_t));
  for (uint64_t e = 0; e < E; ++e) {
    const uint64_t pos = cur[src[e]]++;
    col[pos] = dst[e];
    if (w && wout) wout[pos] = w[e];
  }
  free(cur);
  return OK;
}

int oracle_bfs(uint64_t V, const uint64_t* row_off, const uint32_t* col, uint64_t s,
               uint32_t* level) {
  if (s >= V || !level || !row_off) return EINVAL_;
  uint32_t* queue = (uint32_t*)malloc(V * sizeof(uint32_t));
  if (!queue) return ENOMEM_;
  for (uint64_t v = 0; v < V; ++v) level[v] = ORACLE_INF32;
  uint64_t head = 0, tail = 0;
  level[s] = 0;
  queue[tail++] = (uint32_t)s;
  while (head < tail) {
    const uint32_t u = queue[head++];
    for (uint64_t e = row_off[u]; e < row_off[u + 1]; ++e) {
      const uint32_t v = col[e];
      if (level[v] == ORACLE_INF32) {
        level[v] = level[u] + 1;
        queue[tail++] = v;
      }
    }
  }
  free(queue);
  return OK;
}

/* ---- Dijkstra with an indexed binary min-heap on uint64 distances ---- */
typedef struct {
  uint32_t* heap; /* vertex ids */
  int64_t* pos;   /* position of vertex in heap, -1 if absent */
  uint64_t* key;
  uint64_t n;
} iheap;

static void ih_swap(iheap* h, uint64_t i, uint64_t j) {
  uint32_t a = h->heap[i], b = h->heap[j];
  h->heap[i] = b;
  h->heap[j] = a;
  h->pos[b] = (int64_t)i;
  h->pos[a] = (int64_t)j;
}
static void ih_up(iheap* h, uint64_t i) {
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (h->key[h->heap[p]] <= h->key[h->heap[i]]) break;
    ih_swap(h, i, p);
    i = p;
  }
}
static void ih_down(iheap* h, uint64_t i) {
  for (;;) {
    uint64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && h->key[h->heap[l]] < h->key[h->heap[m]]) m = l;
    if (r < h->n && h->key[h->heap[r]] < h->key[h->heap[m]]) m = r;
    if (m == i) break;
    ih_swap(h, i, m);
    i = m;
  }
}

int oracle_sssp(uint64_t V, const uint64_t* row_off, const uint32_t* col, const uint32_t* w,
                uint64_t s, uint32_t* dist) {
  if (s >= V || !dist || !row_off || !w) return EINVAL_;
  const uint64_t INF = ~0ULL;
  iheap h;
  h.heap = (uint32_t*)malloc(V * sizeof(uint32_t));
  h.pos = (int64_t*)malloc(V * sizeof(int64_t));
  h.key = (uint64_t*)malloc(V * sizeof(uint64_t));
  uint8_t* done = (uint8_t*)calloc(V, 1);
  if (!h.heap || !h.pos || !h.key || !done) {
    free(h.heap); free(h.pos); free(h.key); free(done);
    return ENOMEM_;
  }
  h.n = 0;
  for (uint64_t v = 0; v < V; ++v) { h.key[v] = INF; h.pos[v] = -1; }
  h.key[s] = 0;
  h.heap[0] = (uint32_t)s; h.pos[s] = 0; h.n = 1;
  while (h.n) {
    const uint32_t u = h.heap[0];
    ih_swap(&h, 0, h.n - 1);
    h.pos[u] = -1;
    h.n--;
    if (h.n) ih_down(&h, 0);
    done[u] = 1;
    for (uint64_t e = row_off[u]; e < row_off[u + 1]; ++e) {
      const uint32_t v = col[e];
      if (done[v]) continue;
      const uint64_t nd = h.key[u] + (uint64_t)w[e];
      if (nd < h.key[v]) {
        h.key[v] = nd;
        if (h.pos[v] < 0) { h.heap[h.n] = v; h.pos[v] = (int64_t)h.n; h.n++; }
        ih_up(&h, (uint64_t)h.pos[v]);
      }
    }
  }
  int rc = OK;
  for (uint64_t v = 0; v < V; ++v) {
    if (h.key[v] == INF) dist[v] = ORACLE_INF32;
    else if (h.key[v] >= ORACLE_INF32) { dist[v] = ORACLE_INF32; rc = EINTERNAL_; }
    else dist[v] = (uint32_t)h.key[v];
  }
  free(h.heap); free(h.pos); free(h.key); free(done);
  return rc;
}

int oracle_pagerank(uint64_t V, const uint64_t* row_off, const uint32_t* col, int T, double d,
                    double* rank) {
  if (V == 0 || T < 1 || !rank || !row_off) return EINVAL_;
  double* acc = (double*)malloc(V * sizeof(double));
  if (!acc) return ENOMEM_;
  const double base = (1.0 - d) / (double)V;
  for (uint64_t v = 0; v < V; ++v) rank[v] = 1.0 / (double)V;          /* r_0 */
  for (int t = 0; t < T; ++t) {
    for (uint64_t v = 0; v < V; ++v) acc[v] = 0.0;
    for (uint64_t u = 0; u < V; ++u) {
      const uint64_t deg = row_off[u + 1] - row_off[u];
      if (deg == 0) continue;                                          /* dangling: c = 0 */
      const double c = rank[u] / (double)deg;                          /* c_t[u] */
      for (uint64_t e = row_off[u]; e < row_off[u + 1]; ++e) acc[col[e]] += c;
    }
    for (uint64_t v = 0; v < V; ++v) rank[v] = base + d * acc[v];    /* r_{t+1} */
  }
  free(acc);
  return OK;
}

int oracle_bc(uint64_t V, const uint64_t* row_off, const uint32_t* col, const uint64_t* sources,
              int k, double* bc) {
  if (!bc || !row_off || k < 0 || (k && !sources)) return EINVAL_;
  for (int i = 0; i < k; ++i)
    if (sources[i] >= V) return EINVAL_;
  uint32_t* order = (uint32_t*)malloc((V ? V : 1) * sizeof(uint32_t)); /* BFS order = stack */
  int64_t* dist = (int64_t*)malloc((V ? V : 1) * sizeof(int64_t));
  double* sigma = (double*)malloc((V ? V : 1) * sizeof(double));
  double* delta = (double*)malloc((V ? V : 1) * sizeof(double));
  if (!order || !dist || !sigma || !delta) {
    free(order); free(dist); free(sigma); free(delta);
    return ENOMEM_;
  }
  for (uint64_t v = 0; v < V; ++v) bc[v] = 0.0;
  for (int i = 0; i < k; ++i) {
    const uint64_t s = sources[i];
    for (uint64_t v = 0; v < V; ++v) { dist[v] = -1; sigma[v] = 0.0; delta[v] = 0.0; }
    uint64_t head = 0, tail = 0;
    dist[s] = 0; sigma[s] = 1.0; order[tail++] = (uint32_t)s;
    while (head < tail) {                                   /* forward: BFS + sigma */
      const uint32_t v = order[head++];
      for (uint64_t e = row_off[v]; e < row_off[v + 1]; ++e) {
        const uint32_t w = col[e];
        if (dist[w] < 0) { dist[w] = dist[v] + 1; order[tail++] = w; }
        if (dist[w] == dist[v] + 1) sigma[w] += sigma[v];  /* one term per edge */
      }
    }
    for (uint64_t j = tail; j-- > 0;) {                     /* backward: reverse BFS order */
      const uint32_t v = order[j];
      double dv = 0.0;
      for (uint64_t e = row_off[v]; e < row_off[v + 1]; ++e) {
        const uint32_t w = col[e];
        if (dist[w] == dist[v] + 1) dv += sigma[v] / sigma[w] * (1.0 + delta[w]);
      }
      delta[v] = dv;
      if (v != s) bc[v] += dv;
    }
  }
  free(order); free(dist); free(sigma); free(delta);
  return OK;
}

/* ---- connected components: union-find (oracle.h) ---- */
static uint32_t uf_find(uint32_t* parent, uint32_t x) {
  while (parent[x] != x) {
    parent[x] = parent[parent[x]];  /* path halving */
    x = parent[x];
  }
  return x;
}

static void uf_union(uint32_t* parent, uint32_t a, uint32_t b) {
  a = uf_find(parent, a);
  b = uf_find(parent, b);
  if (a == b) return;
  /* the smaller id becomes the root, so every root is the minimum of its set */
  if (a < b) parent[b] = a;
  else parent[a] = b;
}

int oracle_cc_edges(uint64_t V, uint32_t* parent, uint64_t n, const uint32_t* src,
                    const uint32_t* dst) {
  if (!parent || (n && (!src || !dst))) return EINVAL_;
  for (uint64_t k = 0; k < n; ++k) {
    if (src[k] >= V || dst[k] >= V) return EINVAL_;
    uf_union(parent, src[k], dst[k]);
  }
  return OK;
}

int oracle_cc_finish(uint64_t V, uint32_t* parent, uint32_t* label) {
  if (!parent || !label) return EINVAL_;
  for (uint64_t v = 0; v < V; ++v) label[v] = uf_find(parent, (uint32_t)v);
  return OK;
}

int oracle_cc(uint64_t V, const uint64_t* row_off, const uint32_t* col, uint32_t* label) {
  if (!row_off || !label) return EINVAL_;
  uint32_t* parent = (uint32_t*)malloc((V ? V : 1) * sizeof(uint32_t));
  if (!parent) return ENOMEM_;
  for (uint64_t v = 0; v < V; ++v) parent[v] = (uint32_t)v;
  for (uint64_t u = 0; u < V; ++u)
    for (uint64_t e = row_off[u]; e < row_off[u + 1]; ++e) uf_union(parent, (uint32_t)u, col[e]);
  const int rc = oracle_cc_finish(V, parent, label);
  free(parent);
  return rc;
}

/* qsort comparator context: (degree desc, id asc) */
static const uint64_t* g_cmp_row_off;
static int cmp_deg_desc(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  const uint64_t dx = g_cmp_row_off[x + 1] - g_cmp_row_off[x];
  const uint64_t dy = g_cmp_row_off[y + 1] - g_cmp_row_off[y];
  if (dx != dy) return dx > dy ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int oracle_partition(uint64_t V, const uint64_t* row_off, int P, uint32_t* part, uint32_t* local) {
  if (P < 1 || !row_off || (V && (!part || !local))) return EINVAL_;
  uint32_t* order = (uint32_t*)malloc((V ? V : 1) * sizeof(uint32_t));
  if (!order) return ENOMEM_;
  for (uint64_t v = 0; v < V; ++v) order[v] = (uint32_t)v;
  g_cmp_row_off = row_off;
  qsort(order, V, sizeof(uint32_t), cmp_deg_desc);
  for (uint64_t i = 0; i < V; ++i) {
    const uint64_t r = i / (uint64_t)P, j = i % (uint64_t)P;
    part[order[i]] = (uint32_t)((r % 2 == 0) ? j : (uint64_t)P - 1 - j);
    local[order[i]] = (uint32_t)r;
  }
  free(order);
  return OK;
}

static const uint32_t* g_cmp_key;
static int cmp_key_asc(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  if (g_cmp_key[x] != g_cmp_key[y]) return g_cmp_key[x] < g_cmp_key[y] ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int oracle_partition_random(uint64_t V, const uint64_t* row_off, int P, const uint32_t* key,
                            uint32_t* part, uint32_t* local) {
  if (P < 1 || !row_off || (V && (!part || !local || !key))) return EINVAL_;
  uint32_t* order = (uint32_t*)malloc((V ? V : 1) * sizeof(uint32_t));
  uint64_t* next = (uint64_t*)calloc((size_t)P, sizeof(uint64_t));
  if (!order || !next) { free(order); free(next); return ENOMEM_; }
  /* 1. partition = serpentine deal of the position in (key, id) order */
  for (uint64_t v = 0; v < V; ++v) order[v] = (uint32_t)v;
  g_cmp_key = key;
  qsort(order, V, sizeof(uint32_t), cmp_key_asc);
  for (uint64_t i = 0; i < V; ++i) {
    const uint64_t r = i / (uint64_t)P, j = i % (uint64_t)P;
    part[order[i]] = (uint32_t)((r % 2 == 0) ? j : (uint64_t)P - 1 - j);
  }
  /* 2. local ids: out-degree desc, id asc, counted per partition */
  for (uint64_t v = 0; v < V; ++v) order[v] = (uint32_t)v;
  g_cmp_row_off = row_off;
  qsort(order, V, sizeof(uint32_t), cmp_deg_desc);
  for (uint64_t i = 0; i < V; ++i) local[order[i]] = (uint32_t)next[part[order[i]]]++;
  free(order);
  free(next);
  return OK;
}

int oracle_beta(uint64_t V, uint64_t E, const uint32_t* src, const uint32_t* dst,
                const uint32_t* part, int P, double* beta_raw, double* beta_reduced,
                uint64_t* slots) {
  if (P < 1 || !part || (E && (!src || !dst))) return EINVAL_;
  const uint64_t words = (V + 63) / 64;
  uint64_t* seen = (uint64_t*)calloc((words ? words : 1) * (uint64_t)P, sizeof(uint64_t));
  if (!seen) return ENOMEM_;
  uint64_t cross = 0, distinct = 0;
  if (slots) memset(slots, 0, (size_t)P * P * sizeof(uint64_t));
  for (uint64_t e = 0; e < E; ++e) {
    const uint32_t p = part[src[e]], q = part[dst[e]];
    if (p == q) continue;
    cross++;
    uint64_t* bm = seen + (uint64_t)p * words;
    const uint64_t bit = 1ULL << (dst[e] & 63);
    if (!(bm[dst[e] >> 6] & bit)) {
      bm[dst[e] >> 6] |= bit;
      distinct++;
      if (slots) slots[(uint64_t)p * P + q]++;
    }
  }
  free(seen);
  if (beta_raw) *beta_raw = E ? (double)cross / (double)E : 0.0;
  if (beta_reduced) *beta_reduced = E ? (double)distinct / (double)E : 0.0;
  return OK;
}

int oracle_bfs_certify(uint64_t V, const uint64_t* row_off, const uint32_t* col, uint64_t s,
                       const uint32_t* level, uint64_t* bad) {
  if (s >= V || !level) return EINVAL_;
  uint64_t b = ~0ULL;
  uint8_t* tight = (uint8_t*)calloc(V, 1);
  if (!tight) return ENOMEM_;
  int rc = OK;
  if (level[s] != 0) { rc = 1; b = s; }
  for (uint64_t u = 0; u < V && rc == OK; ++u) {
    if (level[u] == ORACLE_INF32) continue;
    for (uint64_t e = row_off[u]; e < row_off[u + 1]; ++e) {
      const uint32_t v = col[e];
      if (level[v] == ORACLE_INF32 || (uint64_t)level[v] > (uint64_t)level[u] + 1) {
        rc = 1; b = v; break;
      }
      if ((uint64_t)level[v] == (uint64_t)level[u] + 1) tight[v] = 1;
    }
  }
  for (uint64_t v = 0; v < V && rc == OK; ++v)
    if (v != s && level[v] != ORACLE_INF32 && !tight[v]) { rc = 1; b = v; }
  free(tight);
  if (bad) *bad = b;
  return rc;
}

int oracle_sssp_certify(uint64_t V, const uint64_t* row_off, const uint32_t* col,
                        const uint32_t* w, uint64_t s, const uint32_t* dist, uint64_t* bad) {
  if (s >= V || !dist || !w) return EINVAL_;
  uint64_t b = ~0ULL;
  uint8_t* tight = (uint8_t*)calloc(V, 1);
  if (!tight) return ENOMEM_;
  int rc = OK;
  if (dist[s] != 0) { rc = 1; b = s; }
  for (uint64_t u = 0; u < V && rc == OK; ++u) {
    if (dist[u] == ORACLE_INF32) continue;
    for (uint64_t e = row_off[u]; e < row_off[u + 1]; ++e) {
      const uint32_t v = col[e];
      const uint64_t nd = (uint64_t)dist[u] + w[e];
      if (dist[v] == ORACLE_INF32 || nd < (uint64_t)dist[v]) { rc = 1; b = v; break; }
      if (nd == (uint64_t)dist[v]) tight[v] = 1;
    }
  }
  for (uint64_t v = 0; v < V && rc == OK; ++v)
    if (v != s && dist[v] != ORACLE_INF32 && !tight[v]) { rc = 1; b = v; }
  free(tight);
  if (bad) *bad = b;
  return rc;
}

/* ---- streaming certificates (see oracle.h) ---- */
int oracle_outdeg_edges(uint64_t V, uint64_t n, const uint32_t* src, uint32_t* outdeg) {
  if (!outdeg || (n && !src)) return EINVAL_;
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)n; ++i) {
    if (src[i] < V) __atomic_fetch_add(&outdeg[src[i]], 1u, __ATOMIC_RELAXED);
  }
  return OK;
}

int oracle_bfs_cert_edges(uint64_t V, const uint32_t* level, uint64_t n, const uint32_t* src,
                          const uint32_t* dst, uint64_t* tight, uint64_t* bad) {
  if (!level || !tight || !bad || (n && (!src || !dst))) return EINVAL_;
  unsigned long long nbad = 0;
#pragma omp parallel for schedule(static) reduction(+ : nbad)
  for (long long i = 0; i < (long long)n; ++i) {
    const uint32_t u = src[i], v = dst[i];
    if (u >= V || v >= V) { nbad++; continue; }
    if (level[u] == ORACLE_INF32) continue;
    const uint64_t lu = level[u], lv = level[v];
    if (level[v] == ORACLE_INF32 || lv > lu + 1) { nbad++; continue; }
    if (lv == lu + 1) __atomic_fetch_or(&tight[v >> 6], 1ULL << (v & 63), __ATOMIC_RELAXED);
  }
  *bad += nbad;
  return OK;
}

int oracle_sssp_cert_edges(uint64_t V, const uint32_t* dist, uint64_t n, const uint32_t* src,
                           const uint32_t* dst, const uint32_t* w, uint64_t* tight, uint64_t* bad) {
  if (!dist || !tight || !bad || (n && (!src || !dst || !w))) return EINVAL_;
  unsigned long long nbad = 0;
#pragma omp parallel for schedule(static) reduction(+ : nbad)
  for (long long i = 0; i < (long long)n; ++i) {
    const uint32_t u = src[i], v = dst[i];
    if (u >= V || v >= V) { nbad++; continue; }
    if (dist[u] == ORACLE_INF32) continue;
    const uint64_t nd = (uint64_t)dist[u] + w[i];
    if (dist[v] == ORACLE_INF32 || nd < (uint64_t)dist[v]) { nbad++; continue; }
    if (nd == (uint64_t)dist[v]) __atomic_fetch_or(&tight[v >> 6], 1ULL << (v & 63), __ATOMIC_RELAXED);
  }
  *bad += nbad;
  return OK;
}

int oracle_cert_finish(uint64_t V, uint64_t s, const uint32_t* val, const uint64_t* tight,
                       uint64_t* bad) {
  if (s >= V || !val || !tight) return EINVAL_;
  if (val[s] != 0) { if (bad) *bad = s; return 1; }
  for (uint64_t v = 0; v < V; ++v) {
    if (v == s || val[v] == ORACLE_INF32) continue;
    if (!((tight[v >> 6] >> (v & 63)) & 1ULL)) { if (bad) *bad = v; return 1; }
  }
  return OK;
}

int oracle_pr_sample_edges(uint64_t V, uint64_t n, const uint32_t* src, const uint32_t* dst,
                           const uint64_t* mask, const uint32_t* slot, const float* r_prev,
                           const uint32_t* outdeg, double* acc) {
  if (!mask || !slot || !r_prev || !outdeg || !acc || (n && (!src || !dst))) return EINVAL_;
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)n; ++i) {
    const uint32_t u = src[i], v = dst[i];
    if (u >= V || v >= V || !((mask[v >> 6] >> (v & 63)) & 1ULL)) continue;
    const double c = (double)r_prev[u] / (double)outdeg[u];   /* outdeg[u] >= 1: u has this edge */
#pragma omp atomic
    acc[slot[v]] += c;
  }
  return OK;
}
