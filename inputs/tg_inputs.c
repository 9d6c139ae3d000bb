/*
 * tg_inputs.c -- host entry points of the seeded input generators
 * (libtginputs.so).  Used by tests/, the oracle harness and bench.py to
 * materialise the synthetic workload on the host.  No method arithmetic here;
 * see tg_inputs.h for the workload definition.
 */
#include "tg_inputs.h"

#include <stddef.h>

#define TGIN_OK 0
#define TGIN_EINVAL 2

/* Edges [first, first+count) of RMAT(scale, edge_factor, a, b, c, seed).
 * src/dst: caller-owned arrays of length count; w (nullable) receives the
 * SSSP weight of each edge drawn from wseed.  Returns 2 on bad parameters. */
int tgin_rmat_edges(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                    int scramble, uint64_t wseed, uint64_t first, uint64_t count, uint32_t* src,
                    uint32_t* dst, uint32_t* w) {
  if (scale < 1 || scale > 32 || edge_factor < 1) return TGIN_EINVAL;
  if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0 + 1e-12) return TGIN_EINVAL;
  if (count && (!src || !dst)) return TGIN_EINVAL;
  const tgin_rmat g = tgin_make_rmat(scale, a, b, c, seed, scramble);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)count; ++i) {
    const uint64_t k = first + (uint64_t)i;
    tgin_rmat_edge_g(&g, k, &src[i], &dst[i]);
    if (w) w[i] = tgin_weight(wseed, k);
  }
  return TGIN_OK;
}

/* Weights only, for edge lists that did not come from the generator. */
int tgin_weights(uint64_t wseed, uint64_t first, uint64_t count, uint32_t* w) {
  if (count && !w) return TGIN_EINVAL;
  for (uint64_t i = 0; i < count; ++i) w[i] = tgin_weight(wseed, first + i);
  return TGIN_OK;
}

/* k run sources for an RMAT graph: src endpoint of edge tgin_source_edge(sseed, j, E). */
int tgin_rmat_sources(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                      int scramble, uint64_t sseed, uint64_t k, uint64_t* out) {
  if (scale < 1 || scale > 32 || edge_factor < 1 || (k && !out)) return TGIN_EINVAL;
  const tgin_thresholds t = tgin_make_thresholds(a, b, c);
  const uint64_t E = (uint64_t)edge_factor << scale;
  for (uint64_t j = 0; j < k; ++j) {
    uint32_t s, d;
    tgin_rmat_edge(scale, t, seed, scramble, tgin_source_edge(sseed, j, E), &s, &d);
    out[j] = s;
  }
  return TGIN_OK;
}

/* k run sources for an explicit edge list (src endpoint of a seeded edge). */
int tgin_list_sources(uint64_t E, const uint32_t* src, uint64_t sseed, uint64_t k, uint64_t* out) {
  if (E == 0 || !src || (k && !out)) return TGIN_EINVAL;
  for (uint64_t j = 0; j < k; ++j) out[j] = src[tgin_source_edge(sseed, j, E)];
  return TGIN_OK;
}

uint32_t tgin_scramble_one(uint32_t x, int scale, uint64_t seed) {
  return tgin_scramble(x, scale, seed);
}

/* Keys of the TG_PART_RANDOM partitioning draw for vertices [0, V). */
int tgin_part_keys(uint64_t pseed, uint64_t V, uint32_t* out) {
  if (V && !out) return TGIN_EINVAL;
  for (uint64_t v = 0; v < V; ++v) out[v] = tgin_part_key(pseed, v);
  return TGIN_OK;
}
