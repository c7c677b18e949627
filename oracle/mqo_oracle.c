/*
 * mqo_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU oracle of the B200 mQO
 * path.  A plain-C restatement of the reference algorithm, function by
 * function, each citing the reference file:line it follows (paths relative
 * to /root/reference/proj/core/).  It is the checker for tests/, smoke()
 * and bench.py's cpu_baseline leg; the product never links it.
 *
 * Pinned against (a) the reference's own KATs re-hosted in
 * tests/test_oracle_*.py, (b) golden vectors produced by the compiled
 * reference (oracle/_ref, tests/golden/make_golden.py) and (c) direct
 * side-by-side runs against oracle/_ref/libref.so when it is present.
 *
 * Build: -O2 -ffp-contract=off, no -mfma (FMA contraction changes integer
 * outcomes).  Box-Muller uses this host's libm
 * log/sin/cos, exactly like the reference.
 */
#define _POSIX_C_SOURCE 200809L
#include "mqo_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ errors */

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }
const char* orc_impl_name(void) { return "oracle-c"; }

static void* xmalloc(size_t bytes) {
  void* p = malloc(bytes ? bytes : 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory (%zu bytes)\n", bytes);
    abort();
  }
  return p;
}
static void* xcalloc(size_t count, size_t size) {
  void* p = calloc(count ? count : 1, size ? size : 1);
  if (!p) abort();
  return p;
}

/* --------------------------------------------------------------------- RNG */
/* rng.hpp:13-86: xoshiro256** with splitmix64 seeding, Box-Muller spare. */

typedef struct {
  uint64_t s[4];
  double spare;
  int has_spare;
} rng_t;

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t splitmix64(uint64_t* s) { /* rng.hpp:71-76 */
  uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static void rng_seed(rng_t* r, uint64_t seed) { /* rng.hpp:15-18 */
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&s);
  r->spare = 0.0;
  r->has_spare = 0;
}

static uint64_t rng_next(rng_t* r) { /* rng.hpp:20-30 */
  uint64_t* st = r->s;
  const uint64_t result = rotl64(st[1] * 5, 7) * 9;
  const uint64_t t = st[1] << 17;
  st[2] ^= st[0];
  st[3] ^= st[1];
  st[1] ^= st[2];
  st[0] ^= st[3];
  st[2] ^= t;
  st[3] = rotl64(st[3], 45);
  return result;
}

static double rng_u01(rng_t* r) { /* rng.hpp:33 */
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}

static uint64_t rng_index(rng_t* r, uint64_t n) { /* rng.hpp:40-46 */
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t x = rng_next(r);
    if (x >= threshold) return x % n;
  }
}

static double rng_normal(rng_t* r, double mean, double sd) { /* rng.hpp:49-62 */
  if (r->has_spare) {
    r->has_spare = 0;
    return mean + sd * r->spare;
  }
  double u1 = rng_u01(r);
  double u2 = rng_u01(r);
  while (u1 <= 0.0) u1 = rng_u01(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.141592653589793 * u2; /* std::numbers::pi */
  r->spare = rad * sin(theta);
  r->has_spare = 1;
  return mean + sd * rad * cos(theta);
}

uint64_t orc_derive_seed(uint64_t master, uint64_t stream) { /* rng.hpp:80-86 */
  uint64_t s = master ^ (0x9e3779b97f4a7c15ULL + stream * 0xd1342543de82ef95ULL);
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void* orc_rng_new(uint64_t seed) {
  rng_t* r = (rng_t*)xmalloc(sizeof *r);
  rng_seed(r, seed);
  return r;
}
void orc_rng_free(void* r) { free(r); }
uint64_t orc_rng_next_u64(void* r) { return rng_next((rng_t*)r); }
double orc_rng_uniform01(void* r) { return rng_u01((rng_t*)r); }
uint64_t orc_rng_uniform_index(void* r, uint64_t n) { return rng_index((rng_t*)r, n); }
double orc_rng_normal(void* r, double mean, double sd) {
  return rng_normal((rng_t*)r, mean, sd);
}

/* ------------------------------------------------------------------- Graph */
/* graph.hpp:20-63, graph.cpp:8-56: immutable CSR, rows strictly ascending. */

typedef struct {
  int32_t n;
  int64_t m;
  int32_t max_degree;
  int64_t* off; /* n+1 */
  int32_t* nbr; /* 2m */
} graph_t;

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}
static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : x > y;
}

static inline int32_t deg(const graph_t* g, int32_t v) {
  return (int32_t)(g->off[v + 1] - g->off[v]);
}

/* graph.cpp:8-42.  Edge pairs are normalised to u < v, sorted, deduped,
 * counted, prefix-summed, filled and each row sorted. Keys pack (u, v) so
 * the u64 order equals the std::pair order. */
static int graph_build(int32_t n, int64_t ne, uint64_t* keys /* owned */, graph_t** out) {
  if (n < 0) {
    free(keys);
    return fail(ORC_INVALID, "graph: negative vertex count");
  }
  qsort(keys, (size_t)ne, sizeof(uint64_t), cmp_u64);
  int64_t m = 0;
  for (int64_t i = 0; i < ne; ++i)
    if (i == 0 || keys[i] != keys[i - 1]) keys[m++] = keys[i];

  graph_t* g = (graph_t*)xcalloc(1, sizeof *g);
  g->n = n;
  g->m = m;
  g->off = (int64_t*)xcalloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t i = 0; i < m; ++i) {
    const int32_t u = (int32_t)(keys[i] >> 32), v = (int32_t)(keys[i] & 0xffffffffu);
    ++g->off[u + 1];
    ++g->off[v + 1];
  }
  for (int32_t v = 0; v < n; ++v) g->off[v + 1] += g->off[v];
  g->nbr = (int32_t*)xmalloc((size_t)(2 * m) * sizeof(int32_t));
  int64_t* cursor = (int64_t*)xmalloc((size_t)(n + 1) * sizeof(int64_t));
  memcpy(cursor, g->off, (size_t)n * sizeof(int64_t));
  for (int64_t i = 0; i < m; ++i) {
    const int32_t u = (int32_t)(keys[i] >> 32), v = (int32_t)(keys[i] & 0xffffffffu);
    g->nbr[cursor[u]++] = v;
    g->nbr[cursor[v]++] = u;
  }
  free(cursor);
  free(keys);
  for (int32_t v = 0; v < n; ++v)
    qsort(g->nbr + g->off[v], (size_t)deg(g, v), sizeof(int32_t), cmp_i32);
  g->max_degree = 0;
  for (int32_t v = 0; v < n; ++v)
    if (deg(g, v) > g->max_degree) g->max_degree = deg(g, v);
  /* check_invariants, graph.cpp:44-56 */
  int64_t degree_sum = 0;
  for (int32_t v = 0; v < n; ++v) {
    degree_sum += deg(g, v);
    for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
      if (g->nbr[e] == v) return fail(ORC_LOGIC, "graph: self-loop");
      if (e > g->off[v] && g->nbr[e - 1] >= g->nbr[e])
        return fail(ORC_LOGIC, "graph: neighbor list not strictly ascending");
    }
  }
  if (degree_sum != 2 * m) return fail(ORC_LOGIC, "graph: degree sum != 2m");
  *out = g;
  return ORC_OK;
}

int orc_graph_from_edges(int32_t n, int64_t ne, const int32_t* eu, const int32_t* ev,
                         void** out) {
  if (n < 0) return fail(ORC_INVALID, "graph: negative vertex count");
  uint64_t* keys = (uint64_t*)xmalloc((size_t)ne * sizeof(uint64_t));
  for (int64_t i = 0; i < ne; ++i) {
    int32_t u = eu[i], v = ev[i];
    if (u < 0 || u >= n || v < 0 || v >= n) {
      free(keys);
      return fail(ORC_INVALID, "graph: vertex index out of range");
    }
    if (u == v) {
      free(keys);
      return fail(ORC_INVALID, "graph: self-loop rejected");
    }
    if (u > v) {
      const int32_t t = u;
      u = v;
      v = t;
    }
    keys[i] = ((uint64_t)(uint32_t)u << 32) | (uint32_t)v;
  }
  return graph_build(n, ne, keys, (graph_t**)out);
}

/* Test helper (not a reference function): wraps a CSR that is already in
 * Graph's canonical form -- e.g. the device's O(m) ER generator output for
 * C5, where re-sorting 8e7 edge pairs per test would dominate -- after the
 * same invariant checks as Graph::check_invariants (graph.cpp:44-56) plus
 * symmetry.  Reference-side equivalent: Graph::from_edges on the edge list. */
int orc_graph_from_csr(int32_t n, const int64_t* off, const int32_t* nbr, void** out) {
  if (n < 0) return fail(ORC_INVALID, "graph: negative vertex count");
  graph_t* g = (graph_t*)xcalloc(1, sizeof *g);
  g->n = n;
  g->m = off[n] / 2;
  g->off = (int64_t*)xmalloc(((size_t)n + 1) * sizeof(int64_t));
  memcpy(g->off, off, ((size_t)n + 1) * sizeof(int64_t));
  g->nbr = (int32_t*)xmalloc((size_t)off[n] * sizeof(int32_t) + 1);
  memcpy(g->nbr, nbr, (size_t)off[n] * sizeof(int32_t));
  g->max_degree = 0;
  for (int32_t v = 0; v < n; ++v) {
    if (deg(g, v) > g->max_degree) g->max_degree = deg(g, v);
    for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
      const int32_t u = g->nbr[e];
      if (u < 0 || u >= n || u == v) return fail(ORC_LOGIC, "graph: bad neighbour");
      if (e > g->off[v] && g->nbr[e - 1] >= u)
        return fail(ORC_LOGIC, "graph: neighbor list not strictly ascending");
      /* symmetry: v must appear in row u */
      int64_t lo = g->off[u], hi = g->off[u + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (g->nbr[mid] < v) lo = mid + 1; else hi = mid;
      }
      if (lo == g->off[u + 1] || g->nbr[lo] != v) return fail(ORC_LOGIC, "graph: not symmetric");
    }
  }
  if (off[n] % 2) return fail(ORC_LOGIC, "graph: degree sum != 2m");
  *out = g;
  return ORC_OK;
}

/* growable u64 key list for the generators */
typedef struct {
  uint64_t* k;
  int64_t len, cap;
} keyvec;
static void kv_push(keyvec* kv, int32_t u, int32_t v) {
  if (u > v) {
    const int32_t t = u;
    u = v;
    v = t;
  }
  if (kv->len == kv->cap) {
    kv->cap = kv->cap ? 2 * kv->cap : 1024;
    kv->k = (uint64_t*)realloc(kv->k, (size_t)kv->cap * sizeof(uint64_t));
    if (!kv->k) abort();
  }
  kv->k[kv->len++] = ((uint64_t)(uint32_t)u << 32) | (uint32_t)v;
}

int orc_generate_er(int32_t n, double p, uint64_t seed, void** out) { /* graph.cpp:107-116 */
  if (n < 0) return fail(ORC_INVALID, "er: negative n");
  if (p < 0.0 || p > 1.0) return fail(ORC_INVALID, "er: p outside [0,1]");
  rng_t r;
  rng_seed(&r, orc_derive_seed(seed, 0x45521ULL));
  keyvec kv = {0, 0, 0};
  for (int32_t u = 0; u < n; ++u)
    for (int32_t v = u + 1; v < n; ++v)
      if (rng_u01(&r) < p) kv_push(&kv, u, v);
  return graph_build(n, kv.len, kv.k, (graph_t**)out);
}

int orc_generate_ba(int32_t n, int32_t m_attach, uint64_t seed, void** out) {
  /* graph.cpp:118-146 */
  if (m_attach < 1) return fail(ORC_INVALID, "ba: m_attach must be >= 1");
  if (m_attach >= n) return fail(ORC_INVALID, "ba: m_attach must be < n");
  rng_t r;
  rng_seed(&r, orc_derive_seed(seed, 0xBAULL));
  keyvec kv = {0, 0, 0};
  const int64_t cap = 2 * (int64_t)m_attach * n + 2;
  int32_t* endpoints = (int32_t*)xmalloc((size_t)cap * sizeof(int32_t));
  int64_t ne = 0;
  for (int32_t v = 1; v <= m_attach; ++v) {
    kv_push(&kv, 0, v);
    endpoints[ne++] = 0;
    endpoints[ne++] = v;
  }
  int32_t* targets = (int32_t*)xmalloc((size_t)m_attach * sizeof(int32_t));
  for (int32_t v = m_attach + 1; v < n; ++v) {
    int32_t nt = 0;
    while (nt < m_attach) {
      const int32_t t = endpoints[rng_index(&r, (uint64_t)ne)];
      int dup = 0;
      for (int32_t i = 0; i < nt; ++i)
        if (targets[i] == t) dup = 1;
      if (!dup) targets[nt++] = t;
    }
    for (int32_t i = 0; i < nt; ++i) {
      kv_push(&kv, targets[i], v);
      endpoints[ne++] = targets[i];
      endpoints[ne++] = v;
    }
  }
  free(targets);
  free(endpoints);
  return graph_build(n, kv.len, kv.k, (graph_t**)out);
}

int orc_generate_sbm(int32_t n, int32_t k, double p_in, double p_out, uint64_t seed,
                     void** out) { /* graph.cpp:148-165 */
  if (k < 1) return fail(ORC_INVALID, "sbm: k must be >= 1");
  if (p_in < 0.0 || p_in > 1.0 || p_out < 0.0 || p_out > 1.0)
    return fail(ORC_INVALID, "sbm: probabilities outside [0,1]");
  if (p_in <= p_out) return fail(ORC_INVALID, "sbm: requires p_in > p_out");
  rng_t r;
  rng_seed(&r, orc_derive_seed(seed, 0x5B3ULL));
  keyvec kv = {0, 0, 0};
  for (int32_t u = 0; u < n; ++u)
    for (int32_t v = u + 1; v < n; ++v) {
      const int bu = (int)(((int64_t)u * k) / n), bv = (int)(((int64_t)v * k) / n);
      if (rng_u01(&r) < (bu == bv ? p_in : p_out)) kv_push(&kv, u, v);
    }
  return graph_build(n, kv.len, kv.k, (graph_t**)out);
}

void orc_graph_free(void* gp) {
  graph_t* g = (graph_t*)gp;
  if (!g) return;
  free(g->off);
  free(g->nbr);
  free(g);
}

void orc_graph_info(void* gp, int32_t* n, int64_t* m, int32_t* max_degree) {
  const graph_t* g = (const graph_t*)gp;
  *n = g->n;
  *m = g->m;
  *max_degree = g->max_degree;
}

void orc_graph_csr(void* gp, int64_t* offsets, int32_t* nbrs) {
  const graph_t* g = (const graph_t*)gp;
  memcpy(offsets, g->off, (size_t)(g->n + 1) * sizeof(int64_t));
  memcpy(nbrs, g->nbr, (size_t)(2 * g->m) * sizeof(int32_t));
}

/* strip_isolated (graph.cpp:180-198): degree-0 vertices removed in index
 * order; the core is rebuilt from the relabelled edges (v < u). */
int orc_strip_isolated(void* gp, void** core, int32_t* core_to_orig, int32_t* orig_to_core,
                       int32_t* removed, int32_t* n_core, int32_t* n_removed) {
  const graph_t* g = (const graph_t*)gp;
  int32_t nc = 0, nr = 0;
  for (int32_t v = 0; v < g->n; ++v) {
    if (deg(g, v) == 0) {
      orig_to_core[v] = -1;
      removed[nr++] = v;
    } else {
      orig_to_core[v] = nc;
      core_to_orig[nc++] = v;
    }
  }
  uint64_t* keys = (uint64_t*)xmalloc((size_t)(g->m > 0 ? g->m : 1) * sizeof(uint64_t));
  int64_t k = 0;
  for (int32_t v = 0; v < g->n; ++v)
    for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e)
      if (v < g->nbr[e])
        keys[k++] = ((uint64_t)(uint32_t)orig_to_core[v] << 32) | (uint32_t)orig_to_core[g->nbr[e]];
  *n_core = nc;
  *n_removed = nr;
  return graph_build(nc, k, keys, (graph_t**)core);
}

/* connected_components (graph.cpp:200-224): DFS from each unseen vertex in
 * index order; comp[v] = index of v's component (output order). */
int orc_components(void* gp, int32_t* comp, int32_t* count) {
  const graph_t* g = (const graph_t*)gp;
  int32_t* stack = (int32_t*)xmalloc((size_t)(g->n > 0 ? g->n : 1) * sizeof(int32_t));
  for (int32_t v = 0; v < g->n; ++v) comp[v] = -1;
  int32_t c = 0;
  for (int32_t s = 0; s < g->n; ++s) {
    if (comp[s] >= 0) continue;
    int32_t top = 0;
    comp[s] = c;
    stack[top++] = s;
    while (top > 0) {
      const int32_t v = stack[--top];
      for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
        const int32_t u = g->nbr[e];
        if (comp[u] < 0) {
          comp[u] = c;
          stack[top++] = u;
        }
      }
    }
    ++c;
  }
  free(stack);
  *count = c;
  return ORC_OK;
}

static int has_edge(const graph_t* g, int32_t u, int32_t v) { /* graph.cpp:58-61 */
  int64_t lo = g->off[u], hi = g->off[u + 1];
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (g->nbr[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < g->off[u + 1] && g->nbr[lo] == v;
}

static void adj_apply(const graph_t* g, const double* x, double* y) { /* graph.cpp:63-71 */
  for (int32_t v = 0; v < g->n; ++v) {
    double acc = 0.0;
    for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) acc += x[g->nbr[e]];
    y[v] = acc;
  }
}

static void lap_apply(const graph_t* g, const double* x, double* y) { /* graph.cpp:79-88 */
  for (int32_t v = 0; v < g->n; ++v) {
    double acc = 0.0;
    const double xv = x[v];
    for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) acc += xv - x[g->nbr[e]];
    y[v] = acc;
  }
}

int orc_adjacency_apply(void* g, const double* x, double* y) {
  adj_apply((const graph_t*)g, x, y);
  return ORC_OK;
}
int orc_laplacian_apply(void* g, const double* x, double* y) {
  lap_apply((const graph_t*)g, x, y);
  return ORC_OK;
}

/* -------------------------------------------------------------- Objectives */

static int problem_of(int32_t kind) { /* objectives.cpp:8-10 */
  return kind == ORC_MIS_QUBO ? ORC_PROBLEM_MIS : ORC_PROBLEM_MAXCUT;
}

int orc_validate_objective(int32_t kind, double param) { /* objectives.cpp:27-38 */
  if (kind < 0 || kind > 4) return fail(ORC_INVALID, "objective: unknown kind");
  if (kind == ORC_MIS_QUBO && !(param > 1.0))
    return fail(ORC_INVALID, "mis-qubo: gamma must be > 1");
  if (kind == ORC_PERTURBED_LAPLACIAN && !(param > 0.0))
    return fail(ORC_INVALID, "perturbed-laplacian: lambda must be > 0");
  if (kind == ORC_PERTURBED_BIAS && !(param > 0.0 && param < 2.0))
    return fail(ORC_INVALID, "perturbed-bias: lambda must be in (0, 2)");
  return ORC_OK;
}

static void gradient(const graph_t* g, int32_t kind, double param, const double* x,
                     double* out) { /* objectives.cpp:101-134 */
  const int32_t n = g->n;
  if (kind == ORC_MIS_QUBO) {
    adj_apply(g, x, out);
    for (int32_t v = 0; v < n; ++v) out[v] = 1.0 - param * out[v];
  } else if (kind == ORC_LAPLACIAN) {
    lap_apply(g, x, out);
    for (int32_t v = 0; v < n; ++v) out[v] *= 0.5;
  } else if (kind == ORC_PERTURBED_LAPLACIAN) {
    adj_apply(g, x, out);
    for (int32_t v = 0; v < n; ++v)
      out[v] = 2.0 * ((double)deg(g, v) * x[v] - out[v] + param * x[v]);
  } else if (kind == ORC_ADJACENCY) {
    adj_apply(g, x, out);
    for (int32_t v = 0; v < n; ++v) out[v] *= -2.0;
  } else {
    adj_apply(g, x, out);
    for (int32_t v = 0; v < n; ++v) out[v] = -2.0 * out[v] - param;
  }
}

int orc_gradient(void* g, int32_t kind, double param, const double* x, double* out) {
  gradient((const graph_t*)g, kind, param, x, out);
  return ORC_OK;
}

static double quad_adjacency(const graph_t* g, const double* x) { /* objectives.cpp:61-66 */
  double* s = (double*)xmalloc((size_t)g->n * sizeof(double));
  adj_apply(g, x, s);
  double acc = 0.0;
  for (int32_t i = 0; i < g->n; ++i) acc += x[i] * s[i];
  free(s);
  return acc;
}

static double quad_laplacian(const graph_t* g, const double* x) { /* objectives.cpp:69-81 */
  double acc = 0.0;
  for (int32_t v = 0; v < g->n; ++v) {
    const double xv = x[v];
    for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
      const int32_t u = g->nbr[e];
      if (u > v) {
        const double d = xv - x[u];
        acc += d * d;
      }
    }
  }
  return acc;
}

int orc_value(void* gp, int32_t kind, double param, const double* x, double* out) {
  /* objectives.cpp:86-99 */
  const graph_t* g = (const graph_t*)gp;
  double sum = 0.0, dot = 0.0;
  for (int32_t i = 0; i < g->n; ++i) sum += x[i];
  for (int32_t i = 0; i < g->n; ++i) dot += x[i] * x[i];
  if (kind == ORC_MIS_QUBO)
    *out = sum - 0.5 * param * quad_adjacency(g, x);
  else if (kind == ORC_LAPLACIAN)
    *out = 0.25 * quad_laplacian(g, x);
  else if (kind == ORC_PERTURBED_LAPLACIAN)
    *out = quad_laplacian(g, x) + param * dot;
  else if (kind == ORC_ADJACENCY)
    *out = -quad_adjacency(g, x);
  else
    *out = -param * sum - quad_adjacency(g, x);
  return ORC_OK;
}

int64_t orc_cut_value(void* gp, const uint8_t* side) { /* objectives.cpp:163-171 */
  const graph_t* g = (const graph_t*)gp;
  int64_t crossing = 0;
  for (int32_t v = 0; v < g->n; ++v)
    for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
      const int32_t u = g->nbr[e];
      if (v < u && side[v] != side[u]) ++crossing;
    }
  return crossing;
}

int orc_is_independent(void* gp, const uint8_t* in) { /* objectives.cpp:173-180 */
  const graph_t* g = (const graph_t*)gp;
  for (int32_t v = 0; v < g->n; ++v) {
    if (!in[v]) continue;
    for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e)
      if (in[g->nbr[e]]) return 0;
  }
  return 1;
}

static int64_t extract(const graph_t* g, int problem, const double* x, uint8_t* body) {
  /* objectives.cpp:143-161: MIS selects x > 0.5, MaxCut side x > 0 */
  if (problem == ORC_PROBLEM_MIS) {
    int64_t size = 0;
    for (int32_t v = 0; v < g->n; ++v) {
      body[v] = x[v] > 0.5 ? 1 : 0;
      size += body[v];
    }
    return size;
  }
  for (int32_t v = 0; v < g->n; ++v) body[v] = x[v] > 0.0 ? 1 : 0;
  return orc_cut_value((void*)g, body);
}

int orc_extract_solution(void* g, int32_t problem, const double* x, uint8_t* body,
                         int64_t* score) {
  *score = extract((const graph_t*)g, problem, x, body);
  return ORC_OK;
}

/* --------------------------------------------------------------------- PGA */

int orc_validate_optimizer(double alpha, double beta, int32_t max_iters, double conv_tol,
                           int32_t check_every) { /* pga.cpp:9-18 */
  if (!(alpha > 0.0)) return fail(ORC_INVALID, "optimizer: alpha must be > 0");
  if (beta < 0.0 || beta >= 1.0) return fail(ORC_INVALID, "optimizer: beta must be in [0, 1)");
  if (max_iters < 1) return fail(ORC_INVALID, "optimizer: max_iters must be >= 1");
  if (conv_tol < 0.0) return fail(ORC_INVALID, "optimizer: conv_tol must be >= 0");
  if (check_every < 1) return fail(ORC_INVALID, "optimizer: check_every must be >= 1");
  return ORC_OK;
}

/* pga.cpp:31-34: std::min(1.0, std::max(lo, t)); std::max(a,b) = a<b?b:a,
 * std::min(a,b) = b<a?b:a -- spelled out so signed zeros and NaN follow the
 * reference exactly. */
static inline double clamp_to(int problem, double t) {
  const double lo = problem == ORC_PROBLEM_MIS ? 0.0 : -1.0;
  const double a = lo < t ? t : lo;
  return a < 1.0 ? a : 1.0;
}

void orc_project(double* x, int32_t n, int32_t problem) { /* pga.cpp:47-49 */
  for (int32_t i = 0; i < n; ++i) x[i] = clamp_to(problem, x[i]);
}

int orc_step(void* gp, int32_t kind, double param, double* x, double* v, double alpha,
             double beta) { /* pga.cpp:51-61 */
  const graph_t* g = (const graph_t*)gp;
  const int problem = problem_of(kind);
  double* grad = (double*)xmalloc((size_t)g->n * sizeof(double));
  gradient(g, kind, param, x, grad);
  for (int32_t i = 0; i < g->n; ++i) {
    v[i] = beta * v[i] + grad[i];
    x[i] = clamp_to(problem, x[i] + alpha * v[i]);
  }
  free(grad);
  return ORC_OK;
}

static int mis_fixed(const graph_t* g, const double* xb, double* scratch) {
  /* pga.cpp:113-135 (input already known binary) */
  adj_apply(g, xb, scratch);
  for (int32_t v = 0; v < g->n; ++v) {
    if (xb[v] == 1.0) {
      if (scratch[v] > 0.0) return 0;
    } else {
      if (scratch[v] < 1.0) return 0;
    }
  }
  return 1;
}

int orc_mis_fixed_point_check(void* gp, const double* x, double gamma, double alpha,
                              int32_t* fixed) {
  const graph_t* g = (const graph_t*)gp;
  if (!(gamma > 1.0)) return fail(ORC_INVALID, "mis_fixed_point_check: gamma must be > 1");
  if (!(alpha > 0.0)) return fail(ORC_INVALID, "mis_fixed_point_check: alpha must be > 0");
  for (int32_t i = 0; i < g->n; ++i)
    if (x[i] != 0.0 && x[i] != 1.0)
      return fail(ORC_INVALID, "mis_fixed_point_check: state not binary");
  double* s = (double*)xmalloc((size_t)g->n * sizeof(double));
  *fixed = mis_fixed(g, x, s);
  free(s);
  return ORC_OK;
}

static double now_secs(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* pga.cpp:63-111.  deadline < 0 means none. */
static int run_traj(const graph_t* g, int32_t kind, double param, double* x, double alpha,
                    double beta, int32_t max_iters, double conv_tol, int32_t check_every,
                    double deadline, int32_t* iterations) {
  const int problem = problem_of(kind);
  const int32_t n = g->n;
  orc_project(x, n, problem);
  double* vel = (double*)xcalloc((size_t)n, sizeof(double));
  double* grad = (double*)xmalloc((size_t)n * sizeof(double));
  double* bin = (double*)xmalloc((size_t)n * sizeof(double));
  double* scratch = (double*)xmalloc((size_t)n * sizeof(double));
  int reason = ORC_ITER_CAP;
  *iterations = 0;
  for (int32_t iter = 1; iter <= max_iters; ++iter) {
    gradient(g, kind, param, x, grad);
    double max_change = 0.0;
    for (int32_t v = 0; v < n; ++v) {
      vel[v] = beta * vel[v] + grad[v];
      const double next = clamp_to(problem, x[v] + alpha * vel[v]);
      const double d = fabs(next - x[v]);
      max_change = max_change < d ? d : max_change;
      x[v] = next;
    }
    *iterations = iter;
    if (problem == ORC_PROBLEM_MIS) {
      if (iter % check_every == 0) {
        for (int32_t v = 0; v < n; ++v) bin[v] = x[v] > 0.5 ? 1.0 : 0.0;
        if (mis_fixed(g, bin, scratch)) {
          reason = ORC_CHECKER_ACCEPTED;
          goto done;
        }
      }
    } else if (max_change <= conv_tol) {
      reason = ORC_CONVERGED;
      goto done;
    }
    if (deadline >= 0.0 && (iter & 255) == 0 && now_secs() >= deadline) break;
  }
  reason = ORC_ITER_CAP;
done:
  free(vel);
  free(grad);
  free(bin);
  free(scratch);
  return reason;
}

int orc_run_trajectory(void* gp, int32_t kind, double param, double* x, double alpha,
                       double beta, int32_t max_iters, double conv_tol,
                       int32_t check_every, int32_t* iterations, int32_t* reason) {
  int rc = orc_validate_optimizer(alpha, beta, max_iters, conv_tol, check_every);
  if (rc) return rc;
  *reason = run_traj((const graph_t*)gp, kind, param, x, alpha, beta, max_iters, conv_tol,
                     check_every, -1.0, iterations);
  return ORC_OK;
}

/* ------------------------------------------------------------ Solver parts */

static int init_state(const graph_t* g, int problem, double sigma, rng_t* r, double* x) {
  /* solver.cpp:30-46 */
  if (g->n == 0) return fail(ORC_INVALID, "init_state: empty graph");
  if (g->max_degree < 1)
    return fail(ORC_INVALID, "init_state: edgeless graph (strip isolated vertices upstream)");
  const double dmax = (double)g->max_degree;
  for (int32_t v = 0; v < g->n; ++v) {
    const double ratio = 1.0 - (double)deg(g, v) / dmax;
    double base = problem == ORC_PROBLEM_MIS ? ratio : 2.0 * ratio - 1.0;
    if (sigma > 0.0) base += rng_normal(r, 0.0, sigma);
    x[v] = base;
  }
  orc_project(x, g->n, problem);
  return ORC_OK;
}

int orc_init_state(void* g, int32_t problem, double sigma, void* rng, double* x) {
  return init_state((const graph_t*)g, problem, sigma, (rng_t*)rng, x);
}

static int global_reset(double* x, int32_t n, double rho, rng_t* r, int32_t* chosen,
                        int32_t* kout) { /* solver.cpp:48-63 */
  if (rho < 0.0 || rho >= 1.0) return fail(ORC_INVALID, "global_reset: rho must be in [0, 1)");
  const int32_t k = (int32_t)floor(rho * n);
  int32_t* order = (int32_t*)xmalloc((size_t)n * sizeof(int32_t));
  for (int32_t v = 0; v < n; ++v) order[v] = v;
  for (int32_t i = 0; i < k; ++i) {
    const int32_t j = i + (int32_t)rng_index(r, (uint64_t)(n - i));
    const int32_t t = order[i];
    order[i] = order[j];
    order[j] = t;
  }
  qsort(order, (size_t)k, sizeof(int32_t), cmp_i32);
  for (int32_t i = 0; i < k; ++i) x[order[i]] = 0.0;
  if (chosen) memcpy(chosen, order, (size_t)k * sizeof(int32_t));
  if (kout) *kout = k;
  free(order);
  return ORC_OK;
}

int orc_global_reset(double* x, int32_t n, double rho, void* rng, int32_t* chosen,
                     int32_t* k) {
  return global_reset(x, n, rho, (rng_t*)rng, chosen, k);
}

/* ------------------------------------------------------------ Local search */

static void build_tightness(const graph_t* g, const uint8_t* in, int32_t* tight) {
  /* localsearch.cpp:9-15 */
  memset(tight, 0, (size_t)g->n * sizeof(int32_t));
  for (int32_t v = 0; v < g->n; ++v)
    if (in[v])
      for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) ++tight[g->nbr[e]];
}

int orc_build_tightness(void* g, const uint8_t* in, int32_t* tight) {
  build_tightness((const graph_t*)g, in, tight);
  return ORC_OK;
}

static void build_gain(const graph_t* g, const uint8_t* side, int64_t* delta) {
  /* localsearch.cpp:17-26 */
  for (int32_t v = 0; v < g->n; ++v) {
    int64_t same = 0;
    for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e)
      same += side[g->nbr[e]] == side[v] ? 1 : -1;
    delta[v] = same;
  }
}

int orc_build_gain_table(void* g, const uint8_t* side, int64_t* delta) {
  build_gain((const graph_t*)g, side, delta);
  return ORC_OK;
}

static void apply_flip(const graph_t* g, uint8_t* side, int64_t* delta, int32_t v) {
  /* localsearch.cpp:28-33 */
  side[v] ^= 1;
  delta[v] = -delta[v];
  for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
    const int32_t u = g->nbr[e];
    delta[u] += side[u] == side[v] ? 2 : -2;
  }
}

/* (degree, id) ascending, localsearch.cpp:45-47 */
static const graph_t* g_sort_graph;
static int cmp_deg_id(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  const int32_t dx = deg(g_sort_graph, x), dy = deg(g_sort_graph, y);
  if (dx != dy) return dx < dy ? -1 : 1;
  return x < y ? -1 : x > y;
}
static void sort_deg_id(const graph_t* g, int32_t* list, int64_t count) {
  g_sort_graph = g; /* single-threaded test infrastructure */
  qsort(list, (size_t)count, sizeof(int32_t), cmp_deg_id);
}

static int greedy_maximalize(const graph_t* g, uint8_t* sel, int32_t* size) {
  /* localsearch.cpp:35-56 */
  if (!orc_is_independent((void*)g, sel))
    return fail(ORC_INVALID, "greedy_maximalize: input not independent");
  int32_t* tight = (int32_t*)xmalloc((size_t)g->n * sizeof(int32_t));
  build_tightness(g, sel, tight);
  int32_t* freev = (int32_t*)xmalloc((size_t)g->n * sizeof(int32_t));
  int64_t nf = 0;
  for (int32_t v = 0; v < g->n; ++v)
    if (!sel[v] && tight[v] == 0) freev[nf++] = v;
  sort_deg_id(g, freev, nf);
  for (int64_t i = 0; i < nf; ++i) {
    const int32_t v = freev[i];
    if (sel[v] || tight[v] != 0) continue;
    sel[v] = 1;
    for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) ++tight[g->nbr[e]];
  }
  int32_t s = 0;
  for (int32_t v = 0; v < g->n; ++v) s += sel[v];
  *size = s;
  free(tight);
  free(freev);
  return ORC_OK;
}

int orc_greedy_maximalize(void* g, uint8_t* sel, int32_t* size) {
  return greedy_maximalize((const graph_t*)g, sel, size);
}

/* localsearch.cpp:60-74: first (c_i, c_j), i<j, of non-adjacent 1-tight
 * unselected neighbours of v in ascending order. */
static int swap_pair_for(const graph_t* g, int32_t v, const uint8_t* sel,
                         const int32_t* tight, int32_t* cand, int32_t* pu, int32_t* pw) {
  int32_t nc = 0;
  for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
    const int32_t u = g->nbr[e];
    if (!sel[u] && tight[u] == 1) cand[nc++] = u;
  }
  for (int32_t i = 0; i < nc; ++i)
    for (int32_t j = i + 1; j < nc; ++j)
      if (!has_edge(g, cand[i], cand[j])) {
        *pu = cand[i];
        *pw = cand[j];
        return 1;
      }
  return 0;
}

static int one_two_swap(const graph_t* g, uint8_t* sel, int32_t* size) {
  /* localsearch.cpp:88-137 */
  int32_t* tight = (int32_t*)xmalloc((size_t)g->n * sizeof(int32_t));
  build_tightness(g, sel, tight);
  if (!orc_is_independent((void*)g, sel)) { /* require_maximal_is 76-84 */
    free(tight);
    return fail(ORC_INVALID, "one_two_swap: input not an independent set");
  }
  for (int32_t v = 0; v < g->n; ++v)
    if (!sel[v] && tight[v] == 0) {
      free(tight);
      return fail(ORC_INVALID, "one_two_swap: input not maximal");
    }
  int32_t* cand = (int32_t*)xmalloc((size_t)(g->max_degree + 1) * sizeof(int32_t));
  int32_t* freed = (int32_t*)xmalloc((size_t)(g->max_degree + 1) * sizeof(int32_t));
  int applied = 1;
  while (applied) {
    applied = 0;
    for (int32_t v = 0; v < g->n && !applied; ++v) {
      if (!sel[v]) continue;
      int32_t u, w;
      if (!swap_pair_for(g, v, sel, tight, cand, &u, &w)) continue;
      sel[v] = 0;
      for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) --tight[g->nbr[e]];
      const int32_t adds[2] = {u, w};
      for (int a = 0; a < 2; ++a) {
        sel[adds[a]] = 1;
        for (int64_t e = g->off[adds[a]]; e < g->off[adds[a] + 1]; ++e) ++tight[g->nbr[e]];
      }
      int32_t nf = 0;
      for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
        const int32_t z = g->nbr[e];
        if (!sel[z] && tight[z] == 0) freed[nf++] = z;
      }
      sort_deg_id(g, freed, nf);
      for (int32_t i = 0; i < nf; ++i) {
        const int32_t z = freed[i];
        if (sel[z] || tight[z] != 0) continue;
        sel[z] = 1;
        for (int64_t e = g->off[z]; e < g->off[z + 1]; ++e) ++tight[g->nbr[e]];
      }
      applied = 1;
    }
  }
  int32_t s = 0;
  for (int32_t v = 0; v < g->n; ++v) s += sel[v];
  *size = s;
  free(tight);
  free(cand);
  free(freed);
  return ORC_OK;
}

int orc_one_two_swap(void* g, uint8_t* sel, int32_t* size) {
  return one_two_swap((const graph_t*)g, sel, size);
}

static int64_t one_flip_pass(const graph_t* g, uint8_t* side) { /* localsearch.cpp:139-157 */
  int64_t* delta = (int64_t*)xmalloc((size_t)g->n * sizeof(int64_t));
  build_gain(g, side, delta);
  int64_t total = 0;
  int improved = 1;
  while (improved) {
    improved = 0;
    for (int32_t v = 0; v < g->n; ++v)
      if (delta[v] > 0) {
        total += delta[v];
        apply_flip(g, side, delta, v);
        improved = 1;
      }
  }
  free(delta);
  return total;
}

static int64_t two_flip_pass(const graph_t* g, uint8_t* side) { /* localsearch.cpp:159-181 */
  int64_t* delta = (int64_t*)xmalloc((size_t)g->n * sizeof(int64_t));
  build_gain(g, side, delta);
  int64_t total = 0;
  int improved = 1;
  while (improved) {
    improved = 0;
    for (int32_t v = 0; v < g->n; ++v)
      for (int64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
        const int32_t u = g->nbr[e];
        if (u <= v || side[u] == side[v]) continue;
        const int64_t joint = delta[v] + delta[u] + 2;
        if (joint > 0) {
          apply_flip(g, side, delta, v);
          apply_flip(g, side, delta, u);
          total += joint;
          improved = 1;
        }
      }
  }
  free(delta);
  return total;
}

static int64_t one_two_flip(const graph_t* g, uint8_t* side) { /* localsearch.cpp:183-190 */
  int64_t total = 0;
  for (;;) {
    const int64_t round = one_flip_pass(g, side) + two_flip_pass(g, side);
    total += round;
    if (round == 0) return total;
  }
}

int orc_one_flip_pass(void* g, uint8_t* side, int64_t* gain) {
  *gain = one_flip_pass((const graph_t*)g, side);
  return ORC_OK;
}
int orc_two_flip_pass(void* g, uint8_t* side, int64_t* gain) {
  *gain = two_flip_pass((const graph_t*)g, side);
  return ORC_OK;
}
int orc_one_two_flip(void* g, uint8_t* side, int64_t* gain) {
  *gain = one_two_flip((const graph_t*)g, side);
  return ORC_OK;
}

/* ------------------------------------------------------------------ Engine */

typedef struct {
  int64_t score;
  uint8_t* body; /* n bytes, owned */
} sol_t;

/* body_less, solver.cpp:107-112: MIS compares the sorted member lists
 * lexicographically (std::vector operator<), MaxCut the side vectors. */
static int body_less(int problem, int32_t n, const uint8_t* a, const uint8_t* b) {
  if (problem == ORC_PROBLEM_MAXCUT) return memcmp(a, b, (size_t)n) < 0;
  int32_t i = 0, j = 0;
  for (;;) {
    while (i < n && !a[i]) ++i;
    while (j < n && !b[j]) ++j;
    if (j >= n) return 0;    /* b exhausted: a is not less */
    if (i >= n) return 1;    /* a is a proper prefix */
    if (i != j) return i < j;
    ++i;
    ++j;
  }
}
static int body_equal(int32_t n, const uint8_t* a, const uint8_t* b) {
  return memcmp(a, b, (size_t)n) == 0;
}

typedef struct {
  int k, size, problem;
  int32_t n;
  sol_t* e;
} pool_t;

static int pool_before(const pool_t* p, const sol_t* a, const sol_t* b) { /* solver.cpp:137-140 */
  if (a->score != b->score) return a->score > b->score;
  return body_less(p->problem, p->n, a->body, b->body);
}

static void pool_offer(pool_t* p, const sol_t* s) { /* solver.cpp:125-130 */
  int lo = 0, hi = p->size; /* std::lower_bound with `before` */
  while (lo < hi) {
    const int mid = lo + (hi - lo) / 2;
    if (pool_before(p, &p->e[mid], s))
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < p->size && p->e[lo].score == s->score && body_equal(p->n, p->e[lo].body, s->body))
    return;
  /* insert at lo (capacity k+1), then truncate to k */
  uint8_t* copy = (uint8_t*)xmalloc((size_t)p->n);
  memcpy(copy, s->body, (size_t)p->n);
  for (int i = p->size; i > lo; --i) p->e[i] = p->e[i - 1];
  p->e[lo].score = s->score;
  p->e[lo].body = copy;
  ++p->size;
  if (p->size > p->k) {
    free(p->e[p->size - 1].body);
    --p->size;
  }
}

/* harvest, solver.cpp:166-175; returns 0 when the MIS state is dependent */
static int harvest(const graph_t* g, int problem, const double* x, sol_t* out) {
  out->score = extract(g, problem, x, out->body);
  if (problem == ORC_PROBLEM_MIS) {
    if (!orc_is_independent((void*)g, out->body)) return 0;
    int32_t size;
    greedy_maximalize(g, out->body, &size);
    out->score = size;
  }
  return 1;
}

static void encode_solution(int problem, int32_t n, const uint8_t* body, double* x) {
  /* solver.cpp:147-160 */
  for (int32_t v = 0; v < n; ++v)
    x[v] = problem == ORC_PROBLEM_MIS ? (body[v] ? 1.0 : 0.0) : (body[v] ? 1.0 : -1.0);
}

static int validate_cfg(const orc_solver_cfg* c) { /* solver.cpp:14-28 */
  int rc = orc_validate_objective(c->objective, c->param);
  if (rc) return rc;
  rc = orc_validate_optimizer(c->alpha, c->beta, c->max_iters, c->conv_tol, c->check_every);
  if (rc) return rc;
  if (c->reset_fraction < 0.0 || c->reset_fraction >= 1.0)
    return fail(ORC_INVALID, "solver: reset_fraction must be in [0, 1)");
  if (c->reset_rounds < 0) return fail(ORC_INVALID, "solver: reset_rounds must be >= 0");
  if (c->init_noise < 0.0) return fail(ORC_INVALID, "solver: init_noise must be >= 0");
  if (!(c->time_budget_secs > 0.0))
    return fail(ORC_INVALID, "solver: time_budget_secs must be > 0");
  if (c->pool_batch < 1 || c->pool_keep < 1)
    return fail(ORC_INVALID, "solver: pool batch and keep must be >= 1");
  if (c->has_max_outer_loops && c->max_outer_loops < 1)
    return fail(ORC_INVALID, "solver: max_outer_loops must be >= 1");
  return ORC_OK;
}

static void ls_polish(const graph_t* g, int problem, sol_t* s) { /* solver.cpp:318-327 */
  if (problem == ORC_PROBLEM_MIS) {
    int32_t size;
    one_two_swap(g, s->body, &size);
    s->score = size;
  } else {
    s->score += one_two_flip(g, s->body);
  }
}

int orc_solve_pooled(void* gp, const orc_solver_cfg* cfg, orc_report* rep,
                     uint8_t* best_body) { /* solver.cpp:192-372 */
  const graph_t* g = (const graph_t*)gp;
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  const int problem = problem_of(cfg->objective);
  const double t0 = now_secs();
  const double deadline = t0 + cfg->time_budget_secs;
  memset(rep, 0, sizeof *rep);
  rep->last_trajectory_stop = ORC_ITER_CAP;
  if (g->n == 0) return fail(ORC_INVALID, "solver: empty graph");
  const int32_t n = g->n;
  int64_t best_of_gradient = 0, best_of_resets = 0, best_of_ls = 0;

  sol_t best = {0, (uint8_t*)xcalloc((size_t)n, 1)};
  int have_best = 0;

  if (g->m == 0) { /* solver.cpp:221-226, trivial_solution 176-189 */
    rep->n_warnings = 1;
    if (problem == ORC_PROBLEM_MIS) {
      memset(best.body, 1, (size_t)n);
      best.score = n;
    }
    best_of_gradient = best.score;
    have_best = 1;
    goto finish;
  }

  const int batch = cfg->pool_batch;
  if (cfg->reset_rounds > 0 && (int32_t)floor(cfg->reset_fraction * n) == 0)
    rep->n_warnings++;

  rng_t* streams = (rng_t*)xmalloc((size_t)batch * sizeof(rng_t));
  for (int b = 0; b < batch; ++b) rng_seed(&streams[b], orc_derive_seed(cfg->seed, (uint64_t)b + 1));

  pool_t pool = {cfg->pool_keep, 0, problem, n,
                 (sol_t*)xcalloc((size_t)cfg->pool_keep + 1, sizeof(sol_t))};
  sol_t* results = (sol_t*)xmalloc((size_t)batch * sizeof(sol_t));
  int* valid = (int*)xcalloc((size_t)batch, sizeof(int));
  int32_t* iters = (int32_t*)xcalloc((size_t)batch, sizeof(int32_t));
  int32_t* stops = (int32_t*)xcalloc((size_t)batch, sizeof(int32_t));
  for (int b = 0; b < batch; ++b) results[b].body = (uint8_t*)xmalloc((size_t)n);
  double* x = (double*)xmalloc((size_t)n * sizeof(double));
  uint8_t* base = (uint8_t*)xmalloc((size_t)n);

#define PAST_DEADLINE() (now_secs() >= deadline)
#define TARGET_HIT() (have_best && cfg->has_stop_at_score && best.score >= cfg->stop_at_score)

  for (;;) {
    if (PAST_DEADLINE() || TARGET_HIT()) break;
    if (cfg->has_max_outer_loops && rep->outer_loops >= cfg->max_outer_loops) break;

    /* Phase 1, solver.cpp:280-296 */
    for (int b = 0; b < batch; ++b) {
      if (cfg->has_init_constant) {
        for (int32_t v = 0; v < n; ++v) x[v] = cfg->init_constant;
        orc_project(x, n, problem);
      } else {
        init_state(g, problem, cfg->init_noise, &streams[b], x);
      }
      stops[b] = run_traj(g, cfg->objective, cfg->param, x, cfg->alpha, cfg->beta,
                          cfg->max_iters, cfg->conv_tol, cfg->check_every, deadline, &iters[b]);
      valid[b] = harvest(g, problem, x, &results[b]);
    }
    /* merge(false), solver.cpp:252-275 */
    for (int b = 0; b < batch; ++b) {
      rep->total_iterations += iters[b];
      rep->last_trajectory_stop = stops[b];
      ++rep->trajectories;
      if (!valid[b]) continue;
      if (results[b].score > best_of_gradient) best_of_gradient = results[b].score;
      const int better = !have_best || results[b].score > best.score;
      pool_offer(&pool, &results[b]);
      if (better) {
        best.score = results[b].score;
        memcpy(best.body, results[b].body, (size_t)n);
        have_best = 1;
      }
    }

    /* Phase 2, solver.cpp:298-312 */
    for (int round = 0; round < cfg->reset_rounds; ++round) {
      if (PAST_DEADLINE() || TARGET_HIT() || pool.size == 0) break;
      for (int b = 0; b < batch; ++b) {
        const int pi = (int)rng_index(&streams[b], (uint64_t)pool.size);
        memcpy(base, pool.e[pi].body, (size_t)n);
        encode_solution(problem, n, base, x);
        global_reset(x, n, cfg->reset_fraction, &streams[b], NULL, NULL);
        stops[b] = run_traj(g, cfg->objective, cfg->param, x, cfg->alpha, cfg->beta,
                            cfg->max_iters, cfg->conv_tol, cfg->check_every, deadline,
                            &iters[b]);
        valid[b] = harvest(g, problem, x, &results[b]);
      }
      for (int b = 0; b < batch; ++b) { /* merge(true) */
        rep->total_iterations += iters[b];
        rep->last_trajectory_stop = stops[b];
        ++rep->trajectories;
        if (!valid[b]) continue;
        if (results[b].score > best_of_resets) best_of_resets = results[b].score;
        const int better = !have_best || results[b].score > best.score;
        pool_offer(&pool, &results[b]);
        if (better) {
          best.score = results[b].score;
          memcpy(best.body, results[b].body, (size_t)n);
          have_best = 1;
          ++rep->resets_accepted;
        } else {
          ++rep->resets_rejected;
        }
      }
    }

    /* Phase 3, solver.cpp:314-339 */
    if (cfg->local_search && pool.size > 0 && !PAST_DEADLINE() && !TARGET_HIT()) {
      const int members = pool.size;
      sol_t* polished = (sol_t*)xmalloc((size_t)members * sizeof(sol_t));
      for (int i = 0; i < members; ++i) {
        polished[i].score = pool.e[i].score;
        polished[i].body = (uint8_t*)xmalloc((size_t)n);
        memcpy(polished[i].body, pool.e[i].body, (size_t)n);
        ls_polish(g, problem, &polished[i]);
      }
      for (int i = 0; i < members; ++i) {
        if (polished[i].score > best_of_ls) best_of_ls = polished[i].score;
        const int better = !have_best || polished[i].score > best.score;
        pool_offer(&pool, &polished[i]);
        if (better) {
          best.score = polished[i].score;
          memcpy(best.body, polished[i].body, (size_t)n);
          have_best = 1;
        }
        free(polished[i].body);
      }
      free(polished);
    }
    ++rep->outer_loops;
  }

  /* final polish, solver.cpp:344-359 */
  if (cfg->local_search && have_best) {
    sol_t pol = {best.score, (uint8_t*)xmalloc((size_t)n)};
    memcpy(pol.body, best.body, (size_t)n);
    ls_polish(g, problem, &pol);
    if (pol.score > best_of_ls) best_of_ls = pol.score;
    pool_offer(&pool, &pol);
    if (pol.score > best.score) {
      best.score = pol.score;
      memcpy(best.body, pol.body, (size_t)n);
    }
    free(pol.body);
  }

  for (int i = 0; i < pool.size; ++i) free(pool.e[i].body);
  free(pool.e);
  for (int b = 0; b < batch; ++b) free(results[b].body);
  free(results);
  free(valid);
  free(iters);
  free(stops);
  free(x);
  free(base);
  free(streams);

  if (!have_best) { /* solver.cpp:361-370 */
    rep->n_warnings++;
    memset(best.body, 0, (size_t)n);
    best.score = 0; /* MIS: empty set; MaxCut: all-zero side has cut 0 */
  }
#undef PAST_DEADLINE
#undef TARGET_HIT

finish: /* solver.cpp:209-219 */
  rep->found_solution = have_best;
  rep->score = best.score;
  rep->after_gradient = best_of_gradient;
  rep->after_reset_loop = best_of_gradient > best_of_resets ? best_of_gradient : best_of_resets;
  rep->after_local_search =
      rep->after_reset_loop > best_of_ls ? rep->after_reset_loop : best_of_ls;
  rep->elapsed_secs = now_secs() - t0;
  if (best_body) memcpy(best_body, best.body, (size_t)n);
  free(best.body);
  return ORC_OK;
}

/* ----------------------------------------------------------------- Presets */

int orc_preset_for(int32_t problem, int32_t n, double mean_degree, double* alpha,
                   double* momentum, double* rho, int32_t* reset_rounds) {
  /* presets.cpp:17-60 (Appendix-G table, nearest row in log space) */
  static const double mis[][6] = {
      {1000, 100, 0.80, 0.30, 0.70, 60},   {1000, 300, 0.80, 0.45, 0.70, 60},
      {1000, 500, 0.80, 0.45, 0.60, 60},   {3000, 100, 0.80, 0.30, 0.60, 60},
      {3000, 300, 0.80, 0.45, 0.60, 60},   {3000, 1000, 0.80, 0.45, 0.50, 60},
      {10000, 5000, 0.80, 0.75, 0.50, 60}, {20000, 10000, 0.80, 0.75, 0.50, 60},
      {30000, 15000, 0.80, 0.75, 0.50, 60}};
  static const double cut[][6] = {
      {100, 50, 0.0025, 0.90, 0.80, 90},    {1000, 100, 0.0025, 0.80, 0.80, 90},
      {1000, 500, 0.0025, 0.80, 0.80, 90},  {1000, 800, 0.0025, 0.80, 0.80, 90},
      {30000, 15000, 5e-5, 0.80, 0.80, 90}, {30000, 24000, 5e-5, 0.80, 0.80, 90},
      {40000, 20000, 5e-5, 0.80, 0.80, 90}, {40000, 32000, 5e-5, 0.80, 0.80, 90}};
  const double(*rows)[6] = problem == ORC_PROBLEM_MIS ? mis : cut;
  const int nrows = problem == ORC_PROBLEM_MIS ? 9 : 8;
  const double ln = log(n > 1 ? (double)n : 1.0);
  const double ld = log(mean_degree > 1.0 ? mean_degree : 1.0);
  double best_dist = INFINITY;
  int best = 0;
  for (int i = 0; i < nrows; ++i) {
    const double dn = ln - log(rows[i][0]);
    const double dd = ld - log(rows[i][1]);
    const double dist = dn * dn + dd * dd;
    if (dist < best_dist) {
      best_dist = dist;
      best = i;
    }
  }
  *alpha = rows[best][2];
  *momentum = rows[best][3];
  *rho = rows[best][4];
  *reset_rounds = (int32_t)rows[best][5];
  return ORC_OK;
}
