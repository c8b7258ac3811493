/*
 * dg_oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE ONLY; see dg_oracle.h).
 *
 * Sequential restatement of the reference densegraph hot path.  Written
 * for obviousness, not speed: each routine follows the written semantics
 * of the reference (file:line cited per function) with the simplest data
 * structure that reproduces them exactly.
 */
#include "dg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* og_last_error(void) { return g_err; }

/* splitmix64, parallel.hpp:92-97 */
uint64_t og_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* Density{a_e, a_v} > Density{b_e, b_v}: density.hpp:32-36 (u128 cross-multiply) */
static int dens_gt(uint64_t ae, uint64_t av, uint64_t be, uint64_t bv) {
  return (u128)ae * bv > (u128)be * av;
}
static int dens_eq(uint64_t ae, uint64_t av, uint64_t be, uint64_t bv) {
  return (u128)ae * bv == (u128)be * av;
}
/* ceil_scaled, density.hpp:46-51 */
static uint64_t ceil_scaled(uint64_t e, uint64_t v, uint64_t num, uint64_t den) {
  u128 p = (u128)e * num, q = (u128)v * den;
  return (uint64_t)(p / q + (p % q != 0));
}
static uint64_t gcd64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

/* ------------------------------------------------------------------ */
/* CSR build: restates parse_edge_list's cleanup + CSR fill,            */
/* io.cpp:51-92 (tokenising at :29-50 is not on the path).              */
/* ------------------------------------------------------------------ */

typedef struct {
  uint64_t a, b;
} pair64;

static int cmp_pair(const void* x, const void* y) {
  const pair64* p = (const pair64*)x;
  const pair64* q = (const pair64*)y;
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  if (p->b != q->b) return p->b < q->b ? -1 : 1;
  return 0;
}

/* LSD radix sort of u64 keys, 16-bit digits, skipping constant digits. */
static int radix_u64(uint64_t* a, uint64_t n) {
  if (n < 2) return 0;
  uint64_t* tmp = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint64_t* cnt = (uint64_t*)malloc(65536 * sizeof(uint64_t));
  if (!tmp || !cnt) {
    free(tmp);
    free(cnt);
    return -1;
  }
  uint64_t all_or = 0, all_and = ~0ULL;
  for (uint64_t i = 0; i < n; ++i) {
    all_or |= a[i];
    all_and &= a[i];
  }
  uint64_t* src = a;
  uint64_t* dst = tmp;
  for (int sh = 0; sh < 64; sh += 16) {
    if ((((all_or ^ all_and) >> sh) & 0xffff) == 0) continue;
    memset(cnt, 0, 65536 * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) cnt[(src[i] >> sh) & 0xffff]++;
    uint64_t s = 0;
    for (int d = 0; d < 65536; ++d) {
      uint64_t c = cnt[d];
      cnt[d] = s;
      s += c;
    }
    for (uint64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> sh) & 0xffff]++] = src[i];
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  if (src != a) memcpy(a, src, n * sizeof(uint64_t));
  free(tmp);
  free(cnt);
  return 0;
}

static uint64_t lower_bound_u64(const uint64_t* a, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

int og_build(const uint64_t* u, const uint64_t* v, uint64_t k, og_graph* out) {
  memset(out, 0, sizeof *out);
  uint64_t maxid = 0;
  for (uint64_t i = 0; i < k; ++i) {
    if (u[i] > maxid) maxid = u[i];
    if (v[i] > maxid) maxid = v[i];
  }
  /* canonical (min,max), self-loops dropped (io.cpp:51-52), sort+unique (:56-57) */
  pair64* e = NULL;
  uint64_t m = 0;
  if (maxid < (1ULL << 32)) {
    uint64_t* key = (uint64_t*)malloc((k ? k : 1) * sizeof(uint64_t));
    if (!key) return fail(OG_E_NOMEM, "out of memory");
    uint64_t c = 0;
    for (uint64_t i = 0; i < k; ++i) {
      if (u[i] == v[i]) continue;
      uint64_t a = u[i] < v[i] ? u[i] : v[i], b = u[i] < v[i] ? v[i] : u[i];
      key[c++] = (a << 32) | b;
    }
    if (radix_u64(key, c)) {
      free(key);
      return fail(OG_E_NOMEM, "out of memory");
    }
    e = (pair64*)malloc((c ? c : 1) * sizeof(pair64));
    if (!e) {
      free(key);
      return fail(OG_E_NOMEM, "out of memory");
    }
    for (uint64_t i = 0; i < c; ++i)
      if (i == 0 || key[i] != key[i - 1]) {
        e[m].a = key[i] >> 32;
        e[m].b = key[i] & 0xffffffffULL;
        ++m;
      }
    free(key);
  } else {
    e = (pair64*)malloc((k ? k : 1) * sizeof(pair64));
    if (!e) return fail(OG_E_NOMEM, "out of memory");
    uint64_t c = 0;
    for (uint64_t i = 0; i < k; ++i) {
      if (u[i] == v[i]) continue;
      e[c].a = u[i] < v[i] ? u[i] : v[i];
      e[c].b = u[i] < v[i] ? v[i] : u[i];
      ++c;
    }
    qsort(e, c, sizeof(pair64), cmp_pair);
    for (uint64_t i = 0; i < c; ++i)
      if (i == 0 || cmp_pair(&e[i], &e[i - 1]) != 0) e[m++] = e[i];
  }
  if (m == 0) {
    free(e);
    return fail(OG_E_EMPTY, "no edges after removing self-loops and duplicates");
  }
  /* orig = sorted unique endpoints (io.cpp:61-68) */
  uint64_t* ids = (uint64_t*)malloc(2 * m * sizeof(uint64_t));
  if (!ids) {
    free(e);
    return fail(OG_E_NOMEM, "out of memory");
  }
  for (uint64_t i = 0; i < m; ++i) {
    ids[2 * i] = e[i].a;
    ids[2 * i + 1] = e[i].b;
  }
  radix_u64(ids, 2 * m);
  uint64_t n = 0;
  for (uint64_t i = 0; i < 2 * m; ++i)
    if (i == 0 || ids[i] != ids[i - 1]) ids[n++] = ids[i];
  out->n = n;
  out->m = m;
  out->orig = (uint64_t*)realloc(ids, n * sizeof(uint64_t));
  out->offs = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  out->adj = (uint32_t*)malloc(2 * m * sizeof(uint32_t));
  if (!out->orig || !out->offs || !out->adj) {
    free(e);
    og_free(out);
    return fail(OG_E_NOMEM, "out of memory");
  }
  /* dense id = rank of the original id (io.cpp:71-81) */
  for (uint64_t i = 0; i < m; ++i) {
    e[i].a = lower_bound_u64(out->orig, n, e[i].a);
    e[i].b = lower_bound_u64(out->orig, n, e[i].b);
    out->offs[e[i].a + 1]++;
    out->offs[e[i].b + 1]++;
  }
  for (uint64_t x = 0; x < n; ++x) out->offs[x + 1] += out->offs[x];
  /* fill in lexicographic pair order => ascending rows (io.cpp:84-92) */
  uint64_t* cur = (uint64_t*)malloc(n * sizeof(uint64_t));
  if (!cur) {
    free(e);
    og_free(out);
    return fail(OG_E_NOMEM, "out of memory");
  }
  memcpy(cur, out->offs, n * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) {
    out->adj[cur[e[i].a]++] = (uint32_t)e[i].b;
    out->adj[cur[e[i].b]++] = (uint32_t)e[i].a;
  }
  free(cur);
  free(e);
  return OG_OK;
}

int og_from_csr(uint64_t n, const uint64_t* offs, const uint32_t* adj, const uint64_t* orig,
                og_graph* out) {
  memset(out, 0, sizeof *out);
  out->n = n;
  out->m = offs[n] / 2;
  out->offs = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  out->adj = (uint32_t*)malloc((offs[n] ? offs[n] : 1) * sizeof(uint32_t));
  out->orig = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  if (!out->offs || !out->adj || !out->orig) {
    og_free(out);
    return fail(OG_E_NOMEM, "out of memory");
  }
  memcpy(out->offs, offs, (n + 1) * sizeof(uint64_t));
  memcpy(out->adj, adj, offs[n] * sizeof(uint32_t));
  memcpy(out->orig, orig, n * sizeof(uint64_t));
  return OG_OK;
}

void og_free(og_graph* g) {
  free(g->offs);
  free(g->adj);
  free(g->orig);
  memset(g, 0, sizeof *g);
}

/* Graph::stats max degree, graph.hpp:37-41 */
uint64_t og_max_degree(const og_graph* g) {
  uint64_t d = 0;
  for (uint64_t x = 0; x < g->n; ++x)
    if (g->offs[x + 1] - g->offs[x] > d) d = g->offs[x + 1] - g->offs[x];
  return d;
}

/* induced_subgraph, graph.hpp:50-80: new ids in old dense order */
int og_induced(const og_graph* g, const uint8_t* keep, og_graph* out, uint32_t* old_to_new) {
  memset(out, 0, sizeof *out);
  uint32_t* map = (uint32_t*)malloc((g->n ? g->n : 1) * sizeof(uint32_t));
  if (!map) return fail(OG_E_NOMEM, "out of memory");
  uint64_t hn = 0;
  for (uint64_t x = 0; x < g->n; ++x) map[x] = keep[x] ? (uint32_t)hn++ : 0xffffffffu;
  out->n = hn;
  out->offs = (uint64_t*)calloc(hn + 1, sizeof(uint64_t));
  out->orig = (uint64_t*)malloc((hn ? hn : 1) * sizeof(uint64_t));
  if (!out->offs || !out->orig) {
    free(map);
    og_free(out);
    return fail(OG_E_NOMEM, "out of memory");
  }
  for (uint64_t x = 0; x < g->n; ++x) {
    if (map[x] == 0xffffffffu) continue;
    uint64_t d = 0;
    for (uint64_t j = g->offs[x]; j < g->offs[x + 1]; ++j) d += map[g->adj[j]] != 0xffffffffu;
    out->offs[map[x] + 1] = d;
    out->orig[map[x]] = g->orig[x];
  }
  for (uint64_t x = 0; x < hn; ++x) out->offs[x + 1] += out->offs[x];
  out->adj = (uint32_t*)malloc((out->offs[hn] ? out->offs[hn] : 1) * sizeof(uint32_t));
  if (!out->adj) {
    free(map);
    og_free(out);
    return fail(OG_E_NOMEM, "out of memory");
  }
  for (uint64_t x = 0; x < g->n; ++x) {
    if (map[x] == 0xffffffffu) continue;
    uint64_t w = out->offs[map[x]];
    for (uint64_t j = g->offs[x]; j < g->offs[x + 1]; ++j)
      if (map[g->adj[j]] != 0xffffffffu) out->adj[w++] = map[g->adj[j]];
  }
  out->m = out->offs[hn] / 2;
  if (old_to_new) memcpy(old_to_new, map, g->n * sizeof(uint32_t));
  free(map);
  return OG_OK;
}

/* ------------------------------------------------------------------ */
/* Coreness: core.cpp:89-131.  Synchronous threshold rounds: at bound b  */
/* every alive vertex with residual degree <= b leaves in one round      */
/* (labelled with the current label), then its alive neighbours lose one */
/* degree per removed neighbour.  A round with no such vertex advances   */
/* the bound: exact +1 (core.cpp:102-104), approximate geometric phases  */
/* t_{i+1} = max(t_i + 1, ceil(c t_i)) (core.cpp:105-110).  peel_rounds  */
/* counts non-empty rounds (core.cpp:56,117).                            */
/* ------------------------------------------------------------------ */
int og_coreness(const og_graph* g, int approx, uint64_t c_num, uint64_t c_den, uint32_t* labels,
                uint32_t* kmax_out, uint32_t* rounds_out) {
  if (approx && (c_den == 0 || c_num <= c_den))
    return fail(OG_E_PARAM, "approximation factor must be > 1");
  if (g->n == 0) return fail(OG_E_EMPTY, "coreness of empty graph");
  const uint64_t n = g->n;
  uint64_t* deg = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint8_t* alive = (uint8_t*)malloc(n);
  uint32_t* front = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* next = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* live = (uint32_t*)malloc(n * sizeof(uint32_t));
  if (!deg || !alive || !front || !next || !live) {
    free(deg), free(alive), free(front), free(next), free(live);
    return fail(OG_E_NOMEM, "out of memory");
  }
  for (uint64_t x = 0; x < n; ++x) {
    deg[x] = g->offs[x + 1] - g->offs[x];
    alive[x] = 1;
    live[x] = (uint32_t)x;
    labels[x] = 0;
  }
  uint64_t nlive = n, remaining = n, nf = 0;
  uint64_t bound = 0, label = 0, t = 1;
  uint32_t kmax = 0, rounds = 0;
  while (remaining > 0) {
    if (nf == 0) {
      /* drain(bound) found nothing in the previous round: compact the live
         list, then advance the bound until a drain is non-empty */
      uint64_t w = 0, dmin = ~0ULL;
      for (uint64_t i = 0; i < nlive; ++i)
        if (alive[live[i]]) {
          live[w++] = live[i];
          if (deg[live[i]] < dmin) dmin = deg[live[i]];
        }
      nlive = w;
      while (dmin > bound) {
        if (!approx) {
          ++bound;
          label = bound;
        } else {
          label = t;
          uint64_t ct = (t * c_num) / c_den + ((t * c_num) % c_den != 0);
          uint64_t nt = t + 1 > ct ? t + 1 : ct;
          bound = nt - 1;
          t = nt;
        }
      }
      for (uint64_t i = 0; i < nlive; ++i)
        if (deg[live[i]] <= bound) front[nf++] = live[i];
    }
    for (uint64_t i = 0; i < nf; ++i) {
      alive[front[i]] = 0;
      labels[front[i]] = (uint32_t)label;
    }
    if (label > kmax) kmax = (uint32_t)label;
    ++rounds;
    remaining -= nf;
    uint64_t nn = 0;
    for (uint64_t i = 0; i < nf; ++i) {
      uint32_t x = front[i];
      for (uint64_t j = g->offs[x]; j < g->offs[x + 1]; ++j) {
        uint32_t y = g->adj[j];
        if (!alive[y]) continue;
        if (--deg[y] == bound) next[nn++] = y; /* crossed bound+1 -> bound */
      }
    }
    uint32_t* tmp = front;
    front = next;
    next = tmp;
    nf = nn;
  }
  *kmax_out = kmax;
  *rounds_out = rounds;
  free(deg), free(alive), free(front), free(next), free(live);
  return OG_OK;
}

/* ------------------------------------------------------------------ */
/* Greedy++ ordering: min-key batch peel, refine.cpp:20-156 (semantics   */
/* as restated by tests/reference.hpp:60-89).  key = load + residual     */
/* degree; each step removes every alive vertex at the minimum key in    */
/* ascending id (or only the smallest with one_at_a_time), then every    */
/* alive neighbour loses one key unit per removed neighbour.             */
/* ------------------------------------------------------------------ */
int og_peel_order(const og_graph* g, const uint64_t* loads, int one_at_a_time, uint32_t* perm) {
  const uint64_t n = g->n;
  if (n == 0) return OG_OK;
  uint64_t* key = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint8_t* alive = (uint8_t*)malloc(n);
  uint32_t* live = (uint32_t*)malloc(n * sizeof(uint32_t));
  if (!key || !alive || !live) {
    free(key), free(alive), free(live);
    return fail(OG_E_NOMEM, "out of memory");
  }
  for (uint64_t x = 0; x < n; ++x) {
    key[x] = loads[x] + (g->offs[x + 1] - g->offs[x]);
    alive[x] = 1;
    live[x] = (uint32_t)x;
  }
  uint64_t removed = 0, nlive = n;
  while (removed < n) {
    uint64_t mink = ~0ULL;
    uint64_t w = 0;
    for (uint64_t i = 0; i < nlive; ++i) /* live stays in ascending id order */
      if (alive[live[i]]) {
        live[w++] = live[i];
        if (key[live[i]] < mink) mink = key[live[i]];
      }
    nlive = w;
    uint64_t b0 = removed;
    for (uint64_t i = 0; i < nlive; ++i)
      if (key[live[i]] == mink) {
        perm[removed++] = live[i];
        if (one_at_a_time) break;
      }
    for (uint64_t i = b0; i < removed; ++i) alive[perm[i]] = 0;
    for (uint64_t i = b0; i < removed; ++i) {
      uint32_t x = perm[i];
      for (uint64_t j = g->offs[x]; j < g->offs[x + 1]; ++j)
        if (alive[g->adj[j]]) key[g->adj[j]]--;
    }
  }
  free(key), free(alive), free(live);
  return OG_OK;
}

/* load_sort_order, refine.cpp:158-178: stable ascending sort by (load, id) */
static const uint64_t* g_sort_loads;
static int cmp_load_id(const void* x, const void* y) {
  uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  if (g_sort_loads[a] != g_sort_loads[b]) return g_sort_loads[a] < g_sort_loads[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}
int og_sort_order(uint64_t n, const uint64_t* loads, uint32_t* perm) {
  for (uint64_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
  g_sort_loads = loads;
  qsort(perm, n, sizeof(uint32_t), cmp_load_id);
  return OG_OK;
}

/* density_and_load_update, refine.cpp:180-220 (Algorithm 3) */
int og_density_update(const og_graph* g, const uint32_t* perm, uint64_t* loads, og_outcome* out,
                      uint32_t* charges_out, uint64_t* suffix_edges_out) {
  const uint64_t n = g->n;
  uint64_t* pos = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  uint32_t* A = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
  uint64_t* B = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  if (!pos || !A || !B) {
    free(pos), free(A), free(B);
    return fail(OG_E_NOMEM, "out of memory");
  }
  for (uint64_t i = 0; i < n; ++i) pos[i] = ~0ULL;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t x = perm[i];
    if (x >= n || pos[x] != ~0ULL) {
      free(pos), free(A), free(B);
      return fail(OG_E_INVARIANT, "ordering is not a permutation");
    }
    pos[x] = i;
  }
  /* each edge charges the endpoint that leaves first (:195-199) */
  for (uint64_t x = 0; x < n; ++x)
    for (uint64_t j = g->offs[x]; j < g->offs[x + 1]; ++j) {
      uint32_t y = g->adj[j];
      if (y > x) A[pos[x] < pos[y] ? pos[x] : pos[y]]++;
    }
  B[n] = 0;
  for (uint64_t i = n; i-- > 0;) B[i] = B[i + 1] + A[i];
  if (B[0] != g->m) {
    free(pos), free(A), free(B);
    return fail(OG_E_INVARIANT, "charge total does not equal edge count");
  }
  /* first strict maximum of B[i]/(n-i), width = max A (:204-212) */
  uint64_t be = 0, bv = 1, bp = 0, width = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (dens_gt(B[i], n - i, be, bv)) {
      be = B[i];
      bv = n - i;
      bp = i;
    }
    if (A[i] > width) width = A[i];
  }
  for (uint64_t i = 0; i < n; ++i) loads[perm[i]] += A[i]; /* :213 */
  out->rho_edges = be;
  out->rho_verts = bv;
  out->best_prefix = bp;
  out->width = width;
  if (charges_out) memcpy(charges_out, A, n * sizeof(uint32_t));
  if (suffix_edges_out) memcpy(suffix_edges_out, B, n * sizeof(uint64_t));
  free(pos), free(A), free(B);
  return OG_OK;
}

/* slack_violations, refine.cpp:229-242 */
uint64_t og_slack_violations(uint64_t n, const uint32_t* perm, const uint64_t* loads,
                             uint64_t allowed_slack, uint64_t samples, uint64_t seed) {
  if (n < 2) return 0;
  uint64_t bad = 0;
  for (uint64_t t = 0; t < samples; ++t) {
    uint64_t i = og_mix64(seed ^ (2 * t + 1)) % n;
    uint64_t j = og_mix64(seed ^ (2 * t + 2)) % n;
    if (i == j) continue;
    if (i > j) {
      uint64_t s = i;
      i = j;
      j = s;
    }
    if (loads[perm[i]] > loads[perm[j]] + allowed_slack) ++bad;
  }
  return bad;
}

/* default_iterations, framework.cpp:36-44 */
uint64_t og_default_iterations(uint64_t delta, double lower_bound, uint64_t n, double epsilon,
                               uint64_t cap, int* status) {
  *status = OG_OK;
  if (!(epsilon > 0)) return *status = fail(OG_E_PARAM, "epsilon must be positive"), 0;
  if (!(lower_bound >= 1)) return *status = fail(OG_E_PARAM, "density lower bound must be >= 1"), 0;
  if (n == 0) return *status = fail(OG_E_PARAM, "iteration bound needs a nonempty graph"), 0;
  double t = ((double)delta / lower_bound) * log((double)n) / (epsilon * epsilon);
  uint64_t iters = (t >= (double)cap) ? cap : (uint64_t)ceil(t);
  uint64_t lo = iters > 10 ? iters : 10;
  return cap < lo ? cap : lo;
}

/* ------------------------------------------------------------------ */
/* run: Algorithm 1, framework.cpp:46-180                              */
/* ------------------------------------------------------------------ */
static uint64_t threshold_for(uint64_t le, uint64_t lv, int approx_labels, uint64_t cn,
                              uint64_t cd) { /* framework.cpp:22-24 */
  return approx_labels ? ceil_scaled(le, lv, cd, cn) : ceil_scaled(le, lv, 1, 1);
}

static void remap(const uint32_t* labels, const uint32_t* map, uint64_t old_n, uint32_t* out) {
  for (uint64_t x = 0; x < old_n; ++x) /* framework.cpp:26-32 */
    if (map[x] != 0xffffffffu) out[map[x]] = labels[x];
}

static int get_core(const og_graph* g, const uint32_t* labels, uint64_t k, og_graph* out,
                    uint32_t* map) { /* core.cpp:133-140 */
  uint8_t* keep = (uint8_t*)malloc(g->n ? g->n : 1);
  if (!keep) return fail(OG_E_NOMEM, "out of memory");
  for (uint64_t x = 0; x < g->n; ++x) keep[x] = labels[x] >= k;
  int st = og_induced(g, keep, out, map);
  free(keep);
  return st;
}

int og_run(const og_graph* g, const og_config* cfg, og_result* res, og_iter* trace,
           uint64_t trace_cap, uint64_t* witness, uint64_t witness_cap, uint64_t* final_ids,
           uint64_t final_cap) {
  memset(res, 0, sizeof *res);
  if (g->n == 0) return fail(OG_E_EMPTY, "run on empty graph");
  int st = OG_OK;
  og_graph cur;
  memset(&cur, 0, sizeof cur);
  uint32_t* labels = NULL;
  int approx_labels = 0;
  uint64_t thresh = 0, le = 0, lv = 1; /* lower = {0,1} */
  uint64_t* loads = NULL;
  uint32_t* perm = NULL;
  uint64_t* wit = NULL;
  uint64_t nwit = 0;

  if (cfg->pruning == 0) {
    st = og_from_csr(g->n, g->offs, g->adj, g->orig, &cur);
    if (st) return st;
  } else {
    uint32_t* lab = (uint32_t*)malloc(g->n * sizeof(uint32_t));
    uint32_t* map = (uint32_t*)malloc(g->n * sizeof(uint32_t));
    uint32_t kmax = 0, rounds = 0;
    int approx = cfg->pruning != 1;
    st = og_coreness(g, approx, cfg->c_num, cfg->c_den, lab, &kmax, &rounds);
    if (st) {
      free(lab), free(map);
      return st;
    }
    le = kmax;
    lv = 2;
    thresh = approx ? threshold_for(le, lv, 1, cfg->c_num, cfg->c_den) : ceil_scaled(le, lv, 1, 1);
    st = get_core(g, lab, thresh, &cur, map);
    if (st) {
      free(lab), free(map);
      return st;
    }
    labels = (uint32_t*)malloc((cur.n ? cur.n : 1) * sizeof(uint32_t));
    remap(lab, map, g->n, labels);
    approx_labels = approx;
    res->kmax_known = 1;
    res->kmax_exact = !approx;
    res->kmax = kmax;
    res->threshold = (uint32_t)thresh;
    free(lab), free(map);
    if (cfg->pruning == 3) { /* hybrid, framework.cpp:80-91 */
      uint32_t* fine = (uint32_t*)malloc((cur.n ? cur.n : 1) * sizeof(uint32_t));
      uint32_t* map2 = (uint32_t*)malloc((cur.n ? cur.n : 1) * sizeof(uint32_t));
      if (cur.n == 0) {
        free(fine), free(map2), free(labels), og_free(&cur);
        return fail(OG_E_EMPTY, "coreness of empty graph");
      }
      st = og_coreness(&cur, 0, 1, 1, fine, &kmax, &rounds);
      le = kmax;
      lv = 2;
      thresh = ceil_scaled(le, lv, 1, 1);
      og_graph next;
      st = st ? st : get_core(&cur, fine, thresh, &next, map2);
      if (st) {
        free(fine), free(map2), free(labels), og_free(&cur);
        return st;
      }
      free(labels);
      labels = (uint32_t*)malloc((next.n ? next.n : 1) * sizeof(uint32_t));
      remap(fine, map2, cur.n, labels);
      og_free(&cur);
      cur = next;
      approx_labels = 0;
      res->kmax_exact = 1;
      res->kmax = kmax;
      res->threshold = (uint32_t)thresh;
      free(fine), free(map2);
    }
    if (cur.n == 0) {
      free(labels), og_free(&cur);
      return fail(OG_E_INVARIANT, "pruning removed every vertex");
    }
  }
  res->pruned_n = cur.n;
  res->pruned_m = cur.m;

  uint64_t iterations = cfg->iterations;
  if (iterations == 0) {
    double lb = (double)le / (double)lv;
    if (lb < 1.0) lb = 1.0;
    iterations = og_default_iterations(og_max_degree(&cur), lb, cur.n, cfg->epsilon,
                                       cfg->iteration_cap, &st);
    if (st) {
      free(labels), og_free(&cur);
      return st;
    }
  }

  loads = (uint64_t*)calloc(cur.n, sizeof(uint64_t));
  perm = (uint32_t*)malloc(cur.n * sizeof(uint32_t));
  wit = (uint64_t*)malloc(cur.n * sizeof(uint64_t));
  uint64_t be = 0, bv = 1; /* best = {0,1} */
  uint64_t delta_cur = og_max_degree(&cur);
  for (uint64_t it = 1; it <= iterations; ++it) {
    if (cfg->algorithm == 0)
      st = og_peel_order(&cur, loads, 0, perm);
    else
      st = og_sort_order(cur.n, loads, perm);
    if (st) goto done;
    if (cfg->slack_samples > 0)
      res->slack_violations +=
          og_slack_violations(cur.n, perm, loads, cfg->algorithm == 0 ? delta_cur : 0,
                              cfg->slack_samples, 0x5eed0000ULL + it);
    og_outcome out;
    st = og_density_update(&cur, perm, loads, &out, NULL, NULL);
    if (st) goto done;
    if (trace && it - 1 < trace_cap) {
      uint64_t gg = gcd64(out.rho_edges == 0 ? out.rho_verts : out.rho_edges, out.rho_verts);
      og_iter* r = &trace[it - 1];
      r->iter = it;
      r->rho_edges = out.rho_edges / gg;
      r->rho_verts = out.rho_verts / gg;
      r->n = cur.n;
      r->m = cur.m;
      r->width = out.width;
    }
    if (out.width > res->max_width) res->max_width = out.width;
    if (!dens_gt(out.rho_edges, out.rho_verts, be, bv)) continue; /* :126 */
    be = out.rho_edges;
    bv = out.rho_verts;
    nwit = 0;
    for (uint64_t i = out.best_prefix; i < cur.n; ++i) wit[nwit++] = cur.orig[perm[i]];
    if (dens_gt(be, bv, le, lv)) {
      le = be;
      lv = bv;
    }
    if (cfg->pruning != 0) { /* :133-151 */
      uint64_t nt = threshold_for(le, lv, approx_labels, cfg->c_num, cfg->c_den);
      if (nt > thresh) {
        uint8_t* keep = (uint8_t*)malloc(cur.n);
        uint32_t* map = (uint32_t*)malloc(cur.n * sizeof(uint32_t));
        for (uint64_t x = 0; x < cur.n; ++x) keep[x] = labels[x] >= nt;
        og_graph next;
        st = og_induced(&cur, keep, &next, map);
        free(keep);
        if (st) {
          free(map);
          goto done;
        }
        if (next.n == 0) {
          free(map);
          og_free(&next);
          st = fail(OG_E_INVARIANT, "re-pruning removed every vertex");
          goto done;
        }
        uint32_t* nl = (uint32_t*)malloc(next.n * sizeof(uint32_t));
        remap(labels, map, cur.n, nl);
        free(labels);
        labels = nl;
        uint64_t* nloads = (uint64_t*)calloc(next.n, sizeof(uint64_t));
        if (!cfg->reset_loads)
          for (uint64_t x = 0; x < cur.n; ++x)
            if (map[x] != 0xffffffffu) nloads[map[x]] = loads[x];
        free(loads);
        loads = nloads;
        free(map);
        og_free(&cur);
        cur = next;
        delta_cur = og_max_degree(&cur);
        thresh = nt;
      }
    }
  }
  {
    uint64_t gg = gcd64(be == 0 ? bv : be, bv);
    res->best_edges = be / gg;
    res->best_verts = bv / gg;
  }
  res->iterations = iterations;
  /* witness ascending (:156), recount on the input graph (:159-175) */
  radix_u64(wit, nwit);
  {
    uint8_t* in = (uint8_t*)calloc(g->n, 1);
    uint32_t* dense = (uint32_t*)malloc((nwit ? nwit : 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < nwit; ++i) {
      uint64_t p = lower_bound_u64(g->orig, g->n, wit[i]);
      if (p == g->n || g->orig[p] != wit[i]) {
        free(in), free(dense);
        st = fail(OG_E_INVARIANT, "witness vertex not in input graph");
        goto done;
      }
      in[p] = 1;
      dense[i] = (uint32_t)p;
    }
    uint64_t arcs = 0;
    for (uint64_t i = 0; i < nwit; ++i)
      for (uint64_t j = g->offs[dense[i]]; j < g->offs[dense[i] + 1]; ++j) arcs += in[g->adj[j]];
    res->witness_edges = arcs / 2;
    free(in), free(dense);
    if (!dens_eq(res->witness_edges, nwit, res->best_edges, res->best_verts)) {
      st = fail(OG_E_INVARIANT, "witness does not reproduce the reported density");
      goto done;
    }
  }
  res->witness_size = nwit;
  if (witness) memcpy(witness, wit, (nwit < witness_cap ? nwit : witness_cap) * sizeof(uint64_t));
  res->final_n = cur.n;
  if (final_ids)
    memcpy(final_ids, cur.orig, (cur.n < final_cap ? cur.n : final_cap) * sizeof(uint64_t));
done:
  free(loads), free(perm), free(wit), free(labels);
  og_free(&cur);
  return st;
}

/* ------------------------------------------------------------------ */
/* Seeded synthetic inputs.  Counter-based splitmix64 streams with       */
/* integer thresholds, so the device generators in                       */
/* paper_2311_04333_b200/csrc/gen.cu reproduce them bit for bit.          */
/* ------------------------------------------------------------------ */

/* RMAT quadrant thresholds on 32-bit draws: a=.57 b=.19 c=.19 d=.05 */
#define RMAT_TA 2448131358u
#define RMAT_TAB 3264175144u
#define RMAT_TABC 4080218930u

uint64_t og_gen_rmat(uint32_t scale, uint64_t samples, uint64_t seed, uint64_t* u, uint64_t* v) {
  const uint64_t sk = og_mix64(seed ^ 0x524d4154ULL);
  for (uint64_t k = 0; k < samples; ++k) {
    uint64_t a = 0, b = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      uint64_t r = og_mix64(sk ^ ((k << 5) | (l >> 1)));
      uint32_t d = (l & 1) ? (uint32_t)(r >> 32) : (uint32_t)r;
      uint32_t bu = d >= RMAT_TAB, bv = (d >= RMAT_TA && d < RMAT_TAB) || d >= RMAT_TABC;
      a = (a << 1) | bu;
      b = (b << 1) | bv;
    }
    u[k] = a;
    v[k] = b;
  }
  return samples;
}

/* G(n, p) of tests/test_util.hpp:67-79 (p = permille/1000) */
uint64_t og_gen_gnp(uint64_t n, uint64_t permille, uint64_t seed, uint64_t* u, uint64_t* v,
                    uint64_t cap) {
  uint64_t c = 0;
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = i + 1; j < n; ++j)
      if (og_mix64(seed ^ (i * 0x100000001b3ULL + j)) % 1000 < permille) {
        if (c < cap) {
          u[c] = i;
          v[c] = j;
        }
        ++c;
      }
  if (c == 0) {
    if (cap > 0) {
      u[0] = 0;
      v[0] = n > 1 ? 1 : 2;
    }
    c = 1;
  }
  return c;
}

/* Open-addressing set of canonical pairs (ER stream dedup). */
typedef struct {
  uint64_t* slot;
  uint64_t mask;
} pairset;
static int ps_insert(pairset* s, uint64_t key) { /* key != ~0 */
  uint64_t h = og_mix64(key) & s->mask;
  for (;;) {
    if (s->slot[h] == ~0ULL) {
      s->slot[h] = key;
      return 1;
    }
    if (s->slot[h] == key) return 0;
    h = (h + 1) & s->mask;
  }
}

/* ER + planted block (BASELINE config 1).  ER part: stream k draws
   r = mix64(se ^ k), u = hi-mult(lo32(r), n), v = hi-mult(hi32(r), n); loops
   are skipped and the first m_target distinct unordered pairs in stream order
   are kept.  Block: the first `block` distinct ids of the stream
   x_j = hi-mult(lo32(mix64(sb ^ j)), n); pair (a,b), a<b in block order, is
   present iff lo32(mix64(sb ^ (2^32 + a*block + b))) < 2^31 (p = 1/2).
   Output = ER pairs then block pairs (duplicates left to the CSR build). */
uint64_t og_gen_er_planted(uint64_t n, uint64_t m_target, uint64_t block, uint64_t seed,
                           uint64_t* u, uint64_t* v, uint64_t cap) {
  const uint64_t se = og_mix64(seed ^ 0x4552ULL), sb = og_mix64(seed ^ 0x424cULL);
  uint64_t sz = 1;
  while (sz < 2 * m_target + 16) sz <<= 1;
  pairset s = {(uint64_t*)malloc(sz * sizeof(uint64_t)), sz - 1};
  if (!s.slot) return 0;
  memset(s.slot, 0xff, sz * sizeof(uint64_t));
  uint64_t c = 0;
  for (uint64_t k = 0; c < m_target; ++k) {
    uint64_t r = og_mix64(se ^ k);
    uint64_t a = ((r & 0xffffffffULL) * n) >> 32, b = ((r >> 32) * n) >> 32;
    if (a == b) continue;
    uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
    if (ps_insert(&s, (lo << 32) | hi)) {
      if (c < cap) {
        u[c] = lo;
        v[c] = hi;
      }
      ++c;
    }
  }
  free(s.slot);
  uint64_t* ids = (uint64_t*)malloc((block ? block : 1) * sizeof(uint64_t));
  uint64_t nb = 0;
  for (uint64_t j = 0; nb < block; ++j) {
    uint64_t x = ((og_mix64(sb ^ j) & 0xffffffffULL) * n) >> 32;
    int dup = 0;
    for (uint64_t q = 0; q < nb; ++q) dup |= ids[q] == x;
    if (!dup) ids[nb++] = x;
  }
  for (uint64_t a = 0; a < block; ++a)
    for (uint64_t b = a + 1; b < block; ++b)
      if ((og_mix64(sb ^ ((1ULL << 32) + a * block + b)) & 0xffffffffULL) < (1ULL << 31)) {
        if (c < cap) {
          u[c] = ids[a];
          v[c] = ids[b];
        }
        ++c;
      }
  free(ids);
  return c;
}

/* Chung-Lu power law (BASELINE config 3).  Endpoint draw from r:
   x = (r >> 11) * 2^-53, y = 1 + x * (R - 1), z = y^11 by exact-order
   products, id = min(floor(z) - 1, n - 1).  With R = n^(1/11) this gives
   P(id = i) ~ (i+1)^(-10/11): degree exponent 1 + 11/10 = 2.1, mean degree
   2 * pairs / n.  Only IEEE-exact + and * are used (compile with
   -ffp-contract=off; the device side uses __dmul_rn/__dadd_rn). */
static uint64_t cl_endpoint(uint64_t r, double R, uint64_t n) {
  volatile double x = (double)(r >> 11) * (1.0 / 9007199254740992.0);
  volatile double t = x * (R - 1.0);
  volatile double y = 1.0 + t;
  volatile double y2 = y * y;
  volatile double y4 = y2 * y2;
  volatile double y8 = y4 * y4;
  volatile double y10 = y8 * y2;
  volatile double z = y10 * y;
  uint64_t id = (uint64_t)z;
  id = id >= 1 ? id - 1 : 0;
  return id < n ? id : n - 1;
}
uint64_t og_gen_chung_lu(uint64_t n, uint64_t pairs, double n_root11, uint64_t seed, uint64_t* u,
                         uint64_t* v) {
  const uint64_t sc = og_mix64(seed ^ 0x434cULL);
  for (uint64_t k = 0; k < pairs; ++k) {
    u[k] = cl_endpoint(og_mix64(sc ^ (2 * k)), n_root11, n);
    v[k] = cl_endpoint(og_mix64(sc ^ (2 * k + 1)), n_root11, n);
  }
  return pairs;
}
