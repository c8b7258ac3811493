/*
 * og_par.c -- CPU INPUT PREPARATION FOR THE REFERENCE ARM (TEST INFRASTRUCTURE).
 *
 * Builds the seeded RMAT graph of bench.py's configs directly as a CSR on the
 * host with OpenMP, so `bench.py --impl reference` can hand the UNMODIFIED
 * reference library (oracle/_ref) a graph at RMAT-26 size (1.07e9 samples)
 * in seconds instead of the minutes the sequential oracle build needs.  It is
 * NOT the measured path (the reference's exact_coreness / run() are) and the
 * product never loads it.
 *
 * Semantics are the reference's CSR build (io.cpp:51-92) on the samples of
 * og_gen_rmat (dg_oracle.c): canonical pairs, self-loops dropped, duplicates
 * removed, dense id = rank of the original id among vertices with >= 1 edge,
 * rows ascending.  Method: both arc directions of every non-loop sample as
 * (src << scale | dst) keys, parallel LSD radix sort, unique -> the keys ARE
 * the CSR rows in order; dense ids by a prefix count over the sources.
 * Checked equal to og_build (tests/test_oracle_golden.py).
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "dg_oracle.h"

#define RMAT_TA 2448131358u
#define RMAT_TAB 3264175144u
#define RMAT_TABC 4080218930u

static inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* parallel LSD radix sort on the low `bits` bits, 11-bit digits */
static int psort(uint64_t* a, uint64_t n, int bits, int nt) {
  enum { D = 11, R = 1 << D };
  uint64_t* tmp = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  uint64_t* cnt = (uint64_t*)malloc((size_t)nt * R * sizeof(uint64_t));
  if (!tmp || !cnt) {
    free(tmp);
    free(cnt);
    return -1;
  }
  uint64_t *src = a, *dst = tmp;
  for (int sh = 0; sh < bits; sh += D) {
#pragma omp parallel num_threads(nt)
    {
      int t = omp_get_thread_num(), T = omp_get_num_threads();
      uint64_t lo = n * t / T, hi = n * (t + 1) / T;
      uint64_t* c = cnt + (size_t)t * R;
      memset(c, 0, R * sizeof(uint64_t));
      for (uint64_t i = lo; i < hi; ++i) c[(src[i] >> sh) & (R - 1)]++;
#pragma omp barrier
#pragma omp single
      {
        uint64_t s = 0;
        for (int d = 0; d < R; ++d)
          for (int q = 0; q < T; ++q) {
            uint64_t x = cnt[(size_t)q * R + d];
            cnt[(size_t)q * R + d] = s;
            s += x;
          }
      }
      for (uint64_t i = lo; i < hi; ++i) dst[c[(src[i] >> sh) & (R - 1)]++] = src[i];
    }
    uint64_t* x = src;
    src = dst;
    dst = x;
  }
  if (src != a) memcpy(a, src, n * sizeof(uint64_t));
  free(tmp);
  free(cnt);
  return 0;
}

int ogp_rmat_graph(uint32_t scale, uint64_t samples, uint64_t seed, int threads, og_graph* out) {
  memset(out, 0, sizeof *out);
  if (scale < 1 || scale > 31) return OG_E_PARAM;
  int nt = threads > 0 ? threads : omp_get_max_threads();
  const uint64_t sk = mix64(seed ^ 0x524d4154ULL);
  const uint64_t nid = 1ULL << scale, mask = nid - 1;
  uint64_t* key = (uint64_t*)malloc((samples ? 2 * samples : 1) * sizeof(uint64_t));
  uint64_t* tc = (uint64_t*)calloc((size_t)nt + 1, sizeof(uint64_t));
  if (!key || !tc) {
    free(key);
    free(tc);
    return OG_E_NOMEM;
  }
  /* samples -> arc keys, compacted per thread block (loops dropped) */
#pragma omp parallel num_threads(nt)
  {
    int t = omp_get_thread_num(), T = omp_get_num_threads();
    uint64_t lo = samples * t / T, hi = samples * (t + 1) / T, c = 2 * lo;
    for (uint64_t k = lo; k < hi; ++k) {
      uint64_t a = 0, b = 0;
      uint64_t r = 0;
      for (uint32_t l = 0; l < scale; ++l) {
        if (!(l & 1)) r = mix64(sk ^ ((k << 5) | (l >> 1))); /* one draw per 2 levels */
        uint32_t d = (l & 1) ? (uint32_t)(r >> 32) : (uint32_t)r;
        uint32_t bu = d >= RMAT_TAB, bv = (d >= RMAT_TA && d < RMAT_TAB) || d >= RMAT_TABC;
        a = (a << 1) | bu;
        b = (b << 1) | bv;
      }
      if (a == b) continue;
      key[c++] = (a << scale) | b;
      key[c++] = (b << scale) | a;
    }
    tc[t + 1] = c - 2 * lo;
#pragma omp barrier
#pragma omp single
    for (int q = 0; q < T; ++q) tc[q + 1] += tc[q];
    /* close the gaps left by loops (blocks move left only, in order) */
#pragma omp single
    for (int q = 1; q < T; ++q) {
      uint64_t from = 2 * (samples * q / T);
      if (from != tc[q]) memmove(key + tc[q], key + from, (tc[q + 1] - tc[q]) * sizeof(uint64_t));
    }
  }
  uint64_t arcs = tc[nt];
  free(tc);
  if (psort(key, arcs, 2 * (int)scale, nt)) {
    free(key);
    return OG_E_NOMEM;
  }
  /* unique: per-thread counts of run starts, prefix, then each thread writes
   its unique arcs' raw targets and counts their sources (atomics only meet
   at chunk boundaries) */
  uint64_t* uc = (uint64_t*)calloc((size_t)nt + 1, sizeof(uint64_t));
  uint32_t* rank = (uint32_t*)calloc(nid, sizeof(uint32_t));
  uint64_t* deg = (uint64_t*)calloc(nid, sizeof(uint64_t));
  uint32_t* adj = (uint32_t*)malloc((arcs ? arcs : 1) * sizeof(uint32_t));
  if (!uc || !rank || !deg || !adj) {
    free(key);
    free(uc);
    free(rank);
    free(deg);
    free(adj);
    return OG_E_NOMEM;
  }
#pragma omp parallel num_threads(nt)
  {
    int t = omp_get_thread_num(), T = omp_get_num_threads();
    uint64_t lo = arcs * t / T, hi = arcs * (t + 1) / T, c = 0;
    for (uint64_t i = lo; i < hi; ++i) c += (i == 0 || key[i] != key[i - 1]);
    uc[t + 1] = c;
#pragma omp barrier
#pragma omp single
    for (int q = 0; q < T; ++q) uc[q + 1] += uc[q];
    uint64_t p = uc[t];
    for (uint64_t i = lo; i < hi; ++i)
      if (i == 0 || key[i] != key[i - 1]) {
        adj[p++] = (uint32_t)(key[i] & mask);
        uint64_t x = key[i] >> scale;
        if (i == lo || i + 1 == hi) {
#pragma omp atomic
          deg[x]++;
        } else {
          deg[x]++;
        }
      }
  }
  uint64_t u = uc[nt];
  free(uc);
  free(key);
  if (u == 0) {
    free(rank);
    free(deg);
    free(adj);
    return OG_E_EMPTY;
  }
  /* presence -> rank; sources are exactly the vertices with >= 1 edge */
  uint64_t n = 0;
  for (uint64_t x = 0; x < nid; ++x)
    if (deg[x]) rank[x] = (uint32_t)n++;
  out->n = n;
  out->m = u / 2;
  out->offs = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  out->adj = adj; /* u <= arcs entries used */
  out->orig = (uint64_t*)malloc(n * sizeof(uint64_t));
  if (!out->offs || !out->orig) {
    free(rank);
    free(deg);
    og_free(out);
    return OG_E_NOMEM;
  }
  uint64_t s = 0, r = 0;
  for (uint64_t x = 0; x < nid; ++x)
    if (deg[x]) {
      out->offs[r] = s;
      out->orig[r] = x;
      s += deg[x];
      ++r;
    }
  out->offs[n] = s;
#pragma omp parallel for num_threads(nt) schedule(static)
  for (uint64_t i = 0; i < u; ++i) out->adj[i] = rank[out->adj[i]];
  free(rank);
  free(deg);
  return OG_OK;
}
