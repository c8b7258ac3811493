/*
 * dg_oracle.h -- CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * A plain sequential C restatement of the reference's hot path
 * (densegraph, /root/reference/proj): CSR build, exact / approximate
 * coreness, induced-subgraph compaction, Greedy++ min-key batch peel,
 * Algorithm 3 (density + load update), the sampled slack audit and the
 * prune-and-refine driver `run`.  Every function cites the reference
 * file:line it restates.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker.
 * The product (paper_2311_04333_b200/) never links or calls it.
 *
 * Pinning: tests/test_oracle_golden.py checks this restatement against
 * the known-answer vectors of the reference's own unit tests and against
 * fixtures produced by the real reference library (oracle/_ref, built from
 * /root/reference/proj/src by oracle/Makefile; generator script
 * tests/golden/make_golden.py).
 */
#ifndef DG_ORACLE_H
#define DG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: same numbering as include/dg_b200.h */
enum {
  OG_OK = 0,
  OG_E_PARSE = 1,
  OG_E_EMPTY = 2,
  OG_E_IO = 3,
  OG_E_PARAM = 4,
  OG_E_INVARIANT = 5,
  OG_E_NOMEM = 8
};

typedef struct {
  uint64_t n, m;
  uint64_t* offs; /* n + 1 */
  uint32_t* adj;  /* 2m */
  uint64_t* orig; /* n */
} og_graph;

typedef struct {
  uint64_t rho_edges, rho_verts; /* unreduced */
  uint64_t best_prefix;
  uint64_t width;
} og_outcome;

typedef struct {
  int algorithm;        /* 0 peel, 1 sort */
  int pruning;          /* 0 none, 1 exact, 2 approx, 3 hybrid */
  uint64_t iterations;  /* 0 -> epsilon */
  double epsilon;
  uint64_t iteration_cap;
  uint64_t c_num, c_den;
  int reset_loads;
  uint64_t slack_samples;
} og_config;

typedef struct {
  uint64_t iter, rho_edges, rho_verts, n, m, width;
} og_iter;

typedef struct {
  uint64_t best_edges, best_verts; /* reduced */
  uint64_t witness_size, witness_edges, iterations, max_width;
  uint64_t slack_violations;
  int kmax_known, kmax_exact;
  uint32_t kmax, threshold;
  uint64_t pruned_n, pruned_m;
  uint64_t final_n;
} og_result;

const char* og_last_error(void);

uint64_t og_mix64(uint64_t x);

/* ---- graph ---- */
int og_build(const uint64_t* u, const uint64_t* v, uint64_t k, og_graph* out);
int og_from_csr(uint64_t n, const uint64_t* offs, const uint32_t* adj, const uint64_t* orig,
                og_graph* out);
void og_free(og_graph* g);
uint64_t og_max_degree(const og_graph* g);
int og_induced(const og_graph* g, const uint8_t* keep, og_graph* out, uint32_t* old_to_new);

/* ---- coreness ---- */
int og_coreness(const og_graph* g, int approx, uint64_t c_num, uint64_t c_den, uint32_t* labels,
                uint32_t* kmax, uint32_t* peel_rounds);

/* ---- refinement ---- */
int og_peel_order(const og_graph* g, const uint64_t* loads, int one_at_a_time, uint32_t* perm);
int og_sort_order(uint64_t n, const uint64_t* loads, uint32_t* perm);
int og_density_update(const og_graph* g, const uint32_t* perm, uint64_t* loads, og_outcome* out,
                      uint32_t* charges_out, uint64_t* suffix_edges_out);
uint64_t og_slack_violations(uint64_t n, const uint32_t* perm, const uint64_t* loads,
                             uint64_t allowed_slack, uint64_t samples, uint64_t seed);
uint64_t og_default_iterations(uint64_t delta, double lower_bound, uint64_t n, double epsilon,
                               uint64_t cap, int* status);

/* ---- framework ---- */
int og_run(const og_graph* g, const og_config* cfg, og_result* res, og_iter* trace,
           uint64_t trace_cap, uint64_t* witness, uint64_t witness_cap, uint64_t* final_ids,
           uint64_t final_cap);

/* ---- seeded synthetic inputs (bit-identical to the device generators) ---- */
uint64_t og_gen_rmat(uint32_t scale, uint64_t samples, uint64_t seed, uint64_t* u, uint64_t* v);
uint64_t og_gen_gnp(uint64_t n, uint64_t permille, uint64_t seed, uint64_t* u, uint64_t* v,
                    uint64_t cap);
uint64_t og_gen_er_planted(uint64_t n, uint64_t m_target, uint64_t block, uint64_t seed,
                           uint64_t* u, uint64_t* v, uint64_t cap);
uint64_t og_gen_chung_lu(uint64_t n, uint64_t pairs, double n_root11, uint64_t seed,
                         uint64_t* u, uint64_t* v);

#ifdef __cplusplus
}
#endif
#endif
