/*
 * dg_b200.h -- C ABI of the B200-native densegraph hot path.
 *
 * The reference (densegraph, arXiv 2311.04333 artifact) exposes its hot path
 * as a C++ library API (proj/include/densegraph/*.hpp).  This header is the
 * drop-in boundary underneath that API: plain pointers and sizes, no C++ or
 * torch types, status codes instead of exceptions.  include/densegraph/*.hpp
 * re-creates the reference's C++ API on top of it, so reference callers
 * (its CLI and tests) compile unchanged; INTEGRATION.md shows the binding.
 *
 * Every call is externally synchronous (returns finished results), like the
 * reference.  The library owns all device memory behind dg_graph handles;
 * callers own host buffers, sized from dg_graph_info.  Unless a parameter
 * says "device", pointers are host pointers.  Handles are immutable.
 *
 * There is no CPU fallback: every computing entry point runs sm_100a CUDA
 * kernels, and returns DG_E_CUDA when no usable device is present.
 */
#ifndef DG_B200_H
#define DG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes map 1:1 onto the reference's exception types
 * (proj/include/densegraph/errors.hpp:10-42). */
typedef enum {
  DG_OK = 0,
  DG_E_PARSE = 1,        /* ParseError        errors.hpp:10-15 */
  DG_E_EMPTY = 2,        /* EmptyGraphError   errors.hpp:17-19 */
  DG_E_IO = 3,           /* IoError           errors.hpp:21-23 */
  DG_E_PARAM = 4,        /* ParamError        errors.hpp:25-27 */
  DG_E_INVARIANT = 5,    /* InvariantError    errors.hpp:30-32 */
  DG_E_ORACLE_SIZE = 6,  /* OracleSizeError   errors.hpp:35-37 */
  DG_E_CACHE_HASH = 7,   /* CacheHashError    errors.hpp:40-42 */
  DG_E_NOMEM = 8,        /* device/host allocation failure (-> InvariantError, CLI exit 4) */
  DG_E_CUDA = 9          /* CUDA runtime failure / no device (-> InvariantError) */
} dg_status;

typedef struct dg_graph dg_graph; /* device-resident CSR, graph.hpp:24-45 layout */

/* Thread-local message of the last failing call on this thread. */
const char* dg_last_error(void);
/* Library version string, e.g. "densegraph-b200 0.1 sm_100a". */
const char* dg_version(void);

/* ------------------------------------------------------------ graph / CSR */

/* CSR build with the reference's cleanup semantics: canonical (min,max)
 * pairs, self-loops dropped, duplicates collapsed, dense ids = rank of the
 * original id among ids that occur in a non-loop edge, rows ascending.
 * Replaces the CSR-build half of parse_edge_list (io.hpp:18, io.cpp:51-92).
 * `on_device` != 0: u, v are device pointers (e.g. from dg_gen_rmat).
 * DG_E_EMPTY if no edge survives (io.cpp:58). */
dg_status dg_graph_build(const uint64_t* u, const uint64_t* v, uint64_t k, int on_device,
                         dg_graph** out);

/* Wrap an existing CSR (Graph{n,m,offs,adj,orig}, graph.hpp:24-30). Copies
 * host arrays (on_device == 0) or device arrays (on_device != 0). */
/* The CSR of a seeded synthetic graph built straight from the device
 * generator (no pair arrays; source-range parts so the largest BASELINE
 * configuration, RMAT-28, builds on one GPU).  Identical to dg_graph_build on
 * the pairs of dg_gen_rmat / dg_gen_chung_lu.  kind 0: RMAT (size = scale),
 * 1: Chung-Lu (size = n, root = n^(1/11)); part_cap = max arc emissions per
 * part (0: from free memory). */
dg_status dg_graph_generate(int kind, uint64_t size, uint64_t samples, uint64_t seed,
                            double root, uint64_t part_cap, dg_graph** out);
/* parse_edge_list(istream&, ParseOptions) (io.hpp:18-19, io.cpp:25-94): edge-
 * list text (len bytes, host or device memory) tokenised ON THE DEVICE with
 * the reference's rules, then the CSR build of dg_graph_build.  Malformed
 * input returns DG_E_PARSE with *bad_line = the 1-based number of the first
 * malformed line (the caller formats ParseError's message with its text);
 * no edge left returns DG_E_EMPTY. */
dg_status dg_parse_edge_list(const char* text, uint64_t len, char comment, int on_device,
                             dg_graph** out, uint64_t* bad_line);
dg_status dg_graph_from_csr(uint64_t n, const uint64_t* offs, const uint32_t* adj,
                            const uint64_t* orig, int on_device, dg_graph** out);

/* GraphStats (graph.hpp:14-18,37-42). */
dg_status dg_graph_info(const dg_graph* g, uint64_t* n, uint64_t* m, uint64_t* max_degree);

/* Copy the CSR to host buffers of sizes n+1, 2m, n (any may be NULL). */
dg_status dg_graph_download(const dg_graph* g, uint64_t* offs, uint32_t* adj, uint64_t* orig);

/* Device pointers of the CSR (valid until dg_graph_free). */
dg_status dg_graph_device_ptrs(const dg_graph* g, const uint64_t** offs, const uint32_t** adj,
                               const uint64_t** orig);

void dg_graph_free(dg_graph* g);

/* induced_subgraph(g, keep, &old_to_new)  (graph.hpp:50-80).
 * keep: n bytes (host), old_to_new: n entries (host, nullable). */
dg_status dg_induced(const dg_graph* g, const uint8_t* keep, dg_graph** out,
                     uint32_t* old_to_new);

/* get_core(g, dec, k, &old_to_new)  (core.hpp:31-32, core.cpp:133-140):
 * subgraph induced by labels >= k.  labels: n entries (host). */
dg_status dg_get_core(const dg_graph* g, const uint32_t* labels, uint32_t k, dg_graph** out,
                      uint32_t* old_to_new);

/* ------------------------------------------------------------ coreness */

/* exact_coreness (core.hpp:22, core.cpp:123-125) when approx == 0;
 * approx_coreness(g, c_num, c_den) (core.hpp:28, core.cpp:127-131) otherwise.
 * labels: n entries (host, nullable).  DG_E_EMPTY on n == 0,
 * DG_E_PARAM on c_num/c_den <= 1 (approx). */
dg_status dg_coreness(const dg_graph* g, int approx, uint64_t c_num, uint64_t c_den,
                      uint32_t* labels, uint32_t* kmax, uint32_t* peel_rounds);

/* ------------------------------------------------------------ refinement */

typedef struct {
  uint64_t rho_edges, rho_verts; /* RefineOutcome::rho_max, unreduced (refine.hpp:21) */
  uint64_t best_prefix;          /* refine.hpp:22 */
  uint64_t width;                /* refine.hpp:23 */
} dg_outcome;

/* load_peel_order(g, {loads}, one_at_a_time) (refine.hpp:32, refine.cpp:149-156):
 * min-key batch peel on key = load + residual degree.  perm: n entries. */
dg_status dg_peel_order(const dg_graph* g, const uint64_t* loads, int one_at_a_time,
                        uint32_t* perm);

/* load_sort_order({loads}) (refine.hpp:35, refine.cpp:158-178): stable sort by (load, id). */
dg_status dg_sort_order(uint64_t n, const uint64_t* loads, uint32_t* perm);

/* density_and_load_update(g, order, state, want_densities) (refine.hpp:40-41,
 * refine.cpp:180-220).  loads updated in place.  suffix_edges (nullable,
 * n entries): the per-position densities' numerators (denominator n - i).
 * DG_E_INVARIANT if perm is not a permutation (refine.cpp:186-192). */
dg_status dg_density_load_update(const dg_graph* g, const uint32_t* perm, uint64_t* loads,
                                 dg_outcome* out, uint64_t* suffix_edges);

/* charikar_peel (refine.hpp:44, refine.cpp:222-227). */
dg_status dg_charikar_peel(const dg_graph* g, dg_outcome* out);

/* slack_violations (refine.hpp:48-49, refine.cpp:229-242). */
dg_status dg_slack_violations(uint64_t n, const uint32_t* perm, const uint64_t* loads,
                              uint64_t allowed_slack, uint64_t samples, uint64_t seed,
                              uint64_t* violations);

/* default_iterations (framework.hpp:63, framework.cpp:36-44). Host scalar math. */
dg_status dg_default_iterations(uint64_t delta, double lower_bound, uint64_t n, double epsilon,
                                uint64_t cap, uint64_t* out);

/* ------------------------------------------------------------ framework */

typedef struct { /* RunConfig, framework.hpp:15-25 (threads has no meaning here) */
  int algorithm;         /* 0 peel (Greedy++), 1 sort (GreedySorting++) */
  int pruning;           /* 0 none, 1 exact, 2 approx, 3 hybrid */
  uint64_t iterations;   /* explicit T; 0 defers to epsilon */
  double epsilon;
  uint64_t iteration_cap;
  uint64_t c_num, c_den;
  int reset_loads;
  uint64_t slack_samples;
} dg_run_config;

typedef struct { /* IterRecord (framework.hpp:27-33) + device timings */
  uint64_t iter, rho_edges, rho_verts, n, m, width;
  double ms;          /* ordering + audit + Alg. 3, CUDA events */
  double order_ms;    /* ordering kernel alone */
  double update_ms;   /* Alg. 3 kernels alone */
  uint64_t batches;   /* Greedy++ batches in this ordering (0 for sort) */
} dg_iter_record;

typedef struct { /* RunResult + RunTrace/InitRecord (framework.hpp:35-60) */
  uint64_t best_edges, best_verts; /* reduced */
  uint64_t witness_size, witness_edges, iterations, max_width;
  uint64_t slack_violations;
  int kmax_known, kmax_exact;
  uint32_t kmax, threshold;
  uint64_t pruned_n, pruned_m;
  uint64_t final_n;
  uint32_t peel_rounds;  /* of the (first) coreness pass */
  uint32_t reprunes;
  double coreness_ms;    /* InitRecord::coreness_ms: coreness + get_core + remap */
  double coreness_kernel_ms; /* the k-core kernel alone */
  double init_ms, total_ms;
  double reprune_ms;     /* all mid-run re-prune compactions */
  double device_ms;      /* CUDA-event span of the whole run on the library stream */
} dg_run_result;

/* run(g, cfg) (framework.hpp:68, framework.cpp:46-180): Algorithm 1 on the
 * device; only scalars cross PCIe per iteration.  trace: trace_cap records;
 * witness: original ids ascending (witness_cap); final_ids: original ids of
 * the last pruned graph (final_cap).  Any of the arrays may be NULL. */
dg_status dg_run(const dg_graph* g, const dg_run_config* cfg, dg_run_result* res,
                 dg_iter_record* trace, uint64_t trace_cap, uint64_t* witness,
                 uint64_t witness_cap, uint64_t* final_ids, uint64_t final_cap);

/* run() continued after a first prune done elsewhere (framework.cpp:92-180):
 * `core` = get_core(input, labels, threshold) where threshold follows from
 * kmax and cfg->pruning as in framework.cpp:62-79, core_labels (host, core->n)
 * are the coreness labels of the core's vertices, peel_rounds those of the
 * coreness pass.  Produced by the sharded pipeline (sharded coreness +
 * per-shard compaction, one gather); identical result to dg_run on the input
 * graph (the witness recount on the core equals the one on the input: the
 * core is an induced subgraph containing the witness).  pruning 3 (hybrid)
 * runs its exact pass on the core here.  DG_E_INVARIANT if a label is below
 * the threshold, DG_E_PARAM for pruning 0. */
dg_status dg_run_pruned(const dg_graph* core, const uint32_t* core_labels, uint32_t kmax,
                        uint32_t peel_rounds, const dg_run_config* cfg, dg_run_result* res,
                        dg_iter_record* trace, uint64_t trace_cap, uint64_t* witness,
                        uint64_t witness_cap, uint64_t* final_ids, uint64_t final_cap);

/* ------------------------------------------------------------ sharded coreness */

/* One GPU's shard of a 1D vertex-range-partitioned exact coreness
 * (same rounds and labels as exact_coreness, core.cpp:89-119).
 * Rank `rank` of P owns dense ids [bounds[rank], bounds[rank+1]).  Per round:
 * dg_shard_count_remote -> exchange counts -> dg_shard_expand (local
 * decrements + remote ids bucketed by owner into a device send buffer at the
 * given per-rank displacements) -> all-to-all -> dg_shard_apply (received
 * decrements) -> all-reduce of the next frontier sizes; when the global
 * frontier is empty: dg_shard_min_alive -> all-reduce(min) -> dg_shard_collect.
 * The protocol is paper_2311_04333_b200/sharded.py. */
typedef struct dg_shard dg_shard;
dg_status dg_shard_create(const dg_graph* g, const uint64_t* bounds, uint32_t P, uint32_t rank,
                          dg_shard** out);
/* The same shard from the rank's own rows only (memory-scaled: a rank never
 * holds the whole graph): offs = the n_local + 1 row offsets of [lo, hi)
 * (absolute or rebased), adj = their arcs as global dense ids. */
dg_status dg_shard_create_rows(uint64_t n, const uint64_t* bounds, uint32_t P, uint32_t rank,
                               const uint64_t* offs, const uint32_t* adj, int on_device,
                               dg_shard** out);
void dg_shard_free(dg_shard* s);
dg_status dg_shard_min_alive(dg_shard* s, uint32_t* min_degree);  /* UINT32_MAX if none */
dg_status dg_shard_collect(dg_shard* s, uint32_t bound, uint32_t label, uint64_t* nfront);
dg_status dg_shard_count_remote(dg_shard* s, uint64_t* counts /* P entries */);
dg_status dg_shard_expand(dg_shard* s, uint32_t bound, uint32_t label, const uint64_t* displs,
                          uint32_t* d_send /* device */);
dg_status dg_shard_apply(dg_shard* s, const uint32_t* d_recv /* device */, uint64_t nrecv,
                         uint32_t bound, uint32_t label, uint64_t* nnext);
dg_status dg_shard_labels(const dg_shard* s, uint32_t* labels /* hi - lo entries */);

/* Peer mode: the fused form of the round above.  Each shard's decrement
 * targets (degrees, labels, two frontier queues + counters) live in one
 * device allocation that every other rank maps -- by CUDA IPC
 * (dg_shard_ipc_handle on the owner, dg_shard_peer_open on the others: NVLink
 * peer memory on one node) or directly for shards of one process
 * (dg_shard_peer_link).  dg_shard_expand_peer then decrements every
 * neighbour AT ITS OWNER with system-scope atomics and appends crossings to
 * the owner's next queue, returning how many crossings this shard produced;
 * after an all-reduce of those counts (the round barrier) dg_shard_finish_round
 * makes the owner's queue its frontier.  Level advances are unchanged
 * (dg_shard_min_alive / dg_shard_collect).  Every rank must be opened or
 * linked (its own entry is implicit); at most 64 shards. */
dg_status dg_shard_ipc_handle(const dg_shard* s, void* handle /* 64 bytes out */);
dg_status dg_shard_peer_open(dg_shard* s, uint32_t rank, const void* handle /* 64 bytes */);
dg_status dg_shard_peer_link(dg_shard* s, uint32_t rank, const dg_shard* other);
dg_status dg_shard_expand_peer(dg_shard* s, uint32_t bound, uint32_t label, uint64_t* produced);
dg_status dg_shard_finish_round(dg_shard* s, uint64_t* nnext);
/* Distributed CSR build and per-shard get_core, the per-rank device steps
 * (the caller moves buffers between ranks with its collectives; see
 * paper_2311_04333_b200/sharded_build.py).  All array arguments are DEVICE
 * pointers except `id_bounds`, `counts` and `hist` (host).  Original ids must
 * be below 2^32.
 *   max_id        largest endpoint of a non-loop pair (0: none)
 *   endpoint_hist histogram of non-loop endpoints >> shift (nb <= 4096)
 *   route         both arc directions of every non-loop pair as (src << 32 |
 *                 dst) keys, grouped by the owner of src (original-id ranges
 *                 [id_bounds[r], id_bounds[r+1])); counts[r] keys per owner
 *   rows          received keys (sorted in place) -> unique -> rows: offs
 *                 (nverts + 1), distinct sources `verts`, neighbour ids `dst`
 *   unique        distinct values (ascending) and each entry's index into them
 *   lookup        dense ids of asked original ids: base + position in verts
 *   bucket_counts entries of ascending `vals` per owner range (host counts)
 *   take          out[map[i] - base] = in[i] for kept i (4- or 8-byte elements)
 *   relabel       adj[i] = back[inv[i]]
 *   keep_map      map[i] = base + rank among labels >= k, UINT32_MAX if dropped
 *   core_rows     rows of kept vertices, neighbours renamed through full_map
 *                 (global old id -> new id), dropped ones removed in order */
dg_status dg_dist_max_id(const uint64_t* u, const uint64_t* v, uint64_t k, uint64_t* out);
dg_status dg_dist_endpoint_hist(const uint64_t* u, const uint64_t* v, uint64_t k, uint32_t shift,
                                uint32_t nb, uint64_t* hist);
dg_status dg_dist_route(const uint64_t* u, const uint64_t* v, uint64_t k,
                        const uint64_t* id_bounds, uint32_t P, uint64_t* keys, uint64_t* counts);
dg_status dg_dist_rows(uint64_t* keys, uint64_t n, uint64_t* offs, uint64_t* verts,
                       uint32_t* dst, uint64_t* nverts, uint64_t* narcs);
dg_status dg_dist_unique(const uint32_t* vals, uint64_t n, uint32_t* uniq, uint32_t* inv,
                         uint64_t* nuniq);
dg_status dg_dist_lookup(const uint64_t* verts, uint64_t nv, const uint32_t* asked, uint64_t na,
                         uint64_t base, uint32_t* out);
dg_status dg_dist_bucket_counts(const uint32_t* vals, uint64_t n, const uint64_t* id_bounds,
                                uint32_t P, uint64_t* counts);
dg_status dg_dist_take(const void* in, const uint32_t* map, uint64_t nl, uint64_t base,
                       uint32_t elem_bytes, void* out);
dg_status dg_dist_relabel(const uint32_t* back, const uint32_t* inv, uint64_t n, uint32_t* adj);
dg_status dg_dist_keep_map(const uint32_t* labels, uint64_t nl, uint32_t k, uint64_t base,
                           uint32_t* map, uint64_t* kept);
dg_status dg_dist_core_rows(const uint64_t* offs, const uint32_t* adj, uint64_t nl,
                            const uint32_t* local_map, const uint32_t* full_map,
                            uint64_t* noffs, uint32_t* nadj, uint64_t* nkept, uint64_t* narcs);

/* Device-resident round loop: the whole sharded coreness as one
 * persistent cooperative kernel per GPU.  `shards` are the shards THIS
 * process holds (count = 1 per GPU on a multi-GPU job; any count on one GPU,
 * each served by its own group of CTAs); every shard must be linked or opened
 * to every other (peer mode) and all P shards must enter this call (one
 * process per GPU: every rank calls it with its shard).  Rounds are separated
 * by a flip barrier in shard 0's control block with system-scope atomics
 * (NVLink peer memory across GPUs); remote decrements are atomicSub_system at
 * the owner and a crossing appends the vertex to the owner's queue.  The
 * caller resets shard 0's control block first (dg_shard_xctrl_reset, on the
 * process holding shard 0) and makes every rank wait for that reset (e.g. a
 * collective) before entering.  Labels are read with dg_shard_labels;
 * kernel_ms (optional) is the launch's device time. */
dg_status dg_shard_xctrl_reset(dg_shard* shard0);
dg_status dg_shard_coreness_persistent(dg_shard** shards, uint32_t count, int approx,
                                       uint64_t c_num, uint64_t c_den, uint32_t* kmax,
                                       uint32_t* peel_rounds, float* kernel_ms);

/* ------------------------------------------------------------ synthetic inputs */

/* Seeded counter-based generators (bit-identical to oracle/dg_oracle.c).
 * Outputs are device buffers allocated with dg_device_alloc when
 * on_device != 0, else host buffers of `samples` / `pairs` entries. */
dg_status dg_gen_rmat(uint32_t scale, uint64_t samples, uint64_t seed, uint64_t* u, uint64_t* v,
                      int on_device);
/* Samples [first, first + count) of the same RMAT stream (a rank's slice of
 * a distributed input); u, v receive `count` entries. */
dg_status dg_gen_rmat_range(uint32_t scale, uint64_t first, uint64_t count, uint64_t seed,
                            uint64_t* u, uint64_t* v, int on_device);
dg_status dg_gen_chung_lu(uint64_t n, uint64_t pairs, double n_root11, uint64_t seed,
                          uint64_t* u, uint64_t* v, int on_device);

/* Exhaustive densest subgraph over all nonempty vertex subsets (the
 * reference's test oracle, oracle.hpp:16-19 / oracle.cpp:70-108), on the
 * device.  Ties: fewer vertices, then the lexicographically smallest id set.
 * Outputs the reduced density and the witness as ORIGINAL ids, ascending
 * (`witness` may be null; it needs room for n ids).  DG_E_EMPTY on n = 0,
 * DG_E_ORACLE_SIZE when n > limit (or n > 32). */
dg_status dg_brute_force_densest(const dg_graph* g, uint32_t limit, uint64_t* edges,
                                 uint64_t* verts, uint64_t* witness, uint64_t* witness_n);

/* Device memory helpers for callers that keep inputs resident in HBM. */
dg_status dg_device_alloc(uint64_t bytes, void** ptr);
dg_status dg_device_free(void* ptr);
dg_status dg_memcpy(void* dst, const void* src, uint64_t bytes, int kind /* 1 h2d, 2 d2h, 3 d2d */);
dg_status dg_synchronize(void);

/* Select the CUDA device for this thread's subsequent calls (one process per GPU). */
dg_status dg_set_device(int device);
/* Diagnostics (latency microbenchmarks, instrumented-kernel read-outs) live
 * in a separate library, libdg_b200_diag.so (include/dg_b200_diag.h). */
/* Number of this library's own kernels launched so far in this process. */
uint64_t dg_launch_count(void);
/* Return every cached block of the library's private device memory pool to
 * the driver (the pool keeps freed blocks while it holds at most half the
 * device memory). */
dg_status dg_trim_memory(void);
/* Evict L2 by writing a 256 MiB scratch buffer (bench hygiene between steps). */
dg_status dg_flush_l2(void);

/* Tuning / testing knob for the Greedy++ ordering kernel: 0 automatic (batch
 * mode: the thread-block cluster kernel for cores above 16K vertices, the
 * candidate-list kernel when no cluster fits; then the scanning single-CTA
 * kernel; then a thread-block cluster), 1 scanning
 * single-CTA kernel only, 2 cluster (16 or 8 CTAs) whenever it fits, 3
 * candidate-list kernel whenever it fits.  Results are identical in every
 * mode. */
dg_status dg_set_peel_mode(int mode);

#ifdef __cplusplus
}
#endif
#endif
