// internal.cuh -- device-side objects shared by the translation units.
#pragma once

#include <memory>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

#ifndef DG_KCORE_PROFILE_WORDS
#define DG_KCORE_PROFILE_WORDS (8 + 6 * 4096)  // mirrors include/dg_b200_diag.h
#endif

// Device-resident CSR (reference Graph, graph.hpp:24-45): offs u64[n+1],
// adj u32[2m] (rows ascending), orig u64[n] (dense id -> original id).
struct dg_graph {
  uint64_t n = 0, m = 0, maxdeg = 0;
  dgb::DevBuf<uint64_t> offs;
  dgb::DevBuf<uint32_t> adj;
  dgb::DevBuf<uint64_t> orig;
};

namespace dgb {

// NVTX range for the phases of the path (header-only NVTX v3: a no-op unless
// a profiler is attached; ncu --nvtx --nvtx-include "dg.order/" etc.)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

using GraphPtr = std::unique_ptr<dg_graph>;

// ---- graph.cu ----
GraphPtr build_from_pairs(const uint64_t* d_u, const uint64_t* d_v, uint64_t k);
// graph_stream.cu: CSR straight from a device generator, in source-range parts
GraphPtr build_rmat_streamed(uint32_t scale, uint64_t samples, uint64_t seed, uint64_t part_cap);
GraphPtr build_chung_lu_streamed(uint64_t n, uint64_t pairs, double R, uint64_t seed,
                                 uint64_t part_cap);
// parse.cu: edge-list text on the device -> CSR (DG_E_PARSE sets *bad_line)
GraphPtr parse_edge_list(const uint8_t* d_text, uint64_t len, uint8_t comment, uint64_t* bad_line);
GraphPtr graph_from_device_csr(uint64_t n, const uint64_t* d_offs, const uint32_t* d_adj,
                               const uint64_t* d_orig);
uint64_t device_max_degree(const uint64_t* d_offs, uint64_t n);
// Induced subgraph on keep (device u8 mask, or labels >= k when d_keep is
// null).  d_old_to_new (device, n entries) is optional.
GraphPtr induced(const dg_graph& g, const uint8_t* d_keep, const uint32_t* d_labels, uint32_t k,
                 uint32_t* d_old_to_new);
// Arcs of the rows d_rows[0..nrows) whose target is in the vertex set d_bits
// (a bitmap over g's n ids): the witness recount of framework.cpp:159-175.
uint64_t count_arcs_into_set(const dg_graph& g, const uint32_t* d_rows, uint64_t nrows,
                             const uint32_t* d_bits);
// out[map[v]] = in[v] for kept v (labels / loads carried across a prune).
void gather_by_map_u32(const uint32_t* in, const uint32_t* map, uint64_t n, uint32_t* out);
void gather_by_map_u64(const uint64_t* in, const uint32_t* map, uint64_t n, uint64_t* out);

// ---- kcore.cu ----
struct CoreOut {
  uint32_t kmax = 0, rounds = 0;
  float kernel_ms = 0;
};
CoreOut coreness(const dg_graph& g, bool approx, uint64_t c_num, uint64_t c_den,
                 uint32_t* d_labels);
// block-0 cycle split of the last coreness launch (diagnostic)
void kcore_profile(unsigned long long out[DG_KCORE_PROFILE_WORDS]);

// ---- peel.cu ----
struct KeyRange {
  uint64_t min_load = 0;  // base subtracted from every key
  uint64_t max_key = 0;   // max over v of load(v) - base + deg(v)
};
// Greedy++ ordering (refine.cpp:20-156) with Alg. 3 charges fused:
// d_raw[i] = key at removal - #same-batch smaller neighbours, so that
// A[i] = d_raw[i] - (load(perm[i]) - kr.min_load)  (see peel_kernel.cuh).
// *d_batches (device) receives the number of batches.
void peel_order(const dg_graph& g, const uint64_t* d_loads, const KeyRange& kr,
                bool one_at_a_time, uint32_t* d_perm, uint64_t* d_raw,
                unsigned long long* d_batches);
KeyRange key_range(const dg_graph& g, const uint64_t* d_loads);
// thread-0 cycle split (S1, S2, S3, batches) of the last peel launch
void peel_profile(unsigned long long out[16]);
// per-warp phase timeline of kPeelTraceBatches batches (dg_peel_trace_*)
constexpr uint32_t kPeelTraceBatches = 8, kPeelTraceStamps = 12;
constexpr size_t kPeelTraceWords = size_t(kPeelTraceBatches) * 32 * kPeelTraceStamps;
void peel_trace_arm(uint32_t first_batch);
void peel_trace_read(unsigned long long* out);
void sort_order(uint64_t n, const uint64_t* d_loads, uint32_t* d_perm);
// A[i] from an arbitrary permutation (refine.cpp:186-199); throws InvariantError
// on a non-permutation.
void charges_from_perm(const dg_graph& g, const uint32_t* d_perm, uint32_t* d_charges);
// run()-internal forms: the stable (load, id) sort on just the bits the load
// range needs, and charges from a permutation known to be valid
void sort_order_range(uint64_t n, const uint64_t* d_loads, const KeyRange& kr, uint32_t* d_perm);
void charges_trusted(const dg_graph& g, const uint32_t* d_perm, uint32_t* d_charges);

struct Alg3Out {  // device-written scalars of one update
  uint64_t rho_edges, rho_verts, best_prefix, width;
  uint64_t total;       // B[0]
  uint64_t slack_bad;   // slack audit on pre-update loads
  uint64_t min_load, max_key;  // KeyRange for the next ordering
};
// Suffix sums, exact first-strict argmax, width, loads += A, slack audit,
// next KeyRange; result in *d_out (device).  d_suffix optional.
// Charges come either final (d_charges) or raw from the fused peel (d_raw, base).
void alg3(const dg_graph& g, const uint32_t* d_perm, const uint32_t* d_charges,
          const uint64_t* d_raw, uint64_t raw_base,
          uint64_t* d_loads, uint64_t slack_samples, uint64_t slack_allowed, uint64_t slack_seed,
          uint64_t* d_suffix, Alg3Out* d_out);

// ---- gen.cu ----
void gen_rmat_device(uint32_t scale, uint64_t samples, uint64_t seed, uint64_t* d_u,
                     uint64_t* d_v, uint64_t first = 0);
void gen_chung_lu_device(uint64_t n, uint64_t pairs, double R, uint64_t seed, uint64_t* d_u,
                         uint64_t* d_v);

}  // namespace dgb
