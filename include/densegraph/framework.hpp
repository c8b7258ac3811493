// framework.hpp -- drop-in prune-and-refine driver (reference
// proj/include/densegraph/framework.hpp:12-68): Algorithm 1 runs on the
// device behind dg_run; only scalars cross PCIe per iteration.
#pragma once

#include <vector>

#include "densegraph/core.hpp"
#include "densegraph/density.hpp"
#include "densegraph/graph.hpp"
#include "densegraph/refine.hpp"

namespace densegraph {

enum class Algorithm { peel, sort };
enum class Pruning { none, exact, approx, hybrid };

struct RunConfig {
  Algorithm algorithm = Algorithm::peel;
  Pruning pruning = Pruning::exact;
  u64 iterations = 0;
  double epsilon = 0;
  u64 iteration_cap = 1000;
  u64 c_num = 3, c_den = 2;
  int threads = 0;  // accepted for parity; the device path ignores it
  bool reset_loads = false;
  u64 slack_samples = 64;
};

struct IterRecord {
  u64 iter = 0;
  Density rho{0, 1};
  u64 n = 0, m = 0;
  u64 width = 0;
  double ms = 0;
};

struct InitRecord {
  bool kmax_known = false;
  bool kmax_exact = false;
  u32 kmax = 0;
  u32 threshold = 0;
  u64 pruned_n = 0, pruned_m = 0;
  double coreness_ms = 0;
  double init_ms = 0;
};

struct RunTrace {
  InitRecord init;
  std::vector<IterRecord> iters;
  u64 slack_violations = 0;
  std::vector<u64> final_vertices;
};

struct RunResult {
  Density best{0, 1};
  std::vector<u64> witness;
  u64 witness_edges = 0;
  u64 iterations = 0;
  u64 max_width = 0;
  double total_ms = 0;
  RunTrace trace;
};

inline u64 default_iterations(u64 delta, double lower_bound, u64 n, double epsilon,
                              u64 cap = 1000) {
  u64 out = 0;
  detail::check(dg_default_iterations(delta, lower_bound, n, epsilon, cap, &out));
  return out;
}

inline RunResult run(const Graph& g, const RunConfig& cfg) {
  if (g.n == 0) throw EmptyGraphError("run on empty graph");
  if (cfg.threads > 0) set_threads(cfg.threads);
  dg_run_config c{cfg.algorithm == Algorithm::peel ? 0 : 1, static_cast<int>(cfg.pruning),
                  cfg.iterations, cfg.epsilon, cfg.iteration_cap, cfg.c_num, cfg.c_den,
                  cfg.reset_loads ? 1 : 0, cfg.slack_samples};
  dg_run_result r{};
  const u64 cap = cfg.iterations ? cfg.iterations : cfg.iteration_cap;
  std::vector<dg_iter_record> tr(cap);
  std::vector<u64> wit(g.n), fin(g.n);
  detail::check(dg_run(g.device(), &c, &r, tr.data(), cap, wit.data(), g.n, fin.data(), g.n));
  RunResult res;
  res.best = {r.best_edges, r.best_verts};
  wit.resize(r.witness_size);
  res.witness = std::move(wit);
  res.witness_edges = r.witness_edges;
  res.iterations = r.iterations;
  res.max_width = r.max_width;
  res.total_ms = r.total_ms;
  res.trace.init = {bool(r.kmax_known), bool(r.kmax_exact), r.kmax, r.threshold, r.pruned_n,
                    r.pruned_m, r.coreness_ms, r.init_ms};
  for (u64 i = 0; i < r.iterations && i < cap; ++i)
    res.trace.iters.push_back({tr[i].iter, {tr[i].rho_edges, tr[i].rho_verts}, tr[i].n, tr[i].m,
                               tr[i].width, tr[i].ms});
  res.trace.slack_violations = r.slack_violations;
  fin.resize(r.final_n);
  res.trace.final_vertices = std::move(fin);
  return res;
}

}  // namespace densegraph
