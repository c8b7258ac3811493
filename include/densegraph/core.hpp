// core.hpp -- drop-in coreness API (reference proj/include/densegraph/core.hpp:9-32)
// on the B200 persistent k-core kernel.
#pragma once

#include <vector>

#include "densegraph/graph.hpp"

namespace densegraph {

enum class CoreKind { exact, approximate };

struct CoreDecomposition {
  std::vector<u32> labels;
  u32 kmax = 0;
  u32 peel_rounds = 0;
  CoreKind kind = CoreKind::exact;
  u64 c_num = 1, c_den = 1;
};

inline CoreDecomposition exact_coreness(const Graph& g) {
  if (g.n == 0) throw EmptyGraphError("coreness of empty graph");
  CoreDecomposition d;
  d.labels.resize(g.n);
  detail::check(dg_coreness(g.device(), 0, 1, 1, d.labels.data(), &d.kmax, &d.peel_rounds));
  return d;
}

inline CoreDecomposition approx_coreness(const Graph& g, u64 c_num, u64 c_den) {
  if (c_den == 0 || c_num <= c_den) throw ParamError("approximation factor must be > 1");
  if (g.n == 0) throw EmptyGraphError("coreness of empty graph");
  CoreDecomposition d;
  d.kind = CoreKind::approximate;
  d.c_num = c_num;
  d.c_den = c_den;
  d.labels.resize(g.n);
  detail::check(
      dg_coreness(g.device(), 1, c_num, c_den, d.labels.data(), &d.kmax, &d.peel_rounds));
  return d;
}

inline Graph get_core(const Graph& g, const CoreDecomposition& dec, u32 k,
                      std::vector<u32>* old_to_new = nullptr) {
  if (dec.labels.size() != g.n) throw InvariantError("core labels do not match graph size");
  std::vector<u32> map(g.n);
  dg_graph* h = nullptr;
  detail::check(dg_get_core(g.device(), dec.labels.data(), k, &h, map.data()));
  Graph out = Graph::from_device(h);
  if (old_to_new) *old_to_new = std::move(map);
  return out;
}

}  // namespace densegraph
