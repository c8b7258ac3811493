// refine.hpp -- drop-in refinement API (reference proj/include/densegraph/refine.hpp:10-49)
// on the B200 Greedy++ batch-peel and Algorithm-3 kernels.
#pragma once

#include <vector>

#include "densegraph/density.hpp"
#include "densegraph/graph.hpp"

namespace densegraph {

struct LoadState {
  std::vector<u64> loads;
};

enum class OrderKind { peel_by_load, sort_by_load };

struct Ordering {
  std::vector<u32> perm;
  OrderKind kind = OrderKind::peel_by_load;
};

struct RefineOutcome {
  Density rho_max{0, 1};
  u64 best_prefix = 0;
  u64 width = 0;
  std::vector<Density> densities;
};

inline Ordering load_peel_order(const Graph& g, const LoadState& s, bool one_at_a_time = false) {
  if (g.n == 0) return {{}, OrderKind::peel_by_load};
  if (s.loads.size() != g.n) throw InvariantError("load vector does not match graph size");
  Ordering o;
  o.perm.resize(g.n);
  detail::check(dg_peel_order(g.device(), s.loads.data(), one_at_a_time ? 1 : 0, o.perm.data()));
  return o;
}

inline Ordering load_sort_order(const LoadState& s) {
  Ordering o;
  o.kind = OrderKind::sort_by_load;
  o.perm.resize(s.loads.size());
  if (!s.loads.empty()) detail::check(dg_sort_order(s.loads.size(), s.loads.data(), o.perm.data()));
  return o;
}

inline RefineOutcome density_and_load_update(const Graph& g, const Ordering& order, LoadState& s,
                                             bool want_densities = false) {
  if (order.perm.size() != g.n) throw InvariantError("ordering does not match graph size");
  if (s.loads.size() != g.n) throw InvariantError("load vector does not match graph size");
  RefineOutcome r;
  if (g.n == 0) return r;
  dg_outcome o{};
  std::vector<u64> suffix(want_densities ? g.n : 0);
  detail::check(dg_density_load_update(g.device(), order.perm.data(), s.loads.data(), &o,
                                       want_densities ? suffix.data() : nullptr));
  r.rho_max = {o.rho_edges, o.rho_verts};
  r.best_prefix = o.best_prefix;
  r.width = o.width;
  if (want_densities) {
    r.densities.resize(g.n);
    for (u64 i = 0; i < g.n; ++i) r.densities[i] = Density{suffix[i], g.n - i};
  }
  return r;
}

inline RefineOutcome charikar_peel(const Graph& g) {
  dg_outcome o{0, 1, 0, 0};
  detail::check(dg_charikar_peel(g.device(), &o));
  RefineOutcome r;
  r.rho_max = {o.rho_edges, o.rho_verts};
  r.best_prefix = o.best_prefix;
  r.width = o.width;
  return r;
}

inline u64 slack_violations(const Ordering& order, const std::vector<u64>& loads,
                            u64 allowed_slack, u64 samples, u64 seed) {
  u64 bad = 0;
  detail::check(dg_slack_violations(order.perm.size(), order.perm.data(), loads.data(),
                                    allowed_slack, samples, seed, &bad));
  return bad;
}

}  // namespace densegraph
