// oracle.hpp -- drop-in for the reference's exhaustive-search oracle
// (proj/include/densegraph/oracle.hpp:9-28).  brute_force_densest runs on the
// device (dg_brute_force_densest: every Gray-code subset of a <= 32-vertex
// graph, one range per thread); the two lemma checks are scalar host logic
// over it and the device coreness.
#pragma once

#include <algorithm>
#include <vector>

#include "densegraph/core.hpp"
#include "densegraph/density.hpp"
#include "densegraph/graph.hpp"

namespace densegraph {

struct OracleResult {
  Density rho_star{0, 1};    // reduced
  std::vector<u64> witness;  // original ids, ascending
};

// Exhaustive densest subgraph over all nonempty vertex subsets; at most
// `limit` vertices.  Ties prefer fewer vertices, then the lexicographically
// smallest id set (oracle.hpp:16-19).
inline OracleResult brute_force_densest(const Graph& g, u32 limit = 22) {
  if (g.n == 0) throw EmptyGraphError("oracle on empty graph");
  OracleResult r;
  u64 e = 0, v = 0, k = 0;
  std::vector<u64> w(g.n);
  detail::check(dg_brute_force_densest(g.device(), limit, &e, &v, w.data(), &k));
  r.rho_star = Density{e, v};
  w.resize(k);
  r.witness = std::move(w);
  return r;
}

// deg(v) < rho(G) => rho(G - v) > rho(G); vacuous when deg(v) >= rho(G)
// (oracle.hpp:21-24).
inline bool check_degree_lemma(const Graph& g, u32 v) {
  if (v >= g.n) throw ParamError("vertex id out of range");
  const Density rho = g.density();
  if (Density{g.degree(v), 1} >= rho) return true;
  if (g.n == 1) return true;
  return Density{g.m - g.degree(v), g.n - 1} > rho;
}

// The brute-force witness lies inside the k-core (oracle.hpp:26-27).
inline bool check_core_containment(const Graph& g, u32 k) {
  const OracleResult res = brute_force_densest(g);
  const CoreDecomposition dec = exact_coreness(g);
  for (u64 id : res.witness) {
    const auto it = std::lower_bound(g.orig.begin(), g.orig.end(), id);
    if (dec.labels[static_cast<u64>(it - g.orig.begin())] < k) return false;
  }
  return true;
}

}  // namespace densegraph
