// graph.hpp -- drop-in Graph (reference proj/include/densegraph/graph.hpp:12-80)
// over the B200 C ABI.  The public host fields (n, m, offs, adj, orig) are
// kept because reference callers read them directly; a hidden device handle
// caches the CSR in HBM so repeated calls on the same Graph upload it once.
// Like the reference's, a Graph is immutable after construction.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <span>
#include <mutex>
#include <vector>

#include "dg_b200.h"
#include "densegraph/density.hpp"
#include "densegraph/errors.hpp"
#include "densegraph/parallel.hpp"

namespace densegraph {

constexpr u32 kNoVertex = static_cast<u32>(-1);

struct GraphStats {
  u64 n = 0;
  u64 m = 0;
  u64 max_degree = 0;
};

namespace detail {
[[noreturn]] inline void raise(dg_status st) {
  const std::string msg = dg_last_error();
  switch (st) {
    case DG_E_PARSE: throw ParseError(0, msg);
    case DG_E_EMPTY: throw EmptyGraphError(msg);
    case DG_E_IO: throw IoError(msg);
    case DG_E_PARAM: throw ParamError(msg);
    case DG_E_ORACLE_SIZE: throw OracleSizeError(msg);
    case DG_E_CACHE_HASH: throw CacheHashError(msg);
    default: throw InvariantError(msg);  // invariant, CUDA, out of memory
  }
}
inline void check(dg_status st) {
  if (st != DG_OK) raise(st);
}
struct HandleDeleter {
  void operator()(dg_graph* g) const { dg_graph_free(g); }
};
using Handle = std::shared_ptr<dg_graph>;
}  // namespace detail

struct Graph {
  u64 n = 0;
  u64 m = 0;
  std::vector<u64> offs;  // n + 1
  std::vector<u32> adj;   // 2m
  std::vector<u64> orig;  // dense id -> original id, strictly increasing

  u64 degree(u32 v) const { return offs[v + 1] - offs[v]; }
  std::span<const u32> neighbors(u32 v) const {
    return {adj.data() + offs[v], adj.data() + offs[v + 1]};
  }
  GraphStats stats() const {
    GraphStats s{n, m, 0};
    for (u64 v = 0; v < n; ++v) s.max_degree = std::max(s.max_degree, degree(u32(v)));
    return s;
  }
  Density density() const { return {m, n == 0 ? 1 : n}; }

  // ---- B200 device cache (not part of the reference layout) ----
  // The reference's Graph is immutable after construction and safe to share
  // read-only: the cache is keyed on the sizes and storage of
  // offs/adj/orig (a caller that edits those fields in place after the first
  // device call must assign a fresh Graph), and the lazy upload is serialised
  // so concurrent readers of one Graph never race on it.
  dg_graph* device() const {
    std::lock_guard<std::mutex> lk(device_mutex());
    if (!dev_ || dev_n_ != n || dev_adj_ != adj.data() || dev_offs_ != offs.data() ||
        dev_orig_ != orig.data() || dev_arcs_ != adj.size()) {
      dg_graph* h = nullptr;
      detail::check(dg_graph_from_csr(n, offs.empty() ? zero_offs() : offs.data(), adj.data(),
                                      orig.data(), 0, &h));
      dev_ = detail::Handle(h, detail::HandleDeleter{});
      dev_n_ = n;
      dev_adj_ = adj.data();
      dev_offs_ = offs.data();
      dev_orig_ = orig.data();
      dev_arcs_ = adj.size();
    }
    return dev_.get();
  }
  static Graph from_device(dg_graph* h) {  // takes ownership
    Graph g;
    detail::Handle hold(h, detail::HandleDeleter{});
    u64 dn = 0, dm = 0, dd = 0;
    detail::check(dg_graph_info(h, &dn, &dm, &dd));
    g.n = dn;
    g.m = dm;
    g.offs.resize(dn + 1);
    g.adj.resize(2 * dm);
    g.orig.resize(dn);
    detail::check(dg_graph_download(h, g.offs.data(), g.adj.data(), g.orig.data()));
    g.dev_ = std::move(hold);
    g.dev_n_ = dn;
    g.dev_adj_ = g.adj.data();
    g.dev_offs_ = g.offs.data();
    g.dev_orig_ = g.orig.data();
    g.dev_arcs_ = g.adj.size();
    return g;
  }

 private:
  static const u64* zero_offs() {
    static const u64 z = 0;
    return &z;
  }
  static std::mutex& device_mutex() {
    static std::mutex mu;
    return mu;
  }
  mutable detail::Handle dev_;
  mutable u64 dev_n_ = 0;
  mutable const u32* dev_adj_ = nullptr;
  mutable const u64* dev_offs_ = nullptr;
  mutable const u64* dev_orig_ = nullptr;
  mutable std::size_t dev_arcs_ = 0;
};

// Subgraph induced by keep[v] != 0 (graph.hpp:47-80); new ids follow the
// old dense order.  Optionally reports old -> new ids (kNoVertex if dropped).
inline Graph induced_subgraph(const Graph& g, const std::vector<std::uint8_t>& keep,
                              std::vector<u32>* old_to_new = nullptr) {
  if (keep.size() != g.n) throw InvariantError("keep mask does not match graph size");
  std::vector<u32> map(g.n);
  dg_graph* h = nullptr;
  detail::check(dg_induced(g.device(), keep.data(), &h, map.data()));
  Graph out = Graph::from_device(h);
  if (old_to_new) *old_to_new = std::move(map);
  return out;
}

}  // namespace densegraph
