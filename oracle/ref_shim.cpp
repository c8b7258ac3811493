// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C ABI over the UNMODIFIED reference library (densegraph, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libdgref.so).
// It lets Python tests and bench.py's `--impl reference` leg drive the real
// reference through its own public C++ API (proj/include/densegraph/*.hpp):
// no reference source is copied here, this file only converts plain
// pointers <-> the reference's std::vector-based types and exceptions <->
// status codes (same numbering as include/dg_b200.h).
#include <cstring>
#include <exception>
#include <sstream>
#include <string>

#include "densegraph/core.hpp"
#include "densegraph/errors.hpp"
#include "densegraph/framework.hpp"
#include "densegraph/io.hpp"
#include "densegraph/parallel.hpp"
#include "densegraph/refine.hpp"
#include "dg_oracle.h"

namespace dg = densegraph;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const dg::ParseError& e) {
    g_err = e.what();
    return 1;
  } catch (const dg::EmptyGraphError& e) {
    g_err = e.what();
    return 2;
  } catch (const dg::IoError& e) {
    g_err = e.what();
    return 3;
  } catch (const dg::ParamError& e) {
    g_err = e.what();
    return 4;
  } catch (const dg::InvariantError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return 8;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}
dg::Graph& G(void* h) { return *static_cast<dg::Graph*>(h); }
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_set_threads(int t) { dg::set_threads(t); }
int ref_max_threads(void) { return dg::max_threads(); }

int ref_graph_parse_text(const char* text, uint64_t len, void** out) {
  return guard([&] {
    std::istringstream in(std::string(text, len));
    *out = new dg::Graph(dg::parse_edge_list(in));
  });
}

int ref_graph_from_csr(uint64_t n, const uint64_t* offs, const uint32_t* adj,
                       const uint64_t* orig, void** out) {
  return guard([&] {
    auto* g = new dg::Graph;
    g->n = n;
    g->offs.assign(offs, offs + n + 1);
    g->adj.assign(adj, adj + offs[n]);
    g->orig.assign(orig, orig + n);
    g->m = g->adj.size() / 2;
    *out = g;
  });
}

void ref_graph_free(void* h) { delete static_cast<dg::Graph*>(h); }

void ref_graph_info(void* h, uint64_t* n, uint64_t* m, uint64_t* maxdeg) {
  dg::GraphStats s = G(h).stats();
  *n = s.n;
  *m = s.m;
  *maxdeg = s.max_degree;
}

void ref_graph_download(void* h, uint64_t* offs, uint32_t* adj, uint64_t* orig) {
  const dg::Graph& g = G(h);
  std::memcpy(offs, g.offs.data(), g.offs.size() * sizeof(uint64_t));
  std::memcpy(adj, g.adj.data(), g.adj.size() * sizeof(uint32_t));
  std::memcpy(orig, g.orig.data(), g.orig.size() * sizeof(uint64_t));
}

int ref_coreness(void* h, int approx, uint64_t cn, uint64_t cd, uint32_t* labels, uint32_t* kmax,
                 uint32_t* rounds) {
  return guard([&] {
    dg::CoreDecomposition d =
        approx ? dg::approx_coreness(G(h), cn, cd) : dg::exact_coreness(G(h));
    std::memcpy(labels, d.labels.data(), d.labels.size() * sizeof(uint32_t));
    *kmax = d.kmax;
    *rounds = d.peel_rounds;
  });
}

int ref_get_core(void* h, const uint32_t* labels, uint32_t k, void** out, uint32_t* old_to_new) {
  return guard([&] {
    dg::CoreDecomposition d;
    d.labels.assign(labels, labels + G(h).n);
    std::vector<uint32_t> map;
    *out = new dg::Graph(dg::get_core(G(h), d, k, &map));
    if (old_to_new) std::memcpy(old_to_new, map.data(), map.size() * sizeof(uint32_t));
  });
}

int ref_peel_order(void* h, const uint64_t* loads, int one, uint32_t* perm) {
  return guard([&] {
    dg::LoadState s;
    s.loads.assign(loads, loads + G(h).n);
    dg::Ordering o = dg::load_peel_order(G(h), s, one != 0);
    std::memcpy(perm, o.perm.data(), o.perm.size() * sizeof(uint32_t));
  });
}

int ref_sort_order(uint64_t n, const uint64_t* loads, uint32_t* perm) {
  return guard([&] {
    dg::LoadState s;
    s.loads.assign(loads, loads + n);
    dg::Ordering o = dg::load_sort_order(s);
    std::memcpy(perm, o.perm.data(), o.perm.size() * sizeof(uint32_t));
  });
}

int ref_density_update(void* h, const uint32_t* perm, uint64_t* loads, og_outcome* out,
                       uint64_t* suffix_edges) {
  return guard([&] {
    const uint64_t n = G(h).n;
    dg::Ordering o;
    o.perm.assign(perm, perm + n);
    dg::LoadState s;
    s.loads.assign(loads, loads + n);
    dg::RefineOutcome r = dg::density_and_load_update(G(h), o, s, suffix_edges != nullptr);
    std::memcpy(loads, s.loads.data(), n * sizeof(uint64_t));
    out->rho_edges = r.rho_max.edges;
    out->rho_verts = r.rho_max.verts;
    out->best_prefix = r.best_prefix;
    out->width = r.width;
    if (suffix_edges)
      for (uint64_t i = 0; i < n; ++i) suffix_edges[i] = r.densities[i].edges;
  });
}

uint64_t ref_slack_violations(uint64_t n, const uint32_t* perm, const uint64_t* loads,
                              uint64_t slack, uint64_t samples, uint64_t seed) {
  dg::Ordering o;
  o.perm.assign(perm, perm + n);
  std::vector<uint64_t> l(loads, loads + n);
  return dg::slack_violations(o, l, slack, samples, seed);
}

int ref_default_iterations(uint64_t delta, double lb, uint64_t n, double eps, uint64_t cap,
                           uint64_t* out) {
  return guard([&] { *out = dg::default_iterations(delta, lb, n, eps, cap); });
}

// Full Algorithm 1 through dg::run; timings (ms) are the reference's own
// steady_clock figures: times[0] = init.coreness_ms, [1] = init_ms,
// [2] = total_ms; iter_ms[i] = IterRecord.ms.
int ref_run(void* h, const og_config* c, int threads, og_result* res, og_iter* trace,
            uint64_t trace_cap, double* iter_ms, uint64_t* witness, uint64_t witness_cap,
            uint64_t* final_ids, uint64_t final_cap, double* times) {
  return guard([&] {
    dg::RunConfig cfg;
    cfg.algorithm = c->algorithm == 0 ? dg::Algorithm::peel : dg::Algorithm::sort;
    cfg.pruning = static_cast<dg::Pruning>(c->pruning);
    cfg.iterations = c->iterations;
    cfg.epsilon = c->epsilon;
    cfg.iteration_cap = c->iteration_cap;
    cfg.c_num = c->c_num;
    cfg.c_den = c->c_den;
    cfg.threads = threads;
    cfg.reset_loads = c->reset_loads != 0;
    cfg.slack_samples = c->slack_samples;
    dg::RunResult r = dg::run(G(h), cfg);
    std::memset(res, 0, sizeof *res);
    res->best_edges = r.best.edges;
    res->best_verts = r.best.verts;
    res->witness_size = r.witness.size();
    res->witness_edges = r.witness_edges;
    res->iterations = r.iterations;
    res->max_width = r.max_width;
    res->slack_violations = r.trace.slack_violations;
    res->kmax_known = r.trace.init.kmax_known;
    res->kmax_exact = r.trace.init.kmax_exact;
    res->kmax = r.trace.init.kmax;
    res->threshold = r.trace.init.threshold;
    res->pruned_n = r.trace.init.pruned_n;
    res->pruned_m = r.trace.init.pruned_m;
    res->final_n = r.trace.final_vertices.size();
    for (uint64_t i = 0; i < r.trace.iters.size() && i < trace_cap; ++i) {
      const dg::IterRecord& it = r.trace.iters[i];
      if (trace) trace[i] = {it.iter, it.rho.edges, it.rho.verts, it.n, it.m, it.width};
      if (iter_ms) iter_ms[i] = it.ms;
    }
    if (witness)
      for (uint64_t i = 0; i < r.witness.size() && i < witness_cap; ++i) witness[i] = r.witness[i];
    if (final_ids)
      for (uint64_t i = 0; i < r.trace.final_vertices.size() && i < final_cap; ++i)
        final_ids[i] = r.trace.final_vertices[i];
    if (times) {
      times[0] = r.trace.init.coreness_ms;
      times[1] = r.trace.init.init_ms;
      times[2] = r.total_ms;
    }
  });
}

}  // extern "C"
