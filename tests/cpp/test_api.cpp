// test_api.cpp -- the reference's pinned unit-test behaviour, written against
// the drop-in C++ headers (include/densegraph/*.hpp) so a reference caller
// compiles unchanged.  Cases follow test_graph.cpp:12-51, test_core.cpp:10-111,
// test_refine.cpp:29-170 and test_framework.cpp:46-114 (rewritten, not copied).
// Exit code = number of failed checks.  Needs a B200 to run.
#include <cstdio>
#include <filesystem>
#include <numeric>
#include <sstream>

#include "densegraph/core.hpp"
#include "densegraph/framework.hpp"
#include "densegraph/io.hpp"
#include "densegraph/refine.hpp"

using namespace densegraph;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                    \
  do {                                                              \
    ++g_checks;                                                     \
    if (!(c)) {                                                     \
      ++g_fail;                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
    }                                                               \
  } while (0)
#define CHECK_THROWS(expr, T)        \
  do {                               \
    bool thrown_ = false;            \
    try {                            \
      (void)(expr);                  \
    } catch (const T&) {             \
      thrown_ = true;                \
    }                                \
    CHECK(thrown_);                  \
  } while (0)

static Graph text(const std::string& s) {
  std::istringstream in(s);
  return parse_edge_list(in);
}
static Graph edges(const std::vector<std::pair<u64, u64>>& e) {
  std::ostringstream o;
  for (auto [a, b] : e) o << a << ' ' << b << '\n';
  return text(o.str());
}
static Graph clique(u64 k) {
  std::vector<std::pair<u64, u64>> e;
  for (u64 i = 0; i < k; ++i)
    for (u64 j = i + 1; j < k; ++j) e.emplace_back(i, j);
  return edges(e);
}
static Graph path(u64 k) {
  std::vector<std::pair<u64, u64>> e;
  for (u64 i = 0; i + 1 < k; ++i) e.emplace_back(i, i + 1);
  return edges(e);
}
static Graph star(u64 leaves) {
  std::vector<std::pair<u64, u64>> e;
  for (u64 i = 1; i <= leaves; ++i) e.emplace_back(0, i);
  return edges(e);
}
static Graph tri_pendant() { return edges({{0, 1}, {1, 2}, {2, 0}, {2, 3}}); }
static LoadState zeros(u64 n) { return LoadState{std::vector<u64>(n, 0)}; }
static Ordering identity(u64 n) {
  Ordering o;
  o.perm.resize(n);
  std::iota(o.perm.begin(), o.perm.end(), 0u);
  return o;
}

int main() {
  // ---- graph / ingest
  {
    Graph g = text("# c\n0 1\r\n1\t0\n3 3\n  7 5\n");
    CHECK(g.n == 4 && g.m == 2);
    CHECK((g.orig == std::vector<u64>{0, 1, 5, 7}));
    CHECK((g.adj == std::vector<u32>{1, 0, 3, 2}));
    CHECK_THROWS(text("0 1\n1 x\n"), ParseError);
    CHECK_THROWS(text("3 3\n"), EmptyGraphError);
    Graph k4 = clique(4);
    CHECK(k4.stats().max_degree == 3 && k4.density() == (Density{3, 2}));
    std::vector<u32> map;
    Graph t = induced_subgraph(tri_pendant(), {1, 1, 1, 0}, &map);
    CHECK(t.n == 3 && t.m == 3 && map[3] == kNoVertex);
    auto p = std::filesystem::temp_directory_path() / "dg_b200_cache_test.bin";
    write_cache(k4, p.string(), 42);
    u64 src = 0;
    Graph back = read_cache(p.string(), &src);
    CHECK(src == 42 && back.offs == k4.offs && back.adj == k4.adj && back.orig == k4.orig);
    CHECK(is_cache_file(p.string()));
    std::filesystem::remove(p);
  }
  // ---- coreness
  {
    CoreDecomposition d = exact_coreness(clique(5));
    CHECK(d.labels == std::vector<u32>(5, 4) && d.kmax == 4 && d.peel_rounds >= 1);
    d = exact_coreness(tri_pendant());
    CHECK((d.labels == std::vector<u32>{2, 2, 2, 1}) && d.kmax == 2);
    CHECK(exact_coreness(path(4)).labels == std::vector<u32>(4, 1));
    CHECK(approx_coreness(path(4), 3, 2).labels == std::vector<u32>(4, 1));
    CHECK_THROWS(approx_coreness(clique(4), 1, 1), ParamError);
    CHECK_THROWS(exact_coreness(Graph{}), EmptyGraphError);
    Graph g = tri_pendant();
    std::vector<u32> map;
    Graph c = get_core(g, exact_coreness(g), 2, &map);
    CHECK(c.n == 3 && c.m == 3 && (c.orig == std::vector<u64>{0, 1, 2}) && map[3] == kNoVertex);
    CHECK_THROWS(get_core(clique(3), exact_coreness(clique(4)), 1), InvariantError);
    CHECK(exact_coreness(star(3000)).labels == std::vector<u32>(3001, 1));
  }
  // ---- refinement
  {
    CHECK((load_peel_order(path(3), zeros(3)).perm == std::vector<u32>{0, 2, 1}));
    CHECK((load_peel_order(clique(4), zeros(4)).perm == std::vector<u32>{0, 1, 2, 3}));
    LoadState s = zeros(4);
    s.loads[3] = 10;
    CHECK((load_peel_order(tri_pendant(), s).perm == std::vector<u32>{0, 1, 2, 3}));
    CHECK((load_sort_order({{5, 2, 7, 2}}).perm == std::vector<u32>{1, 3, 0, 2}));
    LoadState z = zeros(3);
    RefineOutcome o = density_and_load_update(path(3), identity(3), z, true);
    CHECK(o.rho_max == (Density{2, 3}) && o.best_prefix == 0 && o.width == 1);
    CHECK((z.loads == std::vector<u64>{1, 1, 0}) && o.densities.size() == 3);
    LoadState z4 = zeros(4);
    o = density_and_load_update(edges({{0, 1}, {1, 2}, {2, 3}, {1, 3}}), identity(4), z4, true);
    CHECK(o.rho_max == (Density{1, 1}) && o.best_prefix == 0 && o.width == 2);
    CHECK((z4.loads == std::vector<u64>{1, 2, 1, 0}) && o.densities[1] == (Density{3, 3}));
    Ordering dup{{0, 1, 1}, OrderKind::peel_by_load};
    LoadState z3 = zeros(3);
    CHECK_THROWS(density_and_load_update(clique(3), dup, z3), InvariantError);
    CHECK(charikar_peel(star(5)).rho_max == (Density{5, 6}));
    CHECK(charikar_peel(clique(4)).rho_max == (Density{3, 2}));
    CHECK(charikar_peel(tri_pendant()).rho_max == (Density{1, 1}));
    Ordering desc{{0, 1, 2, 3, 4, 5}, OrderKind::sort_by_load};
    CHECK(slack_violations(desc, {9, 7, 5, 3, 1, 0}, 0, 4000, 1) > 0);
  }
  // ---- framework
  {
    for (Algorithm a : {Algorithm::peel, Algorithm::sort}) {
      RunConfig cfg;
      cfg.algorithm = a;
      cfg.iterations = 1;
      RunResult r = run(clique(4), cfg);
      CHECK(r.best == (Density{3, 2}) && (r.witness == std::vector<u64>{0, 1, 2, 3}));
      CHECK(r.witness_edges == 6 && r.max_width == 3 && r.trace.iters.size() == 1);
      CHECK(r.trace.init.kmax == 3 && r.trace.init.threshold == 2 && r.trace.init.kmax_exact);
    }
    std::vector<std::pair<u64, u64>> e;
    for (u64 r = 0; r < 45; ++r)
      for (u64 l = 45; l < 50; ++l) e.emplace_back(r, l);
    e.insert(e.end(), {{50, 51}, {50, 52}, {50, 53}, {51, 52}, {51, 53}, {52, 53}});
    RunConfig cfg;
    cfg.iterations = 3;
    RunResult r = run(edges(e), cfg);
    CHECK(r.trace.init.kmax == 5 && r.trace.init.threshold == 3 && r.trace.init.pruned_n == 54);
    CHECK(r.trace.iters.size() == 3 && r.trace.iters[0].n == 54 && r.trace.iters[1].n == 50);
    CHECK(r.trace.iters[0].rho == (Density{9, 2}) && r.best == (Density{9, 2}));
    CHECK(r.witness.size() == 50 && r.witness_edges == 225 && r.trace.final_vertices.size() == 50);
    CHECK(default_iterations(100, 50, 7, 0.5) == 16);
    CHECK_THROWS(default_iterations(3, 3, 3, 0.0), ParamError);
    CHECK_THROWS(run(Graph{}, RunConfig{}), EmptyGraphError);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail;
}
