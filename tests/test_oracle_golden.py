"""Pin the CPU oracle (oracle/dg_oracle.c) before trusting it.

1. Known-answer vectors of the reference's own unit tests
   (test_core.cpp:10-28, test_refine.cpp:29-48,89-121,166-170,
   test_framework.cpp:46-114, test_graph.cpp:12-51), rewritten as behaviour.
2. Every fixture in tests/golden/golden.json, produced by the UNMODIFIED
   reference library (tests/golden/make_golden.py).
3. Live cross-checks against the reference library when oracle/_ref is built.
No GPU needed.
"""
import hashlib
import os

import numpy as np
import pytest

import graphs as G
from oracle import OracleError, RunConfig, gnp_edges, mix64, random_loads, reduced


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def build(orc, edges):
    return orc.build(*G.uv(edges))


# ---------------------------------------------------------------- known answers
def test_build_cleanup_rules(orc):
    # loops dropped, reversed duplicates collapsed, ids kept only if in a non-loop edge
    g = orc.build(np.array([0, 1, 3, 7], np.uint64), np.array([1, 0, 3, 5], np.uint64))
    assert g.n == 4 and g.m == 2
    assert g.orig.tolist() == [0, 1, 5, 7]
    assert g.offs.tolist() == [0, 1, 2, 3, 4]
    assert g.adj.tolist() == [1, 0, 3, 2]
    with pytest.raises(OracleError) as e:
        orc.build(np.array([3], np.uint64), np.array([3], np.uint64))
    assert e.value.kind == "EmptyGraphError"


def test_build_rows_sorted_and_symmetric(orc):
    u, v = orc.gen_rmat(10, 16 << 10, 3)
    g = orc.build(u, v)
    for x in range(g.n):
        row = g.adj[g.offs[x]:g.offs[x + 1]]
        assert np.all(np.diff(row.astype(np.int64)) > 0)
    src = np.repeat(np.arange(g.n), np.diff(g.offs).astype(np.int64))
    fwd = set(zip(src.tolist(), g.adj.tolist()))
    assert all((b, a) in fwd for a, b in fwd)
    assert np.all(np.diff(g.orig.astype(np.int64)) > 0)


def test_coreness_pinned(orc):
    lab, kmax, rounds = orc.coreness(build(orc, G.clique(5)))
    assert lab.tolist() == [4] * 5 and kmax == 4 and rounds >= 1
    lab, kmax, _ = orc.coreness(build(orc, G.triangle_pendant()))
    assert lab.tolist() == [2, 2, 2, 1] and kmax == 2
    lab, kmax, _ = orc.coreness(build(orc, G.path_graph(4)))
    assert lab.tolist() == [1] * 4 and kmax == 1
    lab, _, _ = orc.coreness(build(orc, G.path_graph(4)), True, 3, 2)
    assert lab.tolist() == [1] * 4
    lab, _, _ = orc.coreness(build(orc, G.star(3000)))
    assert np.all(lab == 1)


def test_coreness_errors(orc):
    g = build(orc, G.clique(4))
    for cn, cd in ((1, 1), (2, 3), (1, 0)):
        with pytest.raises(OracleError) as e:
            orc.coreness(g, True, cn, cd)
        assert e.value.kind == "ParamError"


def test_get_core_pinned(orc):
    g = build(orc, G.triangle_pendant())
    lab, _, _ = orc.coreness(g)
    c, m = orc.get_core(g, lab, 2)
    assert (c.n, c.m) == (3, 3) and c.orig.tolist() == [0, 1, 2] and m[3] == 0xFFFFFFFF


def test_peel_order_pinned(orc):
    assert orc.peel_order(build(orc, G.path_graph(3)), [0, 0, 0]).tolist() == [0, 2, 1]
    assert orc.peel_order(build(orc, G.clique(4)), [0] * 4).tolist() == [0, 1, 2, 3]
    assert orc.peel_order(build(orc, G.triangle_pendant()), [0, 0, 0, 10]).tolist() == [0, 1, 2, 3]


def test_peel_shift_invariance(orc):
    for seed in range(1, 16):
        g = orc.build(*G.uv(gnp_edges(60, 80, seed * 11)))
        small = random_loads(g.n, 9, seed)
        huge = small + np.uint64(1 << 40)
        assert np.array_equal(orc.peel_order(g, small), orc.peel_order(g, huge))
        assert np.array_equal(orc.peel_order(g, small, True), orc.peel_order(g, huge, True))


def test_sort_order_pinned(orc):
    assert orc.sort_order([5, 2, 7, 2]).tolist() == [1, 3, 0, 2]
    assert orc.sort_order([0, 0, 0, 0]).tolist() == [0, 1, 2, 3]
    assert orc.sort_order([1, 1, 0]).tolist() == [2, 0, 1]


def test_density_update_pinned(orc):
    out, loads, A, B = orc.density_update(build(orc, G.path_graph(3)), [0, 1, 2], [0, 0, 0])
    assert out["rho"] == (2, 3) and out["best_prefix"] == 0 and out["width"] == 1
    assert loads.tolist() == [1, 1, 0] and B.tolist() == [2, 1, 0]
    out, loads, A, B = orc.density_update(build(orc, G.four_chord()), [0, 1, 2, 3], [0] * 4)
    assert out["rho"] == (4, 4) and out["best_prefix"] == 0 and out["width"] == 2
    assert loads.tolist() == [1, 2, 1, 0] and B[1] == 3
    out, loads, _, _ = orc.density_update(build(orc, G.clique(4)), [0, 1, 2, 3], [0] * 4)
    assert reduced(*out["rho"]) == (3, 2) and loads.tolist() == [3, 2, 1, 0] and out["width"] == 3


def test_density_update_contract_errors(orc):
    g = build(orc, G.clique(3))
    for perm in ([0, 1, 1], [0, 1, 7]):
        with pytest.raises(OracleError) as e:
            orc.density_update(g, perm, [0, 0, 0])
        assert e.value.kind == "InvariantError"


def test_charikar_pinned(orc):
    def charikar(edges):
        g = build(orc, edges)
        perm = orc.peel_order(g, np.zeros(g.n, np.uint64))
        out, _, _, _ = orc.density_update(g, perm, np.zeros(g.n, np.uint64))
        return reduced(*out["rho"])
    assert charikar(G.star(5)) == (5, 6)
    assert charikar(G.clique(4)) == (3, 2)
    assert charikar(G.triangle_pendant()) == (1, 1)


def test_slack_audit(orc):
    for seed in range(1, 21):
        g = orc.build(*G.uv(gnp_edges(50, 100, seed * 29)))
        loads = random_loads(g.n, 20, seed)
        assert orc.slack_violations(orc.peel_order(g, loads), loads, g.max_degree(), 2000, seed) == 0
        assert orc.slack_violations(orc.sort_order(loads), loads, 0, 2000, seed) == 0
    assert orc.slack_violations([0, 1, 2, 3, 4, 5], [9, 7, 5, 3, 1, 0], 0, 4000, 1) > 0


def test_default_iterations_pinned(orc):
    assert orc.default_iterations(3, 3, 3, 1.0) == 10
    assert orc.default_iterations(100, 50, 7, 0.5) == 16
    assert orc.default_iterations(1000000, 1, 3, 1.0) == 1000
    assert orc.default_iterations(100, 1, 100, 0.1, 5) == 5
    for args in ((3, 3, 3, 0.0), (3, 3, 3, -1.0), (3, 0.5, 3, 1.0), (3, 3, 0, 1.0)):
        with pytest.raises(OracleError):
            orc.default_iterations(*args)


def test_run_k4_single_iteration(orc):
    for alg in ("peel", "sort"):
        r = orc.run(build(orc, G.clique(4)), RunConfig(algorithm=alg, iterations=1))
        assert r.best == (3, 2) and r.witness.tolist() == [0, 1, 2, 3] and r.witness_edges == 6
        assert r.max_width == 3 and r.trace == [(1, 3, 2, 4, 6, 3)]
        assert (r.kmax, r.threshold, r.pruned_n, r.pruned_m) == (3, 2, 4, 6)


def test_run_ties_and_two_triangles(orc):
    r = orc.run(build(orc, G.triangle_pendant()), RunConfig(iterations=5))
    assert r.best == (1, 1) and len(r.witness) == 4 and r.witness_edges == 4
    r = orc.run(build(orc, G.two_triangles()), RunConfig(iterations=3))
    assert r.best == (6, 5) and len(r.witness) == 5


def test_run_reprune_trace(orc):
    g = build(orc, G.biclique_with_k4())
    r = orc.run(g, RunConfig(iterations=3))
    assert (r.kmax, r.threshold, r.pruned_n) == (5, 3, 54)
    assert [t[3] for t in r.trace] == [54, 50, 50]
    assert reduced(r.trace[0][1], r.trace[0][2]) == (9, 2)
    assert r.best == (9, 2) and len(r.witness) == 50 and r.witness_edges == 225
    assert len(r.final_vertices) == 50


def test_run_errors(orc):
    g = build(orc, G.clique(4))
    with pytest.raises(OracleError) as e:
        orc.run(g, RunConfig(iterations=0, epsilon=0.0))
    assert e.value.kind == "ParamError"
    r = orc.run(g, RunConfig(iterations=0, epsilon=0.9))
    assert r.iterations >= 10 and len(r.trace) == r.iterations


# ---------------------------------------------------------------- golden fixtures
def test_gnp_generator_matches_test_util(orc):
    for n, p, s in ((10, 300, 1), (57, 120, 99), (2, 5, 4)):
        u, v = orc.gen_gnp(n, p, s)
        assert list(zip(u.tolist(), v.tolist())) == gnp_edges(n, p, s)


def test_golden_coreness(orc, golden):
    for c in golden["coreness"]:
        g = orc.build(*orc.gen_gnp(c["n"], c["permille"], c["seed"]))
        lab, kmax, rounds = orc.coreness(g)
        assert lab.tolist() == c["labels"] and kmax == c["kmax"] and rounds == c["rounds"], c["seed"]
        for cn, cd in ((3, 2), (2, 1), (11, 10)):
            a = c[f"approx_{cn}_{cd}"]
            al, ak, ar = orc.coreness(g, True, cn, cd)
            assert al.tolist() == a["labels"] and ak == a["kmax"] and ar == a["rounds"]


def test_golden_peel(orc, golden):
    for c in golden["peel"]:
        g = orc.build(*orc.gen_gnp(c["n"], c["permille"], c["seed"]))
        loads = random_loads(g.n, c["loads_maxload"], c["loads_seed"])
        assert orc.peel_order(g, loads).tolist() == c["perm"]
        assert orc.peel_order(g, loads, True).tolist() == c["perm_one"]
        out, la, _, B = orc.density_update(g, c["perm"], loads)
        assert list(out["rho"]) == c["rho"] and out["best_prefix"] == c["best_prefix"]
        assert out["width"] == c["width"] and la.tolist() == c["loads_after"]
        assert B.tolist() == c["suffix_edges"]


def test_golden_density(orc, golden):
    for c in golden["density"]:
        g = orc.build(*orc.gen_gnp(c["n"], c["permille"], c["seed"]))
        loads = random_loads(g.n, c["maxload"], c["loads_seed"])
        for which in ("peel", "sort"):
            e = c[which]
            perm = orc.peel_order(g, loads) if which == "peel" else orc.sort_order(loads)
            assert perm.tolist() == e["perm"]
            out, la, _, B = orc.density_update(g, perm, loads)
            assert list(out["rho"]) == e["rho"] and out["best_prefix"] == e["best_prefix"]
            assert out["width"] == e["width"] and la.tolist() == e["loads_after"]
            assert B.tolist() == e["suffix_edges"]


def _golden_graph(orc, name):
    if name == "biclique_k4":
        return orc.build(*G.uv(G.biclique_with_k4()))
    _, n, p, s = name.split("_")
    return orc.build(*orc.gen_gnp(int(n), int(p), int(s)))


def _cmp_run(r, e):
    assert list(r.best) == e["best"]
    assert r.witness.tolist() == e["witness"]
    assert r.witness_edges == e["witness_edges"] and r.iterations == e["iterations"]
    assert r.max_width == e["max_width"] and r.slack_violations == e["slack_violations"]
    assert (r.kmax_known, r.kmax_exact, r.kmax, r.threshold) == (
        e["kmax_known"], e["kmax_exact"], e["kmax"], e["threshold"])
    assert (r.pruned_n, r.pruned_m) == (e["pruned_n"], e["pruned_m"])
    assert r.final_vertices.tolist() == e["final_vertices"]
    assert [list(t) for t in r.trace] == e["trace"]


def test_golden_runs(orc, golden):
    cache = {}
    for c in golden["runs"]:
        g = cache.setdefault(c["graph"], _golden_graph(orc, c["graph"]))
        cfg = RunConfig(algorithm=c["algorithm"], pruning=c["pruning"],
                        iterations=c["iterations"], reset_loads=c["reset_loads"])
        _cmp_run(orc.run(g, cfg), c["result"])


def _synthetic_input(orc, s):
    p = s["params"]
    if s["kind"] == "rmat":
        return orc.gen_rmat(p["scale"], p["samples"], p["seed"])
    if s["kind"] == "er_planted":
        return orc.gen_er_planted(p["n"], p["m"], p["block"], p["seed"])
    return orc.gen_chung_lu(p["n"], p["pairs"], p["seed"])


def test_golden_synthetic(orc, golden):
    for s in golden["synthetic"]:
        g = orc.build(*_synthetic_input(orc, s))
        assert (g.n, g.m) == (s["n"], s["m"])
        assert (sha(g.offs), sha(g.adj), sha(g.orig)) == (s["offs"], s["adj"], s["orig"])
        lab, kmax, rounds = orc.coreness(g)
        assert (sha(lab), kmax, rounds) == (s["labels"], s["kmax"], s["rounds"])
        core, _ = orc.get_core(g, lab, (kmax + 1) // 2)
        assert (core.n, core.m, sha(core.adj), sha(core.orig)) == (
            s["core_n"], s["core_m"], s["core_adj"], s["core_orig"])
        loads = np.zeros(core.n, np.uint64)
        for e in s["core_iters"]:
            perm = orc.peel_order(core, loads)
            out, loads, _, _ = orc.density_update(core, perm, loads)
            assert (sha(perm), sha(loads)) == (e["perm"], e["loads"])
            assert list(out["rho"]) == e["rho"] and out["width"] == e["width"]
        r = orc.run(g, RunConfig(iterations=s["run_T"]))
        e = s["run"]
        assert list(r.best) == e["best"] and sha(r.witness) == e["witness"]
        assert [list(t) for t in r.trace] == e["trace"]
        assert sha(r.final_vertices) == e["final_vertices"] and r.max_width == e["max_width"]


# ---------------------------------------------------------------- live reference
def test_live_reference_random(orc, ref):
    """Extra seeds beyond the fixtures, straight against the reference library."""
    for seed in range(1000, 1040):
        n = 3 + mix64(seed) % 150
        edges = gnp_edges(n, 10 + mix64(seed ^ 5) % 400, seed)
        rg = ref.parse_pairs(*G.uv(edges))
        g = orc.build(*G.uv(edges))
        h = rg.download()
        assert np.array_equal(g.offs, h.offs) and np.array_equal(g.adj, h.adj)
        assert ref.coreness(rg)[0].tolist() == orc.coreness(g)[0].tolist()
        loads = random_loads(g.n, seed % 7 * 3, seed)
        assert np.array_equal(ref.peel_order(rg, loads), orc.peel_order(g, loads))
        for alg in ("peel", "sort"):
            cfg = RunConfig(algorithm=alg, iterations=6)
            a, b = ref.run(rg, cfg), orc.run(g, cfg)
            assert a.trace == b.trace and np.array_equal(a.witness, b.witness)


CA_HEPTH = "/root/reference/proj/data/ca-hepth.txt"


@pytest.mark.skipif(not os.path.exists(CA_HEPTH), reason="reference dataset not present")
def test_ca_hepth_acceptance_criterion_1(orc, ref):
    """acceptance.cpp:94-110 on the shipped dataset: kmax 31, 16-core 96 v / 2306 arcs,
    best 31/2, and peel widths 31 pruned / unpruned (:155-177)."""
    with open(CA_HEPTH) as f:
        rg = ref.parse_text(f.read())
    g = rg.download()
    lab, kmax, rounds = orc.coreness(g)
    assert kmax == 31
    core, _ = orc.get_core(g, lab, 16)
    assert core.n == 96 and 2 * core.m == 2306
    r = orc.run(g, RunConfig(iterations=20))
    assert r.best == (31, 2) and r.max_width == 31
    r = orc.run(g, RunConfig(iterations=20, pruning="none"))
    assert r.max_width == 31
    rr = ref.run(rg, RunConfig(iterations=20))
    assert rr.trace == orc.run(g, RunConfig(iterations=20)).trace
