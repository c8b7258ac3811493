"""GPU parity: the CUDA path through the C ABI against the golden fixtures
(produced by the unmodified reference) and the pinned CPU oracle.

Everything integer is compared bit-exactly: CSR arrays, core labels, kmax,
peel_rounds, Greedy++ permutations (batch and one-at-a-time), per-iteration
loads, suffix densities, widths, run traces, witnesses, final vertex sets.
"""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import graphs as G
from oracle import RunConfig as ORunConfig, gnp_edges, mix64, random_loads

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def dgraph(dg, edges):
    u, v = G.uv(edges)
    return dg.Graph.from_pairs(u, v)


def same_csr(g, h):
    return (np.array_equal(g.offs, h.offs) and np.array_equal(g.adj, h.adj)
            and np.array_equal(g.orig, h.orig))


# ------------------------------------------------------------------ CSR build
def test_build_cleanup_rules(dg):
    g = dg.Graph.from_pairs(np.array([0, 1, 3, 7], np.uint64), np.array([1, 0, 3, 5], np.uint64))
    assert (g.n, g.m) == (4, 2)
    assert g.orig.tolist() == [0, 1, 5, 7] and g.adj.tolist() == [1, 0, 3, 2]
    with pytest.raises(dg.EmptyGraphError):
        dg.Graph.from_pairs(np.array([3, 4], np.uint64), np.array([3, 4], np.uint64))
    with pytest.raises(dg.EmptyGraphError):
        dg.Graph.from_pairs(np.array([], np.uint64), np.array([], np.uint64))


@pytest.mark.parametrize("seed", range(1, 9))
def test_build_matches_oracle_gnp(dg, orc, seed):
    n = 2 + mix64(seed) % 150
    u, v = orc.gen_gnp(n, 20 + seed * 97 % 600, seed)
    assert same_csr(dg.Graph.from_pairs(u, v), orc.build(u, v))


def test_build_sparse_64bit_ids(dg, orc):
    """ids above 2^32 take the sort + binary-search relabel path."""
    rng = np.random.default_rng(5)
    ids = np.unique(rng.integers(0, 2**62, 3000, dtype=np.uint64))
    u = ids[rng.integers(0, len(ids), 20000)]
    v = ids[rng.integers(0, len(ids), 20000)]
    u[:50] = v[:50]  # self loops
    assert same_csr(dg.Graph.from_pairs(u, v), orc.build(u, v))


def test_build_rmat_and_generators(dg, orc):
    for scale, seed in ((10, 1), (14, 9)):
        du, dv = dg.gen_rmat(scale, 16 << scale, seed)
        hu, hv = orc.gen_rmat(scale, 16 << scale, seed)
        assert np.array_equal(du, hu) and np.array_equal(dv, hv)
        assert same_csr(dg.Graph.from_pairs(du, dv), orc.build(hu, hv))
    du, dv = dg.gen_chung_lu(200000, 400000, 50)
    hu, hv = orc.gen_chung_lu(200000, 400000, 50)
    assert np.array_equal(du, hu) and np.array_equal(dv, hv)


def test_from_csr_roundtrip(dg, orc):
    h = orc.build(*orc.gen_rmat(12, 16 << 12, 3))
    g = dg.Graph.from_csr(h.offs, h.adj, h.orig)
    assert same_csr(g, h) and g.stats().max_degree == h.max_degree()


# ------------------------------------------------------------------ coreness
def test_coreness_pinned(dg):
    d = dg.exact_coreness(dgraph(dg, G.clique(5)))
    assert d.labels.tolist() == [4] * 5 and d.kmax == 4 and d.peel_rounds >= 1
    assert dg.exact_coreness(dgraph(dg, G.triangle_pendant())).labels.tolist() == [2, 2, 2, 1]
    assert dg.exact_coreness(dgraph(dg, G.path_graph(4))).labels.tolist() == [1] * 4
    assert dg.approx_coreness(dgraph(dg, G.path_graph(4)), 3, 2).labels.tolist() == [1] * 4
    star = dg.exact_coreness(dgraph(dg, G.star(3000)))
    assert np.all(star.labels == 1) and star.kmax == 1
    with pytest.raises(dg.ParamError):
        dg.approx_coreness(dgraph(dg, G.clique(4)), 2, 3)


def test_coreness_golden(dg, orc, golden):
    for c in golden["coreness"]:
        g = dg.Graph.from_pairs(*orc.gen_gnp(c["n"], c["permille"], c["seed"]))
        d = dg.exact_coreness(g)
        assert (d.labels.tolist(), d.kmax, d.peel_rounds) == (c["labels"], c["kmax"], c["rounds"])
        for cn, cd in ((3, 2), (2, 1), (11, 10)):
            a = c[f"approx_{cn}_{cd}"]
            x = dg.approx_coreness(g, cn, cd)
            assert (x.labels.tolist(), x.kmax, x.peel_rounds) == (a["labels"], a["kmax"], a["rounds"])


def test_get_core_pinned(dg):
    g = dgraph(dg, G.triangle_pendant())
    c, m = dg.get_core(g, dg.exact_coreness(g), 2, old_to_new=True)
    assert (c.n, c.m) == (3, 3) and c.orig.tolist() == [0, 1, 2] and m[3] == dg.kNoVertex
    k, m = dg.induced_subgraph(dgraph(dg, G.clique(4)), [1, 1, 1, 1], old_to_new=True)
    assert (k.n, k.m) == (4, 6) and m.tolist() == [0, 1, 2, 3]
    e = dg.induced_subgraph(dgraph(dg, G.clique(4)), [0, 0, 0, 0])
    assert (e.n, e.m) == (0, 0)


def test_induced_matches_oracle_random_masks(dg, orc):
    h = orc.build(*orc.gen_rmat(13, 16 << 13, 11))
    g = dg.Graph.from_csr(h.offs, h.adj, h.orig)
    for s in range(4):
        keep = (np.arange(h.n) * 2654435761 + s * 97) % (3 + s) == 0
        a, am = dg.induced_subgraph(g, keep, old_to_new=True)
        b, bm = orc.induced(h, keep)
        assert same_csr(a, b) and np.array_equal(am, bm)


# ------------------------------------------------------------------ refinement
def test_peel_pinned(dg):
    assert dg.load_peel_order(dgraph(dg, G.path_graph(3)), np.zeros(3, np.uint64)).perm.tolist() == [0, 2, 1]
    assert dg.load_peel_order(dgraph(dg, G.clique(4)), np.zeros(4, np.uint64)).perm.tolist() == [0, 1, 2, 3]
    loads = np.array([0, 0, 0, 10], np.uint64)
    assert dg.load_peel_order(dgraph(dg, G.triangle_pendant()), loads).perm.tolist() == [0, 1, 2, 3]
    assert dg.load_sort_order(np.array([5, 2, 7, 2], np.uint64)).perm.tolist() == [1, 3, 0, 2]


def test_peel_golden(dg, orc, golden):
    for c in golden["peel"]:
        g = dg.Graph.from_pairs(*orc.gen_gnp(c["n"], c["permille"], c["seed"]))
        loads = random_loads(g.n, c["loads_maxload"], c["loads_seed"])
        assert dg.load_peel_order(g, loads).perm.tolist() == c["perm"]
        assert dg.load_peel_order(g, loads, True).perm.tolist() == c["perm_one"]
        la = loads.copy()
        out = dg.density_and_load_update(g, np.array(c["perm"], np.uint32), la, True)
        assert (out.rho_max.edges, out.rho_max.verts) == tuple(c["rho"])
        assert out.best_prefix == c["best_prefix"] and out.width == c["width"]
        assert la.tolist() == c["loads_after"]
        assert [d.edges for d in out.densities] == c["suffix_edges"]


def test_peel_shift_invariance_u64_keys(dg, orc):
    """loads beyond 2^32 force the 64-bit key path; the order must not change."""
    for seed in range(1, 6):
        g = dg.Graph.from_pairs(*G.uv(gnp_edges(60, 80, seed * 11)))
        small = random_loads(g.n, 9, seed)
        huge = small + np.uint64(1 << 40)
        spread = small.copy()
        spread[0] += np.uint64(1 << 36)  # key range itself beyond 32 bits
        a = dg.load_peel_order(g, small).perm
        assert np.array_equal(a, dg.load_peel_order(g, huge).perm)
        h = orc.build(*G.uv(gnp_edges(60, 80, seed * 11)))
        assert np.array_equal(dg.load_peel_order(g, spread).perm, orc.peel_order(h, spread))


def test_density_golden(dg, orc, golden):
    for c in golden["density"]:
        g = dg.Graph.from_pairs(*orc.gen_gnp(c["n"], c["permille"], c["seed"]))
        loads = random_loads(g.n, c["maxload"], c["loads_seed"])
        for which in ("peel", "sort"):
            e = c[which]
            o = dg.load_peel_order(g, loads) if which == "peel" else dg.load_sort_order(loads)
            assert o.perm.tolist() == e["perm"]
            la = loads.copy()
            out = dg.density_and_load_update(g, o, la, True)
            assert (out.rho_max.edges, out.rho_max.verts) == tuple(e["rho"])
            assert out.best_prefix == e["best_prefix"] and out.width == e["width"]
            assert la.tolist() == e["loads_after"]
            assert [d.edges for d in out.densities] == e["suffix_edges"]


def test_density_contract_errors(dg):
    g = dgraph(dg, G.clique(3))
    for perm in ([0, 1, 1], [0, 1, 7]):
        with pytest.raises(dg.InvariantError):
            dg.density_and_load_update(g, np.array(perm, np.uint32), np.zeros(3, np.uint64))
    with pytest.raises(dg.InvariantError):
        dg.load_peel_order(g, np.zeros(2, np.uint64))


def test_charikar_and_slack(dg):
    assert dg.charikar_peel(dgraph(dg, G.star(5))).rho_max == dg.Density(5, 6)
    assert dg.charikar_peel(dgraph(dg, G.clique(4))).rho_max == dg.Density(3, 2)
    assert dg.charikar_peel(dgraph(dg, G.triangle_pendant())).rho_max == dg.Density(1, 1)
    assert dg.slack_violations(np.arange(6, dtype=np.uint32), np.array([9, 7, 5, 3, 1, 0],
                                                                       np.uint64), 0, 4000, 1) > 0
    for seed in range(1, 6):
        g = dg.Graph.from_pairs(*G.uv(gnp_edges(50, 100, seed * 29)))
        loads = random_loads(g.n, 20, seed)
        o = dg.load_peel_order(g, loads)
        assert dg.slack_violations(o, loads, g.stats().max_degree, 2000, seed) == 0


# ------------------------------------------------------------------ framework
def _graph_for(dg, orc, name):
    if name == "biclique_k4":
        return dgraph(dg, G.biclique_with_k4())
    _, n, p, s = name.split("_")
    return dg.Graph.from_pairs(*orc.gen_gnp(int(n), int(p), int(s)))


def _cmp_run(r, e):
    assert [r.best.edges, r.best.verts] == e["best"]
    assert r.witness.tolist() == e["witness"] and r.witness_edges == e["witness_edges"]
    assert r.iterations == e["iterations"] and r.max_width == e["max_width"]
    assert r.trace.slack_violations == e["slack_violations"]
    i = r.trace.init
    assert (i.kmax_known, i.kmax_exact, i.kmax, i.threshold) == (
        e["kmax_known"], e["kmax_exact"], e["kmax"], e["threshold"])
    assert (i.pruned_n, i.pruned_m) == (e["pruned_n"], e["pruned_m"])
    assert r.trace.final_vertices.tolist() == e["final_vertices"]
    assert [[t.iter, t.rho.edges, t.rho.verts, t.n, t.m, t.width] for t in r.trace.iters] == e["trace"]


def test_run_golden(dg, orc, golden):
    cache = {}
    for c in golden["runs"]:
        g = cache.setdefault(c["graph"], _graph_for(dg, orc, c["graph"]))
        cfg = dg.RunConfig(algorithm=c["algorithm"], pruning=c["pruning"],
                           iterations=c["iterations"], reset_loads=c["reset_loads"])
        _cmp_run(dg.run(g, cfg), c["result"])


def test_run_errors(dg):
    g = dgraph(dg, G.clique(4))
    with pytest.raises(dg.ParamError):
        dg.run(g, dg.RunConfig(iterations=0, epsilon=0.0))
    r = dg.run(g, dg.RunConfig(iterations=0, epsilon=0.9))
    assert r.iterations >= 10 and len(r.trace.iters) == r.iterations


def _synthetic_pairs(orc, s):
    p = s["params"]
    if s["kind"] == "rmat":
        return orc.gen_rmat(p["scale"], p["samples"], p["seed"])
    if s["kind"] == "er_planted":
        return orc.gen_er_planted(p["n"], p["m"], p["block"], p["seed"])
    return orc.gen_chung_lu(p["n"], p["pairs"], p["seed"])


def test_synthetic_golden(dg, orc, golden):
    """RMAT / ER+planted / Chung-Lu fixtures: CSR, labels, core, 5 chained
    Greedy++ iterations (perm + loads per iteration) and a full run."""
    for s in golden["synthetic"]:
        g = dg.Graph.from_pairs(*_synthetic_pairs(orc, s))
        assert (g.n, g.m) == (s["n"], s["m"])
        assert (sha(g.offs), sha(g.adj), sha(g.orig)) == (s["offs"], s["adj"], s["orig"])
        d = dg.exact_coreness(g)
        assert (sha(d.labels), d.kmax, d.peel_rounds) == (s["labels"], s["kmax"], s["rounds"])
        core = dg.get_core(g, d, (d.kmax + 1) // 2)
        assert (core.n, core.m, sha(core.adj), sha(core.orig)) == (
            s["core_n"], s["core_m"], s["core_adj"], s["core_orig"])
        loads = np.zeros(core.n, np.uint64)
        for e in s["core_iters"]:
            o = dg.load_peel_order(core, loads)
            out = dg.density_and_load_update(core, o, loads)
            assert (sha(o.perm), sha(loads)) == (e["perm"], e["loads"])
            assert [out.rho_max.edges, out.rho_max.verts] == e["rho"] and out.width == e["width"]
        r = dg.run(g, dg.RunConfig(iterations=s["run_T"]))
        e = s["run"]
        assert [r.best.edges, r.best.verts] == e["best"] and sha(r.witness) == e["witness"]
        assert [[t.iter, t.rho.edges, t.rho.verts, t.n, t.m, t.width] for t in r.trace.iters] == e["trace"]
        assert sha(r.trace.final_vertices) == e["final_vertices"] and r.max_width == e["max_width"]


def test_medium_rmat_vs_oracle(dg, orc):
    """RMAT-17 (beyond the fixtures): every output of a T=10 run and the
    per-iteration Greedy++ state against the oracle."""
    u, v = dg.gen_rmat(17, 16 << 17, 17)
    h = orc.build(u, v)
    g = dg.Graph.from_pairs(u, v)
    assert same_csr(g, h)
    d = dg.exact_coreness(g)
    lab, kmax, rounds = orc.coreness(h)
    assert np.array_equal(d.labels, lab) and (d.kmax, d.peel_rounds) == (kmax, rounds)
    a = dg.approx_coreness(g, 3, 2)
    al, ak, ar = orc.coreness(h, True, 3, 2)
    assert np.array_equal(a.labels, al) and (a.kmax, a.peel_rounds) == (ak, ar)
    core = dg.get_core(g, d, (kmax + 1) // 2)
    hc, _ = orc.get_core(h, lab, (kmax + 1) // 2)
    assert same_csr(core, hc)
    ld, lh = np.zeros(core.n, np.uint64), np.zeros(core.n, np.uint64)
    for _ in range(6):
        p = dg.load_peel_order(core, ld).perm
        assert np.array_equal(p, orc.peel_order(hc, lh))
        dg.density_and_load_update(core, p, ld)
        _, lh, _, _ = orc.density_update(hc, p, lh)
        assert np.array_equal(ld, lh)
    for pr in ("exact", "approx", "hybrid"):
        for alg in ("peel", "sort"):
            r = dg.run(g, dg.RunConfig(algorithm=alg, pruning=pr, iterations=10))
            o = orc.run(h, ORunConfig(algorithm=alg, pruning=pr, iterations=10))
            assert (r.best.edges, r.best.verts) == o.best and np.array_equal(r.witness, o.witness)
            assert [(t.iter, t.rho.edges, t.rho.verts, t.n, t.m, t.width)
                    for t in r.trace.iters] == o.trace
            assert np.array_equal(r.trace.final_vertices, o.final_vertices)


def test_cpp_dropin_api_on_device():
    """The reference's pinned unit-test behaviour through include/densegraph/*.hpp."""
    lib = os.path.join(ROOT, "paper_2311_04333_b200")
    out = os.path.join("/tmp", "dg_test_api.bin")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), "-o", out, "-L", lib, "-ldg_b200",
           f"-Wl,-rpath,{lib}"]
    subprocess.run(cmd, check=True)
    r = subprocess.run([out], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_peel_kernel_modes_agree(dg, orc, golden, mode):
    """The scanning single-CTA (mode 1), thread-block-cluster (mode 2) and
    candidate-list (mode 3) Greedy++ kernels must all reproduce the reference
    bit for bit."""
    dg.set_peel_mode(mode)
    try:
        for c in golden["peel"][::3]:
            g = dg.Graph.from_pairs(*orc.gen_gnp(c["n"], c["permille"], c["seed"]))
            loads = random_loads(g.n, c["loads_maxload"], c["loads_seed"])
            assert dg.load_peel_order(g, loads).perm.tolist() == c["perm"]
            assert dg.load_peel_order(g, loads, True).perm.tolist() == c["perm_one"]
        u, v = dg.gen_rmat(15, 16 << 15, 23)
        g = dg.Graph.from_pairs(u, v)
        h = orc.build(u, v)
        d = dg.exact_coreness(g)
        core = dg.get_core(g, d, (d.kmax + 1) // 2)
        lab, kmax, _ = orc.coreness(h)
        hc, _ = orc.get_core(h, lab, (kmax + 1) // 2)
        ld, lh = np.zeros(core.n, np.uint64), np.zeros(core.n, np.uint64)
        for _ in range(4):
            p = dg.load_peel_order(core, ld).perm
            assert np.array_equal(p, orc.peel_order(hc, lh))
            dg.density_and_load_update(core, p, ld)
            _, lh, _, _ = orc.density_update(hc, p, lh)
            assert np.array_equal(ld, lh)
        r = dg.run(g, dg.RunConfig(iterations=6))
        o = orc.run(h, ORunConfig(iterations=6))
        assert (r.best.edges, r.best.verts) == o.best and np.array_equal(r.witness, o.witness)
        assert [(t.iter, t.rho.edges, t.rho.verts, t.n, t.m, t.width)
                for t in r.trace.iters] == o.trace
    finally:
        dg.set_peel_mode(0)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [3, 1, 2])
def test_peel_queue_paths(dg, orc, mode):
    """Corner paths against the oracle's batch peel (refine.cpp:20-156), for
    the candidate-list kernel (mode 3) and the scanning and cluster kernels
    (modes 1, 2): a tie group larger than the member staging / the CTA (1500
    members), widely spread loads (frequent window rebases), many large
    batches (slice removal) and loads whose keys cross the window."""
    rng = np.random.default_rng(7)
    cases = []
    # K_{1500,40}: 1500 vertices tie at key 40 > 1024 staged members
    e = [(a, 1500 + b) for a in range(1500) for b in range(40)]
    u, v = np.array([x for x, _ in e], np.uint64), np.array([y for _, y in e], np.uint64)
    cases.append((u, v, None))
    gu, gv = orc.gen_gnp(4000, 8, 11)
    cases.append((gu, gv, rng.integers(0, 1 << 20, 4000).astype(np.uint64)))
    cases.append((gu, gv, rng.integers(0, 64, 4000).astype(np.uint64)))
    ru, rv = orc.gen_rmat(14, 8 << 14, 5)
    cases.append((ru, rv, None))
    # 24 twins (identical neighbourhoods: the same 40 hubs of a 20K-vertex
    # G(n,p)) tie in every batch that reaches them: a tie group between the
    # cluster kernel's warp count and its staging limit (flat removal)
    bu, bv = orc.gen_gnp(20000, 1, 3)
    hubs = np.arange(0, 20000, 500, dtype=np.uint64)
    tw = np.repeat(np.arange(20000, 20024, dtype=np.uint64), len(hubs))
    cases.append((np.concatenate([bu, tw]), np.concatenate([bv, np.tile(hubs, 24)]), None))
    dg.set_peel_mode(mode)
    try:
        for u, v, loads in cases:
            g = dg.Graph.from_pairs(u, v)
            h = orc.build(u, v)
            ld = np.zeros(g.n, np.uint64) if loads is None else loads[: g.n].copy()
            lh = ld.copy()
            for _ in range(3):
                p = dg.load_peel_order(g, ld).perm
                assert np.array_equal(p, orc.peel_order(h, lh))
                dg.density_and_load_update(g, p, ld)
                _, lh, _, _ = orc.density_update(h, p, lh)
                assert np.array_equal(ld, lh)
    finally:
        dg.set_peel_mode(0)


@pytest.mark.gpu
def test_full_size_rmat22_vs_oracle(dg, orc):
    """The bench configuration itself (BASELINE configs[1]: RMAT-22, seed 22,
    67M samples) bit-exact against the oracle: CSR, coreness (labels, kmax,
    peel_rounds), and a T=3 run -- iteration 1 on the 35K core takes the
    candidate-list kernel, later ones the scanning kernel.  Plus properties
    that hold at any size: every vertex of label k has >= k neighbours of
    label >= k, and the loads gain exactly m per Greedy++ iteration."""
    u, v = dg.gen_rmat(22, 16 << 22, 22)
    hu, hv = orc.gen_rmat(22, 16 << 22, 22)
    assert np.array_equal(u, hu) and np.array_equal(v, hv)
    del hu, hv
    g = dg.Graph.from_pairs(u, v)
    h = orc.build(u, v)
    del u, v
    assert same_csr(g, h)
    d = dg.exact_coreness(g)
    lab, kmax, rounds = orc.coreness(h)
    assert np.array_equal(d.labels, lab) and (d.kmax, d.peel_rounds) == (kmax, rounds)
    # k-core certificate: label(u) >= label(v) for at least label(v) neighbours
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(h.offs).astype(np.int64))
    hi = (lab[h.adj] >= lab[src]).astype(np.int64)
    support = np.bincount(src, weights=hi, minlength=g.n)
    assert np.all(support >= lab)
    del src, hi, support
    r = dg.run(g, dg.RunConfig(iterations=3))
    o = orc.run(h, ORunConfig(iterations=3))
    assert (r.best.edges, r.best.verts) == o.best and np.array_equal(r.witness, o.witness)
    assert [(t.iter, t.rho.edges, t.rho.verts, t.n, t.m, t.width)
            for t in r.trace.iters] == o.trace
    assert np.array_equal(r.trace.final_vertices, o.final_vertices)
    core = dg.get_core(g, d, (d.kmax + 1) // 2)
    loads = np.zeros(core.n, np.uint64)
    for it in range(1, 3):
        p = dg.load_peel_order(core, loads).perm
        assert np.array_equal(np.sort(p), np.arange(core.n, dtype=p.dtype))
        dg.density_and_load_update(core, p, loads)
        assert int(loads.sum()) == it * core.m


def _parse_fixtures():
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "parse.json")) as f:
        return json.load(f)


def test_parse_edge_list_vs_reference_fixtures(dg):
    """Device tokeniser (csrc/parse.cu) against the reference parser's own
    outcomes (tests/golden/parse.json, made by make_parse_golden.py from
    io.cpp:25-94): CSR arrays, or the status and exact message."""
    for c in _parse_fixtures():
        raw = c["text"].encode("latin-1")
        if c["status"] == 0:
            g = dg.parse_edge_list(raw)
            assert (g.n, g.m) == (c["n"], c["m"]), c["name"]
            assert (sha(g.offs), sha(g.adj), sha(g.orig)) == (c["offs"], c["adj"], c["orig"]), c["name"]
            continue
        err = {1: dg.ParseError, 2: dg.EmptyGraphError}[c["status"]]
        with pytest.raises(err) as e:
            dg.parse_edge_list(raw)
        # the reference message passes a C string: compare up to a NUL byte
        assert str(e.value).split("\0")[0] == c["message"], c["name"]


def test_parse_edge_list_at_scale(dg, orc, tmp_path):
    """RMAT-18 pairs written as text (mixed blanks, CRLF, comments) parse on the
    device into the oracle's CSR; the file and stream entry points agree."""
    u, v = orc.gen_rmat(18, 16 << 18, 181)
    rng = np.random.default_rng(5)
    sep = rng.choice(np.array([" ", "\t", "  "]), len(u))
    eol = rng.choice(np.array(["\n", "\r\n"]), len(u))
    lines = np.char.add(np.char.add(np.char.add(u.astype(str), sep), v.astype(str)), eol)
    text = "# rmat18\n" + "".join(lines.tolist())
    g = dg.parse_edge_list(text)
    h = orc.build(u, v)
    assert same_csr(g, h)
    p = tmp_path / "g.txt"
    p.write_text(text)
    g2 = dg.parse_edge_list_file(str(p))
    assert (sha(g2.offs), sha(g2.adj)) == (sha(g.offs), sha(g.adj))
    with pytest.raises(dg.IoError):
        dg.parse_edge_list_file(str(tmp_path / "missing.txt"))


def test_streamed_generator_build(dg, orc):
    """dg_graph_generate (CSR straight from the device generator, in
    source-range parts) equals the pair-based build of the same samples,
    with one part and with many tiny parts."""
    for scale, cap in ((14, 0), (14, 5000), (17, 0), (17, 200000)):
        u, v = dg.gen_rmat(scale, 16 << scale, 3 * scale)
        ref = dg.Graph.from_pairs(u, v)
        g = dg.Graph.generate_rmat(scale, 16 << scale, 3 * scale, cap)
        assert (g.n, g.m) == (ref.n, ref.m)
        assert (sha(g.offs), sha(g.adj), sha(g.orig)) == (sha(ref.offs), sha(ref.adj), sha(ref.orig))
    for n, pairs, cap in ((20000, 200000, 0), (20000, 200000, 7000)):
        u, v = dg.gen_chung_lu(n, pairs, 5)
        ref = dg.Graph.from_pairs(u, v)
        g = dg.Graph.generate_chung_lu(n, pairs, 5, cap)
        assert (sha(g.offs), sha(g.adj), sha(g.orig)) == (sha(ref.offs), sha(ref.adj), sha(ref.orig))
    with pytest.raises(dg.ParamError):
        dg.Graph.generate_rmat(0, 10, 1)
    with pytest.raises(dg.EmptyGraphError):
        dg.Graph.generate_rmat(1, 0, 1)


def test_coreness_without_alive_bitmap(orc):
    """The k-core kernel's variant without the alive bitmap (DG_KCORE_BITMAP=0;
    the bitmap is the default) on a medium graph: labels, kmax, peel_rounds
    (exact and approximate) against the oracle."""
    code = r"""
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "oracle"))
import paper_2311_04333_b200 as dg
from oracle import Oracle
orc = Oracle()
u, v = orc.gen_rmat(17, 16 << 17, 99)
h = orc.build(u, v)
g = dg.Graph.from_pairs(u, v)
d = dg.exact_coreness(g)
lab, kmax, rounds = orc.coreness(h)
assert np.array_equal(d.labels, lab) and (d.kmax, d.peel_rounds) == (kmax, rounds)
a = dg.approx_coreness(g, 3, 2)
al, ak, ar = orc.coreness(h, True, 3, 2)
assert np.array_equal(a.labels, al) and (a.kmax, a.peel_rounds) == (ak, ar)
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DG_KCORE_BITMAP="0", ROOT=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [30000, 45000, 60000, 75000, 120000])
def test_peel_cluster_chunk_tiers(dg, orc, n):
    """The cluster Greedy++ kernel (mode 2) across its S1 register tiers and
    CTA sizes: per-CTA blocks of ceil(n/16) ids need 4, 6 and 8 keys per
    thread at 512 threads and 5 and 8 at 1024 threads; even counts below 8
    are rounded up to odd ones (conflict-free scans), 8 is the two-vector
    load; the peel order (batch and one-at-a-time) and loads over three
    Greedy++ iterations equal the reference restatement's (refine.cpp:20-220)."""
    u, v = orc.gen_er_planted(n, 10 * n, 60, n % 97)
    h = orc.build(u, v)
    g = dg.Graph.from_csr(h.offs, h.adj, h.orig)
    rng = np.random.default_rng(n)
    ld = rng.integers(0, 48, h.n).astype(np.uint64)
    lh = ld.copy()
    dg.set_peel_mode(2)
    try:
        for it in range(3):
            p = dg.load_peel_order(g, ld).perm
            assert np.array_equal(p, orc.peel_order(h, lh, False)), (n, it)
            dg.density_and_load_update(g, p, ld)
            _, lh, _, _ = orc.density_update(h, p, lh)
            assert np.array_equal(ld, lh), (n, it)
        p = dg.load_peel_order(g, ld, one_at_a_time=True).perm
        assert np.array_equal(p, orc.peel_order(h, lh, True)), n
    finally:
        dg.set_peel_mode(0)


@pytest.mark.gpu
@pytest.mark.parametrize("bitmap", ["1", "0"])
def test_coreness_low_list_paths(orc, bitmap):
    """Level advances through the low list (kcore.cu: theta from a sampled
    degree histogram, theta crossings staged per CTA, dry lists falling back
    to a full pass) forced on small graphs with DG_KCORE_LOWMIN, with and
    without the alive bitmap: labels, kmax, peel_rounds equal the reference
    restatement's (core.cpp:89-119) on three graph families."""
    code = r"""
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "oracle"))
import paper_2311_04333_b200 as dg
from oracle import Oracle
orc = Oracle()
for u, v in (orc.gen_rmat(18, 16 << 18, 7), orc.gen_chung_lu(300000, 2000000, 5),
             orc.gen_er_planted(80000, 600000, 300, 2)):
    h = orc.build(u, v)
    g = dg.Graph.from_pairs(u, v)
    d = dg.exact_coreness(g)
    lab, kmax, rounds = orc.coreness(h)
    assert np.array_equal(d.labels, lab) and (d.kmax, d.peel_rounds) == (kmax, rounds)
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DG_KCORE_BITMAP=bitmap, DG_KCORE_LOWMIN="1", ROOT=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


def _parse_device(dg, raw: bytes, off: int):
    """dg_parse_edge_list on device text starting `off` bytes into an allocation."""
    import ctypes as C
    buf = dg.DeviceBuffer(len(raw) + 16)
    dg._chk(dg.LIB.dg_memcpy(C.c_void_p(buf.ptr + off), raw, len(raw), 1))
    h, bad = C.c_void_p(), C.c_uint64()
    st = dg.LIB.dg_parse_edge_list(C.cast(C.c_void_p(buf.ptr + off), C.c_char_p), len(raw),
                                   b"#", 1, C.byref(h), C.byref(bad))
    return st, (dg.Graph(h) if st == 0 else None), bad.value


def test_parse_tiles_long_lines_and_alignment(dg, orc):
    """Tiled tokeniser edge cases: lines straddling 8 KB tiles at every offset,
    blank runs and comment lines far longer than the 256-byte halo, empty
    lines, CRLF, text starting at every 16-byte misalignment; the first bad
    line after long lines is reported by number."""
    rng = np.random.default_rng(17)
    u, v = orc.gen_rmat(12, 20000, 77)
    lines = []
    for a, b in zip(u.tolist(), v.tolist()):
        r = rng.random()
        if r < 0.02:
            lines.append("#" + "c" * int(rng.integers(200, 20000)))
        elif r < 0.04:
            lines.append("")
        sep = " " * int(rng.integers(1, 600)) if rng.random() < 0.05 else "\t"
        lead = " " * int(rng.integers(0, 400)) if rng.random() < 0.03 else ""
        lines.append(f"{lead}{a}{sep}{b}" + ("\r" if rng.random() < 0.3 else ""))
    text = "\n".join(lines)  # no final newline
    raw = text.encode()
    h = orc.build(u, v)
    for off in (0, 1, 3, 7, 8, 13, 15):
        st, g, _ = _parse_device(dg, raw, off)
        assert st == 0 and same_csr(g, h), off
    # a bad line after the long ones: its 1-based number
    bad_at = len(lines) - 5
    bad_lines = lines[:bad_at] + ["12 x7"] + lines[bad_at:] + ["1 2 3"]
    raw = "\n".join(bad_lines).encode()
    for off in (0, 5):
        st, g, line = _parse_device(dg, raw, off)
        assert st != 0 and line == bad_at + 1, (off, line)


@pytest.mark.gpu
def test_coreness_level_advance_paths(dg, orc):
    """Level advances of k_coreness on three graph families: wide (4 entries
    per thread) and narrow live-list passes, jumps inside and beyond the
    staged window, approximate phases for several c -- labels / kmax /
    peel_rounds equal the reference's (core.cpp:89-119)."""
    graphs = [orc.gen_rmat(18, 16 << 18, 181), orc.gen_chung_lu(200000, 1500000, 9),
              orc.gen_er_planted(60000, 400000, 200, 4)]
    for u, v in graphs:
        h = orc.build(u, v)
        g = dg.Graph.from_pairs(u, v)
        d = dg.exact_coreness(g)
        lab, k, r = orc.coreness(h)
        assert np.array_equal(d.labels, lab) and (d.kmax, d.peel_rounds) == (k, r)
        for cn, cd in ((3, 2), (2, 1), (11, 10), (5, 1)):
            a = dg.approx_coreness(g, cn, cd)
            al, ak, ar = orc.coreness(h, True, cn, cd)
            assert np.array_equal(a.labels, al) and (a.kmax, a.peel_rounds) == (ak, ar), (cn, cd)


@pytest.mark.gpu
def test_peel_large_cores_cluster_and_global_keys(dg, orc):
    """Cores beyond one SM: a ~200K-vertex core (16-CTA cluster kernel, keys in
    distributed shared memory) and a ~600K-vertex core (single-CTA kernel with
    its keys in global memory) give the oracle's peel order and loads, batch
    and (on the smaller one) one-at-a-time (refine.cpp:20-156, 180-220)."""
    for n, m in ((200000, 1600000), (600000, 4800000)):
        u, v = orc.gen_er_planted(n, m, 40, 3)
        h = orc.build(u, v)
        lab, k, _ = orc.coreness(h)
        core, _ = orc.get_core(h, lab, (k + 1) // 2)
        g = dg.Graph.from_csr(core.offs, core.adj, core.orig)
        rng = np.random.default_rng(n)
        ld = rng.integers(0, 64, core.n).astype(np.uint64)
        lh = ld.copy()
        for one in ((False, True) if n < 400000 else (False,)):
            p = dg.load_peel_order(g, ld, one_at_a_time=one).perm
            assert np.array_equal(p, orc.peel_order(core, lh, one)), (n, one)
        dg.density_and_load_update(g, p, ld)
        _, lh, _, _ = orc.density_update(core, p, lh)
        assert np.array_equal(ld, lh)


@pytest.mark.gpu
@pytest.mark.parametrize("slotq", ["256", "32", "off"])
def test_peel_cluster_slice_cache(dg, orc, slotq):
    """The cluster kernel's slice cache (peel_cluster.cuh: losing candidates'
    row slices copied into shared-memory slots with cp.async.bulk, members
    found there removed from shared memory) on a dense core, where a CTA's
    slices run to ~60 quads: default slots, slots of 32 quads (most slices do
    not fit and take the global path) and no cache give the reference
    restatement's peel order and loads (refine.cpp:20-220), batch and
    one-at-a-time."""
    n = 18000
    u, v = orc.gen_er_planted(n, 2200 * n, 500, 11)
    h = orc.build(u, v)
    g = dg.Graph.from_csr(h.offs, h.adj, h.orig)
    rng = np.random.default_rng(7)
    ld = rng.integers(0, 600, h.n).astype(np.uint64)
    lh = ld.copy()
    key = "DG_NO_SLICE_CACHE" if slotq == "off" else "DG_SLICE_SLOTQ"
    os.environ[key] = "1" if slotq == "off" else slotq
    dg.set_peel_mode(2)
    try:
        for it in range(2):
            p = dg.load_peel_order(g, ld).perm
            assert np.array_equal(p, orc.peel_order(h, lh, False)), (slotq, it)
            dg.density_and_load_update(g, p, ld)
            _, lh, _, _ = orc.density_update(h, p, lh)
            assert np.array_equal(ld, lh), (slotq, it)
        p = dg.load_peel_order(g, ld, one_at_a_time=True).perm
        assert np.array_equal(p, orc.peel_order(h, lh, True)), slotq
    finally:
        dg.set_peel_mode(0)
        del os.environ[key]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [30000, 75000])
def test_peel_cluster_64bit_offsets(dg, orc, n):
    """The cluster kernel's 64-bit row-offset instantiation (cores with 2m
    beyond 32 bits; forced here by DG_CLUSTER_O64) at 512 and 1024 threads
    gives the reference restatement's peel order, batch and one-at-a-time
    (refine.cpp:20-156)."""
    u, v = orc.gen_er_planted(n, 12 * n, 80, n % 89)
    h = orc.build(u, v)
    g = dg.Graph.from_csr(h.offs, h.adj, h.orig)
    ld = np.random.default_rng(n + 1).integers(0, 40, h.n).astype(np.uint64)
    os.environ["DG_CLUSTER_O64"] = "1"
    dg.set_peel_mode(2)
    try:
        for one in (False, True):
            p = dg.load_peel_order(g, ld, one_at_a_time=one).perm
            assert np.array_equal(p, orc.peel_order(h, ld, one)), (n, one)
    finally:
        dg.set_peel_mode(0)
        del os.environ["DG_CLUSTER_O64"]
