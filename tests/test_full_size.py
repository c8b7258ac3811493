"""Full-size parity against the REAL reference library (oracle/_ref, compiled
from /root/reference/proj/src by oracle/Makefile), through the CUDA path.

* ca-HepTh, the dataset the reference ships (acceptance.cpp:94-110,155-177):
  the file itself (tests/golden/ca-hepth.txt.gz) goes through the device
  tokeniser, then k-core / get_core / run() for every pruning mode and both
  orderings, against tests/golden/hepth.json (made by the reference,
  make_hepth_golden.py).  The CPU half checks the oracle against the same
  fixture.
* BASELINE configs[0] (C1: ER 100K/1M + planted 300, T=10), configs[2]
  (C3: Chung-Lu 50M, T=20) and configs[3] (C4: RMAT-26, T=10): the seeded
  graph built on the device, the reference run on the downloaded CSR with all
  host threads -- labels, kmax, peel_rounds, the trace, best, witness,
  witness_edges, max_width, final vertices, slack.  RMAT-26's device CSR is
  also checked against an independent host build (og_par.c) of the same
  seeded samples.
"""
import gzip
import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def hepth_text() -> bytes:
    with gzip.open(os.path.join(GOLD, "ca-hepth.txt.gz"), "rb") as f:
        return f.read()


def hepth_fixture():
    with open(os.path.join(GOLD, "hepth.json")) as f:
        return json.load(f)


def _pairs_from_text(raw: bytes):
    """Host split of the SNAP file (two integers per non-comment line)."""
    rows = [ln.split() for ln in raw.decode().splitlines() if ln and not ln.startswith("#")]
    a = np.array(rows, dtype=np.uint64)
    return a[:, 0].copy(), a[:, 1].copy()


# ---------------------------------------------------------------- CPU: the oracle
def test_hepth_fixture_pins_oracle(orc):
    from oracle import RunConfig
    fx = hepth_fixture()
    raw = hepth_text()
    assert hashlib.sha256(raw).hexdigest() == fx["sha_text"]
    g = orc.build(*_pairs_from_text(raw))
    assert (g.n, g.m, sha(g.offs), sha(g.adj), sha(g.orig)) == (
        fx["n"], fx["m"], fx["offs"], fx["adj"], fx["orig"])
    lab, kmax, rounds = orc.coreness(g)
    assert (sha(lab), kmax, rounds) == (fx["labels"], fx["kmax"], fx["peel_rounds"])
    assert kmax == 31                                        # acceptance.cpp:98
    core, _ = orc.get_core(g, lab, 16)
    assert (core.n, int(core.offs[-1])) == (96, 2306)         # acceptance.cpp:99-103
    for key, e in fx["runs"].items():
        alg, pr = key.split("/")
        r = orc.run(g, RunConfig(algorithm=alg, pruning=pr, iterations=20))
        assert list(r.best) == e["best"] and sha(r.witness) == e["witness"], key
        assert [list(t) for t in r.trace] == e["trace"], key
        assert r.max_width == e["max_width"] and r.slack_violations == e["slack_violations"]
        assert sha(r.final_vertices) == e["final_vertices"], key
    assert fx["runs"]["peel/exact"]["best"] == [31, 2]           # acceptance.cpp:100-103
    assert fx["runs"]["peel/exact"]["max_width"] == 31           # :159-176
    assert fx["runs"]["peel/none"]["max_width"] == 31


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_host_rmat_builder_matches_oracle(orc, threads):
    """og_par.c (the reference arm's input preparation) == the oracle build."""
    from oracle import rmat_graph_par
    for scale, seed in ((10, 3), (14, 26)):
        h = orc.build(*orc.gen_rmat(scale, 16 << scale, seed))
        p = rmat_graph_par(scale, 16 << scale, seed, threads)
        assert (np.array_equal(h.offs, p.offs) and np.array_equal(h.adj, p.adj)
                and np.array_equal(h.orig, p.orig))


# ---------------------------------------------------------------- GPU: the product
def _cmp_run_fixture(r, e, key):
    assert [r.best.edges, r.best.verts] == e["best"], key
    assert sha(r.witness) == e["witness"] and r.witness_edges == e["witness_edges"], key
    assert [[t.iter, t.rho.edges, t.rho.verts, t.n, t.m, t.width] for t in r.trace.iters] == e["trace"], key
    assert r.max_width == e["max_width"] and r.trace.slack_violations == e["slack_violations"], key
    assert sha(r.trace.final_vertices) == e["final_vertices"], key


@pytest.mark.gpu
def test_hepth_acceptance_through_cuda(dg):
    """Acceptance criterion 1 (acceptance.cpp:94-110,155-177) on the shipped
    dataset, parsed by the device tokeniser: kmax 31, 16-core 96 v / 2,306
    arcs, best 31/2, max_width 31 pruned and unpruned -- and every other
    output equal to the reference's."""
    fx = hepth_fixture()
    g = dg.parse_edge_list(hepth_text())
    assert (g.n, g.m, sha(g.offs), sha(g.adj), sha(g.orig)) == (
        fx["n"], fx["m"], fx["offs"], fx["adj"], fx["orig"])
    d = dg.exact_coreness(g)
    assert (sha(d.labels), d.kmax, d.peel_rounds) == (fx["labels"], 31, fx["peel_rounds"])
    core = dg.get_core(g, d, 16)
    assert (core.n, int(core.offs[-1])) == (96, 2306)
    assert (sha(core.adj), sha(core.orig)) == (fx["core16"]["adj"], fx["core16"]["orig"])
    for key, e in fx["runs"].items():
        alg, pr = key.split("/")
        r = dg.run(g, dg.RunConfig(algorithm=alg, pruning=pr, iterations=20))
        _cmp_run_fixture(r, e, key)
    r = dg.run(g, dg.RunConfig(iterations=20))
    assert (r.best.edges, r.best.verts) == (31, 2) and r.max_width == 31
    assert dg.run(g, dg.RunConfig(iterations=20, pruning="none")).max_width == 31


def _vs_reference(dg, g, T, extra_modes=()):
    """Run the CUDA path and the reference on the same CSR; compare all outputs."""
    from oracle import HostGraph, Reference, RunConfig, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libdgref.so not built")
    ref = Reference()
    ref.set_threads(os.cpu_count() or 1)
    offs, adj, orig = g.download()
    rg = ref.from_csr(HostGraph(offs, adj, orig))
    del adj
    d = dg.exact_coreness(g)
    lab, kmax, rounds = ref.coreness(rg)
    assert (d.kmax, d.peel_rounds) == (kmax, rounds)
    assert np.array_equal(d.labels, lab)
    del lab
    for alg, pr in (("peel", "exact"),) + tuple(extra_modes):
        r = dg.run(g, dg.RunConfig(algorithm=alg, pruning=pr, iterations=T))
        o = ref.run(rg, RunConfig(algorithm=alg, pruning=pr, iterations=T),
                    threads=os.cpu_count() or 1)
        key = f"{alg}/{pr}"
        assert (r.best.edges, r.best.verts) == o.best, key
        assert np.array_equal(r.witness, o.witness) and r.witness_edges == o.witness_edges, key
        assert [(t.iter, t.rho.edges, t.rho.verts, t.n, t.m, t.width)
                for t in r.trace.iters] == o.trace, key
        assert r.max_width == o.max_width and r.trace.slack_violations == o.slack_violations, key
        assert np.array_equal(r.trace.final_vertices, o.final_vertices), key
    ref.set_threads(1)
    return d


@pytest.mark.gpu
def test_c1_er_planted_vs_reference(dg, orc):
    """BASELINE configs[0]: ER n=100K, m=1M unique + planted 300-block p=.5, T=10."""
    import bench
    cfg = bench.CONFIGS["er_planted"]
    u, v = bench.host_pairs(cfg)
    g = dg.Graph.from_pairs(u, v)
    h = orc.build(u, v)
    assert np.array_equal(g.offs, h.offs) and np.array_equal(g.adj, h.adj)
    assert (g.n, g.m) == (100000, h.m) and h.m >= 1_000_000
    d = _vs_reference(dg, g, cfg["T"], (("peel", "approx"), ("peel", "hybrid"),
                                        ("sort", "exact")))
    # the planted 300-block is the densest part: the witness lies inside it
    r = dg.run(g, dg.RunConfig(iterations=cfg["T"]))
    assert r.best.verts <= 300 and d.kmax >= 100


@pytest.mark.gpu
def test_c3_chung_lu_50m_vs_reference(dg):
    """BASELINE configs[2]: Chung-Lu n=50M, 500M endpoint pairs, T=20."""
    import bench
    cfg = bench.CONFIGS["chunglu50m"]
    g = bench.device_graph(dg, cfg)
    _vs_reference(dg, g, cfg["T"])


@pytest.mark.gpu
def test_c4_rmat26_vs_reference(dg):
    """BASELINE configs[3]: RMAT scale 26 (1.07e9 samples), full core numbers
    + Greedy++ T=10.  The device CSR equals an independent host build of the
    same seeded samples; then every output equals the reference's."""
    import bench
    from oracle import rmat_graph_par
    cfg = bench.CONFIGS["rmat26"]
    g = bench.device_graph(dg, cfg)
    h = rmat_graph_par(cfg["scale"], cfg["edge_factor"] << cfg["scale"], cfg["seed"])
    offs, adj, orig = g.download()
    assert (g.n, g.m) == (h.n, h.m)
    assert np.array_equal(offs, h.offs) and np.array_equal(orig, h.orig)
    assert np.array_equal(adj, h.adj)
    del h, offs, adj, orig
    _vs_reference(dg, g, cfg["T"])
