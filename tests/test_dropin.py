"""The drop-in boundary, exercised the way the reference's own callers use it.

* The reference's OWN unit tests (proj/tests/test_core.cpp, test_refine.cpp,
  test_graph.cpp, test_framework.cpp, test_oracle.cpp), compiled unchanged
  against include/densegraph/*.hpp + libdg_b200.so by `make -C oracle
  ref-tests` (in the build container; the binary travels with the snapshot),
  run on the device.
* The exhaustive-search oracle (oracle.hpp:16-19) on the device against a
  vectorised numpy enumeration of every subset.
"""
import os
import subprocess

import numpy as np
import pytest

import graphs as G
from oracle import gnp_edges, mix64

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests")


@pytest.mark.gpu
def test_reference_unit_tests_on_device():
    if not os.path.exists(REF_TESTS):
        pytest.skip("oracle/_ref/ref_unit_tests not built (needs /root/reference at build time)")
    r = subprocess.run([REF_TESTS], capture_output=True, text=True, timeout=900,
                       cwd="/tmp")
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert "| 0 failed" in r.stdout and "test cases: 50" in r.stdout, tail


def _numpy_densest(n, edges, orig):
    """Every nonempty subset at once: (density, -verts, lexicographic) maximum."""
    adjm = np.zeros(n, np.int64)
    for a, b in edges:
        adjm[a] |= 1 << b
        adjm[b] |= 1 << a
    masks = np.arange(1, 1 << n, dtype=np.int64)
    e2 = np.zeros(len(masks), np.int64)
    for v in range(n):
        inv = (masks >> v) & 1
        e2 += inv * np.bitwise_count(adjm[v] & masks).astype(np.int64)
    e = e2 // 2
    k = np.bitwise_count(masks).astype(np.int64)
    # best density by exact cross-multiplication: scan candidates
    best = 0
    for i in range(1, len(masks)):
        a, b = best, i
        l, r = e[b] * k[a], e[a] * k[b]
        if l > r or (l == r and (k[b] < k[a] or (k[b] == k[a] and _lex(masks[b], masks[a])))):
            best = i
    m = int(masks[best])
    wit = [orig[v] for v in range(n) if (m >> v) & 1]
    from math import gcd
    g = gcd(int(e[best]), int(k[best]))
    return (int(e[best]) // g, int(k[best]) // g), wit


def _lex(a, b):
    d = int(a) ^ int(b)
    return (int(a) & (d & -d)) != 0


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(1, 9))
def test_brute_force_densest_vs_enumeration(dg, seed):
    n = 3 + mix64(seed) % 12
    edges = gnp_edges(n, 150 + seed * 97 % 700, seed * 3)
    if not edges:
        edges = [(0, 1)]
    g = dg.Graph.from_pairs(*G.uv(edges))
    ids = {v: i for i, v in enumerate(g.orig.tolist())}
    dense = [(ids[a], ids[b]) for a, b in edges if a != b]
    want_rho, want_w = _numpy_densest(g.n, dense, g.orig.tolist())
    r = dg.brute_force_densest(g)
    assert (r.rho_star.edges, r.rho_star.verts) == want_rho
    assert r.witness.tolist() == want_w


@pytest.mark.gpu
def test_brute_force_densest_pinned_and_limits(dg):
    # test_oracle.cpp:35-63 behaviour: K4 whole, triangle+pendant -> triangle,
    # disjoint equal triangles -> the lexicographically first, K5 reduced 2/1
    r = dg.brute_force_densest(dg.Graph.from_pairs(*G.uv(G.clique(4))))
    assert (r.rho_star.edges, r.rho_star.verts) == (3, 2) and r.witness.tolist() == [0, 1, 2, 3]
    tp = [(0, 1), (1, 2), (2, 0), (2, 3)]
    r = dg.brute_force_densest(dg.Graph.from_pairs(*G.uv(tp)))
    assert (r.rho_star.edges, r.rho_star.verts) == (1, 1) and r.witness.tolist() == [0, 1, 2]
    two = [(0, 1), (0, 2), (1, 2), (3, 4), (3, 5), (4, 5)]
    r = dg.brute_force_densest(dg.Graph.from_pairs(*G.uv(two)))
    assert r.witness.tolist() == [0, 1, 2]
    r = dg.brute_force_densest(dg.Graph.from_pairs(*G.uv(G.clique(5))))
    assert (r.rho_star.edges, r.rho_star.verts) == (2, 1)
    # original ids in the witness; 22 and 32 vertices (2^32 - 1 subsets)
    r = dg.brute_force_densest(dg.Graph.from_pairs(np.array([7, 7, 900], np.uint64),
                                                   np.array([900, 10, 10], np.uint64)))
    assert r.witness.tolist() == [7, 10, 900]
    for n, lim in ((22, 22), (32, 32)):
        e = [(i, (i + 1) % n) for i in range(n)] + [(0, 2), (0, 3), (2, 3), (1, 3)]
        g = dg.Graph.from_pairs(*G.uv(e))
        r = dg.brute_force_densest(g, lim)
        assert (r.rho_star.edges, r.rho_star.verts) == (3, 2)  # K4 on {0,1,2,3}
        assert r.witness.tolist() == [0, 1, 2, 3]
    star = [(0, i) for i in range(1, 23)]
    with pytest.raises(dg.OracleSizeError):
        dg.brute_force_densest(dg.Graph.from_pairs(*G.uv(star)))
    with pytest.raises(dg.OracleSizeError):
        dg.brute_force_densest(dg.Graph.from_pairs(*G.uv(star[:10])), 10)
    dg.brute_force_densest(dg.Graph.from_pairs(*G.uv(star[:10])), 11)
