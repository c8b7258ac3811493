"""Named test graphs as edge lists (behaviour of tests/test_util.hpp:35-64 and
test_framework.cpp:17-23 in the reference; written fresh)."""
import numpy as np


def path_graph(k):
    return [(i, i + 1) for i in range(k - 1)]


def clique(k):
    return [(i, j) for i in range(k) for j in range(i + 1, k)]


def star(leaves):
    return [(0, i) for i in range(1, leaves + 1)]


def triangle_pendant():
    return [(0, 1), (1, 2), (2, 0), (2, 3)]


def k4_pendant():
    return [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (0, 4)]


def two_triangles():
    return [(0, 1), (0, 2), (1, 2), (0, 3), (0, 4), (3, 4)]


def four_chord():
    return [(0, 1), (1, 2), (2, 3), (1, 3)]


def biclique_with_k4():
    """K_{5,45} (ids 0..49) plus a disjoint K4 (50..53)."""
    e = [(r, l) for r in range(45) for l in range(45, 50)]
    return e + [(50, 51), (50, 52), (50, 53), (51, 52), (51, 53), (52, 53)]


def uv(edges):
    u = np.array([a for a, _ in edges], dtype=np.uint64)
    v = np.array([b for _, b in edges], dtype=np.uint64)
    return u, v
