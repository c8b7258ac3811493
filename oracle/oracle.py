"""CPU ORACLE bindings (TEST INFRASTRUCTURE ONLY).

ctypes + numpy front end for

* ``liboracle.so``   -- the C restatement of the reference hot path
  (oracle/dg_oracle.c; every routine cites the reference file:line), and
* ``_ref/libdgref.so`` -- the UNMODIFIED reference library compiled from
  /root/reference/proj/src (oracle/Makefile) behind oracle/ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module, and only as the checker / the CPU baseline.  The product
package ``paper_2311_04333_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdgref.so")
PAR_SO = os.path.join(HERE, "liboracle_par.so")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u8p = C.POINTER(C.c_uint8)


class OgGraph(C.Structure):
    _fields_ = [("n", C.c_uint64), ("m", C.c_uint64), ("offs", u64p), ("adj", u32p),
                ("orig", u64p)]


class OgOutcome(C.Structure):
    _fields_ = [("rho_edges", C.c_uint64), ("rho_verts", C.c_uint64),
                ("best_prefix", C.c_uint64), ("width", C.c_uint64)]


class OgConfig(C.Structure):
    _fields_ = [("algorithm", C.c_int), ("pruning", C.c_int), ("iterations", C.c_uint64),
                ("epsilon", C.c_double), ("iteration_cap", C.c_uint64), ("c_num", C.c_uint64),
                ("c_den", C.c_uint64), ("reset_loads", C.c_int), ("slack_samples", C.c_uint64)]


class OgIter(C.Structure):
    _fields_ = [("iter", C.c_uint64), ("rho_edges", C.c_uint64), ("rho_verts", C.c_uint64),
                ("n", C.c_uint64), ("m", C.c_uint64), ("width", C.c_uint64)]


class OgResult(C.Structure):
    _fields_ = [("best_edges", C.c_uint64), ("best_verts", C.c_uint64),
                ("witness_size", C.c_uint64), ("witness_edges", C.c_uint64),
                ("iterations", C.c_uint64), ("max_width", C.c_uint64),
                ("slack_violations", C.c_uint64), ("kmax_known", C.c_int),
                ("kmax_exact", C.c_int), ("kmax", C.c_uint32), ("threshold", C.c_uint32),
                ("pruned_n", C.c_uint64), ("pruned_m", C.c_uint64), ("final_n", C.c_uint64)]


ALGORITHMS = {"peel": 0, "sort": 1}
PRUNINGS = {"none": 0, "exact": 1, "approx": 2, "hybrid": 3}
ERRORS = {1: "ParseError", 2: "EmptyGraphError", 3: "IoError", 4: "ParamError",
          5: "InvariantError", 8: "MemoryError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


@dataclass
class HostGraph:
    """CSR in the reference layout (graph.hpp:24-45): offs u64[n+1], adj u32[2m], orig u64[n]."""
    offs: np.ndarray
    adj: np.ndarray
    orig: np.ndarray

    @property
    def n(self) -> int:
        return len(self.orig)

    @property
    def m(self) -> int:
        return int(self.offs[-1]) // 2

    def degrees(self) -> np.ndarray:
        return np.diff(self.offs)

    def max_degree(self) -> int:
        return int(self.degrees().max()) if self.n else 0


@dataclass
class RunConfig:
    """framework.hpp:15-25 (RunConfig)."""
    algorithm: str = "peel"
    pruning: str = "exact"
    iterations: int = 0
    epsilon: float = 0.0
    iteration_cap: int = 1000
    c_num: int = 3
    c_den: int = 2
    reset_loads: bool = False
    slack_samples: int = 64

    def to_c(self) -> OgConfig:
        return OgConfig(ALGORITHMS[self.algorithm], PRUNINGS[self.pruning], self.iterations,
                        self.epsilon, self.iteration_cap, self.c_num, self.c_den,
                        int(self.reset_loads), self.slack_samples)


@dataclass
class RunOut:
    best: tuple
    witness: np.ndarray
    witness_edges: int
    iterations: int
    max_width: int
    slack_violations: int
    kmax_known: bool
    kmax_exact: bool
    kmax: int
    threshold: int
    pruned_n: int
    pruned_m: int
    final_vertices: np.ndarray
    trace: list = field(default_factory=list)  # (iter, rho_e, rho_v, n, m, width)
    iter_ms: list = field(default_factory=list)
    times: tuple = ()


def _p(a, t):
    return a.ctypes.data_as(t)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _og(g: HostGraph) -> OgGraph:
    return OgGraph(g.n, g.m, _p(g.offs, u64p), _p(g.adj, u32p), _p(g.orig, u64p))


def _from_og(lib, og: OgGraph) -> HostGraph:
    n, m = og.n, og.m
    offs = np.ctypeslib.as_array(og.offs, (n + 1,)).copy() if n + 1 else np.zeros(1, np.uint64)
    adj = np.ctypeslib.as_array(og.adj, (2 * m,)).copy() if m else np.zeros(0, np.uint32)
    orig = np.ctypeslib.as_array(og.orig, (n,)).copy() if n else np.zeros(0, np.uint64)
    lib.og_free(C.byref(og))
    return HostGraph(offs, adj, orig)


class Oracle:
    """The C restatement (liboracle.so)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.og_last_error.restype = C.c_char_p
        L.og_mix64.restype = C.c_uint64
        L.og_mix64.argtypes = [C.c_uint64]
        L.og_max_degree.restype = C.c_uint64
        L.og_slack_violations.restype = C.c_uint64
        L.og_slack_violations.argtypes = [C.c_uint64, u32p, u64p, C.c_uint64, C.c_uint64,
                                          C.c_uint64]
        L.og_default_iterations.restype = C.c_uint64
        L.og_default_iterations.argtypes = [C.c_uint64, C.c_double, C.c_uint64, C.c_double,
                                            C.c_uint64, C.POINTER(C.c_int)]
        for fn in ("og_gen_rmat", "og_gen_gnp", "og_gen_er_planted", "og_gen_chung_lu"):
            getattr(L, fn).restype = C.c_uint64
        L.og_gen_rmat.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, u64p, u64p]
        L.og_gen_gnp.argtypes = [C.c_uint64] * 3 + [u64p, u64p, C.c_uint64]
        L.og_gen_er_planted.argtypes = [C.c_uint64] * 4 + [u64p, u64p, C.c_uint64]
        L.og_gen_chung_lu.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, u64p,
                                      u64p]

    def _chk(self, st):
        if st:
            raise OracleError(st, self.lib.og_last_error().decode())

    def mix64(self, x: int) -> int:
        return self.lib.og_mix64(x)

    # ---- graph ----
    def build(self, u, v) -> HostGraph:
        u, v = _u64(u), _u64(v)
        og = OgGraph()
        self._chk(self.lib.og_build(_p(u, u64p), _p(v, u64p), C.c_uint64(len(u)), C.byref(og)))
        return _from_og(self.lib, og)

    def induced(self, g: HostGraph, keep):
        keep = np.ascontiguousarray(keep, dtype=np.uint8)
        og, out = _og(g), OgGraph()
        m = np.zeros(max(g.n, 1), np.uint32)
        self._chk(self.lib.og_induced(C.byref(og), _p(keep, u8p), C.byref(out), _p(m, u32p)))
        return _from_og(self.lib, out), m[: g.n]

    # ---- coreness ----
    def coreness(self, g: HostGraph, approx=False, c_num=3, c_den=2):
        lab = np.zeros(max(g.n, 1), np.uint32)
        kmax, rounds = C.c_uint32(), C.c_uint32()
        og = _og(g)
        self._chk(self.lib.og_coreness(C.byref(og), int(approx), C.c_uint64(c_num),
                                       C.c_uint64(c_den), _p(lab, u32p), C.byref(kmax),
                                       C.byref(rounds)))
        return lab[: g.n], kmax.value, rounds.value

    def get_core(self, g: HostGraph, labels, k: int):
        return self.induced(g, np.asarray(labels) >= k)

    # ---- refinement ----
    def peel_order(self, g: HostGraph, loads, one_at_a_time=False):
        loads = _u64(loads)
        perm = np.zeros(max(g.n, 1), np.uint32)
        og = _og(g)
        self._chk(self.lib.og_peel_order(C.byref(og), _p(loads, u64p), int(one_at_a_time),
                                         _p(perm, u32p)))
        return perm[: g.n]

    def sort_order(self, loads):
        loads = _u64(loads)
        perm = np.zeros(max(len(loads), 1), np.uint32)
        self._chk(self.lib.og_sort_order(C.c_uint64(len(loads)), _p(loads, u64p),
                                         _p(perm, u32p)))
        return perm[: len(loads)]

    def density_update(self, g: HostGraph, perm, loads):
        """Returns (outcome dict, new loads, charges A, suffix edges B)."""
        perm = _u32(perm)
        loads = _u64(loads).copy()
        A = np.zeros(max(g.n, 1), np.uint32)
        B = np.zeros(max(g.n, 1), np.uint64)
        out = OgOutcome()
        og = _og(g)
        self._chk(self.lib.og_density_update(C.byref(og), _p(perm, u32p), _p(loads, u64p),
                                             C.byref(out), _p(A, u32p), _p(B, u64p)))
        return (dict(rho=(out.rho_edges, out.rho_verts), best_prefix=out.best_prefix,
                     width=out.width), loads, A[: g.n], B[: g.n])

    def slack_violations(self, perm, loads, allowed, samples, seed):
        perm, loads = _u32(perm), _u64(loads)
        return self.lib.og_slack_violations(len(perm), _p(perm, u32p), _p(loads, u64p),
                                            allowed, samples, seed)

    def default_iterations(self, delta, lb, n, eps, cap=1000):
        st = C.c_int()
        r = self.lib.og_default_iterations(delta, lb, n, eps, cap, C.byref(st))
        self._chk(st.value)
        return r

    # ---- framework ----
    def run(self, g: HostGraph, cfg: RunConfig) -> RunOut:
        og = _og(g)
        res = OgResult()
        cap = 1 << 16
        trace = (OgIter * cap)()
        wit = np.zeros(max(g.n, 1), np.uint64)
        fin = np.zeros(max(g.n, 1), np.uint64)
        c = cfg.to_c()
        self._chk(self.lib.og_run(C.byref(og), C.byref(c), C.byref(res), trace, C.c_uint64(cap),
                                  _p(wit, u64p), C.c_uint64(g.n), _p(fin, u64p),
                                  C.c_uint64(g.n)))
        return _runout(res, trace, wit, fin)

    # ---- generators ----
    def gen_rmat(self, scale, samples, seed):
        u = np.zeros(samples, np.uint64)
        v = np.zeros(samples, np.uint64)
        self.lib.og_gen_rmat(scale, samples, seed, _p(u, u64p), _p(v, u64p))
        return u, v

    def gen_gnp(self, n, permille, seed):
        cap = max(1, n * (n - 1) // 2)
        u = np.zeros(cap, np.uint64)
        v = np.zeros(cap, np.uint64)
        c = self.lib.og_gen_gnp(n, permille, seed, _p(u, u64p), _p(v, u64p), cap)
        return u[:c], v[:c]

    def gen_er_planted(self, n, m_target, block, seed):
        cap = m_target + block * (block - 1) // 2
        u = np.zeros(cap, np.uint64)
        v = np.zeros(cap, np.uint64)
        c = self.lib.og_gen_er_planted(n, m_target, block, seed, _p(u, u64p), _p(v, u64p), cap)
        return u[:c], v[:c]

    def gen_chung_lu(self, n, pairs, seed):
        u = np.zeros(pairs, np.uint64)
        v = np.zeros(pairs, np.uint64)
        self.lib.og_gen_chung_lu(n, pairs, chung_lu_root(n), seed, _p(u, u64p), _p(v, u64p))
        return u, v


def rmat_graph_par(scale: int, samples: int, seed: int, threads: int = 0) -> HostGraph:
    """Seeded RMAT graph built on the host with OpenMP (og_par.c): the CSR of
    ``Oracle().build(*Oracle().gen_rmat(scale, samples, seed))``, fast enough
    for RMAT-26.  Input preparation for the reference arm only."""
    if not os.path.exists(PAR_SO):
        raise FileNotFoundError(f"{PAR_SO} missing: run `make -C oracle`")
    lib = C.CDLL(PAR_SO)
    lib.ogp_rmat_graph.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_int,
                                   C.POINTER(OgGraph)]
    og = OgGraph()
    st = lib.ogp_rmat_graph(scale, samples, seed, threads, C.byref(og))
    if st:
        raise OracleError(st, "ogp_rmat_graph failed")
    return _from_og(lib, og)


def chung_lu_root(n: int) -> float:
    """R = n^(1/11), the one transcendental constant of the Chung-Lu stream,
    computed once on the host and passed to both host and device generators."""
    return float(n) ** (1.0 / 11.0)


def _runout(res, trace, wit, fin, iter_ms=None, times=None) -> RunOut:
    nt = min(res.iterations, len(trace))
    tr = [(t.iter, t.rho_edges, t.rho_verts, t.n, t.m, t.width) for t in trace[:nt]]
    return RunOut(best=(res.best_edges, res.best_verts), witness=wit[: res.witness_size].copy(),
                  witness_edges=res.witness_edges, iterations=res.iterations,
                  max_width=res.max_width, slack_violations=res.slack_violations,
                  kmax_known=bool(res.kmax_known), kmax_exact=bool(res.kmax_exact),
                  kmax=res.kmax, threshold=res.threshold, pruned_n=res.pruned_n,
                  pruned_m=res.pruned_m, final_vertices=fin[: res.final_n].copy(), trace=tr,
                  iter_ms=list(iter_ms[:nt]) if iter_ms is not None else [],
                  times=tuple(times) if times is not None else ())


class RefGraph:
    def __init__(self, ref: "Reference", h):
        self.ref, self.h = ref, h

    def __del__(self):
        if self.h:
            self.ref.lib.ref_graph_free(self.h)
            self.h = None

    def info(self):
        n, m, d = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.ref.lib.ref_graph_info(self.h, C.byref(n), C.byref(m), C.byref(d))
        return n.value, m.value, d.value

    def download(self) -> HostGraph:
        n, m, _ = self.info()
        offs = np.zeros(n + 1, np.uint64)
        adj = np.zeros(max(2 * m, 1), np.uint32)
        orig = np.zeros(max(n, 1), np.uint64)
        self.ref.lib.ref_graph_download(self.h, _p(offs, u64p), _p(adj, u32p), _p(orig, u64p))
        return HostGraph(offs, adj[: 2 * m], orig[:n])


class Reference:
    """The real reference library (oracle/_ref/libdgref.so) through its C++ API."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_graph_info.argtypes = [C.c_void_p, u64p, u64p, u64p]
        L.ref_graph_download.argtypes = [C.c_void_p, u64p, u32p, u64p]
        L.ref_graph_parse_text.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_graph_from_csr.argtypes = [C.c_uint64, u64p, u32p, u64p, C.POINTER(C.c_void_p)]
        L.ref_coreness.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, u32p,
                                   C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.ref_get_core.argtypes = [C.c_void_p, u32p, C.c_uint32, C.POINTER(C.c_void_p), u32p]
        L.ref_peel_order.argtypes = [C.c_void_p, u64p, C.c_int, u32p]
        L.ref_sort_order.argtypes = [C.c_uint64, u64p, u32p]
        L.ref_density_update.argtypes = [C.c_void_p, u32p, u64p, C.POINTER(OgOutcome), u64p]
        L.ref_slack_violations.restype = C.c_uint64
        L.ref_slack_violations.argtypes = [C.c_uint64, u32p, u64p, C.c_uint64, C.c_uint64,
                                           C.c_uint64]
        L.ref_default_iterations.argtypes = [C.c_uint64, C.c_double, C.c_uint64, C.c_double,
                                             C.c_uint64, u64p]
        L.ref_run.argtypes = [C.c_void_p, C.POINTER(OgConfig), C.c_int, C.POINTER(OgResult),
                              C.POINTER(OgIter), C.c_uint64, C.POINTER(C.c_double), u64p,
                              C.c_uint64, u64p, C.c_uint64, C.POINTER(C.c_double)]
        L.ref_max_threads.restype = C.c_int
        L.ref_set_threads.argtypes = [C.c_int]

    def _chk(self, st):
        if st:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def set_threads(self, t: int):
        self.lib.ref_set_threads(t)

    def max_threads(self) -> int:
        return self.lib.ref_max_threads()

    def parse_text(self, text: str) -> RefGraph:
        b = text.encode()
        h = C.c_void_p()
        self._chk(self.lib.ref_graph_parse_text(b, len(b), C.byref(h)))
        return RefGraph(self, h)

    def parse_pairs(self, u, v) -> RefGraph:
        """The reference's own CSR build (io.cpp parse_edge_list) on "u v" lines."""
        txt = "".join(f"{a} {b}\n" for a, b in zip(np.asarray(u).tolist(), np.asarray(v).tolist()))
        return self.parse_text(txt)

    def from_csr(self, g: HostGraph) -> RefGraph:
        h = C.c_void_p()
        self._chk(self.lib.ref_graph_from_csr(g.n, _p(_u64(g.offs), u64p), _p(_u32(g.adj), u32p),
                                              _p(_u64(g.orig), u64p), C.byref(h)))
        return RefGraph(self, h)

    def coreness(self, rg: RefGraph, approx=False, c_num=3, c_den=2):
        n, _, _ = rg.info()
        lab = np.zeros(max(n, 1), np.uint32)
        kmax, rounds = C.c_uint32(), C.c_uint32()
        self._chk(self.lib.ref_coreness(rg.h, int(approx), c_num, c_den, _p(lab, u32p),
                                        C.byref(kmax), C.byref(rounds)))
        return lab[:n], kmax.value, rounds.value

    def get_core(self, rg: RefGraph, labels, k):
        n, _, _ = rg.info()
        labels = _u32(labels)
        m = np.zeros(max(n, 1), np.uint32)
        h = C.c_void_p()
        self._chk(self.lib.ref_get_core(rg.h, _p(labels, u32p), k, C.byref(h), _p(m, u32p)))
        return RefGraph(self, h), m[:n]

    def peel_order(self, rg: RefGraph, loads, one_at_a_time=False):
        n, _, _ = rg.info()
        loads = _u64(loads)
        perm = np.zeros(max(n, 1), np.uint32)
        self._chk(self.lib.ref_peel_order(rg.h, _p(loads, u64p), int(one_at_a_time),
                                          _p(perm, u32p)))
        return perm[:n]

    def sort_order(self, loads):
        loads = _u64(loads)
        perm = np.zeros(max(len(loads), 1), np.uint32)
        self._chk(self.lib.ref_sort_order(len(loads), _p(loads, u64p), _p(perm, u32p)))
        return perm[: len(loads)]

    def density_update(self, rg: RefGraph, perm, loads):
        n, _, _ = rg.info()
        perm = _u32(perm)
        loads = _u64(loads).copy()
        B = np.zeros(max(n, 1), np.uint64)
        out = OgOutcome()
        self._chk(self.lib.ref_density_update(rg.h, _p(perm, u32p), _p(loads, u64p),
                                              C.byref(out), _p(B, u64p)))
        return (dict(rho=(out.rho_edges, out.rho_verts), best_prefix=out.best_prefix,
                     width=out.width), loads, B[:n])

    def slack_violations(self, perm, loads, allowed, samples, seed):
        perm, loads = _u32(perm), _u64(loads)
        return self.lib.ref_slack_violations(len(perm), _p(perm, u32p), _p(loads, u64p),
                                             allowed, samples, seed)

    def default_iterations(self, delta, lb, n, eps, cap=1000):
        out = C.c_uint64()
        self._chk(self.lib.ref_default_iterations(delta, lb, n, eps, cap, C.byref(out)))
        return out.value

    def run(self, rg: RefGraph, cfg: RunConfig, threads: int = 0) -> RunOut:
        n, _, _ = rg.info()
        res = OgResult()
        cap = 1 << 16
        trace = (OgIter * cap)()
        ms = (C.c_double * cap)()
        times = (C.c_double * 3)()
        wit = np.zeros(max(n, 1), np.uint64)
        fin = np.zeros(max(n, 1), np.uint64)
        c = cfg.to_c()
        self._chk(self.lib.ref_run(rg.h, C.byref(c), threads, C.byref(res), trace, cap, ms,
                                   _p(wit, u64p), n, _p(fin, u64p), n, times))
        return _runout(res, trace, wit, fin, list(ms), list(times))


def reference_available() -> bool:
    return os.path.exists(REF_SO)


_ORACLE = None


def oracle() -> Oracle:
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = Oracle()
    return _ORACLE


def mix64(x: int) -> int:
    """splitmix64, parallel.hpp:92-97 (pure Python, for seeded test sizes)."""
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def gnp_edges(n: int, permille: int, seed: int):
    """tests/test_util.hpp:67-79 random_edges, as (u, v) lists (pure Python)."""
    e = [(i, j) for i in range(n) for j in range(i + 1, n)
         if mix64(seed ^ ((i * 0x100000001B3 + j) & ((1 << 64) - 1))) % 1000 < permille]
    if not e:
        e = [(0, 1 if n > 1 else 2)]
    return e


def random_loads(n: int, maxload: int, seed: int) -> np.ndarray:
    """tests/test_util.hpp:81-86 random_loads."""
    M = (1 << 64) - 1
    return np.array([mix64(seed ^ ((v * 31 + 7) & M)) % (maxload + 1) for v in range(n)],
                    dtype=np.uint64)


def reduced(e: int, v: int):
    """Density::reduced, density.hpp:23-26."""
    g = math.gcd(v if e == 0 else e, v)
    return (e // g, v // g)
