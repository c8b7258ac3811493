"""densegraph-b200: the B200-native hot path of arXiv 2311.04333's
prune-and-refine densest-subgraph framework.

A Python mirror of the reference's C++ API (proj/include/densegraph/*.hpp):
same names, argument meaning and error behaviour, over the C ABI of
include/dg_b200.h (libdg_b200.so, hand-written sm_100a CUDA).  The C++
drop-in headers live in include/densegraph/.

    g   = Graph.from_pairs(u, v)              # parse_edge_list's CSR build, on device
    dec = exact_coreness(g)                   # core.hpp:22
    core = get_core(g, dec, k)                # core.hpp:31
    order = load_peel_order(core, loads)      # refine.hpp:32  (Greedy++ batch peel)
    out = density_and_load_update(core, order, loads)   # refine.hpp:40 (Alg. 3)
    res = run(g, RunConfig(iterations=20))    # framework.hpp:68 (Algorithm 1)
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi
from ._abi import LIB, DgIterRecord, DgOutcome, DgRunConfig, DgRunResult, u8p, u32p, u64p

__all__ = [
    "Density", "Graph", "GraphStats", "CoreDecomposition", "LoadState", "Ordering",
    "RefineOutcome", "RunConfig", "RunResult", "RunTrace", "IterRecord", "InitRecord",
    "parse_edge_list", "parse_edge_list_file", "induced_subgraph", "exact_coreness", "approx_coreness", "get_core",
    "load_peel_order", "load_sort_order", "density_and_load_update", "charikar_peel",
    "slack_violations", "default_iterations", "run", "run_pruned", "gen_rmat", "gen_chung_lu",
    "DensegraphError", "ParseError", "EmptyGraphError", "IoError", "ParamError",
    "InvariantError", "OracleSizeError", "CacheHashError", "kNoVertex", "format_fixed6",
    "ceil_div", "ceil_scaled", "mix64",
]

kNoVertex = 0xFFFFFFFF  # graph.hpp:12


# ------------------------------------------------------------------ errors (errors.hpp:10-42)
class DensegraphError(RuntimeError):
    code = 0


class ParseError(DensegraphError):
    code = 1

    def __init__(self, line: int, what: str):
        super().__init__(f"parse error at line {line}: {what}")
        self.line = line


class EmptyGraphError(DensegraphError):
    code = 2


class IoError(DensegraphError):
    code = 3


class ParamError(DensegraphError):
    code = 4


class InvariantError(DensegraphError):
    code = 5


class OracleSizeError(DensegraphError):
    code = 6


class CacheHashError(DensegraphError):
    code = 7


class CudaError(InvariantError):
    """DG_E_CUDA / DG_E_NOMEM: rethrown as InvariantError (CLI exit 4) like any internal error."""


_ERR = {2: EmptyGraphError, 3: IoError, 4: ParamError, 5: InvariantError, 6: OracleSizeError,
        7: CacheHashError, 8: CudaError, 9: CudaError}


def _chk(st: int):
    if st:
        msg = (LIB.dg_last_error() or b"").decode()
        if st == 1:
            raise ParseError(0, msg)
        raise _ERR.get(st, InvariantError)(msg)


def _p(a, t):
    return a.ctypes.data_as(t)


# ------------------------------------------------------------------ Density (density.hpp:17-67)
@dataclass(frozen=True)
class Density:
    edges: int = 0
    verts: int = 1

    def value(self) -> float:
        return self.edges / self.verts

    def reduced(self) -> "Density":
        g = math.gcd(self.verts if self.edges == 0 else self.edges, self.verts)
        return Density(self.edges // g, self.verts // g)

    def _cmp(self, o: "Density") -> int:
        a, b = self.edges * o.verts, o.edges * self.verts
        return (a > b) - (a < b)

    def __eq__(self, o):  # exact, cross-multiplied
        return isinstance(o, Density) and self._cmp(o) == 0

    def __hash__(self):
        r = self.reduced()
        return hash((r.edges, r.verts))

    def __lt__(self, o):
        return self._cmp(o) < 0

    def __le__(self, o):
        return self._cmp(o) <= 0

    def __gt__(self, o):
        return self._cmp(o) > 0

    def __ge__(self, o):
        return self._cmp(o) >= 0


def ceil_div(a: int, b: int) -> int:  # density.hpp:40-43
    if b == 0:
        raise ParamError("division by zero")
    return a // b + (a % b != 0)


def ceil_scaled(a: Density, num: int, den: int) -> int:  # density.hpp:46-51
    if den == 0 or a.verts == 0:
        raise ParamError("division by zero")
    p, q = a.edges * num, a.verts * den
    return p // q + (p % q != 0)


def format_fixed6(d: Density) -> str:  # density.hpp:55-67, round half to even
    if d.verts == 0:
        raise ParamError("density with zero vertices")
    q, r = divmod(d.edges * 1000000, d.verts)
    if 2 * r > d.verts or (2 * r == d.verts and (q & 1)):
        q += 1
    return f"{q // 1000000}.{q % 1000000:06d}"


def mix64(x: int) -> int:  # parallel.hpp:92-97
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


# ------------------------------------------------------------------ Graph (graph.hpp:14-80)
@dataclass
class GraphStats:
    n: int = 0
    m: int = 0
    max_degree: int = 0


class Graph:
    """Device-resident CSR (offs u64[n+1], adj u32[2m], orig u64[n]); immutable."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        n, m, d = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _chk(LIB.dg_graph_info(self._h, C.byref(n), C.byref(m), C.byref(d)))
        self.n, self.m, self._maxdeg = n.value, m.value, d.value
        self._host = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            LIB.dg_graph_free(h)
            self._h = None

    # -- construction
    @classmethod
    def from_pairs(cls, u, v) -> "Graph":
        """parse_edge_list's CSR build (io.cpp:51-92) on the device."""
        u = np.ascontiguousarray(u, dtype=np.uint64)
        v = np.ascontiguousarray(v, dtype=np.uint64)
        if len(u) != len(v):
            raise ParamError("u and v differ in length")
        h = C.c_void_p()
        _chk(LIB.dg_graph_build(_p(u, u64p), _p(v, u64p), len(u), 0, C.byref(h)))
        return cls(h)

    @classmethod
    def from_device_pairs(cls, d_u: int, d_v: int, k: int) -> "Graph":
        h = C.c_void_p()
        _chk(LIB.dg_graph_build(C.cast(C.c_void_p(d_u), u64p), C.cast(C.c_void_p(d_v), u64p), k,
                                1, C.byref(h)))
        return cls(h)

    @classmethod
    def generate_rmat(cls, scale: int, samples: int, seed: int, part_cap: int = 0) -> "Graph":
        """The CSR of gen_rmat's pairs, built from the device generator without the
        pair arrays (source-range parts; RMAT-28 fits one GPU)."""
        h = C.c_void_p()
        _chk(LIB.dg_graph_generate(0, scale, samples, seed, 0.0, part_cap, C.byref(h)))
        return cls(h)

    @classmethod
    def generate_chung_lu(cls, n: int, pairs: int, seed: int, part_cap: int = 0) -> "Graph":
        """The CSR of gen_chung_lu's pairs, built from the device generator."""
        h = C.c_void_p()
        R = float(n) ** (1.0 / 11.0)
        _chk(LIB.dg_graph_generate(1, n, pairs, seed, R, part_cap, C.byref(h)))
        return cls(h)

    @classmethod
    def from_csr(cls, offs, adj, orig) -> "Graph":
        offs = np.ascontiguousarray(offs, dtype=np.uint64)
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        orig = np.ascontiguousarray(orig, dtype=np.uint64)
        h = C.c_void_p()
        _chk(LIB.dg_graph_from_csr(len(orig), _p(offs, u64p), _p(adj, u32p), _p(orig, u64p), 0,
                                   C.byref(h)))
        return cls(h)

    @classmethod
    def from_device_csr(cls, offs, adj, orig) -> "Graph":
        """CSR already on the GPU (torch CUDA tensors: int64 offsets, int32/uint32
        ids, int64 original ids); copied into the library's graph."""
        import torch
        offs = offs.to(torch.int64).contiguous()
        adj = adj.to(torch.int32).contiguous()
        orig = orig.to(torch.int64).contiguous()
        torch.cuda.synchronize()
        h = C.c_void_p()
        _chk(LIB.dg_graph_from_csr(orig.numel(), C.cast(C.c_void_p(offs.data_ptr()), u64p),
                                   C.cast(C.c_void_p(adj.data_ptr()), u32p),
                                   C.cast(C.c_void_p(orig.data_ptr()), u64p), 1, C.byref(h)))
        return cls(h)

    # -- reference field access (tests read g.offs / g.adj / g.orig)
    def download(self):
        if self._host is None:
            offs = np.zeros(self.n + 1, np.uint64)
            adj = np.zeros(max(2 * self.m, 1), np.uint32)
            orig = np.zeros(max(self.n, 1), np.uint64)
            _chk(LIB.dg_graph_download(self._h, _p(offs, u64p), _p(adj, u32p), _p(orig, u64p)))
            self._host = (offs, adj[: 2 * self.m], orig[: self.n])
        return self._host

    @property
    def offs(self):
        return self.download()[0]

    @property
    def adj(self):
        return self.download()[1]

    @property
    def orig(self):
        return self.download()[2]

    def degree(self, v: int) -> int:
        o = self.offs
        return int(o[v + 1] - o[v])

    def neighbors(self, v: int):
        o = self.offs
        return self.adj[int(o[v]):int(o[v + 1])]

    def stats(self) -> GraphStats:
        return GraphStats(self.n, self.m, self._maxdeg)

    def density(self) -> Density:
        return Density(self.m, self.n if self.n else 1)


def parse_edge_list(text, comment: str = "#") -> Graph:
    """parse_edge_list(istream) (io.hpp:18, io.cpp:25-94): the text is
    tokenised on the device with the reference's rules (csrc/parse.cu), then
    built into the CSR.  `text` is str (UTF-8 bytes, as read from a file) or
    bytes.  Errors are the reference's: ParseError at the first malformed line
    (its text, one trailing CR dropped), EmptyGraphError when no edge is left."""
    raw = bytes(text) if isinstance(text, (bytes, bytearray)) else text.encode("utf-8")
    h, bad = C.c_void_p(), C.c_uint64()
    st = LIB.dg_parse_edge_list(raw, len(raw), comment.encode("latin-1")[:1], 0, C.byref(h),
                                C.byref(bad))
    if st == ParseError.code and bad.value:
        line = raw.split(b"\n")[bad.value - 1]
        if line.endswith(b"\r"):
            line = line[:-1]
        shown = line.decode("latin-1") if isinstance(text, (bytes, bytearray)) else line.decode(
            "utf-8", "replace")
        raise ParseError(bad.value, f'expected two non-negative integers, got "{shown}"')
    _chk(st)
    return Graph(h)


def parse_edge_list_file(path: str, comment: str = "#") -> Graph:
    """parse_edge_list_file (io.hpp:19, io.cpp:96-100)."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    return parse_edge_list(raw, comment)


def induced_subgraph(g: Graph, keep, old_to_new: bool = False):
    """graph.hpp:50-80.  Returns the subgraph (and the old->new map when asked)."""
    keep = np.ascontiguousarray(np.asarray(keep) != 0, dtype=np.uint8)
    if len(keep) != g.n:
        raise InvariantError("keep mask does not match graph size")
    m = np.zeros(max(g.n, 1), np.uint32)
    h = C.c_void_p()
    _chk(LIB.dg_induced(g._h, _p(keep, u8p), C.byref(h), _p(m, u32p)))
    out = Graph(h)
    return (out, m[: g.n]) if old_to_new else out


# ------------------------------------------------------------------ core (core.hpp:9-32)
@dataclass
class CoreDecomposition:
    labels: np.ndarray
    kmax: int = 0
    peel_rounds: int = 0
    kind: str = "exact"
    c_num: int = 1
    c_den: int = 1


def exact_coreness(g: Graph) -> CoreDecomposition:
    lab = np.zeros(max(g.n, 1), np.uint32)
    kmax, rounds = C.c_uint32(), C.c_uint32()
    _chk(LIB.dg_coreness(g._h, 0, 1, 1, _p(lab, u32p), C.byref(kmax), C.byref(rounds)))
    return CoreDecomposition(lab[: g.n], kmax.value, rounds.value, "exact", 1, 1)


def approx_coreness(g: Graph, c_num: int, c_den: int) -> CoreDecomposition:
    lab = np.zeros(max(g.n, 1), np.uint32)
    kmax, rounds = C.c_uint32(), C.c_uint32()
    _chk(LIB.dg_coreness(g._h, 1, c_num, c_den, _p(lab, u32p), C.byref(kmax), C.byref(rounds)))
    return CoreDecomposition(lab[: g.n], kmax.value, rounds.value, "approximate", c_num, c_den)


def get_core(g: Graph, dec: CoreDecomposition, k: int, old_to_new: bool = False):
    if len(dec.labels) != g.n:
        raise InvariantError("core labels do not match graph size")
    lab = np.ascontiguousarray(dec.labels, dtype=np.uint32)
    m = np.zeros(max(g.n, 1), np.uint32)
    h = C.c_void_p()
    _chk(LIB.dg_get_core(g._h, _p(lab, u32p), k, C.byref(h), _p(m, u32p)))
    out = Graph(h)
    return (out, m[: g.n]) if old_to_new else out


# ------------------------------------------------------------------ refine (refine.hpp:10-49)
@dataclass
class LoadState:
    loads: np.ndarray


@dataclass
class Ordering:
    perm: np.ndarray
    kind: str = "peel_by_load"


@dataclass
class RefineOutcome:
    rho_max: Density = field(default_factory=Density)
    best_prefix: int = 0
    width: int = 0
    densities: list = field(default_factory=list)


def _loads(s) -> np.ndarray:
    return s.loads if isinstance(s, LoadState) else s


def load_peel_order(g: Graph, s, one_at_a_time: bool = False) -> Ordering:
    loads = np.ascontiguousarray(_loads(s), dtype=np.uint64)
    if len(loads) != g.n:
        raise InvariantError("load vector does not match graph size")
    perm = np.zeros(max(g.n, 1), np.uint32)
    _chk(LIB.dg_peel_order(g._h, _p(loads, u64p), int(one_at_a_time), _p(perm, u32p)))
    return Ordering(perm[: g.n], "peel_by_load")


def load_sort_order(s) -> Ordering:
    loads = np.ascontiguousarray(_loads(s), dtype=np.uint64)
    perm = np.zeros(max(len(loads), 1), np.uint32)
    _chk(LIB.dg_sort_order(len(loads), _p(loads, u64p), _p(perm, u32p)))
    return Ordering(perm[: len(loads)], "sort_by_load")


def density_and_load_update(g: Graph, order, s, want_densities: bool = False) -> RefineOutcome:
    """Algorithm 3 (refine.cpp:180-220).  `s` is a LoadState (updated in place) or
    a uint64 numpy array (updated in place)."""
    perm = np.ascontiguousarray(order.perm if isinstance(order, Ordering) else order,
                                dtype=np.uint32)
    arr = _loads(s)
    if len(perm) != g.n:
        raise InvariantError("ordering does not match graph size")
    if len(arr) != g.n:
        raise InvariantError("load vector does not match graph size")
    loads = np.ascontiguousarray(arr, dtype=np.uint64)
    suffix = np.zeros(max(g.n, 1), np.uint64) if want_densities else None
    out = DgOutcome()
    _chk(LIB.dg_density_load_update(g._h, _p(perm, u32p), _p(loads, u64p), C.byref(out),
                                     _p(suffix, u64p) if suffix is not None else None))
    if isinstance(s, LoadState):
        s.loads = loads
    elif loads is not arr:
        arr[:] = loads
    r = RefineOutcome(Density(out.rho_edges, out.rho_verts), out.best_prefix, out.width)
    if want_densities:
        r.densities = [Density(int(suffix[i]), g.n - i) for i in range(g.n)]
    return r


def charikar_peel(g: Graph) -> RefineOutcome:
    out = DgOutcome()
    _chk(LIB.dg_charikar_peel(g._h, C.byref(out)))
    return RefineOutcome(Density(out.rho_edges, out.rho_verts), out.best_prefix, out.width)


def slack_violations(order, loads, allowed_slack: int, samples: int, seed: int) -> int:
    perm = np.ascontiguousarray(order.perm if isinstance(order, Ordering) else order,
                                dtype=np.uint32)
    loads = np.ascontiguousarray(_loads(loads), dtype=np.uint64)
    out = C.c_uint64()
    _chk(LIB.dg_slack_violations(len(perm), _p(perm, u32p), _p(loads, u64p), allowed_slack,
                                 samples, seed, C.byref(out)))
    return out.value


def default_iterations(delta: int, lower_bound: float, n: int, epsilon: float,
                       cap: int = 1000) -> int:
    out = C.c_uint64()
    _chk(LIB.dg_default_iterations(delta, lower_bound, n, epsilon, cap, C.byref(out)))
    return out.value


# ------------------------------------------------------------------ framework (framework.hpp)
_ALG = {"peel": 0, "sort": 1}
_PRUNE = {"none": 0, "exact": 1, "approx": 2, "hybrid": 3}


@dataclass
class RunConfig:
    algorithm: str = "peel"
    pruning: str = "exact"
    iterations: int = 0
    epsilon: float = 0.0
    iteration_cap: int = 1000
    c_num: int = 3
    c_den: int = 2
    threads: int = 0  # accepted for API parity; no meaning on the device
    reset_loads: bool = False
    slack_samples: int = 64

    def to_c(self) -> DgRunConfig:
        return DgRunConfig(_ALG[self.algorithm], _PRUNE[self.pruning], self.iterations,
                           self.epsilon, self.iteration_cap, self.c_num, self.c_den,
                           int(self.reset_loads), self.slack_samples)


@dataclass
class IterRecord:
    iter: int
    rho: Density
    n: int
    m: int
    width: int
    ms: float
    order_ms: float = 0.0
    update_ms: float = 0.0
    batches: int = 0


@dataclass
class InitRecord:
    kmax_known: bool = False
    kmax_exact: bool = False
    kmax: int = 0
    threshold: int = 0
    pruned_n: int = 0
    pruned_m: int = 0
    coreness_ms: float = 0.0
    init_ms: float = 0.0
    peel_rounds: int = 0
    coreness_kernel_ms: float = 0.0


@dataclass
class RunTrace:
    init: InitRecord
    iters: List[IterRecord]
    slack_violations: int
    final_vertices: np.ndarray


@dataclass
class RunResult:
    best: Density
    witness: np.ndarray
    witness_edges: int
    iterations: int
    max_width: int
    total_ms: float
    trace: RunTrace
    reprunes: int = 0
    reprune_ms: float = 0.0
    device_ms: float = 0.0


@dataclass
class OracleResult:
    rho_star: Density
    witness: np.ndarray  # original ids, ascending


def brute_force_densest(g: Graph, limit: int = 22) -> OracleResult:
    """oracle.hpp:16-19: exhaustive search over every nonempty subset (device
    kernel, <= 32 vertices); ties -> fewer vertices, then the lexicographically
    smallest id set.  EmptyGraphError / OracleSizeError as the reference."""
    e, v, k = C.c_uint64(), C.c_uint64(), C.c_uint64()
    w = np.zeros(max(1, g.n), np.uint64)
    _chk(LIB.dg_brute_force_densest(g._h, limit, C.byref(e), C.byref(v),
                                    w.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(k)))
    return OracleResult(Density(e.value, v.value), w[:k.value].copy())


def set_device(device: int) -> None:
    _chk(LIB.dg_set_device(device))


def set_peel_mode(mode: int) -> None:
    """0 automatic, 1 scanning single-CTA peel, 2 cluster peel, 3 candidate-list peel
    (each whenever it fits; testing/tuning -- results are identical)."""
    _chk(LIB.dg_set_peel_mode(mode))


def launch_count() -> int:
    """Kernels of this library launched so far in this process."""
    return LIB.dg_launch_count()


def flush_l2() -> None:
    _chk(LIB.dg_flush_l2())


_DIAG = None


def diag():
    """The diagnostics library (microbenchmarks, profiling read-outs; tools only)."""
    global _DIAG
    if _DIAG is None:
        from ._abi import load_diag
        _DIAG = load_diag()
    return _DIAG


def trim_memory() -> None:
    """Return the library's cached device memory to the driver (dg_trim_memory)."""
    _chk(LIB.dg_trim_memory())


def synchronize() -> None:
    _chk(LIB.dg_synchronize())


def _run(g: Graph, cfg: Optional[RunConfig], pruned=None) -> RunResult:
    cfg = cfg or RunConfig()
    res = DgRunResult()
    # explicit T sizes the trace exactly; else the iteration cap bounds it
    cap = max(1, cfg.iterations if cfg.iterations else cfg.iteration_cap)
    trace = (DgIterRecord * cap)()
    wit = np.empty(max(g.n, 1), np.uint64)  # only the returned prefixes are read
    fin = np.empty(max(g.n, 1), np.uint64)
    c = cfg.to_c()
    if pruned is None:
        _chk(LIB.dg_run(g._h, C.byref(c), C.byref(res), trace, cap, _p(wit, u64p), g.n,
                        _p(fin, u64p), g.n))
    else:
        labels, kmax, rounds = pruned
        lab = np.ascontiguousarray(labels, dtype=np.uint32)
        if len(lab) != g.n:
            raise InvariantError("core labels do not match graph size")
        _chk(LIB.dg_run_pruned(g._h, _p(lab, u32p), kmax, rounds, C.byref(c), C.byref(res),
                               trace, cap, _p(wit, u64p), g.n, _p(fin, u64p), g.n))
    iters = [IterRecord(t.iter, Density(t.rho_edges, t.rho_verts), t.n, t.m, t.width, t.ms,
                        t.order_ms, t.update_ms, t.batches)
             for t in trace[: min(res.iterations, cap)]]
    init = InitRecord(bool(res.kmax_known), bool(res.kmax_exact), res.kmax, res.threshold,
                      res.pruned_n, res.pruned_m, res.coreness_ms, res.init_ms, res.peel_rounds,
                      res.coreness_kernel_ms)
    tr = RunTrace(init, iters, res.slack_violations, fin[: res.final_n].copy())
    return RunResult(Density(res.best_edges, res.best_verts), wit[: res.witness_size].copy(),
                     res.witness_edges, res.iterations, res.max_width, res.total_ms, tr,
                     res.reprunes, res.reprune_ms, res.device_ms)


def run(g: Graph, cfg: Optional[RunConfig] = None) -> RunResult:
    """run(g, cfg) (framework.cpp:46-180)."""
    return _run(g, cfg)


def run_pruned(core: Graph, labels, kmax: int, peel_rounds: int,
               cfg: Optional[RunConfig] = None) -> RunResult:
    """run() continued from a first prune computed elsewhere (framework.cpp:92
    onwards): `core` = get_core(input, dec, threshold(kmax)) with its labels --
    what the sharded coreness and per-shard compaction produce
    (sharded_build.run_distributed).  Same result as run() on the input."""
    return _run(core, cfg, (labels, kmax, peel_rounds))


# ------------------------------------------------------------------ synthetic inputs
def gen_rmat(scale: int, samples: int, seed: int):
    """Seeded RMAT (a=.57 b=.19 c=.19 d=.05) pairs, generated on the device (host copy)."""
    u = np.zeros(samples, np.uint64)
    v = np.zeros(samples, np.uint64)
    _chk(LIB.dg_gen_rmat(scale, samples, seed, u.ctypes.data, v.ctypes.data, 0))
    return u, v


def gen_rmat_range(scale: int, first: int, count: int, seed: int, device_ptrs=None):
    """Samples [first, first + count) of the RMAT stream: a rank's slice of a
    distributed input.  device_ptrs=(u_ptr, v_ptr) writes device buffers of
    `count` u64 entries in place (e.g. torch tensors' data_ptr()); otherwise
    host arrays are returned."""
    if device_ptrs is not None:
        _chk(LIB.dg_gen_rmat_range(scale, first, count, seed, device_ptrs[0], device_ptrs[1], 1))
        return None
    u = np.zeros(count, np.uint64)
    v = np.zeros(count, np.uint64)
    _chk(LIB.dg_gen_rmat_range(scale, first, count, seed, u.ctypes.data, v.ctypes.data, 0))
    return u, v


def gen_chung_lu(n: int, pairs: int, seed: int, n_root11: Optional[float] = None):
    R = float(n) ** (1.0 / 11.0) if n_root11 is None else n_root11
    u = np.zeros(pairs, np.uint64)
    v = np.zeros(pairs, np.uint64)
    _chk(LIB.dg_gen_chung_lu(n, pairs, R, seed, u.ctypes.data, v.ctypes.data, 0))
    return u, v


class DeviceBuffer:
    """Raw device allocation (for inputs kept resident in HBM)."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        _chk(LIB.dg_device_alloc(nbytes, C.byref(p)))
        self.ptr, self.nbytes = p.value, nbytes

    def free(self):
        if self.ptr:
            LIB.dg_device_free(C.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        self.free()
