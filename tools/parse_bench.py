"""Edge-list text -> CSR throughput: device tokeniser (dg_parse_edge_list on
HBM-resident text) vs the reference parser (io.cpp parse_edge_list, one host
thread) on the same RMAT text.  python tools/parse_bench.py [scale]"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2311_04333_b200 as dg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
u, v = dg.gen_rmat(scale, 16 << scale, scale)
text = "".join(np.char.add(np.char.add(u.astype(str), " "), np.char.add(v.astype(str), "\n")).tolist())
raw = text.encode()
del text
L = len(raw)
dt = dg.DeviceBuffer(L)
dg._chk(dg.LIB.dg_memcpy(C.c_void_p(dt.ptr), raw, L, 1))
du, dv = dg.DeviceBuffer(8 * len(u)), dg.DeviceBuffer(8 * len(v))
dg._chk(dg.LIB.dg_memcpy(C.c_void_p(du.ptr), u.ctypes.data_as(C.c_void_p), 8 * len(u), 1))
dg._chk(dg.LIB.dg_memcpy(C.c_void_p(dv.ptr), v.ctypes.data_as(C.c_void_p), 8 * len(v), 1))


def parse_dev():
    h, bad = C.c_void_p(), C.c_uint64()
    dg._chk(dg.LIB.dg_parse_edge_list(C.cast(C.c_void_p(dt.ptr), C.c_char_p), L, b"#", 1,
                                      C.byref(h), C.byref(bad)))
    return dg.Graph(h)


def build_dev():
    return dg.Graph.from_device_pairs(du.ptr, dv.ptr, len(u))


def best(f, k=5):
    ts = []
    for _ in range(k):
        dg.synchronize()
        t0 = time.perf_counter()
        g = f()
        dg.synchronize()
        ts.append(time.perf_counter() - t0)
        del g
    return min(ts)


f = parse_dev()
assert (f.n, f.m) == (build_dev().n, build_dev().m)
tp, tb = best(parse_dev), best(build_dev)
out = {"scale": scale, "text_bytes": L, "lines": int(len(u)), "n": f.n, "m": f.m,
       "parse_plus_build_ms": round(1e3 * tp, 3), "build_only_ms": round(1e3 * tb, 3),
       "tokenise_ms": round(1e3 * (tp - tb), 3),
       "tokenise_GBps": round(L / (tp - tb) / 1e9, 1) if tp > tb else None}
try:
    from oracle import Reference, reference_available
    if reference_available():
        ref = Reference()
        b = raw
        h = C.c_void_p()
        t0 = time.perf_counter()
        st = ref.lib.ref_graph_parse_text(b, len(b), C.byref(h))
        out["reference_parse_ms"] = round(1e3 * (time.perf_counter() - t0), 1)
        out["reference_status"] = st
        ref.lib.ref_graph_free(h)
except Exception as e:  # noqa: BLE001
    out["reference_error"] = str(e)
print(json.dumps(out))
