"""Timing of the sharded pipeline stages on ONE GPU (LocalComm: all P shards
in this process, collectives are local copies) vs the single-GPU path.

python tools/sharded_probe.py [scale] [P...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2311_04333_b200 as dg
from paper_2311_04333_b200.sharded import CudaShard, LocalComm, link_local, sharded_coreness
from paper_2311_04333_b200.sharded_build import build_shards, gather_rows, shard_get_core


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
    Ps = [int(x) for x in sys.argv[2:]] or [1, 4]
    u, v = dg.gen_rmat(scale, 16 << scale, scale)
    du = torch.from_numpy(u.astype(np.int64)).cuda()
    dv = torch.from_numpy(v.astype(np.int64)).cuda()
    out = {"scale": scale, "samples": len(u)}
    t0 = t()
    g = dg.Graph.from_device_pairs(du.data_ptr(), dv.data_ptr(), len(u))
    t1 = t()
    dec = dg.exact_coreness(g)
    t2 = t()
    out["single"] = {"build_ms": (t1 - t0) * 1e3, "coreness_ms": (t2 - t1) * 1e3,
                     "n": g.n, "m": g.stats().m}
    for P in Ps:
        cuts = np.linspace(0, len(u), P + 1).astype(int)
        pairs = [(du[cuts[i]:cuts[i + 1]], dv[cuts[i]:cuts[i + 1]]) for i in range(P)]
        comm = LocalComm(P)
        for rep in range(2):  # second pass is the timed one (allocator warm)
            a = t()
            n, bounds, rows = build_shards(pairs, comm)
            b = t()
            shards = [CudaShard.from_rows(n, bounds, r, o, x) for r, (o, x, _) in enumerate(rows)]
            c = t()
            labs, kmax, rounds = sharded_coreness(shards, comm, n)
            d = t()
            shards = [CudaShard.from_rows(n, bounds, r, o, x) for r, (o, x, _) in enumerate(rows)]
            link_local(shards)
            c2 = t()
            labs2, kmax2, rounds2 = sharded_coreness(shards, comm, n, peer=True)
            d2 = t()
            assert np.array_equal(np.concatenate(labs2), np.concatenate(labs)) and rounds2 == rounds
            thresh = (kmax + 1) // 2
            _, _, crow, clab = shard_get_core(comm, bounds, rows, labs, thresh)
            e = t()
            offs, adj, orig, lab = gather_rows(comm, crow, clab)
            f = t()
            del shards
        assert np.array_equal(np.concatenate(labs), dec.labels) and kmax == dec.kmax
        out[f"P{P}"] = {"build_ms": (b - a) * 1e3, "shard_create_ms": (c - b) * 1e3,
                        "coreness_ms": (d - c) * 1e3, "coreness_peer_ms": (d2 - c2) * 1e3,
                        "rounds": rounds,
                        "get_core_ms": (e - d) * 1e3, "gather_ms": (f - e) * 1e3,
                        "core_n": len(orig), "core_arcs": int(offs[-1])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
