"""Device-resident sharded coreness on one GPU: P shards (CTA groups of one
launch) vs the single-GPU kernel.  python tools/sharded_persist_probe.py rmat22 [P ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2311_04333_b200 as dg  # noqa: E402
from paper_2311_04333_b200.sharded import (CudaShard, LocalComm, link_local,  # noqa: E402
                                           partition, sharded_coreness_persistent)

name = sys.argv[1]
Ps = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
g = bench.device_graph(dg, bench.CONFIGS[name])
one = dg.exact_coreness(g)
ts = []
for _ in range(3):
    r = dg.run(g, dg.RunConfig(iterations=1))
    ts.append(r.trace.init.coreness_kernel_ms)
print(f"{name}: n={g.n} m={g.m} single-GPU kernel {min(ts):.2f} ms  kmax={one.kmax} rounds={one.peel_rounds}",
      flush=True)
offs = g.offs
for P in Ps:
    b = partition(offs, P)
    best = None
    for rep in range(3):
        shards = [CudaShard(g, b, r) for r in range(P)]
        link_local(shards)
        labs, kmax, rounds, ms = sharded_coreness_persistent(shards, LocalComm(P), g.n)
        ok = np.array_equal(np.concatenate(labs), one.labels) and (kmax, rounds) == (one.kmax, one.peel_rounds)
        best = ms if best is None else min(best, ms)
        del shards
    print(f"  P={P}: {best:.2f} ms ({best / min(ts):.2f}x single), {1e3 * best / rounds:.2f} us/round, "
          f"bit-exact={ok}", flush=True)
