"""k-core kernel time (production variant) on bench configs, and labels
checked against a previous run's hash: python tools/kcore_time.py rmat22 rmat26 ..."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2311_04333_b200 as dg  # noqa: E402

for name in sys.argv[1:]:
    g = bench.device_graph(dg, bench.CONFIGS[name])
    ts = []
    for _ in range(6):
        dg.flush_l2()
        r = dg.run(g, dg.RunConfig(iterations=1))
        ts.append(r.trace.init.coreness_kernel_ms)
    d = dg.exact_coreness(g)
    h = hashlib.sha256(np.ascontiguousarray(d.labels).tobytes()).hexdigest()[:16]
    a = dg.approx_coreness(g, 3, 2)
    print(f"{name}: n={g.n} m={g.m} kmax={d.kmax} rounds={d.peel_rounds} labels={h} "
          f"approx(kmax={a.kmax},rounds={a.peel_rounds}) kcore_ms median={np.median(ts[1:]):.3f} "
          f"min={min(ts[1:]):.3f} -> {g.m / (np.median(ts[1:]) / 1e3) / 1e9:.2f} G edges/s",
          flush=True)
    del g
