"""A/B of Greedy++ ordering kernels on one graph, one process.

python tools/peel_ab.py [scale] [T] [modes, e.g. 1,4]

Per mode: best-of-3 dg.run(T) with that dg_set_peel_mode; prints the
iteration-2+ order time per batch (the pruned core) and iteration 1's.
Set env vars between runs by listing `mode:VAR=1` (e.g. 4:DG_GMIN_NOPF=1).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04333_b200 as dg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
T = int(sys.argv[2]) if len(sys.argv) > 2 else 20
modes = (sys.argv[3] if len(sys.argv) > 3 else "1,4").split(",")
g = dg.Graph.generate_rmat(scale, 16 << scale, scale)
ref = None
for spec in modes * 2:
    mode, _, env = spec.partition(":")
    if env:
        k, _, v = env.partition("=")
        os.environ[k] = v
    dg.set_peel_mode(int(mode))
    best = None
    for _ in range(3):
        r = dg.run(g, dg.RunConfig(iterations=T))
        it = r.trace.iters
        o1 = it[0].order_ms
        orest = sum(x.order_ms for x in it[1:])
        brest = sum(x.batches for x in it[1:])
        if best is None or orest < best[1]:
            best = (o1, orest, brest, it[0].batches)
    key = (r.best.edges, r.best.verts, tuple(r.witness[:16]))
    ref = ref or key
    assert key == ref, "results differ between modes"
    o1, orest, brest, b1 = best
    print(f"mode {spec:>16}: it1 {o1:7.3f} ms ({1e3 * o1 / b1:.2f} us/batch)  "
          f"it2+ {orest:8.3f} ms ({1e3 * orest / max(1, brest):.3f} us/batch, {brest} batches)",
          flush=True)
    if env:
        del os.environ[env.partition("=")[0]]
dg.set_peel_mode(0)
