#!/usr/bin/env python3
"""Generate tests/golden/golden.json from the REAL reference library.

Runs in the build container only (needs oracle/_ref/libdgref.so, which
oracle/Makefile compiles from /root/reference/proj/src).  Every graph is
built by the reference's own parser (io.cpp parse_edge_list) from seeded
edge lists, and every output is what the unmodified reference computes:

* coreness suites  -- test_core.cpp:30-41 and acceptance.cpp:210-217 recipes
* peel-order suites -- test_refine.cpp:50-59 recipe (batch + one-at-a-time)
* density suites    -- test_refine.cpp:123-150 recipe (peel and sort orders)
* framework runs    -- test_framework.cpp:82-140 graphs, all modes
* medium synthetic  -- RMAT / ER+planted / Chung-Lu (our seeded generators),
                       full run traces plus sha256 of labels / per-iteration
                       perm and loads, for size-independent GPU checks.

Usage:  python tests/golden/make_golden.py   (writes tests/golden/golden.json)
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import (Oracle, Reference, RunConfig, gnp_edges, mix64,  # noqa: E402
                    random_loads)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def L(a):
    return [int(x) for x in np.asarray(a).tolist()]


def run_dict(r):
    return dict(best=list(r.best), witness=L(r.witness), witness_edges=r.witness_edges,
                iterations=r.iterations, max_width=r.max_width,
                slack_violations=r.slack_violations, kmax_known=r.kmax_known,
                kmax_exact=r.kmax_exact, kmax=r.kmax, threshold=r.threshold,
                pruned_n=r.pruned_n, pruned_m=r.pruned_m,
                final_vertices=L(r.final_vertices), trace=[list(t) for t in r.trace])


def biclique_with_k4():
    e = [(r, l) for r in range(45) for l in range(45, 50)]
    e += [(50, 51), (50, 52), (50, 53), (51, 52), (51, 53), (52, 53)]
    return e


def main():
    ref = Reference()
    orc = Oracle()
    ref.set_threads(1)
    G = {"coreness": [], "peel": [], "density": [], "runs": [], "synthetic": []}

    def parse(edges):
        u = [a for a, _ in edges]
        v = [b for _, b in edges]
        return ref.parse_pairs(u, v)

    # coreness: test_core.cpp:30-41 (60 graphs) + acceptance.cpp:210-217 (200 graphs)
    recipes = [(2 + mix64(s) % 99, 20 + mix64(s * 7 + 1) % 300, s) for s in range(1, 61)]
    recipes += [(2 + mix64(s * 31 + 11) % 99, 20 + s * 29 % 500, s ^ 0xC0DE) for s in range(1, 201)]
    for n, p, seed in recipes:
        rg = parse(gnp_edges(n, p, seed))
        lab, kmax, rounds = ref.coreness(rg)
        ent = dict(n=n, permille=p, seed=seed, labels=L(lab), kmax=kmax, rounds=rounds)
        for cn, cd in ((3, 2), (2, 1), (11, 10)):
            al, ak, ar = ref.coreness(rg, True, cn, cd)
            ent[f"approx_{cn}_{cd}"] = dict(labels=L(al), kmax=ak, rounds=ar)
        G["coreness"].append(ent)

    # peel orders: test_refine.cpp:50-59
    for seed in range(1, 41):
        n = 2 + mix64(seed * 5) % 99
        p = 15 + seed * 17 % 400
        rg = parse(gnp_edges(n, p, seed))
        gn = rg.info()[0]
        loads = random_loads(gn, 0 if seed % 3 == 0 else 12, seed ^ 0xF00D)
        perm = ref.peel_order(rg, loads)
        one = ref.peel_order(rg, loads, True)
        out, new_loads, B = ref.density_update(rg, perm, loads)
        G["peel"].append(dict(n=n, permille=p, seed=seed, loads_maxload=0 if seed % 3 == 0 else 12,
                              loads_seed=seed ^ 0xF00D, perm=L(perm), perm_one=L(one),
                              rho=list(out["rho"]), best_prefix=out["best_prefix"],
                              width=out["width"], loads_after=L(new_loads), suffix_edges=L(B)))

    # per-position densities: test_refine.cpp:123-150 and acceptance.cpp:222-236
    rec = [(2 + mix64(s * 3 + 1) % 60, 30 + s * 23 % 300, s ^ 0xBEEF, 6, s) for s in range(1, 26)]
    rec += [(2 + mix64(s * 77 + 5) % 199, 15 + s % 120, s ^ 0xD1CE, 10, s) for s in range(1, 101)]
    for n, p, seed, maxload, lseed in rec:
        rg = parse(gnp_edges(n, p, seed))
        gn = rg.info()[0]
        loads = random_loads(gn, maxload, lseed)
        ent = dict(n=n, permille=p, seed=seed, maxload=maxload, loads_seed=lseed)
        for which in ("peel", "sort"):
            perm = ref.peel_order(rg, loads) if which == "peel" else ref.sort_order(loads)
            out, new_loads, B = ref.density_update(rg, perm, loads)
            ent[which] = dict(perm=L(perm), rho=list(out["rho"]), best_prefix=out["best_prefix"],
                              width=out["width"], loads_after=L(new_loads), suffix_edges=L(B))
        G["density"].append(ent)

    # framework runs: test_framework.cpp:82-140 graphs plus the K4 / tie cases
    graphs = [("biclique_k4", biclique_with_k4())]
    graphs += [(f"gnp_{40 + s * 7}_{80 + s * 53 % 500}_{s * 3}",
                gnp_edges(40 + s * 7, 80 + s * 53 % 500, s * 3)) for s in range(1, 13)]
    graphs += [("gnp_500_25_31415", gnp_edges(500, 25, 31415))]
    for name, edges in graphs:
        rg = parse(edges)
        for alg in ("peel", "sort"):
            for pr in ("exact", "hybrid", "approx", "none"):
                for T, reset in ((8, False), (3, True)):
                    cfg = RunConfig(algorithm=alg, pruning=pr, iterations=T, reset_loads=reset)
                    r = ref.run(rg, cfg, threads=1)
                    G["runs"].append(dict(graph=name, edges=[list(e) for e in edges]
                                          if name == "biclique_k4" else None,
                                          algorithm=alg, pruning=pr, iterations=T,
                                          reset_loads=reset, result=run_dict(r)))

    # medium synthetic: seeded generators -> reference CSR build -> reference outputs
    synth = [
        ("rmat", dict(scale=12, samples=16 << 12, seed=7), 10),
        ("rmat", dict(scale=15, samples=16 << 15, seed=15), 10),
        ("er_planted", dict(n=20000, m=200000, block=150, seed=1), 10),
        ("chung_lu", dict(n=100000, pairs=1000000, seed=50), 5),
    ]
    for kind, kw, T in synth:
        if kind == "rmat":
            u, v = orc.gen_rmat(kw["scale"], kw["samples"], kw["seed"])
        elif kind == "er_planted":
            u, v = orc.gen_er_planted(kw["n"], kw["m"], kw["block"], kw["seed"])
        else:
            u, v = orc.gen_chung_lu(kw["n"], kw["pairs"], kw["seed"])
        rg = ref.parse_pairs(u, v)
        g = rg.download()
        lab, kmax, rounds = ref.coreness(rg)
        thresh = (kmax + 1) // 2
        core, _ = ref.get_core(rg, lab, thresh)
        cg = core.download()
        loads = np.zeros(cg.n, np.uint64)
        iters = []
        for it in range(1, 6):  # manual Greedy++ loop on the ceil(kmax/2)-core
            perm = ref.peel_order(core, loads)
            out, loads, B = ref.density_update(core, perm, loads)
            iters.append(dict(perm=sha(perm), loads=sha(loads), rho=list(out["rho"]),
                              best_prefix=out["best_prefix"], width=out["width"]))
        r = ref.run(rg, RunConfig(iterations=T), threads=1)
        G["synthetic"].append(dict(kind=kind, params=kw, n=g.n, m=g.m, offs=sha(g.offs),
                                   adj=sha(g.adj), orig=sha(g.orig), labels=sha(lab), kmax=kmax,
                                   rounds=rounds, core_n=cg.n, core_m=cg.m, core_offs=sha(cg.offs),
                                   core_adj=sha(cg.adj), core_orig=sha(cg.orig), core_iters=iters,
                                   run_T=T, run=dict(run_dict(r), witness=sha(r.witness),
                                                     final_vertices=sha(r.final_vertices))))
        print(kind, kw, "n", g.n, "m", g.m, "kmax", kmax, "rounds", rounds, "core", cg.n, cg.m,
              "best", r.best, flush=True)

    with open(OUT, "w") as f:
        json.dump(G, f, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
