#!/usr/bin/env python3
"""Generate the ca-HepTh acceptance fixture from the REAL reference library.

The reference ships one dataset, proj/data/ca-hepth.txt (SNAP CA-HepTh,
acceptance criterion 1: proj/tests/acceptance.cpp:94-110,155-177).  This
script (build container only: needs /root/reference and oracle/_ref) stores

* tests/golden/ca-hepth.txt.gz -- the dataset file itself, byte for byte
  (gzip), so GPU boxes without /root/reference can run the acceptance case
  through the device tokeniser;
* tests/golden/hepth.json      -- what the UNMODIFIED reference computes on it:
  the parsed CSR (sha256), labels / kmax / peel_rounds, the 16-core, and
  run() outcomes (T=20) for every pruning mode and both orderings.

Usage:  python tests/golden/make_hepth_golden.py
"""
import gzip
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Reference, RunConfig  # noqa: E402

SRC = "/root/reference/proj/data/ca-hepth.txt"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def main():
    raw = open(SRC, "rb").read()
    with gzip.GzipFile(os.path.join(HERE, "ca-hepth.txt.gz"), "wb", mtime=0) as f:
        f.write(raw)
    ref = Reference()
    ref.set_threads(1)
    rg = ref.parse_text(raw.decode())
    g = rg.download()
    lab, kmax, rounds = ref.coreness(rg)
    core, _ = ref.get_core(rg, lab, 16)
    ch = core.download()
    out = dict(source="proj/data/ca-hepth.txt", bytes=len(raw),
               sha_text=hashlib.sha256(raw).hexdigest(),
               n=g.n, m=g.m, offs=sha(g.offs), adj=sha(g.adj), orig=sha(g.orig),
               labels=sha(lab), kmax=int(kmax), peel_rounds=int(rounds),
               core16=dict(n=ch.n, arcs=int(ch.offs[-1]), adj=sha(ch.adj), orig=sha(ch.orig)),
               runs={})
    for alg in ("peel", "sort"):
        for pr in ("exact", "none", "approx", "hybrid"):
            r = ref.run(rg, RunConfig(algorithm=alg, pruning=pr, iterations=20))
            out["runs"][f"{alg}/{pr}"] = dict(
                best=list(r.best), witness=sha(r.witness), witness_size=len(r.witness),
                witness_edges=r.witness_edges, max_width=r.max_width,
                slack_violations=r.slack_violations, final_vertices=sha(r.final_vertices),
                trace=[list(t) for t in r.trace])
    with open(os.path.join(HERE, "hepth.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("kmax", kmax, "rounds", rounds, "core16", ch.n, int(ch.offs[-1]),
          "best", out["runs"]["peel/exact"]["best"])


if __name__ == "__main__":
    main()
