"""Generate tests/golden/parse.json from the REAL reference parser
(io.cpp:25-94 parse_edge_list, through oracle/_ref/libdgref.so).

Run here (needs /root/reference at build time of oracle/_ref):
    python tests/golden/make_parse_golden.py

Each case records the text (latin-1 code points, so arbitrary bytes
round-trip) and either the CSR the reference builds (n, m, sha256 prefixes of offs /
adj / orig) or its error status and exact message.
"""
import ctypes as C
import hashlib
import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import OracleError, RefGraph, Reference  # noqa: E402


def sha(a):  # as tests/test_gpu_parity.py
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def cases():
    c = {
        "triangle": "0 1\n1 2\n2 0\n",
        "comments": "# header\n0 1\n  # indented comment\n\t#tab comment\n1 2\n",
        "crlf": "0 1\r\n1 2\r\n2 3\r\n",
        "double_cr": "0 1\r\r\n1 2\n",
        "tabs": "0\t1\n1 \t 2\n\t2\t\t3\t\n",
        "trailing_spaces": "0 1   \n1 2\t\n",
        "leading_zeros": "007 0010\n0 7\n",
        "no_final_newline": "0 1\n1 2",
        "self_loops_only": "3 3\n4 4\n",
        "duplicates": "0 1\n1 0\n0 1\n5 6\n",
        "empty": "",
        "blank_lines": "\n\n0 1\n\n\n1 2\n\n",
        "whitespace_lines": " \t \n0 1\n   \n",
        "cr_only_lines": "\r\n0 1\n\r\n",
        "three_tokens": "0 1\n0 1 2\n",
        "one_token": "0 1\n1 2\n5\n",
        "letters": "0 x\n",
        "negative": "-1 2\n",
        "plus_sign": "+1 2\n",
        "overflow": "18446744073709551616 1\n",
        "u64_max": "18446744073709551615 0\n0 1\n",
        "hex": "0x10 1\n",
        "inline_comment": "0 1 # trailing comment\n",
        "comment_in_token": "0 #1\n",
        "cr_in_middle": "0\r1\n",
        "vertical_tab": "0\x0b1 2\n",
        "null_byte": "0\x001 2\n",
        "non_ascii_digit": "0 \xb2\n",
        "comma": "0,1\n",
        "first_error_wins": "0 1\nbad\n1 2 3\n",
        "large_sparse_ids": "1000000000000 5\n5 99999999999999\n1000000000000 99999999999999\n",
        "only_comments": "# a\n# b\n",
    }
    rng = random.Random(2311)
    # an error deep in a long file (line numbering across many windows)
    lines = [f"{rng.randrange(5000)} {rng.randrange(5000)}" for _ in range(20000)]
    lines[17321] = "17 18 19"
    c["deep_error"] = "\n".join(lines) + "\n"
    # long valid files with mixed formatting
    for k in range(4):
        out = []
        for _ in range(6000):
            r = rng.random()
            a, b = rng.randrange(1 << (8 + 6 * k)), rng.randrange(1 << (8 + 6 * k))
            sp = rng.choice([" ", "\t", "  ", " \t"])
            lead = rng.choice(["", "", " ", "\t"])
            tail = rng.choice(["", "", " ", "\t "])
            eol = rng.choice(["\n", "\n", "\r\n"])
            if r < 0.03:
                out.append(lead + "# comment " + str(a) + eol)
            elif r < 0.05:
                out.append(rng.choice(["", " ", "\t"]) + eol)
            else:
                out.append(f"{lead}{a}{sp}{b}{tail}{eol}")
        c[f"random_{k}"] = "".join(out)
    # a long line (spans many 256-byte windows)
    c["long_line"] = "0" * 5000 + "1 " + "0" * 3000 + "2\n3 4\n"
    return c


def main():
    ref = Reference()
    ref.set_threads(1)
    out = []
    for name, text in cases().items():
        rec = {"name": name, "text": text}
        try:
            b = text.encode("latin-1")
            h = C.c_void_p()
            st = ref.lib.ref_graph_parse_text(b, len(b), C.byref(h))
            if st:
                rec["status"] = st
                rec["message"] = ref.lib.ref_last_error().decode("latin-1")
            else:
                g = RefGraph(ref, h).download()
                rec.update(status=0, n=int(g.n), m=int(g.m), offs=sha(g.offs), adj=sha(g.adj),
                           orig=sha(g.orig))
        except OracleError as e:  # pragma: no cover
            rec["status"], rec["message"] = e.code, str(e)
        out.append(rec)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "parse.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(f"wrote {len(out)} cases to {path}")
    for r in out:
        print(f"  {r['name']:20s} status={r['status']} {r.get('message', '')[:70]!r}")


if __name__ == "__main__":
    main()
