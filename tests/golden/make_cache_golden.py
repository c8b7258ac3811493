"""Golden DGRC0001 cache files written by the REFERENCE's own io.cpp
(write_cache / hash_file / parse_edge_list_file), for the byte-compatibility
test of include/densegraph/io.hpp (tests/test_cache.py).

Run here (needs /root/reference; the outputs are committed):
    python tests/golden/make_cache_golden.py
Compiles a small driver (written for this repo) against the reference's
io.cpp where it lies, parses two edge-list texts, writes their caches
(cache_<name>.dgrc) and records n, m and the source hashes (cache.json).
"""
import json
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("REF", "/root/reference/proj")
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"

DRIVER = r'''
#include <cstdio>
#include "densegraph/io.hpp"
int main(int argc, char** argv) {
  using namespace densegraph;
  Graph g = parse_edge_list_file(argv[1]);
  const u64 h = hash_file(argv[1]);
  write_cache(g, argv[2], h);
  std::printf("%llu %llu %llu\n", (unsigned long long)g.n, (unsigned long long)g.m,
              (unsigned long long)h);
  return 0;
}
'''

TEXTS = {
    # K4 on sparse ids plus a pendant path, a duplicate, a loop, a comment, CRLF
    "small": "# small\n10 20\r\n20 30\n30 10\n10 40\n20 40\n30 40\n40 9000000000\n"
             "9000000000 5\n20 10\n7 7\n",
    # a few hundred seeded edges (mix64-style LCG, not a dataset)
    "lcg": "".join(f"{(i * 2654435761) % 977} {(i * 40503 + 7) % 983}\n" for i in range(1, 600)),
}


def main():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "drv.cpp")
        exe = os.path.join(d, "drv")
        with open(src, "w") as f:
            f.write(DRIVER)
        subprocess.run([CXX, "-std=c++20", "-O1", "-fopenmp", "-I", os.path.join(REF, "include"),
                        src, os.path.join(REF, "src", "io.cpp"), "-o", exe], check=True)
        out = {}
        for name, text in TEXTS.items():
            txt = os.path.join(HERE, f"cache_{name}.txt")
            with open(txt, "w", newline="") as f:
                f.write(text)
            dgrc = os.path.join(HERE, f"cache_{name}.dgrc")
            r = subprocess.run([exe, txt, dgrc], check=True, capture_output=True, text=True)
            n, m, h = map(int, r.stdout.split())
            out[name] = {"text": f"cache_{name}.txt", "cache": f"cache_{name}.dgrc", "n": n,
                         "m": m, "source_hash": h}
    with open(os.path.join(HERE, "cache.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
