"""Build a tuning variant of the library from the working tree with some
files taken from a git revision: python tools/build_variant.py TAG REV file... [-- -DFLAG ...]
(-> paper_2311_04333_b200/libdg_b200_TAG.so, load with DG_B200_LIB)."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2311_04333_b200"))
import build  # noqa: E402

args = sys.argv[1:]
flags = args[args.index("--") + 1:] if "--" in args else []
args = args[:args.index("--")] if "--" in args else args
tag, rev, files = args[0], args[1], args[2:]
tmp = f"/tmp/dg_variant_{tag}"
shutil.rmtree(tmp, ignore_errors=True)
shutil.copytree(build.CSRC, tmp)
for f in files:
    src = subprocess.run(["git", "-C", ROOT, "show", f"{rev}:paper_2311_04333_b200/csrc/{f}"],
                         check=True, capture_output=True, text=True).stdout
    open(os.path.join(tmp, f), "w").write(src)
build.FLAGS = [tmp if x == build.CSRC else x for x in build.FLAGS]
build.CSRC = tmp
build.DIAG_SRC = os.path.join(tmp, "microbench.cu")
print(build.build(verbose=False, extra=flags, tag=tag))
