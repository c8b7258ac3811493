"""Build the CUDA library in-tree: paper_2311_04333_b200/libdg_b200.so (sm_100a).

Plain nvcc, one shared object: kernels + the C ABI of include/dg_b200.h.
Objects are compiled in parallel and re-used when their sources are older.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libdg_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


DIAG_SRC = os.path.join(CSRC, "microbench.cu")
DIAG_LIB = os.path.join(PKG, "libdg_b200_diag.so")


def _sources():
    """The product library's sources (diagnostics build separately)."""
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith(".cu") and os.path.join(CSRC, f) != DIAG_SRC)


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "dg_b200.h"),
                 os.path.join(ROOT, "include", "dg_b200_diag.h")]


def _compile(src: str, verbose: bool, extra=(), obj_dir: str = OBJ) -> str:
    obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
    newest = max(os.path.getmtime(p) for p in [src] + _headers())
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(obj_dir, os.path.basename(src) + ".ptxas.log")
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr[-6000:]}")
    if verbose:
        print(f"[build] {os.path.basename(src)}", flush=True)
    return obj


def build(verbose: bool = True, extra=(), tag: str = "") -> str:
    """Build libdg_b200.so; `extra` nvcc flags + `tag` build a tuning variant
    libdg_b200_<tag>.so (load it with DG_B200_LIB=<path>)."""
    obj_dir = OBJ + (f"_{tag}" if tag else "")
    lib = LIB if not tag else os.path.join(PKG, f"libdg_b200_{tag}.so")
    os.makedirs(obj_dir, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, extra, obj_dir), srcs))
    if not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-lrt", "-ldl",
               "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
        if verbose:
            print(f"[build] linked {lib}", flush=True)
    if not tag:
        build_cli(lib, verbose)
    build_diag(lib, obj_dir, verbose)
    return lib


def build_diag(lib: str, obj_dir: str = OBJ, verbose: bool = True) -> str:
    """<lib>_diag.so: latency microbenchmarks and profiling read-outs
    (include/dg_b200_diag.h), linked against the library `lib` (the product
    library, or a tuning build of it)."""
    obj = _compile(DIAG_SRC, verbose, (), obj_dir)
    diag = lib[:-3] + "_diag.so"
    if not os.path.exists(diag) or os.path.getmtime(diag) < max(os.path.getmtime(obj),
                                                               os.path.getmtime(lib)):
        cmd = [NVCC, *ARCH, "-shared", "-o", diag, obj, lib,
               "-Xlinker", "-rpath,$ORIGIN", "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"diag link failed:\n{r.stderr[-4000:]}")
        if verbose:
            print(f"[build] linked {diag}", flush=True)
    return diag


CLI_SRC = os.path.join(PKG, "cli", "densest.cpp")
CLI_BIN = os.path.join(PKG, "densest")


def _json_include():
    """nlohmann/json.hpp (the JSON library the reference CLI uses) as vendored
    in the image's cudnn_frontend package."""
    import glob
    import site
    roots = site.getsitepackages() + [os.path.join(sys.prefix, "lib")]
    for r in roots:
        for h in glob.glob(os.path.join(r, "**", "nlohmann", "json.hpp"), recursive=True):
            return os.path.dirname(os.path.dirname(h))
    return None


def build_cli(lib: str, verbose: bool = True) -> str:
    """The `densest` CLI (cli/densest.cpp, the reference's tools/densest.cpp
    front end) against include/ and libdg_b200.so."""
    deps = [CLI_SRC, lib] + [os.path.join(ROOT, "include", "densegraph", f)
                             for f in os.listdir(os.path.join(ROOT, "include", "densegraph"))]
    if os.path.exists(CLI_BIN) and os.path.getmtime(CLI_BIN) >= max(map(os.path.getmtime, deps)):
        return CLI_BIN
    inc = _json_include()
    if inc is None:
        raise RuntimeError("nlohmann/json.hpp not found: cannot build the densest CLI")
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", inc, CLI_SRC,
           "-o", CLI_BIN, "-L", PKG, "-ldg_b200", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stderr[-4000:]}")
    if verbose:
        print(f"[build] {CLI_BIN}", flush=True)
    return CLI_BIN


if __name__ == "__main__":
    # python build.py [tag -DFLAG ...]
    if len(sys.argv) > 1:
        build(verbose=True, extra=sys.argv[2:], tag=sys.argv[1])
    else:
        build(verbose=True)
    sys.exit(0)
