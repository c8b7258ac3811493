"""CPU-side checks of the drop-in boundary (no GPU calls):
the C-ABI library loads and exports every symbol include/dg_b200.h declares,
the Python mirror's prototype table covers exactly that set, the C++ drop-in
headers compile against it, and the host-side helpers mirror density.hpp."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dg_b200.h")
LIB = os.path.join(ROOT, "paper_2311_04333_b200", "libdg_b200.so")


DIAG_HEADER = os.path.join(ROOT, "include", "dg_b200_diag.h")
DIAG_LIB = os.path.join(ROOT, "paper_2311_04333_b200", "libdg_b200_diag.so")


def declared_symbols(header=HEADER):
    src = open(header).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build first: python -c 'import __graft_entry__ as g; g.build()'"
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_diagnostics_live_in_their_own_library():
    """Latency microbenchmarks and profiling read-outs are not in the product
    library: include/dg_b200_diag.h <-> libdg_b200_diag.so only."""
    from paper_2311_04333_b200 import _abi
    diag = declared_symbols(DIAG_HEADER)
    assert diag and not set(diag) & set(declared_symbols())
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    assert not set(diag) & set(re.findall(r"\b(dg_[a-z0-9_]+)\b", out))
    lib = ctypes.CDLL(DIAG_LIB)
    assert all(hasattr(lib, x) for x in diag)
    assert sorted(_abi.DIAG_PROTOTYPES) == diag


def test_python_prototypes_match_header():
    from paper_2311_04333_b200 import _abi
    assert sorted(_abi.PROTOTYPES) == declared_symbols()


def test_version_and_error_strings_without_gpu():
    from paper_2311_04333_b200._abi import LIB as lib
    assert lib.dg_version().decode().startswith("densegraph-b200")
    assert lib.dg_last_error() is not None


def test_exported_symbols_are_c_linkage():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(dg_[a-z0-9_]+)\b", out))
    assert set(declared_symbols()) <= exported


def test_density_helpers():
    import paper_2311_04333_b200 as dg
    D = dg.Density
    assert D(2, 4) == D(1, 2) and D(3, 2) > D(4, 3) and not (D(1, 1) < D(2, 2))
    assert D(0, 5).reduced() == D(0, 1) and D(6, 4).reduced() == D(3, 2)
    assert dg.ceil_scaled(D(7, 2), 1, 1) == 4 and dg.ceil_scaled(D(31, 2), 2, 3) == 11
    assert dg.format_fixed6(D(1543, 88)) == "17.534091"
    assert dg.format_fixed6(D(1, 8)) == "0.125000"
    assert dg.format_fixed6(D(1, 2000000)) == "0.000000"  # half to even
    assert dg.format_fixed6(D(3, 2000000)) == "0.000002"
    with pytest.raises(dg.ParamError):
        dg.ceil_div(1, 0)


def test_parse_edge_list_fails_loudly_without_gpu():
    """Tokenising runs on the device (csrc/parse.cu): with no GPU the call
    raises instead of falling back to a host parser."""
    import torch
    import paper_2311_04333_b200 as dg
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(dg.CudaError):
        dg.parse_edge_list("0 1\n1 2\n")


def test_cpp_dropin_headers_compile():
    """include/densegraph/*.hpp (the reference's C++ API, re-created over the C ABI)
    compiles and links against libdg_b200.so."""
    src = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
    out = os.path.join(ROOT, "tests", "cpp", "test_api.bin")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", out,
           "-L", os.path.dirname(LIB), "-ldg_b200", f"-Wl,-rpath,{os.path.dirname(LIB)}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
