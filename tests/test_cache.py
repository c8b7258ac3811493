"""DGRC0001 binary cache (reference io.cpp:108-209):
include/densegraph/io.hpp must read the reference's cache files and write
byte-identical ones.  Golden files: tests/golden/make_cache_golden.py (the
reference's own write_cache / hash_file on two edge-list texts)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
LIBDIR = os.path.join(ROOT, "paper_2311_04333_b200")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cache") / "cache_check")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "cache_check.cpp"), "-o", out, "-L", LIBDIR,
           "-ldg_b200", f"-Wl,-rpath,{LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return out


def _cases():
    with open(os.path.join(GOLD, "cache.json")) as f:
        return json.load(f)


def _run(exe, *args):
    return subprocess.run([exe, *args], capture_output=True, text=True)


@pytest.mark.parametrize("name", ["small", "lcg"])
def test_cache_roundtrip_is_byte_identical(exe, tmp_path, name):
    c = _cases()[name]
    gold = os.path.join(GOLD, c["cache"])
    out = str(tmp_path / "out.dgrc")
    r = _run(exe, "roundtrip", gold, out)
    assert r.returncode == 0, r.stdout + r.stderr
    assert list(map(int, r.stdout.split())) == [c["n"], c["m"], c["source_hash"]]
    assert open(out, "rb").read() == open(gold, "rb").read()
    r = _run(exe, "hash", os.path.join(GOLD, c["text"]))
    assert int(r.stdout) == c["source_hash"]
    assert _run(exe, "is", gold).stdout.strip() == "1"
    assert _run(exe, "is", os.path.join(GOLD, c["text"])).stdout.strip() == "0"


def test_fnv1a64_vectors(exe):
    """The published FNV-1a 64-bit test vectors (offset basis 0xcbf29ce484222325,
    prime 0x100000001b3), the hash behind hash_file and the cache payload check."""
    for text, want in (("a", 0xaf63dc4c8601ec8c), ("foobar", 0x85944171f73967e8)):
        assert int(_run(exe, "fnv", text).stdout) == want, text


def test_cache_errors(exe, tmp_path):
    gold = open(os.path.join(GOLD, "cache_lcg.dgrc"), "rb").read()
    bad = tmp_path / "bad.dgrc"
    corrupt = bytearray(gold)
    corrupt[-3] ^= 0x40  # payload byte
    bad.write_bytes(bytes(corrupt))
    r = _run(exe, "roundtrip", str(bad), str(tmp_path / "o.dgrc"))
    assert r.returncode == 6 and r.stdout.startswith("CacheHashError"), r.stdout
    bad.write_bytes(gold[: len(gold) - 5])  # truncated
    r = _run(exe, "roundtrip", str(bad), str(tmp_path / "o.dgrc"))
    assert r.returncode == 3 and "truncated" in r.stdout, r.stdout
    bad.write_bytes(b"DGRC0002" + gold[8:])  # wrong magic
    r = _run(exe, "roundtrip", str(bad), str(tmp_path / "o.dgrc"))
    assert r.returncode == 3 and "not a graph cache" in r.stdout, r.stdout
    r = _run(exe, "roundtrip", str(tmp_path / "missing.dgrc"), str(tmp_path / "o.dgrc"))
    assert r.returncode == 3


def _decode(path):
    b = open(path, "rb").read()
    assert b[:8] == b"DGRC0001"
    n, m, _, _ = np.frombuffer(b, np.uint64, 4, 8)
    n, m = int(n), int(m)
    o = 40
    orig = np.frombuffer(b, np.uint64, n, o)
    offs = np.frombuffer(b, np.uint64, n + 1, o + 8 * n)
    adj = np.frombuffer(b, np.uint32, 2 * m, o + 16 * n + 8)
    return offs, adj, orig


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["small", "lcg"])
def test_device_parse_matches_reference_cache(dg, name):
    """The device tokeniser + CSR build of the text = the CSR the reference
    cached from the same text."""
    c = _cases()[name]
    g = dg.parse_edge_list_file(os.path.join(GOLD, c["text"]))
    offs, adj, orig = _decode(os.path.join(GOLD, c["cache"]))
    assert (g.n, g.m) == (c["n"], c["m"])
    np.testing.assert_array_equal(g.offs, offs)
    np.testing.assert_array_equal(g.adj, adj)
    np.testing.assert_array_equal(g.orig, orig)
