"""The `densest` CLI (paper_2311_04333_b200/cli/densest.cpp) -- the reference's
front end (proj/tools/densest.cpp) on the device path: the behaviour its own
CLI tests pin (proj/tests/test_cli.cpp, restated here), and on the shipped
ca-HepTh dataset the run JSON and trace CSV against what the reference
library computes (tests/golden/hepth.json)."""
import gzip
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2311_04333_b200", "densest")
GOLD = os.path.join(ROOT, "tests", "golden")
pytestmark = pytest.mark.gpu


def cli(*args, env=None):
    if not os.path.exists(BIN):
        pytest.fail("densest CLI not built (paper_2311_04333_b200/build.py)")
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600, env=e)


@pytest.fixture(scope="module")
def files(tmp_path_factory):
    d = tmp_path_factory.mktemp("cli")
    def w(name, text):
        p = d / name
        p.write_text(text)
        return str(p)
    f = {"dir": d,
         "k4": w("k4.txt", "0 1\n0 2\n0 3\n1 2\n1 3\n2 3\n"),
         "tp": w("tri_pendant.txt", "0 1\n1 2\n2 0\n2 3\n"),
         "odd": w("odd_ids.txt", "7 900\n7 10\n900 10\n"),
         "messy": w("messy.txt", "# comment\n2 0\n0 1\n1 2\n2 0\n\n2 3\n"),
         "bad": w("bad.txt", "0 1\nx y\n"),
         "empty": w("empty.txt", "# nothing\n"),
         "star30": w("star30.txt", "".join(f"0 {i}\n" for i in range(1, 30)))}
    with gzip.open(os.path.join(GOLD, "ca-hepth.txt.gz"), "rb") as src:
        p = d / "ca-hepth.txt"
        p.write_bytes(src.read())
    f["hepth"] = str(p)
    return f


def fixed6(a, b):
    """format_fixed6 (density.hpp:55-67): a/b to six decimals, half to even."""
    q, r = divmod(a * 10**6, b)
    if 2 * r > b or (2 * r == b and q % 2):
        q += 1
    return f"{q // 10**6}.{q % 10**6:06d}"


def strip(j):
    j = dict(j)
    j.pop("init_ms")
    j.pop("total_ms")
    j["config"] = {k: v for k, v in j["config"].items() if k != "threads"}
    return j


def test_run_summary_json(files):
    r = cli("run", "--input", files["k4"], "--iterations", "1")
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    assert list(j) == ["input", "config", "kmax", "L0", "best_density", "witness_size",
                       "witness_edges", "iterations", "init_ms", "total_ms", "max_width"]
    assert j["input"] == files["k4"]
    assert j["config"] == {"algorithm": "greedy", "pruning": "exact", "iterations": 1,
                           "epsilon": None, "approx_factor": "1.5", "threads": 0, "repeats": 1,
                           "reset_loads": False, "seed": None}
    assert (j["kmax"], j["L0"]) == (3, 2)
    assert j["best_density"] == {"num": 3, "den": 2, "float": 1.5}
    assert (j["witness_size"], j["witness_edges"], j["iterations"], j["max_width"]) == (4, 6, 1, 3)
    j2 = json.loads(cli("run", "--input", files["k4"], "--iterations", "1", "--pruning", "none").stdout)
    assert j2["kmax"] is None and j2["L0"] is None
    j3 = json.loads(cli("run", "--input", files["k4"], "--iterations=1", "--seed", "7").stdout)
    assert j3["config"]["seed"] == 7


def test_trace_csv(files):
    r = cli("trace", "--input", files["k4"], "--iterations", "2")
    assert r.returncode == 0
    lines = r.stdout.splitlines()
    assert lines[0] == "iter,density_num,density_den,density_float,n,m,width,ms"
    assert lines[1].startswith("1,3,2,1.500000,4,6,3,") and lines[2].startswith("2,3,2,1.500000,4,6,3,")
    out = str(files["dir"] / "trace.csv")
    r2 = cli("trace", "--input", files["k4"], "--iterations", "2", "--trace-csv", out)
    assert open(out).read() == r2.stdout


def test_stats_block(files):
    r = cli("stats", "--input", files["k4"])
    assert r.returncode == 0
    assert r.stdout == ("n              4\nm              6\nmax_degree     3\nkmax           3\n"
                        "core_threshold 2\ncore_vertices  4\ncore_edges     12\n"
                        "vertex_ratio   1.000\nedge_ratio     2.000\n")
    out = str(files["dir"] / "coreness.csv")
    assert cli("stats", "--input", files["tp"], "--coreness-csv", out).returncode == 0
    assert open(out).read() == "orig_id,coreness\n0,2\n1,2\n2,2\n3,1\n"


def test_oracle_line(files):
    assert cli("oracle", "--input", files["tp"]).stdout == "1/1 = 1.000000, witness [0,1,2]\n"
    assert cli("oracle", "--input", files["odd"]).stdout == "1/1 = 1.000000, witness [7,10,900]\n"


def test_convert_round_trip_and_cache(files):
    d = files["dir"]
    canonical = "0 1\n0 2\n1 2\n2 3\n"
    b, back = str(d / "messy.bin"), str(d / "back.txt")
    assert cli("convert", "--input", files["messy"], "--output", b).returncode == 0
    assert cli("convert", "--input", b, "--output", back).returncode == 0
    assert open(back).read() == canonical
    b2, back2 = str(d / "back.bin"), str(d / "back2.txt")
    assert cli("convert", "--input", back, "--output", b2).returncode == 0
    assert cli("convert", "--input", b2, "--output", back2).returncode == 0
    assert open(back2).read() == canonical
    j = json.loads(cli("run", "--input", b, "--iterations", "2").stdout)
    assert (j["best_density"]["num"], j["best_density"]["den"], j["witness_size"]) == (1, 1, 4)
    cache = str(d / "k4.cache")
    first = cli("run", "--input", files["k4"], "--cache", cache, "--iterations", "1")
    second = cli("run", "--input", files["k4"], "--cache", cache, "--iterations", "1")
    assert first.returncode == 0 and second.returncode == 0
    assert strip(json.loads(first.stdout)) == strip(json.loads(second.stdout))
    assert cli("run", "--input", files["tp"], "--cache", cache, "--iterations", "1").returncode == 6


def test_exit_codes(files):
    k4 = files["k4"]
    assert cli("run", "--input", "/nonexistent/g.txt").returncode == 3
    assert cli("run", "--input", files["bad"]).returncode == 3
    assert cli("run", "--input", files["empty"]).returncode == 3
    for extra in (["--bogus"], ["--algorithm", "nope"], ["--iterations", "0"], ["--epsilon", "2.0"],
                  ["--approx-factor", "1.0"], ["--approx-factor", "abc"], ["--repeats", "0"]):
        assert cli("run", "--input", k4, *extra).returncode == 2, extra
    assert cli("run").returncode == 2
    assert cli().returncode == 2
    assert cli("oracle", "--input", files["star30"]).returncode == 5
    assert cli("oracle", "--input", k4, "--limit", "3").returncode == 5
    r = cli("trace", "--input", k4, "--iterations", "2", "--epsilon", "0.5")
    assert r.returncode == 0 and "--iterations wins" in r.stderr and "iter,density_num" in r.stdout
    a = strip(json.loads(cli("run", "--input", k4, "--iterations", "2", "--threads", "1").stdout))
    b = strip(json.loads(cli("run", "--input", k4, "--iterations", "2",
                             env={"DENSEST_THREADS": "4"}).stdout))
    assert a == b
    assert cli("run", "--input", k4, "--iterations", "1", env={"DENSEST_THREADS": "abc"}).returncode == 0
    assert cli("--help").returncode == 0 and cli("run", "--help").returncode == 0


def test_hepth_run_json_and_trace_vs_reference(files):
    """acceptance.cpp's CLI criterion on the shipped dataset: every
    non-timing field of the JSON summary and the trace CSV rows (but ms) equal
    what the reference library computes on the same file."""
    with open(os.path.join(GOLD, "hepth.json")) as f:
        fx = json.load(f)
    for alg, key in (("greedy", "peel"), ("sorting", "sort")):
        for pr in ("exact", "none", "approx", "hybrid"):
            e = fx["runs"][f"{key}/{pr}"]
            r = cli("run", "--input", files["hepth"], "--algorithm", alg, "--pruning", pr)
            assert r.returncode == 0, r.stderr
            j = json.loads(r.stdout)
            from fractions import Fraction
            assert [j["best_density"]["num"], j["best_density"]["den"]] == e["best"]
            assert j["best_density"]["float"] == float(Fraction(*e["best"]))
            assert (j["witness_size"], j["witness_edges"], j["iterations"], j["max_width"]) == (
                e["witness_size"], e["witness_edges"], 20, e["max_width"])
            if pr in ("exact", "hybrid"):
                assert (j["kmax"], j["L0"]) == (fx["kmax"], (fx["kmax"] + 1) // 2)
            t = cli("trace", "--input", files["hepth"], "--algorithm", alg, "--pruning", pr)
            rows = [ln.split(",") for ln in t.stdout.splitlines()[1:]]
            want = [[str(it), str(a), str(b), fixed6(a, b), str(n), str(m), str(w)]
                    for it, a, b, n, m, w in e["trace"]]
            assert [r_[:7] for r_ in rows] == want
    s = cli("stats", "--input", files["hepth"]).stdout.splitlines()
    assert s[3] == f"kmax           {fx['kmax']}" and s[5] == "core_vertices  96"
    assert s[6] == "core_edges     2306"
