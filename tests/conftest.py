import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _ensure_oracle():
    for name in ("liboracle.so", "liboracle_par.so"):
        so = os.path.join(ROOT, "oracle", name)
        if not os.path.exists(so):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), so], check=True,
                           stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def orc():
    _ensure_oracle()
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libdgref.so not built (needs /root/reference at build time)")
    r = Reference()
    r.set_threads(1)
    return r


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def dg():
    """The product: CUDA path through the C ABI (fails loudly without it)."""
    import paper_2311_04333_b200 as dg
    return dg
