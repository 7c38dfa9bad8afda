"""GPU: the C++ drop-in (hitgnn:: API in libhitgnn_gpu.so) driven like the
reference's own callers, compiled from tests/cpp/test_dropin.cpp and checked
against the oracle. The CPU half (it compiles and links) runs everywhere."""
import os
import subprocess

import pytest

from tests.helpers import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")
LIB = os.path.join(ROOT, "paper_2504_04670_b200", "lib")
ORACLE = os.path.join(ROOT, "oracle")


def build():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", ORACLE, SRC,
           "-o", BIN, f"-L{LIB}", "-lhitgnn_gpu", "-lhgs", f"-L{ORACLE}", "-loracle",
           f"-Wl,-rpath,{LIB}:{ORACLE}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return BIN


def test_dropin_builds_and_links():
    assert os.access(build(), os.X_OK)


@pytest.mark.gpu
def test_dropin_against_oracle():
    res = subprocess.run([build()], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "ALL OK" in res.stdout


@pytest.mark.gpu
def test_dropin_frontier_observer_matches_reference():
    """hitgnn::bulk_shadow's FrontierObserver on the GPU drop-in (device
    frontiers exported with HGS_FLAG_KEEP_FRONTIERS, Q/F/P materialised on
    the host) reproduces the reference's per-level FrontierSet bit for bit:
    digests of the reference's own Q, F and P (tests/golden/frontiers.json)."""
    import hashlib
    import json

    import numpy as np
    from paper_2504_04670_b200 import workload as W
    d = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(d, "frontiers.json")) as f:
        idx = json.load(f)
    z = np.load(os.path.join(d, "frontiers.npz"))
    dg = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    for c in idx:
        p = c["name"] + "/"
        lv = W.dropin_frontiers(z[p + "rp"], z[p + "ci"], z[p + "values"] if c["values"] else None,
                                z[p + "roots"], z[p + "boff"], z[p + "seeds"], rng=c["rng"], depth=c["depth"],
                                fanout=c["fanout"], symmetrize=c["sym"])
        assert len(lv) == len(c["levels"]) == c["depth"]
        for got, exp in zip(lv, c["levels"]):
            for k in W.FRONTIER_ARRAYS:
                assert dg(got[k]) == exp[k], (c["name"], k)
