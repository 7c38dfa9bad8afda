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
