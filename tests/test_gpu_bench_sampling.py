"""GPU: `hitgnn bench-sampling`'s CSV (cli.cpp:370-437) through the C++
drop-in (scripts/bench_sampling.py): the reference's columns and formats, and
the bulk and sequential legs return the same batches."""
import csv
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_sampling_csv(tmp_path):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "bench_sampling.py"), "--event", "C1",
                        "--k", "1", "3", "--repeats", "2", "--batch-size", "64", "--out", str(tmp_path)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(open(tmp_path / "bench_sampling.csv")))
    assert rows[0] == ["k", "roots_per_batch", "depth", "fanout", "event_vertices", "event_edges", "repeats",
                       "t_bulk_median_s", "t_sequential_median_s", "speedup"]
    assert [int(x[0]) for x in rows[1:]] == [1, 3]
    for x in rows[1:]:
        assert x[1] == "64" and x[6] == "2"
        assert float(x[7]) > 0 and float(x[8]) > 0
        assert len(x[7].split(".")[1]) == 6 and len(x[9].split(".")[1]) == 4


def test_bulk_and_sequential_legs_agree():
    from paper_2504_04670_b200 import workload as W
    ev = W.preset_event("C1")
    roots, boff, seeds = W.bench_roots(ev.n, 64, 3, 1, 0)
    kw = dict(depth=3, fanout=6, warmup=0, reps=1)
    _, v2, e2 = W.dropin_time(ev, roots, boff, seeds, mode=2, **kw)
    _, v3, e3 = W.dropin_time(ev, roots, boff, seeds, mode=3, **kw)
    assert (v2, e2) == (v3, e3) and v2 > 0 and e2 > 0
    assert np.all(np.diff(boff) == 64)
