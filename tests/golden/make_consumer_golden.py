"""Golden fixtures for the consumer row, generated from the
REFERENCE: slice_components (trainer.cpp:221-269), Tape::gather_rows /
scatter_add forward and backward (autodiff.cpp:121-157, 260-281) and
allreduce_coalesced over InMemoryComm (trainer.cpp:84-157), all from the
unmodified sources built by oracle/Makefile into
oracle/_ref/libhitgnn_ref_consumer.so (ref_consumer_shim.cpp).

    python tests/golden/make_consumer_golden.py   -> tests/golden/consumer.npz

Inputs are regenerated deterministically from the seeds stored in the file;
the sampled batches come from the reference sampler (oracle impl="ref") on a
small random graph, so the fixtures also hold the inputs the checks need.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import consumer as CO  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.helpers import random_graph  # noqa: E402

OUT = os.path.join(HERE, "consumer.npz")


def sampled_case():
    """A reference bulk_shadow + gather_features result: 3 batches of 40 roots."""
    g = random_graph(900, 7000, 41)
    rs = np.random.default_rng(42)
    roots = np.concatenate([rs.permutation(g.n)[:40] for _ in range(3)]).astype(np.int64)
    boff = np.array([0, 40, 80, 120], np.int64)
    seeds = rs.integers(0, 2**63, 120, dtype=np.uint64)
    s = O.bulk_shadow(g, roots, boff, seeds, depth=2, fanout=4, gather=True, impl="ref")
    return g, boff, s


def main() -> None:
    if not CO.ref_available():
        raise SystemExit("oracle/_ref/libhitgnn_ref_consumer.so missing: run `make -f oracle/Makefile ref`")
    d = {}
    # ---- slice_components: several ranges of each batch, incl. empty / full / DDP ranges
    g, boff, s = sampled_case()
    ranges = []
    for b in range(3):
        nb = int(boff[b + 1] - boff[b])
        rr = [(0, nb), (0, 0), (nb, nb), (3, 17), (nb - 1, nb), (5, 6)]
        rr += [(nb * r // 4, nb * (r + 1) // 4) for r in range(4)]  # worker_component_range, world 4
        for (lo, hi) in rr:
            ranges.append((b, lo, hi))
    d["slice_ranges"] = np.array(ranges, np.int64)
    for i, (b, lo, hi) in enumerate(ranges):
        ref = CO.ref_slice_components(CO.batch_of(s, boff, b, 6, 2), lo, hi)
        for k, v in ref.items():
            d[f"slice{i}_{k}"] = v
    # ---- gather_rows / scatter_add, forward; values spanning many magnitudes
    # so that a different summation order would change the bits
    rs = np.random.default_rng(7)
    for case, (n, m, c) in enumerate([(50, 400, 6), (7, 300, 3), (200, 150, 2), (1, 20, 5)]):
        x = rs.standard_normal((n, c)) * np.exp2(rs.integers(-30, 30, (n, c)))
        idx = rs.integers(0, n, m)
        y = rs.standard_normal((m, c)) * np.exp2(rs.integers(-30, 30, (m, c)))
        d[f"gs{case}_x"], d[f"gs{case}_idx"], d[f"gs{case}_y"] = x, idx, y
        d[f"gs{case}_gather"] = CO.ref_gather_rows(x, idx)
        d[f"gs{case}_scatter"] = CO.ref_scatter_add(y, idx, n)
        # backward through linear(w) -> bce(labels)
        w = rs.standard_normal((c, 1)) * 4.0
        lab_g = rs.integers(0, 2, m).astype(np.uint8)
        lab_s = rs.integers(0, 2, n).astype(np.uint8)
        d[f"gs{case}_w"], d[f"gs{case}_labg"], d[f"gs{case}_labs"] = w, lab_g, lab_s
        go, gi = CO.ref_backward(0, x, idx, n, w, lab_g)
        d[f"gs{case}_gather_gout"], d[f"gs{case}_gather_gin"] = go, gi
        go, gi = CO.ref_backward(1, y, idx, n, w, lab_s)
        d[f"gs{case}_scatter_gout"], d[f"gs{case}_scatter_gin"] = go, gi
    # ---- allreduce_coalesced over 1..5 worker threads
    for w in range(1, 6):
        n = 1000 + 7 * w
        parts = rs.standard_normal((w, n)) * np.exp2(rs.integers(-40, 40, (w, n)))
        if w >= 3:  # a cancelling column: (1e16 + 1) - 1e16 != 1e16 + (1 - 1e16) ...
            parts[:, 0] = [(1e16, 1.0, -1e16)[q % 3] for q in range(w)]
        d[f"ar{w}_in"] = parts
        d[f"ar{w}_out"] = CO.ref_allreduce_mean(parts)
    np.savez_compressed(OUT, **d)
    print("wrote", OUT, len(d), "arrays")


if __name__ == "__main__":
    main()
