"""Randomised device-vs-oracle fuzzing (GPU): random graphs (uniform, banded,
hub-heavy, with zeros / negative-free values), random depth / fanout / RNG /
walk / batch shapes, every output array compared bit for bit.
usage: python scripts/fuzz_gpu.py [seconds] [seed]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.helpers import O, compare  # noqa: E402
from paper_2504_04670_b200 import hgs  # noqa: E402


def make_graph(rs):
    kind = rs.integers(0, 3)
    n = int(rs.integers(2, 6000))
    if kind == 0:  # uniform
        m = int(rs.integers(0, 12 * n))
        u, v = rs.integers(0, n, m), rs.integers(0, n, m)
    elif kind == 1:  # banded (id locality)
        w = int(rs.integers(1, 20))
        u = np.repeat(np.arange(n), w)
        v = u + np.tile(np.arange(1, w + 1), n)
        keep = (v < n) & (rs.random(len(u)) < 0.6)
        u, v = u[keep], v[keep]
    else:  # hubs
        h = rs.choice(n, min(n, 5), replace=False)
        u = np.concatenate([np.repeat(h, min(n, 800)), rs.integers(0, n, 4 * n)])
        v = np.concatenate([rs.integers(0, n, len(h) * min(n, 800)), rs.integers(0, n, 4 * n)])
    if rs.random() < 0.7:
        keep = u != v
        u, v = u[keep], v[keep]
    key = np.unique(u.astype(np.int64) * n + v)
    u, v = key // n, key % n
    rp = np.concatenate([[0], np.cumsum(np.bincount(u, minlength=n))]).astype(np.int64)
    g = O.Graph(n=n, rp=rp, ci=v.astype(np.int64))
    if rs.random() < 0.25:
        g.values = rs.uniform(0.5, 2.0, len(v))
        g.values[rs.random(len(v)) < 0.2] = 0.0
    g.node_feat = rs.standard_normal((n, 6))
    g.edge_feat = rs.standard_normal((len(v), 2))
    g.labels = rs.integers(0, 2, len(v)).astype(np.uint8)
    return g


def run(rs, *, secs=None, max_cases=None, log=print):
    """Fuzz until `secs` elapse or `max_cases` cases ran; returns (cases, mismatches)."""
    t0, cases, bad = time.time(), 0, 0
    while (secs is None or time.time() - t0 < secs) and (max_cases is None or cases < max_cases):
        g = make_graph(rs)
        depth = int(rs.integers(1, 5))
        fanout = int(rs.choice([1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 20, 40, 300]))
        # keep the per-root tree bound sane for deep/wide draws
        while sum(fanout ** l for l in range(depth + 1)) > 80000:
            depth -= 1
        sym = bool(rs.random() < 0.7)
        rng = int(rs.integers(0, 2))
        k = int(rs.integers(1, 6))
        sizes = [int(rs.integers(0, min(g.n, 300) + 1)) for _ in range(k)]
        roots = np.concatenate([rs.choice(g.n, s, replace=False) for s in sizes] + [np.zeros(0, np.int64)])
        roots = roots.astype(np.int64)
        boff = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        seeds = rs.integers(0, 2**63, len(roots), dtype=np.uint64)
        gather = g.values is None
        kw = dict(rng=rng, depth=depth, fanout=fanout, symmetrize=sym)
        try:
            ref = O.bulk_shadow(g, roots, boff, seeds, gather=gather, **kw)
        except O.SamplerError:
            continue  # e.g. negative rows; covered by the unit tests
        G = hgs.Graph(g.rp, g.ci, g.values)
        if gather:
            G.attach_features(g.node_feat, g.edge_feat, g.labels)
        S = hgs.Sampler(G)
        S.bulk_shadow(roots, boff, seeds, gather=gather, **kw)
        diff = compare(S.to_host(), ref, gather=gather)
        cases += 1
        if diff:
            bad += 1
            log(f"MISMATCH n={g.n} m={len(g.ci)} {kw} sizes={sizes} fields={diff}")
        S.close()
        G.close()
    log(f"fuzz: {cases} cases, {bad} mismatches in {time.time() - t0:.0f}s")
    return cases, bad


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 300
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 12345
    print(f"fuzz_gpu: seed {seed}, {secs:.0f}s, K2 = {os.environ.get('HGS_K2', 'hash')}",
          flush=True)
    _, bad = run(np.random.default_rng(seed), secs=secs, log=lambda m: print(m, flush=True))
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
