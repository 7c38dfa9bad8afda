"""Shared helpers for the parity tests: workloads and device-vs-oracle
comparison. Imports oracle/ (allowed: tests are the checker side)."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def random_graph(n, m, seed, *, self_loops=False, values=None):
    """Random directed CSR graph (canonical: rows ascending, cols unique)."""
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    if not self_loops:
        keep = u != v
        u, v = u[keep], v[keep]
    key = np.unique(u.astype(np.int64) * n + v)
    u, v = key // n, key % n
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, u + 1, 1)
    rp = np.cumsum(rp)
    g = O.Graph(n=n, rp=rp, ci=v.astype(np.int64))
    mm = len(v)
    g.node_feat = rng.standard_normal((n, 6))
    g.edge_feat = rng.standard_normal((mm, 2))
    g.labels = rng.integers(0, 2, mm).astype(np.uint8)
    return g


def bench_roots(n, b, k, seed=1, rep=0):
    """Roots + per-root seeds of the reference bench protocol (cli.cpp:381-408)."""
    if k * b > n:
        b = max(1, n // k)
    rs = O.derive(seed, [0x62656E6368, k, rep])
    batches = O.epoch_root_batches(n, b, rs)[:k]
    roots = np.concatenate(batches).astype(np.int64)
    boff = np.zeros(len(batches) + 1, np.int64)
    boff[1:] = np.cumsum([len(x) for x in batches])
    seeds = np.array([O.derive(seed, [0x7374726D, k, rep, bi, pos])
                      for bi in range(len(batches)) for pos in range(len(batches[bi]))],
                     np.uint64)
    return roots, boff, seeds


FIELDS = ["batch_voff", "batch_eoff", "comp_off", "l2g", "roots_local", "e_row", "e_col", "e_gid"]


def compare(dev: dict, ref, *, gather=False, counts=True):
    """Bit-exact comparison of a device result (int32 arrays) and an oracle Sample."""
    bad = []
    for f in FIELDS:
        a = np.asarray(dev[f]).astype(np.int64)
        b = getattr(ref, f).astype(np.int64)
        if a.shape != b.shape or not np.array_equal(a, b):
            bad.append(f)
    if gather:
        for f in ["xv", "ye", "lab"]:
            a, b = np.asarray(dev[f]), getattr(ref, f)
            if a.shape != b.shape or not np.array_equal(a.view(np.uint8), b.view(np.uint8)):
                bad.append(f)
    if counts and ref.draws is not None:
        if not np.array_equal(np.asarray(dev["decisions"]).astype(np.int64), ref.decisions):
            bad.append("decisions")
        if not np.array_equal(np.asarray(dev["draws"]).astype(np.int64), ref.draws):
            bad.append("draws")
    return bad


# ---------------------------------------------------------------------------
# golden fixtures (generated from the reference by tests/golden/make_golden.py)

GOLDEN = os.path.join(ROOT, "tests", "golden")
OUT_FIELDS = ["batch_voff", "batch_eoff", "comp_off", "l2g", "roots_local", "e_row", "e_col",
              "e_gid", "e_val", "xv", "ye", "lab"]


def load_small_cases():
    import json
    with open(os.path.join(GOLDEN, "small_cases.json")) as f:
        index = json.load(f)
    z = np.load(os.path.join(GOLDEN, "small_cases.npz"))
    out = []
    for ent in index:
        gp, pre = ent["graph"], ent["prefix"]
        g = O.Graph(n=ent["n"], rp=z[gp + "rp"], ci=z[gp + "ci"],
                    values=z[gp + "values"] if ent["has_values"] else None,
                    node_feat=z[gp + "nf"], edge_feat=z[gp + "ef"], labels=z[gp + "lab"])
        exp = {f: z[pre + "out_" + f] for f in OUT_FIELDS if pre + "out_" + f in z}
        out.append(dict(ent, g=g, roots=z[pre + "roots"], boff=z[pre + "boff"], seeds=z[pre + "seeds"],
                        expected=exp))
    return out


def load_json(name):
    import json
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
