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


# ---------------------------------------------------------------------------
# bench-size parity: slices of one device call against chunked oracle calls

def batch_slice(dev: dict, boff, b0: int, b1: int, f_v: int = 0, f_e: int = 0) -> dict:
    """Outputs of batches [b0, b1) of one device call, in the layout of a call
    over just those batches (batch-local ids need no rebasing; only the call
    offsets do). Per-root streams make that call's result identical."""
    boff = np.asarray(boff, np.int64)
    bv = np.asarray(dev["batch_voff"]).astype(np.int64)
    be = np.asarray(dev["batch_eoff"]).astype(np.int64)
    r0, r1 = int(boff[b0]), int(boff[b1])
    v0, v1, e0, e1 = int(bv[b0]), int(bv[b1]), int(be[b0]), int(be[b1])
    out = {"batch_voff": bv[b0:b1 + 1] - v0, "batch_eoff": be[b0:b1 + 1] - e0,
           "comp_off": np.asarray(dev["comp_off"])[r0 + b0:r1 + b1],
           "roots_local": np.asarray(dev["roots_local"])[r0:r1],
           "l2g": np.asarray(dev["l2g"])[v0:v1],
           "draws": np.asarray(dev["draws"])[r0:r1], "decisions": np.asarray(dev["decisions"])[r0:r1]}
    for f in ("e_row", "e_col", "e_gid", "lab"):
        if dev.get(f) is not None:
            out[f] = np.asarray(dev[f])[e0:e1]
    if dev.get("xv") is not None and f_v:
        out["xv"] = np.asarray(dev["xv"])[v0 * f_v:v1 * f_v]
    if dev.get("ye") is not None and f_e:
        out["ye"] = np.asarray(dev["ye"])[e0 * f_e:e1 * f_e]
    return out


def check_against_oracle_chunks(dev: dict, g, roots, boff, seeds, chunks, *, gather, f_v=0, f_e=0,
                                threads=None, **kw) -> list:
    """Run the oracle on each batch range of `chunks` (host threads in
    parallel; the C oracle releases the GIL) and compare the matching slice of
    the device call bit for bit. Returns [(b0, b1, bad_fields)] for mismatches."""
    import concurrent.futures as cf
    roots = np.asarray(roots, np.int64)
    seeds = np.asarray(seeds, np.uint64)
    boff = np.asarray(boff, np.int64)

    def one(ch):
        b0, b1 = ch
        r0, r1 = int(boff[b0]), int(boff[b1])
        ref = O.bulk_shadow(g, roots[r0:r1], boff[b0:b1 + 1] - r0, seeds[r0:r1], gather=gather, **kw)
        return b0, b1, compare(batch_slice(dev, boff, b0, b1, f_v, f_e), ref, gather=gather)

    with cf.ThreadPoolExecutor(threads or min(len(chunks), os.cpu_count() or 4)) as ex:
        res = list(ex.map(one, chunks))
    return [r for r in res if r[2]]


def even_chunks(k: int, parts: int):
    parts = max(1, min(parts, k))
    return [(k * i // parts, k * (i + 1) // parts) for i in range(parts) if k * i // parts < k * (i + 1) // parts]
