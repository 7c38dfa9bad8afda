"""GPU parity: the CUDA path through the C ABI (libhgs.so) against the
reference's golden results and the oracle, bit for bit.

Covers K0 (walk build), both RNG modes, symmetrized / directed walks,
depths 1-4, fanouts on both choose paths (k <= 8 registers, k > 8 local),
explicit-zero and negative values, self-loops, isolated roots, empty batches,
zero-root calls, gather on/off, resumed (non-fresh) streams, the
capacity-regrow path, error messages, the device-pointer entry point, the
C1 configuration (digests of the reference's own outputs) and the full C2
workload against the oracle plus size-independent properties.
"""
import os

import numpy as np
import pytest

from tests.helpers import O, OUT_FIELDS, compare, load_json, load_small_cases, random_graph, sha

pytestmark = pytest.mark.gpu

CMP = ["batch_voff", "batch_eoff", "comp_off", "l2g", "roots_local", "e_row", "e_col", "e_gid"]


def hgs():
    from paper_2504_04670_b200 import hgs as H
    return H


def device_run(g, roots, boff, seeds, *, gather=False, state=None, sampler=None, **kw):
    H = hgs()
    if sampler is None:
        G = H.Graph(g.rp, g.ci, g.values, n_cols=g.n_cols)
        if gather:
            G.attach_features(g.node_feat, g.edge_feat, g.labels)
        sampler = H.Sampler(G)
    sampler.bulk_shadow(roots, boff, seeds, gather=gather, state=state, **kw)
    return sampler.to_host(), sampler


def assert_same(dev, ref, gather, counts=True, gid=True):
    for f in CMP:
        if f == "e_gid" and not gid:
            continue
        a = np.asarray(dev[f]).astype(np.int64)
        b = getattr(ref, f).astype(np.int64)
        assert a.shape == b.shape and np.array_equal(a, b), f
    if gather:
        for f in ("xv", "ye", "lab"):
            a, b = np.asarray(dev[f]), getattr(ref, f)
            assert a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8)), f
    if counts and ref.draws is not None:
        assert np.array_equal(dev["draws"].astype(np.int64), ref.draws)
        assert np.array_equal(dev["decisions"].astype(np.int64), ref.decisions)


# --------------------------------------------------------------------- K0 ----

@pytest.mark.parametrize("n,m,seed", [(1, 0, 0), (7, 20, 1), (500, 3000, 2), (20000, 250000, 3)])
def test_walk_build_matches_symmetrize_pattern(n, m, seed):
    g = random_graph(n, m, seed, self_loops=seed % 2 == 1)
    G = hgs().Graph(g.rp, g.ci)
    rp, ci = G.walk(True)
    orp, oci = O.symmetrize(g)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)


def test_walk_build_hub_rows():
    # a hub with 6000 in- and out-neighbours: radix transpose + row merge
    n = 8000
    src = np.concatenate([np.zeros(6000, np.int64), np.arange(1, 6001)])
    dst = np.concatenate([np.arange(1, 6001), np.zeros(6000, np.int64) + 7])
    key = np.unique(src * n + dst)
    u, v = key // n, key % n
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, u + 1, 1)
    g = O.Graph(n=n, rp=np.cumsum(rp), ci=v)
    rp2, ci2 = hgs().Graph(g.rp, g.ci).walk(True)
    orp, oci = O.symmetrize(g)
    assert np.array_equal(rp2, orp) and np.array_equal(ci2, oci)


# ----------------------------------------------------------------- golden ----

@pytest.mark.parametrize("case", load_small_cases(), ids=lambda c: c["name"])
def test_golden_cases(case):
    H = hgs()
    g = case["g"]
    kw = dict(rng=case["rng"], depth=case["depth"], fanout=case["fanout"], symmetrize=case["sym"])
    if case["error"]:
        with pytest.raises(H.SamplerError):
            device_run(g, case["roots"], case["boff"], case["seeds"], gather=case["gather"], **kw)
        return
    dev, _ = device_run(g, case["roots"], case["boff"], case["seeds"], gather=case["gather"], **kw)
    exp = case["expected"]
    for f in CMP:
        if f == "e_gid" and np.all(exp[f] == -1) and exp[f].size:
            continue
        assert np.array_equal(np.asarray(dev[f]).astype(np.int64), exp[f]), f
    if case["gather"]:
        for f in ("xv", "ye", "lab"):
            assert np.array_equal(np.asarray(dev[f]).view(np.uint8), exp[f].view(np.uint8)), f


# ------------------------------------------------------------ random sweep ----

SWEEP = [  # (n, m, depth, fanout, values)
    (30, 80, 1, 1, None), (200, 1200, 2, 3, None), (1000, 8000, 3, 6, None),
    (1000, 8000, 4, 2, "zeros"), (3000, 30000, 3, 8, None), (500, 20000, 2, 9, None),
    (300, 9000, 2, 17, "zeros"), (5000, 60000, 3, 6, "zeros"),
]


@pytest.mark.parametrize("n,m,depth,fanout,values", SWEEP)
@pytest.mark.parametrize("rng", [0, 1])
def test_random_graphs(n, m, depth, fanout, values, rng):
    rs = np.random.default_rng(n + depth * 7 + fanout + rng)
    g = random_graph(n, m, n + fanout, self_loops=(n % 3 == 0))
    if values == "zeros":
        g.values = rs.uniform(0.5, 2.0, g.m)
        g.values[rs.random(g.m) < 0.2] = 0.0
    k = 5
    b = min(n // k, 64)
    sizes = [b, 0, b // 2, b, 1]  # includes an empty batch and a single-root batch
    roots = np.concatenate([rs.permutation(n)[:s] for s in sizes]).astype(np.int64)
    boff = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    seeds = rs.integers(0, 2**63, len(roots), dtype=np.uint64)
    gather = values is None
    for sym in (True, False):
        kw = dict(rng=rng, depth=depth, fanout=fanout, symmetrize=sym)
        dev, _ = device_run(g, roots, boff, seeds, gather=gather, **kw)
        ref = O.bulk_shadow(g, roots, boff, seeds, gather=gather, **kw)
        assert_same(dev, ref, gather)


@pytest.mark.parametrize("combine", ["0", "1"])
@pytest.mark.parametrize("n,m,depth,fanout", [(1000, 8000, 3, 6), (3000, 30000, 3, 8), (2000, 16000, 4, 3),
                                              (500, 20000, 2, 17), (4000, 60000, 6, 4)])
def test_k1_store_paths(monkeypatch, combine, n, m, depth, fanout):
    """K1's touched stores with and without the per-lane write combiner
    (HGS_K1_COMBINE; the default picks by call size) over every K1 body:
    fanout 3/4 (KCAP 4), 6, 8, the local-array path (17) and the uncached
    deep tree (depth 6, rows re-read from the walk)."""
    monkeypatch.setenv("HGS_K1_COMBINE", combine)
    rs = np.random.default_rng(n + depth + fanout)
    g = random_graph(n, m, n + 3 * fanout)
    sizes = [100, 0, 37, 1, 64]
    roots = np.concatenate([rs.permutation(n)[:s] for s in sizes]).astype(np.int64)
    boff = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    seeds = rs.integers(0, 2**63, len(roots), dtype=np.uint64)
    for rng in (0, 1):
        for sym in (True, False):
            kw = dict(rng=rng, depth=depth, fanout=fanout, symmetrize=sym)
            dev, _ = device_run(g, roots, boff, seeds, gather=True, **kw)
            ref = O.bulk_shadow(g, roots, boff, seeds, gather=True, **kw)
            assert_same(dev, ref, True)


def banded_graph(n, w, seed, outliers=0):
    """Vertex ids with locality (u -> u+1..u+w) plus a few long-range edges
    to the top ids: a root's set spans a narrow id range with outliers, which
    stresses the order-preserving bucketing of K2's set sort."""
    rs = np.random.default_rng(seed)
    u = np.repeat(np.arange(n), w)
    v = u + np.tile(np.arange(1, w + 1), n)
    keep = (v < n) & (rs.random(len(u)) < 0.7)
    u, v = u[keep], v[keep]
    if outliers:
        ou = rs.integers(0, n, outliers)
        ov = n - 1 - rs.integers(0, 3, outliers)
        u, v = np.concatenate([u, ou]), np.concatenate([v, ov])
    key = np.unique(u.astype(np.int64) * n + v)
    u, v = key // n, key % n
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, u + 1, 1)
    g = O.Graph(n=n, rp=np.cumsum(rp), ci=v.astype(np.int64))
    g.node_feat = rs.standard_normal((n, 6))
    g.edge_feat = rs.standard_normal((len(v), 2))
    g.labels = rs.integers(0, 2, len(v)).astype(np.uint8)
    return g


@pytest.mark.parametrize("n,w,outliers,depth,fanout", [
    (4000, 8, 0, 3, 6), (4000, 8, 200, 3, 6), (100000, 12, 50, 3, 6), (3000, 30, 0, 2, 17)])
def test_clustered_vertex_ids(n, w, outliers, depth, fanout):
    g = banded_graph(n, w, n + w, outliers)
    rs = np.random.default_rng(w)
    k, b = 3, 100
    roots = np.concatenate([rs.permutation(n)[:b] for _ in range(k)]).astype(np.int64)
    boff = np.arange(k + 1, dtype=np.int64) * b
    seeds = rs.integers(0, 2**63, k * b, dtype=np.uint64)
    for sym in (True, False):
        kw = dict(rng=0, depth=depth, fanout=fanout, symmetrize=sym)
        dev, _ = device_run(g, roots, boff, seeds, gather=True, **kw)
        ref = O.bulk_shadow(g, roots, boff, seeds, gather=True, **kw)
        assert_same(dev, ref, True)


@pytest.mark.parametrize("n,m", [(3_000_000, 24_000_000), (9_000_000, 30_000_000)])
def test_large_graph_subset(n, m):
    """Multi-million-vertex graphs: packed hash entries near the 32-bit limit
    (3M) and the unpacked (vertex, rank) path (9M > 2^23), 64-bit CSR sizes
    on the host side; 512 roots against the oracle."""
    rs = np.random.default_rng(n)
    # rows as random ascending progressions: canonical CSR in O(m), no sort
    deg = rs.poisson(m / n, n).astype(np.int64)
    step = rs.integers(1, 64, n)
    start = rs.integers(0, np.maximum(1, n - deg * step))
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    j = np.arange(rp[-1], dtype=np.int64) - np.repeat(rp[:-1], deg)
    v = np.repeat(start, deg) + j * np.repeat(step, deg)
    g = O.Graph(n=n, rp=rp, ci=v)
    g.node_feat = (np.arange(n * 6, dtype=np.float64) * 0.25).reshape(n, 6)
    g.edge_feat = (np.arange(len(v) * 2, dtype=np.float64) * 0.125).reshape(len(v), 2)
    g.labels = (v % 2).astype(np.uint8)
    roots = np.concatenate([rs.choice(n, 256, replace=False) for _ in range(2)]).astype(np.int64)
    boff = np.array([0, 256, 512], np.int64)
    seeds = rs.integers(0, 2**63, 512, dtype=np.uint64)
    for rng in (0, 1):
        kw = dict(rng=rng, depth=3, fanout=6)
        dev, _ = device_run(g, roots, boff, seeds, gather=True, **kw)
        ref = O.bulk_shadow(g, roots, boff, seeds, gather=True, **kw)
        assert_same(dev, ref, True)


@pytest.mark.parametrize("depth,fanout", [(2, 6), (3, 4), (2, 40), (2, 600)])
def test_hub_rows_many_windows(depth, fanout):
    """Hubs with out-degree in the thousands: a root's scanned entries span
    many K2 window passes (more than one pass of win_cap windows), and wide
    fanouts take the local-memory choose path (s=40) or, beyond 256 choices,
    the global-scratch one (s=600)."""
    rs = np.random.default_rng(depth * 100 + fanout)
    n = 3000
    edges = set()
    hubs = rs.choice(n, 12, replace=False)
    for h in hubs:
        for v in rs.choice(n, 2500, replace=False):
            if v != h:
                edges.add((int(h), int(v)))
    for _ in range(20000):
        u, v = rs.integers(0, n, 2)
        if u != v:
            edges.add((int(u), int(v)))
    e = np.array(sorted(edges), np.int64)
    rp = np.concatenate([[0], np.cumsum(np.bincount(e[:, 0], minlength=n))]).astype(np.int64)
    g = O.Graph(n=n, rp=rp, ci=e[:, 1].copy())
    g.node_feat = rs.standard_normal((n, 6))
    g.edge_feat = rs.standard_normal((len(e), 2))
    g.labels = rs.integers(0, 2, len(e)).astype(np.uint8)
    roots = np.concatenate([hubs[:6], rs.choice(n, 90, replace=False)]).astype(np.int64)
    roots = np.unique(roots)
    boff = np.array([0, len(roots) // 2, len(roots)], np.int64)
    seeds = rs.integers(0, 2**63, len(roots), dtype=np.uint64)
    for rng in (0, 1):
        kw = dict(rng=rng, depth=depth, fanout=fanout)
        dev, _ = device_run(g, roots, boff, seeds, gather=True, **kw)
        ref = O.bulk_shadow(g, roots, boff, seeds, gather=True, **kw)
        assert_same(dev, ref, True)


@pytest.mark.parametrize("n,m,depth,fanout", [(4000, 120000, 3, 20), (20000, 300000, 4, 8), (3000, 60000, 5, 5)])
def test_big_trees(n, m, depth, fanout):
    """Tree bounds of 8k-20k vertices per root: K2 runs with 2 or 1 warps per
    CTA, or is sized after K1 from the largest touched list it produced."""
    g = random_graph(n, m, n + depth)
    rs = np.random.default_rng(depth * fanout)
    roots = rs.choice(n, 96, replace=False).astype(np.int64)
    boff = np.array([0, 40, 96], np.int64)
    seeds = rs.integers(0, 2**63, 96, dtype=np.uint64)
    for rng in (0, 1):
        kw = dict(rng=rng, depth=depth, fanout=fanout)
        dev, _ = device_run(g, roots, boff, seeds, gather=True, **kw)
        ref = O.bulk_shadow(g, roots, boff, seeds, gather=True, **kw)
        assert_same(dev, ref, True)


def test_oversize_sets_global_scratch():
    """Touched sets beyond one warp's shared memory (~9k vertices): K2 runs
    with its working sets in global scratch; same results as the oracle."""
    g = random_graph(30000, 1500000, 3)
    roots = np.arange(8, dtype=np.int64)
    boff = np.array([0, 3, 8], np.int64)
    seeds = np.arange(8, dtype=np.uint64)
    for rng in (0, 1):
        kw = dict(rng=rng, depth=3, fanout=30)
        dev, _ = device_run(g, roots, boff, seeds, gather=True, **kw)
        ref = O.bulk_shadow(g, roots, boff, seeds, gather=True, **kw)
        assert ref.V > 8 * 9000 / 2  # really oversize
        assert_same(dev, ref, True)


@pytest.mark.parametrize("depth,fanout", [(4, 16), (3, 40), (6, 6)])
def test_tree_bound_beyond_local_ids(depth, fanout):
    """Tree bounds beyond 32,767 (d=4 s=16: 69,905; d=3 s=40: 65,641; d=6
    s=6: 55,987) with actual sets well below it: K1's slots take the bound,
    K2 is sized from the touched lists; same results as the oracle."""
    g = random_graph(40000, 1000000, depth * fanout)
    rs = np.random.default_rng(fanout)
    roots = rs.choice(g.n, 24, replace=False).astype(np.int64)
    boff = np.array([0, 10, 24], np.int64)
    seeds = rs.integers(0, 2**63, 24, dtype=np.uint64)
    for rng in (0, 1):
        kw = dict(rng=rng, depth=depth, fanout=fanout)
        dev, _ = device_run(g, roots, boff, seeds, gather=True, **kw)
        ref = O.bulk_shadow(g, roots, boff, seeds, gather=True, **kw)
        assert_same(dev, ref, True)


def test_set_beyond_local_ids_is_erange():
    """A root whose induced subgraph has more than 32,767 vertices is
    reported (HGS_ERANGE naming the root), not silently wrapped."""
    H = hgs()
    g = random_graph(60000, 3000000, 5)
    G = H.Graph(g.rp, g.ci)
    S = H.Sampler(G)
    roots = np.array([5, 7], np.int64)
    with pytest.raises(H.HgsRuntimeError, match="per-root limit is 32767"):
        S.bulk_shadow(roots, np.array([0, 2], np.int64), np.arange(2, dtype=np.uint64),
                      rng=0, depth=3, fanout=60)
    # the handle stays usable
    S.bulk_shadow(roots, np.array([0, 2], np.int64), np.arange(2, dtype=np.uint64), rng=0, depth=2, fanout=4)
    S.close()
    G.close()


@pytest.mark.parametrize("rng", [0, 1])
def test_resumed_streams(rng):
    """Non-fresh sources (rng_state): xoshiro states / Philox decision bases."""
    rs = np.random.default_rng(77)
    g = random_graph(800, 6000, 4)
    roots = rs.permutation(800)[:100].astype(np.int64)
    boff = np.array([0, 60, 100], np.int64)
    seeds = rs.integers(0, 2**63, 100, dtype=np.uint64)
    state = (rs.integers(0, 2**63, 400, dtype=np.uint64) if rng == 0
             else rs.integers(0, 1000, 100).astype(np.uint64))
    dev, _ = device_run(g, roots, boff, seeds, state=state, rng=rng, depth=3, fanout=5)
    ref = O.bulk_shadow(g, roots, boff, seeds, state=state, rng=rng, depth=3, fanout=5)
    assert_same(dev, ref, False)


def test_shadow_reference_walk_semantics():
    """HGS_FLAG_SEQ_WALK: raw-row walk of shadow_reference (zeros kept)."""
    rs = np.random.default_rng(5)
    g = random_graph(400, 3000, 8)
    g.values = rs.uniform(0.5, 2.0, g.m)
    g.values[rs.random(g.m) < 0.3] = 0.0
    g.values[rs.random(g.m) < 0.05] = -1.0
    roots = rs.permutation(400)[:50].astype(np.int64)
    boff = np.array([0, 50], np.int64)
    seeds = rs.integers(0, 2**63, 50, dtype=np.uint64)
    dev, _ = device_run(g, roots, boff, seeds, depth=2, fanout=4, symmetrize=False, seq_walk=True)
    ref = O.bulk_shadow(g, roots, boff, seeds, depth=2, fanout=4, symmetrize=False, seq_walk=True)
    assert_same(dev, ref, False)
    # bulk semantics on the same graph rejects the negative rows it visits
    with pytest.raises(hgs().SamplerError, match="negative"):
        device_run(g, roots, boff, seeds, depth=2, fanout=4, symmetrize=False)
    with pytest.raises(O.SamplerError, match="negative"):
        O.bulk_shadow(g, roots, boff, seeds, depth=2, fanout=4, symmetrize=False)


@pytest.mark.parametrize("chunk", ["37", "64", "1000"])
def test_chunked_pipeline(monkeypatch, chunk):
    """Roots split into chunks (K3 of chunk c on the side stream next to K2 of
    chunk c+1): identical results for chunk sizes that cut through batches."""
    monkeypatch.setenv("HGS_CHUNK_ROOTS", chunk)
    g = random_graph(3000, 30000, 12)
    rs = np.random.default_rng(int(chunk))
    sizes = [300, 0, 17, 250, 1, 132]
    roots = np.concatenate([rs.permutation(3000)[:s] for s in sizes]).astype(np.int64)
    boff = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    seeds = rs.integers(0, 2**63, len(roots), dtype=np.uint64)
    for rng in (0, 1):
        kw = dict(rng=rng, depth=3, fanout=6)
        dev, S = device_run(g, roots, boff, seeds, gather=True, **kw)
        ref = O.bulk_shadow(g, roots, boff, seeds, gather=True, **kw)
        assert_same(dev, ref, True)
        dev2, _ = device_run(g, roots, boff, seeds, gather=True, sampler=S, **kw)  # reuse the handle
        assert_same(dev2, ref, True)


@pytest.mark.parametrize("total", [16384, 16385, 65536 + 4001, 131073])
def test_offset_scan_sizes(total):
    """The per-call offset scan at the one-CTA limit (16,384 roots,
    k_scan_small) and beyond it (the three-launch tiled scan) with ragged
    last tiles and an empty batch gives the oracle's outputs. (A one-CTA
    scan looping over up to 8 tiles measured slower at C2: 0.039 ms against
    0.022 ms for scan + finalize.)"""
    n = 3000
    g = random_graph(n, 9000, 7)
    rs = np.random.default_rng(total)
    sizes = [min(n, total - k) for k in range(0, total, n)]  # distinct roots per batch (check_roots)
    sizes.insert(1, 0)  # an empty batch
    roots = np.concatenate([rs.permutation(n)[:s] for s in sizes]).astype(np.int64)
    boff = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    seeds = rs.integers(0, 2**63, len(roots), dtype=np.uint64)
    kw = dict(rng=0, depth=2, fanout=3)
    dev, _ = device_run(g, roots, boff, seeds, **kw)
    ref = O.bulk_shadow(g, roots, boff, seeds, **kw)
    assert_same(dev, ref, False)


def test_capacity_regrow(monkeypatch):
    """Start with 4-edge slots and a 100-edge output: the device reports the
    overflow and the call is re-run with exact sizes."""
    monkeypatch.setenv("HGS_E_STRIDE", "4")
    monkeypatch.setenv("HGS_E_CAP", "100")
    g = random_graph(2000, 20000, 9)
    rs = np.random.default_rng(1)
    roots = rs.permutation(2000)[:300].astype(np.int64)
    boff = np.array([0, 150, 300], np.int64)
    seeds = rs.integers(0, 2**63, 300, dtype=np.uint64)
    dev, S = device_run(g, roots, boff, seeds, depth=3, fanout=6, gather=True)
    ref = O.bulk_shadow(g, roots, boff, seeds, depth=3, fanout=6, gather=True)
    assert_same(dev, ref, True)
    # the regrown workspace is reused without another retry
    dev2, _ = device_run(g, roots, boff, seeds, depth=3, fanout=6, gather=True, sampler=S)
    assert_same(dev2, ref, True)


def test_error_paths():
    H = hgs()
    g = random_graph(50, 200, 3)
    seeds = np.zeros(4, np.uint64)
    with pytest.raises(H.SamplerError, match="^sampler: duplicate root 3$"):
        device_run(g, [1, 3, 3], [0, 3], seeds[:3])
    with pytest.raises(H.SamplerError, match="^sampler: root 50 out of range$"):
        device_run(g, [1, 50], [0, 2], seeds[:2])
    with pytest.raises(H.SamplerError, match="depth must be >= 1"):
        device_run(g, [1], [0, 1], seeds[:1], depth=0)
    with pytest.raises(H.SamplerError, match="fanout must be >= 1"):
        device_run(g, [1], [0, 1], seeds[:1], fanout=0)
    rect = O.Graph(n=50, rp=g.rp, ci=g.ci, n_cols=60)
    with pytest.raises(H.SamplerError, match="symmetrize_pattern: matrix must be square"):
        device_run(rect, [1], [0, 1], seeds[:1])
    with pytest.raises(H.SamplerError, match=r"spgemm: inner dimensions disagree \(60 vs 50\)"):
        device_run(rect, [1], [0, 1], seeds[:1], symmetrize=False)
    # duplicates across batches are allowed (check_roots is per batch)
    device_run(g, [3, 3], [0, 1, 2], seeds[:2])


def test_device_pointer_entry_point():
    import torch
    H = hgs()
    g = random_graph(3000, 25000, 12)
    rs = np.random.default_rng(2)
    roots = np.concatenate([rs.permutation(3000)[:200] for _ in range(4)]).astype(np.int64)
    boff = np.arange(5, dtype=np.int64) * 200
    seeds = rs.integers(0, 2**63, 800, dtype=np.uint64)
    G = H.Graph(g.rp, g.ci).attach_features(g.node_feat, g.edge_feat, g.labels)
    st = torch.cuda.Stream()
    S = H.Sampler(G, stream=st.cuda_stream)
    dr = torch.from_numpy(roots.astype(np.int32)).cuda()
    db = torch.from_numpy(boff).cuda()
    ds = torch.from_numpy(seeds.view(np.int64)).cuda()
    torch.cuda.synchronize()
    S.run_device(dr.data_ptr(), db.data_ptr(), 800, 4, ds.data_ptr(), depth=3, fanout=6, gather=True,
                 profile=True)
    S.wait()
    dev = S.to_host()
    ref = O.bulk_shadow(g, roots, boff, seeds, depth=3, fanout=6, gather=True)
    assert_same(dev, ref, True)
    assert S.launches() >= 5
    assert (S.kernel_times() >= 0).all()
    st_ = S.stats()
    assert st_["V"] == ref.V and st_["E"] == ref.E


@pytest.mark.parametrize("rng", [0, 1])
def test_device_derived_seeds(rng):
    """hgs_sample_run_device_spec: per-root seeds derived inside K1 from a
    stream spec give the same subgraphs as uploading the host-derived seeds
    (bench-sampling and trainer streams, batch_base offsets, ragged batches)."""
    import torch
    H = hgs()
    g = random_graph(4000, 40000, 21)
    rs = np.random.default_rng(3)
    sizes = [100, 37, 0, 64, 1]
    roots = np.concatenate([rs.permutation(4000)[:s] for s in sizes]).astype(np.int64)
    boff = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    G = H.Graph(g.rp, g.ci).attach_features(g.node_feat, g.edge_feat, g.labels)
    S = H.Sampler(G)
    dr = torch.from_numpy(roots.astype(np.int32)).cuda()
    db = torch.from_numpy(boff).cuda()
    for spec in (H.bench_seed_spec(1, 5, 2), H.trainer_seed_spec(9, 1, 4, batch_base=17)):
        seeds = H.derive_seeds(spec, boff)
        kw = dict(rng=rng, depth=3, fanout=5, gather=True)
        S.run_device_spec(dr.data_ptr(), db.data_ptr(), len(roots), len(sizes), spec, **kw)
        S.wait()
        dev = S.to_host()
        ref = O.bulk_shadow(g, roots, boff, seeds, **kw)
        assert_same(dev, ref, True)


def test_epoch_sampler_matches_trainer_streams():
    """EpochSampler (C5 path): several resident events, every minibatch of an
    epoch in trainer order (trainer.cpp:433-459) with device-derived
    root_stream_seed streams, chunked over two handles; each chunk equals the
    oracle's bulk_shadow on the same roots and host-derived trainer seeds."""
    from paper_2504_04670_b200 import epoch as EP, workload as W
    H = hgs()
    graphs_o = [random_graph(n, 8 * n, 30 + n) for n in (700, 1300, 500)]
    graphs = [H.Graph(g.rp, g.ci).attach_features(g.node_feat, g.edge_feat, g.labels) for g in graphs_o]
    es = EP.EpochSampler(graphs, batch_size=64, bulk_batches=3, depth=3, fanout=4, seed=11, gather=True)
    seen = []

    def check(ch):
        g = graphs_o[ch.event_ordinal]
        batches = W.trainer_epoch_batches(g.n, 64, 11, 2, ch.event_ordinal)[ch.batch_base:ch.batch_base + ch.n_batches]
        roots = np.concatenate(batches).astype(np.int64)
        boff = np.concatenate([[0], np.cumsum([len(b) for b in batches])]).astype(np.int64)
        spec = H.trainer_seed_spec(11, 2, ch.event_ordinal, batch_base=ch.batch_base)
        ref = O.bulk_shadow(g, roots, boff, H.derive_seeds(spec, boff), depth=3, fanout=4, gather=True)
        assert_same(ch.sampler.to_host(), ref, True)
        seen.append((ch.event_ordinal, ch.batch_base))

    tot = es.epoch(2, on_chunk=check)
    es.close()
    exp = sum((g.n // 64 + 2) // 3 for g in graphs_o)
    assert tot["calls"] == exp == len(seen)
    assert tot["minibatches"] == sum(g.n // 64 for g in graphs_o)


@pytest.mark.parametrize("rng", [0, 1])
@pytest.mark.parametrize("s", [1, 3, 6, 17])
def test_sample_rows(rng, s):
    """hgs_sample_rows (sample_rows, sampler.cpp:64-86): rows on shared
    streams decided in row order, empty rows make no choose call, fresh and
    resumed sources; equals the oracle restatement."""
    H = hgs()
    rs = np.random.default_rng(100 + s + rng)
    n = 400
    deg = rs.integers(0, 40, n)
    deg[rs.random(n) < 0.15] = 0
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ci = np.concatenate([np.sort(rs.choice(5000, d, replace=False)) for d in deg]).astype(np.int64)
    seeds = rs.integers(0, 2**63, 37, dtype=np.uint64)
    streams = rs.integers(0, 37, n).astype(np.int64)
    for state in (None, "resume"):
        st = None
        if state:
            st = (rs.integers(0, 2**63, 4 * 37, dtype=np.uint64) if rng == 0
                  else rs.integers(0, 500, 37).astype(np.uint64))
        off, cols, draws, decs = H.sample_rows(rp, ci, s, seeds, streams, rng=rng, state=st, n_cols=5000)
        ref, _, ndec, _ = O.sample_rows(rp, ci, s, seeds, streams, rng=rng, state=st)
        got = [cols[off[r]:off[r + 1]].tolist() for r in range(n)]
        assert got == ref
        assert np.array_equal(decs.astype(np.int64), ndec)
    with pytest.raises(H.SamplerError, match="s must be >= 1"):
        H.sample_rows(rp, ci, 0, seeds, streams)
    with pytest.raises(H.SamplerError, match="root ordinal out of range"):
        H.sample_rows(rp, ci, 2, seeds[:3], streams)


@pytest.mark.parametrize("rng", [0, 1])
def test_sample_rows_wide(rng):
    """Rows of up to 2,000 entries with s=700: choices beyond 256 per row take
    the global-scratch choose path; equals the oracle restatement."""
    H = hgs()
    rs = np.random.default_rng(7 + rng)
    n = 60
    deg = rs.integers(0, 2000, n)
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ci = np.concatenate([np.sort(rs.choice(50000, d, replace=False)) for d in deg]).astype(np.int64)
    seeds = rs.integers(0, 2**63, 9, dtype=np.uint64)
    streams = rs.integers(0, 9, n).astype(np.int64)
    off, cols, draws, decs = H.sample_rows(rp, ci, 700, seeds, streams, rng=rng, n_cols=50000)
    ref, _, ndec, _ = O.sample_rows(rp, ci, 700, seeds, streams, rng=rng)
    assert [cols[off[r]:off[r + 1]].tolist() for r in range(n)] == ref
    assert np.array_equal(decs.astype(np.int64), ndec)


def test_threads_share_a_fresh_graph():
    """Sample handles on several host threads, one fresh graph (its walk and
    reciprocal table are built lazily by whichever call comes first): every
    thread's results equal the oracle's."""
    import concurrent.futures as cf
    H = hgs()
    g = random_graph(20000, 200000, 31)
    rs = np.random.default_rng(31)
    jobs = []
    for t in range(4):
        roots = rs.choice(g.n, 300, replace=False).astype(np.int64)
        jobs.append((roots, np.array([0, 100, 300], np.int64), rs.integers(0, 2**63, 300, dtype=np.uint64), t % 2))
    G = H.Graph(g.rp, g.ci)

    def run(job):
        roots, boff, seeds, rng = job
        S = H.Sampler(G)
        S.bulk_shadow(roots, boff, seeds, rng=rng, depth=3, fanout=6)
        out = S.to_host()
        S.close()
        return out

    with cf.ThreadPoolExecutor(4) as ex:
        outs = list(ex.map(run, jobs))
    for (roots, boff, seeds, rng), dev in zip(jobs, outs):
        assert_same(dev, O.bulk_shadow(g, roots, boff, seeds, rng=rng, depth=3, fanout=6), False)
    G.close()


def test_multi_handle_sharding_matches_single_call():
    """Two sample handles on one graph (as two ranks would be): the shard union
    equals the single call, batch for batch."""
    from paper_2504_04670_b200.sharding import shard
    H = hgs()
    g = random_graph(4000, 40000, 21)
    rs = np.random.default_rng(8)
    k, b = 6, 100
    roots = np.concatenate([rs.permutation(4000)[:b] for _ in range(k)]).astype(np.int64)
    boff = np.arange(k + 1, dtype=np.int64) * b
    seeds = rs.integers(0, 2**63, k * b, dtype=np.uint64)
    G = H.Graph(g.rp, g.ci).attach_features(g.node_feat, g.edge_feat, g.labels)
    full, _ = device_run(g, roots, boff, seeds, gather=True, sampler=H.Sampler(G), depth=3, fanout=6)
    parts = []
    for rank in range(2):
        r, bo, s = shard(roots, boff, seeds, rank, 2)
        out, _ = device_run(g, r, bo, s, gather=True, sampler=H.Sampler(G), depth=3, fanout=6)
        parts.append(out)
    for f in ("l2g", "e_row", "e_col", "e_gid", "xv", "ye", "lab"):
        assert np.array_equal(np.concatenate([p[f] for p in parts]), full[f]), f


def _batch_slices(out, boff, f_v, f_e):
    """Per batch: its arrays of a flat device result (batch-local ids)."""
    res = []
    for b in range(len(boff) - 1):
        v0, v1 = int(out["batch_voff"][b]), int(out["batch_voff"][b + 1])
        e0, e1 = int(out["batch_eoff"][b]), int(out["batch_eoff"][b + 1])
        f, nb = int(boff[b]), int(boff[b + 1] - boff[b])
        res.append({"l2g": out["l2g"][v0:v1], "e_row": out["e_row"][e0:e1], "e_col": out["e_col"][e0:e1],
                    "e_gid": out["e_gid"][e0:e1], "comp_off": out["comp_off"][f + b:f + b + nb + 1],
                    "roots_local": out["roots_local"][f:f + nb], "xv": out["xv"][v0 * f_v:v1 * f_v],
                    "ye": out["ye"][e0 * f_e:e1 * f_e], "lab": out["lab"][e0:e1],
                    "draws": out["draws"][f:f + nb], "decisions": out["decisions"][f:f + nb]})
    return res


@pytest.mark.parametrize("rng,k2", [(0, "hash"), (1, "hash"), (0, "bm"), (1, "dir")])
def test_multi_event_call_matches_per_event_calls(rng, k2, monkeypatch):
    """hgs_sample_run_multi (SURVEY §8(e) multi-event launches): one call over
    batches of several resident events (one without batches, different sizes
    and degrees) equals one call per event, batch for batch, and the oracle —
    with every K2 kernel (the bitmap one sizes its directory for the largest
    event)."""
    monkeypatch.setenv("HGS_K2", k2)
    H = hgs()
    graphs = [random_graph(3000, 30000, 31), random_graph(500, 2000, 32), random_graph(8000, 120000, 33)]
    Gs = [H.Graph(g.rp, g.ci).attach_features(g.node_feat, g.edge_feat, g.labels) for g in graphs]
    rs = np.random.default_rng(9)
    plan = [(0, 3, 120), (2, 4, 200)]  # (event, batches, batch size); event 1 has none
    roots, boff, bev, seeds = [], [0], [], []
    per_event = {}
    for e, k, b in plan:
        rr = np.concatenate([rs.permutation(graphs[e].n)[:b] for _ in range(k)]).astype(np.int64)
        ss = rs.integers(0, 2**63, k * b, dtype=np.uint64)
        per_event[e] = (rr, np.arange(k + 1, dtype=np.int64) * b, ss)
        roots.append(rr)
        seeds.append(ss)
        for _ in range(k):
            boff.append(boff[-1] + b)
            bev.append(e)
    roots, seeds, boff = np.concatenate(roots), np.concatenate(seeds), np.array(boff, np.int64)
    S = H.Sampler(Gs[0])
    S.bulk_shadow_multi(Gs, bev, roots, boff, seeds, depth=3, fanout=5, rng=rng, gather=True)
    multi = _batch_slices(S.to_host(), boff, 6, 2)
    got = []
    for e, k, b in plan:
        rr, bo, ss = per_event[e]
        Se = H.Sampler(Gs[e])
        Se.bulk_shadow(rr, bo, ss, depth=3, fanout=5, rng=rng, gather=True)
        got += _batch_slices(Se.to_host(), bo, 6, 2)
        ref = O.bulk_shadow(graphs[e], rr, bo, ss, rng=rng, depth=3, fanout=5, gather=True)
        assert not compare(Se.to_host(), ref, gather=True)
    assert len(got) == len(multi)
    for b, (m, p) in enumerate(zip(multi, got)):
        for f in m:
            assert np.array_equal(np.asarray(m[f]).view(np.uint8), np.asarray(p[f]).view(np.uint8)), (b, f)


def test_slice_after_multi_and_device_runs():
    """hgs_sample_slice reads the last run's batch offsets for host-input,
    device-input and multi-event runs alike."""
    import torch
    from oracle import consumer as CO
    from paper_2504_04670_b200 import consumer
    H = hgs()
    g0, g1 = random_graph(2000, 16000, 51), random_graph(900, 7000, 52)
    Gs = [H.Graph(g.rp, g.ci).attach_features(g.node_feat, g.edge_feat, g.labels) for g in (g0, g1)]
    rs = np.random.default_rng(4)
    r0 = np.concatenate([rs.permutation(2000)[:50] for _ in range(2)])
    r1 = np.concatenate([rs.permutation(900)[:40] for _ in range(3)])
    roots = np.concatenate([r0, r1]).astype(np.int64)
    boff = np.array([0, 50, 100, 140, 180, 220], np.int64)
    seeds = rs.integers(0, 2**63, len(roots), dtype=np.uint64)
    S = H.Sampler(Gs[0])
    S.bulk_shadow_multi(Gs, [0, 0, 1, 1, 1], roots, boff, seeds, depth=2, fanout=4, gather=True)
    ref1 = O.bulk_shadow(g1, r1.astype(np.int64), np.array([0, 40, 80, 120], np.int64), seeds[100:],
                         depth=2, fanout=4, gather=True)
    sl = consumer.slice_components(S, 3, 5, 30)  # event 1's second batch
    want = CO.slice_components(CO.batch_of(ref1, np.array([0, 40, 80, 120]), 1, 6, 2), 5, 30)
    assert np.array_equal(sl.e_col.cpu().numpy(), want["e_col"])
    assert np.array_equal(sl.edge_features.cpu().numpy().view(np.uint64), want["ye"].view(np.uint64))
    # device inputs
    d_r = torch.as_tensor(r1.astype(np.int32), device="cuda")
    d_b = torch.as_tensor(np.array([0, 40, 80, 120], np.int64), device="cuda")
    d_s = torch.as_tensor(seeds[100:].view(np.int64), device="cuda")
    S1 = H.Sampler(Gs[1])
    S1.run_device(d_r.data_ptr(), d_b.data_ptr(), 120, 3, d_s.data_ptr(), depth=2, fanout=4, gather=True)
    S1.wait()
    sl = consumer.slice_components(S1, 1, 5, 30)
    assert np.array_equal(sl.e_col.cpu().numpy(), want["e_col"])
    assert np.array_equal(sl.node_features.cpu().numpy().view(np.uint64), want["xv"].view(np.uint64))


def test_multi_event_call_errors():
    H = hgs()
    g0, g1 = random_graph(300, 2000, 41), random_graph(100, 500, 42)
    Gs = [H.Graph(g.rp, g.ci) for g in (g0, g1)]
    S = H.Sampler(Gs[0])
    roots = np.array([5, 7, 150, 3], np.int64)
    boff = np.array([0, 2, 4], np.int64)
    seeds = np.arange(4, dtype=np.uint64)
    with pytest.raises(H.SamplerError, match="sampler: root 150 out of range"):
        S.bulk_shadow_multi(Gs, [0, 1], roots, boff, seeds, depth=2, fanout=3)
    with pytest.raises(H.SamplerError, match="batch events must be non-decreasing"):
        S.bulk_shadow_multi(Gs, [1, 0], np.array([5, 7, 1, 3], np.int64), boff, seeds, depth=2, fanout=3)
    S.bulk_shadow_multi(Gs, [0, 1], np.array([5, 7, 99, 3], np.int64), boff, seeds, depth=2, fanout=3)
    assert S.counts.k == 2


# ------------------------------------------------------------------ C1 / C2 ----

def test_c1_matches_reference_digests():
    from paper_2504_04670_b200 import workload as W
    c1 = load_json("c1.json")
    ev = W.preset_event("C1")
    roots, boff, seeds = W.bench_roots(ev.n, 256, 16, seed=1, rep=0)
    H = hgs()
    S = H.Sampler(H.Graph(ev.rp, ev.ci).attach_features(ev.node_feat, ev.edge_feat, ev.labels))
    for run in c1["runs"]:
        S.bulk_shadow(roots, boff, seeds, rng=run["rng"], depth=run["depth"], fanout=6, gather=True)
        dev = S.to_host()
        assert (S.counts.V, S.counts.E) == (run["V"], run["E"])
        for f in ("batch_voff", "batch_eoff", "comp_off", "l2g", "roots_local", "e_row", "e_col",
                  "e_gid"):
            assert sha(np.asarray(dev[f]).astype(np.int64)) == run["digests"][f], f
        for f in ("xv", "ye", "lab"):
            assert sha(dev[f]) == run["digests"][f], f


def test_c2_full_workload():
    """BASELINE configs[1] at full size: 64 x 1024 roots, d=3, s=6, gather.
    Bit-exact against the oracle, plus size-independent properties."""
    from paper_2504_04670_b200 import workload as W
    ev = W.preset_event("C2")
    roots, boff, seeds = W.bench_roots(ev.n, 1024, 64, seed=1, rep=0)
    H = hgs()
    S = H.Sampler(H.Graph(ev.rp, ev.ci).attach_features(ev.node_feat, ev.edge_feat, ev.labels))
    S.bulk_shadow(roots, boff, seeds, depth=3, fanout=6, gather=True)
    dev = S.to_host()
    # properties: every component sorted, contains its root, edges in-component
    bv, co, l2g = dev["batch_voff"], dev["comp_off"], dev["l2g"]
    assert bv[-1] == S.counts.V and dev["batch_eoff"][-1] == S.counts.E
    for bi in (0, 31, 63):
        offs = co[boff[bi] + bi: boff[bi + 1] + bi + 1]
        base = bv[bi]
        for c in range(0, 1024, 97):
            seg = l2g[base + offs[c]: base + offs[c + 1]]
            assert np.all(np.diff(seg) > 0)
            assert seg[dev["roots_local"][boff[bi] + c] - offs[c]] == roots[boff[bi] + c]
    rows = dev["e_row"].astype(np.int64)
    assert np.all(ev.ci[dev["e_gid"]] >= 0)
    g = O.Graph(n=ev.n, rp=ev.rp, ci=ev.ci, node_feat=ev.node_feat, edge_feat=ev.edge_feat,
                labels=ev.labels)
    ref = O.bulk_shadow(g, roots, boff, seeds, depth=3, fanout=6, gather=True)
    assert (S.counts.V, S.counts.E) == (ref.V, ref.E) == (14330269, 17161199)
    assert_same(dev, ref, True)
    del rows


def test_hub_root_gets_exact_slots():
    """One root whose induced subgraph has ~11k edges among 4,096 small ones:
    growing every root's edge slot to fit it would take (R+1) x 16,384 slots,
    so the re-run places edges at exact per-root offsets instead (ADVICE r1:
    a hub no longer inflates every slot or fails with an allocation error)."""
    H = hgs()
    rs = np.random.default_rng(17)
    n, clique = 40000, 150
    u = rs.integers(0, n, 120000)
    v = rs.integers(0, n, 120000)
    cu, cv = np.meshgrid(np.arange(clique), np.arange(clique), indexing="ij")
    u = np.concatenate([u, cu.ravel()])
    v = np.concatenate([v, cv.ravel()])
    keep = u != v
    key = np.unique(u[keep].astype(np.int64) * n + v[keep])
    rp = np.concatenate([[0], np.cumsum(np.bincount(key // n, minlength=n))]).astype(np.int64)
    g = O.Graph(n=n, rp=rp, ci=(key % n).astype(np.int64))
    g.node_feat, g.edge_feat = rs.standard_normal((n, 6)), rs.standard_normal((len(key), 2))
    g.labels = rs.integers(0, 2, len(key)).astype(np.uint8)
    roots = np.concatenate([[3], rs.choice(np.arange(clique, n), 4095, replace=False)]).astype(np.int64)
    boff = np.array([0, 2048, 4096], np.int64)
    seeds = rs.integers(0, 2**63, 4096, dtype=np.uint64)
    kw = dict(depth=2, fanout=60, gather=True)
    dev, S = device_run(g, roots, boff, seeds, **kw)
    assert S.reruns() == 1
    ref = O.bulk_shadow(g, roots, boff, seeds, **kw)
    assert ref.batch_eoff[1] > 11000
    assert_same(dev, ref, True)


@pytest.mark.parametrize("every", [0, 1, 3])
def test_k1_xoshiro_serial_fallback(monkeypatch, every):
    """The decision-parallel xoshiro K1 (HGS_K1_GROUPX=1) hands a root whose
    stream saw a rejected draw to the serial per-root path; HGS_K1_FORCE_SERIAL
    forces that path for every `every`-th root (0: none). Mixed roots give the oracle's outputs and
    per-root draw / decision counts."""
    monkeypatch.setenv("HGS_K1_GROUPX", "1")
    monkeypatch.setenv("HGS_K1_FORCE_SERIAL", str(every))
    g = random_graph(6000, 60000, 23)
    rs = np.random.default_rng(23)
    roots = np.concatenate([rs.permutation(6000)[:500] for _ in range(3)]).astype(np.int64)
    boff = np.array([0, 500, 1000, 1500], np.int64)
    seeds = rs.integers(0, 2**63, 1500, dtype=np.uint64)
    state = rs.integers(0, 2**63, 4 * 1500, dtype=np.uint64)
    for st in (None, state):
        dev, _ = device_run(g, roots, boff, seeds, depth=3, fanout=6, gather=True, state=st)
        ref = O.bulk_shadow(g, roots, boff, seeds, depth=3, fanout=6, gather=True, state=st)
        assert_same(dev, ref, True)


def test_event_file_load_matches_arrays(tmp_path):
    """Ingest (§8f #2): a C1 event written with hgs_event_save and loaded
    with hgs_graph_load (mmap, device-side narrowing and validation) samples
    exactly like the graph built from host arrays; reference digests hold."""
    from paper_2504_04670_b200 import workload as W
    H = hgs()
    ev = W.preset_event("C1")
    p = str(tmp_path / "c1.hgsev")
    H.save_event(p, ev.rp, ev.ci, node_feat=ev.node_feat, edge_feat=ev.edge_feat, labels=ev.labels)
    G = H.Graph.load(p)
    assert (G.n, G.nnz, G.f_v, G.f_e) == (ev.n, ev.m, 6, 2)
    roots, boff, seeds = W.bench_roots(ev.n, 256, 16, seed=1, rep=0)
    c1 = load_json("c1.json")
    S = H.Sampler(G)
    for run in c1["runs"]:
        S.bulk_shadow(roots, boff, seeds, rng=run["rng"], depth=run["depth"], fanout=6, gather=True)
        dev = S.to_host()
        for f in ("l2g", "e_row", "e_col", "e_gid"):
            assert sha(np.asarray(dev[f]).astype(np.int64)) == run["digests"][f], f
        for f in ("xv", "ye", "lab"):
            assert sha(dev[f]) == run["digests"][f], f


@pytest.mark.parametrize("values", [False, True])
def test_ingest_validation_messages(values):
    """Device-side ingest (edge-id A) and the host path (general values) report
    the first invalid entry in row-major order with the same text."""
    H = hgs()
    va = np.ones(4) if values else None
    with pytest.raises(H.SamplerError, match=r"^CsrMatrix: entry \(1, 7\) out of range for 3x3$"):
        H.Graph(np.array([0, 1, 3, 4]), np.array([1, 2, 7, 9]), va)
    with pytest.raises(H.SamplerError, match="row_ptr not non-decreasing"):
        H.Graph(np.array([0, 3, 2, 4]), np.array([1, 2, 0, 1]), va)
    # a bad column in a row before the first decreasing row pointer is met first
    with pytest.raises(H.SamplerError, match=r"^CsrMatrix: entry \(0, 5\) out of range for 3x3$"):
        H.Graph(np.array([0, 2, 1, 4]), np.array([5, 2, 0, 1]), va)


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("f_v,f_e", [(1, 1), (2, 2), (3, 5), (8, 2), (510, 3)])
def test_feature_widths(monkeypatch, fused, f_v, f_e):
    """gather_features for any row widths, through the fused K3 and the
    pack + flat-gather path: f_v = 2 (a single 16-byte piece per row, where a
    magic divisor of 2^32 would wrap) and f_v = 510 (q = 255, whose rounded
    reciprocal is inexact beyond ~66k pieces: 4,000 vertices x 255 pieces
    exceed that) included."""
    monkeypatch.setenv("HGS_K3_FUSED", fused)
    H = hgs()
    g = random_graph(5000, 40000, 3)
    rs = np.random.default_rng(f_v + f_e)
    g.node_feat = rs.standard_normal((g.n, f_v))
    g.edge_feat = rs.standard_normal((len(g.ci), f_e))
    roots = np.concatenate([rs.permutation(g.n)[:700] for _ in range(2)]).astype(np.int64)
    boff = np.array([0, 700, 1400], np.int64)
    seeds = rs.integers(0, 2**63, 1400, dtype=np.uint64)
    dev, S = device_run(g, roots, boff, seeds, depth=3, fanout=4, gather=True)
    assert S.counts.V > 4000
    ref = O.bulk_shadow(g, roots, boff, seeds, depth=3, fanout=4, gather=True)
    assert_same(dev, ref, True)
