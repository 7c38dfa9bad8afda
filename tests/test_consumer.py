"""CPU: the consumer row. The oracle restatements
(oracle/consumer.py) against golden vectors from the unmodified reference
(tests/golden/consumer.npz, tests/golden/make_consumer_golden.py) and, where
oracle/_ref exists, against the live reference on random cases; and the
multi-rank plumbing of consumer.allreduce_coalesced (all-to-all of chunks,
rank-ordered reduction, all-gather) over gloo with world sizes 2 and 3, the
oracle's reducer injected so no CUDA is needed."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import consumer as CO
from tests.helpers import GOLDEN, O, random_graph

G = np.load(os.path.join(GOLDEN, "consumer.npz"))
REF = CO.ref_available()


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def sampled_case():
    g = random_graph(900, 7000, 41)
    rs = np.random.default_rng(42)
    roots = np.concatenate([rs.permutation(g.n)[:40] for _ in range(3)]).astype(np.int64)
    boff = np.array([0, 40, 80, 120], np.int64)
    seeds = rs.integers(0, 2**63, 120, dtype=np.uint64)
    return g, boff, O.bulk_shadow(g, roots, boff, seeds, depth=2, fanout=4, gather=True)


def test_slice_components_matches_reference_golden():
    g, boff, s = sampled_case()
    for i, (b, lo, hi) in enumerate(G["slice_ranges"]):
        got = CO.slice_components(CO.batch_of(s, boff, int(b), 6, 2), int(lo), int(hi))
        for k in ("comp_off", "l2g", "roots_local", "e_row", "e_col", "e_gid", "lab"):
            assert np.array_equal(np.asarray(got[k]).astype(np.int64), G[f"slice{i}_{k}"].astype(np.int64)), (i, k)
        for k in ("xv", "ye"):
            assert np.array_equal(bits(got[k]), bits(G[f"slice{i}_{k}"])), (i, k)


def test_slice_components_bad_range():
    g, boff, s = sampled_case()
    batch = CO.batch_of(s, boff, 0, 6, 2)
    for lo, hi in ((-1, 3), (4, 3), (0, 41)):
        with pytest.raises(CO.ConsumerError, match="slice_components: bad component range"):
            CO.slice_components(batch, lo, hi)
        if REF:
            with pytest.raises(CO.ConsumerError, match="slice_components: bad component range"):
                CO.ref_slice_components(batch, lo, hi)


@pytest.mark.parametrize("case", range(4))
def test_gather_scatter_match_reference_golden(case):
    x, idx, y = G[f"gs{case}_x"], G[f"gs{case}_idx"], G[f"gs{case}_y"]
    n = x.shape[0]
    assert np.array_equal(bits(CO.gather_rows(x, idx)), bits(G[f"gs{case}_gather"]))
    assert np.array_equal(bits(CO.scatter_add(y, idx, n)), bits(G[f"gs{case}_scatter"]))
    # backward: gather's input gradient = scatter-add of its output gradient, scatter's = gather
    assert np.array_equal(bits(CO.scatter_add(G[f"gs{case}_gather_gout"], idx, n)), bits(G[f"gs{case}_gather_gin"]))
    assert np.array_equal(bits(CO.gather_rows(G[f"gs{case}_scatter_gout"], idx)), bits(G[f"gs{case}_scatter_gin"]))


def test_scatter_add_is_order_sensitive():
    """The fixtures would catch a different summation order: a pairwise or
    reversed sum of the same rows changes the bits."""
    y, idx = G["gs1_y"], G["gs1_idx"]
    ref = G["gs1_scatter"]
    rev = CO.scatter_add(y[::-1], idx[::-1], 7)
    assert not np.array_equal(bits(rev), bits(ref))


@pytest.mark.parametrize("w", range(1, 6))
def test_allreduce_mean_matches_reference_golden(w):
    assert np.array_equal(bits(CO.allreduce_mean(G[f"ar{w}_in"])), bits(G[f"ar{w}_out"]))


def test_errors_match_reference_text():
    x = np.zeros((3, 2))
    with pytest.raises(CO.ConsumerError, match="gather_rows: index 3 out of range"):
        CO.gather_rows(x, [0, 3])
    with pytest.raises(CO.ConsumerError, match="scatter_add: index -1 out of range"):
        CO.scatter_add(np.zeros((2, 2)), [1, -1], 3)
    with pytest.raises(CO.ConsumerError, match="scatter_add: index list length must equal row count"):
        CO.scatter_add(np.zeros((2, 2)), [1], 3)
    if REF:
        with pytest.raises(CO.ConsumerError, match="gather_rows: index 3 out of range"):
            CO.ref_gather_rows(x, [0, 3])
        with pytest.raises(CO.ConsumerError, match="scatter_add: index -1 out of range"):
            CO.ref_scatter_add(np.zeros((2, 2)), [1, -1], 3)


@pytest.mark.skipif(not REF, reason="oracle/_ref (the compiled reference) not built here")
def test_oracle_matches_live_reference_random():
    rs = np.random.default_rng(99)
    for _ in range(20):
        n, m, c = int(rs.integers(1, 60)), int(rs.integers(0, 300)), int(rs.integers(1, 7))
        x = rs.standard_normal((n, c)) * np.exp2(rs.integers(-20, 20, (n, c)))
        y = rs.standard_normal((m, c)) * np.exp2(rs.integers(-20, 20, (m, c)))
        idx = rs.integers(0, n, m)
        assert np.array_equal(bits(CO.gather_rows(x, idx)), bits(CO.ref_gather_rows(x, idx)))
        assert np.array_equal(bits(CO.scatter_add(y, idx, n)), bits(CO.ref_scatter_add(y, idx, n)))
        w = int(rs.integers(1, 7))
        parts = rs.standard_normal((w, 50)) * np.exp2(rs.integers(-30, 30, (w, 50)))
        assert np.array_equal(bits(CO.allreduce_mean(parts)), bits(CO.ref_allreduce_mean(parts)))
    g, boff, s = sampled_case()
    for b in range(3):
        batch = CO.batch_of(s, boff, b, 6, 2)
        for _ in range(5):
            lo = int(rs.integers(0, 41))
            hi = int(rs.integers(lo, 41))
            got, ref = CO.slice_components(batch, lo, hi), CO.ref_slice_components(batch, lo, hi)
            for k in ref:
                assert np.array_equal(np.asarray(got[k]).view(np.uint8), np.asarray(ref[k]).view(np.uint8)), k


def _np_reducer(parts: torch.Tensor) -> torch.Tensor:
    return torch.from_numpy(CO.allreduce_mean(parts.numpy()))


def _ar_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_04670_b200 import consumer
    data = G[f"ar{world}_in"]
    flat = torch.from_numpy(data[rank].copy())
    consumer.allreduce_coalesced(flat, reducer=_np_reducer)
    q.put((rank, bool(np.array_equal(flat.numpy().view(np.uint64), G[f"ar{world}_out"].view(np.uint64)))))
    # mismatched lengths raise the reference's error on every rank
    bad = torch.zeros(5 + rank, dtype=torch.float64)
    try:
        consumer.allreduce_coalesced(bad, reducer=_np_reducer)
        q.put((rank, "no error"))
    except ValueError as e:
        q.put((rank, str(e)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allreduce_coalesced_plumbing_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + world
    procs = [ctx.Process(target=_ar_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2 * world)]
    for p in procs:
        p.join(timeout=60)
    assert all(v is True for (_, v) in res if isinstance(v, bool)), res
    errs = [v for (_, v) in res if isinstance(v, str)]
    assert errs == ["allreduce: buffer lengths differ across ranks"] * world, errs
