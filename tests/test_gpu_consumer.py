"""GPU: the consumer row through the C ABI — device
slice_components over a run's outputs, gather_rows / scatter_add forward and
backward (also as torch autograd functions), the rank-ordered reduction of
the coalesced all-reduce, and one IGNN message-passing step on a sliced
batch — bit for bit against the oracle / the reference's golden vectors."""
import os

import numpy as np
import pytest
import torch

from oracle import consumer as CO
from tests.helpers import GOLDEN, O, random_graph

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(GOLDEN, "consumer.npz"))


def H():
    from paper_2504_04670_b200 import hgs
    return hgs


def C():
    from paper_2504_04670_b200 import consumer
    return consumer


def bits(a):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def cuda(a, dt=None):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda", dtype=dt)


@pytest.fixture(scope="module")
def run():
    hg = H()
    g = random_graph(900, 7000, 41)
    rs = np.random.default_rng(42)
    roots = np.concatenate([rs.permutation(g.n)[:40] for _ in range(3)]).astype(np.int64)
    boff = np.array([0, 40, 80, 120], np.int64)
    seeds = rs.integers(0, 2**63, 120, dtype=np.uint64)
    S = hg.Sampler(hg.Graph(g.rp, g.ci).attach_features(g.node_feat, g.edge_feat, g.labels))
    S.bulk_shadow(roots, boff, seeds, depth=2, fanout=4, gather=True)
    ref = O.bulk_shadow(g, roots, boff, seeds, depth=2, fanout=4, gather=True)
    return S, boff, ref


def test_device_slice_matches_reference_golden(run):
    S, boff, ref = run
    for i, (b, lo, hi) in enumerate(G["slice_ranges"]):
        sl = C().slice_components(S, int(b), int(lo), int(hi))
        got = {"comp_off": sl.component_offsets, "l2g": sl.local_to_global, "roots_local": sl.roots_local,
               "e_row": sl.e_row, "e_col": sl.e_col, "e_gid": sl.edge_global_ids, "lab": sl.edge_labels}
        for k, v in got.items():
            assert np.array_equal(v.cpu().numpy().astype(np.int64), G[f"slice{i}_{k}"].astype(np.int64)), (i, k)
        assert np.array_equal(bits(sl.node_features), bits(G[f"slice{i}_xv"])), i
        assert np.array_equal(bits(sl.edge_features), bits(G[f"slice{i}_ye"])), i


def test_device_slice_errors(run):
    S, boff, ref = run
    for b, lo, hi in ((0, -1, 2), (1, 5, 4), (2, 0, 41)):
        with pytest.raises(H().SamplerError, match="slice_components: bad component range"):
            C().slice_components(S, b, lo, hi)


@pytest.mark.parametrize("case", range(4))
def test_gather_scatter_forward_backward_golden(case):
    co = C()
    x, idx, y = G[f"gs{case}_x"], G[f"gs{case}_idx"], G[f"gs{case}_y"]
    n = x.shape[0]
    di = cuda(idx, torch.int32)
    plan = co.ScatterPlan(di, n)
    assert np.array_equal(bits(co.gather_rows(cuda(x), di)), bits(G[f"gs{case}_gather"]))
    assert np.array_equal(bits(co.scatter_add(cuda(y), plan)), bits(G[f"gs{case}_scatter"]))
    # backward passes as the reference tape computes them
    assert np.array_equal(bits(co.scatter_add(cuda(G[f"gs{case}_gather_gout"]), plan)), bits(G[f"gs{case}_gather_gin"]))
    assert np.array_equal(bits(co.gather_rows(cuda(G[f"gs{case}_scatter_gout"]), di)), bits(G[f"gs{case}_scatter_gin"]))
    # the planned gather (no re-check) gives the same rows; a sorted list takes the no-sort plan
    assert np.array_equal(bits(co.gather_rows_planned(cuda(x), plan)), bits(G[f"gs{case}_gather"]))
    sidx = np.sort(idx)
    splan = co.ScatterPlan(cuda(sidx, torch.int32), n)
    assert np.array_equal(bits(co.scatter_add(cuda(y), splan)), bits(CO.scatter_add(y, sidx, n)))
    splan.close()
    # the same through torch autograd
    xt = cuda(x).requires_grad_(True)
    out = co.GatherRows.apply(xt, di, plan)
    out.backward(cuda(G[f"gs{case}_gather_gout"]))
    assert np.array_equal(bits(xt.grad), bits(G[f"gs{case}_gather_gin"]))
    yt = cuda(y).requires_grad_(True)
    out = co.ScatterAdd.apply(yt, plan)
    out.backward(cuda(G[f"gs{case}_scatter_gout"]))
    assert np.array_equal(bits(yt.grad), bits(G[f"gs{case}_scatter_gin"]))
    # accumulate onto an existing buffer (gradient fan-in) = the oracle's ordered adds
    base = np.random.default_rng(case).standard_normal((n, x.shape[1]))
    acc = co.scatter_add(cuda(y), plan, out=cuda(base.copy()), accumulate=True)
    assert np.array_equal(bits(acc), bits(CO.scatter_add(y, idx, n, out=base)))
    plan.close()


def test_gather_scatter_errors():
    co = C()
    x = cuda(np.zeros((3, 2)))
    with pytest.raises(H().SamplerError, match="gather_rows: index 3 out of range"):
        co.gather_rows(x, cuda([0, 3], torch.int32))
    with pytest.raises(H().SamplerError, match="scatter_add: index -1 out of range"):
        co.ScatterPlan(cuda([1, -1], torch.int32), 3)


@pytest.mark.parametrize("w", range(1, 6))
def test_ordered_mean_golden(w):
    assert np.array_equal(bits(C().ordered_mean(cuda(G[f"ar{w}_in"]))), bits(G[f"ar{w}_out"]))


def test_allreduce_coalesced_world1_nccl():
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("process group already initialised")
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29651", rank=0, world_size=1)
    try:
        flat = cuda(G["ar1_in"][0].copy())
        C().allreduce_coalesced(flat)
        assert np.array_equal(bits(flat), bits(G["ar1_out"]))
    finally:
        dist.destroy_process_group()


def test_message_passing_step_on_slice(run):
    """One IGNN message-passing step (ignn.cpp:156-167 minus the MLPs) on a
    DDP slice of a batch: x_src/x_dst gathers and the two scatters, plus
    their backward passes, against the oracle on the same slice."""
    S, boff, ref = run
    co = C()
    batch = CO.batch_of(ref, boff, 1, 6, 2)
    lo, hi = 10, 30
    sl = co.slice_components(S, 1, lo, hi)
    want = CO.slice_components(batch, lo, hi)
    nv = sl.n_vertices
    rows, cols = sl.e_row, sl.e_col
    x, y = sl.node_features, sl.edge_features
    prow, pcol = co.ScatterPlan(rows, nv), co.ScatterPlan(cols, nv)
    x_src, x_dst = co.gather_rows(x, rows), co.gather_rows(x, cols)
    m_src, m_dst = co.scatter_add(y, prow), co.scatter_add(y, pcol)
    wr, wc = want["e_row"], want["e_col"]
    assert np.array_equal(bits(x_src), bits(CO.gather_rows(want["xv"], wr)))
    assert np.array_equal(bits(x_dst), bits(CO.gather_rows(want["xv"], wc)))
    assert np.array_equal(bits(m_src), bits(CO.scatter_add(want["ye"], wr, nv)))
    assert np.array_equal(bits(m_dst), bits(CO.scatter_add(want["ye"], wc, nv)))
    # x_src and x_dst both feed the loss: gradient fan-in accumulates in tape order
    g1 = np.random.default_rng(5).standard_normal(tuple(x_src.shape))
    g2 = np.random.default_rng(6).standard_normal(tuple(x_dst.shape))
    gx = co.scatter_add(cuda(g1), prow)
    gx = co.scatter_add(cuda(g2), pcol, out=gx, accumulate=True)
    want_gx = CO.scatter_add(g2, wc, nv, out=CO.scatter_add(g1, wr, nv))
    assert np.array_equal(bits(gx), bits(want_gx))
