"""CPU, multi-process: the N>1 data path shards minibatches across ranks with
no collective. world_size=2 over gloo: each rank samples its contiguous batch
range (paper_2504_04670_b200.sharding) with the checker; the gathered union
must equal the single-process result batch for batch (per-root streams make
the output shard-invariant)."""
import os

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.helpers import O, random_graph

FIELDS = ["l2g", "e_row", "e_col", "e_gid", "roots_local"]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_04670_b200.sharding import shard
    g = random_graph(300, 1500, 11)
    rs = np.random.default_rng(3)
    k, b = 7, 20
    roots = np.concatenate([rs.permutation(300)[:b] for _ in range(k)]).astype(np.int64)
    boff = np.arange(k + 1, dtype=np.int64) * b
    seeds = rs.integers(0, 2**63, k * b, dtype=np.uint64)
    r, bo, s = shard(roots, boff, seeds, rank, world)
    out = O.bulk_shadow(g, r, bo, s, depth=2, fanout=4, gather=True)
    parts = [None] * world
    dist.all_gather_object(parts, {f: getattr(out, f) for f in FIELDS} | {"bv": out.batch_voff})
    if rank == 0:
        full = O.bulk_shadow(g, roots, boff, seeds, depth=2, fanout=4, gather=True)
        ok = True
        for f in ("l2g", "e_gid"):
            ok &= np.array_equal(np.concatenate([p[f] for p in parts]), getattr(full, f))
        ok &= np.array_equal(np.concatenate([p["roots_local"] for p in parts]),
                             np.concatenate([full.roots_local[boff[b0]:boff[b1]]
                                             for b0, b1 in ((0, 3), (3, 7))]))
        q.put(bool(ok))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_is_exact():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10)


def test_batch_range_partition():
    from paper_2504_04670_b200.sharding import batch_range
    for k in (1, 7, 64, 512):
        for world in (1, 2, 3, 8):
            rs = [batch_range(k, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == k
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
