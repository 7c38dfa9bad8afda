"""Small sampling calls for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): K0, K1 (serial, Philox group, xoshiro group), K2 (hash-set,
directory and bitmap-directory variants), offset scan, K3 pack + gathers, the standalone gather,
the ingest kernels and the consumer kernels, each checked against the oracle.
usage: compute-sanitizer --tool <tool> python scripts/sanitize_case.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.helpers import O, compare, random_graph  # noqa: E402
from paper_2504_04670_b200 import hgs  # noqa: E402

g = random_graph(1500, 12000, 5)
G = hgs.Graph(g.rp, g.ci).attach_features(g.node_feat, g.edge_feat, g.labels)
rs = np.random.default_rng(5)
roots = np.concatenate([rs.permutation(1500)[:64] for _ in range(3)]).astype(np.int64)
boff = np.array([0, 64, 128, 192], np.int64)
seeds = rs.integers(0, 2**63, 192, dtype=np.uint64)
bad = 0
for env in ({}, {"HGS_K2": "dir"}, {"HGS_K2": "bm"}, {"HGS_K1_GROUPX": "1"}):
    for k, v in env.items():
        os.environ[k] = v
    S = hgs.Sampler(G)
    for rng in (0, 1):
        S.bulk_shadow(roots, boff, seeds, rng=rng, depth=3, fanout=5, gather=True)
        diff = compare(S.to_host(), O.bulk_shadow(g, roots, boff, seeds, rng=rng, depth=3, fanout=5, gather=True),
                       gather=True)
        bad += bool(diff)
        print(env, "rng", rng, "diff", diff, flush=True)
    S.close()
    for k in env:
        del os.environ[k]
# consumer kernels (slice_components, gather_rows / scatter_add, ordered mean) on the last run
import torch  # noqa: E402
from oracle import consumer as CO  # noqa: E402
from paper_2504_04670_b200 import consumer  # noqa: E402
S = hgs.Sampler(G)
S.bulk_shadow(roots, boff, seeds, rng=0, depth=2, fanout=5, gather=True)
ref = O.bulk_shadow(g, roots, boff, seeds, rng=0, depth=2, fanout=5, gather=True)
sl = consumer.slice_components(S, 1, 7, 40)
want = CO.slice_components(CO.batch_of(ref, boff, 1, 6, 2), 7, 40)
plan = consumer.ScatterPlan(sl.e_col, sl.n_vertices)
ok = np.array_equal(sl.e_col.cpu().numpy(), want["e_col"])
ok &= np.array_equal(consumer.scatter_add(sl.edge_features, plan).cpu().numpy().view(np.uint64),
                     CO.scatter_add(want["ye"], want["e_col"], sl.n_vertices).view(np.uint64))
ok &= np.array_equal(consumer.gather_rows(sl.node_features, sl.e_row).cpu().numpy().view(np.uint64),
                     CO.gather_rows(want["xv"], want["e_row"]).view(np.uint64))
parts = np.random.default_rng(1).standard_normal((3, 100))
ok &= np.array_equal(consumer.ordered_mean(torch.as_tensor(parts, device="cuda")).cpu().numpy().view(np.uint64),
                     CO.allreduce_mean(parts).view(np.uint64))
torch.cuda.synchronize()
plan.close()
S.close()
bad += not ok
print("consumer", "ok" if ok else "MISMATCH", flush=True)
xv, ye, lab = np.zeros(10 * 6), np.zeros(10 * 2), np.zeros(10, np.uint8)
out = hgs.lib().hgs_graph_gather(G._h, hgs._p(np.arange(10, dtype=np.int64)), 10,
                                 hgs._p(np.arange(10, dtype=np.int64)), 10, hgs._p(xv), hgs._p(ye), hgs._p(lab))
print("gather rc", out, flush=True)
print("SANITIZE CASE", "FAIL" if bad or out else "OK")
sys.exit(1 if bad or out else 0)
