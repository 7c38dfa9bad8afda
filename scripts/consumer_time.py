"""Per-op wall times of the consumer on C2 batches (sync after each op).
usage: python scripts/consumer_time.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2504_04670_b200 import hgs, workload as W, consumer as C
ev = W.preset_event("C2")
G = hgs.Graph(ev.rp, ev.ci).attach_features(ev.node_feat, ev.edge_feat, ev.labels)
side = torch.cuda.Stream()  # the sampler on its own (non-blocking) torch stream, as in bench.py
S = hgs.Sampler(G, stream=side.cuda_stream)
roots, boff, seeds = W.bench_roots(ev.n, 1024, 64, seed=1, rep=0)
S.bulk_shadow(roots, boff, seeds, depth=3, fanout=6, gather=True)
acc = {}
def t(name, f):
    torch.cuda.synchronize(); a = time.perf_counter(); r = f(); torch.cuda.synchronize()
    acc[name] = acc.get(name, 0.0) + time.perf_counter() - a
    return r
for it in range(2):
    acc.clear()
    for b in range(16):
        sl = t("slice", lambda: C.slice_components(S, b, 0, S.batch_components(b)))
        pr = t("plan rows", lambda: C.ScatterPlan(sl.e_row, sl.n_vertices))
        pc = t("plan cols", lambda: C.ScatterPlan(sl.e_col, sl.n_vertices))
        t("gather x rows", lambda: C.gather_rows_planned(sl.node_features, pr))
        t("gather x cols", lambda: C.gather_rows_planned(sl.node_features, pc))
        t("scatter y rows", lambda: C.scatter_add(sl.edge_features, pr))
        t("scatter y cols", lambda: C.scatter_add(sl.edge_features, pc))
        t("close", lambda: (pr.close(), pc.close()))
print({k: round(v / 16 * 1e3, 3) for k, v in acc.items()}, "ms per minibatch")
