import sys, time, numpy as np
sys.path.insert(0, '.')
from tests.helpers import random_graph, compare, O
from paper_2504_04670_b200 import hgs
print("devices", hgs.device_count())
for n, m, seed in [(50, 200, 1), (1000, 8000, 2), (20000, 200000, 3)]:
    g = random_graph(n, m, seed)
    G = hgs.Graph(g.rp, g.ci).attach_features(g.node_feat, g.edge_feat, g.labels)
    info = G.info()
    wrp, wci = G.walk(True)
    orp, oci = O.symmetrize(g)
    print(n, m, info, "walk ok", np.array_equal(wrp, orp) and np.array_equal(wci, oci))
    S = hgs.Sampler(G)
    k = 4; b = min(64, n // k)
    rng = np.random.default_rng(seed)
    roots = np.concatenate([rng.permutation(n)[:b] for _ in range(k)]).astype(np.int64)
    boff = np.arange(k + 1, dtype=np.int64) * b
    seeds = rng.integers(0, 2**63, k * b, dtype=np.uint64)
    for rngk in (0, 1):
        for sym in (True, False):
            for d in (1, 2, 3):
                t = time.time()
                S.bulk_shadow(roots, boff, seeds, depth=d, fanout=6, symmetrize=sym, rng=rngk, gather=True)
                dev = S.to_host()
                ref = O.bulk_shadow(g, roots, boff, seeds, rng=rngk, depth=d, fanout=6, symmetrize=sym, gather=True)
                bad = compare(dev, ref, gather=True)
                print(f"  rng={rngk} sym={sym} d={d} V={S.counts.V}/{ref.V} E={S.counts.E}/{ref.E} bad={bad}")
