import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2504_04670_b200 import hgs, workload as W
ev = W.preset_event("C1")
G = hgs.Graph(ev.rp, ev.ci).attach_features(ev.node_feat, ev.edge_feat, ev.labels)
st = torch.cuda.Stream()
S = hgs.Sampler(G, stream=st.cuda_stream)
roots, boff, seeds = W.bench_roots(ev.n, 256, 16, seed=1, rep=0)
dr = torch.from_numpy(roots.astype(np.int32)).cuda(); db = torch.from_numpy(boff).cuda(); ds = torch.from_numpy(seeds.view(np.int64)).cuda()
for i in range(5):
    with torch.cuda.stream(st):
        S.run_device(dr.data_ptr(), db.data_ptr(), dr.numel(), db.numel()-1, ds.data_ptr(), depth=2, fanout=6, gather=True, profile=True)
    S.wait()
print(os.environ.get("HGS_K2", "hash"), "C1 kernel ms (expand, extract, scan, pack, finalize, total):", np.round(S.kernel_times(), 4))
