"""Profiling driver: generate C2, run N bulk calls (device inputs) with per-kernel events.
usage: python scripts/prof.py [--calls N] [--no-gather] [--philox] [--k K]"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2504_04670_b200 import hgs, workload as W
ap = argparse.ArgumentParser()
ap.add_argument("--calls", type=int, default=3)
ap.add_argument("--no-gather", action="store_true")
ap.add_argument("--philox", action="store_true")
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--event", default="C2")
a = ap.parse_args()
ev = W.preset_event(a.event)
G = hgs.Graph(ev.rp, ev.ci).attach_features(ev.node_feat, ev.edge_feat, ev.labels)
st = torch.cuda.Stream()
S = hgs.Sampler(G, stream=st.cuda_stream)
roots, boff, seeds = W.bench_roots(ev.n, 1024, a.k, seed=1, rep=0)
dr = torch.from_numpy(roots.astype(np.int32)).cuda(); db = torch.from_numpy(boff).cuda(); ds = torch.from_numpy(seeds.view(np.int64)).cuda()
torch.cuda.synchronize()
for i in range(a.calls):
    with torch.cuda.stream(st):
        S.run_device(dr.data_ptr(), db.data_ptr(), dr.numel(), db.numel()-1, ds.data_ptr(), depth=3, fanout=6,
                     rng=1 if a.philox else 0, gather=not a.no_gather, profile=True)
    c = S.wait()
    print("call", i, c, "kernel ms (expand, extract, finalize, total):", S.kernel_times(), file=sys.stderr)
print(S.stats(), file=sys.stderr)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for i in range(a.calls + 2):
    with torch.cuda.stream(st):
        ev[0].record(st)
        S.run_device(dr.data_ptr(), db.data_ptr(), dr.numel(), db.numel()-1, ds.data_ptr(), depth=3, fanout=6,
                     rng=1 if a.philox else 0, gather=not a.no_gather, profile=False)
        ev[1].record(st)
    S.wait()
    ts.append(ev[0].elapsed_time(ev[1]))
print("unprofiled call ms:", " ".join(f"{t:.3f}" for t in ts), file=sys.stderr)
# calibration: write-only and copy streams on this box
buf = torch.empty(1 << 30, dtype=torch.uint8, device="cuda"); buf2 = torch.empty_like(buf)
for name, fn, nbytes in [("memset 1GiB", lambda: buf.zero_(), 1 << 30), ("copy 1GiB", lambda: buf2.copy_(buf), 2 << 30)]:
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(5)]; e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name}: {ms:.3f} ms = {nbytes / ms / 1e6:.0f} GB/s", file=sys.stderr)
