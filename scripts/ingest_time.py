"""Time event ingest: hgs_graph_create + attach_features + K0 (first call builds the walk)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2504_04670_b200 import hgs, workload as W
ev = W.preset_event(sys.argv[1] if len(sys.argv) > 1 else "C2")
for rep in range(3):
    t0 = time.perf_counter()
    G = hgs.Graph(ev.rp, ev.ci)
    t1 = time.perf_counter()
    G.attach_features(ev.node_feat, ev.edge_feat, ev.labels)
    t2 = time.perf_counter()
    G.walk(True)
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  features {1e3*(t2-t1):.1f} ms  walk(K0 + D2H) {1e3*(t3-t2):.1f} ms", flush=True)
    G.close()
import tempfile
path = os.path.join(tempfile.mkdtemp(prefix="hgs_ingest_"), "event.hgsev")
hgs.save_event(path, ev.rp, ev.ci, node_feat=ev.node_feat, edge_feat=ev.edge_feat, labels=ev.labels)
for rep in range(5):
    t0 = time.perf_counter()
    G = hgs.Graph.load(path)
    t1 = time.perf_counter()
    G.info()
    t2 = time.perf_counter()
    G.close()
    t3 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.1f} ms  walk {1e3*(t2-t1):.1f} ms  close {1e3*(t3-t2):.1f} ms", flush=True)
os.remove(path)
