"""`hitgnn bench-sampling` (cli.cpp:340-445) through the C++ drop-in.

Same root sets and per-root streams as the reference command (workload.bench_roots:
epoch_root_batches under Rng(derive(seed, {'bench', k, rep})), seeds
derive(seed, {'strm', k, rep, bi, pos})), same legs (bulk: one bulk_shadow call
over k batches; sequential: k shadow_reference calls), same CSV columns and
number formats (bench_sampling.csv, cli.cpp:370-437). The event is a preset
(C1 / C2 shapes) instead of a dataset directory's largest event.

usage: python scripts/bench_sampling.py [--event C2] [--k 1 2 4 8] [--repeats 5]
                                        [--batch-size 256] [--seed 1] [--out DIR]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_04670_b200 import workload as W  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--event", default="C2")
    ap.add_argument("--k", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--batch-size", type=int, default=256)
    ap.add_argument("--depth", type=int, default=3)
    ap.add_argument("--fanout", type=int, default=6)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default="gpurun_out")
    args = ap.parse_args()
    if args.repeats < 1:
        raise SystemExit("bench-sampling: repeats must be >= 1")
    ev = W.preset_event(args.event)
    m = int(ev.rp[-1])
    os.makedirs(args.out, exist_ok=True)
    path = os.path.join(args.out, "bench_sampling.csv")
    with open(path, "w") as f:
        f.write("k,roots_per_batch,depth,fanout,event_vertices,event_edges,repeats,"
                "t_bulk_median_s,t_sequential_median_s,speedup\n")
        for k in args.k:
            if k < 1:
                raise SystemExit("bench-sampling: k must be >= 1")
            b = args.batch_size if k * args.batch_size <= ev.n else max(1, ev.n // k)
            t_bulk, t_seq = [], []
            for rep in range(args.repeats):
                roots, boff, seeds = W.bench_roots(ev.n, b, k, args.seed, rep)
                kw = dict(depth=args.depth, fanout=args.fanout, warmup=1, reps=1)
                t_bulk.append(W.dropin_time(ev, roots, boff, seeds, mode=2, **kw)[0][0])
                t_seq.append(W.dropin_time(ev, roots, boff, seeds, mode=3, **kw)[0][0])
            bulk, seq = float(np.median(t_bulk)), float(np.median(t_seq))
            line = (f"{k},{b},{args.depth},{args.fanout},{ev.n},{m},{args.repeats},"
                    f"{bulk:.6f},{seq:.6f},{seq / bulk:.4f}\n")
            f.write(line)
            print(line, end="", flush=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
