#!/usr/bin/env python
"""bench.py — bulk ShaDow sampling throughput on B200 (BASELINE.json metric).

One step = one bulk_shadow + gather_features call (the trainer's `sample_s`
region, reference trainer.cpp:456-459) over k=64 minibatches x 1024 roots of
the synthetic TrackML-shaped event C2 (n=120,373 hits, m=1,509,282 edges),
depth 3, fanout 6, symmetrized walk, per-root xoshiro streams
(PerRootChoiceSource) — BASELINE.json configs[1]. Roots and seeds follow the
reference's `bench-sampling` protocol (cli.cpp:381-408) with rep = step index.

  value  device-resident throughput: inputs already in HBM, CUDA events on the
         launching stream around each step, L2 flushed (512 MiB memset)
         before every timed step; minibatches/s over all ranks (max rank time).
  e2e    the same metric through the C ABI with host buffers: pinned H2D of
         roots/offsets/seeds, the call, and D2H of every output array the
         reference API returns (vertex maps, edges, edge ids, gathered node/edge
         features, labels), wall-clocked.
  roofline  of the dominant kernel (k_extract): algorithmic bytes per launch
         (SURVEY.md §8(d) model) / its CUDA-event duration.
  cpu_baseline  the reference CPU sampler (oracle/_ref: the unmodified
         reference sources built by oracle/Makefile) on a bounded sample, all
         host threads, batch-sharded.

Multi-GPU (torchrun): weak scaling — every rank samples its own 64 batches
(rep offset by rank); no collective on the data path; timing = max over ranks.
`--impl reference` times the reference CPU sampler instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sampled minibatches/sec (and edges/sec) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "minibatches/s"
K_BATCHES, BATCH, DEPTH, FANOUT = 64, 1024, 3, 6
RNG = 0  # 0: per-root xoshiro streams (the reference's PerRootChoiceSource), 1: Philox
WORKLOAD = "C2"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


WORKLOAD_TEXT = {
    "C1": "C1: synthetic 10k-hit event (reference CPU-runnable case)",
    "C2": "C2: synthetic TrackML-shaped event",
    "C3": "C3: C2's event, 512 minibatches per step (trainer root/seed streams over consecutive epochs)"
          " sharded over the GPUs",
    "C4": "C4: high-pileup synthetic event (windowed generator)",
    "C5": "C5: multi-event epoch, C2-shaped events resident in HBM, every minibatch of one epoch"
          " (trainer root/seed streams, device-derived seeds)",
}


def set_workload(name, world):
    """BASELINE.json configs: C2 (default, weak scaling: 64 minibatches per
    GPU), C3 (512 minibatches per step split over the GPUs: strong scaling),
    C1 / C4 (4096-root minibatches on a ~1M-hit event), per GPU."""
    global WORKLOAD, K_BATCHES, BATCH, DEPTH, FANOUT
    from paper_2504_04670_b200 import workload as W
    WORKLOAD = name
    K_BATCHES, BATCH, DEPTH, FANOUT = W.SHAPE[name]
    if name == "C3":
        K_BATCHES = max(1, K_BATCHES // world)
    if name == "C5":
        K_BATCHES, BATCH, DEPTH, FANOUT = W.SHAPE["C2"]


RNG_TEXT = {0: "per-root xoshiro streams", 1: "per-root Philox streams"}


def config_dict(n_gpus, ev):
    return {"workload": "%s, n=%d hits / m=%d edges, %d minibatches"
            " x %d seeds per GPU, %d-hop, fanout %d, symmetrized walk, %s,"
            " bulk_shadow+gather_features" % (WORKLOAD_TEXT[WORKLOAD], ev.n, ev.m, K_BATCHES, BATCH, DEPTH,
                                               FANOUT, RNG_TEXT[RNG]),
            "minibatches_per_step_per_gpu": K_BATCHES, "roots_per_minibatch": BATCH,
            "depth": DEPTH, "fanout": FANOUT, "parallelism": f"shard{n_gpus} (replicated graph)",
            "l2": "flushed (512 MiB memset) before every timed step"}


# ----------------------------------------------------------------------------
# clocks


class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.path = tempfile.mktemp(suffix=".csv")
        self.p = None

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.close()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------
# reference / CPU baseline


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_sample_time(ev, n_batches, threads, rep0=1000):
    """Reference bulk_shadow + gather_features (oracle/_ref) on n_batches of the
    workload, batch-sharded over `threads`. Falls back to the C restatement
    ("port") if the reference build is absent."""
    from oracle import oracle as O
    from paper_2504_04670_b200 import workload as W
    roots, boff, seeds = W.bench_roots(ev.n, BATCH, n_batches, seed=1, rep=rep0)
    g = O.Graph(n=ev.n, rp=ev.rp, ci=ev.ci, node_feat=ev.node_feat, edge_feat=ev.edge_feat,
                labels=ev.labels)
    if O.ref_available():
        t, V, E = O.ref_time_sample(g, roots, boff, seeds, rng=RNG, depth=DEPTH, fanout=FANOUT,
                                    threads=threads)
        return t, V, E, "reference"
    t, V, E = O.port_time_sample(g, roots, boff, seeds, rng=RNG, depth=DEPTH, fanout=FANOUT,
                                 threads=threads)
    return t, V, E, "port"


def run_reference(args, world, rank):
    if rank != 0:
        return
    from paper_2504_04670_b200 import workload as W
    ev = W.preset_event(WORKLOAD)
    threads = os.cpu_count() or 1
    # one step = the GPU arm's own call (K_BATCHES minibatches of BATCH roots),
    # as one bulk_shadow + gather_features over contiguous batch ranges on all
    # host threads (each thread one reference call: one symmetrize_pattern per
    # thread per step, sampler.cpp:129)
    nb = K_BATCHES
    times = []
    kind = None
    for i in range(args.warmup + args.steps):
        t, V, E, kind = cpu_sample_time(ev, nb, threads, rep0=2000 + i)
        if i >= args.warmup:
            times.append(t)
    total = sum(times)
    value = nb * len(times) / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
            "scaling": "strong" if WORKLOAD == "C3" else "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "impl": "reference", "config": config_dict(world, ev),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                             "sample": f"{nb} minibatches x {BATCH} roots of {WORKLOAD} per step (the GPU arm's "
                                       f"call), bulk_shadow+gather_features over contiguous batch ranges on "
                                       f"{threads} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# the GPU arm


def measure_ingest(ev, device) -> dict:
    """Event ingest (§8f #2): the event as a binary file (hgs_event_save),
    then hgs_graph_load (mmap, device-side narrowing / validation, features
    attached) + the walk build (K0), wall clock, page cache warm; the median
    of 3 loads."""
    import torch
    from paper_2504_04670_b200 import hgs
    path = os.path.join(tempfile.mkdtemp(prefix="hgs_ingest_"), "event.hgsev")
    hgs.save_event(path, ev.rp, ev.ci, node_feat=ev.node_feat, edge_feat=ev.edge_feat, labels=ev.labels)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G = hgs.Graph.load(path, device=device)
        G.info()  # builds the symmetrized walk (K0)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        G.close()
    size = os.path.getsize(path)
    os.remove(path)
    return {"ms_per_event": 1e3 * float(np.median(ts)), "file_bytes": size,
            "path": "hgs_event_save file -> hgs_graph_load (mmap, device narrowing/validation, features) + K0 walk"}


def measure_consumer(S, k: int) -> dict:
    """The training step's device-side use of the last call's batches
    (SURVEY §8f #3): per minibatch slice_components (the whole batch), scatter
    plans for the row and column lists, the four IGNN message-passing ops of
    ignn.cpp:158-164 on the gathered features (x by rows / cols, y into rows /
    cols), then the rank-ordered reduction of a gradient-sized buffer. Wall
    clock with a device sync; slices include their small host reads."""
    import torch
    from paper_2504_04670_b200 import consumer as C
    phase = {"slice": 0.0, "plans": 0.0, "ops": 0.0}

    def tick(name, t):
        torch.cuda.synchronize()
        now = time.perf_counter()
        phase[name] += now - t
        return now

    for b in range(min(k, 4)):  # warm-up (pool growth, first launches)
        sl = C.slice_components(S, b, 0, int(S.batch_components(b)))
        C.ScatterPlan(sl.e_col, sl.n_vertices).close()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nbytes = 0
    for b in range(k):
        ta = time.perf_counter()
        sl = C.slice_components(S, b, 0, int(S.batch_components(b)))
        ta = tick("slice", ta)
        prow, pcol = C.ScatterPlan(sl.e_row, sl.n_vertices), C.ScatterPlan(sl.e_col, sl.n_vertices)
        ta = tick("plans", ta)
        x, y = sl.node_features, sl.edge_features
        for t in (C.gather_rows_planned(x, prow), C.gather_rows_planned(x, pcol), C.scatter_add(y, prow),
                  C.scatter_add(y, pcol)):
            nbytes += 2 * t.numel() * 8
        tick("ops", ta)
        prow.close()
        pcol.close()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    parts = torch.randn(8, 1 << 20, dtype=torch.float64, device="cuda")
    C.ordered_mean(parts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        C.ordered_mean(parts)
    e1.record()
    torch.cuda.synchronize()
    om = e0.elapsed_time(e1) / 10
    return {"ms_per_minibatch": (t1 - t0) * 1e3 / k, "minibatches": k,
            "breakdown_ms_per_minibatch": {n: v * 1e3 / k for n, v in phase.items()},
            "gather_scatter_gbs": nbytes / (t1 - t0) / 1e9,
            "ordered_mean_8x1M_ms": om, "ordered_mean_gbs": 9 * (1 << 20) * 8 / (om / 1e3) / 1e9,
            "path": "consumer.slice_components + 2 ScatterPlans + gather_rows_planned(x, rows/cols) + scatter_add(y, rows/cols) "
                    "per minibatch of the last e2e call (wall, synchronised per phase, incl. plan builds and slice "
                    "host reads; after a 4-batch warm-up); "
                    "hgs_ordered_mean over 8 ranks x 1M doubles (CUDA events)"}


def distinct_devices(world, dev) -> int:
    """Number of distinct physical GPUs the ranks run on (device UUIDs). A
    multi-rank line is only printed when every rank has its own GPU; the
    HGS_FORCE_DEVICE test hook (several ranks on one GPU over gloo) reports
    the true device count and marks the line."""
    import torch
    uuid = str(torch.cuda.get_device_properties(dev).uuid)
    if world == 1:
        return 1
    import torch.distributed as dist
    allu = [None] * world
    dist.all_gather_object(allu, uuid)
    n = len(set(allu))
    if n < world and os.environ.get("HGS_FORCE_DEVICE") is None:
        raise SystemExit(f"bench: {world} ranks share {n} GPU(s); refusing to report a multi-GPU number")
    return n


def byte_model(st, f_v, f_e, gather=True):
    """Algorithmic bytes of one call (split per stage; see
    DESIGN.md): expand = roots + seeds + offsets + walk row_ptr pairs of the
    expanded rows + chosen walk col_idx; extract = A row_ptr pairs of the set
    vertices + scanned A col_idx; pack = the outputs (vtx, comp_off,
    roots_local, 3 x E edge arrays, batch offsets) + the feature/label gather
    (read + write). Scratch traffic (touched lists, edge slots) earns nothing."""
    R, k, V, E, S = st["R"], st["k"], st["V"], st["E"], st["S"]
    expand = 12 * R + 4 * (k + 1) + 8 * st["F_expand"] + 4 * st["F_children"]
    extract = 8 * V + 4 * S
    pack = 4 * V + 4 * (R + k) + 4 * R + 12 * E + 8 * (k + 1)
    if gather:
        pack += 16 * f_v * V + (16 * f_e + 2) * E
    return expand, extract, pack


def run_gpu(args, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2504_04670_b200 import hgs, workload as W

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n_dev = distinct_devices(world, dev)
    t0 = time.time()
    ev = W.preset_event(WORKLOAD)
    log(f"[rank {rank}] event n={ev.n} m={ev.m} generated in {time.time() - t0:.1f}s")
    G = hgs.Graph(ev.rp, ev.ci, device=local_rank).attach_features(ev.node_feat, ev.edge_feat,
                                                                    ev.labels)
    ingest = measure_ingest(ev, local_rank) if rank == 0 else None
    stream = torch.cuda.Stream(dev)  # a real (non-default) stream shared with the C ABI
    S = hgs.Sampler(G, stream=stream.cuda_stream)
    cfg = dict(depth=DEPTH, fanout=FANOUT, symmetrize=True, rng=RNG, gather=True,
               batch_size=BATCH, bulk_batches=K_BATCHES)
    nsteps = args.warmup + args.steps
    host_in, dev_in = [], []
    for i in range(nsteps):
        if WORKLOAD == "C3":  # the step's 512 trainer-order minibatches, this rank's slice
            total_k = W.SHAPE["C3"][0]
            roots, boff, seeds, _ = W.trainer_roots(ev.n, BATCH, total_k, seed=1, epoch0=8 * i)
            b0, b1 = rank * K_BATCHES, (rank + 1) * K_BATCHES
            r0, r1 = int(boff[b0]), int(boff[b1])
            roots, seeds, boff = roots[r0:r1], seeds[r0:r1], boff[b0:b1 + 1] - r0
        else:
            roots, boff, seeds = W.bench_roots(ev.n, BATCH, K_BATCHES, seed=1, rep=rank * nsteps + i)
        host_in.append((roots, boff, seeds))
        dev_in.append((torch.from_numpy(roots.astype(np.int32)).to(dev),
                       torch.from_numpy(boff).to(dev),
                       torch.from_numpy(seeds.view(np.int64)).to(dev)))
    with torch.cuda.stream(stream):
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step_device(i, profile):
        r, b, s = dev_in[i]
        S.run_device(r.data_ptr(), b.data_ptr(), r.numel(), b.numel() - 1, s.data_ptr(),
                     profile=profile, **cfg)

    for i in range(args.warmup):
        step_device(i, True)
        S.wait()

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    step_ms, wall_ms, kern, stats, launches = [], [], [], [], 0
    with Clocks(local_rank) as clk:
        for j in range(args.steps):
            i = args.warmup + j
            with torch.cuda.stream(stream):
                flush.zero_()
            if world > 1:  # every rank starts the step together; the wall clock runs to the last rank's end
                stream.synchronize()
                dist.barrier()
            tw = time.perf_counter()
            ev0[j].record(stream)
            step_device(i, False)
            ev1[j].record(stream)
            S.wait()
            if world > 1:
                dist.barrier()
            wall_ms.append(1e3 * (time.perf_counter() - tw))
            if S.reruns():  # a capacity re-run inside wait() would run outside ev0..ev1
                raise RuntimeError("bench: a timed step needed a capacity re-run; warm-up did not size the buffers")
            step_ms.append(ev0[j].elapsed_time(ev1[j]))
            launches += S.launches()
            stats.append(S.stats())
        torch.cuda.synchronize()
        # per-stage kernel times: the same steps again as profiled calls
        # (one serial chunk, CUDA events between the stages on the stream)
        for j in range(min(args.steps, 5)):
            with torch.cuda.stream(stream):
                flush.zero_()
            step_device(args.warmup + j, True)
            S.wait()
            kern.append(S.kernel_times())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # ---- e2e through the C ABI with host buffers (pinned)
        cap_v = int(max(s["V"] for s in stats) * 1.25) + 1024
        cap_e = int(max(s["E"] for s in stats) * 1.25) + 1024
        R = K_BATCHES * BATCH

        def pin(n, dt):
            return torch.empty(max(n, 1), dtype=dt, pin_memory=True).numpy()

        hout = dict(batch_voff=pin(K_BATCHES + 1, torch.int32), batch_eoff=pin(K_BATCHES + 1, torch.int32),
                    comp_off=pin(R + K_BATCHES, torch.int32), l2g=pin(cap_v, torch.int32),
                    roots_local=pin(R, torch.int32), e_row=pin(cap_e, torch.int32),
                    e_col=pin(cap_e, torch.int32), e_gid=pin(cap_e, torch.int32),
                    draws=pin(R, torch.int32).view(np.uint32),
                    decisions=pin(R, torch.int32).view(np.uint32),
                    xv=pin(cap_v * G.f_v, torch.float64), ye=pin(cap_e * G.f_e, torch.float64),
                    lab=pin(cap_e, torch.uint8))
        hin = []
        for (roots, boff, seeds) in host_in:
            pr, pb, ps = pin(len(roots), torch.int64), pin(len(boff), torch.int64), pin(len(seeds), torch.int64)
            pr[:] = roots
            pb[:] = boff
            ps[:] = seeds.view(np.int64)
            hin.append((pr, pb, ps.view(np.uint64)))
        e2e_s, h2d, d2h = [], 0, 0
        e2e_n = min(nsteps, args.e2e_steps)
        e2e_warm = args.warmup if e2e_n == nsteps else 1
        for i in range(e2e_n):
            pr, pb, ps = hin[i]
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            c = S.bulk_shadow(pr, pb, ps, **cfg)
            S.to_host(hout)
            t2 = time.perf_counter()
            if i >= e2e_warm:
                e2e_s.append(t2 - t1)
                h2d = pr.nbytes + pb.nbytes + ps.nbytes
                d2h = (4 * 2 * (c.k + 1) + 4 * (c.R + c.k) + 4 * c.V + 4 * c.R + 12 * c.E
                       + 8 * c.V * G.f_v + 8 * c.E * G.f_e + c.E + 8 * c.R)
    e2e_total = float(sum(e2e_s))
    if world > 1:  # per step: the slowest rank's device time; then the sum over steps
        t = torch.tensor(step_ms + [e2e_total], device=dev if dist.get_backend() == "nccl" else "cpu",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms, e2e_total = [float(x) for x in t[:-1]], float(t[-1])
    total_ms = float(sum(step_ms))
    # C++ drop-in end to end (rank 0, one GPU): std::vector<SampledBatch> out
    e2e_cpp = None
    if rank == 0 and not args.no_dropin_e2e and WORKLOAD in ("C1", "C2"):
        roots_h, boff_h, seeds_h = host_in[args.warmup]
        e2e_cpp = {}
        for mode, name in ((0, "device_event"), (1, "trainer_two_lines")):
            sec, V, E = W.dropin_time(ev, roots_h, boff_h, seeds_h, depth=DEPTH, fanout=FANOUT, mode=mode,
                                      warmup=1, reps=3)
            e2e_cpp[name] = {"value": K_BATCHES / float(np.mean(sec)), "unit": UNIT, "s_per_call": float(np.mean(sec)),
                             "V": V, "E": E}
        e2e_cpp["path"] = ("C++ drop-in, host int64 vectors in, std::vector<SampledBatch> with gathered fp64 "
                           "features out, wall clock: device_event = gpu::DeviceEvent::bulk_shadow(gather); "
                           "trainer_two_lines = hitgnn::bulk_shadow(edge-id A) + gather_features per batch "
                           "(trainer.cpp:457-458) through the resident-graph cache")
    consumer_leg = None
    if rank == 0 and world == 1 and WORKLOAD in ("C1", "C2") and cfg.get("gather"):
        consumer_leg = measure_consumer(S, K_BATCHES)
    if rank != 0:
        return
    mb = world * K_BATCHES * args.steps
    value = mb / (total_ms / 1e3)
    edges = sum(s["E"] for s in stats)
    kern = np.array(kern)
    kt_mean = kern.mean(axis=0)  # expand, extract, scan, pack, finalize, total
    bm = np.mean([byte_model(s, G.f_v, G.f_e, True) for s in stats], axis=0)
    b_exp, b_ext, b_pack = (float(x) for x in bm)
    bt = b_exp + b_ext + b_pack
    peak, peak_kind = peaks()
    stage_ms = {"expand": float(kt_mean[0]), "extract": float(kt_mean[1]), "scan": float(kt_mean[2]),
                "pack": float(kt_mean[3]), "finalize": float(kt_mean[4])}
    stage_bytes = {"expand": b_exp, "extract": b_ext, "pack": b_pack}
    top = max(("expand", "extract", "pack"), key=lambda n: stage_ms[n])
    ext_ms = stage_ms[top]
    bx = stage_bytes[top]
    achieved = bx / (ext_ms / 1e3) / 1e9
    call_gbs = bt / (float(np.mean(step_ms)) / 1e3) / 1e9
    prof = os.path.join(ROOT, "profiles", "extract_dram_bytes.json")
    traffic = None
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_dev, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if WORKLOAD == "C3" else "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": config_dict(world, ev),
        "edges_per_s": world * edges / (total_ms / 1e3),
        "roofline": {"bound": "hbm", "kernel": {"expand": "k_expand", "extract": "k_extract",
                                                "pack": "k_pack"}[top], "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "alg_bytes_per_launch": bx,
                     "kernel_ms": ext_ms,
                     "kernel_share_of_step": ext_ms / float(np.mean(step_ms)),
                     "call_alg_bytes": bt, "call_frac": call_gbs / peak,
                     "stage_ms": stage_ms, "stage_alg_bytes": stage_bytes,
                     "stage_frac": {n: stage_bytes[n] / (stage_ms[n] / 1e3) / 1e9 / peak
                                    for n in stage_bytes}},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": {"value": world * K_BATCHES * len(e2e_s) / e2e_total if e2e_total > 0 else None, "unit": UNIT,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "path": "hgs_sample_run (host int64 inputs, pinned) + hgs_sample_copy_to_host "
                        "(all outputs, pinned), wall clock"},
        "counts_per_step": {k: int(np.mean([s[k] for s in stats])) for k in ("V", "E", "S")},
        "timing": ("CUDA events on the sampling stream around each step, per step the max over ranks, summed"
                   + ("; wall_ms_per_step = barrier -> all ranks done" if world > 1 else "")),
    }
    if world > 1:
        line["wall_ms_per_step"] = float(np.mean(wall_ms))
        line["ranks"] = world
    if e2e_cpp:
        line["e2e_cpp"] = e2e_cpp
    if ingest:
        line["ingest"] = ingest
    if consumer_leg:
        line["consumer"] = consumer_leg
    if world == 1 and not args.no_cpu_baseline:
        # (i) all host threads on the call's own shape (K_BATCHES minibatches,
        # contiguous batch ranges per thread); (ii) one thread, the reference as
        # shipped (trainer.cpp:457 samples on the caller thread), on a
        # 2-minibatch sample
        threads = os.cpu_count() or 1
        nb = K_BATCHES
        t, V, E, kind = cpu_sample_time(ev, nb, threads)
        nb1 = 2
        t1, _, _, _ = cpu_sample_time(ev, nb1, 1, rep0=1500)
        line["cpu_baseline"] = {"value": nb / t, "unit": UNIT, "cores": threads, "kind": kind,
                                "cpu_model": cpu_model(),
                                "value_1thread": nb1 / t1,
                                "sample": f"{nb} minibatches x {BATCH} roots of {WORKLOAD} (the GPU call), "
                                          f"bulk_shadow+gather_features over contiguous batch ranges on "
                                          f"{threads} host threads ({t:.1f}s wall); 1-thread figure: {nb1} "
                                          f"minibatches on one thread ({t1:.1f}s)"}
    print(json.dumps(line), flush=True)


def run_epoch(args, world, rank, local_rank):
    """C5: this rank's share of the events (ordinals rank, rank+world, ...)
    resident on its GPU; one step = one full epoch of sampling over them
    (EpochSampler: host shuffles + int32 root uploads + device calls, all
    inside the timed region). Timed with CUDA events (max over ranks)."""
    import concurrent.futures as cf

    import torch
    import torch.distributed as dist
    from paper_2504_04670_b200 import epoch as EP, hgs, workload as W

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n_dev = distinct_devices(world, dev)
    mine = list(range(rank, args.events, world))
    t0 = time.time()
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        evs = list(ex.map(lambda e: W.generate_event(**W.GEN["C2"], event_id=e), mine))
    gen_s = time.time() - t0
    log(f"[rank {rank}] {len(evs)} events generated in {gen_s:.1f}s")
    torch.cuda.synchronize()
    t0 = time.time()
    graphs = [hgs.Graph(e.rp, e.ci, device=local_rank).attach_features(e.node_feat, e.edge_feat, e.labels)
              for e in evs]
    for g in graphs:
        g.info()  # walk build (K0) per event
    torch.cuda.synchronize()
    ingest_s = time.time() - t0
    n_v = sum(e.n for e in evs)
    del evs
    es = EP.EpochSampler(graphs, batch_size=BATCH, bulk_batches=args.bulk_batches, depth=DEPTH, fanout=FANOUT,
                         seed=1)
    for i in range(args.warmup):
        es.epoch(1000 + i, max_batches_per_event=es.k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms, tots = [], []
    with Clocks(local_rank) as clk:
        for j in range(args.steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in es.streams:
                s.wait_event(e0)
            tot = es.epoch(j)
            ends = []
            for s in es.streams:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(s)
                ends.append(e1)
            torch.cuda.synchronize()
            ms.append(max(e0.elapsed_time(e1) for e1 in ends))
            tots.append(tot)
    total_ms = float(sum(ms))
    mbs = sum(t["minibatches"] for t in tots)
    if world > 1:
        t = torch.tensor([total_ms, float(mbs)], device=dev if dist.get_backend() == "nccl" else "cpu",
                         dtype=torch.float64)
        dist.all_reduce(t[0:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:2], op=dist.ReduceOp.SUM)
        total_ms, mbs = float(t[0]), int(t[1])
    if rank != 0:
        return
    line = {"metric": METRIC, "value": mbs / (total_ms / 1e3), "unit": UNIT, "n_gpus": n_dev,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT["C5"] + f": {args.events} events (generate_event C2 preset,"
                                   f" event_id 0..{args.events - 1}), b={BATCH}, bulk_batches="
                                   f"{args.bulk_batches or 'all batches of the event'},"
                                   f" {DEPTH}-hop, fanout {FANOUT}, with gather",
                       "events": args.events, "events_per_gpu": len(graphs), "vertices_per_gpu": n_v,
                       "minibatches_per_epoch": mbs // args.steps, "parallelism": f"events split over {world} GPU(s)",
                       "setup_s": {"generate": round(gen_s, 2), "ingest_and_walk_build": round(ingest_s, 2)},
                       "l2": "not flushed (the epoch streams ~100 events, far beyond L2)"},
            "edges_per_s": world * sum(t["E"] for t in tots) / (total_ms / 1e3),
            "calls_per_epoch": tots[0]["calls"], "gpu_launches": None, "clocks": clk.summary(),
            "e2e": None}
    print(json.dumps(line), flush=True)
    es.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--events", type=int, default=100, help="C5: events in the epoch (split over ranks)")
    ap.add_argument("--rng", default="xoshiro", choices=["xoshiro", "philox"],
                    help="choice streams: per-root xoshiro (reference default) or counter-based Philox")
    ap.add_argument("--bulk-batches", type=int, default=0,
                    help="C5: minibatches per sampling call (0 = all batches of an event in one call)")
    ap.add_argument("--workload", default="C2", choices=["C1", "C2", "C3", "C4", "C5"],
                    help="BASELINE.json config (C2 = the headline line)")
    ap.add_argument("--no-dropin-e2e", action="store_true", help="skip the C++ drop-in e2e legs")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="steps of the host-buffer e2e leg (default: all; fewer for C3/C4)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: run several ranks on one GPU over gloo (exercises the
    # multi-rank timing / reduction path where only one GPU is available)
    backend = os.environ.get("HGS_DIST_BACKEND", "nccl")
    if os.environ.get("HGS_FORCE_DEVICE") is not None:
        local_rank = int(os.environ["HGS_FORCE_DEVICE"])
    set_workload(args.workload, world)
    global RNG
    RNG = 1 if args.rng == "philox" else 0
    if args.e2e_steps is None:
        args.e2e_steps = args.warmup + args.steps if args.workload in ("C1", "C2") else 3
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        if args.workload == "C5":
            run_epoch(args, world, rank, local_rank)
        else:
            run_gpu(args, world, rank, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
