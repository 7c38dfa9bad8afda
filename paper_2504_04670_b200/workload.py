"""Synthetic TrackML-shaped workloads (BASELINE.json configs) for the bench
and the parity tests: the event generator (C++, libhitgnn_gpu.so), the
reference's bench-sampling root/seed protocol (cli.cpp:378-408) and the
trainer's seed streams (trainer.cpp:195-206)."""
from __future__ import annotations

import ctypes as C
import hashlib
import os
from dataclasses import dataclass

import numpy as np

from . import hgs

_PKG = os.path.dirname(os.path.abspath(__file__))
TOOLS_PATH = os.path.join(_PKG, "lib", "libhitgnn_gpu.so")

# GenConfig presets of SURVEY.md §8(d).
GEN = {
    "C1": dict(n_tracks=1100, hits_min=7, hits_max=10, layers=12, noise=650, false_factor=11.0,
               f_v=6, f_e=2, seed=1),
    "C2": dict(n_tracks=13000, hits_min=7, hits_max=10, layers=12, noise=10000,
               false_factor=14.5, f_v=6, f_e=2, seed=1),
    # C4 "high-pileup ~1M hits / ~15M edges": 8.5x C2's hits per layer. The
    # reference generator is quadratic in hits per layer (data.cpp:193-221);
    # this preset uses the windowed variant with C2's candidate density
    # (phi window scaled by the inverse hit density), so it is linear.
    "C4": dict(n_tracks=110000, hits_min=7, hits_max=10, layers=12, noise=85000,
               false_factor=17.5, f_v=6, f_e=2, seed=1, phi_window=0.45 * 23000 / 195000),
}
GEN["C3"] = GEN["C2"]
# sampler shapes: (batches k, roots per batch b, depth d, fanout s)
SHAPE = {"C1": (16, 256, 2, 6), "C2": (64, 1024, 3, 6), "C3": (512, 1024, 3, 6), "C4": (16, 4096, 3, 6),
         "C5": (64, 1024, 3, 6)}

_tools: C.CDLL | None = None


def tools() -> C.CDLL:
    global _tools
    if _tools is None:
        if not os.path.exists(TOOLS_PATH):
            raise hgs.HgsRuntimeError(f"{TOOLS_PATH} missing; run python -m paper_2504_04670_b200.build")
        hgs.lib()  # load libhgs first (libhitgnn_gpu depends on it)
        L = C.CDLL(TOOLS_PATH)
        vp = C.c_void_p
        L.hgs_generate_event.argtypes = [C.c_int64] * 5 + [C.c_double, C.c_int64, C.c_int64,
                                                           C.c_uint64, C.c_uint64, C.POINTER(vp)]
        L.hgs_generate_event_windowed.argtypes = [C.c_int64] * 5 + [C.c_double, C.c_int64, C.c_int64,
                                                                    C.c_uint64, C.c_uint64, C.c_double,
                                                                    C.POINTER(vp)]
        L.hgs_event_sizes.argtypes = [vp, vp]
        L.hgs_event_copy.argtypes = [vp] * 6
        L.hgs_event_free.argtypes = [vp]
        L.hgs_tools_last_error.restype = C.c_char_p
        L.hgs_epoch_root_batches.restype = C.c_int64
        L.hgs_epoch_root_batches.argtypes = [C.c_int64, C.c_int64, C.c_uint64, vp]
        L.hgs_derive_grid.argtypes = [C.c_uint64, vp, C.c_int32, C.c_int64, C.c_int64, vp]
        L.hgs_tools_frontiers.argtypes = [C.c_int64, C.c_int64, vp, vp, vp, vp, vp, C.c_int64, vp, C.c_int32,
                                          C.c_int64, C.c_int64, C.c_int32, C.POINTER(vp)]
        L.hgs_tools_frontiers_levels.restype = C.c_int64
        L.hgs_tools_frontiers_levels.argtypes = [vp]
        L.hgs_tools_frontier_array.restype = C.c_int64
        L.hgs_tools_frontier_array.argtypes = [vp, C.c_int64, C.c_int32, vp]
        L.hgs_tools_frontiers_free.argtypes = [vp]
        L.hgs_dropin_time.argtypes = [C.c_int64, vp, vp, vp, C.c_int64, vp, C.c_int64, vp, vp, vp, C.c_int64, vp,
                                      C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int32, vp, vp]
        _tools = L
    return _tools


@dataclass
class Event:
    n: int
    rp: np.ndarray  # int64 [n+1] (make_edge_id_matrix CSR)
    ci: np.ndarray  # int64 [m]
    node_feat: np.ndarray  # (n, f_v) f64
    edge_feat: np.ndarray  # (m, f_e) f64
    labels: np.ndarray  # (m,) u8

    @property
    def m(self) -> int:
        return int(self.rp[-1])


def generate_event(n_tracks=1100, hits_min=7, hits_max=10, layers=12, noise=650,
                   false_factor=11.0, f_v=6, f_e=2, seed=1, event_id=0, phi_window=0.45) -> Event:
    """generate_event (data.cpp:124-268); phi_window < 0.45 selects the
    scalable windowed variant (not in the reference)."""
    L = tools()
    h = C.c_void_p()
    if L.hgs_generate_event_windowed(n_tracks, hits_min, hits_max, layers, noise, false_factor, f_v, f_e,
                                     seed, event_id, phi_window, C.byref(h)) != 0:
        raise ValueError(L.hgs_tools_last_error().decode())
    sz = np.zeros(4, np.int64)
    L.hgs_event_sizes(h, sz.ctypes.data)
    n, m, fv, fe = (int(x) for x in sz)
    ev = Event(n=n, rp=np.zeros(n + 1, np.int64), ci=np.zeros(m, np.int64),
               node_feat=np.zeros((n, fv)), edge_feat=np.zeros((m, fe)),
               labels=np.zeros(m, np.uint8))
    L.hgs_event_copy(h, ev.rp.ctypes.data, ev.ci.ctypes.data, ev.node_feat.ctypes.data,
                     ev.edge_feat.ctypes.data, ev.labels.ctypes.data)
    L.hgs_event_free(h)
    return ev


FRONTIER_ARRAYS = ["q_ci", "f_rp", "f_ci", "p_rp", "p_ci", "p_val"]


def dropin_frontiers(rp, ci, values, roots, batch_off, seeds, *, rng=0, depth=3, fanout=6,
                     symmetrize=True, n_cols=None) -> list[dict]:
    """The C++ drop-in hitgnn::bulk_shadow (GPU) with a FrontierObserver: per
    level the FrontierSet's Q col_idx, F and P CSR arrays (sampler.hpp:52-58)."""
    L = tools()
    rp = np.ascontiguousarray(rp, np.int64)
    ci = np.ascontiguousarray(ci, np.int64)
    va = None if values is None else np.ascontiguousarray(values, np.float64)
    r = np.ascontiguousarray(roots, np.int64)
    b = np.ascontiguousarray(batch_off, np.int64)
    sd = np.ascontiguousarray(seeds, np.uint64)
    n = len(rp) - 1
    h = C.c_void_p()
    if L.hgs_tools_frontiers(n, n if n_cols is None else n_cols, rp.ctypes.data, ci.ctypes.data,
                             None if va is None else va.ctypes.data, r.ctypes.data, b.ctypes.data, len(b) - 1,
                             sd.ctypes.data, rng, depth, fanout, int(symmetrize), C.byref(h)) != 0:
        raise ValueError(L.hgs_tools_last_error().decode())
    out = []
    for lvl in range(L.hgs_tools_frontiers_levels(h)):
        d = {}
        for which, name in enumerate(FRONTIER_ARRAYS):
            m = L.hgs_tools_frontier_array(h, lvl, which, None)
            a = np.zeros(m, np.float64 if which == 5 else np.int64)
            L.hgs_tools_frontier_array(h, lvl, which, a.ctypes.data)
            d[name] = a
        out.append(d)
    L.hgs_tools_frontiers_free(h)
    return out


def save_event(path: str, ev: Event) -> None:
    """Binary event file (numpy .npz: make_edge_id_matrix CSR, features,
    labels) — the fast on-disk form of an EventGraph (§8f #2; the
    reference's JSON write_event, data.cpp:270-302, is its slow twin)."""
    np.savez(path, n=ev.n, rp=ev.rp, ci=ev.ci, nf=ev.node_feat, ef=ev.edge_feat, lab=ev.labels)


def load_event(path: str) -> Event:
    z = np.load(path)
    return Event(n=int(z["n"]), rp=z["rp"], ci=z["ci"], node_feat=z["nf"], edge_feat=z["ef"], labels=z["lab"])


def preset_event(name: str, event_id: int = 0) -> Event:
    """The preset's event. Large presets (C4: ~1-2 min to generate) are cached
    as .npz under $HGS_EVENT_CACHE (default /tmp/hgs_events): a convenience
    for repeated runs on one box, never needed for correctness or timing."""
    cfg = GEN[name]
    if cfg["n_tracks"] < 50000:
        return generate_event(**cfg, event_id=event_id)
    d = os.environ.get("HGS_EVENT_CACHE", "/tmp/hgs_events")
    key = "_".join(f"{k}{v}" for k, v in sorted(cfg.items())) + f"_e{event_id}"
    path = os.path.join(d, f"{name}_{hashlib.sha1(key.encode()).hexdigest()[:12]}.npz")
    if os.path.exists(path):
        return load_event(path)
    ev = generate_event(**cfg, event_id=event_id)
    try:
        os.makedirs(d, exist_ok=True)
        save_event(path + ".tmp.npz", ev)
        os.replace(path + ".tmp.npz", path)
    except OSError:
        pass
    return ev


def epoch_root_batches(n: int, b: int, rng_seed: int) -> list[np.ndarray]:
    """sampler.cpp:245-263 (host utility): Fisher-Yates with Rng(rng_seed)."""
    perm = np.zeros(n, np.int64)
    nb = int(tools().hgs_epoch_root_batches(n, b, rng_seed, perm.ctypes.data))
    size = n if n < b else b
    return [perm[i * size:(i + 1) * size] for i in range(nb)]


def epoch_root_perm(n: int, b: int, rng_seed: int) -> tuple[np.ndarray, int, int]:
    """epoch_root_batches as one contiguous int32 array: (perm, n_batches,
    batch size); batch i is perm[i*size:(i+1)*size]. The C shuffle runs
    without the GIL, so several events can be shuffled in parallel."""
    perm = np.zeros(n, np.int64)
    nb = int(tools().hgs_epoch_root_batches(n, b, rng_seed, perm.ctypes.data))
    size = n if n < b else b
    return perm[:nb * size].astype(np.int32), nb, size


def derive_grid(seed: int, prefix, k: int, b: int) -> np.ndarray:
    pre = np.ascontiguousarray(prefix, np.uint64)
    out = np.zeros(k * b, np.uint64)
    tools().hgs_derive_grid(seed, pre.ctypes.data, len(pre), k, b, out.ctypes.data)
    return out


STREAM_ROOTS, STREAM_SAMPLE = 0x726F6F7473, 0x73616D706C  # trainer.cpp:21-22


def trainer_epoch_batches(n: int, b: int, seed: int, epoch: int, event: int = 0):
    """Trainer::epoch_minibatch's roots for one (epoch, event) (trainer.cpp:433-437):
    epoch_root_batches(n, b, roots_rng(seed, epoch, event))."""
    return epoch_root_batches(n, b, hgs.derive(seed, [STREAM_ROOTS, epoch, event]))


def trainer_epoch_perm(n: int, b: int, seed: int, epoch: int, event: int = 0):
    """trainer_epoch_batches as (contiguous int32 perm, n_batches, size)."""
    return epoch_root_perm(n, b, hgs.derive(seed, [STREAM_ROOTS, epoch, event]))


def trainer_roots(n: int, b: int, k: int, seed: int = 1, epoch0: int = 0, event: int = 0):
    """k minibatches in the trainer's order over consecutive epochs epoch0,
    epoch0+1, ... of one event (C3: 512 minibatches of 1024 roots need ~5
    epochs of a 120k-hit event). Seeds are root_stream_seed(seed, epoch,
    event, batch, pos) (trainer.cpp:200-206). Returns roots, batch offsets,
    seeds and the (epoch, batch) of every minibatch."""
    roots, seeds, ids = [], [], []
    epoch = epoch0
    while len(ids) < k:
        batches = trainer_epoch_batches(n, b, seed, epoch, event)
        take = min(len(batches), k - len(ids))
        roots.extend(batches[:take])
        seeds.append(derive_grid(seed, [STREAM_SAMPLE, epoch, event], take, len(batches[0])))
        ids.extend((epoch, bi) for bi in range(take))
        epoch += 1
    boff = np.zeros(k + 1, np.int64)
    boff[1:] = np.cumsum([len(x) for x in roots])
    return np.concatenate(roots).astype(np.int64), boff, np.concatenate(seeds), ids


def bench_roots(n: int, b: int, k: int, seed: int = 1, rep: int = 0):
    """Roots, batch offsets and per-root seeds of `hitgnn bench-sampling`
    (cli.cpp:381-408): roots = epoch_root_batches(n, b,
    Rng(derive(seed,{'bench',k,rep}))) truncated to k; seeds
    derive(seed,{'strm',k,rep,bi,pos})."""
    if k * b > n:
        b = max(1, n // k)
    batches = epoch_root_batches(n, b, hgs.derive(seed, [0x62656E6368, k, rep]))
    if len(batches) < k:
        raise ValueError(f"event too small for k={k} batches of {b}")
    batches = batches[:k]
    roots = np.concatenate(batches).astype(np.int64)
    boff = np.arange(k + 1, dtype=np.int64) * b
    seeds = derive_grid(seed, [0x7374726D, k, rep], k, b)
    return roots, boff, seeds


def dropin_time(ev: Event, roots, batch_off, seeds, *, depth=3, fanout=6, mode=0, warmup=1, reps=3):
    """Wall-clock seconds per call of the C++ drop-in end to end (host arrays
    in, std::vector<SampledBatch> with gathered features out): mode 0 =
    gpu::DeviceEvent::bulk_shadow(gather), mode 1 = the reference trainer's two
    lines (bulk_shadow + gather_features per batch), mode 2 = bulk_shadow
    alone and mode 3 = one shadow_reference call per batch (the two legs of
    `hitgnn bench-sampling`). Returns (seconds, V, E)."""
    L = tools()
    r = np.ascontiguousarray(roots, np.int64)
    b = np.ascontiguousarray(batch_off, np.int64)
    sd = np.ascontiguousarray(seeds, np.uint64)
    nf = np.ascontiguousarray(ev.node_feat, np.float64)
    ef = np.ascontiguousarray(ev.edge_feat, np.float64)
    lab = np.ascontiguousarray(ev.labels, np.uint8)
    rp = np.ascontiguousarray(ev.rp, np.int64)
    ci = np.ascontiguousarray(ev.ci, np.int64)
    sec = np.zeros(reps, np.float64)
    ve = np.zeros(2, np.int64)
    if L.hgs_dropin_time(ev.n, rp.ctypes.data, ci.ctypes.data, nf.ctypes.data, nf.shape[1], ef.ctypes.data,
                         ef.shape[1], lab.ctypes.data, r.ctypes.data, b.ctypes.data, len(b) - 1, sd.ctypes.data,
                         depth, fanout, mode, warmup, reps, sec.ctypes.data, ve.ctypes.data) != 0:
        raise ValueError(L.hgs_tools_last_error().decode())
    return sec, int(ve[0]), int(ve[1])
