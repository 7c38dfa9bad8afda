"""Python bindings (ctypes) of the C ABI in include/hgs.h.

Mirrors the reference's sampler API shape for use from Python harnesses
(tests, bench): a device-resident :class:`Graph` (one per event, the
reference's ``make_edge_id_matrix`` + features) and a reusable
:class:`Sampler` workspace whose :meth:`Sampler.bulk_shadow` is
``hitgnn::bulk_shadow`` (+ ``gather_features`` when ``gather=True``).

There is no CPU fallback: if ``lib/libhgs.so`` is missing or no CUDA device
is visible, every sampling call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HGS_LIB") or os.path.join(_PKG, "lib", "libhgs.so")

HGS_OK, HGS_EINVAL, HGS_ECUDA, HGS_ERANGE = 0, 1, 2, 3
RNG_XOSHIRO, RNG_PHILOX = 0, 1
FLAG_SEQ_WALK = 1

# Exported symbols declared in include/hgs.h (checked by tests/test_abi.py).
EXPORTS = [
    "hgs_last_error", "hgs_abi_version", "hgs_device_count", "hgs_graph_create",
    "hgs_graph_attach_features", "hgs_graph_info", "hgs_graph_walk", "hgs_graph_destroy",
    "hgs_graph_gather",
    "hgs_sample_create", "hgs_sample_destroy", "hgs_sample_run", "hgs_sample_run_device",
    "hgs_sample_wait", "hgs_sample_copy_to_host", "hgs_sample_device_views",
    "hgs_sample_kernel_times", "hgs_sample_stats", "hgs_sample_launches", "hgs_derive", "hgs_philox4x32_10",
    "hgs_sample_run_device_spec", "hgs_derive_seeds", "hgs_sample_bind", "hgs_sample_copy_frontiers",
    "hgs_sample_rows", "hgs_sample_reruns",
    "hgs_sample_slice", "hgs_gather_rows", "hgs_scatter_plan_create", "hgs_scatter_add",
    "hgs_scatter_plan_destroy", "hgs_ordered_mean", "hgs_gather_rows_planned", "hgs_sample_run_multi",
]


class SamplerError(ValueError):
    """std::invalid_argument of the reference (HGS_EINVAL)."""


class HgsRuntimeError(RuntimeError):
    """CUDA / runtime failure or implementation limit (HGS_ECUDA, HGS_ERANGE)."""


class Config(C.Structure):
    _fields_ = [("depth", C.c_int64), ("fanout", C.c_int64), ("batch_size", C.c_int64),
                ("bulk_batches", C.c_int64), ("symmetrize", C.c_int32), ("rng", C.c_int32),
                ("gather", C.c_int32), ("profile", C.c_int32), ("flags", C.c_int32)]


class HostOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("batch_voff", "batch_eoff", "comp_off", "l2g",
                                            "roots_local", "e_row", "e_col", "e_gid", "xv", "ye",
                                            "lab", "draws", "decisions")]


class DeviceViews(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("batch_voff", "batch_eoff", "comp_off", "l2g",
                                            "roots_local", "e_row", "e_col", "e_gid",
                                            "root_voff", "root_eoff", "xv", "ye", "lab", "draws",
                                            "decisions", "touched", "touched_count",
                                            "level_counts")] + [("touched_stride", C.c_int64)]


class SliceViews(C.Structure):
    """hgs_slice_views: one slice_components result (device pointers)."""
    _fields_ = [("n_vertices", C.c_int64), ("n_edges", C.c_int64), ("n_components", C.c_int64),
                ("f_v", C.c_int64), ("f_e", C.c_int64)] + \
               [(n, C.c_void_p) for n in ("e_row", "e_col", "comp_off", "roots_local", "l2g", "e_gid",
                                            "xv", "ye", "lab")]


class SeedSpec(C.Structure):
    """hgs_seed_spec: per-root seed = derive(seed, path + [batch_base + bi, pos])."""
    _fields_ = [("seed", C.c_uint64), ("path", C.c_uint64 * 6), ("path_len", C.c_int32),
                ("batch_base", C.c_int64)]

    @classmethod
    def make(cls, seed: int, path, batch_base: int = 0) -> "SeedSpec":
        path = [int(x) for x in path]
        if len(path) > 6:
            raise SamplerError("seed path longer than 6")
        arr = (C.c_uint64 * 6)(*(path + [0] * (6 - len(path))))
        return cls(seed, arr, len(path), batch_base)


# Stream prefixes of the reference: trainer root streams (trainer.cpp:22,
# 200-206: {kStreamSample, epoch, event}) and bench-sampling (cli.cpp:404-408).
STREAM_SAMPLE = 0x73616D706C
STREAM_BENCH = 0x7374726D


def trainer_seed_spec(seed: int, epoch: int, event_ordinal: int, batch_base: int = 0) -> SeedSpec:
    return SeedSpec.make(seed, [STREAM_SAMPLE, epoch, event_ordinal], batch_base)


def bench_seed_spec(seed: int, k: int, rep: int) -> SeedSpec:
    return SeedSpec.make(seed, [STREAM_BENCH, k, rep], 0)


def derive_seeds(spec: SeedSpec, batch_off) -> np.ndarray:
    """Host copy of the device-derived seeds (hgs_derive_seeds)."""
    b = np.ascontiguousarray(batch_off, np.int64)
    out = np.zeros(int(b[-1]) if len(b) else 0, np.uint64)
    _check(lib().hgs_derive_seeds(C.byref(spec), _p(b), len(b) - 1, _p(out)))
    return out


def sample_rows(row_ptr, col_idx, s: int, seeds, row_streams, *, values=None, rng=RNG_XOSHIRO,
                state=None, n_cols=None, device=0):
    """hitgnn::sample_rows on the device (hgs_sample_rows): per-row chosen
    columns as (offsets, cols) plus per-stream draws / decisions consumed."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx, np.int64)
    va = None if values is None else np.ascontiguousarray(values, np.float64)
    sd = np.ascontiguousarray(seeds, np.uint64)
    rs = np.ascontiguousarray(row_streams, np.int64)
    st = None if state is None else np.ascontiguousarray(state, np.uint64)
    n = len(rp) - 1
    off = np.zeros(n + 1, np.int64)
    deg = np.diff(rp)
    cols = np.zeros(max(int(np.minimum(deg, max(int(s), 0)).sum()), 1), np.int64)
    dr = np.zeros(max(len(sd), 1), np.uint32)
    dc = np.zeros(max(len(sd), 1), np.uint32)
    _check(lib().hgs_sample_rows(device, n, n if n_cols is None else n_cols, _p(rp), _p(ci), _p(va), int(s), rng,
                                 _p(sd), len(sd), _p(st), _p(rs), _p(off), _p(cols), _p(dr), _p(dc)))
    return off, cols[:off[-1]], dr[:len(sd)], dc[:len(sd)]


_lib_cache: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib_cache
    if _lib_cache is None:
        if not os.path.exists(LIB_PATH):
            raise HgsRuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2504_04670_b200.build` "
                "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        L.hgs_last_error.restype = C.c_char_p
        L.hgs_derive.restype = C.c_uint64
        L.hgs_derive.argtypes = [C.c_uint64, vp, i32]
        L.hgs_philox4x32_10.argtypes = [vp, vp, vp]
        L.hgs_device_count.argtypes = [C.POINTER(C.c_int)]
        L.hgs_graph_create.argtypes = [C.c_int, i64, i64, vp, vp, vp, C.POINTER(vp)]
        L.hgs_graph_attach_features.argtypes = [vp, vp, i64, vp, i64, vp]
        L.hgs_graph_info.argtypes = [vp, vp]
        L.hgs_graph_walk.argtypes = [vp, i32, vp, vp]
        L.hgs_graph_destroy.argtypes = [vp]
        L.hgs_graph_gather.argtypes = [vp, vp, i64, vp, i64, vp, vp, vp]
        L.hgs_sample_create.argtypes = [vp, vp, C.POINTER(vp)]
        L.hgs_sample_destroy.argtypes = [vp]
        L.hgs_sample_run.argtypes = [vp, C.POINTER(Config), vp, vp, i64, vp, vp]
        L.hgs_sample_run_device.argtypes = [vp, C.POINTER(Config), vp, vp, i64, i64, vp]
        L.hgs_sample_wait.argtypes = [vp, vp]
        L.hgs_sample_run_device_spec.argtypes = [vp, C.POINTER(Config), vp, vp, i64, i64, C.POINTER(SeedSpec)]
        L.hgs_derive_seeds.argtypes = [C.POINTER(SeedSpec), vp, i64, vp]
        L.hgs_sample_bind.argtypes = [vp, vp]
        L.hgs_sample_rows.argtypes = [C.c_int, i64, i64, vp, vp, vp, i64, i32, vp, i64, vp, vp, vp, vp, vp, vp]
        L.hgs_sample_copy_to_host.argtypes = [vp, C.POINTER(HostOut)]
        L.hgs_sample_device_views.argtypes = [vp, C.POINTER(DeviceViews)]
        L.hgs_sample_kernel_times.argtypes = [vp, vp]
        L.hgs_sample_launches.argtypes = [vp, vp]
        L.hgs_sample_reruns.argtypes = [vp, vp]
        L.hgs_sample_stats.argtypes = [vp, vp, i32]
        L.hgs_current_device.argtypes = [C.POINTER(C.c_int)]
        L.hgs_event_save.argtypes = [C.c_char_p, i64, i64, vp, vp, vp, vp, i64, vp, i64, vp]
        L.hgs_event_info.argtypes = [C.c_char_p, vp]
        L.hgs_graph_load.argtypes = [C.c_int, C.c_char_p, C.POINTER(vp)]
        L.hgs_sample_slice.argtypes = [vp, i64, i64, i64, C.POINTER(SliceViews)]
        L.hgs_gather_rows.argtypes = [vp, i64, i64, vp, i64, vp, vp]
        L.hgs_scatter_plan_create.argtypes = [C.c_int, vp, i64, i64, vp, C.POINTER(vp)]
        L.hgs_scatter_add.argtypes = [vp, vp, i64, vp, i32, vp]
        L.hgs_scatter_plan_destroy.argtypes = [vp]
        L.hgs_ordered_mean.argtypes = [vp, i32, i64, vp, vp]
        L.hgs_gather_rows_planned.argtypes = [vp, vp, i64, i64, vp, vp]
        L.hgs_sample_run_multi.argtypes = [vp, C.POINTER(Config), vp, i32, vp, vp, vp, i64, vp]
        _lib_cache = L
    return _lib_cache


def _check(rc: int) -> None:
    if rc == HGS_OK:
        return
    msg = lib().hgs_last_error().decode()
    if rc == HGS_EINVAL:
        raise SamplerError(msg)
    raise HgsRuntimeError(msg)


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def device_count() -> int:
    c = C.c_int(0)
    _check(lib().hgs_device_count(C.byref(c)))
    return c.value


def derive(seed: int, path) -> int:
    p = np.ascontiguousarray(path, dtype=np.uint64)
    return int(lib().hgs_derive(C.c_uint64(seed), _p(p), len(p)))


def derive_many(seed: int, prefix, n_batches: int, batch_size: int) -> np.ndarray:
    """Per-root seeds derive(seed, prefix + [bi, pos]) for the bench protocol
    (cli.cpp:401-408) and trainer streams (trainer.cpp:200-206)."""
    out = np.empty(n_batches * batch_size, np.uint64)
    pre = list(prefix)
    w = 0
    for bi in range(n_batches):
        for pos in range(batch_size):
            out[w] = derive(seed, pre + [bi, pos])
            w += 1
    return out


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().hgs_philox4x32_10(_p(c), _p(k), _p(o))
    return o


def save_event(path: str, row_ptr, col_idx, *, values=None, node_feat=None, edge_feat=None, labels=None,
               n_cols=None) -> None:
    """Binary event file (hgs_event_save): the ingest format hgs_graph_load /
    Graph.load read back with mmap (no CUDA needed to write it)."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx, np.int64)
    va = None if values is None else np.ascontiguousarray(values, np.float64)
    nf = None if node_feat is None else np.ascontiguousarray(node_feat, np.float64)
    ef = None if edge_feat is None else np.ascontiguousarray(edge_feat, np.float64)
    lb = None if labels is None else np.ascontiguousarray(labels, np.uint8)
    n = len(rp) - 1
    nnz = int(rp[-1]) if n >= 0 else 0
    f_v = 0 if nf is None else (nf.shape[1] if nf.ndim == 2 else nf.size // max(n, 1))
    f_e = 0 if ef is None else (ef.shape[1] if ef.ndim == 2 else ef.size // max(nnz, 1))
    # the C entry point reads exactly these extents from the pointers
    if n < 0 or ci.size < nnz or (va is not None and va.size < nnz) or (nf is not None and nf.size < n * f_v) \
            or (ef is not None and ef.size < nnz * f_e) or (lb is not None and lb.size < nnz):
        raise SamplerError("hgs_event_save: array shorter than row_ptr / feature widths require")
    _check(lib().hgs_event_save(os.fsencode(path), n, n if n_cols is None else int(n_cols), _p(rp), _p(ci), _p(va),
                                _p(nf), f_v, _p(ef), f_e, _p(lb)))


def event_info(path: str) -> dict:
    a = np.zeros(6, np.int64)
    _check(lib().hgs_event_info(os.fsencode(path), _p(a)))
    return dict(zip(["n_rows", "n_cols", "nnz", "f_v", "f_e", "flags"], (int(x) for x in a)))


class Graph:
    """Device-resident event graph (CSR A with edge ids; optional features)."""

    @classmethod
    def load(cls, path: str, device: int = 0) -> "Graph":
        """hgs_graph_load: an event file (save_event) mmapped and built on the
        device, features attached."""
        info = event_info(path)
        g = cls.__new__(cls)
        g.n, g.n_cols, g.nnz = info["n_rows"], info["n_cols"], info["nnz"]
        g.f_v, g.f_e = info["f_v"], info["f_e"]
        g.device = device
        g._h = C.c_void_p()
        _check(lib().hgs_graph_load(device, os.fsencode(path), C.byref(g._h)))
        return g

    def __init__(self, row_ptr, col_idx, values=None, n_cols=None, device=0):
        rp = np.ascontiguousarray(row_ptr, np.int64)
        ci = np.ascontiguousarray(col_idx, np.int64)
        va = None if values is None else np.ascontiguousarray(values, np.float64)
        self.n = len(rp) - 1
        self.n_cols = self.n if n_cols is None else int(n_cols)
        self.nnz = int(rp[-1])
        self.device = device
        self._h = C.c_void_p()
        _check(lib().hgs_graph_create(device, self.n, self.n_cols, _p(rp), _p(ci), _p(va),
                                      C.byref(self._h)))
        self.f_v = self.f_e = 0

    def attach_features(self, node_feat, edge_feat, labels):
        nf = np.ascontiguousarray(node_feat, np.float64)
        ef = np.ascontiguousarray(edge_feat, np.float64)
        lb = np.ascontiguousarray(labels, np.uint8)
        self.f_v = nf.shape[1] if nf.ndim == 2 else (nf.size // max(self.n, 1))
        self.f_e = ef.shape[1] if ef.ndim == 2 else (ef.size // max(self.nnz, 1))
        _check(lib().hgs_graph_attach_features(self._h, _p(nf), self.f_v, _p(ef), self.f_e,
                                               _p(lb)))
        return self

    def info(self) -> dict:
        a = np.zeros(8, np.int64)
        _check(lib().hgs_graph_info(self._h, _p(a)))
        keys = ["n_rows", "n_cols", "nnz", "walk_nnz", "max_walk_deg", "max_out_deg", "f_v", "f_e"]
        return dict(zip(keys, (int(x) for x in a)))

    def walk(self, symmetrize=True):
        info = self.info()
        nnz = info["walk_nnz"] if symmetrize else self.nnz
        rp = np.zeros(self.n + 1, np.int64)
        ci = np.zeros(max(nnz, 1), np.int64)
        _check(lib().hgs_graph_walk(self._h, int(symmetrize), _p(rp), _p(ci)))
        return rp, ci[:int(rp[-1])]

    def close(self):
        if self._h:
            lib().hgs_graph_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class SampleCounts:
    R: int
    k: int
    V: int
    E: int


class Sampler:
    """A reusable device workspace bound to one Graph and one CUDA stream."""

    def __init__(self, graph: Graph, stream: int | None = None):
        self.graph = graph
        self._h = C.c_void_p()
        _check(lib().hgs_sample_create(graph._h, C.c_void_p(stream) if stream else None,
                                       C.byref(self._h)))
        self.counts = SampleCounts(0, 0, 0, 0)
        self.gathered = False
        self._batch_off = None

    @staticmethod
    def config(depth=3, fanout=6, symmetrize=True, rng=RNG_XOSHIRO, gather=False, profile=False,
               batch_size=1, bulk_batches=1, seq_walk=False) -> Config:
        return Config(depth, fanout, batch_size, bulk_batches, int(symmetrize), int(rng),
                      int(gather), int(profile), FLAG_SEQ_WALK if seq_walk else 0)

    def bulk_shadow(self, roots, batch_off, seeds, *, state=None, **cfg) -> SampleCounts:
        """hitgnn::bulk_shadow (+ gather_features) from host arrays; blocks."""
        r = np.ascontiguousarray(roots, np.int64)
        b = np.ascontiguousarray(batch_off, np.int64)
        s = np.ascontiguousarray(seeds, np.uint64)
        st = None if state is None else np.ascontiguousarray(state, np.uint64)
        c = self.config(**cfg)
        _check(lib().hgs_sample_run(self._h, C.byref(c), _p(r), _p(b), len(b) - 1, _p(s), _p(st)))
        self.gathered = bool(c.gather)
        self._batch_off = b.copy()
        return self.wait()

    def bulk_shadow_multi(self, graphs, batch_event, roots, batch_off, seeds, **cfg) -> SampleCounts:
        """One call over batches of several resident events (hgs_sample_run_multi):
        batch b samples graphs[batch_event[b]]; batch_event non-decreasing."""
        hs = (C.c_void_p * len(graphs))(*[g._h.value for g in graphs])
        be = np.ascontiguousarray(batch_event, np.int32)
        r = np.ascontiguousarray(roots, np.int64)
        b = np.ascontiguousarray(batch_off, np.int64)
        s = np.ascontiguousarray(seeds, np.uint64)
        c = self.config(**cfg)
        _check(lib().hgs_sample_run_multi(self._h, C.byref(c), C.cast(hs, C.c_void_p), len(graphs), _p(be), _p(r),
                                          _p(b), len(b) - 1, _p(s)))
        self.gathered = bool(c.gather)
        self._batch_off = b.copy()
        return self.wait()

    def run_device(self, d_roots: int, d_batch_off: int, n_roots: int, n_batches: int,
                   d_seeds: int, **cfg) -> None:
        """Enqueue with device pointers (int32 roots, int64 batch_off, u64 seeds)."""
        self._batch_off = None
        c = self.config(**cfg)
        self.gathered = bool(c.gather)
        _check(lib().hgs_sample_run_device(self._h, C.byref(c), C.c_void_p(d_roots),
                                           C.c_void_p(d_batch_off), n_roots, n_batches,
                                           C.c_void_p(d_seeds)))

    def bind(self, graph: "Graph") -> None:
        """Re-bind this workspace to another graph on the same device."""
        _check(lib().hgs_sample_bind(self._h, graph._h))
        self.graph = graph

    def run_device_spec(self, d_roots: int, d_batch_off: int, n_roots: int, n_batches: int,
                        spec: SeedSpec, **cfg) -> None:
        """Enqueue with device roots/offsets; per-root seeds derived on the device."""
        self._batch_off = None
        c = self.config(**cfg)
        self.gathered = bool(c.gather)
        _check(lib().hgs_sample_run_device_spec(self._h, C.byref(c), C.c_void_p(d_roots),
                                                C.c_void_p(d_batch_off), n_roots, n_batches,
                                                C.byref(spec)))

    def wait(self) -> SampleCounts:
        a = np.zeros(4, np.int64)
        _check(lib().hgs_sample_wait(self._h, _p(a)))
        self.counts = SampleCounts(*(int(x) for x in a))
        return self.counts

    def alloc_host(self, pinned_alloc=None) -> dict:
        c = self.counts
        g = self.graph
        mk = pinned_alloc or (lambda n, dt: np.empty(n, dt))
        out = dict(batch_voff=mk(c.k + 1, np.int32), batch_eoff=mk(c.k + 1, np.int32),
                   comp_off=mk(c.R + c.k, np.int32), l2g=mk(c.V, np.int32),
                   roots_local=mk(c.R, np.int32), e_row=mk(c.E, np.int32),
                   e_col=mk(c.E, np.int32), e_gid=mk(c.E, np.int32),
                   draws=mk(c.R, np.uint32), decisions=mk(c.R, np.uint32))
        if self.gathered:
            out.update(xv=mk(c.V * g.f_v, np.float64), ye=mk(c.E * g.f_e, np.float64),
                       lab=mk(c.E, np.uint8))
        return out

    def to_host(self, out: dict | None = None) -> dict:
        out = out if out is not None else self.alloc_host()
        ho = HostOut(**{k: (v.ctypes.data if v is not None and v.size else None)
                        for k, v in out.items()})
        _check(lib().hgs_sample_copy_to_host(self._h, C.byref(ho)))
        return out

    def device_views(self) -> DeviceViews:
        v = DeviceViews()
        _check(lib().hgs_sample_device_views(self._h, C.byref(v)))
        return v

    def batch_components(self, batch: int) -> int:
        """Number of components (roots) of batch `batch` of the last host-input run."""
        if self._batch_off is None:
            raise SamplerError("batch_components: last run had device inputs (batch offsets not on the host)")
        return int(self._batch_off[batch + 1] - self._batch_off[batch])

    def slice(self, batch: int, begin: int, end: int) -> SliceViews:
        """slice_components (trainer.cpp:221-269) of batch `batch` of the last
        run on the device: see paper_2504_04670_b200.consumer."""
        v = SliceViews()
        _check(lib().hgs_sample_slice(self._h, batch, begin, end, C.byref(v)))
        return v

    def kernel_times(self) -> np.ndarray:
        ms = np.zeros(6, np.float32)
        _check(lib().hgs_sample_kernel_times(self._h, _p(ms)))
        return ms

    def stats(self) -> dict:
        a = np.zeros(32, np.int64)
        _check(lib().hgs_sample_stats(self._h, _p(a), 32))
        keys = ["R", "k", "V", "E", "S", "F_expand", "F_children", "decisions", "draws"]
        d = dict(zip(keys, (int(x) for x in a[:9])))
        d["F_levels"] = [int(x) for x in a[9:]]
        return d

    def reruns(self) -> int:
        """Capacity re-runs the last run needed (0 once buffers fit)."""
        n = np.zeros(1, np.int64)
        _check(lib().hgs_sample_reruns(self._h, _p(n)))
        return int(n[0])

    def launches(self) -> int:
        n = np.zeros(1, np.int64)
        _check(lib().hgs_sample_launches(self._h, _p(n)))
        return int(n[0])

    def close(self):
        if self._h:
            lib().hgs_sample_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
