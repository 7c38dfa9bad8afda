"""ctypes bindings to the TEST-ONLY checkers in oracle/.

* ``liboracle.so`` — the plain-C restatement (hgs_oracle.c) of the reference
  bulk ShaDow sampler; always buildable (gcc).
* ``_ref/libhitgnn_ref.so`` — the unmodified reference sources compiled in
  place from /root/reference by oracle/Makefile, plus ref_shim.cpp. Present
  in this container and on GPU boxes that received the built .so; absent
  otherwise (``ref_available()``).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module: it is the checker, never
the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhitgnn_ref.so")

RNG_XOSHIRO = 0
RNG_PHILOX = 1

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_vp = C.c_void_p

_libs: dict[str, C.CDLL] = {}


def build(ref: bool = True) -> None:
    """Build the checkers (the recipe is oracle/Makefile)."""
    targets = ["oracle"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")] + targets, check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_vp)


def _oracle() -> C.CDLL:
    if "oracle" not in _libs:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        lib = C.CDLL(ORACLE_SO)
        lib.or_splitmix64.restype = C.c_uint64
        lib.or_xoshiro_next.restype = C.c_uint64
        lib.or_xoshiro_bounded.restype = C.c_uint64
        lib.or_derive.restype = C.c_uint64
        lib.or_derive.argtypes = [C.c_uint64, _u64p, C.c_int]
        lib.or_choose_philox.restype = C.c_uint32
        lib.or_choose_philox.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, _u32p]
        lib.or_choose_xoshiro.restype = C.c_uint32
        lib.or_choose_xoshiro.argtypes = [_vp, C.c_uint32, C.c_uint32, _vp]
        lib.or_xoshiro_seed.argtypes = [_vp, C.c_uint64]
        lib.or_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        lib.or_epoch_root_batches.restype = C.c_int64
        lib.or_epoch_root_batches.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _i64p]
        lib.or_symmetrize.restype = C.c_int64
        lib.or_symmetrize.argtypes = [C.c_int64, _i64p, _i64p, _i64p, _i64p]
        lib.or_bulk_shadow.restype = _vp
        lib.or_bulk_shadow.argtypes = [C.c_int64, C.c_int64, _vp, _vp, _vp, _vp, _vp, C.c_int64,
                                       _vp, C.c_int, C.c_int64, C.c_int64, C.c_int, _vp, C.c_int64,
                                       _vp, C.c_int64, _vp, C.c_char_p, C.c_int]
        lib.or_bulk_shadow_ex.restype = _vp
        lib.or_bulk_shadow_ex.argtypes = [C.c_int64, C.c_int64, _vp, _vp, _vp, _vp, _vp, C.c_int64,
                                          _vp, _vp, C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                          _vp, C.c_int64, _vp, C.c_int64, _vp, C.c_char_p, C.c_int]
        lib.or_result_counts.argtypes = [_vp, _i64p]
        lib.or_result_touched_total.restype = C.c_int64
        lib.or_result_touched_total.argtypes = [_vp]
        lib.or_result_copy.argtypes = [_vp] + [_vp] * 16
        lib.or_result_free.argtypes = [_vp]
        _libs["oracle"] = lib
    return _libs["oracle"]


def _ref() -> C.CDLL:
    if "ref" not in _libs:
        if not ref_available():
            raise RuntimeError("oracle/_ref/libhitgnn_ref.so not built (reference sources absent)")
        lib = C.CDLL(REF_SO)
        lib.ref_rng_first.argtypes = [C.c_uint64, C.c_int64, _u64p]
        lib.ref_derive.restype = C.c_uint64
        lib.ref_derive.argtypes = [C.c_uint64, _u64p, C.c_int]
        lib.ref_bounded_seq.argtypes = [C.c_uint64, _u64p, C.c_int64, _u64p]
        lib.ref_choose_seq.restype = C.c_int64
        lib.ref_choose_seq.argtypes = [C.c_uint64, _u32p, _u32p, C.c_int64, _u32p]
        lib.ref_epoch_root_batches.restype = C.c_int64
        lib.ref_epoch_root_batches.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _i64p]
        lib.ref_symmetrize.restype = C.c_int64
        lib.ref_symmetrize.argtypes = [C.c_int64, _i64p, _i64p, _i64p, _i64p]
        lib.ref_generate_event.restype = _vp
        lib.ref_generate_event.argtypes = [C.c_int64] * 5 + [C.c_double, C.c_int64, C.c_int64,
                                                             C.c_uint64, C.c_uint64]
        lib.ref_event_sizes.argtypes = [_vp, _i64p]
        lib.ref_event_copy.argtypes = [_vp, _i64p, _i64p, _f64p, _f64p, _u8p]
        lib.ref_event_free.argtypes = [_vp]
        lib.ref_bulk_shadow.restype = _vp
        lib.ref_bulk_shadow.argtypes = [C.c_int64, C.c_int64, _vp, _vp, _vp, _vp, _vp, C.c_int64,
                                        _vp, C.c_int, C.c_int64, C.c_int64, C.c_int, _vp,
                                        C.c_int64, _vp, C.c_int64, _vp, C.c_int, C.c_char_p,
                                        C.c_int]
        lib.ref_result_counts.argtypes = [_vp, _i64p]
        lib.ref_result_copy.argtypes = [_vp] + [_vp] * 12
        lib.ref_result_level_size.restype = C.c_int64
        lib.ref_result_level_size.argtypes = [_vp, C.c_int64]
        lib.ref_result_level_copy.argtypes = [_vp, C.c_int64, _i64p]
        lib.ref_result_level_array.restype = C.c_int64
        lib.ref_result_level_array.argtypes = [_vp, C.c_int64, C.c_int, _vp]
        lib.ref_result_free.argtypes = [_vp]
        lib.ref_time_sample.restype = C.c_double
        lib.ref_time_sample.argtypes = [C.c_int64, _vp, _vp, _vp, C.c_int64, _vp, C.c_int64, _vp,
                                        _vp, _vp, C.c_int64, _vp, C.c_int, C.c_int64, C.c_int64,
                                        C.c_int, _i64p]
        _libs["ref"] = lib
    return _libs["ref"]


# --------------------------------------------------------------------------
# data containers


@dataclass
class Graph:
    """A directed graph in the reference's CSR layout (int64 Index)."""

    n: int
    rp: np.ndarray
    ci: np.ndarray
    values: np.ndarray | None = None
    node_feat: np.ndarray | None = None  # (n, f_v) float64
    edge_feat: np.ndarray | None = None  # (m, f_e) float64
    labels: np.ndarray | None = None  # (m,) uint8
    n_cols: int | None = None

    @property
    def m(self) -> int:
        return int(self.rp[-1])


@dataclass
class Sample:
    """Flat SampledBatch list (batch-local indices), the device output layout."""

    batch_voff: np.ndarray
    batch_eoff: np.ndarray
    comp_off: np.ndarray
    l2g: np.ndarray
    roots_local: np.ndarray
    e_row: np.ndarray
    e_col: np.ndarray
    e_gid: np.ndarray
    e_val: np.ndarray
    xv: np.ndarray | None = None
    ye: np.ndarray | None = None
    lab: np.ndarray | None = None
    draws: np.ndarray | None = None
    decisions: np.ndarray | None = None
    level_counts: np.ndarray | None = None
    touched: np.ndarray | None = None
    level_q: list = field(default_factory=list)
    levels: list = field(default_factory=list)  # ref mode 2: per level dict of Q/F/P arrays

    @property
    def V(self) -> int:
        return int(self.batch_voff[-1])

    @property
    def E(self) -> int:
        return int(self.batch_eoff[-1])


class SamplerError(ValueError):
    pass


# FrontierSet arrays per level (sampler.hpp:52-58), in shim/tools order
FRONTIER_ARRAYS = ["q_ci", "f_rp", "f_ci", "p_rp", "p_ci", "p_val"]


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def bulk_shadow(g: Graph, roots, batch_off, seeds, *, rng=RNG_XOSHIRO, depth=3, fanout=6,
                symmetrize=True, gather=False, impl="oracle", mode=0, state=None,
                seq_walk=False) -> Sample:
    """Run the checker. impl="oracle" (C restatement) or "ref" (reference).
    mode (ref only): 0 bulk_shadow, 1 per-batch shadow_reference, 2 bulk with
    a FrontierObserver capturing Q per level."""
    roots = _c(roots, np.int64)
    batch_off = _c(batch_off, np.int64)
    seeds = _c(seeds, np.uint64)
    rp, ci = _c(g.rp, np.int64), _c(g.ci, np.int64)
    vals = _c(g.values, np.float64)
    nf = _c(g.node_feat, np.float64) if gather else None
    ef = _c(g.edge_feat, np.float64) if gather else None
    lab = _c(g.labels, np.uint8) if gather else None
    f_v = 0 if nf is None else nf.shape[1]
    f_e = 0 if ef is None else ef.shape[1]
    k = len(batch_off) - 1
    n_cols = g.n if g.n_cols is None else g.n_cols
    err = C.create_string_buffer(512)
    if impl == "oracle":
        lib = _oracle()
        st = _c(state, np.uint64)
        h = lib.or_bulk_shadow_ex(g.n, n_cols, _ptr(rp), _ptr(ci), _ptr(vals), _ptr(roots),
                                  _ptr(batch_off), k, _ptr(seeds), _ptr(st), rng, depth, fanout,
                                  int(symmetrize), 1 if seq_walk else 0, _ptr(nf), f_v, _ptr(ef),
                                  f_e, _ptr(lab), err, 512)
        if not h:
            raise SamplerError(err.value.decode())
        cnt = np.zeros(8, np.int64)
        lib.or_result_counts(h, cnt)
        _, R, V, E = (int(x) for x in cnt[:4])
        T = lib.or_result_touched_total(h)
        s = _alloc(k, R, V, E, f_v, f_e, bool(cnt[6]))
        s.draws = np.zeros(R, np.int64)
        s.decisions = np.zeros(R, np.int64)
        s.level_counts = np.zeros(R * (depth + 1), np.int64)
        s.touched = np.zeros(T, np.int64)
        lib.or_result_copy(h, *[_ptr(x) for x in (s.batch_voff, s.batch_eoff, s.comp_off, s.l2g,
                                                   s.roots_local, s.e_row, s.e_col, s.e_gid,
                                                   s.e_val, s.xv, s.ye, s.lab, s.draws,
                                                   s.decisions, s.level_counts, s.touched)])
        s.level_counts = s.level_counts.reshape(R, depth + 1)
        lib.or_result_free(h)
        return s
    lib = _ref()
    h = lib.ref_bulk_shadow(g.n, n_cols, _ptr(rp), _ptr(ci), _ptr(vals), _ptr(roots),
                            _ptr(batch_off), k, _ptr(seeds), rng, depth, fanout, int(symmetrize),
                            _ptr(nf), f_v, _ptr(ef), f_e, _ptr(lab), mode, err, 512)
    if not h:
        raise SamplerError(err.value.decode())
    cnt = np.zeros(8, np.int64)
    lib.ref_result_counts(h, cnt)
    kk, R, V, E = (int(x) for x in cnt[:4])
    s = _alloc(kk, R, V, E, f_v, f_e, bool(cnt[6]))
    lib.ref_result_copy(h, *[_ptr(x) for x in (s.batch_voff, s.batch_eoff, s.comp_off, s.l2g,
                                                s.roots_local, s.e_row, s.e_col, s.e_gid,
                                                s.e_val, s.xv, s.ye, s.lab)])
    for lvl in range(int(cnt[7])):
        q = np.zeros(lib.ref_result_level_size(h, lvl), np.int64)
        lib.ref_result_level_copy(h, lvl, q)
        s.level_q.append(q)
        if mode == 2:
            d = {}
            for which, name in enumerate(FRONTIER_ARRAYS):
                n = lib.ref_result_level_array(h, lvl, which, None)
                a = np.zeros(n, np.float64 if which == 5 else np.int64)
                lib.ref_result_level_array(h, lvl, which, a.ctypes.data)
                d[name] = a
            s.levels.append(d)
    lib.ref_result_free(h)
    return s


def _alloc(k, R, V, E, f_v, f_e, gathered) -> Sample:
    z = lambda n, dt=np.int64: np.zeros(n, dt)  # noqa: E731
    return Sample(
        batch_voff=z(k + 1), batch_eoff=z(k + 1), comp_off=z(R + k), l2g=z(V),
        roots_local=z(R), e_row=z(E), e_col=z(E), e_gid=z(E), e_val=z(E, np.float64),
        xv=z(V * f_v, np.float64) if gathered else None,
        ye=z(E * f_e, np.float64) if gathered else None,
        lab=z(E, np.uint8) if gathered else None)


# --------------------------------------------------------------------------
# RNG helpers


class _Xo(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4)]


def sample_rows(rp, ci, s: int, seeds, row_streams=None, *, values=None, rng=RNG_XOSHIRO, state=None,
                current: int = 0):
    """sample_rows (sampler.cpp:64-86) over one ChoiceSource of per-root
    streams (PerRootChoiceSource / PhiloxChoiceSource): returns (per-row choice
    lists, per-stream draws-or-states, per-stream decisions)."""
    lib = _oracle()
    if s < 1:
        raise SamplerError("sample_rows: s must be >= 1")
    n_rows = len(rp) - 1
    if row_streams is not None and len(row_streams) != n_rows:
        raise SamplerError("sample_rows: row_streams length must equal row count")
    if values is not None and np.any(np.asarray(values) < 0.0):
        raise SamplerError("sample_rows: row with negative mass")
    ns = len(seeds)
    xs = []
    for i in range(ns):
        x = _Xo()
        if state is not None and rng == RNG_XOSHIRO:
            for w in range(4):
                x.s[w] = int(state[4 * i + w])
        else:
            lib.or_xoshiro_seed(C.byref(x), C.c_uint64(int(seeds[i])))
        xs.append(x)
    dec = [int(state[i]) if (state is not None and rng != RNG_XOSHIRO) else 0 for i in range(ns)]
    ndec = [0] * ns
    out = []
    buf = np.zeros(max(int(s), 1), np.uint32)
    for r in range(n_rows):
        b, e = int(rp[r]), int(rp[r + 1])
        if e == b:
            out.append([])
            continue
        if row_streams is not None:
            st = int(row_streams[r])
            if st < 0 or st >= ns:
                raise SamplerError("PerRootChoiceSource: root ordinal out of range" if rng == RNG_XOSHIRO
                                   else "PhiloxChoiceSource: root ordinal out of range")
            current = st
        if ns == 0:
            raise SamplerError("PerRootChoiceSource: no streams configured" if rng == RNG_XOSHIRO
                               else "PhiloxChoiceSource: no streams configured")
        k = min(int(s), e - b)
        if rng == RNG_XOSHIRO:
            got = lib.or_choose_xoshiro(C.byref(xs[current]), e - b, k, buf.ctypes.data)
        else:
            got = lib.or_choose_philox(C.c_uint64(int(seeds[current])), dec[current], e - b, k, buf)
            dec[current] += 1
        ndec[current] += 1
        out.append([int(ci[b + int(x)]) for x in buf[:got]])
    states = np.array([x.s[w] for x in xs for w in range(4)], np.uint64)
    return out, states, np.array(ndec, np.int64), current


def derive(seed: int, path, impl="oracle") -> int:
    p = np.ascontiguousarray(path, dtype=np.uint64)
    if impl == "oracle":
        return int(_oracle().or_derive(seed, p, len(p)))
    return int(_ref().ref_derive(seed, p, len(p)))


def philox(ctr, key) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    _oracle().or_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


def rng_first(seed: int, n: int) -> np.ndarray:
    """First n xoshiro256** outputs of Rng(seed), from the restatement."""
    lib = _oracle()

    class X(C.Structure):
        _fields_ = [("s", C.c_uint64 * 4)]

    st = X()
    lib.or_xoshiro_seed(C.byref(st), C.c_uint64(seed))
    lib.or_xoshiro_next.argtypes = [C.c_void_p]
    return np.array([lib.or_xoshiro_next(C.byref(st)) for _ in range(n)], np.uint64)


def epoch_root_batches(n: int, b: int, rng_seed: int, impl="oracle") -> list[np.ndarray]:
    perm = np.zeros(n, np.int64)
    if impl == "oracle":
        nb = _oracle().or_epoch_root_batches(n, b, rng_seed, perm)
        if n < b:
            return [perm]
        return [perm[i * b:(i + 1) * b].copy() for i in range(nb)]
    nb = _ref().ref_epoch_root_batches(n, b, rng_seed, perm)
    size = n if n < b else b
    return [perm[i * size:(i + 1) * size].copy() for i in range(nb)]


def symmetrize(g: Graph, impl="oracle"):
    rp = np.zeros(g.n + 1, np.int64)
    ci = np.zeros(2 * g.m + 1, np.int64)
    f = _oracle().or_symmetrize if impl == "oracle" else _ref().ref_symmetrize
    nnz = f(g.n, _c(g.rp, np.int64), _c(g.ci, np.int64), rp, ci)
    return rp, ci[:nnz].copy()


# --------------------------------------------------------------------------
# reference generator (only where the reference was compiled)


def ref_generate_event(n_tracks=1100, hits_min=7, hits_max=10, layers=12, noise=650,
                       false_factor=11.0, f_v=6, f_e=2, seed=1, event_id=0) -> Graph:
    lib = _ref()
    h = lib.ref_generate_event(n_tracks, hits_min, hits_max, layers, noise, false_factor, f_v,
                               f_e, seed, event_id)
    sz = np.zeros(4, np.int64)
    lib.ref_event_sizes(h, sz)
    n, m, fv, fe = (int(x) for x in sz)
    rp, ci = np.zeros(n + 1, np.int64), np.zeros(m, np.int64)
    nf, ef = np.zeros(n * fv, np.float64), np.zeros(m * fe, np.float64)
    lab = np.zeros(m, np.uint8)
    lib.ref_event_copy(h, rp, ci, nf, ef, lab)
    lib.ref_event_free(h)
    return Graph(n=n, rp=rp, ci=ci, node_feat=nf.reshape(n, fv), edge_feat=ef.reshape(m, fe),
                 labels=lab)


def ref_time_sample(g: Graph, roots, batch_off, seeds, *, rng=RNG_XOSHIRO, depth=3, fanout=6,
                    threads=1):
    """Wall seconds of reference bulk_shadow + gather_features, batch-sharded
    over `threads` host threads. Returns (seconds, V, E)."""
    lib = _ref()
    ve = np.zeros(2, np.int64)
    roots = _c(roots, np.int64)
    batch_off = _c(batch_off, np.int64)
    seeds = _c(seeds, np.uint64)
    nf = _c(g.node_feat, np.float64)
    ef = _c(g.edge_feat, np.float64)
    lab = _c(g.labels, np.uint8)
    rp, ci = _c(g.rp, np.int64), _c(g.ci, np.int64)
    t = lib.ref_time_sample(g.n, _ptr(rp), _ptr(ci), _ptr(nf), nf.shape[1], _ptr(ef),
                            ef.shape[1], _ptr(lab), _ptr(roots), _ptr(batch_off),
                            len(batch_off) - 1, _ptr(seeds), rng, depth, fanout, threads, ve)
    return t, int(ve[0]), int(ve[1])


def port_time_sample(g: Graph, roots, batch_off, seeds, *, rng=RNG_XOSHIRO, depth=3, fanout=6,
                     threads=1):
    """Wall seconds of the C restatement (bulk_shadow + gather) batch-sharded
    over `threads` Python threads (ctypes releases the GIL). (seconds, V, E)"""
    import time
    from concurrent.futures import ThreadPoolExecutor

    roots = np.asarray(roots, np.int64)
    batch_off = np.asarray(batch_off, np.int64)
    seeds = np.asarray(seeds, np.uint64)
    k = len(batch_off) - 1
    threads = max(1, min(threads, k))

    def work(t):
        b0, b1 = k * t // threads, k * (t + 1) // threads
        if b1 <= b0:
            return 0, 0
        r0, r1 = batch_off[b0], batch_off[b1]
        s = bulk_shadow(g, roots[r0:r1], batch_off[b0:b1 + 1] - r0, seeds[r0:r1], rng=rng,
                        depth=depth, fanout=fanout, gather=True)
        return s.V, s.E

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(work, range(threads)))
    return time.perf_counter() - t0, sum(r[0] for r in res), sum(r[1] for r in res)
