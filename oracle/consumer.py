"""Consumer oracle — TEST INFRASTRUCTURE ONLY.

numpy restatements of what the reference trainer does with a sampled batch,
each following the cited reference lines, plus ctypes bindings of the
unmodified reference code (oracle/_ref/libhitgnn_ref_consumer.so, built by
oracle/Makefile from ref_consumer_shim.cpp) used to pin them:

  slice_components   trainer.cpp:221-269
  gather_rows        autodiff.cpp:121-136    backward :260-270
  scatter_add        autodiff.cpp:138-157    backward :271-281
  allreduce_mean     trainer.cpp:84-123 (allreduce_coalesced :155-157)

Only tests/ and the golden-fixture script import this module; the product
path (paper_2504_04670_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_CONSUMER_SO = os.path.join(HERE, "_ref", "libhitgnn_ref_consumer.so")


class ConsumerError(ValueError):
    """std::invalid_argument of the reference."""


# ---------------------------------------------------------------------------
# restatements


def slice_components(batch: dict, begin: int, end: int) -> dict:
    """trainer.cpp:221-269 over one batch given as a dict of arrays:
    comp_off[C+1], l2g[V], roots_local[C], e_row/e_col[E] (row-major,
    batch-local), e_gid[E], optional xv[V, f_v], ye[E, f_e], lab[E]."""
    comp = np.asarray(batch["comp_off"], np.int64)
    n_comp = len(comp) - 1
    if begin < 0 or end < begin or end > n_comp:  # trainer.cpp:223-224
        raise ConsumerError("slice_components: bad component range")
    v0, v1 = int(comp[begin]), int(comp[end])
    rows = np.asarray(batch["e_row"], np.int64)
    p0 = int(np.searchsorted(rows, v0, side="left"))  # lower_bound on row (:232-237)
    p1 = int(np.searchsorted(rows, v1, side="left"))
    out = {
        "comp_off": comp[begin:end + 1] - v0,
        "l2g": np.asarray(batch["l2g"], np.int64)[v0:v1],
        "roots_local": np.asarray(batch["roots_local"], np.int64)[begin:end] - v0,
        "e_row": rows[p0:p1] - v0,
        "e_col": np.asarray(batch["e_col"], np.int64)[p0:p1] - v0,
        "e_gid": np.asarray(batch["e_gid"], np.int64)[p0:p1],
    }
    for k, lo, hi in (("xv", v0, v1), ("ye", p0, p1), ("lab", p0, p1)):
        if batch.get(k) is not None:
            out[k] = np.asarray(batch[k])[lo:hi]
    return out


def batch_of(sample, batch_off, b: int, f_v: int = 0, f_e: int = 0) -> dict:
    """Batch b of a flat oracle Sample (oracle.py) as a slice_components input."""
    f = int(batch_off[b])
    nb = int(batch_off[b + 1]) - f
    v0, v1 = int(sample.batch_voff[b]), int(sample.batch_voff[b + 1])
    e0, e1 = int(sample.batch_eoff[b]), int(sample.batch_eoff[b + 1])
    d = {"comp_off": sample.comp_off[f + b:f + b + nb + 1], "l2g": sample.l2g[v0:v1],
         "roots_local": sample.roots_local[f:f + nb], "e_row": sample.e_row[e0:e1], "e_col": sample.e_col[e0:e1],
         "e_gid": sample.e_gid[e0:e1]}
    if sample.xv is not None:
        d["xv"] = sample.xv[v0 * f_v:v1 * f_v].reshape(-1, f_v)
        d["ye"] = sample.ye[e0 * f_e:e1 * f_e].reshape(-1, f_e)
        d["lab"] = sample.lab[e0:e1]
    return d


def gather_rows(x: np.ndarray, idx) -> np.ndarray:
    """out[i] = x[idx[i]] (autodiff.cpp:121-136)."""
    idx = np.asarray(idx, np.int64)
    for i in idx:
        if i < 0 or i >= x.shape[0]:
            raise ConsumerError(f"gather_rows: index {int(i)} out of range")
    return x[idx].copy()


def scatter_add(y: np.ndarray, idx, n_rows: int, out: np.ndarray | None = None) -> np.ndarray:
    """out[idx[i]] += y[i] for i ascending, from zeros or onto `out`
    (autodiff.cpp:138-157; the backward of gather_rows accumulates onto the
    gradient buffer the same way, :260-270). np.add.at is unbuffered and
    applies the additions in index order."""
    idx = np.asarray(idx, np.int64)
    if len(idx) != y.shape[0]:
        raise ConsumerError("scatter_add: index list length must equal row count")
    for i in idx:
        if i < 0 or i >= n_rows:
            raise ConsumerError(f"scatter_add: index {int(i)} out of range")
    res = np.zeros((n_rows, y.shape[1]), np.float64) if out is None else out.copy()
    np.add.at(res, idx, y)
    return res


def allreduce_mean(parts: np.ndarray) -> np.ndarray:
    """InMemoryComm::allreduce_mean (trainer.cpp:98-108): per element the
    ranks' values added in rank order, then times 1/w."""
    w = parts.shape[0]
    s = parts[0].astype(np.float64).copy()
    for q in range(1, w):
        s = s + parts[q]
    return s * (1.0 / float(w))


# ---------------------------------------------------------------------------
# the unmodified reference (where oracle/_ref was built)

_lib = None


def ref_available() -> bool:
    return os.path.exists(REF_CONSUMER_SO)


def _ref() -> C.CDLL:
    global _lib
    if _lib is None:
        L = C.CDLL(REF_CONSUMER_SO)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        L.refc_last_error.restype = C.c_char_p
        L.refc_slice.argtypes = [i64, i64, i64] + [vp] * 8 + [i64, vp, i64, vp, i64, i64, C.POINTER(vp)]
        L.refc_batch_sizes.argtypes = [vp, vp]
        L.refc_batch_copy.argtypes = [vp] * 11
        L.refc_batch_free.argtypes = [vp]
        L.refc_gather_rows.argtypes = [vp, i64, i64, vp, i64, vp]
        L.refc_scatter_add.argtypes = [vp, i64, i64, vp, i64, vp]
        L.refc_backward.argtypes = [i32, vp, i64, i64, vp, i64, i64, vp, vp, vp, vp]
        L.refc_allreduce.argtypes = [i32, vp, i64]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _rc(rc):
    if rc:
        raise ConsumerError(_ref().refc_last_error().decode())


def ref_slice_components(batch: dict, begin: int, end: int) -> dict:
    L = _ref()
    i64 = lambda a: np.ascontiguousarray(a, np.int64)  # noqa: E731
    comp, l2g, roots = i64(batch["comp_off"]), i64(batch["l2g"]), i64(batch["roots_local"])
    rows, cols, gid = i64(batch["e_row"]), i64(batch["e_col"]), i64(batch["e_gid"])
    val = np.ones(len(rows), np.float64)
    xv = batch.get("xv")
    ye = batch.get("ye")
    lab = batch.get("lab")
    f_v = xv.shape[1] if xv is not None else 0
    f_e = ye.shape[1] if ye is not None else 0
    xv = None if xv is None else np.ascontiguousarray(xv, np.float64)
    ye = None if ye is None else np.ascontiguousarray(ye, np.float64)
    lab = None if lab is None else np.ascontiguousarray(lab, np.uint8)
    h = C.c_void_p()
    _rc(L.refc_slice(len(l2g), len(rows), len(comp) - 1, _p(comp), _p(l2g), _p(roots), _p(rows), _p(cols), _p(val),
                     _p(gid), _p(xv), f_v, _p(ye), f_e, _p(lab), begin, end, C.byref(h)))
    try:
        s = np.zeros(5, np.int64)
        L.refc_batch_sizes(h, _p(s))
        nv, ne, nc = int(s[0]), int(s[1]), int(s[2])
        out = {"comp_off": np.zeros(nc + 1, np.int64), "l2g": np.zeros(nv, np.int64),
               "roots_local": np.zeros(nc, np.int64), "e_row": np.zeros(ne, np.int64),
               "e_col": np.zeros(ne, np.int64), "e_gid": np.zeros(ne, np.int64)}
        ev = np.zeros(ne, np.float64)
        if xv is not None:
            out["xv"] = np.zeros((nv, f_v), np.float64)
            out["ye"] = np.zeros((ne, f_e), np.float64)
            out["lab"] = np.zeros(ne, np.uint8)
        L.refc_batch_copy(h, _p(out["comp_off"]), _p(out["l2g"]), _p(out["roots_local"]), _p(out["e_row"]),
                          _p(out["e_col"]), _p(ev), _p(out["e_gid"]), _p(out.get("xv")), _p(out.get("ye")),
                          _p(out.get("lab")))
    finally:
        L.refc_batch_free(h)
    return out


def ref_gather_rows(x: np.ndarray, idx) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    idx = np.ascontiguousarray(idx, np.int64)
    out = np.zeros((len(idx), x.shape[1]), np.float64)
    _rc(_ref().refc_gather_rows(_p(x), x.shape[0], x.shape[1], _p(idx), len(idx), _p(out)))
    return out


def ref_scatter_add(y: np.ndarray, idx, n_rows: int) -> np.ndarray:
    y = np.ascontiguousarray(y, np.float64)
    idx = np.ascontiguousarray(idx, np.int64)
    out = np.zeros((n_rows, y.shape[1]), np.float64)
    _rc(_ref().refc_scatter_add(_p(y), y.shape[0], y.shape[1], _p(idx), n_rows, _p(out)))
    return out


def ref_backward(op: int, inp: np.ndarray, idx, n_rows: int, w: np.ndarray, labels: np.ndarray):
    """Gradients from the reference tape for gather_rows (op 0) or
    scatter_add (op 1) feeding linear(w) -> bce_with_logits(labels):
    returns (incoming gradient of the op's output, gradient of its input)."""
    inp = np.ascontiguousarray(inp, np.float64)
    idx = np.ascontiguousarray(idx, np.int64)
    w = np.ascontiguousarray(w, np.float64)
    labels = np.ascontiguousarray(labels, np.uint8)
    c = inp.shape[1]
    ro = len(idx) if op == 0 else n_rows
    g_out = np.zeros((ro, c), np.float64)
    g_in = np.zeros_like(inp)
    _rc(_ref().refc_backward(op, _p(inp), inp.shape[0], c, _p(idx), len(idx), n_rows, _p(w), _p(labels), _p(g_out),
                             _p(g_in)))
    return g_out, g_in


def ref_allreduce_mean(parts: np.ndarray) -> np.ndarray:
    """The reference's allreduce_coalesced on parts.shape[0] worker threads;
    returns rank 0's buffer (every rank's is the same)."""
    bufs = np.ascontiguousarray(parts, np.float64).copy()
    _rc(_ref().refc_allreduce(bufs.shape[0], _p(bufs), bufs.shape[1]))
    assert all(np.array_equal(bufs[0].view(np.uint64), b.view(np.uint64)) for b in bufs)
    return bufs[0]
