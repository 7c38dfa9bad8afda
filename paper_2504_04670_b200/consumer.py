"""The training step's device-side use of a sampled batch.

Host mirror of the reference consumer interface over the C ABI
(include/hgs.h, "consumer" section), on device-resident torch tensors:

  slice_components(sampler, batch, begin, end)
      trainer.cpp:221-269 — the components [begin, end) of one batch of the
      last run, as device tensors (COO rebased to the slice, component offsets,
      roots_local; l2g / features / labels / edge ids are views of the run).
  gather_rows(x, idx) / scatter_add(y, plan, ...)
      Tape::gather_rows / scatter_add (autodiff.cpp:121-157) as used by the
      IGNN message passing (ignn.cpp:158-164), bit-identical in fp64 (sums in
      index order, no floating-point atomics). GatherRows / ScatterAdd wrap
      them as torch autograd functions whose backward passes are each other
      (autodiff.cpp:260-281).
  allreduce_coalesced(flat_grads, group)
      trainer.cpp:155-157 -> InMemoryComm::allreduce_mean (trainer.cpp:84-123):
      one collective over the flat gradient buffer: every rank's chunk
      [n*r/w, n*(r+1)/w) goes to rank r (NCCL all-to-all), rank r adds the
      ranks' values in rank order and scales by 1/w (hgs_ordered_mean), and the
      reduced chunks go back to every rank (NCCL all-gather) — the reference's
      reduce-scatter + all-gather, bit-identical to it for any world size.

There is no CPU path: the ops raise if the CUDA library is missing or a
tensor is not on a CUDA device (tests inject the oracle's reducer explicitly
to exercise the collective plumbing over gloo on CPU).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import hgs


def _stream(t: torch.Tensor) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _need_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if not t.is_cuda:
            raise hgs.HgsRuntimeError("consumer ops run on CUDA tensors only (no CPU path)")


class _Cai:
    """A device pointer exposed through __cuda_array_interface__ (zero copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr or 0, False),
                                         "version": 3, "strides": None}


def _view(ptr, shape, dtype: torch.dtype, device) -> torch.Tensor | None:
    if not ptr:
        return None if any(shape) else torch.empty(shape, dtype=dtype, device=device)
    ts = {torch.int32: "<i4", torch.float64: "<f8", torch.uint8: "|u1"}[dtype]
    return torch.as_tensor(_Cai(int(ptr), shape, ts), device=device)


@dataclass
class BatchSlice:
    """slice_components result (SampledBatch fields, trainer.cpp:227-268)."""

    e_row: torch.Tensor          # adjacency.entries[i].row, slice-local
    e_col: torch.Tensor          # adjacency.entries[i].col
    component_offsets: torch.Tensor
    roots_local: torch.Tensor
    local_to_global: torch.Tensor
    edge_global_ids: torch.Tensor
    node_features: torch.Tensor | None   # [V, f_v] (None without gather)
    edge_features: torch.Tensor | None   # [E, f_e]
    edge_labels: torch.Tensor | None     # [E]

    @property
    def n_vertices(self) -> int:
        return int(self.local_to_global.numel())

    @property
    def n_edges(self) -> int:
        return int(self.e_row.numel())


def slice_components(sampler: "hgs.Sampler", batch: int, begin: int, end: int) -> BatchSlice:
    """Components [begin, end) of batch `batch` of the sampler's last run
    (device tensors; the rebased arrays stay valid until the sampler's next
    slice or run, the views until its next run)."""
    v = sampler.slice(batch, begin, end)
    dev = torch.device("cuda", sampler.graph.device)
    nv, ne, nc = v.n_vertices, v.n_edges, v.n_components
    return BatchSlice(
        e_row=_view(v.e_row, (ne,), torch.int32, dev), e_col=_view(v.e_col, (ne,), torch.int32, dev),
        component_offsets=_view(v.comp_off, (nc + 1,), torch.int32, dev),
        roots_local=_view(v.roots_local, (nc,), torch.int32, dev),
        local_to_global=_view(v.l2g, (nv,), torch.int32, dev),
        edge_global_ids=_view(v.e_gid, (ne,), torch.int32, dev),
        node_features=_view(v.xv, (nv, v.f_v), torch.float64, dev) if v.xv else None,
        edge_features=_view(v.ye, (ne, v.f_e), torch.float64, dev) if v.ye else None,
        edge_labels=_view(v.lab, (ne,), torch.uint8, dev) if v.lab else None)


def gather_rows(x: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """out[i] = x[idx[i]] (Tape::gather_rows forward, autodiff.cpp:121-136)."""
    _need_cuda(x, idx)
    x = x.contiguous()
    idx = idx.to(torch.int32).contiguous()
    cols = x.shape[1] if x.dim() == 2 else 1
    out = torch.empty((idx.numel(), cols), dtype=torch.float64, device=x.device)
    hgs._check(hgs.lib().hgs_gather_rows(C.c_void_p(x.data_ptr()), x.shape[0], cols, C.c_void_p(idx.data_ptr()),
                                         idx.numel(), C.c_void_p(out.data_ptr()), _stream(x)))
    return out


class ScatterPlan:
    """Stable sort of an index list + per-destination segments (built once,
    used by scatter_add, by gather_rows_planned and by the backward passes).
    The indices are range-checked once here; a non-decreasing list (a batch's
    rows) needs no sort. Buffers are stream-ordered on the current stream."""

    def __init__(self, idx: torch.Tensor, n_rows: int):
        _need_cuda(idx)
        self.idx = idx.to(torch.int32).contiguous()
        self.n_rows = int(n_rows)
        self._h = C.c_void_p()
        hgs._check(hgs.lib().hgs_scatter_plan_create(self.idx.device.index or 0, C.c_void_p(self.idx.data_ptr()),
                                                     self.idx.numel(), self.n_rows, _stream(self.idx),
                                                     C.byref(self._h)))

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            hgs.lib().hgs_scatter_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gather_rows_planned(x: torch.Tensor, plan: ScatterPlan) -> torch.Tensor:
    """gather_rows(x, plan.idx) without a second range check or host sync
    (x must have plan.n_rows rows)."""
    _need_cuda(x)
    x = x.contiguous()
    cols = x.shape[1] if x.dim() == 2 else 1
    out = torch.empty((plan.idx.numel(), cols), dtype=torch.float64, device=x.device)
    hgs._check(hgs.lib().hgs_gather_rows_planned(plan._h, C.c_void_p(x.data_ptr()), x.shape[0], cols,
                                                 C.c_void_p(out.data_ptr()), _stream(x)))
    return out


def scatter_add(y: torch.Tensor, plan: ScatterPlan, out: torch.Tensor | None = None,
                accumulate: bool = False) -> torch.Tensor:
    """out[j] = sum over i ascending with idx[i] == j of y[i]
    (Tape::scatter_add, autodiff.cpp:138-157); accumulate=True adds onto
    `out` in the same order (gather_rows backward, autodiff.cpp:260-270)."""
    _need_cuda(y)
    y = y.contiguous()
    cols = y.shape[1] if y.dim() == 2 else 1
    if y.shape[0] != plan.idx.numel():
        raise hgs.SamplerError("scatter_add: index list length must equal row count")
    if out is None:
        out = torch.empty((plan.n_rows, cols), dtype=torch.float64, device=y.device)
        accumulate = False
    hgs._check(hgs.lib().hgs_scatter_add(plan._h, C.c_void_p(y.data_ptr()), cols, C.c_void_p(out.data_ptr()),
                                         1 if accumulate else 0, _stream(y)))
    return out


class GatherRows(torch.autograd.Function):
    """gather_rows with the reference's backward (scatter-add of the output
    gradient into the input's rows in index order)."""

    @staticmethod
    def forward(ctx, x, idx, plan):
        ctx.plan = plan
        return gather_rows_planned(x, plan) if plan.n_rows == x.shape[0] else gather_rows(x, idx)

    @staticmethod
    def backward(ctx, g):
        return scatter_add(g, ctx.plan), None, None


class ScatterAdd(torch.autograd.Function):
    """scatter_add with the reference's backward (gather of the output
    gradient's rows, autodiff.cpp:271-281)."""

    @staticmethod
    def forward(ctx, y, plan):
        ctx.plan = plan
        return scatter_add(y, plan)

    @staticmethod
    def backward(ctx, g):
        return gather_rows_planned(g, ctx.plan), None


def ordered_mean(parts: torch.Tensor) -> torch.Tensor:
    """parts[w, n] -> (parts[0] + ... + parts[w-1]) * (1/w), in rank order."""
    _need_cuda(parts)
    parts = parts.contiguous()
    w, n = parts.shape
    out = torch.empty(n, dtype=torch.float64, device=parts.device)
    hgs._check(hgs.lib().hgs_ordered_mean(C.c_void_p(parts.data_ptr()), w, n, C.c_void_p(out.data_ptr()),
                                          _stream(parts)))
    return out


def chunk_bounds(n: int, w: int) -> list[tuple[int, int]]:
    """Rank r's chunk of an n-element buffer: [n*r/w, n*(r+1)/w) (trainer.cpp:102-103)."""
    return [(n * r // w, n * (r + 1) // w) for r in range(w)]


def allreduce_coalesced(flat: torch.Tensor, group=None, reducer=ordered_mean) -> torch.Tensor:
    """In-place mean of `flat` over the process group, bit-identical with
    InMemoryComm::allreduce_mean (trainer.cpp:84-123): reduce-scatter with
    rank-ordered accumulation, then all-gather. One collective pair for the
    whole flat gradient buffer (allreduce_coalesced, trainer.cpp:155-157).
    `reducer` maps a [w, chunk] tensor to its rank-ordered mean (the CUDA
    kernel; tests substitute the oracle to drive the plumbing over gloo)."""
    import torch.distributed as dist

    w = dist.get_world_size(group)
    r = dist.get_rank(group)
    n = flat.numel()
    lens = torch.tensor([n], dtype=torch.int64, device=flat.device)
    all_lens = [torch.empty_like(lens) for _ in range(w)]
    dist.all_gather(all_lens, lens, group=group)
    if any(int(t.item()) != n for t in all_lens):
        raise hgs.SamplerError("allreduce: buffer lengths differ across ranks")
    if w == 1:
        flat.copy_(reducer(flat.reshape(1, n)))
        return flat
    bounds = chunk_bounds(n, w)
    lo, hi = bounds[r]
    # every rank's copy of chunk r, stacked in rank order
    recv = torch.empty((w, hi - lo), dtype=flat.dtype, device=flat.device)
    send_splits = [b - a for a, b in bounds]
    dist.all_to_all_single(recv.reshape(-1), flat.contiguous(), output_split_sizes=[hi - lo] * w,
                           input_split_sizes=send_splits, group=group)
    mine = reducer(recv)
    # reduced chunks back to every rank (padded to the largest chunk)
    cmax = max(send_splits)
    padded = torch.zeros(cmax, dtype=flat.dtype, device=flat.device)
    padded[:hi - lo] = mine
    gathered = torch.empty((w, cmax), dtype=flat.dtype, device=flat.device)
    dist.all_gather_into_tensor(gathered.reshape(-1), padded, group=group)
    for q, (a, b) in enumerate(bounds):
        flat[a:b] = gathered[q, :b - a]
    return flat
