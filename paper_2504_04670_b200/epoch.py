"""Epoch-level sampling over many device-resident events (BASELINE.json C5).

Restates the sampling side of ``Trainer::epoch_minibatch``
(reference trainer.cpp:433-459): for every training event, the epoch's root
batches come from ``epoch_root_batches(n, b, roots_rng(seed, epoch, event))``
(host, sequential Fisher-Yates, sampler.cpp:245-263), are split into chunks
of ``bulk_batches``, and every chunk is one ``bulk_shadow`` + ``gather_features``
call whose per-root streams are ``root_stream_seed(seed, epoch, event,
batch, pos)`` (trainer.cpp:200-206).

On the device the per-root seeds are derived inside K1 from a stream spec
(SURVEY.md §8f #1), so a chunk uploads only its int32 roots. Chunks rotate
over ``n_slots`` sample handles, each on its own stream, so the next chunk is
enqueued while the previous one finishes; the host shuffle of the next event
runs on a worker thread while the current event is sampled. Every event's
graph stays resident (one ``hgs.Graph`` per event).
"""
from __future__ import annotations

import concurrent.futures as cf
from dataclasses import dataclass

import numpy as np

from . import hgs
from . import workload as W


@dataclass
class Chunk:
    event_ordinal: int
    batch_base: int  # index of the chunk's first batch in the event's epoch
    n_batches: int
    sampler: hgs.Sampler
    counts: hgs.SampleCounts


class EpochSampler:
    def __init__(self, graphs: list[hgs.Graph], *, batch_size: int = 1024, bulk_batches: int = 64,
                 depth: int = 3, fanout: int = 6, seed: int = 1, gather: bool = True,
                 symmetrize: bool = True, rng: int = hgs.RNG_XOSHIRO, n_slots: int = 2):
        import torch

        if batch_size < 1 or bulk_batches < 0:
            raise hgs.SamplerError("SamplerConfig: batch_size must be >= 1 and bulk_batches >= 0")
        self.graphs = graphs
        # bulk_batches=0: every batch of an event in one call (the epoch's
        # minibatches bulk-sampled per event, BASELINE C5)
        if bulk_batches == 0:
            bulk_batches = max(g.n // batch_size + 1 for g in graphs)
        self.b, self.k = batch_size, bulk_batches
        self.seed = seed
        self.cfg = dict(depth=depth, fanout=fanout, symmetrize=symmetrize, rng=rng, gather=gather,
                        batch_size=batch_size, bulk_batches=bulk_batches)
        self._torch = torch
        self.streams = [torch.cuda.Stream() for _ in range(n_slots)]
        self.slots = [hgs.Sampler(graphs[0], stream=s.cuda_stream) for s in self.streams]
        self._slot_graph = [0] * n_slots
        # per-slot device roots / offsets and pinned staging
        cap = batch_size * bulk_batches
        self.d_roots = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(n_slots)]
        self.d_boff = [torch.empty(bulk_batches + 1, dtype=torch.int64, device="cuda") for _ in range(n_slots)]
        self.h_roots = [torch.empty(cap, dtype=torch.int32).pin_memory() for _ in range(n_slots)]
        self.h_boff = [torch.empty(bulk_batches + 1, dtype=torch.int64).pin_memory() for _ in range(n_slots)]
        # host shuffles of upcoming events run ahead on a few worker threads
        self.lookahead = 8
        self._pool = cf.ThreadPoolExecutor(max_workers=4)

    def _sampler_for(self, slot: int, ev: int) -> hgs.Sampler:
        if self._slot_graph[slot] != ev:  # keep the workspace, switch the event
            self.slots[slot].bind(self.graphs[ev])
            self._slot_graph[slot] = ev
        return self.slots[slot]

    def epoch(self, epoch: int, *, events=None, max_batches_per_event: int = 0, on_chunk=None) -> dict:
        """Sample every minibatch of the epoch. ``on_chunk(chunk)`` is called
        once a chunk's results are ready (device views valid until the slot is
        reused). Returns totals."""
        events = list(range(len(self.graphs))) if events is None else list(events)
        shuffle = lambda e: W.trainer_epoch_perm(self.graphs[e].n, self.b, self.seed, epoch, e)  # noqa: E731
        futs = [self._pool.submit(shuffle, e) for e in events[:self.lookahead]]
        pending: list[Chunk | None] = [None] * len(self.slots)
        tot = dict(minibatches=0, roots=0, V=0, E=0, calls=0)
        slot = 0

        def finish(s):
            ch = pending[s]
            if ch is None:
                return
            ch.counts = ch.sampler.wait()
            tot["V"] += ch.counts.V
            tot["E"] += ch.counts.E
            if on_chunk:
                on_chunk(ch)
            pending[s] = None

        for i, ev in enumerate(events):
            perm, nb, size = futs[i].result()
            futs[i] = None
            if i + self.lookahead < len(events):
                futs.append(self._pool.submit(shuffle, events[i + self.lookahead]))
            if max_batches_per_event > 0:
                nb = min(nb, max_batches_per_event)
            for b0 in range(0, nb, self.k):
                kc = min(self.k, nb - b0)
                R = kc * size
                finish(slot)
                S = self._sampler_for(slot, ev)
                hr, hb = self.h_roots[slot].numpy(), self.h_boff[slot].numpy()
                hr[:R] = perm[b0 * size:b0 * size + R]
                hb[:kc + 1] = np.arange(kc + 1, dtype=np.int64) * size
                st = self.streams[slot]
                with self._torch.cuda.stream(st):
                    self.d_roots[slot][:R].copy_(self.h_roots[slot][:R], non_blocking=True)
                    self.d_boff[slot][:kc + 1].copy_(self.h_boff[slot][:kc + 1], non_blocking=True)
                spec = hgs.trainer_seed_spec(self.seed, epoch, ev, batch_base=b0)
                S.run_device_spec(self.d_roots[slot].data_ptr(), self.d_boff[slot].data_ptr(), R, kc,
                                  spec, **self.cfg)
                pending[slot] = Chunk(ev, b0, kc, S, hgs.SampleCounts(R, kc, 0, 0))
                tot["minibatches"] += kc
                tot["roots"] += R
                tot["calls"] += 1
                slot = (slot + 1) % len(self.slots)
        for s in range(len(self.slots)):
            finish((slot + s) % len(self.slots))
        return tot

    def close(self):
        for S in self.slots:
            S.close()
        self._pool.shutdown(wait=False)
