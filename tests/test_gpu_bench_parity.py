"""Parity at bench size for every BASELINE.json config (north_star: "bit-exact
subgraphs versus the CPU oracle"), through the C ABI on the GPU:

  C2  full call under both choice streams against the REFERENCE's own
      digests (tests/golden/c2.json, from oracle/_ref) and, for Philox,
      batch for batch against the oracle; the generator against the
      reference generator's digests.
  C3  one step = 512 trainer-order minibatches (trainer.cpp:433-459) in one
      call; 64 of them (8 runs of 8 spread over the step) against the oracle.
  C4  the ~1M-hit windowed event, 16 x 4096 roots, every batch against the
      oracle (no reference counterpart: the reference generator cannot build
      it).
  C5  an epoch over 3 resident C2-shaped events (device-derived trainer
      streams, one call per event), every minibatch against the per-event
      oracle.
plus a seeded slice of scripts/fuzz_gpu.py and the opt-in directory K2.

Per-root streams make any batch range of a call identical to a call over just
that range, so the oracle runs batch ranges on host threads
in parallel (tests/helpers.py: batch_slice, check_against_oracle_chunks).
"""
import os
import sys

import numpy as np
import pytest

from tests.helpers import O, check_against_oracle_chunks, even_chunks, load_json, random_graph, sha

pytestmark = pytest.mark.gpu

INT_FIELDS = ("batch_voff", "batch_eoff", "comp_off", "l2g", "roots_local", "e_row", "e_col", "e_gid")


def H():
    from paper_2504_04670_b200 import hgs
    return hgs


def W():
    from paper_2504_04670_b200 import workload
    return workload


def oracle_graph(ev):
    return O.Graph(n=ev.n, rp=ev.rp, ci=ev.ci, node_feat=ev.node_feat, edge_feat=ev.edge_feat, labels=ev.labels)


@pytest.fixture(scope="module")
def c2():
    ev = W().preset_event("C2")
    G = H().Graph(ev.rp, ev.ci).attach_features(ev.node_feat, ev.edge_feat, ev.labels)
    return ev, G


def test_c2_generator_matches_reference_digests(c2):
    ev, _ = c2
    ref = load_json("c2.json")["graph"]
    assert (ev.n, ev.m) == (ref["n"], ref["m"]) == (120373, 1509282)
    assert sha(ev.rp.astype(np.int64)) == ref["rp"]
    assert sha(ev.ci.astype(np.int64)) == ref["ci"]
    assert sha(ev.node_feat) == ref["node_feat"]
    assert sha(ev.edge_feat) == ref["edge_feat"]
    assert sha(ev.labels) == ref["labels"]


@pytest.mark.parametrize("rng", [0, 1])
def test_c2_full_call_matches_reference_digests(c2, rng):
    """The full bench call (64 x 1024 roots, d=3, s=6, gather) equals the
    reference bulk_shadow + gather_features output, digest for digest."""
    ev, G = c2
    gold = load_json("c2.json")
    run = next(r for r in gold["runs"] if r["rng"] == rng)
    roots, boff, seeds = W().bench_roots(ev.n, 1024, 64, seed=1, rep=0)
    assert sha(roots.astype(np.int64)) == gold["roots"] and sha(seeds) == gold["seeds"]
    S = H().Sampler(G)
    S.bulk_shadow(roots, boff, seeds, rng=rng, depth=3, fanout=6, gather=True)
    dev = S.to_host()
    assert (S.counts.V, S.counts.E) == (run["V"], run["E"])
    for f in INT_FIELDS:
        assert sha(np.asarray(dev[f]).astype(np.int64)) == run["digests"][f], f
    for f in ("xv", "ye", "lab"):
        assert sha(dev[f]) == run["digests"][f], f
    S.close()


def test_c2_philox_full_against_oracle(c2):
    ev, G = c2
    roots, boff, seeds = W().bench_roots(ev.n, 1024, 64, seed=1, rep=0)
    S = H().Sampler(G)
    S.bulk_shadow(roots, boff, seeds, rng=1, depth=3, fanout=6, gather=True)
    dev = S.to_host()
    bad = check_against_oracle_chunks(dev, oracle_graph(ev), roots, boff, seeds, even_chunks(64, 16),
                                      gather=True, f_v=6, f_e=2, rng=1, depth=3, fanout=6)
    assert not bad, bad
    S.close()


def test_c3_step_trainer_order(c2):
    """BASELINE configs[2]: 512 minibatches bulk-sampled in one call, roots and
    seeds in the trainer's order over consecutive epochs of the C2 event."""
    ev, G = c2
    roots, boff, seeds, ids = W().trainer_roots(ev.n, 1024, 512, seed=1, epoch0=0)
    assert len(ids) == 512 and ids[-1][0] >= 4  # spans five epochs of 117 minibatches
    S = H().Sampler(G)
    S.bulk_shadow(roots, boff, seeds, depth=3, fanout=6, gather=True)
    dev = S.to_host()
    bv = np.asarray(dev["batch_voff"]).astype(np.int64)
    assert bv[0] == 0 and np.all(np.diff(bv) > 0) and bv[-1] == S.counts.V
    chunks = [(64 * i, 64 * i + 8) for i in range(8)]
    bad = check_against_oracle_chunks(dev, oracle_graph(ev), roots, boff, seeds, chunks, gather=True,
                                      f_v=6, f_e=2, depth=3, fanout=6)
    assert not bad, bad
    S.close()


def test_c4_full_against_oracle():
    """BASELINE configs[3] shape: the ~1M-hit / ~15M-edge windowed event,
    16 minibatches x 4096 roots, d=3, every batch against the oracle."""
    ev = W().preset_event("C4")
    assert ev.n > 1_000_000 and ev.m > 14_000_000
    roots, boff, seeds = W().bench_roots(ev.n, 4096, 16, seed=1, rep=0)
    G = H().Graph(ev.rp, ev.ci).attach_features(ev.node_feat, ev.edge_feat, ev.labels)
    S = H().Sampler(G)
    S.bulk_shadow(roots, boff, seeds, depth=3, fanout=6, gather=True)
    dev = S.to_host()
    bad = check_against_oracle_chunks(dev, oracle_graph(ev), roots, boff, seeds, even_chunks(16, 16),
                                      gather=True, f_v=6, f_e=2, depth=3, fanout=6)
    assert not bad, bad
    S.close()
    G.close()


def test_c5_epoch_three_c2_events():
    """BASELINE configs[4] path: several C2-shaped events resident in HBM, every
    minibatch of epoch 0 (trainer order, device-derived root_stream_seed
    streams, trainer.cpp:195-206, 433-459), one call per event."""
    from paper_2504_04670_b200 import epoch as EP
    hg, w = H(), W()
    evs = [w.generate_event(**w.GEN["C2"], event_id=e) for e in range(3)]
    graphs = [hg.Graph(e.rp, e.ci).attach_features(e.node_feat, e.edge_feat, e.labels) for e in evs]
    es = EP.EpochSampler(graphs, batch_size=1024, bulk_batches=0, depth=3, fanout=6, seed=1, gather=True)
    seen, bad = [], []

    def check(ch):
        ev = evs[ch.event_ordinal]
        batches = w.trainer_epoch_batches(ev.n, 1024, 1, 0, ch.event_ordinal)[ch.batch_base:ch.batch_base + ch.n_batches]
        roots = np.concatenate(batches).astype(np.int64)
        boff = np.concatenate([[0], np.cumsum([len(b) for b in batches])]).astype(np.int64)
        seeds = hg.derive_seeds(hg.trainer_seed_spec(1, 0, ch.event_ordinal, batch_base=ch.batch_base), boff)
        dev = ch.sampler.to_host()
        bad.extend(check_against_oracle_chunks(dev, oracle_graph(ev), roots, boff, seeds,
                                               even_chunks(ch.n_batches, 16), gather=True, f_v=6, f_e=2,
                                               depth=3, fanout=6))
        seen.append((ch.event_ordinal, ch.batch_base, ch.n_batches))

    tot = es.epoch(0, on_chunk=check)
    es.close()
    assert not bad, bad
    assert tot["calls"] == 3 == len(seen)
    assert tot["minibatches"] == sum(e.n // 1024 for e in evs) == sum(s[2] for s in seen)


def test_fuzz_slice():
    """A fixed, seeded slice of scripts/fuzz_gpu.py: random graphs (uniform,
    banded, hubs, explicit zeros), depths 1-4, fanouts 1-300, both streams,
    both walks, ragged / empty batches, all outputs bit for bit."""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    import fuzz_gpu
    log = []
    cases, mism = fuzz_gpu.run(np.random.default_rng(20260), max_cases=120, log=log.append)
    assert cases == 120 and mism == 0, log


@pytest.mark.parametrize("iters", [0, 1, 2])
def test_k2_cuckoo_fallback(monkeypatch, iters):
    """The hash kernel's scan probes a cuckoo re-layout of its table; a root
    whose insert chain exceeds the bound rebuilds the 4-slot table instead
    (HGS_K2_CK_ITERS: 0 forces the fallback on every root, 1-2 on a mix of
    roots). Outputs stay equal to the reference digests on C1 (both RNGs)."""
    monkeypatch.setenv("HGS_K2_CK_ITERS", str(iters))
    hg = H()
    c1 = load_json("c1.json")
    ev = W().preset_event("C1")
    roots, boff, seeds = W().bench_roots(ev.n, 256, 16, seed=1, rep=0)
    S = hg.Sampler(hg.Graph(ev.rp, ev.ci).attach_features(ev.node_feat, ev.edge_feat, ev.labels))
    for run in c1["runs"]:
        S.bulk_shadow(roots, boff, seeds, rng=run["rng"], depth=run["depth"], fanout=6, gather=True)
        dev = S.to_host()
        for f in INT_FIELDS:
            assert sha(np.asarray(dev[f]).astype(np.int64)) == run["digests"][f], (f, iters)


@pytest.mark.parametrize("case", ["random", "clustered", "c1"])
@pytest.mark.parametrize("kernel", ["dir", "bm"])
def test_k2_alternative_kernels(monkeypatch, case, kernel):
    """The opt-in K2 kernels give the same outputs as the oracle: the
    rank-directory kernel with a shared-memory counting sort (HGS_K2=dir,
    csrc/extract_dir.cu) and the CTA-per-root bitmap-directory kernel over
    A's 4-entry quads (HGS_K2=bm, csrc/extract_bm.cu)."""
    monkeypatch.setenv("HGS_K2", kernel)
    hg = H()
    if case == "c1":
        c1 = load_json("c1.json")
        ev = W().preset_event("C1")
        roots, boff, seeds = W().bench_roots(ev.n, 256, 16, seed=1, rep=0)
        S = hg.Sampler(hg.Graph(ev.rp, ev.ci).attach_features(ev.node_feat, ev.edge_feat, ev.labels))
        for run in c1["runs"]:
            S.bulk_shadow(roots, boff, seeds, rng=run["rng"], depth=run["depth"], fanout=6, gather=True)
            dev = S.to_host()
            for f in INT_FIELDS:
                assert sha(np.asarray(dev[f]).astype(np.int64)) == run["digests"][f], f
        return
    if case == "random":
        g = random_graph(20000, 250000, 5)
    else:  # ids with locality: many keys per directory bucket (slow-path walks)
        n, w = 30000, 12
        u = np.repeat(np.arange(n), w)
        v = u + np.tile(np.arange(1, w + 1), n)
        keep = v < n
        key = np.unique(u[keep] * n + v[keep])
        rp = np.concatenate([[0], np.cumsum(np.bincount(key // n, minlength=n))]).astype(np.int64)
        g = O.Graph(n=n, rp=rp, ci=(key % n).astype(np.int64))
        rs = np.random.default_rng(3)
        g.node_feat, g.edge_feat = rs.standard_normal((n, 6)), rs.standard_normal((len(key), 2))
        g.labels = rs.integers(0, 2, len(key)).astype(np.uint8)
    rs = np.random.default_rng(11)
    k, b = 8, 256
    roots = np.concatenate([rs.permutation(g.n)[:b] for _ in range(k)]).astype(np.int64)
    boff = np.arange(k + 1, dtype=np.int64) * b
    seeds = rs.integers(0, 2**63, k * b, dtype=np.uint64)
    G = hg.Graph(g.rp, g.ci).attach_features(g.node_feat, g.edge_feat, g.labels)
    S = hg.Sampler(G)
    for rng in (0, 1):
        S.bulk_shadow(roots, boff, seeds, rng=rng, depth=3, fanout=6, gather=True)
        bad = check_against_oracle_chunks(S.to_host(), g, roots, boff, seeds, even_chunks(k, 4), gather=True,
                                          f_v=6, f_e=2, rng=rng, depth=3, fanout=6)
        assert not bad, bad
