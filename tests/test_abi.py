"""CPU: the C-ABI boundary — libraries load, every symbol declared in
include/*.h is exported, host-only helpers agree with the oracle, and the
compute entry points fail cleanly (no crash, no CPU fallback) without a GPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from tests.conftest import has_gpu
from tests.helpers import O, ROOT, load_json

LIB = os.path.join(ROOT, "paper_2504_04670_b200", "lib")


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hgs_[a-z0-9_]+)\s*\(", text)))


def exported(so):
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_hgs_exports_every_declared_symbol():
    from paper_2504_04670_b200 import hgs
    names = declared("hgs.h")
    assert len(names) >= 20
    ex = exported(os.path.join(LIB, "libhgs.so"))
    missing = [n for n in names if n not in ex]
    assert not missing, missing
    assert set(hgs.EXPORTS) <= set(names)
    L = hgs.lib()
    for n in names:
        getattr(L, n)


def test_tools_exports():
    names = declared("hgs_tools.h")
    ex = exported(os.path.join(LIB, "libhitgnn_gpu.so"))
    assert not [n for n in names if n not in ex]


def test_dropin_exports_reference_api():
    ex = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(LIB, "libhitgnn_gpu.so")],
                        capture_output=True, text=True).stdout
    for sym in ["hitgnn::bulk_shadow(", "hitgnn::shadow_reference(", "hitgnn::gather_features(",
                "hitgnn::make_edge_id_matrix(", "hitgnn::epoch_root_batches(",
                "hitgnn::symmetrize_pattern(", "hitgnn::generate_event(", "hitgnn::coo_to_csr(",
                "hitgnn::csr_to_coo(", "hitgnn::Rng::derive(", "hitgnn::PerRootChoiceSource::choose(",
                "hitgnn::PhiloxChoiceSource::choose(", "hitgnn::gpu::DeviceEvent::bulk_shadow("]:
        assert sym in ex, sym


def test_host_helpers_match_oracle():
    from paper_2504_04670_b200 import hgs
    assert hgs.lib().hgs_abi_version() == 1
    for seed, path, val in load_json("kat.json")["derive"]:
        assert f"{hgs.derive(int(seed), [int(p) for p in path]):016x}" == val
    for ctr, key, out in load_json("kat.json")["philox_random123"]:
        assert [f"{int(x):08x}" for x in hgs.philox4x32_10(ctr, key)] == out


def test_seed_spec_matches_reference_streams():
    """hgs_derive_seeds = the reference's per-root stream seeds: the trainer's
    root_stream_seed (trainer.cpp:200-206) and bench-sampling (cli.cpp:404-408),
    restated by the oracle's derive (pinned to the reference KATs)."""
    from paper_2504_04670_b200 import hgs
    boff = np.array([0, 3, 3, 7, 12], np.int64)
    for spec, pre, base in [(hgs.trainer_seed_spec(7, 2, 5, batch_base=10), [0x73616D706C, 2, 5], 10),
                            (hgs.bench_seed_spec(1, 64, 3), [0x7374726D, 64, 3], 0)]:
        got = hgs.derive_seeds(spec, boff)
        exp = [O.derive(spec.seed, pre + [base + b, r - boff[b]])
               for b in range(len(boff) - 1) for r in range(boff[b], boff[b + 1])]
        assert [int(x) for x in got] == exp
    with pytest.raises(hgs.SamplerError):
        hgs.SeedSpec.make(1, [1] * 7)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure path")
def test_compute_fails_loudly_without_gpu():
    from paper_2504_04670_b200 import hgs
    assert hgs.device_count() == 0
    with pytest.raises(hgs.HgsRuntimeError):
        hgs.Graph(np.array([0, 1, 1]), np.array([1]))


def test_graph_create_validates_before_touching_the_device():
    # host-side checks (O(n) row pointers; general-valued A entirely); the
    # column range of an edge-id A is checked on the device
    # (test_gpu_parity.py::test_ingest_validation_messages)
    from paper_2504_04670_b200 import hgs
    with pytest.raises(hgs.SamplerError, match="out of range"):
        hgs.Graph(np.array([0, 1, 1]), np.array([5]), np.ones(1))
    with pytest.raises(hgs.SamplerError, match="row_ptr"):
        hgs.Graph(np.array([1, 1, 1]), np.array([0]))
    with pytest.raises(hgs.SamplerError, match="row_ptr not non-decreasing"):
        hgs.Graph(np.array([0, 2, 1, 2]), np.array([0, 1]))


def test_generator_matches_reference_digest():
    """The product-side event generator (libhitgnn_gpu) reproduces the
    reference generator bit for bit on C1 (digests from the reference)."""
    from paper_2504_04670_b200 import workload as W
    from tests.helpers import sha
    c1 = load_json("c1.json")["graph"]
    ev = W.preset_event("C1")
    assert (ev.n, ev.m) == (c1["n"], c1["m"])
    for k, a in (("rp", ev.rp), ("ci", ev.ci), ("node_feat", ev.node_feat),
                 ("edge_feat", ev.edge_feat), ("labels", ev.labels)):
        assert sha(a) == c1[k], k


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")
def test_generator_matches_reference_presets():
    from paper_2504_04670_b200 import workload as W
    for kw in (dict(n_tracks=110, hits_min=7, hits_max=10, layers=12, noise=65, false_factor=1.0,
                    f_v=9, f_e=7, seed=3),
               dict(n_tracks=1500, hits_min=7, hits_max=10, layers=12, noise=250, false_factor=3.25,
                    f_v=6, f_e=2, seed=1)):
        for eid in (0, 5):
            a = W.generate_event(**kw, event_id=eid)
            r = O.ref_generate_event(kw["n_tracks"], kw["hits_min"], kw["hits_max"], kw["layers"],
                                     kw["noise"], kw["false_factor"], kw["f_v"], kw["f_e"],
                                     kw["seed"], eid)
            assert np.array_equal(a.rp, r.rp) and np.array_equal(a.ci, r.ci)
            assert np.array_equal(a.node_feat.view(np.uint64), r.node_feat.view(np.uint64))
            assert np.array_equal(a.edge_feat.view(np.uint64), r.edge_feat.view(np.uint64))
            assert np.array_equal(a.labels, r.labels)


def test_event_save_load_roundtrip(tmp_path):
    from paper_2504_04670_b200 import workload as W
    ev = W.preset_event("C1")
    f = str(tmp_path / "c1.npz")
    W.save_event(f, ev)
    ev2 = W.load_event(f)
    assert ev2.n == ev.n and ev2.m == ev.m
    for a in ("rp", "ci", "node_feat", "edge_feat", "labels"):
        assert np.array_equal(getattr(ev, a), getattr(ev2, a)), a


def test_event_file_round_trip_and_corruption(tmp_path):
    """hgs_event_save / hgs_event_info (no GPU needed): header round trip,
    64-byte-aligned sections, truncated and foreign files rejected."""
    from paper_2504_04670_b200 import hgs
    rp = np.array([0, 2, 3, 3], np.int64)
    ci = np.array([1, 2, 0], np.int64)
    nf = np.arange(6, dtype=np.float64).reshape(3, 2)
    ef = np.arange(3, dtype=np.float64).reshape(3, 1)
    lab = np.array([1, 0, 1], np.uint8)
    p = str(tmp_path / "ev.hgsev")
    hgs.save_event(p, rp, ci, node_feat=nf, edge_feat=ef, labels=lab)
    assert hgs.event_info(p) == {"n_rows": 3, "n_cols": 3, "nnz": 3, "f_v": 2, "f_e": 1, "flags": 0}
    raw = open(p, "rb").read()
    assert len(raw) % 64 == 0
    open(p + ".cut", "wb").write(raw[:-64])
    with pytest.raises(hgs.SamplerError, match="truncated or corrupt"):
        hgs.event_info(p + ".cut")
    open(p + ".bad", "wb").write(b"NOTANEVT" + raw[8:])
    with pytest.raises(hgs.SamplerError, match="bad magic"):
        hgs.event_info(p + ".bad")
    with pytest.raises(hgs.SamplerError, match="cannot open"):
        hgs.event_info(str(tmp_path / "missing"))
    with pytest.raises(hgs.SamplerError, match="bad row_ptr"):
        hgs.save_event(str(tmp_path / "bad_rp"), np.array([1, 2, 3, 3]), ci)
    with pytest.raises(hgs.SamplerError, match="shorter"):
        hgs.save_event(str(tmp_path / "short_ci"), rp, ci[:2])
    with pytest.raises(hgs.SamplerError, match="shorter"):
        hgs.save_event(str(tmp_path / "short_lab"), rp, ci, labels=lab[:1])
