"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Every expected output here comes from the unmodified reference sampler
compiled in place by oracle/Makefile (oracle/_ref/libhitgnn_ref.so, only
available where /root/reference exists). The fixtures then travel with the
repo, so the oracle restatement and the CUDA path are checked against the
reference's own results on machines without it.

    python tests/golden/make_golden.py          # KATs, small cases, C1, frontiers
    python tests/golden/make_golden.py --c2     # C2 event + sampler digests (~3 min)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT_FIELDS = ["batch_voff", "batch_eoff", "comp_off", "l2g", "roots_local", "e_row", "e_col",
              "e_gid", "e_val", "xv", "ye", "lab"]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_graph(n, m, seed, values_kind=None, self_loops=False):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    if not self_loops:
        keep = u != v
        u, v = u[keep], v[keep]
    key = np.unique(u.astype(np.int64) * n + v)
    u, v = key // n, key % n
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, u + 1, 1)
    rp = np.cumsum(rp)
    mm = len(v)
    vals = None
    if values_kind == "zeros":
        vals = rng.uniform(0.5, 2.0, mm)
        vals[rng.random(mm) < 0.2] = 0.0
    g = O.Graph(n=n, rp=rp, ci=v.astype(np.int64), values=vals,
                node_feat=rng.standard_normal((n, 3)), edge_feat=rng.standard_normal((mm, 2)),
                labels=rng.integers(0, 2, mm).astype(np.uint8))
    return g


def coo_graph(n, edges):
    edges = sorted(set(edges))
    rp = np.zeros(n + 1, np.int64)
    ci = []
    for (a, b) in edges:
        rp[a + 1] += 1
        ci.append(b)
    rp = np.cumsum(rp)
    m = len(edges)
    return O.Graph(n=n, rp=rp, ci=np.array(ci, np.int64), node_feat=np.arange(n * 3, dtype=float).reshape(n, 3),
                   edge_feat=np.arange(m * 2, dtype=float).reshape(m, 2) / 7.0,
                   labels=(np.arange(m) % 2).astype(np.uint8))


def cases():
    out = []
    rs = np.random.default_rng(2024)
    # random graphs x configurations
    for gi, (n, m) in enumerate([(5, 12), (20, 60), (60, 240), (200, 900)]):
        for vk in (None, "zeros"):
            g = random_graph(n, m, 100 + gi, vk, self_loops=(gi == 2))
            for d, s in ((1, 2), (2, 1), (2, 6), (3, 3)):
                for rng in (0, 1):
                    for sym in (True, False):
                        k = 3 if n >= 20 else 1
                        b = min(n // k, 7)
                        roots = np.concatenate([rs.permutation(n)[:b] for _ in range(k)])
                        boff = np.arange(k + 1, dtype=np.int64) * b
                        seeds = rs.integers(0, 2**63, len(roots), dtype=np.uint64)
                        out.append(dict(name=f"rand{gi}_{vk}_d{d}s{s}_r{rng}_{int(sym)}", g=g,
                                        roots=roots, boff=boff, seeds=seeds, depth=d, fanout=s,
                                        rng=rng, sym=sym, gather=vk is None))
    # an empty batch and a zero-root call
    g = random_graph(30, 100, 7)
    out.append(dict(name="empty_batch", g=g, roots=np.array([3, 4, 9, 1], np.int64),
                    boff=np.array([0, 2, 2, 4], np.int64), seeds=np.arange(4, dtype=np.uint64) + 5,
                    depth=2, fanout=3, rng=0, sym=True, gather=True))
    out.append(dict(name="no_roots", g=g, roots=np.zeros(0, np.int64), boff=np.array([0, 0], np.int64),
                    seeds=np.zeros(0, np.uint64), depth=2, fanout=3, rng=0, sym=True, gather=True))
    # SPEC.md:152-174 known answers
    path = coo_graph(4, [(0, 1), (1, 2), (2, 3)])
    out.append(dict(name="spec_path_d1s1", g=path, roots=np.array([0], np.int64),
                    boff=np.array([0, 1], np.int64), seeds=np.array([11], np.uint64), depth=1,
                    fanout=1, rng=0, sym=True, gather=True))
    star = coo_graph(6, [(0, i) for i in range(1, 6)])
    out.append(dict(name="spec_star", g=star, roots=np.array([0], np.int64), boff=np.array([0, 1], np.int64),
                    seeds=np.array([3], np.uint64), depth=1, fanout=5, rng=1, sym=True, gather=True))
    tri = coo_graph(9, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5), (6, 7), (7, 8), (6, 8)])
    out.append(dict(name="spec_triangles", g=tri, roots=np.array([0, 4, 8], np.int64),
                    boff=np.array([0, 1, 2, 3], np.int64), seeds=np.array([1, 2, 3], np.uint64),
                    depth=2, fanout=2, rng=0, sym=True, gather=True))
    iso = coo_graph(5, [(0, 1), (1, 2)])
    out.append(dict(name="spec_isolated", g=iso, roots=np.array([4, 0], np.int64),
                    boff=np.array([0, 2], np.int64), seeds=np.array([9, 10], np.uint64), depth=3,
                    fanout=2, rng=1, sym=True, gather=True))
    return out


def frontier_cases():
    """FrontierObserver fixtures (sampler.hpp:52-58; sampler.cpp:149-158, 186):
    the reference's per-level Q / F / P of small bulk calls."""
    out = []
    g = random_graph(300, 1500, 41)
    rs = np.random.default_rng(41)
    roots = np.concatenate([rs.permutation(300)[:20] for _ in range(3)]).astype(np.int64)
    boff = np.array([0, 20, 40, 60], np.int64)
    seeds = rs.integers(0, 2**63, 60, dtype=np.uint64)
    out.append(dict(name="sym_xoshiro", g=g, roots=roots, boff=boff, seeds=seeds, depth=3, fanout=4, rng=0,
                    sym=True))
    out.append(dict(name="ids_philox", g=g, roots=roots, boff=boff, seeds=seeds, depth=3, fanout=3, rng=1,
                    sym=False))
    gz = random_graph(200, 1200, 42, values_kind="zeros")
    out.append(dict(name="values_zeros", g=gz, roots=roots[:30] % 200, boff=np.array([0, 15, 30], np.int64),
                    seeds=seeds[:30], depth=2, fanout=5, rng=0, sym=False))
    return out


def write_frontiers():
    arrays, index = {}, []
    for c in frontier_cases():
        g = c["g"]
        s = O.bulk_shadow(g, c["roots"], c["boff"], c["seeds"], rng=c["rng"], depth=c["depth"],
                          fanout=c["fanout"], symmetrize=c["sym"], impl="ref", mode=2)
        pre = c["name"] + "/"
        arrays[pre + "rp"], arrays[pre + "ci"] = g.rp, g.ci
        if g.values is not None:
            arrays[pre + "values"] = g.values
        arrays[pre + "roots"], arrays[pre + "boff"], arrays[pre + "seeds"] = c["roots"], c["boff"], c["seeds"]
        index.append({"name": c["name"], "n": g.n, "depth": c["depth"], "fanout": c["fanout"], "rng": c["rng"],
                      "sym": c["sym"], "values": g.values is not None,
                      "levels": [{k: digest(v) for k, v in lv.items()} for lv in s.levels]})
    np.savez_compressed(os.path.join(HERE, "frontiers.npz"), **arrays)
    with open(os.path.join(HERE, "frontiers.json"), "w") as f:
        json.dump(index, f, indent=1)
    print("frontier fixtures written:", len(index))


def write_c2():
    """C2 (BASELINE configs[1]) digests from the reference generator and
    sampler: the event arrays, and the full bench-protocol call (64 x 1024
    roots, d=3, s=6, gather) under both choice streams."""
    g = O.ref_generate_event(n_tracks=13000, noise=10000, false_factor=14.5)
    c2 = {"graph": {"n": g.n, "m": g.m, "rp": digest(g.rp), "ci": digest(g.ci),
                    "node_feat": digest(g.node_feat), "edge_feat": digest(g.edge_feat),
                    "labels": digest(g.labels)}, "runs": []}
    k, b = 64, 1024
    rsd = O.derive(1, [0x62656E6368, k, 0])
    batches = O.epoch_root_batches(g.n, b, rsd, impl="ref")[:k]
    roots = np.concatenate(batches)
    boff = np.arange(k + 1, dtype=np.int64) * b
    seeds = np.array([O.derive(1, [0x7374726D, k, 0, bi, pos]) for bi in range(k) for pos in range(b)],
                     np.uint64)
    c2["roots"] = digest(roots)
    c2["seeds"] = digest(seeds)
    for rng in (0, 1):
        s = O.bulk_shadow(g, roots, boff, seeds, rng=rng, depth=3, fanout=6, gather=True, impl="ref")
        c2["runs"].append({"rng": rng, "depth": 3, "V": s.V, "E": s.E,
                           "digests": {f: digest(getattr(s, f)) for f in OUT_FIELDS}})
    with open(os.path.join(HERE, "c2.json"), "w") as f:
        json.dump(c2, f, indent=1)
    print("C2 reference digests written:", [(r["rng"], r["V"], r["E"]) for r in c2["runs"]])


def main():
    if "--frontiers" in sys.argv:
        write_frontiers()
        return
    if "--c2" in sys.argv:
        write_c2()
        return
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: run `make -f oracle/Makefile` where /root/reference exists")
    # ---- known answers
    kat = {"rng_first": {}, "derive": [], "bounded": {}, "choose": {}, "epoch_root_batches": {}}
    for seed in (0, 1, 7, 42):
        out = np.zeros(3, np.uint64)
        O._ref().ref_rng_first(seed, 3, out)
        kat["rng_first"][str(seed)] = [f"{int(x):016x}" for x in out]
    for seed, path in ((1, [0x7374726D, 1, 0, 0, 0]), (1, [0x73616D706C, 0, 0, 0, 0]),
                       (1, [0x62656E6368, 64, 0]), (5, []), (2**63 + 3, [1, 2, 3, 4, 5, 6])):
        kat["derive"].append([str(seed), [str(x) for x in path], f"{O.derive(seed, path, 'ref'):016x}"])
    bounds = np.array([10, 9, 8, 1, 2, 1000, 2**40], np.uint64)
    bo = np.zeros(len(bounds), np.uint64)
    O._ref().ref_bounded_seq(7, bounds, len(bounds), bo)
    kat["bounded"] = {"seed": 7, "bounds": [str(int(x)) for x in bounds], "out": [int(x) for x in bo]}
    ns = np.array([10, 4, 25, 1, 7, 100, 3], np.uint32)
    ks = np.array([3, 4, 6, 1, 9, 6, 0], np.uint32)
    co = np.zeros(int(np.minimum(ns, ks).sum()), np.uint32)
    O._ref().ref_choose_seq(7, ns, ks, len(ns), co)
    kat["choose"] = {"seed": 7, "n": ns.tolist(), "k": ks.tolist(), "out": co.tolist()}
    perm = np.zeros(50, np.int64)
    nb = O._ref().ref_epoch_root_batches(50, 8, 99, perm)
    kat["epoch_root_batches"] = {"n": 50, "b": 8, "seed": 99, "n_batches": int(nb), "perm": perm[:nb * 8].tolist()}
    kat["philox_random123"] = [  # published Random123 KATs for philox4x32-10
        [[0, 0, 0, 0], [0, 0], ["6627e8d5", "e169c58d", "bc57ac4c", "9b00dbd8"]],
        [[0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, ["408f276d", "41c83b0e", "a20bc7c6", "6d5451fd"]],
        [[0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         ["d16cfe09", "94fdcceb", "5001e420", "24126ea1"]]]
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)

    # ---- small cases, full expected outputs from the reference
    arrays, index, graphs = {}, [], {}
    for i, c in enumerate(cases()):
        g = c["g"]
        pre = f"c{i}_"
        if id(g) not in graphs:  # each graph stored once
            gp = f"g{len(graphs)}_"
            graphs[id(g)] = gp
            arrays[gp + "rp"] = g.rp
            arrays[gp + "ci"] = g.ci
            if g.values is not None:
                arrays[gp + "values"] = g.values
            arrays[gp + "nf"] = g.node_feat
            arrays[gp + "ef"] = g.edge_feat
            arrays[gp + "lab"] = g.labels
        arrays[pre + "roots"] = c["roots"]
        arrays[pre + "boff"] = c["boff"]
        arrays[pre + "seeds"] = c["seeds"]
        ent = {k: c[k] for k in ("name", "depth", "fanout", "rng", "sym", "gather")}
        ent.update(n=g.n, has_values=g.values is not None, prefix=pre, graph=graphs[id(g)])
        try:
            s = O.bulk_shadow(g, c["roots"], c["boff"], c["seeds"], rng=c["rng"], depth=c["depth"],
                              fanout=c["fanout"], symmetrize=c["sym"], gather=c["gather"], impl="ref")
            for fld in OUT_FIELDS:
                a = getattr(s, fld)
                if a is not None:
                    arrays[pre + "out_" + fld] = a
            ent["error"] = None
        except O.SamplerError as e:
            ent["error"] = str(e)
        index.append(ent)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    with open(os.path.join(HERE, "small_cases.json"), "w") as f:
        json.dump(index, f, indent=1)

    # ---- C1 (BASELINE configs[0]) digests from the reference generator + sampler
    g = O.ref_generate_event()
    c1 = {"graph": {"n": g.n, "m": g.m, "rp": digest(g.rp), "ci": digest(g.ci),
                    "node_feat": digest(g.node_feat), "edge_feat": digest(g.edge_feat),
                    "labels": digest(g.labels)}, "runs": []}
    k, b = 16, 256
    rsd = O.derive(1, [0x62656E6368, k, 0])
    batches = O.epoch_root_batches(g.n, b, rsd, impl="ref")[:k]
    roots = np.concatenate(batches)
    boff = np.arange(k + 1, dtype=np.int64) * b
    seeds = np.array([O.derive(1, [0x7374726D, k, 0, bi, pos]) for bi in range(k) for pos in range(b)],
                     np.uint64)
    c1["roots"] = digest(roots)
    c1["seeds"] = digest(seeds)
    for rng in (0, 1):
        for d in (2, 3):
            s = O.bulk_shadow(g, roots, boff, seeds, rng=rng, depth=d, fanout=6, gather=True, impl="ref")
            c1["runs"].append({"rng": rng, "depth": d, "V": s.V, "E": s.E,
                               "digests": {f: digest(getattr(s, f)) for f in OUT_FIELDS}})
    with open(os.path.join(HERE, "c1.json"), "w") as f:
        json.dump(c1, f, indent=1)
    print("golden fixtures written:", len(index), "small cases;", len(c1["runs"]), "C1 runs")
    write_frontiers()


if __name__ == "__main__":
    main()
