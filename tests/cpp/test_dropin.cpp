// test_dropin.cpp — the C++ drop-in API (include/hitgnn/*.hpp,
// libhitgnn_gpu.so) used exactly as the reference's callers use it
// (Trainer::epoch_minibatch, trainer.cpp:433-459; cmd_bench_sampling,
// cli.cpp:393-430), checked against the C oracle (oracle/liboracle.so).
// Prints "ALL OK" on success; needs a GPU.
#include <algorithm>
#include <cmath>
#include <memory>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "hgs_oracle.h"
#include "hitgnn/data.hpp"
#include "hitgnn/rng.hpp"
#include "hitgnn/sampler.hpp"
#include "hitgnn/sparse.hpp"

using namespace hitgnn;

static int failures = 0;
#define CHECK(cond)                                                      \
    do {                                                                 \
        if (!(cond)) {                                                   \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
            ++failures;                                                  \
        }                                                                \
    } while (0)

template <class E, class F>
static std::string expect_throw(F&& f) {
    try {
        f();
    } catch (const E& e) {
        return e.what();
    } catch (...) {
        return "<wrong exception type>";
    }
    return "<no exception>";
}

struct Flat {
    std::vector<int64_t> bvoff, beoff, comp, l2g, rl, er, ec, eg, draws, decisions;
    std::vector<double> ev, xv, ye;
    std::vector<uint8_t> lab;
};

static Flat oracle(const CsrMatrix& a, const EventGraph* evg, const std::vector<std::vector<Index>>& batches,
                   const std::vector<uint64_t>& seeds, const std::vector<uint64_t>* state, int rng,
                   const SamplerConfig& cfg, int flags = 0) {
    std::vector<int64_t> roots, boff{0};
    for (auto& b : batches) {
        roots.insert(roots.end(), b.begin(), b.end());
        boff.push_back((int64_t)roots.size());
    }
    char err[256] = {0};
    or_result* r = or_bulk_shadow_ex(a.n_rows, a.n_cols, a.row_ptr.data(), a.col_idx.data(), a.values.data(),
                                     roots.data(), boff.data(), (int64_t)batches.size(), seeds.data(),
                                     state ? state->data() : nullptr, rng, cfg.depth, cfg.fanout,
                                     cfg.symmetrize, flags, evg ? evg->node_features.data.data() : nullptr,
                                     evg ? evg->node_features.cols : 0,
                                     evg ? evg->edge_features.data.data() : nullptr,
                                     evg ? evg->edge_features.cols : 0, evg ? evg->labels.data() : nullptr,
                                     err, sizeof err);
    if (!r) throw std::runtime_error(std::string("oracle failed: ") + err);
    int64_t c[8];
    or_result_counts(r, c);
    Flat f;
    const int64_t k = c[0], R = c[1], V = c[2], E = c[3];
    f.bvoff.resize(k + 1); f.beoff.resize(k + 1); f.comp.resize(R + k); f.l2g.resize(V); f.rl.resize(R);
    f.er.resize(E); f.ec.resize(E); f.eg.resize(E); f.ev.resize(E); f.draws.resize(R); f.decisions.resize(R);
    if (c[6]) { f.xv.resize(V * c[4]); f.ye.resize(E * c[5]); f.lab.resize(E); }
    or_result_copy(r, f.bvoff.data(), f.beoff.data(), f.comp.data(), f.l2g.data(), f.rl.data(), f.er.data(),
                   f.ec.data(), f.eg.data(), f.ev.data(), c[6] ? f.xv.data() : nullptr,
                   c[6] ? f.ye.data() : nullptr, c[6] ? f.lab.data() : nullptr, f.draws.data(),
                   f.decisions.data(), nullptr, nullptr);
    or_result_free(r);
    return f;
}

// Compare the reference-layout batches with the oracle's flat layout.
static void compare(const std::vector<SampledBatch>& got, const Flat& f, bool gathered, const char* what) {
    const int before = failures;
    int64_t roff = 0;
    CHECK(got.size() + 1 == f.bvoff.size());
    for (size_t b = 0; b < got.size(); ++b) {
        const SampledBatch& sb = got[b];
        const int64_t v0 = f.bvoff[b], v1 = f.bvoff[b + 1], e0 = f.beoff[b], e1 = f.beoff[b + 1];
        const int64_t nr = (int64_t)sb.roots_local.size();
        CHECK(sb.n_vertices() == v1 - v0);
        CHECK(sb.n_edges() == e1 - e0);
        CHECK(sb.n_components() == nr);
        for (int64_t i = 0; i <= nr; ++i) CHECK(sb.component_offsets[i] == f.comp[roff + b + i]);
        for (int64_t i = 0; i < nr; ++i) CHECK(sb.roots_local[i] == f.rl[roff + i]);
        for (int64_t i = 0; i < v1 - v0; ++i) CHECK(sb.local_to_global[i] == f.l2g[v0 + i]);
        for (int64_t e = 0; e < e1 - e0; ++e) {
            const CooEntry& ce = sb.adjacency.entries[e];
            CHECK(ce.row == f.er[e0 + e] && ce.col == f.ec[e0 + e]);
            CHECK(ce.value == (gathered ? 1.0 : f.ev[e0 + e]));
        }
        if (gathered) {
            CHECK(std::memcmp(sb.node_features.data.data(), f.xv.data() + v0 * sb.node_features.cols,
                              sizeof(double) * sb.node_features.data.size()) == 0);
            CHECK(std::memcmp(sb.edge_features.data.data(), f.ye.data() + e0 * sb.edge_features.cols,
                              sizeof(double) * sb.edge_features.data.size()) == 0);
            for (int64_t e = 0; e < e1 - e0; ++e) {
                CHECK(sb.edge_labels[e] == f.lab[e0 + e]);
                CHECK(sb.edge_global_ids[e] == f.eg[e0 + e]);
            }
        }
        roff += nr;
        if (failures > before + 5) break;
    }
    std::printf("%s: %s (%zu batches)\n", what, failures == before ? "ok" : "MISMATCH", got.size());
}

int main() {
    // ---- an event exactly as `hitgnn generate` produces it (C1 preset)
    GenConfig gc;
    gc.n_tracks = 1100; gc.hits_min = 7; gc.hits_max = 10; gc.detector_layers = 12;
    gc.noise_hits = 650; gc.false_edge_factor = 11.0; gc.f_v = 6; gc.f_e = 2; gc.seed = 1;
    const EventGraph event = generate_event(gc, 0);
    CHECK(event.n == 10069 && event.m() == 99828);
    const CsrMatrix adj = make_edge_id_matrix(event);

    // ---- bench-sampling protocol (cli.cpp:393-408)
    const Index k = 8, b = 256;
    Rng rng(Rng::derive(1, {0x62656e6368ULL, (uint64_t)k, 0}));
    auto batches = epoch_root_batches(event.n, b, rng);
    batches.resize(k);
    std::vector<uint64_t> seeds;
    for (Index bi = 0; bi < k; ++bi)
        for (Index pos = 0; pos < b; ++pos)
            seeds.push_back(Rng::derive(1, {0x7374726dULL, (uint64_t)k, 0, (uint64_t)bi, (uint64_t)pos}));
    SamplerConfig cfg;
    cfg.depth = 2; cfg.fanout = 6; cfg.batch_size = b; cfg.bulk_batches = k;

    {   // trainer path: bulk_shadow then gather_features per batch
        PerRootChoiceSource src(seeds);
        auto out = bulk_shadow(adj, batches, cfg, src);
        compare(out, oracle(adj, nullptr, batches, seeds, nullptr, 0, cfg), false, "bulk_shadow");
        for (auto& sb : out) gather_features(sb, event);
        compare(out, oracle(adj, &event, batches, seeds, nullptr, 0, cfg), true, "bulk_shadow+gather_features");
    }
    {   // resident-graph cache: the trainer's repeated calls reuse one upload;
        // an in-place change of A's content is detected (new entry, new results)
        gpu::release_cached();
        for (int rep = 0; rep < 3; ++rep) {
            PerRootChoiceSource src(seeds);
            auto out = bulk_shadow(adj, batches, cfg, src);
            for (auto& sb : out) gather_features(sb, event);
            compare(out, oracle(adj, &event, batches, seeds, nullptr, 0, cfg), true, "cached trainer path");
        }
        CHECK(gpu::cached_entries() == 2);  // A and the event
        // reps 1 and 2 found the event resident: their gathers were prefetched
        CHECK(gpu::prefetched_gathers() >= static_cast<std::size_t>(2 * k));
        {   // a copied batch, a reordered gather and an untouched batch still get exact features
            const std::size_t before = gpu::prefetched_gathers();
            PerRootChoiceSource src(seeds);
            auto out = bulk_shadow(adj, batches, cfg, src);
            compare(out, oracle(adj, nullptr, batches, seeds, nullptr, 0, cfg), false, "prefetch: values before gather");
            std::vector<SampledBatch> copy(out.begin(), out.end());  // new buffers: no prefetch match
            for (Index bi = k - 1; bi >= 0; --bi) gather_features(out[bi], event);
            for (auto& sb : copy) gather_features(sb, event);
            compare(out, oracle(adj, &event, batches, seeds, nullptr, 0, cfg), true, "prefetch: reverse order");
            compare(copy, oracle(adj, &event, batches, seeds, nullptr, 0, cfg), true, "prefetch: copies");
            CHECK(gpu::prefetched_gathers() == before + static_cast<std::size_t>(k));
        }
        CsrMatrix adj2 = adj;
        {
            PerRootChoiceSource src(seeds);
            auto out = bulk_shadow(adj2, batches, cfg, src);
            compare(out, oracle(adj2, nullptr, batches, seeds, nullptr, 0, cfg), false, "cache: copy of A");
        }
        // drop one edge of row 0 in place (same arrays, same sizes are not
        // possible: rebuild row 0 with its last column replaced)
        const Index r0b = adj2.row_ptr[0], r0e = adj2.row_ptr[1];
        if (r0e > r0b) {
            std::vector<bool> used(static_cast<std::size_t>(adj2.n_cols), false);
            for (Index t = r0b; t < r0e; ++t) used[adj2.col_idx[t]] = true;
            Index c = adj2.n_cols - 1;
            while (c >= 0 && used[c]) --c;
            if (c > adj2.col_idx[r0e - 1]) {
                adj2.col_idx[r0e - 1] = c;  // still sorted and unique
                PerRootChoiceSource src(seeds);
                auto out = bulk_shadow(adj2, batches, cfg, src);
                compare(out, oracle(adj2, nullptr, batches, seeds, nullptr, 0, cfg), false, "cache: A changed in place");
            }
        }
        gpu::release_cached();
        CHECK(gpu::cached_entries() == 0);
    }
    {   // resident event, fused gather, reused (non-fresh) source on a second call
        gpu::DeviceEvent dev(event);
        PerRootChoiceSource src(seeds);
        auto out1 = dev.bulk_shadow(batches, cfg, src, true);
        const Flat f1 = oracle(adj, &event, batches, seeds, nullptr, 0, cfg);
        compare(out1, f1, true, "DeviceEvent::bulk_shadow(gather)");
        std::vector<uint64_t> st(4 * seeds.size());
        for (size_t r = 0; r < seeds.size(); ++r) {
            or_xoshiro x;
            or_xoshiro_seed(&x, seeds[r]);
            for (int64_t i = 0; i < f1.draws[r]; ++i) or_xoshiro_next(&x);
            std::memcpy(&st[4 * r], x.s, sizeof x.s);
        }
        auto out2 = dev.bulk_shadow(batches, cfg, src, true);
        compare(out2, oracle(adj, &event, batches, seeds, &st, 0, cfg), true, "resumed PerRootChoiceSource");
        // host use after device use replays the device's draws first
        src.begin_root(3);
        auto pos = src.choose(10, 3);
        or_xoshiro x;
        std::memcpy(x.s, &st[12], sizeof x.s);
        const Flat f2 = oracle(adj, &event, batches, seeds, &st, 0, cfg);
        for (int64_t i = 0; i < f2.draws[3]; ++i) or_xoshiro_next(&x);
        uint32_t exp[3];
        or_choose_xoshiro(&x, 10, 3, exp);
        CHECK(pos.size() == 3 && pos[0] == exp[0] && pos[1] == exp[1] && pos[2] == exp[2]);
    }
    {   // Philox streams, d = 3
        SamplerConfig c3 = cfg;
        c3.depth = 3;
        PhiloxChoiceSource src(seeds);
        auto out = bulk_shadow(adj, batches, c3, src);
        compare(out, oracle(adj, nullptr, batches, seeds, nullptr, 1, c3), false, "bulk_shadow(Philox)");
        // host PhiloxChoiceSource == oracle choose for the next decision
        src.begin_root(5);
        auto pos = src.choose(20, 4);
        const Flat f = oracle(adj, nullptr, batches, seeds, nullptr, 1, c3);
        uint32_t exp[4];
        or_choose_philox(seeds[5], (uint32_t)f.decisions[5], 20, 4, exp);
        CHECK(pos.size() == 4 && pos[0] == exp[0] && pos[3] == exp[3]);
    }
    {   // k x shadow_reference with seed slices == bulk (cli.cpp:418-430)
        std::vector<SampledBatch> seq;
        for (Index bi = 0; bi < k; ++bi) {
            PerRootChoiceSource src(std::vector<uint64_t>(seeds.begin() + bi * b, seeds.begin() + (bi + 1) * b));
            seq.push_back(shadow_reference(adj, batches[bi], cfg, src));
        }
        compare(seq, oracle(adj, nullptr, batches, seeds, nullptr, 0, cfg), false, "k x shadow_reference");
    }
    {   // errors: the reference's exception types and texts
        PerRootChoiceSource src(seeds);
        auto bad = batches;
        bad[1][7] = bad[1][3];
        CHECK(expect_throw<std::invalid_argument>([&] { bulk_shadow(adj, bad, cfg, src); }) ==
              "sampler: duplicate root " + std::to_string(bad[1][3]));
        bad = batches;
        bad[0][0] = event.n;
        CHECK(expect_throw<std::invalid_argument>([&] { bulk_shadow(adj, bad, cfg, src); }) ==
              "sampler: root " + std::to_string(event.n) + " out of range");
        SamplerConfig c0 = cfg;
        c0.depth = 0;
        CHECK(expect_throw<std::invalid_argument>([&] { bulk_shadow(adj, batches, c0, src); }) ==
              "SamplerConfig: depth must be >= 1");
        RandomChoiceSource single(3);
        CHECK(expect_throw<std::invalid_argument>([&] { bulk_shadow(adj, batches, cfg, single); }) !=
              "<no exception>");
        CsrMatrix rect(3, 4);
        CHECK(expect_throw<std::invalid_argument>([&] { symmetrize_pattern(rect); }) ==
              "symmetrize_pattern: matrix must be square");
        SampledBatch plain;
        plain.local_to_global = {0, 1};
        plain.adjacency = CooMatrix{2, 2, {{0, 1, 0.25}}};  // llround(0.25) - 1 = -1
        CHECK(expect_throw<std::invalid_argument>([&] { gather_features(plain, event); }).find(
                  "do not carry edge ids") != std::string::npos);
        std::printf("errors: %s\n", failures ? "see above" : "ok");
    }
    {   // symmetrize_pattern (device K0) == oracle
        const CsrMatrix w = symmetrize_pattern(adj);
        std::vector<int64_t> rp(adj.n_rows + 1), ci(2 * adj.nnz());
        const int64_t nnz = or_symmetrize(adj.n_rows, adj.row_ptr.data(), adj.col_idx.data(), rp.data(), ci.data());
        CHECK(w.nnz() == nnz);
        CHECK(std::equal(rp.begin(), rp.end(), w.row_ptr.begin()));
        CHECK(std::equal(ci.begin(), ci.begin() + nnz, w.col_idx.begin()));
        CHECK(w.values.size() == (size_t)nnz && w.values[0] == 1.0);
        std::printf("symmetrize_pattern: ok\n");
    }
    {   // host containers (test_sparse.cpp:10-44 semantics)
        CooMatrix m{2, 2, {{1, 1, 2.0}, {0, 0, 1.5}, {1, 1, -2.0}, {0, 1, 0.5}}};
        m.canonicalize();
        CHECK((m.entries == std::vector<CooEntry>{{0, 0, 1.5}, {0, 1, 0.5}}));
        CooMatrix dups{2, 2, {{0, 0, 1.0}, {0, 0, 2.0}}};
        CHECK(expect_throw<std::invalid_argument>([&] { coo_to_csr(dups); }) != "<no exception>");
        const CsrMatrix round = coo_to_csr(csr_to_coo(adj));
        CHECK(round == adj);
    }
    {   // sample_rows (sampler.cpp:64-86) on the GPU vs the host choice sources,
        // then both sources must continue identically (device draws replayed)
        CsrMatrix p(6, 40);
        p.row_ptr = {0, 5, 5, 17, 18, 30, 40};
        for (Index i = 0; i < 40; ++i) p.col_idx.push_back(i % 40);
        for (Index r = 0; r < 6; ++r) std::sort(p.col_idx.begin() + p.row_ptr[r], p.col_idx.begin() + p.row_ptr[r + 1]);
        p.values.assign(40, 0.5);
        const std::vector<Index> streams = {2, 0, 2, 1, 0, 2};
        const std::vector<uint64_t> sd = {11, 22, 33};
        for (int mode = 0; mode < 2; ++mode) {
            std::unique_ptr<ChoiceSource> dev_src, host_src;
            if (mode == 0) {
                dev_src = std::make_unique<PerRootChoiceSource>(sd);
                host_src = std::make_unique<PerRootChoiceSource>(sd);
            } else {
                dev_src = std::make_unique<PhiloxChoiceSource>(sd);
                host_src = std::make_unique<PhiloxChoiceSource>(sd);
            }
            const auto got = sample_rows(p, 4, *dev_src, streams);
            for (Index r = 0; r < 6; ++r) {
                const auto sup = p.row_cols(r);
                std::vector<Index> exp;
                if (!sup.empty()) {
                    host_src->begin_root((uint64_t)streams[r]);
                    for (auto q : host_src->choose((uint32_t)sup.size(), std::min<uint32_t>(4, (uint32_t)sup.size())))
                        exp.push_back(sup[q]);
                }
                CHECK(got[r] == exp);
            }
            for (uint64_t st = 0; st < 3; ++st) {
                dev_src->begin_root(st);
                host_src->begin_root(st);
                CHECK(dev_src->choose(50, 5) == host_src->choose(50, 5));
            }
        }
        PerRootChoiceSource src(sd);
        CHECK(expect_throw<std::invalid_argument>([&] { sample_rows(p, 0, src, streams); }) ==
              "sample_rows: s must be >= 1");
    }
    {   // FrontierObserver through the resident-event path: shapes of Q / F / P
        gpu::DeviceEvent dev(event);
        PerRootChoiceSource src(seeds);
        Index levels = 0, prev_q = (Index)(k * b);
        auto out = dev.bulk_shadow(batches, cfg, src, false, [&](Index level, const FrontierSet& fs) {
            ++levels;
            CHECK(level == levels);
            CHECK(fs.f.n_rows == k * b && fs.q.n_cols == event.n);
            CHECK(fs.p.n_rows == prev_q);  // P: one row per frontier row of the level before
            for (Index r = 0; r < fs.p.n_rows; ++r) {
                double sum = 0;
                for (Index t = fs.p.row_ptr[r]; t < fs.p.row_ptr[r + 1]; ++t) sum += fs.p.values[t];
                CHECK(fs.p.row_ptr[r + 1] == fs.p.row_ptr[r] || std::fabs(sum - 1.0) < 1e-12);
            }
            prev_q = fs.q.n_rows;
        });
        CHECK(levels == cfg.depth);
        compare(out, oracle(adj, nullptr, batches, seeds, nullptr, 0, cfg), false, "bulk_shadow(observer)");
    }
    std::printf(failures ? "FAILURES: %d\n" : "ALL OK\n", failures);
    return failures ? 1 : 0;
}
