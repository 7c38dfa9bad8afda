// eventgen.cpp — synthetic TrackML-shaped events: the workload source for the
// sampler benchmarks and parity tests on machines without the reference.
//
// Semantics are those of the reference generator (data.cpp:124-268): the same
// random-call sequence, geometry, false-edge candidate rule, 90th-percentile
// distance cut, shuffle, truncation, canonical edge order and features, so
// the produced EventGraph is bit-identical (checked against the compiled
// reference in tests/test_abi.py::test_generator_matches_reference_digest and
// _presets, and at C2 size in tests/test_gpu_bench_parity.py). The one
// algorithmic change is the
// false-edge candidate search: the reference scans all pairs of adjacent
// layers (O(|L_i|·|L_{i+1}|), 3 GB and 30 s at 120k hits); here each inner hit
// binary-searches the phi window of the phi-sorted outer layer and tests the
// exact predicate only on that window, visiting candidates in the same order.
#include <algorithm>
#include <cmath>
#include <numbers>
#include <vector>

#include "hitgnn/core.hpp"

namespace hitgnn {

namespace {

constexpr double kInnerRadius = 1.0;
constexpr double kLayerGap = 1.0;
constexpr double kMaxCurvature = 0.10;
constexpr double kMaxZSlope = 0.5;
constexpr double kPhiNoise = 0.01;
constexpr double kZNoise = 0.02;
constexpr double kPhiWindow = 0.45;
constexpr double kZWindow = 1.1;
constexpr double kCandidatePercentile = 0.9;
constexpr double kTwoPi = 2.0 * std::numbers::pi;

struct Hit {
    double r, phi, z;
    Index layer;
    Index track;  // -1: noise
};

double wrap(double a) {
    while (a > std::numbers::pi) a -= kTwoPi;
    while (a < -std::numbers::pi) a += kTwoPi;
    return a;
}

double distance(const Hit& a, const Hit& b) {
    const double xa = a.r * std::cos(a.phi), ya = a.r * std::sin(a.phi);
    const double xb = b.r * std::cos(b.phi), yb = b.r * std::sin(b.phi);
    const double dz = a.z - b.z;
    return std::sqrt((xa - xb) * (xa - xb) + (ya - yb) * (ya - yb) + dz * dz);
}

struct Cand {
    std::int32_t src, dst;
    double dist;
};

}  // namespace

EventGraph generate_event(const GenConfig& cfg, std::uint64_t event_id) {
    return generate_event_windowed(cfg, event_id, kPhiWindow);
}

// phi_window == kPhiWindow: the reference generator. A narrower window is the
// scalable variant for events the reference cannot generate (SURVEY.md §8(d)
// C4: ~1M hits): the candidate count per inner hit, and with it the cost,
// stays constant as the layers fill up, so generation is linear in the hits.
EventGraph generate_event_windowed(const GenConfig& cfg, std::uint64_t event_id, double phi_window) {
    cfg.validate();
    if (!(phi_window > 0.0 && phi_window <= kPhiWindow))
        fail_invalid("generate_event: phi window must be in (0, 0.45]");
    Rng rng(Rng::derive(cfg.seed, {0x6576656e74ULL, event_id}));
    const double r_outer = kInnerRadius + kLayerGap * static_cast<double>(cfg.detector_layers - 1);

    std::vector<Hit> hits;
    std::vector<std::pair<std::int32_t, std::int32_t>> true_pairs;
    for (Index t = 0; t < cfg.n_tracks; ++t) {
        const Index len = cfg.hits_min + static_cast<Index>(rng.bounded(
                                             static_cast<std::uint64_t>(cfg.hits_max - cfg.hits_min + 1)));
        const Index first = static_cast<Index>(
            rng.bounded(static_cast<std::uint64_t>(cfg.detector_layers - len + 1)));
        const double phi0 = rng.uniform(0.0, kTwoPi);
        const double curv = rng.uniform(-kMaxCurvature, kMaxCurvature);
        const double slope = rng.uniform(-kMaxZSlope, kMaxZSlope);
        const double z0 = rng.uniform(-0.5, 0.5);
        for (Index j = 0; j < len; ++j) {
            Hit h{};
            h.layer = first + j;
            h.r = kInnerRadius + kLayerGap * static_cast<double>(h.layer);
            h.phi = wrap(phi0 + curv * static_cast<double>(j) + kPhiNoise * rng.normal());
            h.z = z0 + slope * h.r + kZNoise * rng.normal();
            h.track = t;
            hits.push_back(h);
            if (j > 0) {
                const auto last = static_cast<std::int32_t>(hits.size()) - 1;
                true_pairs.emplace_back(last - 1, last);
            }
        }
    }
    const double z_half = kMaxZSlope * r_outer + 0.5;
    for (Index i = 0; i < cfg.noise_hits; ++i) {
        Hit h{};
        h.layer = static_cast<Index>(rng.bounded(static_cast<std::uint64_t>(cfg.detector_layers)));
        h.r = kInnerRadius + kLayerGap * static_cast<double>(h.layer);
        h.phi = rng.uniform(-std::numbers::pi, std::numbers::pi);
        h.z = rng.uniform(-z_half, z_half);
        h.track = -1;
        hits.push_back(h);
    }
    const Index n = static_cast<Index>(hits.size());

    std::vector<Index> new_id(static_cast<std::size_t>(n));
    for (Index i = 0; i < n; ++i) new_id[i] = i;
    for (Index i = n - 1; i > 0; --i)
        std::swap(new_id[i], new_id[static_cast<Index>(rng.bounded(static_cast<std::uint64_t>(i) + 1))]);

    std::vector<std::vector<Index>> by_layer(static_cast<std::size_t>(cfg.detector_layers));
    for (Index i = 0; i < n; ++i) by_layer[hits[i].layer].push_back(i);
    for (auto& L : by_layer)
        std::sort(L.begin(), L.end(), [&](Index a, Index b) { return hits[a].phi < hits[b].phi; });

    // Candidate sweep. For inner hit u the admissible outer phis form up to
    // three intervals of the sorted outer layer (the direct window and its
    // images across ±pi); their union is visited in index order, so the
    // candidate sequence equals the reference's full scan.
    std::vector<Cand> cand;
    constexpr double kSlack = 1e-9;
    for (Index layer = 0; layer + 1 < cfg.detector_layers; ++layer) {
        const auto& inner = by_layer[layer];
        const auto& outer = by_layer[layer + 1];
        std::vector<double> ophi(outer.size());
        for (std::size_t i = 0; i < outer.size(); ++i) ophi[i] = hits[outer[i]].phi;
        auto index_range = [&](double lo, double hi) {
            const auto b = std::lower_bound(ophi.begin(), ophi.end(), lo) - ophi.begin();
            const auto e = std::upper_bound(ophi.begin(), ophi.end(), hi) - ophi.begin();
            return std::pair<std::ptrdiff_t, std::ptrdiff_t>(b, std::max(b, e));
        };
        for (Index u : inner) {
            const Hit& hu = hits[u];
            const double w = phi_window + kSlack;
            std::pair<std::ptrdiff_t, std::ptrdiff_t> iv[3] = {
                index_range(hu.phi - w, hu.phi + w),
                index_range(hu.phi - w + kTwoPi, hu.phi + w + kTwoPi),
                index_range(hu.phi - w - kTwoPi, hu.phi + w - kTwoPi)};
            std::sort(std::begin(iv), std::end(iv));
            std::ptrdiff_t done = 0;
            for (auto [b, e] : iv) {
                for (std::ptrdiff_t i = std::max(b, done); i < e; ++i) {
                    const Index v = outer[static_cast<std::size_t>(i)];
                    const Hit& hv = hits[v];
                    if (hu.track >= 0 && hu.track == hv.track) continue;
                    if (std::abs(wrap(hv.phi - hu.phi)) > phi_window) continue;
                    if (std::abs(hv.z - hu.z) > kZWindow) continue;
                    cand.push_back({static_cast<std::int32_t>(u), static_cast<std::int32_t>(v), distance(hu, hv)});
                }
                done = std::max(done, e);
            }
        }
    }

    const auto n_true = static_cast<Index>(true_pairs.size());
    const auto n_false = static_cast<Index>(std::llround(cfg.false_edge_factor * static_cast<double>(n_true)));
    if (!cand.empty()) {
        std::vector<double> d(cand.size());
        for (std::size_t i = 0; i < cand.size(); ++i) d[i] = cand[i].dist;
        const auto cut = static_cast<std::size_t>(kCandidatePercentile * static_cast<double>(d.size() - 1));
        std::nth_element(d.begin(), d.begin() + static_cast<std::ptrdiff_t>(cut), d.end());
        const double thr = d[cut];
        std::erase_if(cand, [&](const Cand& c) { return c.dist > thr; });
    }
    for (std::size_t i = cand.size(); i > 1; --i)
        std::swap(cand[i - 1], cand[static_cast<std::size_t>(rng.bounded(i))]);
    if (static_cast<Index>(cand.size()) > n_false) cand.resize(static_cast<std::size_t>(n_false));

    struct Rec {
        Index src, dst;
        std::int32_t gsrc, gdst;
        std::uint8_t label;
    };
    std::vector<Rec> recs;
    recs.reserve(true_pairs.size() + cand.size());
    for (auto [u, v] : true_pairs) recs.push_back({new_id[u], new_id[v], u, v, 1});
    for (const Cand& c : cand) recs.push_back({new_id[c.src], new_id[c.dst], c.src, c.dst, 0});
    std::sort(recs.begin(), recs.end(),
              [](const Rec& a, const Rec& b) { return a.src != b.src ? a.src < b.src : a.dst < b.dst; });

    EventGraph ev;
    ev.event_id = event_id;
    ev.n = n;
    ev.edges.n_rows = ev.edges.n_cols = n;
    ev.node_features = DenseMatrix(n, cfg.f_v);
    ev.edge_features = DenseMatrix(static_cast<Index>(recs.size()), cfg.f_e);
    for (Index i = 0; i < n; ++i) {
        const Hit& h = hits[i];
        const double ch[8] = {h.r * std::cos(h.phi) / r_outer,
                              h.r * std::sin(h.phi) / r_outer,
                              h.z / r_outer,
                              h.r / r_outer,
                              std::cos(h.phi),
                              std::sin(h.phi),
                              static_cast<double>(h.layer) / static_cast<double>(cfg.detector_layers),
                              h.z / std::max(h.r, 1e-9)};
        double* row = ev.node_features.row_ptr(new_id[i]);
        for (Index c = 0; c < cfg.f_v; ++c) row[c] = c < 8 ? ch[c] : 0.1 * rng.normal();
    }
    ev.edges.entries.reserve(recs.size());
    ev.labels.reserve(recs.size());
    for (std::size_t i = 0; i < recs.size(); ++i) {
        const Rec& rc = recs[i];
        ev.edges.entries.push_back({rc.src, rc.dst, 1.0});
        ev.labels.push_back(rc.label);
        const Hit& s = hits[rc.gsrc];
        const Hit& t = hits[rc.gdst];
        const double dphi = wrap(t.phi - s.phi), dz = t.z - s.z, dr = t.r - s.r;
        const double ch[6] = {dphi, dz, dr, distance(s, t), dphi / std::max(dr, 1e-9), dz / std::max(dr, 1e-9)};
        double* row = ev.edge_features.row_ptr(static_cast<Index>(i));
        for (Index c = 0; c < cfg.f_e; ++c) row[c] = c < 6 ? ch[c] : 0.1 * rng.normal();
    }
    ev.validate();
    return ev;
}

}  // namespace hitgnn
