// tools.cpp — extern "C" wrappers (include/hgs_tools.h) for Python harnesses.
#include <algorithm>
#include <chrono>
#include <memory>
#include <string>

#include "hgs_tools.h"
#include "hitgnn/core.hpp"
#include "../hgs_rng.cuh"

struct hgs_frontiers {
    std::vector<std::vector<int64_t>> a[5];  // q_ci, f_rp, f_ci, p_rp, p_ci per level
    std::vector<std::vector<double>> p_val;
};

struct hgs_event {
    hitgnn::EventGraph ev;
    hitgnn::CsrMatrix a;
};

namespace {
thread_local std::string g_tools_err;
}

extern "C" {

const char* hgs_tools_last_error(void) { return g_tools_err.c_str(); }

// End-to-end timing of the C++ drop-in: host arrays in, the reference's
// std::vector<SampledBatch> (with gathered features) out, wall clock per rep.
//   mode 0: gpu::DeviceEvent::bulk_shadow(batches, cfg, source, gather = true)
//   mode 1: the reference trainer's unmodified two lines (trainer.cpp:457-458):
//           bulk_shadow(make_edge_id_matrix(event), chunk, cfg, source) and
//           gather_features(batch, event) per batch, served by the
//           resident-graph cache
//   mode 2: bench-sampling's bulk leg (cli.cpp:411-418): bulk_shadow only
//   mode 3: bench-sampling's sequential leg (cli.cpp:419-431): one
//           shadow_reference call per batch, each on its batch's seeds
// Each rep builds a fresh PerRootChoiceSource from the seeds, as the trainer
// does (trainer.cpp:453). ve[0..1] = V, E of the last rep.
int hgs_dropin_time(int64_t n, const int64_t* rp, const int64_t* ci, const double* nf, int64_t f_v,
                    const double* ef, int64_t f_e, const uint8_t* lab, const int64_t* roots,
                    const int64_t* boff, int64_t k, const uint64_t* seeds, int64_t depth, int64_t fanout,
                    int32_t mode, int32_t warmup, int32_t reps, double* seconds, int64_t* ve) {
    try {
        hitgnn::EventGraph ev;
        ev.n = n;
        ev.edges = hitgnn::CooMatrix(n, n);
        const int64_t m = rp[n];
        ev.edges.entries.resize(static_cast<size_t>(m));
        for (int64_t u = 0; u < n; ++u)
            for (int64_t t = rp[u]; t < rp[u + 1]; ++t) ev.edges.entries[t] = {u, ci[t], 1.0};
        ev.node_features = hitgnn::DenseMatrix(n, f_v, std::vector<double>(nf, nf + n * f_v));
        ev.edge_features = hitgnn::DenseMatrix(m, f_e, std::vector<double>(ef, ef + m * f_e));
        ev.labels.assign(lab, lab + m);
        const hitgnn::CsrMatrix a = hitgnn::make_edge_id_matrix(ev);
        std::vector<std::vector<hitgnn::Index>> batches(static_cast<size_t>(k));
        for (int64_t b = 0; b < k; ++b) batches[b].assign(roots + boff[b], roots + boff[b + 1]);
        const std::vector<uint64_t> sv(seeds, seeds + boff[k]);
        hitgnn::SamplerConfig cfg;
        cfg.depth = depth;
        cfg.fanout = fanout;
        cfg.batch_size = k > 0 ? boff[1] - boff[0] : 1;
        cfg.bulk_batches = std::max<int64_t>(k, 1);
        std::unique_ptr<hitgnn::gpu::DeviceEvent> dev;
        if (mode == 0) dev = std::make_unique<hitgnn::gpu::DeviceEvent>(ev);
        for (int32_t i = 0; i < warmup + reps; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            hitgnn::PerRootChoiceSource src(sv);
            std::vector<hitgnn::SampledBatch> out;
            if (mode == 0) {
                out = dev->bulk_shadow(batches, cfg, src, true);
            } else if (mode == 1) {
                out = hitgnn::bulk_shadow(a, batches, cfg, src);
                for (auto& sb : out) hitgnn::gather_features(sb, ev);
            } else if (mode == 2) {
                out = hitgnn::bulk_shadow(a, batches, cfg, src);
            } else {
                for (int64_t b = 0; b < k; ++b) {
                    hitgnn::PerRootChoiceSource one(std::vector<uint64_t>(seeds + boff[b], seeds + boff[b + 1]));
                    out.push_back(hitgnn::shadow_reference(a, batches[b], cfg, one));
                }
            }
            const auto t1 = std::chrono::steady_clock::now();
            if (i >= warmup) seconds[i - warmup] = std::chrono::duration<double>(t1 - t0).count();
            int64_t V = 0, E = 0;
            for (const auto& sb : out) {
                V += sb.n_vertices();
                E += sb.n_edges();
            }
            ve[0] = V;
            ve[1] = E;
        }
        return 0;
    } catch (const std::exception& e) {
        g_tools_err = e.what();
        return 1;
    }
}

int hgs_generate_event(int64_t n_tracks, int64_t hits_min, int64_t hits_max, int64_t layers,
                       int64_t noise_hits, double false_edge_factor, int64_t f_v, int64_t f_e,
                       uint64_t seed, uint64_t event_id, hgs_event** out) {
    return hgs_generate_event_windowed(n_tracks, hits_min, hits_max, layers, noise_hits, false_edge_factor, f_v,
                                       f_e, seed, event_id, 0.45, out);
}

int hgs_generate_event_windowed(int64_t n_tracks, int64_t hits_min, int64_t hits_max, int64_t layers,
                                int64_t noise_hits, double false_edge_factor, int64_t f_v, int64_t f_e,
                                uint64_t seed, uint64_t event_id, double phi_window, hgs_event** out) {
    try {
        hitgnn::GenConfig cfg;
        cfg.n_tracks = n_tracks;
        cfg.hits_min = hits_min;
        cfg.hits_max = hits_max;
        cfg.detector_layers = layers;
        cfg.noise_hits = noise_hits;
        cfg.false_edge_factor = false_edge_factor;
        cfg.f_v = f_v;
        cfg.f_e = f_e;
        cfg.seed = seed;
        auto* e = new hgs_event;
        e->ev = hitgnn::generate_event_windowed(cfg, event_id, phi_window);
        e->a = hitgnn::make_edge_id_matrix(e->ev);
        *out = e;
        return 0;
    } catch (const std::exception& ex) {
        g_tools_err = ex.what();
        return 1;
    }
}

void hgs_event_sizes(const hgs_event* e, int64_t* s) {
    s[0] = e->ev.n;
    s[1] = e->ev.m();
    s[2] = e->ev.node_features.cols;
    s[3] = e->ev.edge_features.cols;
}

void hgs_event_copy(const hgs_event* e, int64_t* rp, int64_t* ci, double* nf, double* ef, uint8_t* lab) {
    if (rp) std::copy(e->a.row_ptr.begin(), e->a.row_ptr.end(), rp);
    if (ci) std::copy(e->a.col_idx.begin(), e->a.col_idx.end(), ci);
    if (nf) std::copy(e->ev.node_features.data.begin(), e->ev.node_features.data.end(), nf);
    if (ef) std::copy(e->ev.edge_features.data.begin(), e->ev.edge_features.data.end(), ef);
    if (lab) std::copy(e->ev.labels.begin(), e->ev.labels.end(), lab);
}

void hgs_event_free(hgs_event* e) { delete e; }

int64_t hgs_epoch_root_batches(int64_t n, int64_t b, uint64_t rng_seed, int64_t* perm) {
    hitgnn::Rng rng(rng_seed);
    const auto batches = hitgnn::epoch_root_batches(n, b, rng);
    int64_t w = 0;
    for (const auto& bb : batches)
        for (auto v : bb) perm[w++] = v;
    return static_cast<int64_t>(batches.size());
}

void hgs_derive_grid(uint64_t seed, const uint64_t* prefix, int32_t plen, int64_t k, int64_t b,
                     uint64_t* seeds) {
    std::vector<uint64_t> path(prefix, prefix + plen);
    path.push_back(0);
    path.push_back(0);
    for (int64_t bi = 0; bi < k; ++bi)
        for (int64_t pos = 0; pos < b; ++pos) {
            path[plen] = static_cast<uint64_t>(bi);
            path[plen + 1] = static_cast<uint64_t>(pos);
            seeds[bi * b + pos] = hgs::derive_seed(seed, path.data(), plen + 2);
        }
}

// hitgnn::bulk_shadow (the GPU drop-in) with a FrontierObserver recording
// every level's FrontierSet (sampler.hpp:52-58); per-root seeds, rng 0 =
// PerRootChoiceSource, 1 = PhiloxChoiceSource.
int hgs_tools_frontiers(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci, const double* values,
                        const int64_t* roots, const int64_t* batch_off, int64_t n_batches, const uint64_t* seeds,
                        int32_t rng, int64_t depth, int64_t fanout, int32_t symmetrize, hgs_frontiers** out) {
    try {
        hitgnn::CsrMatrix a(n_rows, n_cols);
        a.row_ptr.assign(rp, rp + n_rows + 1);
        a.col_idx.assign(ci, ci + rp[n_rows]);
        a.values.resize(a.col_idx.size());
        for (size_t k = 0; k < a.values.size(); ++k) a.values[k] = values ? values[k] : double(k) + 1.0;
        std::vector<std::vector<hitgnn::Index>> batches;
        for (int64_t b = 0; b < n_batches; ++b) batches.emplace_back(roots + batch_off[b], roots + batch_off[b + 1]);
        std::vector<uint64_t> sd(seeds, seeds + batch_off[n_batches]);
        hitgnn::SamplerConfig cfg;
        cfg.depth = depth;
        cfg.fanout = fanout;
        cfg.symmetrize = symmetrize != 0;
        auto* f = new hgs_frontiers;
        hitgnn::FrontierObserver obs = [&](hitgnn::Index, const hitgnn::FrontierSet& fs) {
            f->a[0].push_back(fs.q.col_idx);
            f->a[1].push_back(fs.f.row_ptr);
            f->a[2].push_back(fs.f.col_idx);
            f->a[3].push_back(fs.p.row_ptr);
            f->a[4].push_back(fs.p.col_idx);
            f->p_val.push_back(fs.p.values);
        };
        try {
            if (rng == 1) {
                hitgnn::PhiloxChoiceSource src(std::move(sd));
                hitgnn::bulk_shadow(a, batches, cfg, src, obs);
            } else {
                hitgnn::PerRootChoiceSource src(std::move(sd));
                hitgnn::bulk_shadow(a, batches, cfg, src, obs);
            }
        } catch (...) {
            delete f;
            throw;
        }
        *out = f;
        return 0;
    } catch (const std::exception& ex) {
        g_tools_err = ex.what();
        return 1;
    }
}

int64_t hgs_tools_frontiers_levels(const hgs_frontiers* f) { return static_cast<int64_t>(f->p_val.size()); }

int64_t hgs_tools_frontier_array(const hgs_frontiers* f, int64_t level, int32_t which, void* out) {
    if (which == 5) {
        const auto& d = f->p_val[level];
        if (out) std::copy(d.begin(), d.end(), static_cast<double*>(out));
        return static_cast<int64_t>(d.size());
    }
    const auto& v = f->a[which][level];
    if (out) std::copy(v.begin(), v.end(), static_cast<int64_t*>(out));
    return static_cast<int64_t>(v.size());
}

void hgs_tools_frontiers_free(hgs_frontiers* f) { delete f; }

}  // extern "C"
