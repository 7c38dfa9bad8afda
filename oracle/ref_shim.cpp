// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper around the UNMODIFIED reference sampler, compiled from
// /root/reference/proj/src/{rng,sparse,sampler,data}.cpp in place by
// oracle/Makefile with -Dhitgnn=hitgnn_ref (so it can sit beside the product
// namespace). Nothing here re-implements the reference algorithm: every
// sampled result comes from hitgnn_ref::bulk_shadow / shadow_reference /
// gather_features / generate_event. Used to
//   * pin the C restatement (hgs_oracle.c) and generate tests/golden/,
//   * time the reference CPU sampler for bench.py's cpu_baseline and
//     `--impl reference` legs (kind "reference").
// The one addition is PhiloxSource, a ChoiceSource implementing the Philox
// decision stream of SURVEY.md Appendix A.3 on top of the reference's own
// interface (rng.hpp:48-54), so the Philox-mode oracle is the unmodified
// reference bulk_shadow fed by that source.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hitgnn/data.hpp"
#include "hitgnn/rng.hpp"
#include "hitgnn/sampler.hpp"
#include "hitgnn/sparse.hpp"

extern "C" {
#include "hgs_oracle.h"
}

namespace R = hitgnn_ref;

namespace {

class PhiloxSource final : public R::ChoiceSource {
public:
    explicit PhiloxSource(std::vector<std::uint64_t> seeds)
        : seeds_(std::move(seeds)), decisions_(seeds_.size(), 0) {}
    void begin_root(std::uint64_t r) override {
        if (r >= seeds_.size()) throw std::invalid_argument("PhiloxSource: root ordinal out of range");
        cur_ = r;
    }
    std::vector<std::uint32_t> choose(std::uint32_t n, std::uint32_t k) override {
        if (k > n) k = n;
        const std::uint64_t seed = seeds_[cur_];
        const std::uint32_t key[2] = {static_cast<std::uint32_t>(seed),
                                      static_cast<std::uint32_t>(seed >> 32)};
        const std::uint32_t dec = decisions_[cur_]++;
        std::vector<std::uint32_t> a(n);
        std::iota(a.begin(), a.end(), 0u);
        for (std::uint32_t i = 0; i < k; ++i) {
            const std::uint64_t m = n - i;
            const std::uint64_t lim = (0ULL - m) % m;
            std::uint64_t x = 0;
            for (std::uint32_t att = 0;; ++att) {
                const std::uint32_t ctr[4] = {dec, i, att, 0x43484f53u};
                std::uint32_t o[4];
                or_philox4x32_10(ctr, key, o);
                x = (static_cast<std::uint64_t>(o[1]) << 32) | o[0];
                if (x >= lim) break;
            }
            std::swap(a[i], a[i + static_cast<std::uint32_t>(x % m)]);
        }
        std::vector<std::uint32_t> out(a.begin(), a.begin() + k);
        std::sort(out.begin(), out.end());
        return out;
    }

private:
    std::vector<std::uint64_t> seeds_;
    std::vector<std::uint32_t> decisions_;
    std::size_t cur_ = 0;
};

struct Result {
    std::int64_t k = 0, R = 0, V = 0, E = 0, f_v = 0, f_e = 0, gathered = 0;
    std::vector<std::int64_t> bvoff, beoff, comp_off, l2g, roots_local, e_row, e_col, e_gid;
    std::vector<double> e_val, xv, ye;
    std::vector<std::uint8_t> lab;
    std::vector<std::vector<std::int64_t>> level_q;  // observer: Q col ids per level
    std::vector<std::int64_t> level_f_nnz;
    // observer, full: per level F (row_ptr, col_idx) and P (row_ptr, col_idx, values)
    std::vector<std::vector<std::int64_t>> level_f_rp, level_f_ci, level_p_rp, level_p_ci;
    std::vector<std::vector<double>> level_p_val;
};

void put_err(char* err, int len, const std::string& s) {
    if (err && len > 0) std::snprintf(err, static_cast<std::size_t>(len), "%s", s.c_str());
}

R::CsrMatrix make_csr(std::int64_t n_rows, std::int64_t n_cols, const std::int64_t* rp,
                      const std::int64_t* ci, const double* values) {
    R::CsrMatrix a(n_rows, n_cols);
    const std::int64_t nnz = rp[n_rows];
    a.row_ptr.assign(rp, rp + n_rows + 1);
    a.col_idx.assign(ci, ci + nnz);
    a.values.resize(static_cast<std::size_t>(nnz));
    for (std::int64_t k = 0; k < nnz; ++k) a.values[k] = values ? values[k] : double(k) + 1.0;
    return a;
}

R::EventGraph make_event(std::int64_t n, const std::int64_t* rp, const std::int64_t* ci,
                         const double* nf, std::int64_t f_v, const double* ef,
                         std::int64_t f_e, const std::uint8_t* lab) {
    R::EventGraph ev;
    ev.n = n;
    ev.edges.n_rows = ev.edges.n_cols = n;
    const std::int64_t m = rp[n];
    ev.edges.entries.reserve(static_cast<std::size_t>(m));
    for (std::int64_t u = 0; u < n; ++u)
        for (std::int64_t k = rp[u]; k < rp[u + 1]; ++k) ev.edges.entries.push_back({u, ci[k], 1.0});
    ev.node_features = R::DenseMatrix(n, f_v, std::vector<double>(nf, nf + n * f_v));
    ev.edge_features = R::DenseMatrix(m, f_e, std::vector<double>(ef, ef + m * f_e));
    ev.labels.assign(lab, lab + m);
    return ev;
}

void flatten(Result& res, std::vector<R::SampledBatch>& out, bool values_are_ids) {
    res.k = static_cast<std::int64_t>(out.size());
    res.bvoff.push_back(0);
    res.beoff.push_back(0);
    for (auto& sb : out) {
        const std::int64_t vb = res.V, eb = res.E;
        for (auto c : sb.component_offsets) res.comp_off.push_back(c);
        for (auto v : sb.local_to_global) res.l2g.push_back(v);
        for (auto r : sb.roots_local) res.roots_local.push_back(r);
        std::size_t i = 0;
        for (auto& e : sb.adjacency.entries) {
            res.e_row.push_back(e.row);
            res.e_col.push_back(e.col);
            res.e_val.push_back(e.value);
            if (!sb.edge_global_ids.empty()) res.e_gid.push_back(sb.edge_global_ids[i]);
            else res.e_gid.push_back(values_are_ids ? std::llround(e.value) - 1 : -1);
            ++i;
        }
        if (res.gathered) {
            res.xv.insert(res.xv.end(), sb.node_features.data.begin(), sb.node_features.data.end());
            res.ye.insert(res.ye.end(), sb.edge_features.data.begin(), sb.edge_features.data.end());
            res.lab.insert(res.lab.end(), sb.edge_labels.begin(), sb.edge_labels.end());
        }
        res.R += sb.n_components();
        res.V = vb + static_cast<std::int64_t>(sb.local_to_global.size());
        res.E = eb + sb.n_edges();
        res.bvoff.push_back(res.V);
        res.beoff.push_back(res.E);
    }
}

std::vector<std::vector<R::Index>> split_batches(const std::int64_t* roots,
                                                 const std::int64_t* batch_off,
                                                 std::int64_t k) {
    std::vector<std::vector<R::Index>> b(static_cast<std::size_t>(k));
    for (std::int64_t i = 0; i < k; ++i) b[i].assign(roots + batch_off[i], roots + batch_off[i + 1]);
    return b;
}

}  // namespace

extern "C" {

// ---- RNG known answers -------------------------------------------------
void ref_rng_first(std::uint64_t seed, std::int64_t n, std::uint64_t* out) {
    R::Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
std::uint64_t ref_derive(std::uint64_t seed, const std::uint64_t* path, int len) {
    // derive takes an initializer_list; fold the same recurrence through
    // nested calls is not possible, so dispatch on length (tests use <= 6).
    switch (len) {
        case 0: return R::Rng::derive(seed, {});
        case 1: return R::Rng::derive(seed, {path[0]});
        case 2: return R::Rng::derive(seed, {path[0], path[1]});
        case 3: return R::Rng::derive(seed, {path[0], path[1], path[2]});
        case 4: return R::Rng::derive(seed, {path[0], path[1], path[2], path[3]});
        case 5: return R::Rng::derive(seed, {path[0], path[1], path[2], path[3], path[4]});
        default: return R::Rng::derive(seed, {path[0], path[1], path[2], path[3], path[4], path[5]});
    }
}
void ref_bounded_seq(std::uint64_t seed, const std::uint64_t* bounds, std::int64_t n,
                     std::uint64_t* out) {
    R::Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.bounded(bounds[i]);
}
// RandomChoiceSource(seed): successive choose(n_i, k_i); positions appended.
std::int64_t ref_choose_seq(std::uint64_t seed, const std::uint32_t* ns, const std::uint32_t* ks,
                            std::int64_t calls, std::uint32_t* out) {
    R::RandomChoiceSource src(seed);
    std::int64_t w = 0;
    for (std::int64_t i = 0; i < calls; ++i)
        for (auto p : src.choose(ns[i], ks[i])) out[w++] = p;
    return w;
}
std::int64_t ref_epoch_root_batches(std::int64_t n, std::int64_t b, std::uint64_t seed,
                                    std::int64_t* flat) {
    R::Rng r(seed);
    const auto batches = R::epoch_root_batches(n, b, r);
    std::int64_t w = 0;
    for (const auto& bb : batches)
        for (auto v : bb) flat[w++] = v;
    return static_cast<std::int64_t>(batches.size());
}

// ---- symmetrize_pattern ---------------------------------------------------
std::int64_t ref_symmetrize(std::int64_t n, const std::int64_t* rp, const std::int64_t* ci,
                            std::int64_t* out_rp, std::int64_t* out_ci) {
    const R::CsrMatrix w = R::symmetrize_pattern(make_csr(n, n, rp, ci, nullptr));
    std::copy(w.row_ptr.begin(), w.row_ptr.end(), out_rp);
    std::copy(w.col_idx.begin(), w.col_idx.end(), out_ci);
    return w.nnz();
}

// ---- synthetic event generator (data.cpp:124-268) --------------------------
void* ref_generate_event(std::int64_t n_tracks, std::int64_t hits_min, std::int64_t hits_max,
                         std::int64_t layers, std::int64_t noise, double false_factor,
                         std::int64_t f_v, std::int64_t f_e, std::uint64_t seed,
                         std::uint64_t event_id) {
    R::GenConfig cfg;
    cfg.n_tracks = n_tracks; cfg.hits_min = hits_min; cfg.hits_max = hits_max;
    cfg.detector_layers = layers; cfg.noise_hits = noise; cfg.false_edge_factor = false_factor;
    cfg.f_v = f_v; cfg.f_e = f_e; cfg.seed = seed;
    return new R::EventGraph(R::generate_event(cfg, event_id));
}
void ref_event_sizes(const void* h, std::int64_t* out) {
    const auto* ev = static_cast<const R::EventGraph*>(h);
    out[0] = ev->n; out[1] = ev->m(); out[2] = ev->node_features.cols; out[3] = ev->edge_features.cols;
}
void ref_event_copy(const void* h, std::int64_t* rp, std::int64_t* ci, double* nf, double* ef,
                    std::uint8_t* lab) {
    const auto* ev = static_cast<const R::EventGraph*>(h);
    const R::CsrMatrix a = R::make_edge_id_matrix(*ev);
    std::copy(a.row_ptr.begin(), a.row_ptr.end(), rp);
    std::copy(a.col_idx.begin(), a.col_idx.end(), ci);
    std::copy(ev->node_features.data.begin(), ev->node_features.data.end(), nf);
    std::copy(ev->edge_features.data.begin(), ev->edge_features.data.end(), ef);
    std::copy(ev->labels.begin(), ev->labels.end(), lab);
}
void ref_event_free(void* h) { delete static_cast<R::EventGraph*>(h); }

// ---- the sampler ---------------------------------------------------------
// mode: 0 = bulk_shadow over all batches, 1 = one shadow_reference per batch
// (seed slices), 2 = bulk_shadow with a FrontierObserver recording Q per level.
void* ref_bulk_shadow(std::int64_t n_rows, std::int64_t n_cols, const std::int64_t* rp,
                      const std::int64_t* ci, const double* values, const std::int64_t* roots,
                      const std::int64_t* batch_off, std::int64_t n_batches,
                      const std::uint64_t* seeds, int rng_kind, std::int64_t depth,
                      std::int64_t fanout, int symmetrize, const double* nf, std::int64_t f_v,
                      const double* ef, std::int64_t f_e, const std::uint8_t* lab, int mode,
                      char* err, int errlen) {
    auto* res = new Result;
    try {
        const R::CsrMatrix a = make_csr(n_rows, n_cols, rp, ci, values);
        const auto batches = split_batches(roots, batch_off, n_batches);
        const std::int64_t nr = batch_off[n_batches];
        std::vector<std::uint64_t> sd(seeds, seeds + nr);
        R::SamplerConfig cfg;
        cfg.depth = depth; cfg.fanout = fanout; cfg.symmetrize = symmetrize != 0;
        cfg.bulk_batches = std::max<std::int64_t>(1, n_batches);
        std::vector<R::SampledBatch> out;
        auto make_src = [&](std::vector<std::uint64_t> s) -> std::unique_ptr<R::ChoiceSource> {
            if (rng_kind == 0) return std::make_unique<R::PerRootChoiceSource>(std::move(s));
            return std::make_unique<PhiloxSource>(std::move(s));
        };
        if (mode == 1) {
            for (std::int64_t b = 0; b < n_batches; ++b) {
                auto src = make_src(std::vector<std::uint64_t>(sd.begin() + batch_off[b],
                                                               sd.begin() + batch_off[b + 1]));
                out.push_back(R::shadow_reference(a, batches[b], cfg, *src));
            }
        } else {
            auto src = make_src(sd);
            R::FrontierObserver obs;
            if (mode == 2)
                obs = [&](R::Index, const R::FrontierSet& fs) {
                    res->level_q.push_back(fs.q.col_idx);
                    res->level_f_nnz.push_back(fs.f.nnz());
                    res->level_f_rp.push_back(fs.f.row_ptr);
                    res->level_f_ci.push_back(fs.f.col_idx);
                    res->level_p_rp.push_back(fs.p.row_ptr);
                    res->level_p_ci.push_back(fs.p.col_idx);
                    res->level_p_val.push_back(fs.p.values);
                };
            out = R::bulk_shadow(a, batches, cfg, *src, obs);
        }
        if (nf && ef && lab) {
            const R::EventGraph ev = make_event(n_rows, rp, ci, nf, f_v, ef, f_e, lab);
            for (auto& sb : out) R::gather_features(sb, ev);
            res->gathered = 1; res->f_v = f_v; res->f_e = f_e;
        }
        flatten(*res, out, values == nullptr);
    } catch (const std::invalid_argument& e) {
        put_err(err, errlen, std::string("invalid_argument: ") + e.what());
        delete res;
        return nullptr;
    } catch (const std::exception& e) {
        put_err(err, errlen, std::string("runtime_error: ") + e.what());
        delete res;
        return nullptr;
    }
    return res;
}

void ref_result_counts(const void* h, std::int64_t* c) {
    const auto* r = static_cast<const Result*>(h);
    c[0] = r->k; c[1] = r->R; c[2] = r->V; c[3] = r->E; c[4] = r->f_v; c[5] = r->f_e;
    c[6] = r->gathered; c[7] = static_cast<std::int64_t>(r->level_q.size());
}
void ref_result_copy(const void* h, std::int64_t* bvoff, std::int64_t* beoff,
                     std::int64_t* comp_off, std::int64_t* l2g, std::int64_t* roots_local,
                     std::int64_t* e_row, std::int64_t* e_col, std::int64_t* e_gid, double* e_val,
                     double* xv, double* ye, std::uint8_t* lab) {
    const auto* r = static_cast<const Result*>(h);
    auto cp = [](auto* dst, const auto& v) { if (dst) std::copy(v.begin(), v.end(), dst); };
    cp(bvoff, r->bvoff); cp(beoff, r->beoff); cp(comp_off, r->comp_off); cp(l2g, r->l2g);
    cp(roots_local, r->roots_local); cp(e_row, r->e_row); cp(e_col, r->e_col);
    cp(e_gid, r->e_gid); cp(e_val, r->e_val); cp(xv, r->xv); cp(ye, r->ye); cp(lab, r->lab);
}
std::int64_t ref_result_level_size(const void* h, std::int64_t level) {
    return static_cast<std::int64_t>(static_cast<const Result*>(h)->level_q[level].size());
}
void ref_result_level_copy(const void* h, std::int64_t level, std::int64_t* out) {
    const auto& q = static_cast<const Result*>(h)->level_q[level];
    std::copy(q.begin(), q.end(), out);
}
// which: 0 Q col_idx, 1 F row_ptr, 2 F col_idx, 3 P row_ptr, 4 P col_idx
// (int64), 5 P values (double). Returns the length; copies when out != null.
std::int64_t ref_result_level_array(const void* h, std::int64_t level, int which, void* out) {
    const auto* r = static_cast<const Result*>(h);
    const std::vector<std::int64_t>* v = nullptr;
    switch (which) {
        case 0: v = &r->level_q[level]; break;
        case 1: v = &r->level_f_rp[level]; break;
        case 2: v = &r->level_f_ci[level]; break;
        case 3: v = &r->level_p_rp[level]; break;
        case 4: v = &r->level_p_ci[level]; break;
        default: {
            const auto& d = r->level_p_val[level];
            if (out) std::copy(d.begin(), d.end(), static_cast<double*>(out));
            return static_cast<std::int64_t>(d.size());
        }
    }
    if (out) std::copy(v->begin(), v->end(), static_cast<std::int64_t*>(out));
    return static_cast<std::int64_t>(v->size());
}
void ref_result_free(void* h) { delete static_cast<Result*>(h); }

// ---- timing for the CPU baseline -----------------------------------------
// bulk_shadow + gather_features (the trainer's sample_s region,
// trainer.cpp:456-459) over `n_batches` batches, sharded across `threads`
// host threads by contiguous batch ranges, each with its own seed slice.
// Returns wall seconds; total V/E through out_ve.
double ref_time_sample(std::int64_t n, const std::int64_t* rp, const std::int64_t* ci,
                       const double* nf, std::int64_t f_v, const double* ef, std::int64_t f_e,
                       const std::uint8_t* lab, const std::int64_t* roots,
                       const std::int64_t* batch_off, std::int64_t n_batches,
                       const std::uint64_t* seeds, int rng_kind, std::int64_t depth,
                       std::int64_t fanout, int threads, std::int64_t* out_ve) {
    const R::CsrMatrix a = make_csr(n, n, rp, ci, nullptr);
    const R::EventGraph ev = make_event(n, rp, ci, nf, f_v, ef, f_e, lab);
    const auto batches = split_batches(roots, batch_off, n_batches);
    R::SamplerConfig cfg;
    cfg.depth = depth; cfg.fanout = fanout;
    threads = std::max(1, std::min<int>(threads, static_cast<int>(std::max<std::int64_t>(1, n_batches))));
    std::atomic<std::int64_t> V{0}, E{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            const std::int64_t b0 = n_batches * t / threads, b1 = n_batches * (t + 1) / threads;
            if (b1 <= b0) return;
            std::vector<std::vector<R::Index>> mine(batches.begin() + b0, batches.begin() + b1);
            std::vector<std::uint64_t> sd(seeds + batch_off[b0], seeds + batch_off[b1]);
            std::unique_ptr<R::ChoiceSource> src;
            if (rng_kind == 0) src = std::make_unique<R::PerRootChoiceSource>(std::move(sd));
            else src = std::make_unique<PhiloxSource>(std::move(sd));
            R::SamplerConfig c = cfg;
            c.bulk_batches = b1 - b0;
            auto out = R::bulk_shadow(a, mine, c, *src);
            for (auto& sb : out) {
                R::gather_features(sb, ev);
                V += sb.n_vertices();
                E += sb.n_edges();
            }
        });
    }
    for (auto& th : pool) th.join();
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    out_ve[0] = V.load();
    out_ve[1] = E.load();
    return s;
}

}  // extern "C"
