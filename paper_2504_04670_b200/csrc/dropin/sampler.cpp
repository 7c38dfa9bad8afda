// sampler.cpp — hitgnn:: sampler API (sampler.hpp:60-102 of the reference)
// implemented over the C ABI (include/hgs.h). All sampling runs on the GPU;
// this file validates inputs with the reference's error semantics, moves
// inputs/outputs across the host boundary and lays the results out as the
// reference's SampledBatch values.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

#include "hgs.h"
#include "hitgnn/core.hpp"

namespace hitgnn {

namespace {

void check(int rc) {
    if (rc == HGS_OK) return;
    const std::string msg = hgs_last_error();
    if (rc == HGS_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

struct GraphGuard {
    hgs_graph* g = nullptr;
    ~GraphGuard() { if (g) hgs_graph_destroy(g); }
};
struct SampleGuard {
    hgs_sample* s = nullptr;
    ~SampleGuard() { if (s) hgs_sample_destroy(s); }
};

hgs_graph* upload_csr(const CsrMatrix& a, int device, bool with_values) {
    hgs_graph* g = nullptr;
    check(hgs_graph_create(device, a.n_rows, a.n_cols, a.row_ptr.data(), a.col_idx.data(),
                           with_values ? a.values.data() : nullptr, &g));
    return g;
}

bool values_are_ids(const CsrMatrix& a) {
    for (std::size_t k = 0; k < a.values.size(); ++k)
        if (a.values[k] != static_cast<double>(k) + 1.0) return false;
    return true;
}

// Run one bulk call on a resident graph and materialise SampledBatch values.
// values == nullptr: values are edge ids (gid + 1), as make_edge_id_matrix.
// FrontierObserver (sampler.cpp:149-158, 186) from the device's frontiers:
// per level l = 1..d, Q = the level's chosen vertices (one row each, roots in
// order, BFS order within a root), F = per root the canonical set of the
// root and everything touched so far, P = row_normalize(spgemm(Q_{l-1}, walk))
// restated for one-hot rows: the walk row of the parent with zeros dropped,
// each value divided by the row's sequential sum (sparse.cpp:78-144, 193-206).
void emit_frontiers(hgs_graph* g, hgs_sample* s, const CsrMatrix& a, const std::vector<Index>& roots,
                    const SamplerConfig& cfg, const FrontierObserver& observer) {
    const std::size_t R = roots.size();
    const Index d = cfg.depth;
    int64_t stride = 0;
    check(hgs_sample_copy_frontiers(s, nullptr, nullptr, nullptr, &stride));
    std::vector<int32_t> touched(R * static_cast<std::size_t>(stride)), tcount(R),
        lc(R * static_cast<std::size_t>(d + 1));
    check(hgs_sample_copy_frontiers(s, touched.data(), tcount.data(), lc.data(), &stride));
    CsrMatrix walk;
    const CsrMatrix* w = &a;
    if (cfg.symmetrize) {
        int64_t info[8];
        check(hgs_graph_info(g, info));
        walk = CsrMatrix(a.n_rows, a.n_cols);
        walk.col_idx.resize(static_cast<std::size_t>(info[3]));
        check(hgs_graph_walk(g, 1, walk.row_ptr.data(), walk.col_idx.data()));
        walk.values.assign(walk.col_idx.size(), 1.0);
        w = &walk;
    }
    auto level_begin = [&](std::size_t r, Index l) {  // offset of level l in root r's list
        Index off = 0;
        for (Index j = 0; j < l; ++j) off += lc[r * (d + 1) + j];
        return off;
    };
    for (Index level = 1; level <= d; ++level) {
        FrontierSet fs;
        // Q: the level's rows
        Index nq = 0;
        for (std::size_t r = 0; r < R; ++r) nq += lc[r * (d + 1) + level];
        fs.q = CsrMatrix(nq, a.n_cols);
        fs.q.col_idx.reserve(static_cast<std::size_t>(nq));
        for (std::size_t r = 0; r < R; ++r) {
            const Index b = level_begin(r, level), n = lc[r * (d + 1) + level];
            for (Index i = 0; i < n; ++i) fs.q.col_idx.push_back(touched[r * stride + b + i]);
        }
        fs.q.values.assign(fs.q.col_idx.size(), 1.0);
        for (Index i = 0; i < nq; ++i) fs.q.row_ptr[i + 1] = i + 1;
        // F: root + touched through this level, canonical, values 1
        fs.f = CsrMatrix(static_cast<Index>(R), a.n_cols);
        for (std::size_t r = 0; r < R; ++r) {
            const Index end = level_begin(r, level + 1);
            std::vector<Index> row(touched.begin() + r * stride, touched.begin() + r * stride + end);
            if (row.empty()) row.push_back(roots[r]);
            std::sort(row.begin(), row.end());
            row.erase(std::unique(row.begin(), row.end()), row.end());
            fs.f.col_idx.insert(fs.f.col_idx.end(), row.begin(), row.end());
            fs.f.row_ptr[r + 1] = static_cast<Index>(fs.f.col_idx.size());
        }
        fs.f.values.assign(fs.f.col_idx.size(), 1.0);
        // P: one row per frontier row of level-1
        Index np = 0;
        for (std::size_t r = 0; r < R; ++r) np += lc[r * (d + 1) + level - 1];
        fs.p = CsrMatrix(np, a.n_cols);
        Index row = 0;
        for (std::size_t r = 0; r < R; ++r) {
            const Index b = level_begin(r, level - 1), n = lc[r * (d + 1) + level - 1];
            for (Index i = 0; i < n; ++i, ++row) {
                const Index v = touched[r * stride + b + i];
                const std::size_t k0 = fs.p.col_idx.size();
                double sum = 0.0;
                for (Index k = w->row_ptr[v]; k < w->row_ptr[v + 1]; ++k) {
                    const double x = w->values.empty() ? 1.0 : w->values[k];
                    if (x == 0.0) continue;  // spgemm drops exact zeros
                    fs.p.col_idx.push_back(w->col_idx[k]);
                    fs.p.values.push_back(x);
                    sum += x;
                }
                if (sum != 0.0)
                    for (std::size_t k = k0; k < fs.p.values.size(); ++k) fs.p.values[k] /= sum;
                fs.p.row_ptr[row + 1] = static_cast<Index>(fs.p.col_idx.size());
            }
        }
        observer(level, fs);
    }
}

std::vector<SampledBatch> run_bulk(hgs_graph* g, hgs_sample* s,
                                   const std::vector<std::vector<Index>>& batches,
                                   const SamplerConfig& cfg, ChoiceSource& choice, bool gather,
                                   const std::vector<double>* values, Index f_v, Index f_e,
                                   bool seq_walk = false, const FrontierObserver* observer = nullptr,
                                   const CsrMatrix* a_host = nullptr) {
    cfg.validate();
    auto* per_root = dynamic_cast<PerRootChoiceSource*>(&choice);
    auto* philox = dynamic_cast<PhiloxChoiceSource*>(&choice);
    if (!per_root && !philox)
        fail_invalid("bulk_shadow: the GPU sampler needs a PerRootChoiceSource or PhiloxChoiceSource");
    std::vector<Index> roots, boff{0};
    for (const auto& b : batches) {
        roots.insert(roots.end(), b.begin(), b.end());
        boff.push_back(static_cast<Index>(roots.size()));
    }
    const std::size_t R = roots.size();
    const std::size_t have = per_root ? per_root->size() : philox->size();
    if (have < R) {
        if (have == 0 && R > 0)
            fail_invalid(per_root ? "PerRootChoiceSource: no streams configured"
                                  : "PhiloxChoiceSource: no streams configured");
        if (R > 0) fail_invalid(per_root ? "PerRootChoiceSource: root ordinal out of range"
                                         : "PhiloxChoiceSource: root ordinal out of range");
    }
    const std::vector<std::uint64_t>& seeds = per_root ? per_root->seeds() : philox->seeds();
    std::vector<std::uint64_t> state;
    const std::uint64_t* state_ptr = nullptr;
    if (per_root && !per_root->fresh()) {
        state = per_root->states();
        state_ptr = state.data();
    } else if (philox && !philox->fresh()) {
        state.assign(philox->decisions().begin(), philox->decisions().end());
        state_ptr = state.data();
    }
    hgs_config hc{};
    hc.depth = cfg.depth;
    hc.fanout = cfg.fanout;
    hc.batch_size = cfg.batch_size;
    hc.bulk_batches = cfg.bulk_batches;
    hc.symmetrize = cfg.symmetrize ? 1 : 0;
    hc.rng = philox ? HGS_RNG_PHILOX : HGS_RNG_XOSHIRO;
    hc.gather = gather ? 1 : 0;
    hc.flags = (seq_walk ? HGS_FLAG_SEQ_WALK : 0) | (observer ? HGS_FLAG_KEEP_FRONTIERS : 0);
    check(hgs_sample_run(s, &hc, roots.data(), boff.data(), static_cast<int64_t>(batches.size()),
                         seeds.data(), state_ptr));
    int64_t counts[4];
    check(hgs_sample_wait(s, counts));
    const Index V = counts[2], E = counts[3], k = static_cast<Index>(batches.size());

    std::vector<int32_t> bvoff(k + 1), beoff(k + 1), comp(R + k), l2g(V), rl(R), er(E), ec(E), eg(E);
    std::vector<std::uint32_t> draws(R), decisions(R);
    std::vector<double> xv, ye;
    std::vector<std::uint8_t> lab;
    hgs_host_out o{};
    o.batch_voff = bvoff.data(); o.batch_eoff = beoff.data(); o.comp_off = comp.data();
    o.l2g = l2g.data(); o.roots_local = rl.data(); o.e_row = er.data(); o.e_col = ec.data();
    o.e_gid = eg.data(); o.draws = draws.data(); o.decisions = decisions.data();
    if (gather) {
        xv.resize(static_cast<std::size_t>(V * f_v));
        ye.resize(static_cast<std::size_t>(E * f_e));
        lab.resize(static_cast<std::size_t>(E));
        o.xv = xv.data(); o.ye = ye.data(); o.lab = lab.data();
    }
    check(hgs_sample_copy_to_host(s, &o));
    if (per_root) per_root->advance(draws);
    else philox->advance(decisions);
    if (observer) emit_frontiers(g, s, *a_host, roots, cfg, *observer);

    std::vector<SampledBatch> out(static_cast<std::size_t>(k));
    for (Index b = 0; b < k; ++b) {
        SampledBatch& sb = out[b];
        const Index v0 = bvoff[b], v1 = bvoff[b + 1], e0 = beoff[b], e1 = beoff[b + 1];
        const Index r0 = boff[b], r1 = boff[b + 1];
        sb.adjacency.n_rows = sb.adjacency.n_cols = v1 - v0;
        sb.adjacency.entries.resize(static_cast<std::size_t>(e1 - e0));
        for (Index e = e0; e < e1; ++e) {
            double val = 1.0;
            if (!gather) val = values ? (*values)[eg[e]] : static_cast<double>(eg[e]) + 1.0;
            sb.adjacency.entries[e - e0] = {er[e], ec[e], val};
        }
        sb.component_offsets.assign(comp.begin() + (r0 + b), comp.begin() + (r1 + b + 1));
        sb.local_to_global.assign(l2g.begin() + v0, l2g.begin() + v1);
        sb.roots_local.assign(rl.begin() + r0, rl.begin() + r1);
        if (gather) {
            sb.node_features = DenseMatrix(v1 - v0, f_v, std::vector<double>(xv.begin() + v0 * f_v, xv.begin() + v1 * f_v));
            sb.edge_features = DenseMatrix(e1 - e0, f_e, std::vector<double>(ye.begin() + e0 * f_e, ye.begin() + e1 * f_e));
            sb.edge_labels.assign(lab.begin() + e0, lab.begin() + e1);
            sb.edge_global_ids.assign(eg.begin() + e0, eg.begin() + e1);
        }
    }
    return out;
}

}  // namespace

std::vector<SampledBatch> bulk_shadow(const CsrMatrix& a, const std::vector<std::vector<Index>>& batches,
                                      const SamplerConfig& cfg, ChoiceSource& choice,
                                      const FrontierObserver& observer) {
    cfg.validate();
    const bool ids = values_are_ids(a);
    GraphGuard g;
    g.g = upload_csr(a, 0, !ids);
    SampleGuard s;
    check(hgs_sample_create(g.g, nullptr, &s.s));
    return run_bulk(g.g, s.s, batches, cfg, choice, false, ids ? nullptr : &a.values, 0, 0, false,
                    observer ? &observer : nullptr, &a);
}

SampledBatch shadow_reference(const CsrMatrix& a, std::span<const Index> roots,
                              const SamplerConfig& cfg, ChoiceSource& choice) {
    // One batch, root ordinal = position (sampler.cpp:96-98); the walk uses
    // the raw rows of A when unsymmetrized (sampler.cpp:104-106).
    cfg.validate();
    std::vector<std::vector<Index>> one{std::vector<Index>(roots.begin(), roots.end())};
    const bool ids = values_are_ids(a);
    GraphGuard g;
    g.g = upload_csr(a, 0, !ids);
    SampleGuard s;
    check(hgs_sample_create(g.g, nullptr, &s.s));
    return std::move(run_bulk(g.g, s.s, one, cfg, choice, false, ids ? nullptr : &a.values, 0, 0, true).front());
}

std::vector<std::vector<Index>> sample_rows(const CsrMatrix& p, Index s, ChoiceSource& choice,
                                            std::span<const Index> row_streams) {
    if (s < 1) fail_invalid("sample_rows: s must be >= 1");
    if (!row_streams.empty() && static_cast<Index>(row_streams.size()) != p.n_rows)
        fail_invalid("sample_rows: row_streams length must equal row count");
    for (double v : p.values)
        if (v < 0.0) fail_invalid("sample_rows: row with negative mass");
    auto* per_root = dynamic_cast<PerRootChoiceSource*>(&choice);
    auto* philox = dynamic_cast<PhiloxChoiceSource*>(&choice);
    if (!per_root && !philox)
        fail_invalid("sample_rows: the GPU sampler needs a PerRootChoiceSource or PhiloxChoiceSource");
    const std::size_t n_streams = per_root ? per_root->size() : philox->size();
    const std::size_t cur = per_root ? per_root->current() : philox->current();
    std::vector<Index> streams(row_streams.begin(), row_streams.end());
    if (streams.empty()) streams.assign(static_cast<std::size_t>(p.n_rows), static_cast<Index>(cur));
    Index last = -1, total = 0;
    for (Index r = 0; r < p.n_rows; ++r) {
        const Index deg = p.row_ptr[r + 1] - p.row_ptr[r];
        if (deg == 0) continue;
        total += std::min(s, deg);
        if (last < 0) {  // the reference's first begin_root / choose sees these first
            if (!row_streams.empty() && (streams[r] < 0 || static_cast<std::size_t>(streams[r]) >= n_streams))
                fail_invalid(per_root ? "PerRootChoiceSource: root ordinal out of range"
                                      : "PhiloxChoiceSource: root ordinal out of range");
            if (n_streams == 0)
                fail_invalid(per_root ? "PerRootChoiceSource: no streams configured"
                                      : "PhiloxChoiceSource: no streams configured");
        }
        last = r;
    }
    std::vector<std::uint64_t> state;
    const std::uint64_t* state_ptr = nullptr;
    if (per_root && !per_root->fresh()) {
        state = per_root->states();
        state_ptr = state.data();
    } else if (philox && !philox->fresh()) {
        state.assign(philox->decisions().begin(), philox->decisions().end());
        state_ptr = state.data();
    }
    const std::vector<std::uint64_t>& seeds = per_root ? per_root->seeds() : philox->seeds();
    std::vector<int64_t> off(static_cast<std::size_t>(p.n_rows) + 1), cols(static_cast<std::size_t>(std::max<Index>(total, 1)));
    std::vector<std::uint32_t> draws(n_streams + 1), decs(n_streams + 1);
    check(hgs_sample_rows(0, p.n_rows, p.n_cols, p.row_ptr.data(), p.col_idx.data(), nullptr, s,
                          philox ? HGS_RNG_PHILOX : HGS_RNG_XOSHIRO, seeds.data(), static_cast<int64_t>(n_streams),
                          state_ptr, streams.data(), off.data(), cols.data(), draws.data(), decs.data()));
    draws.resize(n_streams);
    decs.resize(n_streams);
    if (per_root) per_root->advance(draws);
    else philox->advance(decs);
    if (last >= 0 && !row_streams.empty()) choice.begin_root(static_cast<std::uint64_t>(streams[last]));
    std::vector<std::vector<Index>> out(static_cast<std::size_t>(p.n_rows));
    for (Index r = 0; r < p.n_rows; ++r) out[r].assign(cols.begin() + off[r], cols.begin() + off[r + 1]);
    return out;
}

CsrMatrix make_edge_id_matrix(const EventGraph& event) {
    event.validate();
    CsrMatrix out(event.n, event.n);
    out.col_idx.resize(event.edges.entries.size());
    out.values.resize(event.edges.entries.size());
    for (std::size_t i = 0; i < event.edges.entries.size(); ++i) {
        const CooEntry& e = event.edges.entries[i];
        out.row_ptr[static_cast<std::size_t>(e.row) + 1] += 1;
        out.col_idx[i] = e.col;
        out.values[i] = static_cast<double>(i) + 1.0;
    }
    for (Index r = 0; r < event.n; ++r) out.row_ptr[r + 1] += out.row_ptr[r];
    return out;
}

void gather_features(SampledBatch& batch, const EventGraph& event) {
    for (Index v : batch.local_to_global)
        if (v < 0 || v >= event.n) fail_invalid("gather_features: batch vertex out of range for event");
    const Index m = batch.adjacency.nnz();
    std::vector<Index> ids(static_cast<std::size_t>(m));
    for (Index i = 0; i < m; ++i) {
        const Index id = static_cast<Index>(std::llround(batch.adjacency.entries[i].value)) - 1;
        if (id < 0 || id >= event.m())
            fail_invalid("gather_features: adjacency values do not carry edge ids; "
                         "sample from make_edge_id_matrix(event)");
        ids[i] = id;
    }
    const CsrMatrix a = make_edge_id_matrix(event);
    GraphGuard g;
    g.g = upload_csr(a, 0, false);
    check(hgs_graph_attach_features(g.g, event.node_features.data.data(), event.node_features.cols,
                                    event.edge_features.data.data(), event.edge_features.cols,
                                    event.labels.data()));
    const Index V = static_cast<Index>(batch.local_to_global.size());
    batch.node_features = DenseMatrix(V, event.node_features.cols);
    batch.edge_features = DenseMatrix(m, event.edge_features.cols);
    batch.edge_labels.resize(static_cast<std::size_t>(m));
    check(hgs_graph_gather(g.g, batch.local_to_global.data(), V, ids.data(), m,
                           batch.node_features.data.data(), batch.edge_features.data.data(),
                           batch.edge_labels.data()));
    batch.edge_global_ids = std::move(ids);
    for (auto& e : batch.adjacency.entries) e.value = 1.0;
}

std::vector<std::vector<Index>> epoch_root_batches(Index n_vertices, Index batch_size, Rng& rng) {
    if (n_vertices < 1) fail_invalid("epoch_root_batches: empty vertex set");
    if (batch_size < 1) fail_invalid("epoch_root_batches: batch_size must be >= 1");
    std::vector<Index> perm(static_cast<std::size_t>(n_vertices));
    std::iota(perm.begin(), perm.end(), Index{0});
    for (Index i = n_vertices - 1; i > 0; --i)
        std::swap(perm[i], perm[static_cast<Index>(rng.bounded(static_cast<std::uint64_t>(i) + 1))]);
    std::vector<std::vector<Index>> out;
    if (n_vertices < batch_size) {
        out.push_back(std::move(perm));
        return out;
    }
    for (Index s = 0; s + batch_size <= n_vertices; s += batch_size)
        out.emplace_back(perm.begin() + s, perm.begin() + s + batch_size);
    return out;
}

CsrMatrix symmetrize_pattern(const CsrMatrix& a) {
    if (a.n_rows != a.n_cols) fail_invalid("symmetrize_pattern: matrix must be square");
    GraphGuard g;
    g.g = upload_csr(a, 0, false);
    int64_t info[8];
    check(hgs_graph_info(g.g, info));
    CsrMatrix w(a.n_rows, a.n_cols);
    w.col_idx.resize(static_cast<std::size_t>(info[3]));
    check(hgs_graph_walk(g.g, 1, w.row_ptr.data(), w.col_idx.data()));
    w.values.assign(w.col_idx.size(), 1.0);
    return w;
}

// ---- resident events ---------------------------------------------------------------

namespace gpu {

DeviceEvent::DeviceEvent(const EventGraph& event, int device) : device_(device) {
    const CsrMatrix a = make_edge_id_matrix(event);
    graph_ = upload_csr(a, device, false);
    host_a_ = std::make_unique<CsrMatrix>(a);
    n_ = event.n;
    nnz_ = event.m();
    f_v_ = event.node_features.cols;
    f_e_ = event.edge_features.cols;
    check(hgs_graph_attach_features(static_cast<hgs_graph*>(graph_), event.node_features.data.data(), f_v_,
                                    event.edge_features.data.data(), f_e_, event.labels.data()));
    hgs_sample* s = nullptr;
    check(hgs_sample_create(static_cast<hgs_graph*>(graph_), nullptr, &s));
    sampler_ = s;
}

DeviceEvent::DeviceEvent(const CsrMatrix& a, int device) : device_(device) {
    ids_ = values_are_ids(a);
    if (!ids_) values_ = a.values;
    graph_ = upload_csr(a, device, !ids_);
    host_a_ = std::make_unique<CsrMatrix>(a);
    n_ = a.n_rows;
    nnz_ = a.nnz();
    hgs_sample* s = nullptr;
    check(hgs_sample_create(static_cast<hgs_graph*>(graph_), nullptr, &s));
    sampler_ = s;
}

DeviceEvent::~DeviceEvent() {
    if (sampler_) hgs_sample_destroy(static_cast<hgs_sample*>(sampler_));
    if (graph_) hgs_graph_destroy(static_cast<hgs_graph*>(graph_));
}

std::vector<SampledBatch> DeviceEvent::bulk_shadow(const std::vector<std::vector<Index>>& batches,
                                                   const SamplerConfig& cfg, ChoiceSource& choice,
                                                   bool gather, const FrontierObserver& observer) {
    if (gather && f_v_ == 0 && f_e_ == 0) fail_invalid("gather_features: no features attached to the graph");
    return run_bulk(static_cast<hgs_graph*>(graph_), static_cast<hgs_sample*>(sampler_), batches, cfg,
                    choice, gather, ids_ ? nullptr : &values_, f_v_, f_e_, false,
                    observer ? &observer : nullptr, host_a_.get());
}

}  // namespace gpu
}  // namespace hitgnn
