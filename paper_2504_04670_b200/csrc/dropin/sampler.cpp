// sampler.cpp — hitgnn:: sampler API (sampler.hpp:60-102 of the reference)
// implemented over the C ABI (include/hgs.h). All sampling runs on the GPU;
// this file validates inputs with the reference's error semantics, moves
// inputs/outputs across the host boundary and lays the results out as the
// reference's SampledBatch values.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
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

int current_device() {
    int d = 0;
    check(hgs_current_device(&d));
    return d;
}

// ---- resident-graph cache (see include/hitgnn/core.hpp, gpu::release_cached)

std::uint64_t rotl64(std::uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

// Content hash for change detection: four independent multiply-rotate lanes.
std::uint64_t hash_bytes(const void* p, std::size_t bytes, std::uint64_t h) {
    constexpr std::uint64_t K = 0x9E3779B97F4A7C15ULL;
    const auto* c = static_cast<const unsigned char*>(p);
    std::uint64_t a = h ^ 0x243F6A8885A308D3ULL, b = h ^ 0x13198A2E03707344ULL, d = h ^ 0xA4093822299F31D0ULL,
                  e = h ^ 0x082EFA98EC4E6C89ULL;
    std::size_t i = 0;
    for (; i + 32 <= bytes; i += 32) {
        std::uint64_t w[4];
        std::memcpy(w, c + i, 32);
        a = rotl64(a ^ w[0], 29) * K;
        b = rotl64(b ^ w[1], 29) * K;
        d = rotl64(d ^ w[2], 29) * K;
        e = rotl64(e ^ w[3], 29) * K;
    }
    for (; i < bytes; ++i) a = rotl64(a ^ c[i], 29) * K;
    return rotl64(a, 1) ^ rotl64(b, 7) ^ rotl64(d, 13) ^ rotl64(e, 19) ^ (bytes * K);
}

// Sampled fingerprint: 4,096 strided elements plus the first and last 4 KB.
std::uint64_t fingerprint_bytes(const void* p, std::size_t bytes, std::uint64_t h, bool full) {
    if (full || bytes <= 65536) return hash_bytes(p, bytes, h);
    const auto* c = static_cast<const unsigned char*>(p);
    h = hash_bytes(c, 4096, h);
    h = hash_bytes(c + bytes - 4096, 4096, h);
    const std::size_t step = (bytes - 8) / 4096;
    for (std::size_t i = 0; i < 4096; ++i) h = hash_bytes(c + i * step, 8, h);
    return h;
}

struct CacheKey {
    int device = 0;
    int kind = 0;  // 0: A (sampling), 1: event (features)
    const void* obj = nullptr;
    const void* ptr[4] = {};
    std::int64_t size[4] = {};
    std::uint64_t hash = 0;
    bool operator==(const CacheKey& o) const {
        return device == o.device && kind == o.kind && obj == o.obj && hash == o.hash &&
               std::equal(ptr, ptr + 4, o.ptr) && std::equal(size, size + 4, o.size);
    }
};

struct CacheEntry {
    CacheKey key;
    hgs_graph* g = nullptr;
    std::vector<hgs_sample*> idle;  // sample handles not in use
    int in_use = 0;
    std::uint64_t tick = 0;
    bool ids = true;  // A: values are make_edge_id_matrix ids
    std::uint64_t a_hash = 0;  // events: content hash of make_edge_id_matrix(event), as lease_csr keys A
    ~CacheEntry() {
        for (hgs_sample* s : idle) hgs_sample_destroy(s);
        if (g) hgs_graph_destroy(g);
    }
};

struct Cache {
    std::mutex mu;
    std::vector<std::unique_ptr<CacheEntry>> entries;
    std::uint64_t tick = 0;
};
Cache& cache() {
    static Cache* c = new Cache;  // never destroyed: handles may outlive static teardown order
    return *c;
}

bool cache_enabled() {
    const char* e = std::getenv("HGS_DROPIN_CACHE");
    return !(e && std::string(e) == "0");
}
bool verify_full() {
    const char* e = std::getenv("HGS_DROPIN_VERIFY");
    return e && std::string(e) == "full";
}

// A borrowed (graph, sample handle) pair; returned to the cache on scope exit
// (or destroyed with the graph when the cache is off).
struct Lease {
    CacheEntry* entry = nullptr;
    std::unique_ptr<CacheEntry> owned;  // cache disabled: private entry
    hgs_sample* s = nullptr;
    Lease() = default;
    Lease(const Lease&) = delete;
    ~Lease() {
        if (owned) {
            if (s) hgs_sample_destroy(s);
            return;
        }
        if (!entry) return;
        std::lock_guard<std::mutex> lk(cache().mu);
        if (s) entry->idle.push_back(s);
        --entry->in_use;
    }
    hgs_graph* graph() const { return owned ? owned->g : entry->g; }
};

// Find or build the entry for `key`, then borrow a sample handle of it.
template <class Build>
void lease(Lease& out, const CacheKey& key, Build&& build) {
    if (!cache_enabled()) {
        out.owned = std::make_unique<CacheEntry>();
        out.owned->key = key;
        build(*out.owned);
        check(hgs_sample_create(out.owned->g, nullptr, &out.s));
        return;
    }
    Cache& c = cache();
    std::unique_lock<std::mutex> lk(c.mu);
    CacheEntry* e = nullptr;
    for (auto& p : c.entries)
        if (p->key == key) e = p.get();
    if (!e) {
        lk.unlock();  // build (uploads) outside the lock
        auto fresh = std::make_unique<CacheEntry>();
        fresh->key = key;
        build(*fresh);
        lk.lock();
        for (auto& p : c.entries)  // another thread may have built it meanwhile
            if (p->key == key) e = p.get();
        if (!e) {
            constexpr std::size_t kMax = 16;
            while (c.entries.size() >= kMax) {  // evict the least recently used idle entry
                auto victim = c.entries.end();
                for (auto it = c.entries.begin(); it != c.entries.end(); ++it)
                    if ((*it)->in_use == 0 && (victim == c.entries.end() || (*it)->tick < (*victim)->tick))
                        victim = it;
                if (victim == c.entries.end()) break;
                c.entries.erase(victim);
            }
            c.entries.push_back(std::move(fresh));
            e = c.entries.back().get();
        }
    }
    e->tick = ++c.tick;
    ++e->in_use;
    out.entry = e;
    if (!e->idle.empty()) {
        out.s = e->idle.back();
        e->idle.pop_back();
    }
    lk.unlock();
    if (!out.s) check(hgs_sample_create(e->g, nullptr, &out.s));
}

std::uint64_t csr_hash(const CsrMatrix& a) {
    std::uint64_t h = hash_bytes(a.row_ptr.data(), a.row_ptr.size() * sizeof(Index), 1);
    h = hash_bytes(a.col_idx.data(), a.col_idx.size() * sizeof(Index), h);
    return hash_bytes(a.values.data(), a.values.size() * sizeof(double), h);
}

// Borrow an existing event entry (features attached) whose edge-id matrix is
// A, if the cache holds one on this device; false otherwise.
bool lease_event_for(Lease& out, std::uint64_t a_hash, Index n, Index nnz, CacheKey* key_out) {
    if (!cache_enabled()) return false;
    Cache& c = cache();
    std::unique_lock<std::mutex> lk(c.mu);
    const int dev = current_device();
    CacheEntry* e = nullptr;
    for (auto& p : c.entries)
        if (p->key.kind == 1 && p->key.device == dev && p->a_hash == a_hash && p->key.size[0] == n &&
            p->key.size[1] == nnz)
            e = p.get();
    if (!e) return false;
    e->tick = ++c.tick;
    ++e->in_use;
    out.entry = e;
    *key_out = e->key;
    if (!e->idle.empty()) {
        out.s = e->idle.back();
        e->idle.pop_back();
    }
    lk.unlock();
    if (!out.s) check(hgs_sample_create(e->g, nullptr, &out.s));
    return true;
}

// A (sampling matrix): full content hash, values checked for the id pattern
void lease_csr(Lease& out, const CsrMatrix& a, const std::uint64_t* hash = nullptr) {
    CacheKey key;
    key.device = current_device();
    key.kind = 0;
    key.obj = &a;
    key.ptr[0] = a.row_ptr.data(); key.ptr[1] = a.col_idx.data(); key.ptr[2] = a.values.data();
    key.size[0] = a.n_rows; key.size[1] = a.n_cols; key.size[2] = static_cast<std::int64_t>(a.col_idx.size());
    key.size[3] = static_cast<std::int64_t>(a.values.size());
    key.hash = hash ? *hash : csr_hash(a);
    lease(out, key, [&](CacheEntry& e) {
        e.ids = values_are_ids(a);
        e.g = upload_csr(a, key.device, !e.ids);
    });
}

CacheKey event_key(const EventGraph& event) {
    CacheKey key;
    key.device = current_device();
    key.kind = 1;
    key.obj = &event;
    key.ptr[0] = event.edges.entries.data(); key.ptr[1] = event.node_features.data.data();
    key.ptr[2] = event.edge_features.data.data(); key.ptr[3] = event.labels.data();
    key.size[0] = event.n; key.size[1] = event.m();
    key.size[2] = event.node_features.cols; key.size[3] = event.edge_features.cols;
    const bool full = verify_full();
    std::uint64_t h = fingerprint_bytes(event.edges.entries.data(), event.edges.entries.size() * sizeof(CooEntry), 2, full);
    h = fingerprint_bytes(event.node_features.data.data(), event.node_features.data.size() * sizeof(double), h, full);
    h = fingerprint_bytes(event.edge_features.data.data(), event.edge_features.data.size() * sizeof(double), h, full);
    h = fingerprint_bytes(event.labels.data(), event.labels.size(), h, full);
    key.hash = h;
    return key;
}

void lease_event(Lease& out, const EventGraph& event, CacheKey* key_out = nullptr) {
    const CacheKey key = event_key(event);
    if (key_out) *key_out = key;
    lease(out, key, [&](CacheEntry& e) {
        const CsrMatrix a = make_edge_id_matrix(event);
        e.a_hash = csr_hash(a);
        e.g = upload_csr(a, key.device, false);
        check(hgs_graph_attach_features(e.g, event.node_features.data.data(), event.node_features.cols,
                                        event.edge_features.data.data(), event.edge_features.cols,
                                        event.labels.data()));
    });
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

// Page-locked host staging for one thread's calls (grow-only slots).
struct Staging {
    void* p[13] = {};
    std::size_t cap[13] = {};
    template <class T>
    T* get(int slot, std::size_t n) {
        const std::size_t bytes = std::max<std::size_t>(n, 1) * sizeof(T);
        if (cap[slot] < bytes) {
            if (p[slot]) hgs_host_free(p[slot]);
            p[slot] = nullptr;
            cap[slot] = 0;
            const std::size_t want = bytes + bytes / 8;
            check(hgs_host_alloc(want, &p[slot]));
            cap[slot] = want;
        }
        return static_cast<T*>(p[slot]);
    }
    ~Staging() {
        for (void* q : p)
            if (q) hgs_host_free(q);
    }
};
Staging& staging() {
    thread_local Staging st;
    return st;
}

// f(i) for i in [0, n) on up to hardware_concurrency host threads (the
// per-batch SampledBatch values are independent).
template <class F>
void parallel_for(Index n, F&& f) {
    const Index T = std::min<Index>(n, std::max<Index>(1, std::thread::hardware_concurrency()));
    if (T <= 1) {
        for (Index i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> pool;
    std::exception_ptr err;
    std::mutex emu;
    for (Index t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            try {
                for (Index i = t; i < n; i += T) f(i);
            } catch (...) {
                std::lock_guard<std::mutex> lk(emu);
                if (!err) err = std::current_exception();
            }
        });
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
}

// Gather prefetch for the reference's two-line pattern (trainer.cpp:457-458:
// bulk_shadow(edge-id A) then gather_features(batch, event) per batch). When
// the cache already holds the event with its features (any earlier
// gather_features call), bulk_shadow samples on that graph WITH the device
// gather and keeps each batch's features here, built batch-parallel; the
// batches it returns are the reference's (edge-id values, no features). A
// later gather_features(batch, event) on this thread that names the same
// event and the same batch (its local_to_global buffer, sizes and edge ids)
// moves the prebuilt features in instead of gathering again. Anything else
// (a copied batch, another event, an older call) takes the ordinary path.
struct StashItem {
    const Index* l2g = nullptr;
    std::size_t V = 0, E = 0;
    DenseMatrix nf, ef;
    std::vector<std::uint8_t> lab;
    std::vector<Index> gid;
    bool used = true;
};
struct Stash {
    CacheKey event;
    std::vector<StashItem> items;
    std::size_t served = 0;
};
Stash& stash() {
    thread_local Stash st;
    return st;
}

std::vector<SampledBatch> run_bulk(hgs_graph* g, hgs_sample* s,
                                   const std::vector<std::vector<Index>>& batches,
                                   const SamplerConfig& cfg, ChoiceSource& choice, bool gather,
                                   const std::vector<double>* values, Index f_v, Index f_e,
                                   bool seq_walk = false, const FrontierObserver* observer = nullptr,
                                   const CsrMatrix* a_host = nullptr, const CacheKey* stash_event = nullptr) {
    cfg.validate();
    const bool prefetch = stash_event != nullptr;  // gather on the device, hand features out later
    if (prefetch) gather = true;
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

    // D2H into page-locked staging owned by this thread (grow-only), then the
    // reference's SampledBatch layout built batch-parallel on host threads
    Staging& st = staging();
    auto* bvoff = st.get<int32_t>(0, static_cast<std::size_t>(k + 1));
    auto* beoff = st.get<int32_t>(1, static_cast<std::size_t>(k + 1));
    auto* comp = st.get<int32_t>(2, R + static_cast<std::size_t>(k));
    auto* l2g = st.get<int32_t>(3, static_cast<std::size_t>(V));
    auto* rl = st.get<int32_t>(4, R);
    auto* er = st.get<int32_t>(5, static_cast<std::size_t>(E));
    auto* ec = st.get<int32_t>(6, static_cast<std::size_t>(E));
    auto* eg = st.get<int32_t>(7, static_cast<std::size_t>(E));
    auto* draws_p = st.get<std::uint32_t>(8, R);
    auto* decs_p = st.get<std::uint32_t>(9, R);
    double *xv = nullptr, *ye = nullptr;
    std::uint8_t* lab = nullptr;
    hgs_host_out o{};
    o.batch_voff = bvoff; o.batch_eoff = beoff; o.comp_off = comp;
    o.l2g = l2g; o.roots_local = rl; o.e_row = er; o.e_col = ec;
    o.e_gid = eg; o.draws = draws_p; o.decisions = decs_p;
    if (gather) {
        xv = st.get<double>(10, static_cast<std::size_t>(V * f_v));
        ye = st.get<double>(11, static_cast<std::size_t>(E * f_e));
        lab = st.get<std::uint8_t>(12, static_cast<std::size_t>(E));
        o.xv = xv; o.ye = ye; o.lab = lab;
    }
    check(hgs_sample_copy_to_host(s, &o));
    const std::vector<std::uint32_t> draws(draws_p, draws_p + R), decisions(decs_p, decs_p + R);
    if (per_root) per_root->advance(draws);
    else philox->advance(decisions);
    if (observer) emit_frontiers(g, s, *a_host, roots, cfg, *observer);

    std::vector<SampledBatch> out(static_cast<std::size_t>(k));
    Stash& stsh = stash();
    if (prefetch) {
        stsh.event = *stash_event;
        stsh.items.clear();
        stsh.items.resize(static_cast<std::size_t>(k));
    }
    auto build = [&](Index b) {
        SampledBatch& sb = out[b];
        const Index v0 = bvoff[b], v1 = bvoff[b + 1], e0 = beoff[b], e1 = beoff[b + 1];
        const Index r0 = boff[b], r1 = boff[b + 1];
        sb.adjacency.n_rows = sb.adjacency.n_cols = v1 - v0;
        sb.adjacency.entries.resize(static_cast<std::size_t>(e1 - e0));
        for (Index e = e0; e < e1; ++e) {
            double val = 1.0;
            if (!gather || prefetch) val = values ? (*values)[eg[e]] : static_cast<double>(eg[e]) + 1.0;
            sb.adjacency.entries[e - e0] = {er[e], ec[e], val};
        }
        sb.component_offsets.assign(comp + (r0 + b), comp + (r1 + b + 1));
        sb.local_to_global.assign(l2g + v0, l2g + v1);
        sb.roots_local.assign(rl + r0, rl + r1);
        if (prefetch) {
            StashItem& it = stsh.items[b];
            it.l2g = sb.local_to_global.data();
            it.V = static_cast<std::size_t>(v1 - v0);
            it.E = static_cast<std::size_t>(e1 - e0);
            it.nf = DenseMatrix(v1 - v0, f_v, std::vector<double>(xv + v0 * f_v, xv + v1 * f_v));
            it.ef = DenseMatrix(e1 - e0, f_e, std::vector<double>(ye + e0 * f_e, ye + e1 * f_e));
            it.lab.assign(lab + e0, lab + e1);
            it.gid.assign(eg + e0, eg + e1);
            it.used = false;
        } else if (gather) {
            sb.node_features = DenseMatrix(v1 - v0, f_v, std::vector<double>(xv + v0 * f_v, xv + v1 * f_v));
            sb.edge_features = DenseMatrix(e1 - e0, f_e, std::vector<double>(ye + e0 * f_e, ye + e1 * f_e));
            sb.edge_labels.assign(lab + e0, lab + e1);
            sb.edge_global_ids.assign(eg + e0, eg + e1);
        }
    };
    parallel_for(k, build);
    return out;
}

}  // namespace

std::vector<SampledBatch> bulk_shadow(const CsrMatrix& a, const std::vector<std::vector<Index>>& batches,
                                      const SamplerConfig& cfg, ChoiceSource& choice,
                                      const FrontierObserver& observer) {
    cfg.validate();
    std::uint64_t h = 0;
    const bool hashed = !observer && cache_enabled() && values_are_ids(a);
    if (hashed) {  // the event is resident with its features: gather prefetch
        h = csr_hash(a);
        Lease le;
        CacheKey ek;
        if (lease_event_for(le, h, a.n_rows, a.nnz(), &ek)) {
            int64_t info[8];
            check(hgs_graph_info(le.graph(), info));
            return run_bulk(le.graph(), le.s, batches, cfg, choice, true, nullptr, info[6], info[7], false, nullptr,
                            &a, &ek);
        }
    }
    Lease l;
    lease_csr(l, a, hashed ? &h : nullptr);
    const bool ids = l.owned ? l.owned->ids : l.entry->ids;
    return run_bulk(l.graph(), l.s, batches, cfg, choice, false, ids ? nullptr : &a.values, 0, 0, false,
                    observer ? &observer : nullptr, &a);
}

SampledBatch shadow_reference(const CsrMatrix& a, std::span<const Index> roots,
                              const SamplerConfig& cfg, ChoiceSource& choice) {
    // One batch, root ordinal = position (sampler.cpp:96-98); the walk uses
    // the raw rows of A when unsymmetrized (sampler.cpp:104-106).
    cfg.validate();
    std::vector<std::vector<Index>> one{std::vector<Index>(roots.begin(), roots.end())};
    Lease l;
    lease_csr(l, a);
    const bool ids = l.owned ? l.owned->ids : l.entry->ids;
    return std::move(run_bulk(l.graph(), l.s, one, cfg, choice, false, ids ? nullptr : &a.values, 0, 0, true).front());
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
    const Index V = static_cast<Index>(batch.local_to_global.size());
    const Index fv = event.node_features.cols, fe = event.edge_features.cols;
    // ids and outputs through this thread's page-locked staging (slots 0-4)
    Staging& st = staging();
    auto* l2g = st.get<int64_t>(0, static_cast<std::size_t>(V));
    auto* ids = st.get<int64_t>(1, static_cast<std::size_t>(m));
    for (Index i = 0; i < m; ++i) {
        const Index id = static_cast<Index>(std::llround(batch.adjacency.entries[i].value)) - 1;
        if (id < 0 || id >= event.m())
            fail_invalid("gather_features: adjacency values do not carry edge ids; "
                         "sample from make_edge_id_matrix(event)");
        ids[i] = id;
    }
    {  // prefetched by bulk_shadow on this thread for exactly this batch and event?
        Stash& sh = stash();
        for (StashItem& it : sh.items) {
            if (it.used || it.l2g != batch.local_to_global.data() || it.V != static_cast<std::size_t>(V) ||
                it.E != static_cast<std::size_t>(m) || it.nf.cols != fv || it.ef.cols != fe)
                continue;
            if (!(sh.event == event_key(event))) break;
            if (!std::equal(it.gid.begin(), it.gid.end(), ids)) break;
            batch.node_features = std::move(it.nf);
            batch.edge_features = std::move(it.ef);
            batch.edge_labels = std::move(it.lab);
            batch.edge_global_ids = std::move(it.gid);
            it.used = true;
            ++sh.served;
            for (auto& e : batch.adjacency.entries) e.value = 1.0;
            return;
        }
    }
    std::memcpy(l2g, batch.local_to_global.data(), sizeof(int64_t) * static_cast<std::size_t>(V));
    auto* xv = st.get<double>(2, static_cast<std::size_t>(V * fv));
    auto* ye = st.get<double>(3, static_cast<std::size_t>(m * fe));
    auto* lab = st.get<std::uint8_t>(4, static_cast<std::size_t>(m));
    Lease l;
    lease_event(l, event);  // the event's features stay resident across calls
    check(hgs_graph_gather(l.graph(), l2g, V, ids, m, xv, ye, lab));
    batch.node_features = DenseMatrix(V, fv, std::vector<double>(xv, xv + V * fv));
    batch.edge_features = DenseMatrix(m, fe, std::vector<double>(ye, ye + m * fe));
    batch.edge_labels.assign(lab, lab + m);
    batch.edge_global_ids.assign(ids, ids + m);
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

void release_cached() {
    Cache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    // entries borrowed by running calls stay until their next release
    c.entries.erase(std::remove_if(c.entries.begin(), c.entries.end(),
                                   [](const std::unique_ptr<CacheEntry>& e) { return e->in_use == 0; }),
                    c.entries.end());
}

std::size_t prefetched_gathers() { return stash().served; }

std::size_t cached_entries() {
    Cache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    return c.entries.size();
}

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
