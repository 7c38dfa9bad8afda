// abi.cu — the C ABI (include/hgs.h) over the device graph store and the
// sampling pipeline. Host work here is input validation with the reference's
// error semantics, graph ingest (int64 -> int32 narrowing, explicit-zero and
// negative-value bookkeeping) and host<->device copies; all sampling
// arithmetic runs in the kernels (graph.cu, expand.cu, extract*.cu, consumer.cu).
#include <cuda_runtime.h>

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "hgs_internal.cuh"
#include "kernels.cuh"

using namespace hgs;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return HGS_OK;
    } catch (const Failure& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "hgs: host allocation failed";
        return HGS_ECUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return HGS_ECUDA;
    }
}

}  // namespace

int hgs::abi_guard(const std::function<void()>& f) { return guarded(f); }

namespace {

void upload(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes) HGS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
}

void upload_csr(DevCsr& d, int32_t n, const std::vector<int32_t>& rp, const std::vector<int32_t>& ci,
                cudaStream_t st) {
    d.n = n;
    d.nnz = (int64_t)ci.size();
    d.rp.reserve(rp.size());
    d.ci.reserve(std::max<size_t>(ci.size(), 1));
    upload(d.rp.p, rp.data(), rp.size() * sizeof(int32_t), st);
    upload(d.ci.p, ci.data(), ci.size() * sizeof(int32_t), st);
    int32_t md = 0;
    for (int32_t u = 0; u < n; ++u) md = std::max(md, rp[u + 1] - rp[u]);
    d.max_deg = md;
}

// SamplerConfig::validate (sampler.cpp:57-62), verbatim messages.
void validate_cfg(const hgs_config* cfg) {
    if (!cfg) fail(HGS_EINVAL, "hgs: null config");
    if (cfg->depth < 1) fail(HGS_EINVAL, "SamplerConfig: depth must be >= 1");
    if (cfg->fanout < 1) fail(HGS_EINVAL, "SamplerConfig: fanout must be >= 1");
    if (cfg->batch_size < 1) fail(HGS_EINVAL, "SamplerConfig: batch_size must be >= 1");
    if (cfg->bulk_batches < 1) fail(HGS_EINVAL, "SamplerConfig: bulk_batches must be >= 1");
    if (cfg->rng != HGS_RNG_XOSHIRO && cfg->rng != HGS_RNG_PHILOX) fail(HGS_EINVAL, "hgs: unknown rng kind");
}

// The walk's squareness checks of the reference: symmetrize_pattern
// (sparse.cpp:261) or, unsymmetrized, spgemm(q, walk) (sparse.cpp:79-81).
void check_square(const DevGraph& g, int32_t symmetrize) {
    if (g.n_rows == g.n_cols) return;
    if (symmetrize) fail(HGS_EINVAL, "symmetrize_pattern: matrix must be square");
    fail(HGS_EINVAL, "spgemm: inner dimensions disagree (" + std::to_string(g.n_cols) + " vs " +
                         std::to_string(g.n_rows) + ")");
}

}  // namespace

extern "C" {

const char* hgs_last_error(void) { return g_err.c_str(); }
int hgs_abi_version(void) { return HGS_ABI_VERSION; }

int hgs_device_count(int* count) {
    return guarded([&] {
        int c = 0;
        const cudaError_t e = cudaGetDeviceCount(&c);
        if (e != cudaSuccess) { cudaGetLastError(); c = 0; }
        *count = c;
    });
}

int hgs_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        if (!out) fail(HGS_EINVAL, "hgs_host_alloc: null argument");
        *out = nullptr;
        if (bytes) HGS_CUDA(cudaMallocHost(out, bytes));
    });
}

int hgs_host_free(void* p) {
    return guarded([&] {
        if (p) HGS_CUDA(cudaFreeHost(p));
    });
}

int hgs_current_device(int* device) {
    return guarded([&] {
        if (!device) fail(HGS_EINVAL, "hgs_current_device: null argument");
        HGS_CUDA(cudaGetDevice(device));
    });
}

uint64_t hgs_derive(uint64_t seed, const uint64_t* path, int32_t len) { return derive_seed(seed, path, len); }

void hgs_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    philox4x32_10(c, key[0], key[1]);
    std::memcpy(out, c, sizeof(c));
}

// ---- graph -------------------------------------------------------------------

int hgs_graph_create(int device, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                     const int64_t* col_idx, const double* values, hgs_graph** out) {
    return guarded([&] {
        if (!out) fail(HGS_EINVAL, "hgs_graph_create: null out");
        *out = nullptr;
        if (n_rows < 0 || n_cols < 0) fail(HGS_EINVAL, "hgs_graph_create: negative dimension");
        if (n_rows >= ((int64_t)1 << 31) - 1 || n_cols >= ((int64_t)1 << 31) - 1)
            fail(HGS_ERANGE, "hgs_graph_create: more than 2^31-2 vertices");
        if (!row_ptr) fail(HGS_EINVAL, "hgs_graph_create: null row_ptr");
        if (row_ptr[0] != 0) fail(HGS_EINVAL, "hgs_graph_create: row_ptr[0] must be 0");
        const int64_t nnz = row_ptr[n_rows];
        if (nnz >= ((int64_t)1 << 31) - 1) fail(HGS_ERANGE, "hgs_graph_create: more than 2^31-2 entries");
        if (nnz > 0 && !col_idx) fail(HGS_EINVAL, "hgs_graph_create: null col_idx");
        const int32_t n = (int32_t)n_rows;
        bool rp_ok = true;  // O(n) on the host; an invalid row_ptr takes the host loop below,
        for (int32_t u = 0; u < n && rp_ok; ++u) rp_ok = row_ptr[u + 1] >= row_ptr[u];  // which orders errors
        if (!values && rp_ok) {  // edge-id matrix: narrowing and column checks run on the device
            auto* h = new hgs_graph;
            DevGraph& g = h->g;
            try {
                g.device = device;
                HGS_CUDA(cudaSetDevice(device));
                HGS_CUDA(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
                g.n_rows = n_rows;
                g.n_cols = n_cols;
                g.nnz = nnz;
                graph_ingest_device(g, row_ptr, col_idx, g.stream);
            } catch (...) {
                if (g.stream) cudaStreamDestroy(g.stream);
                delete h;
                throw;
            }
            *out = h;
            return;
        }
        std::vector<int32_t> rp(n + 1), ci, gid, frp, fci;
        ci.reserve(nnz);
        bool zeros = false, neg = false;
        std::vector<uint8_t> negrow;
        for (int32_t u = 0; u < n; ++u) {
            if (row_ptr[u + 1] < row_ptr[u]) fail(HGS_EINVAL, "hgs_graph_create: row_ptr not non-decreasing");
            for (int64_t k = row_ptr[u]; k < row_ptr[u + 1]; ++k) {
                const int64_t c = col_idx[k];
                if (c < 0 || c >= n_cols)
                    fail(HGS_EINVAL, "CsrMatrix: entry (" + std::to_string(u) + ", " + std::to_string(c) +
                                         ") out of range for " + std::to_string(n_rows) + "x" +
                                         std::to_string(n_cols));
                if (values && values[k] == 0.0) {  // dropped by spgemm (sparse.cpp:118-121)
                    zeros = true;
                    continue;
                }
                if (values && values[k] < 0.0) {
                    if (negrow.empty()) negrow.assign(n, 0);
                    negrow[u] = 1;
                    neg = true;
                }
                ci.push_back((int32_t)c);
                gid.push_back((int32_t)k);
            }
            rp[u + 1] = (int32_t)ci.size();
        }
        std::vector<int2> ari;  // (row start, out-degree) per vertex of A
        auto* h = new hgs_graph;
        DevGraph& g = h->g;
        try {
            g.device = device;
            HGS_CUDA(cudaSetDevice(device));
            HGS_CUDA(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
            g.n_rows = n_rows;
            g.n_cols = n_cols;
            g.nnz = nnz;
            upload_csr(g.a, n, rp, ci, g.stream);
            ari.resize((size_t)std::max<int32_t>(n, 1));
            for (int32_t u = 0; u < n; ++u) ari[u] = make_int2(rp[u], rp[u + 1] - rp[u]);
            g.a_ri.reserve(ari.size());
            upload(g.a_ri.p, ari.data(), ari.size() * sizeof(int2), g.stream);
            if (zeros) {
                g.has_gid = true;
                g.a_gid.reserve(gid.size());
                upload(g.a_gid.p, gid.data(), gid.size() * sizeof(int32_t), g.stream);
                frp.resize(n + 1);
                fci.resize(nnz);
                for (int32_t u = 0; u <= n; ++u) frp[u] = (int32_t)row_ptr[u];
                for (int64_t k = 0; k < nnz; ++k) fci[k] = (int32_t)col_idx[k];
                g.has_full = true;
                upload_csr(g.a_full, n, frp, fci, g.stream);
            }
            if (neg) {
                g.has_neg = true;
                g.neg_row.reserve(n);
                upload(g.neg_row.p, negrow.data(), n, g.stream);
            }
            HGS_CUDA(cudaStreamSynchronize(g.stream));
        } catch (...) {
            if (g.stream) cudaStreamDestroy(g.stream);
            delete h;
            throw;
        }
        *out = h;
    });
}

int hgs_graph_attach_features(hgs_graph* h, const double* node_feat, int64_t f_v,
                              const double* edge_feat, int64_t f_e, const uint8_t* labels) {
    return guarded([&] {
        if (!h) fail(HGS_EINVAL, "hgs: null graph");
        DevGraph& g = h->g;
        if (f_v < 0 || f_e < 0) fail(HGS_EINVAL, "hgs_graph_attach_features: negative width");
        HGS_CUDA(cudaSetDevice(g.device));
        g.f_v = (int32_t)f_v;
        g.f_e = (int32_t)f_e;
        g.node_feat.reserve((size_t)std::max<int64_t>(1, g.n_rows * f_v));
        g.edge_feat.reserve((size_t)std::max<int64_t>(1, g.nnz * f_e));
        g.labels.reserve((size_t)std::max<int64_t>(1, g.nnz));
        upload(g.node_feat.p, node_feat, sizeof(double) * g.n_rows * f_v, g.stream);
        upload(g.edge_feat.p, edge_feat, sizeof(double) * g.nnz * f_e, g.stream);
        upload(g.labels.p, labels, g.nnz, g.stream);
        build_edge_records(g, g.stream);
        HGS_CUDA(cudaStreamSynchronize(g.stream));
        g.has_features = true;
    });
}

// ---- binary event files (hgs_event_save / hgs_graph_load) ------------------

namespace {

constexpr char kEventMagic[8] = {'H', 'G', 'S', 'E', 'V', 'T', '0', '1'};
struct EventHeader {
    char magic[8];
    int64_t n_rows, n_cols, nnz, f_v, f_e, flags;  // flags: 1 = values present
    int64_t off[6];  // row_ptr, col_idx, values, node_feat, edge_feat, labels (bytes from file start)
    int64_t bytes[6];
    int64_t file_bytes;
};
constexpr int64_t kAlign = 64;
int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Mapping {
    void* p = MAP_FAILED;
    size_t len = 0;
    int fd = -1;
    ~Mapping() {
        if (p != MAP_FAILED) munmap(p, len);
        if (fd >= 0) close(fd);
    }
};

const EventHeader& map_event(Mapping& m, const char* path) {
    if (!path) fail(HGS_EINVAL, "hgs_graph_load: null path");
    m.fd = open(path, O_RDONLY);
    if (m.fd < 0) fail(HGS_EINVAL, std::string("hgs_graph_load: cannot open ") + path);
    struct stat sb {};
    if (fstat(m.fd, &sb) != 0 || sb.st_size < (off_t)sizeof(EventHeader))
        fail(HGS_EINVAL, std::string("hgs_graph_load: not an event file: ") + path);
    m.len = (size_t)sb.st_size;
    m.p = mmap(nullptr, m.len, PROT_READ, MAP_PRIVATE | MAP_POPULATE, m.fd, 0);
    if (m.p == MAP_FAILED) fail(HGS_ECUDA, std::string("hgs_graph_load: mmap failed: ") + path);
    const auto& h = *static_cast<const EventHeader*>(m.p);
    if (std::memcmp(h.magic, kEventMagic, 8) != 0) fail(HGS_EINVAL, std::string("hgs_graph_load: bad magic: ") + path);
    if (h.file_bytes != (int64_t)m.len || h.n_rows < 0 || h.n_cols < 0 || h.nnz < 0 || h.f_v < 0 || h.f_e < 0)
        fail(HGS_EINVAL, std::string("hgs_graph_load: truncated or corrupt event file: ") + path);
    const int64_t want[6] = {8 * (h.n_rows + 1), 8 * h.nnz, (h.flags & 1) ? 8 * h.nnz : 0, 8 * h.n_rows * h.f_v,
                             8 * h.nnz * h.f_e, h.nnz};
    for (int i = 0; i < 6; ++i)
        if (h.bytes[i] != want[i] || h.off[i] < (int64_t)sizeof(EventHeader) || h.off[i] + h.bytes[i] > h.file_bytes)
            fail(HGS_EINVAL, std::string("hgs_graph_load: truncated or corrupt event file: ") + path);
    return h;
}

}  // namespace

int hgs_event_save(const char* path, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                   const double* values, const double* node_feat, int64_t f_v, const double* edge_feat, int64_t f_e,
                   const uint8_t* labels) {
    return guarded([&] {
        if (!path || !row_ptr || n_rows < 0 || n_cols < 0 || f_v < 0 || f_e < 0)
            fail(HGS_EINVAL, "hgs_event_save: bad arguments");
        if (row_ptr[0] != 0 || row_ptr[n_rows] < 0 || (row_ptr[n_rows] > 0 && !col_idx))
            fail(HGS_EINVAL, "hgs_event_save: bad row_ptr or null col_idx");
        EventHeader h{};
        std::memcpy(h.magic, kEventMagic, 8);
        h.n_rows = n_rows;
        h.n_cols = n_cols;
        h.nnz = row_ptr[n_rows];
        h.f_v = node_feat ? f_v : 0;
        h.f_e = edge_feat ? f_e : 0;
        h.flags = values ? 1 : 0;
        const void* src[6] = {row_ptr, col_idx, values, node_feat, edge_feat, labels};
        const int64_t bytes[6] = {8 * (n_rows + 1), 8 * h.nnz, values ? 8 * h.nnz : 0, 8 * n_rows * h.f_v,
                                  8 * h.nnz * h.f_e, labels ? h.nnz : 0};
        int64_t pos = align_up((int64_t)sizeof(EventHeader));
        for (int i = 0; i < 6; ++i) {
            h.off[i] = pos;
            h.bytes[i] = bytes[i];
            pos = align_up(pos + bytes[i]);
        }
        h.file_bytes = pos;
        const std::string tmp = std::string(path) + ".tmp";
        FILE* f = std::fopen(tmp.c_str(), "wb");
        if (!f) fail(HGS_EINVAL, std::string("hgs_event_save: cannot write ") + path);
        bool ok = std::fwrite(&h, sizeof h, 1, f) == 1;
        static const char zeros[kAlign] = {};
        int64_t at = (int64_t)sizeof h;
        for (int i = 0; i < 6 && ok; ++i) {
            ok = ok && std::fwrite(zeros, 1, (size_t)(h.off[i] - at), f) == (size_t)(h.off[i] - at);
            if (bytes[i]) ok = ok && std::fwrite(src[i], 1, (size_t)bytes[i], f) == (size_t)bytes[i];
            at = h.off[i] + bytes[i];
        }
        ok = ok && std::fwrite(zeros, 1, (size_t)(h.file_bytes - at), f) == (size_t)(h.file_bytes - at);
        ok = (std::fclose(f) == 0) && ok;
        if (!ok || std::rename(tmp.c_str(), path) != 0) {
            std::remove(tmp.c_str());
            fail(HGS_EINVAL, std::string("hgs_event_save: write failed: ") + path);
        }
    });
}

int hgs_event_info(const char* path, int64_t* info) {
    return guarded([&] {
        if (!info) fail(HGS_EINVAL, "hgs_event_info: null argument");
        Mapping m;
        const EventHeader& h = map_event(m, path);
        info[0] = h.n_rows; info[1] = h.n_cols; info[2] = h.nnz; info[3] = h.f_v; info[4] = h.f_e; info[5] = h.flags;
    });
}

int hgs_graph_load(int device, const char* path, hgs_graph** out) {
    if (!out) {
        g_err = "hgs_graph_load: null out";
        return HGS_EINVAL;
    }
    *out = nullptr;
    Mapping m;
    const EventHeader* hp = nullptr;
    const int rc0 = guarded([&] { hp = &map_event(m, path); });
    if (rc0 != HGS_OK) return rc0;
    const EventHeader& h = *hp;
    const auto* base = static_cast<const char*>(m.p);
    auto at = [&](int i) { return h.bytes[i] ? base + h.off[i] : nullptr; };
    hgs_graph* g = nullptr;
    int rc = hgs_graph_create(device, h.n_rows, h.n_cols, reinterpret_cast<const int64_t*>(at(0)),
                              reinterpret_cast<const int64_t*>(at(1)), reinterpret_cast<const double*>(at(2)), &g);
    if (rc != HGS_OK) return rc;
    if (h.bytes[5] || h.f_v || h.f_e) {
        rc = hgs_graph_attach_features(g, reinterpret_cast<const double*>(at(3)), h.f_v,
                                       reinterpret_cast<const double*>(at(4)), h.f_e,
                                       reinterpret_cast<const uint8_t*>(at(5)));
        if (rc != HGS_OK) {
            const std::string keep = g_err;
            hgs_graph_destroy(g);
            g_err = keep;
            return rc;
        }
    }
    *out = g;
    return HGS_OK;
}

int hgs_graph_info(hgs_graph* h, int64_t* info) {
    return guarded([&] {
        if (!h || !info) fail(HGS_EINVAL, "hgs_graph_info: null argument");
        DevGraph& g = h->g;
        HGS_CUDA(cudaSetDevice(g.device));
        if (g.n_rows == g.n_cols) graph_build_walk_sym(g);
        info[0] = g.n_rows;
        info[1] = g.n_cols;
        info[2] = g.nnz;
        info[3] = g.sym_built ? g.walk_sym.nnz : -1;
        info[4] = g.sym_built ? g.walk_sym.max_deg : -1;
        info[5] = g.a.max_deg;
        info[6] = g.f_v;
        info[7] = g.f_e;
    });
}

int hgs_graph_walk(hgs_graph* h, int32_t symmetrize, int64_t* row_ptr, int64_t* col_idx) {
    return guarded([&] {
        if (!h || !row_ptr || !col_idx) fail(HGS_EINVAL, "hgs_graph_walk: null argument");
        DevGraph& g = h->g;
        HGS_CUDA(cudaSetDevice(g.device));
        check_square(g, symmetrize);
        if (symmetrize) graph_build_walk_sym(g);
        const DevCsr& w = symmetrize ? g.walk_sym : g.a;
        std::vector<int32_t> rp(w.n + 1), ci(w.nnz);
        HGS_CUDA(cudaMemcpy(rp.data(), w.rp.p, sizeof(int32_t) * (w.n + 1), cudaMemcpyDeviceToHost));
        if (w.nnz) HGS_CUDA(cudaMemcpy(ci.data(), w.ci.p, sizeof(int32_t) * w.nnz, cudaMemcpyDeviceToHost));
        for (int32_t u = 0; u <= w.n; ++u) row_ptr[u] = rp[u];
        for (int64_t k = 0; k < w.nnz; ++k) col_idx[k] = ci[k];
    });
}

int hgs_graph_destroy(hgs_graph* h) {
    return guarded([&] {
        if (!h) return;
        cudaSetDevice(h->g.device);
        cudaStream_t st = h->g.stream;
        delete h;
        if (st) cudaStreamDestroy(st);
    });
}

int hgs_graph_gather(hgs_graph* h, const int64_t* l2g, int64_t V, const int64_t* eid, int64_t E,
                     double* xv, double* ye, uint8_t* lab) {
    return guarded([&] {
        if (!h) fail(HGS_EINVAL, "hgs: null graph");
        DevGraph& g = h->g;
        if (!g.has_features) fail(HGS_EINVAL, "gather_features: no features attached to the graph");
        if (V < 0 || E < 0 || (V && !l2g) || (E && (!eid || !lab)) || (V * g.f_v && !xv) || (E * g.f_e && !ye))
            fail(HGS_EINVAL, "hgs_graph_gather: bad sizes or null buffers");
        for (int64_t i = 0; i < V; ++i)
            if (l2g[i] < 0 || l2g[i] >= g.n_rows)
                fail(HGS_EINVAL, "gather_features: batch vertex out of range for event");
        for (int64_t i = 0; i < E; ++i)
            if (eid[i] < 0 || eid[i] >= g.nnz)
                fail(HGS_EINVAL, "gather_features: adjacency values do not carry edge ids; "
                                 "sample from make_edge_id_matrix(event)");
        HGS_CUDA(cudaSetDevice(g.device));
        // per-graph grow-only scratch (no cudaMalloc per batch); one gather at a time per graph
        std::lock_guard<std::mutex> lk(g.gather_mu);
        cudaStream_t st = g.stream;
        DevBuf<int64_t>& dl = g.g_l2g;
        DevBuf<int64_t>& de = g.g_eid;
        DevBuf<double>& dx = g.g_xv;
        DevBuf<double>& dy = g.g_ye;
        DevBuf<uint8_t>& db = g.g_lab;
        dl.reserve((size_t)V + 1); de.reserve((size_t)E + 1);
        dx.reserve((size_t)(V * g.f_v) + 1); dy.reserve((size_t)(E * g.f_e) + 1); db.reserve((size_t)E + 1);
        upload(dl.p, l2g, sizeof(int64_t) * V, st);
        upload(de.p, eid, sizeof(int64_t) * E, st);
        gather_rows(g, dl.p, V, de.p, E, dx.p, dy.p, db.p, st);
        if (V * g.f_v) HGS_CUDA(cudaMemcpyAsync(xv, dx.p, sizeof(double) * V * g.f_v, cudaMemcpyDeviceToHost, st));
        if (E * g.f_e) HGS_CUDA(cudaMemcpyAsync(ye, dy.p, sizeof(double) * E * g.f_e, cudaMemcpyDeviceToHost, st));
        if (E) HGS_CUDA(cudaMemcpyAsync(lab, db.p, E, cudaMemcpyDeviceToHost, st));
        HGS_CUDA(cudaStreamSynchronize(st));
    });
}

// ---- sampling -------------------------------------------------------------------

int hgs_sample_create(hgs_graph* g, void* stream, hgs_sample** out) {
    return guarded([&] {
        if (!g || !out) fail(HGS_EINVAL, "hgs_sample_create: null argument");
        HGS_CUDA(cudaSetDevice(g->g.device));
        auto* s = new hgs_sample;
        s->graph = g;
        // test hooks: start with tiny capacities to exercise the regrow path
        if (const char* e = getenv("HGS_E_STRIDE")) s->e_stride = std::max(1, atoi(e));
        if (const char* e = getenv("HGS_E_CAP")) s->e_cap = (size_t)std::max(1, atoi(e));
        if (stream) s->stream = (cudaStream_t)stream;
        else {
            HGS_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
            s->own_stream = true;
        }
        *out = s;
    });
}

int hgs_sample_bind(hgs_sample* s, hgs_graph* g) {
    return guarded([&] {
        if (!s || !g) fail(HGS_EINVAL, "hgs_sample_bind: null argument");
        if (s->pending) fail(HGS_EINVAL, "hgs_sample_bind: run not waited for");
        if (g->g.device != s->graph->g.device) fail(HGS_EINVAL, "hgs_sample_bind: graph is on another device");
        s->graph = g;
    });
}

int hgs_sample_destroy(hgs_sample* s) {
    return guarded([&] {
        if (!s) return;
        cudaSetDevice(s->graph->g.device);
        if (s->pending) cudaStreamSynchronize(s->stream);
        for (auto& e : s->ev) if (e) cudaEventDestroy(e);
        for (auto& e : s->chunk_ev) cudaEventDestroy(e);
        if (s->aux) cudaStreamDestroy(s->aux);
        if (s->h_state) cudaFreeHost(s->h_state);
        cudaStream_t st = s->own_stream ? s->stream : nullptr;
        delete s;
        if (st) cudaStreamDestroy(st);
    });
}

int hgs_sample_run(hgs_sample* s, const hgs_config* cfg, const int64_t* roots,
                   const int64_t* batch_off, int64_t n_batches, const uint64_t* seeds,
                   const uint64_t* rng_state) {
    return guarded([&] {
        if (!s) fail(HGS_EINVAL, "hgs: null sample handle");
        validate_cfg(cfg);
        DevGraph& g = s->graph->g;
        if (n_batches < 0 || !batch_off) fail(HGS_EINVAL, "hgs_sample_run: bad batch offsets");
        if (batch_off[0] != 0) fail(HGS_EINVAL, "hgs_sample_run: batch_off[0] must be 0");
        for (int64_t b = 0; b < n_batches; ++b)
            if (batch_off[b + 1] < batch_off[b]) fail(HGS_EINVAL, "hgs_sample_run: batch_off not non-decreasing");
        const int64_t R = batch_off[n_batches];
        if (R >= ((int64_t)1 << 31) - 1) fail(HGS_ERANGE, "hgs_sample_run: too many roots");
        // check_roots per batch (sampler.cpp:12-20), in order, verbatim messages
        static thread_local std::vector<uint8_t> seen;
        if ((int64_t)seen.size() < g.n_rows) seen.assign((size_t)g.n_rows, 0);
        for (int64_t b = 0; b < n_batches; ++b) {
            int64_t i = batch_off[b];
            for (; i < batch_off[b + 1]; ++i) {
                const int64_t r = roots[i];
                if (r < 0 || r >= g.n_rows) {
                    for (int64_t j = batch_off[b]; j < i; ++j) seen[roots[j]] = 0;
                    fail(HGS_EINVAL, "sampler: root " + std::to_string(r) + " out of range");
                }
                if (seen[r]) {
                    for (int64_t j = batch_off[b]; j < i; ++j) seen[roots[j]] = 0;
                    fail(HGS_EINVAL, "sampler: duplicate root " + std::to_string(r));
                }
                seen[r] = 1;
            }
            for (int64_t j = batch_off[b]; j < batch_off[b + 1]; ++j) seen[roots[j]] = 0;
        }
        check_square(g, cfg->symmetrize);
        if (R > 0 && !seeds) fail(HGS_EINVAL, "hgs_sample_run: null seeds");
        HGS_CUDA(cudaSetDevice(g.device));
        if (s->pending) HGS_CUDA(cudaStreamSynchronize(s->stream));
        s->pending = false;
        s->boff64.reserve((size_t)n_batches + 1);
        s->seeds.reserve((size_t)R + 1);
        s->roots64.reserve((size_t)R + 1);
        upload(s->roots64.p, roots, sizeof(int64_t) * R, s->stream);
        upload(s->boff64.p, batch_off, sizeof(int64_t) * (n_batches + 1), s->stream);
        upload(s->seeds.p, seeds, sizeof(uint64_t) * R, s->stream);
        const bool philox = cfg->rng == HGS_RNG_PHILOX;
        if (rng_state) {
            const size_t words = philox ? (size_t)R : 4 * (size_t)R;
            s->rng_state.reserve(words + 1);
            upload(s->rng_state.p, rng_state, sizeof(uint64_t) * words, s->stream);
        }
        CallInputs in;
        in.roots64 = s->roots64.p;
        in.batch_off = s->boff64.p;
        in.seeds = s->seeds.p;
        in.state = rng_state ? s->rng_state.p : nullptr;
        in.R = R;
        in.k = n_batches;
        s->last_in = in;  // device copies: hgs_sample_slice reads the batch offsets
        s->last_cfg = *cfg;
        sample_enqueue(s, *cfg, in);
        sample_finish(s, *cfg, in);
    });
}

int hgs_sample_run_multi(hgs_sample* s, const hgs_config* cfg, hgs_graph* const* graphs, int32_t n_graphs,
                         const int32_t* batch_event, const int64_t* roots, const int64_t* batch_off,
                         int64_t n_batches, const uint64_t* seeds) {
    return guarded([&] {
        if (!s) fail(HGS_EINVAL, "hgs: null sample handle");
        validate_cfg(cfg);
        if (n_graphs < 1 || !graphs) fail(HGS_EINVAL, "hgs_sample_run_multi: no graphs");
        if (n_batches < 0 || !batch_off || (n_batches > 0 && !batch_event))
            fail(HGS_EINVAL, "hgs_sample_run_multi: bad batch offsets");
        if (batch_off[0] != 0) fail(HGS_EINVAL, "hgs_sample_run_multi: batch_off[0] must be 0");
        const int device = s->graph->g.device;
        for (int32_t e = 0; e < n_graphs; ++e) {
            if (!graphs[e]) fail(HGS_EINVAL, "hgs_sample_run_multi: null graph");
            if (graphs[e]->g.device != device)
                fail(HGS_EINVAL, "hgs_sample_run_multi: every graph must be on the sample handle's device");
            check_square(graphs[e]->g, cfg->symmetrize);
            if (cfg->gather && (graphs[e]->g.f_v != graphs[0]->g.f_v || graphs[e]->g.f_e != graphs[0]->g.f_e))
                fail(HGS_EINVAL, "hgs_sample_run_multi: feature widths differ across graphs");
        }
        // events contiguous in batch order: event e owns the roots [ev_r0[e], ev_r0[e+1])
        std::vector<int64_t> ev_r0((size_t)n_graphs + 1, 0);
        int32_t prev = 0;
        for (int64_t b = 0; b < n_batches; ++b) {
            const int32_t e = batch_event[b];
            if (e < 0 || e >= n_graphs) fail(HGS_EINVAL, "hgs_sample_run_multi: batch event out of range");
            if (e < prev) fail(HGS_EINVAL, "hgs_sample_run_multi: batch events must be non-decreasing");
            if (batch_off[b + 1] < batch_off[b]) fail(HGS_EINVAL, "hgs_sample_run_multi: batch_off not non-decreasing");
            prev = e;
        }
        for (int32_t e = 0, b = 0; e <= n_graphs; ++e) {  // first root of each event
            while (b < n_batches && batch_event[b] < e) ++b;
            ev_r0[(size_t)e] = batch_off[b];
        }
        const int64_t R = batch_off[n_batches];
        if (R >= ((int64_t)1 << 31) - 1) fail(HGS_ERANGE, "hgs_sample_run_multi: too many roots");
        // check_roots per batch (sampler.cpp:12-20) against the batch's event
        static thread_local std::vector<uint8_t> seen;
        for (int64_t b = 0; b < n_batches; ++b) {
            const int64_t n = graphs[batch_event[b]]->g.n_rows;
            if ((int64_t)seen.size() < n) seen.assign((size_t)n, 0);
            int64_t i = batch_off[b];
            for (; i < batch_off[b + 1]; ++i) {
                const int64_t r = roots[i];
                if (r < 0 || r >= n) {
                    for (int64_t j = batch_off[b]; j < i; ++j) seen[roots[j]] = 0;
                    fail(HGS_EINVAL, "sampler: root " + std::to_string(r) + " out of range");
                }
                if (seen[r]) {
                    for (int64_t j = batch_off[b]; j < i; ++j) seen[roots[j]] = 0;
                    fail(HGS_EINVAL, "sampler: duplicate root " + std::to_string(r));
                }
                seen[r] = 1;
            }
            for (int64_t j = batch_off[b]; j < batch_off[b + 1]; ++j) seen[roots[j]] = 0;
        }
        if (R > 0 && !seeds) fail(HGS_EINVAL, "hgs_sample_run_multi: null seeds");
        HGS_CUDA(cudaSetDevice(device));
        if (s->pending) HGS_CUDA(cudaStreamSynchronize(s->stream));
        s->pending = false;
        s->boff64.reserve((size_t)n_batches + 1);
        s->seeds.reserve((size_t)R + 1);
        s->roots64.reserve((size_t)R + 1);
        upload(s->roots64.p, roots, sizeof(int64_t) * R, s->stream);
        upload(s->boff64.p, batch_off, sizeof(int64_t) * (n_batches + 1), s->stream);
        upload(s->seeds.p, seeds, sizeof(uint64_t) * R, s->stream);
        s->multi_graphs.assign(graphs, graphs + n_graphs);
        s->multi_r0 = ev_r0;
        CallInputs in;
        in.roots64 = s->roots64.p;
        in.batch_off = s->boff64.p;
        in.seeds = s->seeds.p;
        in.R = R;
        in.k = n_batches;
        in.n_events = n_graphs;
        in.events = s->multi_graphs.data();
        in.ev_r0 = s->multi_r0.data();
        s->last_in = in;
        s->last_cfg = *cfg;
        sample_enqueue(s, *cfg, in);
        sample_finish(s, *cfg, in);
    });
}

int hgs_sample_run_device(hgs_sample* s, const hgs_config* cfg, const int32_t* d_roots,
                          const int64_t* d_batch_off, int64_t n_roots, int64_t n_batches,
                          const uint64_t* d_seeds) {
    return guarded([&] {
        if (!s) fail(HGS_EINVAL, "hgs: null sample handle");
        if (n_roots < 0 || n_batches < 0) fail(HGS_EINVAL, "hgs_sample_run_device: negative count");
        if (n_roots > 0 && n_batches < 1) fail(HGS_EINVAL, "hgs_sample_run_device: roots without batches");
        if (n_roots >= ((int64_t)1 << 31) - 1) fail(HGS_ERANGE, "hgs_sample_run_device: too many roots");
        if (n_batches > 0 && !d_batch_off) fail(HGS_EINVAL, "hgs_sample_run_device: null batch offsets");
        if (n_roots > 0 && (!d_roots || !d_seeds)) fail(HGS_EINVAL, "hgs_sample_run_device: null roots or seeds");
        validate_cfg(cfg);
        DevGraph& g = s->graph->g;
        check_square(g, cfg->symmetrize);
        HGS_CUDA(cudaSetDevice(g.device));
        if (s->pending) fail(HGS_EINVAL, "hgs_sample_run_device: previous run not waited for");
        CallInputs in;
        in.roots32 = d_roots;
        in.batch_off = d_batch_off;
        in.seeds = d_seeds;
        in.R = n_roots;
        in.k = n_batches;
        sample_enqueue(s, *cfg, in);
        // remembered for a possible capacity re-run in hgs_sample_wait
        s->last_in = in;
        s->last_cfg = *cfg;
    });
}

int hgs_sample_run_device_spec(hgs_sample* s, const hgs_config* cfg, const int32_t* d_roots,
                               const int64_t* d_batch_off, int64_t n_roots, int64_t n_batches,
                               const hgs_seed_spec* spec) {
    return guarded([&] {
        if (!s) fail(HGS_EINVAL, "hgs: null sample handle");
        if (!spec) fail(HGS_EINVAL, "hgs_sample_run_device_spec: null seed spec");
        if (spec->path_len < 0 || spec->path_len > 6)
            fail(HGS_EINVAL, "hgs_sample_run_device_spec: path_len must be in [0, 6]");
        if (n_roots < 0 || n_batches < 0) fail(HGS_EINVAL, "hgs_sample_run_device_spec: negative count");
        if (n_roots > 0 && n_batches < 1)
            fail(HGS_EINVAL, "hgs_sample_run_device_spec: roots without batches");
        if (n_roots >= ((int64_t)1 << 31) - 1) fail(HGS_ERANGE, "hgs_sample_run_device_spec: too many roots");
        if (n_batches > 0 && !d_batch_off) fail(HGS_EINVAL, "hgs_sample_run_device_spec: null batch offsets");
        if (n_roots > 0 && !d_roots) fail(HGS_EINVAL, "hgs_sample_run_device_spec: null roots");
        validate_cfg(cfg);
        DevGraph& g = s->graph->g;
        check_square(g, cfg->symmetrize);
        HGS_CUDA(cudaSetDevice(g.device));
        if (s->pending) fail(HGS_EINVAL, "hgs_sample_run_device_spec: previous run not waited for");
        s->last_spec = *spec;
        CallInputs in;
        in.roots32 = d_roots;
        in.batch_off = d_batch_off;
        in.seeds = nullptr;
        in.spec = &s->last_spec;
        in.R = n_roots;
        in.k = n_batches;
        sample_enqueue(s, *cfg, in);
        s->last_in = in;
        s->last_cfg = *cfg;
    });
}

int hgs_derive_seeds(const hgs_seed_spec* spec, const int64_t* batch_off, int64_t n_batches, uint64_t* out) {
    return guarded([&] {
        if (!spec || (n_batches > 0 && (!batch_off || !out))) fail(HGS_EINVAL, "hgs_derive_seeds: null argument");
        if (spec->path_len < 0 || spec->path_len > 6) fail(HGS_EINVAL, "hgs_derive_seeds: path_len must be in [0, 6]");
        uint64_t path[8];
        for (int i = 0; i < spec->path_len; ++i) path[i] = spec->path[i];
        for (int64_t b = 0; b < n_batches; ++b)
            for (int64_t r = batch_off[b]; r < batch_off[b + 1]; ++r) {
                path[spec->path_len] = (uint64_t)(spec->batch_base + b);
                path[spec->path_len + 1] = (uint64_t)(r - batch_off[b]);
                out[r] = derive_seed(spec->seed, path, spec->path_len + 2);
            }
    });
}

int hgs_sample_copy_frontiers(hgs_sample* s, int32_t* touched, int32_t* tcount, int32_t* level_counts,
                              int64_t* stride) {
    return guarded([&] {
        if (!s) fail(HGS_EINVAL, "hgs: null sample handle");
        if (s->pending) fail(HGS_EINVAL, "hgs_sample_copy_frontiers: run not waited for");
        if (!s->frontier_kept) fail(HGS_EINVAL, "hgs_sample_copy_frontiers: last run did not keep frontiers");
        HGS_CUDA(cudaSetDevice(s->graph->g.device));
        const size_t R = (size_t)s->R;
        cudaStream_t st = s->stream;
        if (stride) *stride = s->touched_stride;
        if (touched && R)
            HGS_CUDA(cudaMemcpyAsync(touched, s->frontier.p, sizeof(int32_t) * R * s->touched_stride,
                                     cudaMemcpyDeviceToHost, st));
        if (tcount && R)
            HGS_CUDA(cudaMemcpyAsync(tcount, s->tcount.p, sizeof(int32_t) * R, cudaMemcpyDeviceToHost, st));
        if (level_counts && R)
            HGS_CUDA(cudaMemcpyAsync(level_counts, s->level_counts.p, sizeof(int32_t) * R * (s->depth + 1),
                                     cudaMemcpyDeviceToHost, st));
        HGS_CUDA(cudaStreamSynchronize(st));
    });
}

int hgs_sample_rows(int device, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                    const double* values, int64_t s, int32_t rng, const uint64_t* seeds, int64_t n_streams,
                    const uint64_t* rng_state, const int64_t* row_streams, int64_t* out_off, int64_t* out_cols,
                    uint32_t* draws, uint32_t* decisions) {
    return guarded([&] {
        // validation in the reference's order and words (sampler.cpp:67-72)
        if (s < 1) fail(HGS_EINVAL, "sample_rows: s must be >= 1");
        if (n_rows < 0 || !row_ptr || !out_off || !row_streams) fail(HGS_EINVAL, "hgs_sample_rows: null argument");
        const int64_t nnz = row_ptr[n_rows];
        if (values)
            for (int64_t k = 0; k < nnz; ++k)
                if (values[k] < 0.0) fail(HGS_EINVAL, "sample_rows: row with negative mass");
        const char* src = rng == HGS_RNG_PHILOX ? "PhiloxChoiceSource" : "PerRootChoiceSource";
        // choices per row, stream groups (counting sort by stream, row order kept)
        out_off[0] = 0;
        int64_t maxdeg = 0;
        std::vector<int64_t> cnt((size_t)std::max<int64_t>(n_streams, 0) + 1, 0);
        for (int64_t r = 0; r < n_rows; ++r) {
            const int64_t deg = row_ptr[r + 1] - row_ptr[r];
            out_off[r + 1] = out_off[r] + std::min<int64_t>(s, deg);
            if (deg == 0) continue;
            maxdeg = std::max(maxdeg, deg);
            const int64_t st = row_streams[r];
            if (n_streams == 0) fail(HGS_EINVAL, std::string(src) + ": no streams configured");
            if (st < 0 || st >= n_streams) fail(HGS_EINVAL, std::string(src) + ": root ordinal out of range");
            ++cnt[st + 1];
        }
        const int64_t kmax = std::min<int64_t>(s, maxdeg);
        if (kmax > ((int64_t)1 << 24))
            fail(HGS_ERANGE, "hgs_sample_rows: more than 2^24 choices per row is not supported by this build");
        if (maxdeg >= ((int64_t)1 << 31)) fail(HGS_ERANGE, "hgs_sample_rows: row too wide");
        std::vector<int64_t> sptr{0}, sid, srows;
        std::vector<int64_t> start(cnt.size(), 0);
        for (size_t i = 1; i < cnt.size(); ++i) start[i] = start[i - 1] + cnt[i];
        srows.resize((size_t)start.back());
        std::vector<int64_t> fill(start.begin(), start.end() - 1);
        for (int64_t r = 0; r < n_rows; ++r)
            if (row_ptr[r + 1] > row_ptr[r]) srows[(size_t)fill[row_streams[r]]++] = r;
        for (int64_t st = 0; st < n_streams; ++st)
            if (cnt[st + 1]) { sid.push_back(st); sptr.push_back(start[st + 1]); }
        const int64_t groups = (int64_t)sid.size();
        std::vector<uint32_t> gd(groups), gc(groups);
        if (groups > 0) {
            HGS_CUDA(cudaSetDevice(device));
            cudaStream_t st;
            HGS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            DevBuf<int64_t> d_rp, d_ci, d_srows, d_sptr, d_sid, d_off, d_out;
            DevBuf<uint64_t> d_seeds, d_state, d_recip;
            DevBuf<uint32_t> d_draws, d_dec, d_big;
            std::vector<uint64_t> recip((size_t)maxdeg + 1, 0);
            for (int64_t m = 1; m <= maxdeg; ++m) recip[m] = recip_of((uint64_t)m);
            auto up = [&](auto& buf, const auto* src_, size_t n) {
                buf.reserve(std::max<size_t>(n, 1));
                upload(buf.p, src_, n * sizeof(*src_), st);
            };
            up(d_rp, row_ptr, (size_t)n_rows + 1);
            up(d_ci, col_idx, (size_t)nnz);
            up(d_srows, srows.data(), srows.size());
            up(d_sptr, sptr.data(), sptr.size());
            up(d_sid, sid.data(), sid.size());
            up(d_off, out_off, (size_t)n_rows + 1);
            up(d_seeds, seeds, (size_t)n_streams);
            up(d_recip, recip.data(), recip.size());
            if (rng_state) up(d_state, rng_state, (size_t)n_streams * (rng == HGS_RNG_PHILOX ? 1 : 4));
            d_out.reserve(std::max<int64_t>(out_off[n_rows], 1));
            d_draws.reserve(groups);
            d_dec.reserve(groups);
            RowsParams p{};
            p.row_ptr = d_rp.p; p.col = d_ci.p; p.srows = d_srows.p; p.sptr = d_sptr.p; p.sid = d_sid.p;
            p.out_off = d_off.p; p.out_cols = d_out.p; p.seeds = d_seeds.p;
            p.state = rng_state ? d_state.p : nullptr; p.recip = d_recip.p;
            p.fanout = (int32_t)std::min<int64_t>(s, 1 << 30); p.groups = (int32_t)groups;
            p.draws = d_draws.p; p.decisions = d_dec.p;
            if (kmax > (int64_t)kLocalK) {
                d_big.reserve((size_t)groups * 3 * (size_t)kmax);
                p.big = d_big.p;
                p.big_k = (int32_t)kmax;
            }
            launch_sample_rows(p, rng == HGS_RNG_PHILOX, st);
            if (out_off[n_rows] > 0)
                HGS_CUDA(cudaMemcpyAsync(out_cols, d_out.p, sizeof(int64_t) * out_off[n_rows], cudaMemcpyDeviceToHost, st));
            HGS_CUDA(cudaMemcpyAsync(gd.data(), d_draws.p, sizeof(uint32_t) * groups, cudaMemcpyDeviceToHost, st));
            HGS_CUDA(cudaMemcpyAsync(gc.data(), d_dec.p, sizeof(uint32_t) * groups, cudaMemcpyDeviceToHost, st));
            HGS_CUDA(cudaStreamSynchronize(st));
            HGS_CUDA(cudaStreamDestroy(st));
        }
        if (draws) std::fill(draws, draws + n_streams, 0u);
        if (decisions) std::fill(decisions, decisions + n_streams, 0u);
        for (int64_t g = 0; g < groups; ++g) {
            if (draws) draws[sid[g]] = gd[g];
            if (decisions) decisions[sid[g]] = gc[g];
        }
    });
}

int hgs_sample_wait(hgs_sample* s, int64_t* counts) {
    return guarded([&] {
        if (!s) fail(HGS_EINVAL, "hgs: null sample handle");
        HGS_CUDA(cudaSetDevice(s->graph->g.device));
        if (s->pending) sample_finish(s, s->last_cfg, s->last_in);
        if (counts) {
            counts[0] = s->R;
            counts[1] = s->k;
            counts[2] = s->V;
            counts[3] = s->E;
        }
    });
}

int hgs_sample_copy_to_host(hgs_sample* s, const hgs_host_out* o) {
    return guarded([&] {
        if (!s || !o) fail(HGS_EINVAL, "hgs: null argument");
        HGS_CUDA(cudaSetDevice(s->graph->g.device));
        if (s->pending) fail(HGS_EINVAL, "hgs_sample_copy_to_host: run not waited for");
        cudaStream_t st = s->stream;
        const DevGraph& g = s->graph->g;
        auto cp = [&](void* dst, const void* src, size_t bytes) {
            if (dst && bytes) HGS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        };
        const size_t R = s->R, k = s->k, V = s->V, E = s->E;
        cp(o->batch_voff, s->batch_voff.p, 4 * (k + 1));
        cp(o->batch_eoff, s->batch_eoff.p, 4 * (k + 1));
        cp(o->comp_off, s->comp_off.p, 4 * (R + k));
        cp(o->l2g, s->l2g.p, 4 * V);
        cp(o->roots_local, s->roots_local.p, 4 * R);
        cp(o->e_row, s->e_row.p, 4 * E);
        cp(o->e_col, s->e_col.p, 4 * E);
        cp(o->e_gid, s->e_gid.p, 4 * E);
        if (s->gathered) {
            cp(o->xv, s->xv.p, 8 * V * g.f_v);
            cp(o->ye, s->ye.p, 8 * E * g.f_e);
            cp(o->lab, s->lab.p, E);
        }
        if (R) {
            cp(o->draws, s->draws.p, 4 * R);
            cp(o->decisions, s->decisions.p, 4 * R);
        }
        HGS_CUDA(cudaStreamSynchronize(st));
    });
}

int hgs_sample_device_views(hgs_sample* s, hgs_device_views* v) {
    return guarded([&] {
        if (!s || !v) fail(HGS_EINVAL, "hgs: null argument");
        // a pending run may still be re-run with larger buffers inside
        // hgs_sample_wait (capacity overflow), which can move every output
        if (s->pending) fail(HGS_EINVAL, "hgs_sample_device_views: run not waited for");
        v->batch_voff = s->batch_voff.p; v->batch_eoff = s->batch_eoff.p; v->comp_off = s->comp_off.p;
        v->l2g = s->l2g.p; v->roots_local = s->roots_local.p; v->e_row = s->e_row.p;
        v->e_col = s->e_col.p; v->e_gid = s->e_gid.p; v->root_voff = s->root_voff.p;
        v->root_eoff = s->root_eoff.p; v->xv = s->gathered ? s->xv.p : nullptr;
        v->ye = s->gathered ? s->ye.p : nullptr; v->lab = s->gathered ? s->lab.p : nullptr;
        v->draws = s->draws.p; v->decisions = s->decisions.p; v->touched = s->touched.p;
        v->touched_count = s->tcount.p; v->touched_stride = s->touched_stride;
        v->level_counts = s->level_counts.p;
    });
}

int hgs_sample_kernel_times(hgs_sample* s, float* ms) {  // 6 entries
    return guarded([&] {
        if (!s || !s->profiled) fail(HGS_EINVAL, "hgs_sample_kernel_times: last run was not profiled");
        HGS_CUDA(cudaSetDevice(s->graph->g.device));
        HGS_CUDA(cudaEventSynchronize(s->ev[5]));
        for (int i = 0; i < 5; ++i) HGS_CUDA(cudaEventElapsedTime(&ms[i], s->ev[i], s->ev[i + 1]));
        HGS_CUDA(cudaEventElapsedTime(&ms[5], s->ev[0], s->ev[5]));
    });
}

int hgs_sample_stats(hgs_sample* s, int64_t* stats, int32_t n) {
    return guarded([&] {
        if (!s || !stats) fail(HGS_EINVAL, "hgs: null argument");
        if (s->pending) fail(HGS_EINVAL, "hgs_sample_stats: run not waited for");
        if (n < 10 + s->depth) fail(HGS_EINVAL, "hgs_sample_stats: stats array too short");
        HGS_CUDA(cudaSetDevice(s->graph->g.device));
        sample_stats(s, stats, n);
    });
}

int hgs_sample_launches(hgs_sample* s, int64_t* n) {
    return guarded([&] {
        if (!s) fail(HGS_EINVAL, "hgs: null sample handle");
        *n = s->launches;
    });
}

int hgs_sample_reruns(hgs_sample* s, int64_t* n) {
    return guarded([&] {
        if (!s || !n) fail(HGS_EINVAL, "hgs: null argument");
        if (s->pending) fail(HGS_EINVAL, "hgs_sample_reruns: run not waited for");
        *n = s->reruns;
    });
}

}  // extern "C"
