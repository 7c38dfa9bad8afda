// hgs_internal.cuh — device graph store, workspaces and shared device helpers.
#pragma once
#include <functional>
#include <mutex>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "hgs.h"
#include "hgs_rng.cuh"

namespace hgs {

// Failure carried up to the C ABI: code = HGS_E*, message = reference text.
struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure(code, msg); }
[[noreturn]] void fail_cuda(cudaError_t e, const char* what);

#define HGS_CUDA(expr)                                          \
    do {                                                        \
        cudaError_t hgs_e_ = (expr);                            \
        if (hgs_e_ != cudaSuccess) ::hgs::fail_cuda(hgs_e_, #expr); \
    } while (0)

// Grow-only device buffer.
// L2 residency hints for the gathers: the feature tables are re-read ~10x
// per call by random rows while the outputs stream past them, so table loads
// carry an evict_last policy and output stores are evict-first (.cs).
#ifndef HGS_GATHER_HINT
#define HGS_GATHER_HINT 1
#endif
#ifndef HGS_KEEP_FRAC
#define HGS_KEEP_FRAC 1.0
#endif
__device__ __forceinline__ uint64_t l2_keep_policy() {
    uint64_t p = 0;
#if HGS_GATHER_HINT
    asm("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(p) : "f"((float)HGS_KEEP_FRAC));
#endif
    return p;
}
__device__ __forceinline__ uint4 ldg_keep(const uint4* a, uint64_t pol) {
#if HGS_GATHER_HINT
    uint4 r;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(a), "l"(pol));
    return r;
#else
    (void)pol;
    return __ldg(a);
#endif
}
__device__ __forceinline__ uint32_t ldg_keep(const uint32_t* a, uint64_t pol) {
#if HGS_GATHER_HINT
    uint32_t r;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol));
    return r;
#else
    (void)pol;
    return __ldg(a);
#endif
}

// The stream-ordered pool trims its memory back to the driver at every
// synchronisation by default (release threshold 0), which turns each
// cudaMallocAsync after a sync into a driver allocation; the library keeps
// the memory in the device's pool instead (like torch's caching allocator).
inline void pool_keep(int device) {
    static std::once_flag once[64];
    if (device < 0 || device >= 64) return;
    std::call_once(once[device], [device] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
}

// Device buffer from the device's stream-ordered pool. cudaMalloc/cudaFree
// cost milliseconds each on B200 boxes (a free unmaps; both synchronise), so
// graph builds and teardown allocate from the pool: reserve completes the
// allocation before returning, release waits for the device (cudaFree's
// implicit synchronisation) and hands the block back to the pool.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;
    void reserve(size_t n) {
        if (n <= cap) return;
        release();
        int dev = 0;
        HGS_CUDA(cudaGetDevice(&dev));
        pool_keep(dev);
        HGS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), (n ? n : 1) * sizeof(T), 0));
        HGS_CUDA(cudaStreamSynchronize(0));
        cap = n;
    }
    void release() {
        if (p) {
            cudaDeviceSynchronize();
            cudaFreeAsync(p, 0);
        }
        p = nullptr;
        cap = 0;
    }
    ~DevBuf() { release(); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// One CSR pattern on the device (int32 positions; n, nnz < 2^31).
struct DevCsr {
    DevBuf<int32_t> rp, ci;
    int32_t n = 0;
    int64_t nnz = 0;
    int32_t max_deg = 0;
    DevBuf<int2> ri;  // per row (start, degree): K1's row loads; built on first use as a walk
    bool ri_built = false;
};

// Device-resident event: the extraction matrix A (directed, edge ids), the
// walk matrices the expansion samples from, the bounded() reciprocal table
// and optional features. Built once per event.
struct DevGraph {
    int device = 0;
    int64_t n_rows = 0, n_cols = 0, nnz = 0;  // as given by the caller
    DevCsr a;                // extraction matrix: A minus explicit zeros
    DevBuf<int2> a_ri;       // per vertex of a: (row start, out-degree), one 8-byte load
    DevBuf<int32_t> a_gid;   // a position -> input CSR position (only if zeros dropped)
    bool has_gid = false;
    DevCsr a_full;           // full pattern of A (only if zeros dropped; else == a)
    bool has_full = false;
    DevBuf<int4> a_q;        // A's rows padded to 4-entry quads (pad entry = n_rows), built lazily for K2
    DevBuf<int4> a_qid;      // edge id (input CSR position) of every a_q entry, -1 for pads
    DevBuf<int2> a_rq;       // per vertex: (first quad, out-degree)
    bool quads_built = false;
    DevCsr walk_sym;         // pattern(A ∪ Aᵀ), built lazily by K0
    bool sym_built = false;
    DevBuf<uint8_t> neg_row; // rows of A holding a negative value (only if any)
    bool has_neg = false;
    DevBuf<uint64_t> recip;  // recip[m] = floor((2^64-1)/m), m in [1, recip_n)
    int32_t recip_n = 0;
    // features (gather_features)
    DevBuf<double> node_feat, edge_feat;
    DevBuf<uint8_t> labels;
    DevBuf<uint4> erec;      // f_e == 2: per edge 32 B = {features, label}: one sector per gathered edge
    int32_t f_v = 0, f_e = 0;
    bool has_features = false;
    cudaStream_t stream = nullptr;  // ingest stream
    // guards the lazily built parts (walk_sym, recip): sample handles on
    // different host threads may share one graph
    std::recursive_mutex lazy_mu;
    // hgs_graph_gather scratch (grow-only), guarded by gather_mu
    std::mutex gather_mu;
    DevBuf<int64_t> g_l2g, g_eid;
    DevBuf<double> g_xv, g_ye;
    DevBuf<uint8_t> g_lab;

    const DevCsr& full_pattern() const { return has_full ? a_full : a; }
    DevCsr& full_pattern() { return has_full ? a_full : a; }
};

void graph_build_walk_sym(DevGraph& g);  // K0 (graph.cu)
void graph_ensure_quads(DevGraph& g);    // a_q / a_rq for k_extract_bm (graph.cu)
// int64 edge-id CSR (host) -> device int32 A + a_ri, validated on the device (graph.cu)
void graph_ingest_device(DevGraph& g, const int64_t* row_ptr, const int64_t* col_idx, cudaStream_t st);

// Inputs of one sampling call (device pointers).
struct CallInputs {
    const int32_t* roots32 = nullptr;  // one of roots32 / roots64
    const int64_t* roots64 = nullptr;
    const int64_t* batch_off = nullptr;
    const uint64_t* seeds = nullptr;
    const uint64_t* state = nullptr;
    const hgs_seed_spec* spec = nullptr;  // seeds derived on the device when seeds == nullptr
    int64_t R = 0, k = 0;
    // multi-event call (hgs_sample_run_multi): event e samples graph events[e]
    // for the roots [ev_r0[e], ev_r0[e+1]) (host arrays, owned by the handle)
    int32_t n_events = 0;
    hgs_graph* const* events = nullptr;
    const int64_t* ev_r0 = nullptr;
};
void graph_ensure_recip(DevGraph& g, int32_t max_m);
// (row start, degree) per row of a walk CSR, built once (call under the graph's lazy_mu)
void csr_ensure_row_info(DevCsr& c, cudaStream_t st);

// Device exclusive scan: out[0..n] with out[n] = total (int32, total < 2^31).
void scan_exclusive_i32(const int32_t* in, int32_t* out, int64_t n, cudaStream_t st);
// Stable LSD radix sort of (uint32 key, int32 value) pairs in place (graph.cu).
void radix_sort_pairs(uint32_t* keys, int32_t* vals, uint32_t* tkeys, int32_t* tvals, int64_t n, int key_bits,
                      cudaStream_t st);
// Runs f with the C ABI's error convention (HGS_* code + hgs_last_error text).
int abi_guard(const std::function<void()>& f);

// ---- warp helpers -----------------------------------------------------------
#if defined(__CUDACC__)
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Full-warp ballot for code the caller knows to be converged: plain
// vote.sync without the divergence fallback ptxas wraps __ballot_sync in.
__device__ __forceinline__ unsigned ballot_nonneg(int x) {  // ballot(x >= 0)
    unsigned r;
    asm volatile("{ .reg .pred q; setp.ge.s32 q, %1, 0; vote.sync.ballot.b32 %0, q, 0xffffffff; }"
                 : "=r"(r) : "r"(x));
    return r;
}

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// Bitonic sort of 32*E keys held lane-major (lane l owns keys l*E .. l*E+E-1),
// ascending. Merges of width <= E are unrolled register compare-exchanges;
// wider merges run as (non-unrolled) loops over shuffle stages followed by
// the E-wide in-register tail, keeping the code small enough to stay in the
// instruction cache next to the extraction loop.
template <int E>
__device__ __forceinline__ void bitonic_lane_tail(uint32_t (&k)[E], bool up) {
#pragma unroll
    for (int stride = E >> 1; stride > 0; stride >>= 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if ((e & stride) == 0) {
                const int e2 = e | stride;
                const uint32_t x = k[e], y = k[e2];
                const bool sw = up ? (x > y) : (x < y);
                k[e] = sw ? y : x;
                k[e2] = sw ? x : y;
            }
        }
    }
}

template <int E>
__device__ __forceinline__ void warp_bitonic_sort(uint32_t (&k)[E]) {
    const int lane = lane_id();
    // merges of width 2..E: entirely inside a lane
#pragma unroll
    for (int size = 2; size <= E; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if ((e & stride) == 0) {
                    const int e2 = e | stride;
                    const bool up = (((lane * E + e) & size) == 0);
                    const uint32_t x = k[e], y = k[e2];
                    const bool sw = up ? (x > y) : (x < y);
                    k[e] = sw ? y : x;
                    k[e2] = sw ? x : y;
                }
            }
        }
    }
    // merges of width 2E..32E: shuffle stages, then the in-lane tail
#pragma unroll 1
    for (int size = 2 * E; size <= 32 * E; size <<= 1) {
        const bool up = ((lane * E) & size) == 0;
#pragma unroll 1
        for (int lm = size / (2 * E); lm > 0; lm >>= 1) {
            const bool keep_min = ((lane & lm) == 0) == up;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const uint32_t other = __shfl_xor_sync(kFull, k[e], lm);
                k[e] = keep_min ? min(k[e], other) : max(k[e], other);
            }
        }
        bitonic_lane_tail<E>(k, up);
    }
}
#endif

}  // namespace hgs

// Opaque handle types of the C ABI.
struct hgs_graph {
    hgs::DevGraph g;
};

struct hgs_sample {
    hgs_graph* graph = nullptr;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // inputs (device copies of host inputs)
    hgs::DevBuf<int64_t> roots64, boff64;
    hgs::DevBuf<uint64_t> seeds, rng_state;
    hgs::CallInputs last_in;
    hgs_seed_spec last_spec{};
    hgs_config last_cfg{};
    // expand scratch
    hgs::DevBuf<int32_t> touched, tcount, level_counts;
    hgs::DevBuf<int32_t> frontier;  // BFS-order copy of touched (HGS_FLAG_KEEP_FRONTIERS)
    bool frontier_kept = false;
    hgs::DevBuf<uint32_t> draws, decisions;
    int64_t touched_stride = 0;
    // extract scratch + offsets
    hgs::DevBuf<int32_t> root_nv, root_ne, root_rloc;
    hgs::DevBuf<int2> escratch;
    hgs::DevBuf<uint32_t> kbig;       // K1 choose() scratch for choices > kLocalK (wide rows only)
    hgs::DevBuf<unsigned char> k2g;  // K2 working sets in global memory (oversized sets only)
    int32_t e_stride = 512;
    hgs::DevBuf<int32_t> eoff_exact;  // exact per-root edge-slot offsets for an overflow re-run
    bool exact_slots = false;
    hgs::DevBuf<int64_t> scan_tmp;
    hgs::DevBuf<unsigned long long> stats_tmp;
    hgs::DevBuf<int32_t> ticket;  // [1]=error code [2..3]=error detail [4]=max E_r seen
    // outputs
    hgs::DevBuf<int32_t> l2g, roots_local, comp_off, batch_voff, batch_eoff;
    hgs::DevBuf<int32_t> e_row, e_col, e_gid, root_voff, root_eoff, root_scan;
    hgs::DevBuf<double> xv, ye;
    hgs::DevBuf<uint8_t> lab;
    size_t v_cap = 0, e_cap = 0;
    // pinned host mirror of small per-call state
    int32_t* h_state = nullptr;  // [0..4] error words, [8]=V, [9]=E
    // last call
    int64_t R = 0, k = 0, V = 0, E = 0;
    int64_t depth = 0, fanout = 0;
    int32_t gathered = 0, symmetrize = 1, rng = 0;
    bool pending = false;
    bool profiled = false;
    cudaEvent_t ev[6] = {};
    int64_t launches = 0;     // kernels launched by the last run, re-runs included
    int64_t reruns = 0;       // capacity re-runs of the last run (0 in a steady state)
    // multi-event call inputs (kept for a capacity re-run)
    std::vector<hgs_graph*> multi_graphs;
    std::vector<int64_t> multi_r0;
    // slice_components outputs (hgs_sample_slice)
    hgs::DevBuf<int32_t> sl_row, sl_col, sl_comp, sl_roots;
    // chunked pipeline: packing runs on a higher-priority side stream
    cudaStream_t aux = nullptr;
    std::vector<cudaEvent_t> chunk_ev;
};

namespace hgs {
void sample_enqueue(hgs_sample* s, const hgs_config& cfg, const CallInputs& in, bool rerun = false);
void sample_finish(hgs_sample* s, const hgs_config& cfg, const CallInputs& in);
void sample_stats(hgs_sample* s, int64_t* out, int n);
void gather_rows(DevGraph& g, const int64_t* d_l2g, int64_t V, const int64_t* d_eid, int64_t E,
                 double* d_xv, double* d_ye, uint8_t* d_lab, cudaStream_t st);
}  // namespace hgs
