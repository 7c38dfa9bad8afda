// graph.cu — device graph store and K0 (walk CSR build).
//
// K0 restates symmetrize_pattern (sparse.cpp:260-272: pattern of A ∪ Aᵀ,
// canonical = rows ascending, columns strictly ascending) as
//   (1) a stable LSD radix sort of A's entries by column with the row as
//       payload — the transpose, whose in-lists come out row-ascending
//       because the input is row-major;
//   (2) a per-row merge of the (sorted) out-list with the (sorted) in-list,
//       dropping duplicates: a count pass, a scan, a write pass.
// It runs once per graph (ingest), not per sampling call.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "hgs_internal.cuh"

namespace hgs {

void fail_cuda(cudaError_t e, const char* what) {
    fail(HGS_ECUDA, std::string("CUDA error ") + cudaGetErrorName(e) + ": " +
                        cudaGetErrorString(e) + " (" + what + ")");
}

// ---------------------------------------------------------------------------
// exclusive scan (int32), out[n] = total

namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* warp_tot, int32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t inc = warp_incl_scan(v);
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        int32_t t = lane < nw ? warp_tot[lane] : 0;
        const int32_t ti = warp_incl_scan(t);
        if (lane < nw) warp_tot[lane] = ti - t;
        if (lane == nw - 1) warp_tot[32] = ti;
    }
    __syncthreads();
    total = warp_tot[32];
    const int32_t r = warp_tot[warp] + inc - v;
    __syncthreads();
    return r;
}

__global__ void k_scan_tiles(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                             int64_t n, int32_t* __restrict__ tile_sums) {
    __shared__ int32_t wt[33];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int32_t x[kScanItems];
    int32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        x[i] = (base + i < n) ? in[base + i] : 0;
        s += x[i];
    }
    int32_t total;
    int32_t run = block_excl_scan(s, wt, total);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = run;
        run += x[i];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void k_scan_add(int32_t* __restrict__ out, int64_t n,
                           const int32_t* __restrict__ tile_off) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    const int32_t add = tile_off[blockIdx.x];
    for (int i = threadIdx.x; i < kScanTile; i += blockDim.x)
        if (base + i < n) out[base + i] += add;
}

__global__ void k_set_total(int32_t* out, int64_t n, const int32_t* tile_off, int64_t tiles) {
    out[n] = tile_off[tiles];
}

}  // namespace

void scan_exclusive_i32(const int32_t* in, int32_t* out, int64_t n, cudaStream_t st) {
    if (n <= 0) {
        HGS_CUDA(cudaMemsetAsync(out, 0, sizeof(int32_t), st));
        return;
    }
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles == 1) {  // one tile: its sum is the total
        k_scan_tiles<<<1, kScanThreads, 0, st>>>(in, out, n, out + n);
        HGS_CUDA(cudaGetLastError());
        return;
    }
    int32_t* sums = nullptr;
    HGS_CUDA(cudaMallocAsync(&sums, sizeof(int32_t) * (2 * tiles + 2), st));
    int32_t* offs = sums + tiles + 1;
    k_scan_tiles<<<(unsigned)tiles, kScanThreads, 0, st>>>(in, out, n, sums);
    HGS_CUDA(cudaGetLastError());
    scan_exclusive_i32(sums, offs, tiles, st);  // offs[tiles] = total
    k_scan_add<<<(unsigned)tiles, kScanThreads, 0, st>>>(out, n, offs);
    k_set_total<<<1, 1, 0, st>>>(out, n, offs, tiles);
    HGS_CUDA(cudaGetLastError());
    HGS_CUDA(cudaFreeAsync(sums, st));
}

// ---------------------------------------------------------------------------
// stable LSD radix sort of (uint32 key, int32 value) pairs, 8-bit digits.
// Each 256-thread block owns a tile of 2048 keys; every warp a contiguous
// 256-key sub-tile it walks in order, so ranks are stable: peers with the
// same digit are ranked with __match_any_sync + lane order, warps in warp
// order, tiles in tile order (digit-major histogram scan).

namespace {

constexpr int kRadix = 256;
constexpr int kSortThreads = 256;
constexpr int kWarpKeys = 256;
constexpr int kSortTile = (kSortThreads / 32) * kWarpKeys;

__global__ void k_radix_hist(const uint32_t* __restrict__ keys, int64_t n, int shift,
                             int32_t* __restrict__ hist, int64_t tiles) {
    __shared__ int32_t cnt[kRadix];
    for (int i = threadIdx.x; i < kRadix; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int i = threadIdx.x; i < kSortTile; i += blockDim.x)
        if (base + i < n) atomicAdd(&cnt[(keys[base + i] >> shift) & 0xff], 1);
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += blockDim.x) hist[(int64_t)d * tiles + blockIdx.x] = cnt[d];
}

__global__ void k_radix_scatter(const uint32_t* __restrict__ keys, const int32_t* __restrict__ vals,
                                int64_t n, int shift, const int32_t* __restrict__ offs,
                                int64_t tiles, uint32_t* __restrict__ okeys,
                                int32_t* __restrict__ ovals) {
    __shared__ int32_t wc[kSortThreads / 32][kRadix];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (kSortThreads / 32) * kRadix; i += blockDim.x) (&wc[0][0])[i] = 0;
    __syncthreads();
    const int64_t wbase = (int64_t)blockIdx.x * kSortTile + (int64_t)warp * kWarpKeys;
    for (int step = 0; step < kWarpKeys / 32; ++step) {
        const int64_t idx = wbase + step * 32 + lane;
        const bool ok = idx < n;
        const unsigned act = __ballot_sync(kFull, ok);
        if (ok) {
            const uint32_t d = (keys[idx] >> shift) & 0xff;
            const unsigned peers = __match_any_sync(act, d);
            if ((__ffs(peers) - 1) == lane) wc[warp][d] += __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += blockDim.x) {
        int32_t run = offs[(int64_t)d * tiles + blockIdx.x];
        for (int w = 0; w < kSortThreads / 32; ++w) {
            const int32_t t = wc[w][d];
            wc[w][d] = run;
            run += t;
        }
    }
    __syncthreads();
    for (int step = 0; step < kWarpKeys / 32; ++step) {
        const int64_t idx = wbase + step * 32 + lane;
        const bool ok = idx < n;
        const unsigned act = __ballot_sync(kFull, ok);
        uint32_t key = 0, d = 0;
        unsigned peers = 0;
        int32_t pos = 0;
        if (ok) {
            key = keys[idx];
            d = (key >> shift) & 0xff;
            peers = __match_any_sync(act, d);
            pos = wc[warp][d] + __popc(peers & ((1u << lane) - 1u));
            okeys[pos] = key;
            ovals[pos] = vals[idx];
        }
        __syncwarp();
        if (ok && (__ffs(peers) - 1) == lane) wc[warp][d] += __popc(peers);
        __syncwarp();
    }
}

}  // namespace

// Sorts (keys, vals) in place using the given temporaries; key_bits = number
// of low bits that can be nonzero.
void radix_sort_pairs(uint32_t* keys, int32_t* vals, uint32_t* tkeys, int32_t* tvals, int64_t n, int key_bits,
                      cudaStream_t st) {
    if (n <= 1) return;
    const int64_t tiles = (n + kSortTile - 1) / kSortTile;
    int32_t* hist = nullptr;
    HGS_CUDA(cudaMallocAsync(&hist, sizeof(int32_t) * (kRadix * tiles * 2 + 1), st));
    int32_t* offs = hist + kRadix * tiles;
    uint32_t *ka = keys, *kb = tkeys;
    int32_t *va = vals, *vb = tvals;
    int passes = 0;
    for (int shift = 0; shift < key_bits; shift += 8, ++passes) {
        k_radix_hist<<<(unsigned)tiles, kSortThreads, 0, st>>>(ka, n, shift, hist, tiles);
        scan_exclusive_i32(hist, offs, kRadix * tiles, st);
        k_radix_scatter<<<(unsigned)tiles, kSortThreads, 0, st>>>(ka, va, n, shift, offs, tiles, kb, vb);
        HGS_CUDA(cudaGetLastError());
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (passes & 1) {
        HGS_CUDA(cudaMemcpyAsync(keys, ka, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st));
        HGS_CUDA(cudaMemcpyAsync(vals, va, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
    }
    HGS_CUDA(cudaFreeAsync(hist, st));
}

// ---------------------------------------------------------------------------
// K0 kernels

namespace {

__global__ void k_row_ids(const int32_t* __restrict__ rp, int32_t n, int32_t* __restrict__ rows) {
    for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x)
        for (int32_t k = rp[u]; k < rp[u + 1]; ++k) rows[k] = u;
}

// t_rp[v] = first position of key >= v in the sorted column keys.
__global__ void k_lower_bound(const uint32_t* __restrict__ sorted, int64_t nnz, int32_t n,
                              int32_t* __restrict__ t_rp) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (sorted[mid] < (uint32_t)v) lo = mid + 1; else hi = mid;
        }
        t_rp[v] = (int32_t)lo;
    }
}

// Merge out-list and in-list of row u (both ascending), unique. WRITE=false
// counts into cnt[u]; WRITE=true writes at w_ci[w_rp[u]...].
template <bool WRITE>
__global__ void k_merge_rows(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                             const int32_t* __restrict__ t_rp, const int32_t* __restrict__ t_ci,
                             int32_t n, int32_t* __restrict__ cnt, const int32_t* __restrict__ w_rp,
                             int32_t* __restrict__ w_ci, int32_t* __restrict__ max_deg) {
    for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        int32_t i = rp[u];
        const int32_t ie = rp[u + 1];
        int32_t j = t_rp[u];
        const int32_t je = t_rp[u + 1];
        int32_t w = WRITE ? w_rp[u] : 0;
        int32_t c = 0;
        int64_t last = -1;
        while (i < ie || j < je) {
            int32_t v;
            if (j >= je || (i < ie && ci[i] <= t_ci[j])) v = ci[i++];
            else v = t_ci[j++];
            if (v == last) continue;
            last = v;
            if (WRITE) w_ci[w++] = v;
            ++c;
        }
        if (!WRITE) {
            cnt[u] = c;
            atomicMax(max_deg, c);
        }
    }
}

__global__ void k_recip(uint64_t* r, int32_t n) {
    for (int32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < n; m += gridDim.x * blockDim.x)
        r[m] = m ? (~0ULL / (uint64_t)m) : 0ULL;
}

}  // namespace

namespace {
__global__ void k_csr_row_info(const int32_t* __restrict__ rp, int32_t n, int2* __restrict__ ri) {
    for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        const int32_t b = rp[u];
        ri[u] = make_int2(b, rp[u + 1] - b);
    }
}
}  // namespace

void csr_ensure_row_info(DevCsr& c, cudaStream_t st) {
    if (c.ri_built) return;
    c.ri.reserve((size_t)std::max<int32_t>(c.n, 1));
    if (c.n > 0) {
        k_csr_row_info<<<(unsigned)std::min<int64_t>((c.n + 255) / 256, 148 * 8), 256, 0, st>>>(c.rp.p, c.n, c.ri.p);
        HGS_CUDA(cudaGetLastError());
    }
    HGS_CUDA(cudaStreamSynchronize(st));
    c.ri_built = true;
}

void graph_build_walk_sym(DevGraph& g) {
    std::lock_guard<std::recursive_mutex> lock(g.lazy_mu);
    if (g.sym_built) return;
    const DevCsr& a = g.full_pattern();
    const int32_t n = a.n;
    const int64_t nnz = a.nnz;
    cudaStream_t st = g.stream;
    DevCsr& w = g.walk_sym;
    w.n = n;
    w.rp.reserve((size_t)n + 1);
    DevBuf<uint32_t> keys, tkeys;
    DevBuf<int32_t> vals, tvals, t_rp, cnt, maxd;
    keys.reserve(nnz); tkeys.reserve(nnz); vals.reserve(nnz); tvals.reserve(nnz);
    t_rp.reserve((size_t)n + 1); cnt.reserve((size_t)n + 1); maxd.reserve(1);
    const int threads = 256;
    const unsigned rows_grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 1 << 16));
    if (nnz > 0) {
        HGS_CUDA(cudaMemcpyAsync(keys.p, a.ci.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, st));
        k_row_ids<<<rows_grid, threads, 0, st>>>(a.rp.p, n, vals.p);
        int bits = 1;
        while (bits < 32 && ((int64_t)1 << bits) < (int64_t)n) ++bits;
        radix_sort_pairs(keys.p, vals.p, tkeys.p, tvals.p, nnz, bits, st);
    }
    k_lower_bound<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 1 + threads - 1) / threads, 1 << 16)), threads, 0, st>>>(
        keys.p, nnz, n, t_rp.p);
    HGS_CUDA(cudaMemsetAsync(maxd.p, 0, sizeof(int32_t), st));
    k_merge_rows<false><<<rows_grid, threads, 0, st>>>(a.rp.p, a.ci.p, t_rp.p, vals.p, n, cnt.p,
                                                       nullptr, nullptr, maxd.p);
    HGS_CUDA(cudaGetLastError());
    scan_exclusive_i32(cnt.p, w.rp.p, n, st);
    int32_t h[2];
    HGS_CUDA(cudaMemcpyAsync(&h[0], w.rp.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaMemcpyAsync(&h[1], maxd.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaStreamSynchronize(st));
    w.nnz = h[0];
    w.max_deg = h[1];
    w.ci.reserve((size_t)w.nnz);
    k_merge_rows<true><<<rows_grid, threads, 0, st>>>(a.rp.p, a.ci.p, t_rp.p, vals.p, n, nullptr,
                                                      w.rp.p, w.ci.p, nullptr);
    HGS_CUDA(cudaGetLastError());
    HGS_CUDA(cudaStreamSynchronize(st));
    g.sym_built = true;
    graph_ensure_recip(g, w.max_deg);
}

// ---------------------------------------------------------------------------
// ingest on the device (edge-id A, no values): int64 CSR -> int32 CSR + a_ri,
// validated as CsrMatrix::validate does (row_ptr[0] == 0, non-decreasing,
// columns in range), max out-degree reduced on the way. The first offending
// entry in row-major order is reported (atomicMin over its position).

__global__ void k_ingest_rows(const int64_t* __restrict__ rp64, int32_t n, int32_t* __restrict__ rp32,
                              int2* __restrict__ ari, int32_t* __restrict__ st) {
    // st[0] = max degree, st[1] = first row with row_ptr decreasing (or INT_MAX)
    int32_t md = 0;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= n; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = rp64[u];
        rp32[u] = (int32_t)b;
        if (u < n) {
            const int64_t e = rp64[u + 1];
            if (e < b) atomicMin(&st[1], (int32_t)u);
            const int32_t d = e > b ? (int32_t)(e - b) : 0;
            ari[u] = make_int2((int32_t)b, d);
            md = max(md, d);
        }
    }
    md = __reduce_max_sync(kFull, md);
    if ((threadIdx.x & 31) == 0) atomicMax(&st[0], md);
}

__global__ void k_ingest_cols(const int64_t* __restrict__ ci64, int64_t nnz, int64_t n_cols,
                              int32_t* __restrict__ ci32, unsigned long long* __restrict__ first_bad) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = ci64[k];
        ci32[k] = (int32_t)c;
        if (c < 0 || c >= n_cols) atomicMin(first_bad, (unsigned long long)k);
    }
}

void graph_ingest_device(DevGraph& g, const int64_t* row_ptr, const int64_t* col_idx, cudaStream_t st) {
    const int32_t n = (int32_t)g.n_rows;
    const int64_t nnz = g.nnz;
    DevBuf<int64_t> rp64, ci64;
    DevBuf<int32_t> stat;
    DevBuf<unsigned long long> bad;
    rp64.reserve((size_t)n + 1);
    ci64.reserve((size_t)std::max<int64_t>(nnz, 1));
    stat.reserve(2);
    bad.reserve(1);
    HGS_CUDA(cudaMemcpyAsync(rp64.p, row_ptr, sizeof(int64_t) * ((size_t)n + 1), cudaMemcpyHostToDevice, st));
    if (nnz) HGS_CUDA(cudaMemcpyAsync(ci64.p, col_idx, sizeof(int64_t) * (size_t)nnz, cudaMemcpyHostToDevice, st));
    const int32_t init[2] = {0, 0x7fffffff};
    HGS_CUDA(cudaMemcpyAsync(stat.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    HGS_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
    g.a.n = n;
    g.a.nnz = nnz;
    g.a.rp.reserve((size_t)n + 1);
    g.a.ci.reserve((size_t)std::max<int64_t>(nnz, 1));
    g.a_ri.reserve((size_t)std::max<int32_t>(n, 1));
    k_ingest_rows<<<148 * 4, 256, 0, st>>>(rp64.p, n, g.a.rp.p, g.a_ri.p, stat.p);
    if (nnz) k_ingest_cols<<<148 * 8, 256, 0, st>>>(ci64.p, nnz, g.n_cols, g.a.ci.p, bad.p);
    HGS_CUDA(cudaGetLastError());
    int32_t hs[2];
    unsigned long long hb = 0;
    HGS_CUDA(cudaMemcpyAsync(hs, stat.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaStreamSynchronize(st));
    // the first failure in row-major order, as the host loop would meet it:
    // row u's pointers are checked before its entries
    const int64_t u_bad = hs[1] != 0x7fffffff ? hs[1] : (int64_t)n;  // row_ptr monotone on [0, u_bad]
    const bool col_first = hb != ~0ULL && (int64_t)hb < row_ptr[u_bad];
    if (hs[1] != 0x7fffffff && !col_first) fail(HGS_EINVAL, "hgs_graph_create: row_ptr not non-decreasing");
    if (hb != ~0ULL) {  // first bad entry in row-major order: its row by binary search
        const int64_t k = (int64_t)hb;
        const int64_t u = std::upper_bound(row_ptr, row_ptr + u_bad + 1, k) - row_ptr - 1;
        fail(HGS_EINVAL, "CsrMatrix: entry (" + std::to_string(u) + ", " + std::to_string(col_idx[k]) +
                             ") out of range for " + std::to_string(g.n_rows) + "x" + std::to_string(g.n_cols));
    }
    g.a.max_deg = hs[0];
}

// ---------------------------------------------------------------------------
// Quad layout of A for k_extract_bm: every row padded to a multiple of 4
// entries (pad = n, never a vertex) so a lane reads 4 entries of ONE row with
// one 16-byte load. Entries are stored as probe words of k_extract_bm's
// directory: ((c >> 4) * 4) << 8 | (15 - (c & 15)) = the byte offset of the
// directory word holding column c and the left shift that moves c's member bit
// to bit 15. a_qid holds the entries' edge ids (input CSR positions, through
// a_gid when explicit zeros were dropped) and a_rq[v] = (first quad, out-degree).

__global__ void k_quad_counts(const int32_t* __restrict__ rp, int32_t n, int32_t* __restrict__ qc) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        qc[v] = (rp[v + 1] - rp[v] + 3) >> 2;
}

__global__ void k_quad_fill(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const int32_t* __restrict__ gid, int32_t n, const int32_t* __restrict__ qrp,
                            int4* __restrict__ aq, int4* __restrict__ aqid, int2* __restrict__ arq) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int32_t b = rp[v], d = rp[v + 1] - b, q0 = qrp[v];
        arq[v] = make_int2(q0, d);
        for (int32_t i = 0; 4 * i < d; ++i) {
            int32_t c[4], e[4];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const int32_t k = b + 4 * i + s;
                const bool in = 4 * i + s < d;
                const uint32_t col = in ? (uint32_t)ci[k] : (uint32_t)n;
                c[s] = (int32_t)((((col >> 4) << 2) << 8) | (15u - (col & 15u)));
                e[s] = in ? (gid ? gid[k] : k) : -1;
            }
            aq[q0 + i] = make_int4(c[0], c[1], c[2], c[3]);
            aqid[q0 + i] = make_int4(e[0], e[1], e[2], e[3]);
        }
    }
}

void graph_ensure_quads(DevGraph& g) {
    std::lock_guard<std::recursive_mutex> lock(g.lazy_mu);
    if (g.quads_built) return;
    const int32_t n = g.a.n;
    cudaStream_t st = g.stream;
    DevBuf<int32_t> qc, qrp;
    qc.reserve((size_t)n + 1);
    qrp.reserve((size_t)n + 1);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
    k_quad_counts<<<grid, 256, 0, st>>>(g.a.rp.p, n, qc.p);
    HGS_CUDA(cudaGetLastError());
    scan_exclusive_i32(qc.p, qrp.p, n, st);
    int32_t nq = 0;
    HGS_CUDA(cudaMemcpyAsync(&nq, qrp.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaStreamSynchronize(st));
    g.a_q.reserve((size_t)std::max(nq, 1));
    g.a_qid.reserve((size_t)std::max(nq, 1));
    g.a_rq.reserve((size_t)std::max(n, 1));
    k_quad_fill<<<grid, 256, 0, st>>>(g.a.rp.p, g.a.ci.p, g.has_gid ? g.a_gid.p : nullptr, n, qrp.p, g.a_q.p,
                                      g.a_qid.p, g.a_rq.p);
    HGS_CUDA(cudaGetLastError());
    HGS_CUDA(cudaStreamSynchronize(st));
    g.quads_built = true;
}

void graph_ensure_recip(DevGraph& g, int32_t max_m) {
    std::lock_guard<std::recursive_mutex> lock(g.lazy_mu);
    const int32_t need = max_m + 1;
    if (need <= g.recip_n) return;
    g.recip.release();
    g.recip.reserve((size_t)need);
    k_recip<<<(unsigned)std::max(1, std::min((need + 255) / 256, 1 << 16)), 256, 0, g.stream>>>(g.recip.p, need);
    HGS_CUDA(cudaGetLastError());
    HGS_CUDA(cudaStreamSynchronize(g.stream));
    g.recip_n = need;
}

}  // namespace hgs
