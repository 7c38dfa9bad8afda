// consumer.cu — the training step's device-side use of a sampled batch
// (SURVEY.md §8f #3): slice_components over the device outputs of a run, the
// IGNN message-passing gather / scatter (forward and backward) and the
// rank-ordered reduction step of the coalesced gradient all-reduce.
//
//   slice_components   trainer.cpp:221-269. A batch's components are
//                      contiguous in the run's outputs (root_voff/root_eoff),
//                      so a slice is an offset range; only the batch-local
//                      ids are rebased (k_slice).
//   gather_rows        autodiff.cpp:121-136 (ignn.cpp:158-159): k_gather_rows.
//   scatter_add        autodiff.cpp:138-157 (ignn.cpp:163-164) and the
//                      backward of gather_rows, autodiff.cpp:260-270: the
//                      reference adds rows into each destination in index
//                      order, so the device sums each destination's segment of
//                      a stable sort of the indices in that order (k_scatter),
//                      bit-identical, no fp64 atomics.
//   allreduce_mean     trainer.cpp:84-123: per element the ranks' values are
//                      added in rank order, then scaled by 1/w (k_ordered_mean).
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "kernels.cuh"

struct hgs_scatter_plan {
    int device = 0;
    int64_t m = 0, n_rows = 0;
    const int32_t* idx = nullptr;  // the caller's index list (must outlive the plan)
    int32_t* perm = nullptr;       // positions of idx, stably sorted by destination (stream-ordered pool)
    int32_t* seg = nullptr;        // [n_rows + 1] segment offsets into perm
    cudaStream_t stream = nullptr;
};

namespace hgs {

namespace {

__global__ void k_slice(const int32_t* __restrict__ e_row, const int32_t* __restrict__ e_col, int64_t ne,
                        const int32_t* __restrict__ comp_off, const int32_t* __restrict__ roots_local, int64_t nc,
                        int32_t vshift, int32_t* __restrict__ o_row, int32_t* __restrict__ o_col,
                        int32_t* __restrict__ o_comp, int32_t* __restrict__ o_roots) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ne; t += stride) {
        o_row[t] = e_row[t] - vshift;
        o_col[t] = e_col[t] - vshift;
    }
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= nc; c += stride) {
        o_comp[c] = comp_off[c] - vshift;
        if (c < nc) o_roots[c] = roots_local[c] - vshift;
    }
}

// first position i with idx[i] outside [0, n) (atomicMin over positions);
// first[1] != 0 when the list is not non-decreasing
__global__ void k_first_bad(const int32_t* __restrict__ idx, int64_t m, int64_t n,
                            unsigned long long* __restrict__ first) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = idx[i];
        if (v < 0 || v >= n) atomicMin(first, (unsigned long long)i);
        if (i + 1 < m && idx[i + 1] < v) first[1] = 1ull;
    }
}

__global__ void k_iota(int32_t* __restrict__ p, int64_t m) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int32_t)i;
}

// seg[j] = first position with idx >= j over a non-decreasing index list
__global__ void k_segments_i32(const int32_t* __restrict__ sorted, int64_t m, int64_t n, int32_t* __restrict__ seg) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= n; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)sorted[mid] < j) lo = mid + 1; else hi = mid;
        }
        seg[j] = (int32_t)lo;
    }
}

__global__ void k_gather_rows(const double* __restrict__ x, int64_t cols, const int32_t* __restrict__ idx,
                              int64_t m, double* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if ((cols & 1) == 0) {  // rows as 16-byte pieces
        const int64_t q = cols >> 1, n2 = m * q;
        const double2* src = reinterpret_cast<const double2*>(x);
        double2* dst = reinterpret_cast<double2*>(out);
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += stride) {
            const int64_t i = e / q;
            dst[e] = __ldg(src + (int64_t)__ldg(idx + i) * q + (e - i * q));
        }
    } else {
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m * cols; e += stride) {
            const int64_t i = e / cols;
            out[e] = __ldg(x + (int64_t)__ldg(idx + i) * cols + (e - i * cols));
        }
    }
}

__global__ void k_iota_keys(const int32_t* __restrict__ idx, int64_t m, uint32_t* __restrict__ keys,
                            int32_t* __restrict__ vals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = (uint32_t)idx[i];
        vals[i] = (int32_t)i;
    }
}

// seg[j] = first position of the sorted keys with key >= j, j in [0, n]
__global__ void k_segments(const uint32_t* __restrict__ sorted, int64_t m, int64_t n, int32_t* __restrict__ seg) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= n; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)sorted[mid] < j) lo = mid + 1; else hi = mid;
        }
        seg[j] = (int32_t)lo;
    }
}

// out[j, c] (+)= y[perm[p], c] for p over j's segment, in ascending index order
__global__ void k_scatter(const double* __restrict__ y, int64_t cols, const int32_t* __restrict__ perm,
                          const int32_t* __restrict__ seg, int64_t n, int32_t accumulate, double* __restrict__ out) {
    const int64_t total = n * cols;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / cols, c = t - j * cols;
        double acc = accumulate ? out[t] : 0.0;
        const int32_t p1 = seg[j + 1];
        for (int32_t p = seg[j]; p < p1; ++p) acc = __dadd_rn(acc, __ldg(y + (int64_t)__ldg(perm + p) * cols + c));
        out[t] = acc;
    }
}

__global__ void k_ordered_mean(const double* __restrict__ parts, int32_t w, int64_t n, double inv_w,
                               double* __restrict__ out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        double s = parts[e];
        for (int32_t q = 1; q < w; ++q) s = __dadd_rn(s, parts[(int64_t)q * n + e]);
        out[e] = __dmul_rn(s, inv_w);
    }
}


unsigned grid_for(int64_t work) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 16));
}

// First out-of-range index, or -1 (synchronizes st); *sorted = non-decreasing.
int64_t first_bad_index(const int32_t* idx, int64_t m, int64_t n, cudaStream_t st, bool* sorted = nullptr) {
    if (sorted) *sorted = true;
    if (m <= 0) return -1;
    unsigned long long* d = nullptr;
    HGS_CUDA(cudaMallocAsync(&d, 2 * sizeof(unsigned long long), st));
    HGS_CUDA(cudaMemsetAsync(d, 0xff, sizeof(unsigned long long), st));
    HGS_CUDA(cudaMemsetAsync(d + 1, 0, sizeof(unsigned long long), st));
    k_first_bad<<<grid_for(m), 256, 0, st>>>(idx, m, n, d);
    HGS_CUDA(cudaGetLastError());
    unsigned long long h[2] = {0, 0};
    HGS_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaFreeAsync(d, st));
    HGS_CUDA(cudaStreamSynchronize(st));
    if (sorted) *sorted = h[1] == 0;
    return h[0] == ~0ULL ? -1 : (int64_t)h[0];
}

int32_t read_i32(const int32_t* p, cudaStream_t st) {
    int32_t v = 0;
    HGS_CUDA(cudaMemcpyAsync(&v, p, sizeof(v), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaStreamSynchronize(st));
    return v;
}

}  // namespace

}  // namespace hgs

using namespace hgs;

extern "C" {

int hgs_sample_slice(hgs_sample* s, int64_t batch, int64_t begin, int64_t end, hgs_slice_views* out) {
    return abi_guard([&] {
        if (!s || !out) fail(HGS_EINVAL, "hgs: null argument");
        if (s->pending) fail(HGS_EINVAL, "hgs_sample_slice: run not waited for");
        if (batch < 0 || batch >= s->k) fail(HGS_EINVAL, "hgs_sample_slice: batch out of range");
        HGS_CUDA(cudaSetDevice(s->graph->g.device));
        cudaStream_t st = s->stream;
        int64_t bo[2];
        HGS_CUDA(cudaMemcpyAsync(bo, s->last_in.batch_off + batch, sizeof(bo), cudaMemcpyDeviceToHost, st));
        HGS_CUDA(cudaStreamSynchronize(st));
        const int64_t f = bo[0], n_comp = bo[1] - bo[0];
        if (begin < 0 || end < begin || end > n_comp) fail(HGS_EINVAL, "slice_components: bad component range");
        int32_t h[5];  // root_voff[f], [f+begin], [f+end], root_eoff[f+begin], [f+end]
        HGS_CUDA(cudaMemcpyAsync(&h[0], s->root_voff.p + f, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HGS_CUDA(cudaMemcpyAsync(&h[1], s->root_voff.p + f + begin, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HGS_CUDA(cudaMemcpyAsync(&h[2], s->root_voff.p + f + end, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HGS_CUDA(cudaMemcpyAsync(&h[3], s->root_eoff.p + f + begin, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HGS_CUDA(cudaMemcpyAsync(&h[4], s->root_eoff.p + f + end, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HGS_CUDA(cudaStreamSynchronize(st));
        const int64_t nv = h[2] - h[1], ne = h[4] - h[3], nc = end - begin;
        const int32_t vshift = h[1] - h[0];  // batch-local id of the slice's first vertex
        s->sl_row.reserve((size_t)ne + 1);
        s->sl_col.reserve((size_t)ne + 1);
        s->sl_comp.reserve((size_t)nc + 1);
        s->sl_roots.reserve((size_t)nc + 1);
        k_slice<<<grid_for(std::max<int64_t>(ne, nc + 1)), 256, 0, st>>>(
            s->e_row.p + h[3], s->e_col.p + h[3], ne, s->comp_off.p + f + batch + begin, s->roots_local.p + f + begin,
            nc, vshift, s->sl_row.p, s->sl_col.p, s->sl_comp.p, s->sl_roots.p);
        HGS_CUDA(cudaGetLastError());
        // the slice is consumed on the caller's streams: make it complete here
        HGS_CUDA(cudaStreamSynchronize(st));
        const DevGraph& g = s->graph->g;
        out->n_vertices = nv;
        out->n_edges = ne;
        out->n_components = nc;
        out->f_v = s->gathered ? g.f_v : 0;
        out->f_e = s->gathered ? g.f_e : 0;
        out->e_row = s->sl_row.p;
        out->e_col = s->sl_col.p;
        out->comp_off = s->sl_comp.p;
        out->roots_local = s->sl_roots.p;
        out->l2g = s->l2g.p + h[1];
        out->e_gid = s->e_gid.p + h[3];
        out->xv = s->gathered ? s->xv.p + (size_t)h[1] * g.f_v : nullptr;
        out->ye = s->gathered ? s->ye.p + (size_t)h[3] * g.f_e : nullptr;
        out->lab = s->gathered ? s->lab.p + h[3] : nullptr;
    });
}

int hgs_gather_rows(const double* x, int64_t n_rows, int64_t cols, const int32_t* idx, int64_t m, double* out,
                    void* stream) {
    return abi_guard([&] {
        if (m < 0 || cols < 0 || n_rows < 0) fail(HGS_EINVAL, "gather_rows: negative size");
        cudaStream_t st = (cudaStream_t)stream;
        int dev = 0;
        HGS_CUDA(cudaGetDevice(&dev));
        pool_keep(dev);
        const int64_t bad = first_bad_index(idx, m, n_rows, st);
        if (bad >= 0)
            fail(HGS_EINVAL, "gather_rows: index " + std::to_string(read_i32(idx + bad, st)) + " out of range");
        if (m * cols == 0) return;
        k_gather_rows<<<grid_for(m * cols), 256, 0, st>>>(x, cols, idx, m, out);
        HGS_CUDA(cudaGetLastError());
    });
}

int hgs_scatter_plan_create(int device, const int32_t* idx, int64_t m, int64_t n_rows, void* stream,
                            hgs_scatter_plan** out) {
    return abi_guard([&] {
        if (!out) fail(HGS_EINVAL, "hgs: null argument");
        if (m < 0 || n_rows < 0 || m >= ((int64_t)1 << 31) || n_rows >= ((int64_t)1 << 31))
            fail(HGS_ERANGE, "scatter_add: sizes beyond 2^31 are not supported by this build");
        HGS_CUDA(cudaSetDevice(device));
        pool_keep(device);
        cudaStream_t st = (cudaStream_t)stream;
        bool sorted = true;
        const int64_t bad = first_bad_index(idx, m, n_rows, st, &sorted);
        if (bad >= 0)
            fail(HGS_EINVAL, "scatter_add: index " + std::to_string(read_i32(idx + bad, st)) + " out of range");
        auto* p = new hgs_scatter_plan();
        p->device = device;
        p->m = m;
        p->n_rows = n_rows;
        p->idx = idx;
        p->stream = st;
        // plan buffers and temporaries come from the stream-ordered pool: no
        // cudaMalloc / device-wide synchronisation per plan
        HGS_CUDA(cudaMallocAsync(&p->perm, sizeof(int32_t) * (size_t)std::max<int64_t>(m, 1), st));
        HGS_CUDA(cudaMallocAsync(&p->seg, sizeof(int32_t) * (size_t)(n_rows + 1), st));
        if (sorted) {  // e.g. the row list of a batch (CSR order): identity permutation
            if (m > 0) k_iota<<<grid_for(m), 256, 0, st>>>(p->perm, m);
            k_segments_i32<<<grid_for(n_rows + 1), 256, 0, st>>>(idx, m, n_rows, p->seg);
        } else {
            uint32_t *keys = nullptr, *tkeys = nullptr;
            int32_t* tvals = nullptr;
            HGS_CUDA(cudaMallocAsync(&keys, sizeof(uint32_t) * (size_t)m, st));
            HGS_CUDA(cudaMallocAsync(&tkeys, sizeof(uint32_t) * (size_t)m, st));
            HGS_CUDA(cudaMallocAsync(&tvals, sizeof(int32_t) * (size_t)m, st));
            k_iota_keys<<<grid_for(m), 256, 0, st>>>(idx, m, keys, p->perm);
            int bits = 1;
            while (bits < 32 && ((int64_t)1 << bits) < n_rows) ++bits;
            radix_sort_pairs(keys, p->perm, tkeys, tvals, m, bits, st);
            k_segments<<<grid_for(n_rows + 1), 256, 0, st>>>(keys, m, n_rows, p->seg);
            HGS_CUDA(cudaFreeAsync(keys, st));
            HGS_CUDA(cudaFreeAsync(tkeys, st));
            HGS_CUDA(cudaFreeAsync(tvals, st));
        }
        HGS_CUDA(cudaGetLastError());
        *out = p;
    });
}

int hgs_scatter_add(const hgs_scatter_plan* plan, const double* y, int64_t cols, double* out, int32_t accumulate,
                    void* stream) {
    return abi_guard([&] {
        if (!plan) fail(HGS_EINVAL, "hgs: null plan");
        if (cols < 0) fail(HGS_EINVAL, "scatter_add: negative size");
        if (plan->n_rows * cols == 0) return;
        HGS_CUDA(cudaSetDevice(plan->device));
        cudaStream_t st = (cudaStream_t)stream;
        if (st != plan->stream) HGS_CUDA(cudaStreamSynchronize(plan->stream));  // plan built on another stream
        k_scatter<<<grid_for(plan->n_rows * cols), 256, 0, st>>>(y, cols, plan->perm, plan->seg, plan->n_rows,
                                                                  accumulate, out);
        HGS_CUDA(cudaGetLastError());
    });
}

int hgs_gather_rows_planned(const hgs_scatter_plan* plan, const double* x, int64_t n_rows, int64_t cols, double* out,
                            void* stream) {
    return abi_guard([&] {
        if (!plan) fail(HGS_EINVAL, "hgs: null plan");
        if (n_rows != plan->n_rows) fail(HGS_EINVAL, "gather_rows: table rows differ from the plan's");
        if (plan->m * cols == 0) return;
        HGS_CUDA(cudaSetDevice(plan->device));
        cudaStream_t st = (cudaStream_t)stream;
        if (st != plan->stream) HGS_CUDA(cudaStreamSynchronize(plan->stream));
        k_gather_rows<<<grid_for(plan->m * cols), 256, 0, st>>>(x, cols, plan->idx, plan->m, out);
        HGS_CUDA(cudaGetLastError());
    });
}

int hgs_scatter_plan_destroy(hgs_scatter_plan* plan) {
    return abi_guard([&] {
        if (!plan) return;
        HGS_CUDA(cudaSetDevice(plan->device));
        HGS_CUDA(cudaFreeAsync(plan->perm, plan->stream));
        HGS_CUDA(cudaFreeAsync(plan->seg, plan->stream));
        delete plan;
    });
}

int hgs_ordered_mean(const double* parts, int32_t w, int64_t n, double* out, void* stream) {
    return abi_guard([&] {
        if (w < 1) fail(HGS_EINVAL, "run_workers: world_size must be >= 1");
        if (n < 0) fail(HGS_EINVAL, "allreduce: negative length");
        if (n == 0) return;
        const double inv_w = 1.0 / static_cast<double>(w);
        k_ordered_mean<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(parts, w, n, inv_w, out);
        HGS_CUDA(cudaGetLastError());
    });
}

}  // extern "C"
