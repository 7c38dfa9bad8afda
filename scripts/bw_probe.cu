// HBM bandwidth probe for write-dominated streams (calibrates the pack /
// gather kernels): write-only (default and evict-first stores), copy, and
// gather-from-an-L2-resident-table + write.
// build+run: nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/bw_probe.cu -o /tmp/bw && /tmp/bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write(double2* __restrict__ d, size_t n, int cs) {
    const size_t st = (size_t)gridDim.x * blockDim.x;
    const double2 v = make_double2(1.0, 2.0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += st) {
        if (cs) __stcs(d + i, v); else d[i] = v;
    }
}
__global__ void k_copy(const double2* __restrict__ s, double2* __restrict__ d, size_t n) {
    const size_t st = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += st) __stcs(d + i, __ldg(s + i));
}
__global__ void k_gather(const double2* __restrict__ t, int tn, double2* __restrict__ d, size_t n) {
    const size_t st = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += st) {
        const unsigned h = (unsigned)(i * 2654435761u) % (unsigned)tn;
        __stcs(d + i, __ldg(t + h));
    }
}

// gather rows of W 16-byte pieces (row = W*16 B, rows aligned), W adjacent
// threads per row: one warp instruction touches 32/W rows
template <int W>
__global__ void k_gather_rows(const double2* __restrict__ t, int rows, double2* __restrict__ d, size_t n) {
    const size_t st = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += st) {
        const size_t row = i / W;
        const unsigned h = (unsigned)(row * 2654435761u) % (unsigned)rows;
        __stcs(d + i, __ldg(t + (size_t)h * W + (i % W)));
    }
}

int main() {
    const size_t bytes = 1ull << 30, n = bytes / 16;
    double2 *a, *b, *t;
    cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&t, 6 << 20);
    cudaMemset(a, 0, bytes); cudaMemset(b, 0, bytes); cudaMemset(t, 0, 6 << 20);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int gm : {8, 32}) {
        const int grid = sms * gm;
        auto run = [&](const char* name, auto fn, double gb) {
            fn(); cudaDeviceSynchronize();
            cudaEventRecord(e0); for (int r = 0; r < 10; ++r) fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
            printf("grid %3dx%d  %-22s %7.3f ms  %6.0f GB/s\n", gm, 256, name, ms, gb / ms * 1e3);
        };
        run("write (evict-first)", [&] { k_write<<<grid, 256>>>(a, n, 1); }, bytes / 1e9);
        run("write (default)", [&] { k_write<<<grid, 256>>>(a, n, 0); }, bytes / 1e9);
        run("copy (r+w)", [&] { k_copy<<<grid, 256>>>(a, b, n); }, 2 * bytes / 1e9);
        run("L2 gather + write", [&] { k_gather<<<grid, 256>>>(t, (6 << 20) / 16, a, n); }, bytes / 1e9);
        run("L1 gather(64KB) + write", [&] { k_gather<<<grid, 256>>>(t, (64 << 10) / 16, a, n); }, bytes / 1e9);
        run("L2 gather 32B rows", [&] { k_gather_rows<2><<<grid, 256>>>(t, (6 << 20) / 32, a, n); }, bytes / 1e9);
        run("L2 gather 64B rows", [&] { k_gather_rows<4><<<grid, 256>>>(t, (6 << 20) / 64, a, n); }, bytes / 1e9);
        run("L2 gather 128B rows", [&] { k_gather_rows<8><<<grid, 256>>>(t, (6 << 20) / 128, a, n); }, bytes / 1e9);
        run("L2 gather 48B rows", [&] { k_gather_rows<3><<<grid, 256>>>(t, (6 << 20) / 48, a, n); }, bytes / 1e9);
    }
    return 0;
}
