// kernels.cuh — parameter blocks and launchers shared by the sampling kernels.
#pragma once
#include <algorithm>

#include "hgs_internal.cuh"

namespace hgs {

enum : int32_t { kErrNone = 0, kErrRootRange = 1, kErrNegative = 2, kErrOverflow = 3, kErrCapacity = 4, kErrSetRange = 5 };
// largest distinct vertex set of one root (16-bit local ids in K2's edge slots)
constexpr int32_t kMaxSet = 32767;
// choose() keeps up to this many slots in local memory; larger choices use
// a global scratch slot per lane (ExpandParams/RowsParams::big)
constexpr uint32_t kLocalK = 256;

__device__ __forceinline__ void report(int32_t* t, int32_t code, int32_t a, int32_t b) {
    if (atomicCAS(&t[1], 0, code) == 0) {
        t[2] = a;
        t[3] = b;
    }
}

struct ExpandParams {
    const int2* __restrict__ w_ri;      // walk rows: (row start, degree), one 8-byte load
    int32_t combine;                    // touched stores through the per-lane write combiner (large calls)
    const int32_t* __restrict__ w_ci;
    const uint64_t* __restrict__ recip;
    const uint8_t* __restrict__ neg_row;  // nullable
    const int32_t* __restrict__ roots32;  // one of roots32 / roots64
    const int64_t* __restrict__ roots64;
    const uint64_t* __restrict__ seeds;
    const uint64_t* __restrict__ state;   // nullable: resume states
    const int64_t* __restrict__ batch_off;  // for device-derived seeds (seeds == nullptr)
    int32_t k;
    hgs_seed_spec spec;
    int32_t r0, R, depth, fanout, n;     // roots [r0, R) of the call
    int64_t stride;
    int32_t cache_entries;                // (b,deg) entries cached per lane in smem
    int32_t recip_smem;                   // recip entries staged in smem (0: read global)
    int32_t* __restrict__ touched;
    int32_t* __restrict__ tcount;
    int32_t* __restrict__ level_counts;
    uint32_t* __restrict__ draws;
    uint32_t* __restrict__ decisions;
    int32_t* __restrict__ ticket;         // [0] ticket, [1] error code, [2] root, [3] aux
    uint32_t* __restrict__ big;           // choices > kLocalK: 3 x big_k words per root of the launch
    int32_t big_k;
    int32_t force_serial;                 // test hook: roots r % force_serial == 0 take the serial path
};

void launch_expand(int threads, size_t smem, int64_t kmax, const ExpandParams& ep, bool philox,
                   cudaStream_t st);

// sample_rows on the device: rows grouped by choice stream.
struct RowsParams {
    const int64_t* __restrict__ row_ptr;  // P's pattern
    const int64_t* __restrict__ col;
    const int64_t* __restrict__ srows;    // nonempty rows, grouped by stream, row order within
    const int64_t* __restrict__ sptr;     // [groups + 1]
    const int64_t* __restrict__ sid;      // stream ordinal of each group
    const int64_t* __restrict__ out_off;  // per row: offset of its choices
    int64_t* __restrict__ out_cols;
    const uint64_t* __restrict__ seeds;
    const uint64_t* __restrict__ state;   // nullable: resume (xoshiro 4 words / philox decisions)
    const uint64_t* __restrict__ recip;
    int32_t fanout, groups;
    uint32_t* __restrict__ draws;         // per group
    uint32_t* __restrict__ decisions;
    uint32_t* __restrict__ big;           // choices > kLocalK: 3 x big_k words per group
    int32_t big_k;
};
void launch_sample_rows(const RowsParams& p, bool philox, cudaStream_t st);

// K2: dedup + induced-subgraph extraction into per-root scratch.
struct ExtractParams {
    const int32_t* __restrict__ a_rp;
    const int32_t* __restrict__ a_ci;
    const int32_t* __restrict__ a_gid;  // nullable
    const int2* __restrict__ a_ri;      // per vertex: (A row start, out-degree)
    int32_t* __restrict__ touched;      // in: touched lists; out: sorted sets
    const int32_t* __restrict__ tcount;
    int64_t stride;
    int32_t r0, R;                      // roots [r0, R)
    int32_t* __restrict__ root_nv;
    int32_t* __restrict__ root_ne;
    int32_t* __restrict__ root_rloc;
    int32_t* __restrict__ root_scan;
    int2* __restrict__ escratch;        // per root: e_stride x (local i<<16 | j, edge id)
    int32_t e_stride;
    int32_t* __restrict__ ticket;
    int32_t n_buckets, set_cap, row_cap, win_cap, warp_bytes, rank_bits;
    int32_t cnt_lg;                     // log2 of the bucket-counter capacity (<= 2*row_cap)
    int32_t* __restrict__ work;         // root counter (zeroed before each launch)
    unsigned char* gscratch;            // nullable: per-warp working sets in global memory
    int32_t lnb;                        // k_extract_dir: log2 of the rank-directory buckets
    const int32_t* __restrict__ e_off;  // nullable: exact edge-slot offsets [R+1] (re-run after overflow)
    int32_t ck_iters;                   // k_extract: cuckoo insert chain bound (beyond it: 4-slot table)
    int32_t tab_n;                      // k_extract_bm: directory words (multiple of 32, > n / 16)
    const int4* __restrict__ a_q;       // k_extract_bm: A in 4-entry quads (DevGraph::a_q)
    const int4* __restrict__ a_qid;     // k_extract_bm: edge ids of the a_q entries
    const int2* __restrict__ a_rq;      // k_extract_bm: per vertex (first quad, out-degree)
};

// K3: packing + gather.
struct PackParams {
    const int32_t* __restrict__ touched;
    int64_t stride;
    const int32_t* __restrict__ root_voff;
    const int32_t* __restrict__ root_eoff;
    const int32_t* __restrict__ root_rloc;
    const int2* __restrict__ escratch;
    int32_t e_stride;
    const int32_t* __restrict__ e_off;  // nullable: exact edge-slot offsets (see ExtractParams)
    const int64_t* __restrict__ batch_off;
    int32_t k, r0, R;                   // roots [r0, R)
    int32_t* __restrict__ l2g;
    int32_t* __restrict__ roots_local;
    int32_t* __restrict__ comp_off;
    int32_t* __restrict__ e_row;
    int32_t* __restrict__ e_col;
    int32_t* __restrict__ e_gid;
    double* __restrict__ xv;
    double* __restrict__ ye;
    uint8_t* __restrict__ lab;
    const double* __restrict__ node_feat;
    const double* __restrict__ edge_feat;
    const uint8_t* __restrict__ labels;
    int32_t f_v, f_e, gather;
    uint32_t fv_magic;  // ceil(2^32 / (f_v/2)) for even f_v (0 when f_v/2 == 1)
    uint32_t fv_err;    // (f_v/2) * fv_magic - 2^32: the magic quotient is exact for e * fv_err < 2^32
    uint32_t fv_magic_local;  // the same magic when exact for every per-root piece index (< set_cap * f_v/2), else 0
    int64_t v_cap, e_cap;
    int32_t set_cap;  // per-warp staging of the root's set (>= max set size)
    int32_t* __restrict__ ticket;
};

void launch_extract(int grid, int warps, size_t smem, const ExtractParams& xp, bool packed, cudaStream_t st);
int extract_blocks_per_sm(size_t smem, int warps, bool packed);
// K2, directory variant (extract_dir.cu): the default path
void launch_extract_dir(int grid, int warps, size_t smem, const ExtractParams& xp, cudaStream_t st);
int extract_dir_prepare(size_t smem, int warps);
// K2, one root per CTA with a bitmap rank directory (extract_bm.cu): the default
// for touched lists of <= 512 entries on graphs whose directory fits shared memory
#ifndef HGS_K2M_WARPS
#define HGS_K2M_WARPS 4  // warps per k_extract_bm CTA (one root per CTA)
#endif
void launch_extract_bm(int grid, int warps, size_t smem, const ExtractParams& xp, cudaStream_t st);
int extract_bm_prepare(size_t smem, int warps);
// Shared-memory opt-in + occupancy (CTAs per SM, min over the kernels) of
// kernels launched with `smem` dynamic bytes and 32*warps threads, cached per
// (device, kernels, smem, warps): no driver calls on the per-call path.
int prepare_kernel(const void* const* kerns, int n, size_t smem, int warps);
// *out = max(x[0..n)) (>= 0), on the device
void launch_max_i32(const int32_t* x, int32_t n, int32_t* out, cudaStream_t st);
// Exclusive scan of (V_r, E_r) over roots [r0, r1) into voff/eoff[r0..r1];
// for r0 > 0 the carry-in is voff/eoff[r0] as written by the previous chunk.
// scan + batch offsets in one launch for R <= 16384 (false: use launch_scan + launch_finalize)
bool launch_scan_small(const int32_t* nv, const int32_t* ne, int32_t R, int32_t* voff, int32_t* eoff, int32_t* ticket,
                       const int64_t* batch_off, int32_t k, int32_t* bvoff, int32_t* beoff, int32_t* comp_off,
                       cudaStream_t st);
void launch_scan(const int32_t* nv, const int32_t* ne, int32_t r0, int32_t r1, int64_t* tmp, int32_t* voff,
                 int32_t* eoff, int32_t* ticket, cudaStream_t st);
int64_t scan_tmp_words(int64_t R);
void launch_pack(int grid, const PackParams& pp, cudaStream_t st);
// K3 fused: pack + node/edge gathers per root (erec nullable: general f_e)
void launch_pack_gather(int grid, const PackParams& pp, const uint4* erec, cudaStream_t st);
// node / edge feature gather over the packed call outputs
// over vertices [*vb, *ve) and edges [*eb, *ee) of the call (device pointers)
void launch_gather_packed(int blocks, const PackParams& pp, const uint4* erec, const int32_t* vb,
                          const int32_t* ve, const int32_t* eb, const int32_t* ee, cudaStream_t st);
// DevGraph::erec from the attached edge features + labels (f_e == 2 only)
void build_edge_records(DevGraph& g, cudaStream_t st);
void launch_finalize(const int64_t* batch_off, int32_t k, int32_t R, const int32_t* voff,
                     const int32_t* eoff, int32_t* bvoff, int32_t* beoff, int32_t* comp_off,
                     cudaStream_t st);
void launch_gather(const DevGraph& g, const int64_t* d_l2g, int64_t V, const int64_t* d_eid, int64_t E,
                   double* d_xv, double* d_ye, uint8_t* d_lab, cudaStream_t st);
void launch_stats(const int32_t* level_counts, int32_t depth, const int32_t* root_scan,
                  const uint32_t* decisions, const uint32_t* draws, int32_t R,
                  unsigned long long* out, cudaStream_t st);

}  // namespace hgs
