// sampler.cu — the per-call hot path of bulk ShaDow sampling on sm_100a.
//
// Reference semantics: hitgnn::bulk_shadow (sampler.cpp:123-201) +
// gather_features (sampler.cpp:211-243). Under per-root choice streams the
// result is independent of the order roots are processed in (the reference's
// bulk ≡ shadow_reference property), so the device processes
// each root's tree independently:
//
//   K1 k_expand   (lane per root)  stacked-Q expansion: d levels of
//                 "row v of the walk, choose min(s,deg) sorted positions,
//                 append children" in the root's BFS order, consuming the
//                 root's stream exactly like sample_rows (sampler.cpp:64-86,
//                 173-182). Output: the root's touched list (root, then level
//                 1..d children) in a per-root scratch slot.
//   K2-K5 k_extract (warp per root, persistent, single pass):
//                 dedup (smem hash) + bitonic sort = sorted_vertex_set
//                 (sampler.cpp:48-53); induced subgraph S·A·Sᵀ
//                 (sparse.cpp:177-191) as a load-balanced scan of the set's
//                 A rows with hash membership; block_diag packing
//                 (sparse.cpp:245-258) through a decoupled look-back scan
//                 over roots (global + per-batch offsets); feature/label
//                 gather fused into the output writes.
//   k_finalize    per-batch offsets (k+1 threads).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

#include "hgs_internal.cuh"

namespace hgs {

// ===========================================================================
// K1: expansion
// ===========================================================================

struct ExpandParams {
    const int32_t* __restrict__ w_rp;
    const int32_t* __restrict__ w_ci;
    const uint64_t* __restrict__ recip;
    const uint8_t* __restrict__ neg_row;  // nullable
    const int32_t* __restrict__ roots32;  // one of roots32 / roots64
    const int64_t* __restrict__ roots64;
    const uint64_t* __restrict__ seeds;
    const uint64_t* __restrict__ state;   // nullable: resume states
    int32_t R, depth, fanout, n;
    int64_t stride;
    int32_t cache_entries;                // (b,deg) entries cached per lane in smem
    int32_t* __restrict__ touched;
    int32_t* __restrict__ tcount;
    int32_t* __restrict__ level_counts;
    uint32_t* __restrict__ draws;
    uint32_t* __restrict__ decisions;
    unsigned long long* __restrict__ status;
    int32_t* __restrict__ ticket;         // [0] ticket, [1] error code, [2] root, [3] aux
};

enum : int32_t { kErrNone = 0, kErrRootRange = 1, kErrNegative = 2, kErrOverflow = 3, kErrCapacity = 4 };

__device__ __forceinline__ void report(int32_t* t, int32_t code, int32_t a, int32_t b) {
    if (atomicCAS(&t[1], 0, code) == 0) {
        t[2] = a;
        t[3] = b;
    }
}

// A random stream for one root, in either mode; draw(i, m) returns the
// accepted bounded(m) result of Fisher-Yates step i (Rng::bounded
// semantics, rng.cpp:43-50).
template <bool PHILOX>
struct RootStream;

template <>
struct RootStream<false> {
    Xoshiro256 x;
    uint32_t draws = 0;
    __device__ void init(uint64_t seed, const uint64_t* st) {
        if (st) { x.a = st[0]; x.b = st[1]; x.c = st[2]; x.d = st[3]; }
        else x.seed(seed);
    }
    __device__ __forceinline__ void begin_decision(uint32_t) {}
    __device__ __forceinline__ uint32_t draw(uint32_t, uint64_t m, uint64_t rc) {
        uint64_t v;
        do {
            v = x.next();
            ++draws;
        } while (rejected(v, m, rc));
        return (uint32_t)mod_by_recip(v, m, rc);
    }
};

template <>
struct RootStream<true> {
    uint64_t seed = 0;
    uint32_t dec = 0, draws = 0;
    __device__ void init(uint64_t s, const uint64_t*) { seed = s; }
    __device__ __forceinline__ void begin_decision(uint32_t d) { dec = d; }
    __device__ __forceinline__ uint32_t draw(uint32_t step, uint64_t m, uint64_t rc) {
        uint64_t v;
        uint32_t att = 0;
        do {
            v = philox_draw(seed, dec, step, att++);
            ++draws;
        } while (rejected(v, m, rc));
        return (uint32_t)mod_by_recip(v, m, rc);
    }
};

// choose(n, k) of RandomChoiceSource (rng.cpp:105-119) over a virtual
// identity array, for k <= KCAP: slots < k live in registers; slots >= k that
// a swap displaced live in a short (pos, val) list. Output sorted ascending.
template <int KCAP, bool PHILOX>
__device__ __forceinline__ void choose_regs(RootStream<PHILOX>& rs, uint32_t n, uint32_t k,
                                            const uint64_t* __restrict__ recip,
                                            uint32_t (&val)[KCAP]) {
    uint32_t dpos[KCAP], dval[KCAP];
#pragma unroll
    for (int q = 0; q < KCAP; ++q) { val[q] = q; dpos[q] = 0xffffffffu; dval[q] = 0; }
    int nd = 0;
#pragma unroll
    for (int i = 0; i < KCAP; ++i) {
        if (i < (int)k) {
            const uint64_t m = n - (uint32_t)i;
            const uint32_t j = (uint32_t)i + rs.draw((uint32_t)i, m, __ldg(recip + m));
            const uint32_t vi = val[i];
            uint32_t vj = j;
            if (j < k) {
#pragma unroll
                for (int q = 0; q < KCAP; ++q) if ((uint32_t)q == j) vj = val[q];
#pragma unroll
                for (int q = 0; q < KCAP; ++q) if ((uint32_t)q == j) val[q] = vi;
            } else {
                bool found = false;
#pragma unroll
                for (int q = 0; q < KCAP; ++q)
                    if (dpos[q] == j) { vj = dval[q]; dval[q] = vi; found = true; }
                if (!found) {
#pragma unroll
                    for (int q = 0; q < KCAP; ++q)
                        if (q == nd) { dpos[q] = j; dval[q] = vi; }
                    ++nd;
                }
            }
            val[i] = vj;
        }
    }
#pragma unroll
    for (int q = 0; q < KCAP; ++q) if (q >= (int)k) val[q] = 0xffffffffu;
    // odd-even transposition network
#pragma unroll
    for (int round = 0; round < KCAP; ++round) {
#pragma unroll
        for (int q = round & 1; q + 1 < KCAP; q += 2) {
            const uint32_t a = val[q], b = val[q + 1];
            val[q] = min(a, b);
            val[q + 1] = max(a, b);
        }
    }
}

// Generic variant for large fanouts (local-memory arrays, k <= 256).
template <bool PHILOX>
__device__ void choose_local(RootStream<PHILOX>& rs, uint32_t n, uint32_t k,
                             const uint64_t* __restrict__ recip, uint32_t* val) {
    uint32_t dpos[256], dval[256];
    int nd = 0;
    for (uint32_t q = 0; q < k; ++q) val[q] = q;
    for (uint32_t i = 0; i < k; ++i) {
        const uint64_t m = n - i;
        const uint32_t j = i + rs.draw(i, m, __ldg(recip + m));
        const uint32_t vi = val[i];
        uint32_t vj = j;
        if (j < k) {
            vj = val[j];
            val[j] = vi;
        } else {
            int f = -1;
            for (int q = 0; q < nd; ++q) if (dpos[q] == j) f = q;
            if (f >= 0) { vj = dval[f]; dval[f] = vi; }
            else { dpos[nd] = j; dval[nd] = vi; ++nd; }
        }
        val[i] = vj;
    }
    for (uint32_t a = 1; a < k; ++a) {  // insertion sort
        const uint32_t x = val[a];
        uint32_t b = a;
        while (b > 0 && val[b - 1] > x) { val[b] = val[b - 1]; --b; }
        val[b] = x;
    }
}

template <int KCAP, bool PHILOX, bool LOCAL>
__global__ void __launch_bounds__(128) k_expand(ExpandParams p) {
    extern __shared__ int2 cache[];  // [entry][thread]: (row start, degree)
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.R) return;
    p.status[r] = 0ull;
    const int bd = blockDim.x, ti = threadIdx.x;

    const int32_t root = p.roots32 ? p.roots32[r] : (int32_t)p.roots64[r];
    if (root < 0 || root >= p.n) {
        report(p.ticket, kErrRootRange, r, root);
        p.tcount[r] = 0;
        return;
    }
    RootStream<PHILOX> rs;
    rs.init(p.seeds[r], (!PHILOX && p.state) ? p.state + 4 * (size_t)r : nullptr);
    uint32_t ndec = (PHILOX && p.state) ? (uint32_t)p.state[r] : 0u;
    const uint32_t dec0 = ndec;

    int32_t* out = p.touched + (size_t)r * p.stride;
    int32_t* lc = p.level_counts + (size_t)r * (p.depth + 1);
    out[0] = root;
    lc[0] = 1;
    const bool cached = p.cache_entries > 0;
    {
        const int32_t b = p.w_rp[root];
        if (cached) cache[ti] = make_int2(b, p.w_rp[root + 1] - b);
    }
    int T = 1, lvl_begin = 0, lvl_end = 1;
    for (int level = 0; level < p.depth; ++level) {
        const bool expand_next = level + 1 < p.depth;
        const int next_begin = T;
        for (int idx = lvl_begin; idx < lvl_end; ++idx) {
            int2 row;
            if (cached) row = cache[(size_t)idx * bd + ti];
            else {
                const int32_t v = out[idx];
                row.x = p.w_rp[v];
                row.y = p.w_rp[v + 1] - row.x;
            }
            if (row.y == 0) continue;  // empty rows make no choose call (sampler.cpp:75)
            if (p.neg_row && p.neg_row[out[idx]]) {
                report(p.ticket, kErrNegative, r, level);
                p.tcount[r] = T;
                return;
            }
            const uint32_t deg = (uint32_t)row.y;
            const uint32_t k = min((uint32_t)p.fanout, deg);
            rs.begin_decision(ndec);
            ++ndec;
            if (!LOCAL) {
                uint32_t pos[KCAP];
                choose_regs<KCAP, PHILOX>(rs, deg, k, p.recip, pos);
#pragma unroll
                for (int q = 0; q < KCAP; ++q) {
                    if (q < (int)k) {
                        const int32_t c = __ldg(p.w_ci + row.x + pos[q]);
                        out[T] = c;
                        if (expand_next && cached) {
                            const int32_t cb = __ldg(p.w_rp + c);
                            cache[(size_t)T * bd + ti] = make_int2(cb, __ldg(p.w_rp + c + 1) - cb);
                        }
                        ++T;
                    }
                }
            } else {
                uint32_t pos[256];
                choose_local<PHILOX>(rs, deg, k, p.recip, pos);
                for (uint32_t q = 0; q < k; ++q) {
                    const int32_t c = __ldg(p.w_ci + row.x + pos[q]);
                    out[T] = c;
                    if (expand_next && cached) {
                        const int32_t cb = __ldg(p.w_rp + c);
                        cache[(size_t)T * bd + ti] = make_int2(cb, __ldg(p.w_rp + c + 1) - cb);
                    }
                    ++T;
                }
            }
        }
        lc[level + 1] = T - next_begin;
        lvl_begin = next_begin;
        lvl_end = T;
    }
    p.tcount[r] = T;
    p.draws[r] = rs.draws;
    p.decisions[r] = ndec - dec0;
}

// ===========================================================================
// K2-K5: fused extract
// ===========================================================================

struct ExtractParams {
    const int32_t* __restrict__ a_rp;
    const int32_t* __restrict__ a_ci;
    const int32_t* __restrict__ a_gid;  // nullable
    const double* __restrict__ node_feat;
    const double* __restrict__ edge_feat;
    const uint8_t* __restrict__ labels;
    int32_t f_v, f_e, gather;
    const int32_t* __restrict__ touched;
    const int32_t* __restrict__ tcount;
    int64_t stride;
    const int64_t* __restrict__ batch_off;
    int32_t k, R;
    int32_t* __restrict__ l2g;
    int32_t* __restrict__ roots_local;
    int32_t* __restrict__ comp_off;
    int32_t* __restrict__ e_row;
    int32_t* __restrict__ e_col;
    int32_t* __restrict__ e_gid;
    int32_t* __restrict__ root_voff;
    int32_t* __restrict__ root_eoff;
    double* __restrict__ xv;
    double* __restrict__ ye;
    uint8_t* __restrict__ lab;
    int64_t v_cap, e_cap;
    unsigned long long* __restrict__ status;
    unsigned long long* __restrict__ bbase;
    int32_t* __restrict__ ticket;
    // per-warp shared-memory geometry
    int32_t hs_bits, set_cap, row_cap, stage_cap, warp_bytes;
};

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62;
constexpr int32_t kMask31 = 0x7fffffff;

__device__ __forceinline__ unsigned long long pack_status(unsigned long long flag, int64_t v, int64_t e) {
    return flag | ((unsigned long long)(v & kMask31) << 31) | (unsigned long long)(e & kMask31);
}

struct WarpSmem {
    int32_t* hkey;
    int16_t* hval;
    int32_t* set;
    int32_t* rstart;
    int32_t* rbase;
    int16_t* rrank;
    int32_t* sgid;
    uint32_t* sij;
};

__device__ __forceinline__ uint32_t hslot(int32_t v, int bits) {
    return ((uint32_t)v * 0x9E3779B1u) >> (32 - bits);
}

__device__ __forceinline__ int find_rank(const WarpSmem& s, int32_t v, int bits) {
    const uint32_t mask = (1u << bits) - 1u;
    uint32_t h = hslot(v, bits);
    for (;;) {
        const int32_t key = s.hkey[h];
        if (key == v) return s.hval[h];
        if (key == -1) return -1;
        h = (h + 1) & mask;
    }
}

template <int E>
__device__ __forceinline__ void sort_set_regs(int32_t* set, int U) {
    const int lane = lane_id();
    uint32_t kk[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        kk[e] = i < U ? (uint32_t)set[i] : 0xffffffffu;
    }
    warp_bitonic_sort<E>(kk);
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        if (i < U) set[i] = (int32_t)kk[e];
    }
}

// In-place warp bitonic sort over a power-of-two smem array (large sets).
__device__ void sort_set_smem(int32_t* set, int U, int N) {
    const int lane = lane_id();
    for (int i = U + lane; i < N; i += 32) set[i] = 0x7fffffff;
    __syncwarp();
    for (int size = 2; size <= N; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = lane; t < N / 2; t += 32) {
                const int i = 2 * t - (t & (stride - 1));
                const int j = i + stride;
                const bool up = (i & size) == 0;
                const int32_t a = set[i], b = set[j];
                if ((a > b) == up) { set[i] = b; set[j] = a; }
            }
            __syncwarp();
        }
    }
}

// Scan the flattened A-row entries of the set (local order, columns
// ascending) in 32-wide windows; emit hits in output order.
// MODE 0: stage into smem (returns count, staging only below stage_cap);
// MODE 1: write edges directly to global at ebase.
template <int MODE>
__device__ __forceinline__ int scan_edges(const ExtractParams& p, const WarpSmem& s, int NR, int S,
                                          int64_t ebase, int32_t loc) {
    const int lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    const unsigned le = (2u << lane) - 1u;
    int cursor = 0, count = 0;
    for (int w = 0; w < S; w += 32) {
        const int rr = cursor + 1 + lane;
        const int rs = rr <= NR ? s.rstart[rr] : 0x7fffffff;
        const int off = rs - w;
        const unsigned bit = (off > 0 && off < 32) ? (1u << off) : 0u;
        const unsigned M = __reduce_or_sync(kFull, bit);
        const int own = cursor + __popc(M & le);
        const int pos = w + lane;
        int j = -1, gid = 0, li = 0;
        if (pos < S) {
            const int kk = s.rbase[own] + (pos - s.rstart[own]);
            const int32_t v = __ldg(p.a_ci + kk);
            j = find_rank(s, v, p.hs_bits);
            gid = p.a_gid ? __ldg(p.a_gid + kk) : kk;
            li = s.rrank[own];
        }
        const bool hit = j >= 0;
        const unsigned hb = __ballot_sync(kFull, hit);
        if (hit) {
            const int t = count + __popc(hb & lt);
            if (MODE == 0) {
                if (t < p.stage_cap) {
                    s.sgid[t] = gid;
                    s.sij[t] = ((uint32_t)li << 16) | (uint32_t)j;
                }
            } else {
                p.e_row[ebase + t] = loc + li;
                p.e_col[ebase + t] = loc + j;
                p.e_gid[ebase + t] = gid;
            }
        }
        count += __popc(hb);
        const int own31 = __shfl_sync(kFull, own, 31);
        cursor = (own31 + 1 <= NR && s.rstart[own31 + 1] == w + 32) ? own31 + 1 : own31;
    }
    return count;
}

__global__ void __launch_bounds__(128) k_extract(ExtractParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = lane_id();
    const int warp = threadIdx.x >> 5;
    unsigned char* base = smem_raw + (size_t)warp * p.warp_bytes;
    const int HS = 1 << p.hs_bits;
    WarpSmem s;
    {
        unsigned char* q = base;
        s.hkey = (int32_t*)q; q += 4 * HS;
        s.set = (int32_t*)q; q += 4 * p.set_cap;
        s.rstart = (int32_t*)q; q += 4 * (p.row_cap + 1);
        s.rbase = (int32_t*)q; q += 4 * p.row_cap;
        s.sgid = (int32_t*)q; q += 4 * p.stage_cap;
        s.sij = (uint32_t*)q; q += 4 * p.stage_cap;
        s.hval = (int16_t*)q; q += 2 * HS;
        s.rrank = (int16_t*)q;
    }
    const uint32_t hmask = (uint32_t)HS - 1u;

    for (;;) {
        int r = 0;
        if (lane == 0) r = atomicAdd(&p.ticket[0], 1);
        r = __shfl_sync(kFull, r, 0);
        if (r >= p.R) break;
        const int32_t* tl = p.touched + (size_t)r * p.stride;
        const int T = p.tcount[r];

        // ---- dedup into the hash set (sorted_vertex_set, sampler.cpp:48-53)
        for (int i = lane; i < HS; i += 32) s.hkey[i] = -1;
        __syncwarp();
        int U = 0;
        for (int b0 = 0; b0 < T; b0 += 32) {
            const int idx = b0 + lane;
            bool fresh = false;
            int32_t v = -1;
            if (idx < T) {
                v = tl[idx];
                uint32_t h = hslot(v, p.hs_bits);
                for (;;) {
                    const int32_t prev = atomicCAS(&s.hkey[h], -1, v);
                    if (prev == -1) { fresh = true; break; }
                    if (prev == v) break;
                    h = (h + 1) & hmask;
                }
            }
            const unsigned fb = __ballot_sync(kFull, fresh);
            if (fresh) s.set[U + __popc(fb & ((1u << lane) - 1u))] = v;
            U += __popc(fb);
        }
        __syncwarp();
        if (U <= 32) sort_set_regs<1>(s.set, U);
        else if (U <= 64) sort_set_regs<2>(s.set, U);
        else if (U <= 128) sort_set_regs<4>(s.set, U);
        else if (U <= 256) sort_set_regs<8>(s.set, U);
        else if (U <= 512) sort_set_regs<16>(s.set, U);
        else {
            int N = 1024;
            while (N < U) N <<= 1;
            sort_set_smem(s.set, U, N);
        }
        __syncwarp();

        // ---- ranks + nonempty A rows with flattened offsets
        int NR = 0, S = 0;
        for (int b0 = 0; b0 < U; b0 += 32) {
            const int i = b0 + lane;
            int32_t rb = 0, deg = 0;
            if (i < U) {
                const int32_t u = s.set[i];
                uint32_t h = hslot(u, p.hs_bits);
                while (s.hkey[h] != u) h = (h + 1) & hmask;
                s.hval[h] = (int16_t)i;
                rb = __ldg(p.a_rp + u);
                deg = __ldg(p.a_rp + u + 1) - rb;
            }
            const bool ne = deg > 0;
            const unsigned nb = __ballot_sync(kFull, ne);
            const int incl = warp_incl_scan(deg);
            if (ne) {
                const int q = NR + __popc(nb & ((1u << lane) - 1u));
                s.rstart[q] = S + incl - deg;
                s.rbase[q] = rb;
                s.rrank[q] = (int16_t)i;
            }
            NR += __popc(nb);
            S += __shfl_sync(kFull, incl, 31);
        }
        if (lane == 0) s.rstart[NR] = S;
        __syncwarp();
        const int32_t root = tl[0];
        const int rloc = find_rank(s, root, p.hs_bits);

        // ---- induced subgraph edges (staged)
        const int Er = scan_edges<0>(p, s, NR, S, 0, 0);

        // ---- decoupled look-back over roots: global + batch-base offsets
        int b;
        {
            int lo = 0, hi = p.k;  // largest b with batch_off[b] <= r
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (p.batch_off[mid] <= r) lo = mid; else hi = mid - 1;
            }
            b = lo;
        }
        const int f = (int)p.batch_off[b];
        if (lane == 0 && r > 0) st_release(p.status + r, pack_status(kFlagAgg, U, Er));
        int64_t exV = 0, exE = 0, segV = 0, segE = 0, bV = 0, bE = 0;
        bool base_known = false;
        if (r > 0) {
            int pos = r - 1;
            for (;;) {
                const int idx = pos - lane;
                unsigned long long sw = kFlagInc;
                if (idx >= 0) {
                    do { sw = ld_acquire(p.status + idx); } while ((sw >> 62) == 0);
                }
                const bool inc = (sw >> 62) == 2;
                const unsigned ib = __ballot_sync(kFull, inc);
                const int stop = ib ? __ffs(ib) - 1 : 32;
                const bool contrib = lane <= stop;
                const int64_t sv = contrib ? (int64_t)((sw >> 31) & kMask31) : 0;
                const int64_t se = contrib ? (int64_t)(sw & kMask31) : 0;
                const bool seg = contrib && lane < stop && idx >= f;
                exV += warp_sum(sv);
                exE += warp_sum(se);
                segV += warp_sum(seg ? sv : 0);
                segE += warp_sum(seg ? se : 0);
                if (ib) {
                    const int idx_s = pos - stop;
                    if (idx_s >= f && idx_s >= 0) {
                        unsigned long long bb = 0;
                        if (lane == stop) bb = p.bbase[idx_s];
                        bb = __shfl_sync(kFull, bb, stop);
                        bV = (int64_t)(bb >> 32);
                        bE = (int64_t)(bb & 0xffffffffull);
                        base_known = true;
                    }
                    break;
                }
                pos -= 32;
            }
        }
        if (!base_known) { bV = exV - segV; bE = exE - segE; }
        const int64_t incV = exV + U, incE = exE + Er;
        if (lane == 0) {
            if (incV > kMask31 || incE > kMask31) report(p.ticket, kErrOverflow, r, 0);
            p.bbase[r] = ((unsigned long long)bV << 32) | (unsigned long long)(uint32_t)bE;
            st_release(p.status + r, pack_status(kFlagInc, incV, incE));
        }

        // ---- outputs (block_diag packing, sampler.cpp:26-46)
        const int32_t loc = (int32_t)(exV - bV);
        const int32_t eloc = (int32_t)(exE - bE);
        (void)eloc;
        if (lane == 0) {
            p.root_voff[r] = (int32_t)exV;
            p.root_eoff[r] = (int32_t)exE;
            if (r == p.R - 1) {
                p.root_voff[p.R] = (int32_t)incV;
                p.root_eoff[p.R] = (int32_t)incE;
            }
        }
        if (incV > p.v_cap || incE > p.e_cap) {
            if (lane == 0) report(p.ticket, kErrCapacity, r, 0);
            continue;
        }
        if (lane == 0) {
            p.roots_local[r] = loc + rloc;
            p.comp_off[r + b] = loc;
            if (r == p.batch_off[b + 1] - 1) p.comp_off[r + 1 + b] = loc + U;
        }
        for (int i = lane; i < U; i += 32) p.l2g[exV + i] = s.set[i];
        if (Er <= p.stage_cap) {
            for (int t = lane; t < Er; t += 32) {
                const uint32_t ij = s.sij[t];
                p.e_row[exE + t] = loc + (int32_t)(ij >> 16);
                p.e_col[exE + t] = loc + (int32_t)(ij & 0xffffu);
                p.e_gid[exE + t] = s.sgid[t];
            }
        } else {
            scan_edges<1>(p, s, NR, S, exE, loc);
        }
        if (p.gather) {
            // node rows: xv[(exV+i)*f_v + c] = node_feat[set[i]*f_v + c]
            const int fv = p.f_v;
            double* dst = p.xv + (size_t)exV * fv;
            for (int e = lane; e < U * fv; e += 32) {
                const int i = e / fv, c = e - i * fv;
                __stcs(dst + e, __ldg(p.node_feat + (size_t)s.set[i] * fv + c));
            }
            const int fe = p.f_e;
            double* edst = p.ye + (size_t)exE * fe;
            __syncwarp();
            for (int t = lane; t < Er; t += 32) {
                const int32_t g = (Er <= p.stage_cap) ? s.sgid[t] : p.e_gid[exE + t];
                p.lab[exE + t] = __ldg(p.labels + g);
                for (int c = 0; c < fe; ++c)
                    __stcs(edst + (size_t)t * fe + c, __ldg(p.edge_feat + (size_t)g * fe + c));
            }
        }
        __syncwarp();
    }
}

__global__ void k_finalize(const int64_t* __restrict__ batch_off, int32_t k, int32_t R,
                           const int32_t* __restrict__ root_voff, const int32_t* __restrict__ root_eoff,
                           int32_t* __restrict__ batch_voff, int32_t* __restrict__ batch_eoff,
                           int32_t* __restrict__ comp_off) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= k; b += gridDim.x * blockDim.x) {
        const int64_t f = batch_off[b];
        const int32_t tv = R > 0 ? root_voff[R] : 0, te = R > 0 ? root_eoff[R] : 0;
        batch_voff[b] = f < R ? root_voff[f] : tv;
        batch_eoff[b] = f < R ? root_eoff[f] : te;
        if (b < k && batch_off[b + 1] == f) comp_off[f + b] = 0;  // empty batch
    }
}

// ===========================================================================
// host side
// ===========================================================================

static int64_t tree_bound(int64_t kmax, int64_t depth, int64_t upto) {
    // 1 + kmax + ... + kmax^upto, saturating at 2^40
    int64_t total = 0, term = 1;
    for (int64_t l = 0; l <= upto; ++l) {
        total += term;
        if (total > ((int64_t)1 << 40)) return (int64_t)1 << 40;
        term *= kmax;
        if (term > ((int64_t)1 << 40)) term = (int64_t)1 << 40;
    }
    (void)depth;
    return total;
}

struct CallPlan {
    int64_t kmax, max_t, cache_entries;
    int expand_threads;
    size_t expand_smem;
    int32_t hs_bits, set_cap, row_cap, stage_cap, warp_bytes;
};

static CallPlan plan_call(const DevCsr& walk, int64_t depth, int64_t fanout) {
    CallPlan c{};
    c.kmax = std::min<int64_t>(fanout, walk.max_deg);
    if (c.kmax > 256)
        fail(HGS_ERANGE, "hgs: min(fanout, max degree) > 256 is not supported by this build");
    c.max_t = tree_bound(c.kmax, depth, depth);
    if (c.max_t > 32767)
        fail(HGS_ERANGE, "hgs: per-root tree bound " + std::to_string(c.max_t) +
                             " exceeds this build's limit (32767); reduce depth/fanout");
    c.cache_entries = tree_bound(c.kmax, depth, depth - 1);
    c.expand_threads = 128;
    c.expand_smem = (size_t)c.cache_entries * 128 * sizeof(int2);
    if (c.expand_smem > 96 * 1024) {
        c.expand_threads = 64;
        c.expand_smem = (size_t)c.cache_entries * 64 * sizeof(int2);
        if (c.expand_smem > 96 * 1024) { c.cache_entries = 0; c.expand_smem = 0; c.expand_threads = 128; }
    }
    int bits = 6;
    while ((1 << bits) < (int)(c.max_t + c.max_t / 2 + 1)) ++bits;
    c.hs_bits = bits;
    c.set_cap = (int32_t)((c.max_t + 31) / 32 * 32);
    if (c.max_t > 512) {
        int n = 1024;
        while (n < c.max_t) n <<= 1;
        c.set_cap = n;
    }
    c.row_cap = (int32_t)((c.max_t + 31) / 32 * 32);
    c.stage_cap = 512;
    const int HS = 1 << c.hs_bits;
    size_t bytes = 4 * (size_t)HS + 4 * (size_t)c.set_cap + 4 * (size_t)(c.row_cap + 1) +
                   4 * (size_t)c.row_cap + 8 * (size_t)c.stage_cap + 2 * (size_t)HS +
                   2 * (size_t)c.row_cap;
    bytes = (bytes + 15) / 16 * 16;
    c.warp_bytes = (int32_t)bytes;
    if (4 * bytes > 200 * 1024) fail(HGS_ERANGE, "hgs: per-root working set too large for shared memory");
    return c;
}

static int sm_count(int device) {
    int n = 0;
    HGS_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    return n;
}

template <int KCAP, bool PH, bool LOCAL>
static void launch_expand_t(const CallPlan& c, const ExpandParams& ep, cudaStream_t st) {
    auto kern = k_expand<KCAP, PH, LOCAL>;
    if (c.expand_smem > 48 * 1024)
        HGS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.expand_smem));
    const unsigned grid = (unsigned)((ep.R + c.expand_threads - 1) / c.expand_threads);
    kern<<<grid, c.expand_threads, c.expand_smem, st>>>(ep);
    HGS_CUDA(cudaGetLastError());
}

static void launch_expand(const CallPlan& c, const ExpandParams& ep, bool philox, cudaStream_t st) {
    const bool local = c.kmax > 8;  // register fast path covers fanouts up to 8
    if (philox) {
        if (local) launch_expand_t<8, true, true>(c, ep, st);
        else launch_expand_t<8, true, false>(c, ep, st);
    } else {
        if (local) launch_expand_t<8, false, true>(c, ep, st);
        else launch_expand_t<8, false, false>(c, ep, st);
    }
}

static void launch_extract(hgs_sample* s, const CallPlan& c, const ExtractParams& xp) {
    const size_t smem = (size_t)4 * c.warp_bytes;
    HGS_CUDA(cudaFuncSetAttribute(k_extract, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    HGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_extract, 128, smem));
    per_sm = std::max(per_sm, 1);
    const int64_t warps_needed = (xp.R + 3) / 4;
    const int64_t grid = std::min<int64_t>((int64_t)per_sm * sm_count(s->graph->g.device), warps_needed);
    k_extract<<<(unsigned)std::max<int64_t>(grid, 1), 128, smem, s->stream>>>(xp);
    HGS_CUDA(cudaGetLastError());
}

// ---- the call -----------------------------------------------------------------

void sample_enqueue(hgs_sample* s, const hgs_config& cfg, const CallInputs& in) {
    DevGraph& g = s->graph->g;
    HGS_CUDA(cudaSetDevice(g.device));
    if (cfg.symmetrize) graph_build_walk_sym(g);
    const DevCsr& walk = cfg.symmetrize ? g.walk_sym : g.a;
    graph_ensure_recip(g, walk.max_deg);
    if (cfg.gather && !g.has_features)
        fail(HGS_EINVAL, "gather_features: no features attached to the graph");
    const CallPlan c = plan_call(walk, cfg.depth, cfg.fanout);
    const int64_t R = in.R, k = in.k;
    if (R >= ((int64_t)1 << 31) / std::max<int64_t>(1, c.max_t) && R * c.max_t >= ((int64_t)1 << 40))
        fail(HGS_ERANGE, "hgs: too many roots for one call");
    cudaStream_t st = s->stream;

    s->R = R; s->k = k; s->depth = cfg.depth; s->fanout = cfg.fanout;
    s->gathered = cfg.gather; s->symmetrize = cfg.symmetrize; s->rng = cfg.rng;
    s->launches = 0;
    s->touched_stride = c.max_t;
    s->touched.reserve((size_t)std::max<int64_t>(R, 1) * c.max_t);
    s->tcount.reserve((size_t)R + 1);
    s->level_counts.reserve((size_t)(R + 1) * (cfg.depth + 1));
    s->draws.reserve((size_t)R + 1);
    s->decisions.reserve((size_t)R + 1);
    s->status.reserve((size_t)R + 1);
    s->bbase.reserve((size_t)R + 1);
    s->ticket.reserve(8);
    s->root_voff.reserve((size_t)R + 1);
    s->root_eoff.reserve((size_t)R + 1);
    s->roots_local.reserve((size_t)R + 1);
    s->comp_off.reserve((size_t)(R + k) + 1);
    s->batch_voff.reserve((size_t)k + 1);
    s->batch_eoff.reserve((size_t)k + 1);
    const size_t vneed = (size_t)std::max<int64_t>(1, R * c.max_t);
    if (s->v_cap < vneed) {
        s->l2g.reserve(vneed);
        s->v_cap = vneed;
    }
    if (s->e_cap < s->v_cap * 2) s->e_cap = s->v_cap * 2;
    s->e_row.reserve(s->e_cap); s->e_col.reserve(s->e_cap); s->e_gid.reserve(s->e_cap);
    if (cfg.gather) {
        s->xv.reserve(s->v_cap * (size_t)std::max(1, g.f_v));
        s->ye.reserve(s->e_cap * (size_t)std::max(1, g.f_e));
        s->lab.reserve(s->e_cap);
    }
    HGS_CUDA(cudaMemsetAsync(s->ticket.p, 0, 8 * sizeof(int32_t), st));
    if (R == 0) HGS_CUDA(cudaMemsetAsync(s->root_voff.p, 0, sizeof(int32_t), st));
    if (R == 0) HGS_CUDA(cudaMemsetAsync(s->root_eoff.p, 0, sizeof(int32_t), st));

    if (!s->ev[0]) for (auto& e : s->ev) HGS_CUDA(cudaEventCreate(&e));
    s->profiled = cfg.profile != 0;
    if (s->profiled) HGS_CUDA(cudaEventRecord(s->ev[0], st));

    if (R > 0) {
        ExpandParams ep{};
        ep.w_rp = walk.rp.p; ep.w_ci = walk.ci.p; ep.recip = g.recip.p;
        ep.neg_row = (!cfg.symmetrize && g.has_neg) ? g.neg_row.p : nullptr;
        ep.roots32 = in.roots32; ep.roots64 = in.roots64; ep.seeds = in.seeds; ep.state = in.state;
        ep.R = (int32_t)R; ep.depth = (int32_t)cfg.depth; ep.fanout = (int32_t)std::min<int64_t>(cfg.fanout, 1 << 30);
        ep.n = (int32_t)g.n_rows; ep.stride = c.max_t; ep.cache_entries = (int32_t)c.cache_entries;
        ep.touched = s->touched.p; ep.tcount = s->tcount.p; ep.level_counts = s->level_counts.p;
        ep.draws = s->draws.p; ep.decisions = s->decisions.p; ep.status = s->status.p;
        ep.ticket = s->ticket.p;
        launch_expand(c, ep, cfg.rng == HGS_RNG_PHILOX, st);
        ++s->launches;
    }
    if (s->profiled) HGS_CUDA(cudaEventRecord(s->ev[1], st));

    ExtractParams xp{};
    xp.a_rp = g.a.rp.p; xp.a_ci = g.a.ci.p; xp.a_gid = g.has_gid ? g.a_gid.p : nullptr;
    xp.node_feat = g.node_feat.p; xp.edge_feat = g.edge_feat.p; xp.labels = g.labels.p;
    xp.f_v = g.f_v; xp.f_e = g.f_e; xp.gather = cfg.gather;
    xp.touched = s->touched.p; xp.tcount = s->tcount.p; xp.stride = c.max_t;
    xp.batch_off = in.batch_off; xp.k = (int32_t)k; xp.R = (int32_t)R;
    xp.l2g = s->l2g.p; xp.roots_local = s->roots_local.p; xp.comp_off = s->comp_off.p;
    xp.e_row = s->e_row.p; xp.e_col = s->e_col.p; xp.e_gid = s->e_gid.p;
    xp.root_voff = s->root_voff.p; xp.root_eoff = s->root_eoff.p;
    xp.xv = s->xv.p; xp.ye = s->ye.p; xp.lab = s->lab.p;
    xp.v_cap = (int64_t)s->v_cap; xp.e_cap = (int64_t)s->e_cap;
    xp.status = s->status.p; xp.bbase = s->bbase.p; xp.ticket = s->ticket.p;
    xp.hs_bits = c.hs_bits; xp.set_cap = c.set_cap; xp.row_cap = c.row_cap;
    xp.stage_cap = c.stage_cap; xp.warp_bytes = c.warp_bytes;
    if (R > 0) {
        launch_extract(s, c, xp);
        ++s->launches;
    }
    if (s->profiled) HGS_CUDA(cudaEventRecord(s->ev[2], st));
    k_finalize<<<(unsigned)((k + 1 + 255) / 256), 256, 0, st>>>(in.batch_off, (int32_t)k, (int32_t)R,
                                                               s->root_voff.p, s->root_eoff.p,
                                                               s->batch_voff.p, s->batch_eoff.p,
                                                               s->comp_off.p);
    HGS_CUDA(cudaGetLastError());
    ++s->launches;
    if (s->profiled) HGS_CUDA(cudaEventRecord(s->ev[3], st));
    // small state back to pinned host memory: error words + totals
    if (!s->h_state) HGS_CUDA(cudaMallocHost(&s->h_state, 16 * sizeof(int32_t)));
    HGS_CUDA(cudaMemcpyAsync(s->h_state, s->ticket.p, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaMemcpyAsync(s->h_state + 4, s->batch_voff.p + k, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaMemcpyAsync(s->h_state + 5, s->batch_eoff.p + k, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    s->pending = true;
    // keep the extract parameters for a capacity re-run
    static_assert(sizeof(ExtractParams) < 1024, "");
}

// Completes a call: checks device-side errors and re-runs the extract stage
// with grown outputs if the edge capacity estimate was too small.
void sample_finish(hgs_sample* s, const hgs_config& cfg, const CallInputs& in) {
    if (!s->pending) return;
    HGS_CUDA(cudaStreamSynchronize(s->stream));
    s->pending = false;
    const int32_t code = s->h_state[1];
    if (code == kErrRootRange)
        fail(HGS_EINVAL, "sampler: root " + std::to_string(s->h_state[3]) + " out of range");
    if (code == kErrNegative)
        fail(HGS_EINVAL, "row_normalize: negative value in a visited walk row (root ordinal " +
                             std::to_string(s->h_state[2]) + ", level " + std::to_string(s->h_state[3]) + ")");
    if (code == kErrOverflow)
        fail(HGS_ERANGE, "hgs: more than 2^31-1 sampled vertices/edges in one call; split the call");
    s->V = s->h_state[4];
    s->E = s->h_state[5];
    if (code == kErrCapacity) {
        // grow to the exact totals and run the whole call again (K1 is cheap)
        s->e_cap = (size_t)s->E + (size_t)s->E / 8 + 1024;
        s->e_row.release(); s->e_col.release(); s->e_gid.release(); s->ye.release(); s->lab.release();
        if ((size_t)s->V > s->v_cap) { s->v_cap = (size_t)s->V; s->l2g.release(); s->xv.release(); }
        sample_enqueue(s, cfg, in);
        sample_finish(s, cfg, in);
    }
}

}  // namespace hgs
