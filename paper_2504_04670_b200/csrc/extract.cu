// extract.cu — K2 (dedup + induced-subgraph extraction), the per-call offset
// scan, K3 (block-diagonal packing + feature/label gather) and small helpers.
//
// K2 k_extract, one warp per root:
//   sorted_vertex_set (sampler.cpp:48-53): the touched list is inserted into a
//   shared-memory hash set (4-slot buckets probed with one 16-byte LDS), the
//   unique vertices are bitonic-sorted in registers and written back over the
//   touched slot; ranks (local ids) go into the table.
//   induced_subgraph = S·A·Sᵀ (sparse.cpp:177-191) on the directed edge-id
//   matrix A: the A rows of the set, in local order, are flattened into one
//   index space and scanned in 32-wide coalesced windows (row owner of every
//   lane from a __reduce_or_sync bitmask of row starts), each column probed in
//   the hash set; hits come out row-major with ascending columns, i.e. in the
//   reference's CSR order, and are appended to the root's edge slot.
// Offsets: exclusive scan of (V_r, E_r) over roots (block_diag offsets,
//   sparse.cpp:245-258) — three small launches.
// K3 k_pack, one warp per root: rebases into batch-local ids, writes
//   local_to_global / roots_local / component offsets / COO edges / edge ids,
//   and gathers node rows, edge rows and labels (gather_features,
//   sampler.cpp:211-243) with 16-byte vector stores.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace hgs {

namespace {

constexpr uint32_t kEmpty = 0xffffffffu;

// Shared-memory hash set of the root's vertex set mapping vertex -> local id
// (rank in the sorted set). 4-slot buckets, one 16-byte LDS per probed
// bucket; slots of a bucket fill in order, so a bucket with a free slot ends
// a miss. PACKED: entry = vertex << rank_bits | rank (32 bit) and a bucket is
// 4 entries; otherwise entry = (vertex, rank) and a bucket spans 2 x 16 B.
template <bool PACKED>
struct HashSet;

template <>
struct HashSet<true> {
    uint32_t* slot;
    uint32_t bmask, rmask;
    int bits, rb;
    static constexpr int kBytesPerSlot = 4;
    __device__ __forceinline__ uint32_t bucket(uint32_t v) const { return (v * 0x9E3779B1u) >> (32 - bits); }
    __device__ __forceinline__ void clear(int nslots) const {
        for (int i = lane_id(); i < nslots / 4; i += 32)
            reinterpret_cast<uint4*>(slot)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    }
    __device__ __forceinline__ bool insert(uint32_t v) const {
        const uint32_t e = (v << rb) | rmask, hi = v << rb;
        uint32_t b = bucket(v);
        for (;;) {
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint32_t prev = atomicCAS(slot + 4 * b + s, kEmpty, e);
                if (prev == kEmpty) return true;
                if ((prev ^ hi) <= rmask) return false;
            }
            b = (b + 1) & bmask;
        }
    }
    __device__ __forceinline__ int find_slot(uint32_t v) const {
        const uint32_t hi = v << rb;
        uint32_t b = bucket(v);
        for (;;) {
            const uint4 q = *reinterpret_cast<const uint4*>(slot + 4 * b);
            if ((q.x ^ hi) <= rmask) return 4 * b;
            if ((q.y ^ hi) <= rmask) return 4 * b + 1;
            if ((q.z ^ hi) <= rmask) return 4 * b + 2;
            if ((q.w ^ hi) <= rmask) return 4 * b + 3;
            if (q.w == kEmpty) return -1;
            b = (b + 1) & bmask;
        }
    }
    __device__ __forceinline__ void set_rank(uint32_t v, uint32_t r) const { slot[find_slot(v)] = (v << rb) | r; }
    // (entry ^ (v << rb)) is the entry's rank for the matching entry and
    // exceeds rmask for every other entry (keys are distinct), so the
    // bucket's minimum decides a hit without per-slot branches.
    __device__ __forceinline__ int find_rank(uint32_t v) const {
        const uint32_t hi = v << rb;
        uint32_t b = bucket(v);
        uint4 q = *reinterpret_cast<const uint4*>(slot + 4 * b);
        uint32_t d = min(min(q.x ^ hi, q.y ^ hi), min(q.z ^ hi, q.w ^ hi));
        if (d > rmask && q.w != kEmpty) {  // full bucket without a match: rare
            do {
                b = (b + 1) & bmask;
                q = *reinterpret_cast<const uint4*>(slot + 4 * b);
                d = min(min(q.x ^ hi, q.y ^ hi), min(q.z ^ hi, q.w ^ hi));
            } while (d > rmask && q.w != kEmpty);
        }
        return d <= rmask ? (int)d : -1;
    }
};

template <>
struct HashSet<false> {
    uint2* slot;  // (vertex, rank)
    uint32_t bmask, rmask;
    int bits, rb;
    static constexpr int kBytesPerSlot = 8;
    __device__ __forceinline__ uint32_t bucket(uint32_t v) const { return (v * 0x9E3779B1u) >> (32 - bits); }
    __device__ __forceinline__ void clear(int nslots) const {
        for (int i = lane_id(); i < nslots; i += 32) slot[i] = make_uint2(kEmpty, 0);
    }
    __device__ __forceinline__ bool insert(uint32_t v) const {
        uint32_t b = bucket(v);
        for (;;) {
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint32_t prev = atomicCAS(&slot[4 * b + s].x, kEmpty, v);
                if (prev == kEmpty) return true;
                if (prev == v) return false;
            }
            b = (b + 1) & bmask;
        }
    }
    __device__ __forceinline__ int find_slot(uint32_t v) const {
        uint32_t b = bucket(v);
        for (;;) {
            const uint4 q0 = *reinterpret_cast<const uint4*>(slot + 4 * b);
            const uint4 q1 = *reinterpret_cast<const uint4*>(slot + 4 * b + 2);
            if (q0.x == v) return 4 * b;
            if (q0.z == v) return 4 * b + 1;
            if (q1.x == v) return 4 * b + 2;
            if (q1.z == v) return 4 * b + 3;
            if (q1.z == kEmpty) return -1;
            b = (b + 1) & bmask;
        }
    }
    __device__ __forceinline__ void set_rank(uint32_t v, uint32_t r) const { slot[find_slot(v)].y = r; }
    __device__ __forceinline__ int find_rank(uint32_t v) const {
        uint32_t b = bucket(v);
        for (;;) {
            const uint4 q0 = *reinterpret_cast<const uint4*>(slot + 4 * b);
            const uint4 q1 = *reinterpret_cast<const uint4*>(slot + 4 * b + 2);
            int r = -1;
            r = (q1.z == v) ? (int)q1.w : r;
            r = (q1.x == v) ? (int)q1.y : r;
            r = (q0.z == v) ? (int)q0.w : r;
            r = (q0.x == v) ? (int)q0.y : r;
            if (r >= 0 || q1.z == kEmpty) return r;
            b = (b + 1) & bmask;
        }
    }
};

template <int E>
__device__ __forceinline__ void sort_regs(int32_t* set, int U) {
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
    __syncwarp();
}

__device__ void sort_smem(int32_t* set, int U, int N) {
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

}  // namespace

// ===========================================================================
// K2
// ===========================================================================

template <bool PACKED, bool HAS_GID>
__global__ void __launch_bounds__(128, 6) k_extract(ExtractParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = lane_id();
    const int warp = threadIdx.x >> 5;
    unsigned char* q = smem_raw + (size_t)warp * p.warp_bytes;
    const int nslots = 4 << p.nb_bits;
    HashSet<PACKED> hs;
    hs.slot = reinterpret_cast<decltype(hs.slot)>(q);
    q += HashSet<PACKED>::kBytesPerSlot * nslots;
    int32_t* set = (int32_t*)q; q += 4 * p.set_cap;
    // after the set is dead its space holds, per 32-entry window, the row of
    // the window's first entry (wcur) and a bitmask of rows starting inside it
    uint32_t* wmask = reinterpret_cast<uint32_t*>(set);
    uint16_t* wcur = reinterpret_cast<uint16_t*>(set + p.win_cap);
    int32_t* rstart = (int32_t*)q; q += 4 * (p.row_cap + 36);
    int2* rinfo = (int2*)q;  // per nonempty row: (A position - flat index, local id)
    hs.bits = p.nb_bits;
    hs.bmask = (1u << p.nb_bits) - 1u;
    hs.rb = p.rank_bits;
    hs.rmask = (1u << p.rank_bits) - 1u;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned le = (2u << lane) - 1u;

    const int nwarps = gridDim.x * (blockDim.x >> 5);
    for (int r = blockIdx.x * (blockDim.x >> 5) + warp; r < p.R; r += nwarps) {
        int32_t* tl = p.touched + (size_t)r * p.stride;
        const int T = p.tcount[r];
        const int32_t root = tl[0];  // before the slot is overwritten by the set

        // ---- dedup: hash-insert the touched list, compact the new keys
        hs.clear(nslots);
        __syncwarp();
        int U = 0;
        for (int b0 = 0; b0 < T; b0 += 32) {
            const int idx = b0 + lane;
            bool fresh = false;
            int32_t v = 0;
            if (idx < T) {
                v = tl[idx];
                fresh = hs.insert((uint32_t)v);
            }
            const unsigned fb = __ballot_sync(kFull, fresh);
            if (fresh) set[U + __popc(fb & lt)] = v;
            U += __popc(fb);
        }
        __syncwarp();
        if (U <= 32) sort_regs<1>(set, U);
        else if (U <= 64) sort_regs<2>(set, U);
        else if (U <= 128) sort_regs<4>(set, U);
        else if (U <= 256) sort_regs<8>(set, U);
        else {  // large sets: bitonic in the (not yet used) row arrays
            int N = 512;
            while (N < U) N <<= 1;
            int32_t* scr = rstart;
            for (int i = lane; i < U; i += 32) scr[i] = set[i];
            __syncwarp();
            sort_smem(scr, U, N);
            for (int i = lane; i < U; i += 32) set[i] = scr[i];
            __syncwarp();
        }

        // ---- ranks, the sorted set back to global, nonempty A rows
        int NR = 0, S = 0;
        for (int b0 = 0; b0 < U; b0 += 32) {
            const int i = b0 + lane;
            int32_t rb = 0, deg = 0;
            if (i < U) {
                const int32_t u = set[i];
                hs.set_rank((uint32_t)u, (uint32_t)i);
                tl[i] = u;
                rb = __ldg(p.a_rp + u);
                deg = __ldg(p.a_rp + u + 1) - rb;
            }
            const bool ne = deg > 0;
            const unsigned nb = __ballot_sync(kFull, ne);
            const int incl = warp_incl_scan(deg);
            if (ne) {
                const int qi = NR + __popc(nb & lt);
                const int st = S + incl - deg;
                rstart[qi] = st;
                rinfo[qi] = make_int2(rb - st, i);
            }
            NR += __popc(nb);
            S += __shfl_sync(kFull, incl, 31);
        }
        if (lane == 0) rstart[NR] = S;
        __syncwarp();

        // ---- window cursors: row holding the first entry of each 32-window
        for (int i = NR + 1 + lane; i <= NR + 32; i += 32) rstart[i] = 0x7fffffff;  // sentinels
        const int nwin = (S + 31) >> 5;
        const bool direct = nwin <= p.win_cap;
        if (direct) {
            for (int w = lane; w < nwin; w += 32) wmask[w] = 0u;
            __syncwarp();
            for (int qi = lane; qi < NR; qi += 32) {
                const int s0 = rstart[qi], s1 = rstart[qi + 1];
                if (s0 & 31) atomicOr(&wmask[s0 >> 5], 1u << (s0 & 31));
                for (int w = (s0 + 31) >> 5; (w << 5) < s1; ++w) wcur[w] = (uint16_t)qi;
            }
        }
        __syncwarp();

        // ---- induced subgraph: scan the flattened rows in 32-entry windows
        int2* const ed = p.escratch + (size_t)r * p.e_stride;
        const unsigned es = (unsigned)p.e_stride;
        int count = 0;
        // Row owning lane's entry of window w, given the row c holding the
        // window's first entry: c + #row starts in (base, base + lane].
        auto owner = [&](int c, int base) -> int {
            const int off = rstart[c + 1 + lane] - base;
            const unsigned bit = ((unsigned)(off - 1) < 31u) ? (1u << off) : 0u;
            return c + __popc(__reduce_or_sync(kFull, bit) & le);
        };
        // Emit the hits of one window in scan order. The capacity check is
        // hoisted: `room` says every lane's slot fits (count + 32 <= stride).
        auto emit = [&](int j, int own, int kk) {
            const unsigned hb = __ballot_sync(kFull, j >= 0);
            const unsigned t = (unsigned)count + __popc(hb & lt);
            if (j >= 0 && t < es) {
                const int32_t gid = HAS_GID ? __ldg(p.a_gid + kk) : kk;
                ed[t] = make_int2((rinfo[own].y << 16) | j, gid);
            }
            count += __popc(hb);
        };
        constexpr int G = 4;  // windows in flight per iteration
        auto group = [&](int w, bool guard) {
            int own[G], kk[G];
            uint32_t v[G];
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const int base = (w + u) << 5;
                if (!guard || w + u < nwin) {
                    own[u] = (int)wcur[w + u] + __popc(wmask[w + u] & le);
                    if (guard) own[u] = min(own[u], NR - 1);
                    kk[u] = base + lane + rinfo[own[u]].x;
                    if (guard && base + lane >= S) kk[u] = -1;
                } else {
                    own[u] = 0;
                    kk[u] = -1;
                }
            }
#pragma unroll
            for (int u = 0; u < G; ++u) v[u] = (!guard || kk[u] >= 0) ? (uint32_t)__ldg(p.a_ci + kk[u]) : 0u;
#pragma unroll
            for (int u = 0; u < G; ++u) {
                if (!guard || w + u < nwin) emit((!guard || kk[u] >= 0) ? hs.find_rank(v[u]) : -1, own[u], kk[u]);
            }
        };
        // Full groups are software-pipelined: the column loads of group g+1
        // are in flight while group g is probed and emitted.
        auto fetch = [&](int w, int (&own)[G], int (&kk)[G], uint32_t (&v)[G]) {
#pragma unroll
            for (int u = 0; u < G; ++u) {
                own[u] = (int)wcur[w + u] + __popc(wmask[w + u] & le);
                kk[u] = ((w + u) << 5) + lane + rinfo[own[u]].x;
            }
#pragma unroll
            for (int u = 0; u < G; ++u) v[u] = (uint32_t)__ldg(p.a_ci + kk[u]);
        };
        auto consume = [&](const int (&own)[G], const int (&kk)[G], const uint32_t (&v)[G]) {
#pragma unroll
            for (int u = 0; u < G; ++u) emit(hs.find_rank(v[u]), own[u], kk[u]);
        };
        int w = 0;
        if (direct) {
            const int nfg = (S >> 5) / G;  // groups whose windows are all full
            if (nfg > 0) {
                int ownA[G], kkA[G], ownB[G], kkB[G];
                uint32_t vA[G], vB[G];
                fetch(0, ownA, kkA, vA);
                for (int gi = 0; gi < nfg; gi += 2) {
                    if (gi + 1 < nfg) fetch((gi + 1) * G, ownB, kkB, vB);
                    consume(ownA, kkA, vA);
                    if (gi + 1 < nfg) {
                        if (gi + 2 < nfg) fetch((gi + 2) * G, ownA, kkA, vA);
                        consume(ownB, kkB, vB);
                    }
                }
                w = nfg * G;
            }
            for (; w < nwin; w += G) group(w, true);
        } else {
            int cursor = 0;  // huge sets: serial window cursor
            for (; w < nwin; ++w) {
                const int base = w << 5;
                const int own = min(owner(cursor, base), NR - 1);
                const int own31 = __shfl_sync(kFull, own, 31);
                cursor = (rstart[own31 + 1] == base + 32) ? own31 + 1 : own31;
                const int pos = base + lane;
                const int kk = pos < S ? pos + rinfo[own].x : -1;
                const int j = kk >= 0 ? hs.find_rank((uint32_t)__ldg(p.a_ci + kk)) : -1;
                emit(j, own, kk);
            }
        }
        if (lane == 0) {
            p.root_nv[r] = U;
            p.root_ne[r] = count;
            p.root_rloc[r] = hs.find_rank((uint32_t)root);
            p.root_scan[r] = S;
            if (count > p.e_stride) {
                atomicMax(&p.ticket[4], count);
                report(p.ticket, kErrCapacity, r, count);
            }
        }
        __syncwarp();
    }
}

// ===========================================================================
// offsets: exclusive scan of (V_r, E_r)
// ===========================================================================

constexpr int kPairTile = 1024;  // roots per tile, 256 threads x 4

__device__ __forceinline__ void block_scan_pair(int64_t& a, int64_t& b, int64_t* sh, int64_t& ta, int64_t& tb) {
    // exclusive block scan of two int64 values; sh holds 2*33 entries
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int64_t ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t xa = __shfl_up_sync(kFull, ia, o), xb = __shfl_up_sync(kFull, ib, o);
        if (lane >= o) { ia += xa; ib += xb; }
    }
    if (lane == 31) { sh[wid] = ia; sh[33 + wid] = ib; }
    __syncthreads();
    if (wid == 0) {
        int64_t wa = lane < nw ? sh[lane] : 0, wb = lane < nw ? sh[33 + lane] : 0;
        int64_t sa = wa, sb = wb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t xa = __shfl_up_sync(kFull, sa, o), xb = __shfl_up_sync(kFull, sb, o);
            if (lane >= o) { sa += xa; sb += xb; }
        }
        if (lane < nw) { sh[lane] = sa - wa; sh[33 + lane] = sb - wb; }
        if (lane == nw - 1) { sh[32] = sa; sh[65] = sb; }
    }
    __syncthreads();
    ta = sh[32];
    tb = sh[65];
    a = sh[wid] + ia - a;
    b = sh[33 + wid] + ib - b;
    __syncthreads();
}

__global__ void k_scan_reduce(const int32_t* __restrict__ nv, const int32_t* __restrict__ ne, int32_t R,
                              int64_t* __restrict__ tile_sums) {
    __shared__ int64_t sh[66];
    int64_t a = 0, b = 0;
    const int base = blockIdx.x * kPairTile + threadIdx.x * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (base + i < R) { a += nv[base + i]; b += ne[base + i]; }
    int64_t ta, tb;
    block_scan_pair(a, b, sh, ta, tb);
    if (threadIdx.x == 0) { tile_sums[2 * blockIdx.x] = ta; tile_sums[2 * blockIdx.x + 1] = tb; }
}

__global__ void k_scan_tiles(int64_t* __restrict__ tile_sums, int32_t tiles, int32_t* __restrict__ ticket) {
    __shared__ int64_t sh[66];
    __shared__ int64_t carry[2];
    if (threadIdx.x == 0) { carry[0] = 0; carry[1] = 0; }
    __syncthreads();
    for (int t0 = 0; t0 < tiles; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        int64_t a = t < tiles ? tile_sums[2 * t] : 0, b = t < tiles ? tile_sums[2 * t + 1] : 0;
        int64_t ta, tb;
        block_scan_pair(a, b, sh, ta, tb);
        if (t < tiles) { tile_sums[2 * t] = carry[0] + a; tile_sums[2 * t + 1] = carry[1] + b; }
        __syncthreads();
        if (threadIdx.x == 0) { carry[0] += ta; carry[1] += tb; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        tile_sums[2 * tiles] = carry[0];
        tile_sums[2 * tiles + 1] = carry[1];
        if (carry[0] > 0x7fffffff || carry[1] > 0x7fffffff) report(ticket, kErrOverflow, 0, 0);
    }
}

__global__ void k_scan_apply(const int32_t* __restrict__ nv, const int32_t* __restrict__ ne, int32_t R,
                             const int64_t* __restrict__ tile_offs, int32_t tiles,
                             int32_t* __restrict__ voff, int32_t* __restrict__ eoff) {
    __shared__ int64_t sh[66];
    int64_t x[4], y[4], a = 0, b = 0;
    const int base = blockIdx.x * kPairTile + threadIdx.x * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        x[i] = base + i < R ? nv[base + i] : 0;
        y[i] = base + i < R ? ne[base + i] : 0;
        a += x[i];
        b += y[i];
    }
    int64_t ta, tb;
    block_scan_pair(a, b, sh, ta, tb);
    a += tile_offs[2 * blockIdx.x];
    b += tile_offs[2 * blockIdx.x + 1];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (base + i < R) { voff[base + i] = (int32_t)a; eoff[base + i] = (int32_t)b; }
        a += x[i];
        b += y[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        voff[R] = (int32_t)tile_offs[2 * tiles];
        eoff[R] = (int32_t)tile_offs[2 * tiles + 1];
    }
}

void launch_scan(const int32_t* nv, const int32_t* ne, int32_t R, int64_t* tmp, int32_t* voff,
                 int32_t* eoff, int32_t* ticket, cudaStream_t st) {
    const int tiles = (R + kPairTile - 1) / kPairTile;
    k_scan_reduce<<<tiles, 256, 0, st>>>(nv, ne, R, tmp);
    k_scan_tiles<<<1, 1024, 0, st>>>(tmp, tiles, ticket);
    k_scan_apply<<<tiles, 256, 0, st>>>(nv, ne, R, tmp, tiles, voff, eoff);
    HGS_CUDA(cudaGetLastError());
}

int64_t scan_tmp_words(int64_t R) { return 2 * ((R + kPairTile - 1) / kPairTile) + 4; }

// ===========================================================================
// K3
// ===========================================================================

__global__ void __launch_bounds__(256) k_pack(PackParams p) {
    extern __shared__ int32_t pack_smem[];
    const int lane = lane_id();
    int32_t* sset = pack_smem + (size_t)(threadIdx.x >> 5) * p.set_cap;  // the root's set, staged
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    constexpr int U = 4;  // independent loads in flight per lane
    for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < p.R; r += nwarps) {
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
        const int64_t vb = p.root_voff[r], eb = p.root_eoff[r];
        const int Vr = p.root_voff[r + 1] - (int32_t)vb;
        const int Er = p.root_eoff[r + 1] - (int32_t)eb;
        if (vb + Vr > p.v_cap || eb + Er > p.e_cap) {
            if (lane == 0) report(p.ticket, kErrCapacity, r, -1);
            continue;
        }
        const int32_t loc = (int32_t)vb - p.root_voff[f];
        const int32_t* set = p.touched + (size_t)r * p.stride;
        for (int i = lane; i < Vr; i += 32) {
            const int32_t u = set[i];
            sset[i] = u;
            __stcs(p.l2g + vb + i, u);
        }
        if (lane == 0) {
            p.roots_local[r] = loc + p.root_rloc[r];
            p.comp_off[r + b] = loc;
            if (r == p.batch_off[b + 1] - 1) p.comp_off[r + 1 + b] = loc + Vr;
        }
        const int2* ed = p.escratch + (size_t)r * p.e_stride;
        const bool fe2 = p.gather && p.f_e == 2;
        for (int t0 = 0; t0 < Er; t0 += 32 * U) {
            int2 e[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = t0 + 32 * u + lane;
                e[u] = t < Er ? ed[t] : make_int2(0, -1);
            }
            double2 x[U];
            uint8_t lb[U];
            if (p.gather) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (e[u].y >= 0) {
                        lb[u] = __ldg(p.labels + e[u].y);
                        if (fe2) x[u] = __ldg(reinterpret_cast<const double2*>(p.edge_feat) + e[u].y);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = t0 + 32 * u + lane;
                if (t < Er) {
                    __stcs(p.e_row + eb + t, loc + (e[u].x >> 16));
                    __stcs(p.e_col + eb + t, loc + (e[u].x & 0xffff));
                    __stcs(p.e_gid + eb + t, e[u].y);
                    if (p.gather) {
                        p.lab[eb + t] = lb[u];
                        if (fe2) {
                            __stcs(reinterpret_cast<double2*>(p.ye) + eb + t, x[u]);
                        } else {
                            for (int c = 0; c < p.f_e; ++c)
                                __stcs(p.ye + (eb + t) * p.f_e + c,
                                       __ldg(p.edge_feat + (int64_t)e[u].y * p.f_e + c));
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (p.gather) {
            if ((p.f_v & 1) == 0) {  // rows as f_v/2 16-byte pieces
                const int q2 = p.f_v >> 1;
                const int n2 = Vr * q2;
                const double2* src = reinterpret_cast<const double2*>(p.node_feat);
                double2* dst = reinterpret_cast<double2*>(p.xv) + vb * q2;
                for (int e0 = 0; e0 < n2; e0 += 32 * U) {
                    double2 x[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int e = e0 + 32 * u + lane;
                        if (e < n2) {
                            const int i = (int)__umulhi((unsigned)e, p.fv_magic);
                            x[u] = __ldg(src + (int64_t)sset[i] * q2 + (e - i * q2));
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int e = e0 + 32 * u + lane;
                        if (e < n2) __stcs(dst + e, x[u]);
                    }
                }
            } else {
                double* dst = p.xv + vb * p.f_v;
                for (int e = lane; e < Vr * p.f_v; e += 32) {
                    const int i = e / p.f_v;
                    __stcs(dst + e, __ldg(p.node_feat + (int64_t)sset[i] * p.f_v + (e - i * p.f_v)));
                }
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
        batch_voff[b] = root_voff[f];
        batch_eoff[b] = root_eoff[f];
        if (b < k && batch_off[b + 1] == f) comp_off[f + b] = 0;  // empty batch
    }
}

// ===========================================================================
// standalone gather + stats
// ===========================================================================

__global__ void k_gather(const double* __restrict__ node_feat, int32_t f_v,
                         const double* __restrict__ edge_feat, int32_t f_e,
                         const uint8_t* __restrict__ labels, const int64_t* __restrict__ l2g,
                         int64_t V, const int64_t* __restrict__ eid, int64_t E,
                         double* __restrict__ xv, double* __restrict__ ye, uint8_t* __restrict__ lab) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t e = t0; e < V * f_v; e += stride) {
        const int64_t i = e / f_v;
        xv[e] = node_feat[l2g[i] * f_v + (e - i * f_v)];
    }
    for (int64_t e = t0; e < E * f_e; e += stride) {
        const int64_t i = e / f_e;
        ye[e] = edge_feat[eid[i] * f_e + (e - i * f_e)];
    }
    for (int64_t i = t0; i < E; i += stride) lab[i] = labels[eid[i]];
}

__global__ void k_stats(const int32_t* __restrict__ level_counts, int32_t depth,
                        const int32_t* __restrict__ root_scan, const uint32_t* __restrict__ decisions,
                        const uint32_t* __restrict__ draws, int32_t R,
                        unsigned long long* __restrict__ out) {
    unsigned long long acc[3 + 16] = {};
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
        acc[0] += (unsigned)root_scan[r];
        acc[1] += decisions[r];
        acc[2] += draws[r];
        for (int l = 0; l <= depth && l < 16; ++l) acc[3 + l] += (unsigned)level_counts[(size_t)r * (depth + 1) + l];
    }
    for (int i = 0; i < 3 + 16; ++i) {
        unsigned long long v = acc[i];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(out + i, v);
    }
}

// ---- launchers -----------------------------------------------------------------

void launch_extract(int grid, size_t smem, const ExtractParams& xp, bool packed, cudaStream_t st) {
    auto kern = packed ? (xp.a_gid ? k_extract<true, true> : k_extract<true, false>)
                       : (xp.a_gid ? k_extract<false, true> : k_extract<false, false>);
    HGS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, 128, smem, st>>>(xp);
    HGS_CUDA(cudaGetLastError());
}

int extract_blocks_per_sm(size_t smem, bool packed) {
    auto kern = packed ? k_extract<true, false> : k_extract<false, false>;
    HGS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    HGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
    return per_sm > 0 ? per_sm : 1;
}

void launch_pack(int grid, const PackParams& pp, cudaStream_t st) {
    const size_t smem = (size_t)8 * pp.set_cap * sizeof(int32_t);
    if (smem > 48 * 1024)
        HGS_CUDA(cudaFuncSetAttribute(k_pack, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_pack<<<grid, 256, smem, st>>>(pp);
    HGS_CUDA(cudaGetLastError());
}

void launch_finalize(const int64_t* batch_off, int32_t k, int32_t R, const int32_t* voff,
                     const int32_t* eoff, int32_t* bvoff, int32_t* beoff, int32_t* comp_off,
                     cudaStream_t st) {
    k_finalize<<<(unsigned)((k + 1 + 255) / 256), 256, 0, st>>>(batch_off, k, R, voff, eoff, bvoff, beoff,
                                                               comp_off);
    HGS_CUDA(cudaGetLastError());
}

void launch_gather(const DevGraph& g, const int64_t* d_l2g, int64_t V, const int64_t* d_eid, int64_t E,
                   double* d_xv, double* d_ye, uint8_t* d_lab, cudaStream_t st) {
    const int64_t work = std::max<int64_t>(std::max<int64_t>(V * g.f_v, E * g.f_e), std::max<int64_t>(E, 1));
    const unsigned grid = (unsigned)std::min<int64_t>((work + 255) / 256, 148 * 16);
    k_gather<<<grid, 256, 0, st>>>(g.node_feat.p, g.f_v, g.edge_feat.p, g.f_e, g.labels.p, d_l2g, V, d_eid,
                                   E, d_xv, d_ye, d_lab);
    HGS_CUDA(cudaGetLastError());
}

void launch_stats(const int32_t* level_counts, int32_t depth, const int32_t* root_scan,
                  const uint32_t* decisions, const uint32_t* draws, int32_t R,
                  unsigned long long* out, cudaStream_t st) {
    if (R <= 0) return;
    k_stats<<<(unsigned)std::min<int64_t>((R + 255) / 256, 1024), 256, 0, st>>>(
        level_counts, depth, root_scan, decisions, draws, R, out);
    HGS_CUDA(cudaGetLastError());
}

}  // namespace hgs
