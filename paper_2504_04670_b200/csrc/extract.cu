// extract.cu — K2 (dedup + induced-subgraph extraction), the per-call offset
// scan, K3 (block-diagonal packing + feature/label gather) and small helpers.
//
// K2 k_extract, one warp per root:
//   sorted_vertex_set (sampler.cpp:48-53): the touched list is deduplicated
//   through a shared-memory hash set (4-slot buckets, CAS inserts), the unique
//   vertices are sorted by an order-preserving bucket sort and written back
//   over the touched slot; their ranks are the local ids.
//   The hash words are then re-laid as two one-slot cuckoo tables of packed
//   (vertex, rank) entries, so a scan probe is two independent 4-byte loads.
//   induced_subgraph = S·A·Sᵀ (sparse.cpp:177-191) on the directed edge-id
//   matrix A: the A rows of the set, in local order, are flattened into one
//   index space and scanned in 32-wide coalesced windows (row owner of every
//   lane from a bitmask of row starts per window), each column probed in the
//   cuckoo tables; hits come out row-major with ascending columns, i.e. in the
//   reference's CSR order, and are appended to the root's edge slot.
// Offsets: exclusive scan of (V_r, E_r) over roots (block_diag offsets,
//   sparse.cpp:245-258) — three small launches.
// K3 k_pack, one warp per root: rebases into batch-local ids, writes
//   local_to_global / roots_local / component offsets / COO edges / edge ids,
//   and gathers node rows, edge rows and labels (gather_features,
//   sampler.cpp:211-243) with 16-byte vector stores.
#include <cuda_runtime.h>

#include <type_traits>

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

#ifndef HGS_K2_BW
#define HGS_K2_BW 4  // slots per bucket of the packed hash (2: one 8-byte LDS per probe)
#endif
template <>
struct HashSet<true> {
    static constexpr int BW = HGS_K2_BW;
    using Vec = std::conditional_t<BW == 4, uint4, std::conditional_t<BW == 2, uint2, uint32_t>>;
    uint32_t* slot;
    uint32_t nb, rmask;  // nb buckets of BW slots (any count)
    int rb;
    static constexpr int kBytesPerSlot = 4;
    __device__ __forceinline__ void set_buckets(uint32_t nb4) { nb = nb4 * (4 / BW); }
    __device__ __forceinline__ uint32_t bucket(uint32_t v) const { return __umulhi(v * 0x9E3779B1u, nb); }
    __device__ __forceinline__ uint32_t next(uint32_t b) const { return b + 1 == nb ? 0u : b + 1; }
    __device__ __forceinline__ void clear(int nslots) const {
        for (int i = lane_id(); i < nslots / 4; i += 32)
            reinterpret_cast<uint4*>(slot)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    }
    // spill is set when the key lands outside its home bucket
    __device__ __forceinline__ bool insert(uint32_t v, bool& spill) const {
        const uint32_t e = (v << rb) | rmask, hi = v << rb;
        uint32_t b = bucket(v);
        for (;;) {
#pragma unroll
            for (int s = 0; s < BW; ++s) {
                const uint32_t prev = atomicCAS(slot + BW * b + s, kEmpty, e);
                if (prev == kEmpty) return true;
                if ((prev ^ hi) <= rmask) return false;
            }
            b = next(b);
            spill = true;
        }
    }
    __device__ __forceinline__ int find_slot(uint32_t v) const {
        const uint32_t hi = v << rb;
        uint32_t b = bucket(v);
        for (;;) {
#pragma unroll
            for (int s = 0; s < BW; ++s)
                if ((slot[BW * b + s] ^ hi) <= rmask) return BW * b + s;
            if (slot[BW * b + BW - 1] == kEmpty) return -1;
            b = next(b);
        }
    }
    __device__ __forceinline__ void set_slot_rank(int sl, uint32_t v, uint32_t r) const { slot[sl] = (v << rb) | r; }
    __device__ __forceinline__ static uint32_t bmin(const uint4& q, uint32_t hi) {
        return min(min(q.x ^ hi, q.y ^ hi), min(q.z ^ hi, q.w ^ hi));
    }
    __device__ __forceinline__ static uint32_t bmin(const uint2& q, uint32_t hi) { return min(q.x ^ hi, q.y ^ hi); }
    __device__ __forceinline__ static uint32_t bmin(const uint32_t& q, uint32_t hi) { return q ^ hi; }
    __device__ __forceinline__ static uint32_t blast(const uint32_t& q) { return q; }
    __device__ __forceinline__ static uint32_t blast(const uint4& q) { return q.w; }
    __device__ __forceinline__ static uint32_t blast(const uint2& q) { return q.y; }
    // (entry ^ (v << rb)) is the entry's rank for the matching entry and
    // exceeds rmask for every other entry (keys are distinct), so the
    // bucket's minimum decides a hit without per-slot branches.
    __device__ __forceinline__ int find_rank(uint32_t v) const {
        const uint32_t hi = v << rb;
        uint32_t b = bucket(v);
        Vec q = *reinterpret_cast<const Vec*>(slot + BW * b);
        uint32_t d = bmin(q, hi);
        if (d > rmask && blast(q) != kEmpty) {  // full bucket without a match: rare
            do {
                b = next(b);
                q = *reinterpret_cast<const Vec*>(slot + BW * b);
                d = bmin(q, hi);
            } while (d > rmask && blast(q) != kEmpty);
        }
        return d <= rmask ? (int)d : -1;
    }
    // insert a final (vertex, rank) entry of a key known to be absent
    __device__ __forceinline__ void insert_entry(uint32_t v, uint32_t r) const {
        const uint32_t e = (v << rb) | r;
        uint32_t b = bucket(v);
        for (;;) {
#pragma unroll
            for (int s = 0; s < BW; ++s)
                if (atomicCAS(slot + BW * b + s, kEmpty, e) == kEmpty) return;
            b = next(b);
        }
    }
    // Scan-time cuckoo layout of the same words: two one-slot tables of H
    // entries each; a key sits in T1[h1(v)] or T2[h2(v)], so a probe is two
    // independent 4-byte loads (~3.5 wavefronts each for 32 random lanes,
    // against ~10 for one 16-byte bucket load) and one compare.
    static constexpr uint32_t kC2 = 0x85EBCA77u;
    __device__ __forceinline__ uint32_t probe_cuckoo(uint32_t v, uint32_t H) const {
        const uint32_t hi = v << rb;
        const uint32_t e1 = slot[__umulhi(v * 0x9E3779B1u, H)];
        const uint32_t e2 = slot[H + __umulhi(v * kC2, H)];
        return min(e1 ^ hi, e2 ^ hi);
    }
    // concurrent cuckoo insert (atomicExch chains); false when the chain
    // exceeds its bound (the evicted entry is then dropped: caller rebuilds)
    __device__ __forceinline__ bool insert_cuckoo(uint32_t v, uint32_t r, uint32_t H, int iters) const {
        uint32_t e = (v << rb) | r;
        int t = 0;
        for (int it = 0; it < iters; ++it) {
            uint32_t* sl = t ? slot + H + __umulhi(v * kC2, H) : slot + __umulhi(v * 0x9E3779B1u, H);
            const uint32_t old = atomicExch(sl, e);
            if (old == kEmpty) return true;
            e = old;
            v = old >> rb;
            t ^= 1;
        }
        return false;
    }
    // home-bucket probe, raw: the rank on a hit, a value > rmask on a miss
    __device__ __forceinline__ uint32_t probe_home(uint32_t v) const {
        return bmin(*reinterpret_cast<const Vec*>(slot + BW * bucket(v)), v << rb);
    }
    // find_rank when no key of the set left its home bucket: one probe, no loop
    __device__ __forceinline__ int find_rank_home(uint32_t v) const {
        const uint32_t hi = v << rb;
        const uint32_t d = bmin(*reinterpret_cast<const Vec*>(slot + BW * bucket(v)), hi);
        return d <= rmask ? (int)d : -1;
    }
};

template <>
struct HashSet<false> {
    uint2* slot;  // (vertex, rank)
    uint32_t nb, rmask;
    int rb;
    static constexpr int kBytesPerSlot = 8;
    __device__ __forceinline__ uint32_t bucket(uint32_t v) const { return __umulhi(v * 0x9E3779B1u, nb); }
    __device__ __forceinline__ uint32_t next(uint32_t b) const { return b + 1 == nb ? 0u : b + 1; }
    __device__ __forceinline__ void clear(int nslots) const {
        for (int i = lane_id(); i < nslots; i += 32) slot[i] = make_uint2(kEmpty, 0);
    }
    __device__ __forceinline__ bool insert(uint32_t v, bool& spill) const {
        uint32_t b = bucket(v);
        for (;;) {
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint32_t prev = atomicCAS(&slot[4 * b + s].x, kEmpty, v);
                if (prev == kEmpty) return true;
                if (prev == v) return false;
            }
            b = next(b);
            spill = true;
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
            b = next(b);
        }
    }
    __device__ __forceinline__ void set_slot_rank(int sl, uint32_t, uint32_t r) const { slot[sl].y = r; }
    __device__ __forceinline__ uint32_t probe_home(uint32_t v) const { return (uint32_t)find_rank_home(v); }
    // cuckoo layout is packed-only (never called)
    __device__ __forceinline__ uint32_t probe_cuckoo(uint32_t v, uint32_t) const { return (uint32_t)find_rank(v); }
    __device__ __forceinline__ bool insert_cuckoo(uint32_t, uint32_t, uint32_t, int) const { return false; }
    __device__ __forceinline__ void insert_entry(uint32_t, uint32_t) const {}
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
            b = next(b);
        }
    }
    __device__ __forceinline__ int find_rank_home(uint32_t v) const {
        const uint32_t b = bucket(v);
        const uint4 q0 = *reinterpret_cast<const uint4*>(slot + 4 * b);
        const uint4 q1 = *reinterpret_cast<const uint4*>(slot + 4 * b + 2);
        int r = -1;
        r = (q1.z == v) ? (int)q1.w : r;
        r = (q1.x == v) ? (int)q1.y : r;
        r = (q0.z == v) ? (int)q0.w : r;
        r = (q0.x == v) ? (int)q0.y : r;
        return r;
    }
};

}  // namespace

// ===========================================================================
// K2
// ===========================================================================

// Per-warp shared memory of K2 (set_cap == row_cap == max tree size rounded
// up to 32; the regions are reused phase by phase):
//   hash   4<<nb_bits slots                   vertex -> rank
//   keys   set_cap x i32   unsorted keys -> sorted keys -> per-window (mask, cursor)
//   tmp    row_cap+36 x i32  bucketed keys -> row starts (+ sentinels)
//   aux    row_cap x int2  bucket counters -> per nonempty row (A pos - flat pos, rank<<16)
#ifndef HGS_K2_MINB
#define HGS_K2_MINB 6  // CTAs per SM the register budget is sized for (80 registers; 7 CTAs at 72 measured slower)
#endif
// GMEM: the per-warp working set lives in a global scratch slot instead of
// shared memory (sets too large for one warp's shared memory; slow, rare).
template <bool PACKED, bool HAS_GID, bool GMEM>
__global__ void __launch_bounds__(128, HGS_K2_MINB) k_extract(ExtractParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = lane_id();
    const int warp = threadIdx.x >> 5;
    unsigned char* q = GMEM ? p.gscratch + ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * p.warp_bytes
                            : smem_raw + (size_t)warp * p.warp_bytes;
    const int nslots = 4 * p.n_buckets;
#ifndef HGS_K2_CUCKOO
#define HGS_K2_CUCKOO 1
#endif
    // the scan probes a cuckoo re-layout of the hash words (packed entries)
    constexpr bool CK = HGS_K2_CUCKOO && PACKED;
    HashSet<PACKED> hs;
    hs.slot = reinterpret_cast<decltype(hs.slot)>(q);
    q += HashSet<PACKED>::kBytesPerSlot * nslots;
    int32_t* keys = (int32_t*)q; q += 4 * p.set_cap;
    uint2* winfo = reinterpret_cast<uint2*>(keys);  // per window: (row-start mask, cursor row)
    int32_t* tmp = (int32_t*)q; q += 4 * (p.row_cap + 36);
    int32_t* rstart = tmp;
    int32_t* cnt = (int32_t*)q;
    int2* rinfo = (int2*)q;
    if constexpr (PACKED) hs.set_buckets((uint32_t)p.n_buckets);
    else hs.nb = (uint32_t)p.n_buckets;
    hs.rb = p.rank_bits;
    hs.rmask = (1u << p.rank_bits) - 1u;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned le = (2u << lane) - 1u;
    constexpr int CH = 4;  // 32-key chunks of row loads in flight

    // roots are handed out dynamically (per-root work varies ~6x), which
    // shortens the tail of the persistent grid
    auto next_root = [&]() -> int {
        int r = 0;
        if (lane == 0) r = p.r0 + atomicAdd(p.work, 1);
        return __shfl_sync(kFull, r, 0);
    };
    for (int r = next_root(); r < p.R; r = next_root()) {
        int32_t* tl = p.touched + (size_t)r * p.stride;
        const int T = p.tcount[r];

        // ---- dedup: hash-insert the touched list (next chunk's load in
        // flight), compact the fresh keys, track the id range
        hs.clear(nslots);
        __syncwarp();
        int U = 0;
        uint32_t lo = 0xffffffffu, hi = 0u;
        bool spill = false;
        int32_t nxt = lane < T ? tl[lane] : 0;
        const int32_t root = __shfl_sync(kFull, nxt, 0);
#pragma unroll 1
        for (int b0 = 0; b0 < T; b0 += 32) {
            const int32_t v = nxt;
            const bool valid = b0 + lane < T;
            nxt = b0 + 32 + lane < T ? tl[b0 + 32 + lane] : 0;
            const bool fresh = valid && hs.insert((uint32_t)v, spill);
            const unsigned fb = __ballot_sync(kFull, fresh);
            if (fresh) {
                keys[U + __popc(fb & lt)] = v;
                lo = min(lo, (uint32_t)v);
                hi = max(hi, (uint32_t)v);
            }
            U += __popc(fb);
        }
        if (U > kMaxSet) {  // local ids would not fit the edge slots: report, skip the root
            if (lane == 0) {
                report(p.ticket, kErrSetRange, r, U);
                p.root_nv[r] = 0; p.root_ne[r] = 0; p.root_rloc[r] = -1; p.root_scan[r] = 0;
            }
            __syncwarp();
            continue;
        }
        // every key in its home bucket (~80% of C2 roots): probes need no
        // chain walk. (Rebuilding the other roots' tables with another hash
        // multiplier measured no faster.)
        const bool home = !__any_sync(kFull, spill);
        lo = __reduce_min_sync(kFull, lo);
        hi = __reduce_max_sync(kFull, hi);
        // ---- order-preserving buckets b = (v - lo) >> shift, ~2U of them
        const int lg = min(p.cnt_lg, max(5, 32 - __clz(max(2 * U - 1, 1))));
        const int shift = max(0, (32 - __clz(hi - lo)) - lg);
        const int lp = lg - 5;  // counters per lane = 1 << lp
        const uint32_t pm = (1u << lp) - 1u;
        // counter of bucket b lives at ((b & pm) << 5) | (b >> lp): lane l's
        // consecutive buckets are one bank apart (conflict-free scan)
        auto cidx = [&](uint32_t b) -> int { return (int)(((b & pm) << 5) | (b >> lp)); };
        for (int i = lane; i < (8 << lp); i += 32) reinterpret_cast<int4*>(cnt)[i] = make_int4(0, 0, 0, 0);
        __syncwarp();
        for (int i = lane; i < U; i += 32) atomicAdd(&cnt[cidx(((uint32_t)keys[i] - lo) >> shift)], 1);
        __syncwarp();

        // ---- exclusive scan of the bucket counts (lane l owns buckets l<<lp ..)
        {
            int s = 0;
            for (int e = 0; e <= (int)pm; ++e) s += cnt[(e << 5) | lane];
            const int incl = warp_incl_scan(s);
            int run = incl - s;
            for (int e = 0; e <= (int)pm; ++e) {
                const int c = cnt[(e << 5) | lane];
                cnt[(e << 5) | lane] = run;
                run += c;
            }
        }
        __syncwarp();
        // ---- place keys into their buckets (counter becomes the bucket end)
        for (int i = lane; i < U; i += 32) {
            const uint32_t v = (uint32_t)keys[i];
            tmp[atomicAdd(&cnt[cidx((v - lo) >> shift)], 1)] = (int32_t)v;
        }
        __syncwarp();
        // ---- rank = bucket start + smaller keys of the same bucket; the
        // rank goes into the key's hash slot, found before any lane of the
        // chunk rewrites a slot (no lane reads a slot another lane writes)
        for (int i0 = 0; i0 < U; i0 += 32) {
            const int i = i0 + lane;
            int rank = 0, sl = -1;
            uint32_t v = 0;
            if (i < U) {
                v = (uint32_t)tmp[i];
                const uint32_t b = (v - lo) >> shift;
                const int e = cnt[cidx(b)];
                const int s = b ? cnt[cidx(b - 1)] : 0;
                // buckets hold ~1-2 keys: the first two compares without a loop
                const uint32_t t0 = (uint32_t)tmp[s], t1 = s + 1 < e ? (uint32_t)tmp[s + 1] : v;
                rank = s + (t0 < v) + (t1 < v);
                for (int j = s + 2; j < e; ++j) rank += (uint32_t)tmp[j] < v;
                keys[rank] = (int32_t)v;
                if constexpr (!CK) sl = hs.find_slot(v);
            }
            if constexpr (!CK) {
                __syncwarp();
                if (sl >= 0) hs.set_slot_rank(sl, v, (uint32_t)rank);
            }
            __syncwarp();
        }
        // ---- CK: re-lay the hash words as two one-slot cuckoo tables of
        // (vertex, rank) from the sorted keys; if a chain exceeds its bound,
        // the 4-slot table is rebuilt with final entries instead
        const uint32_t H = (uint32_t)nslots >> 1;
        bool ck = false;
        if constexpr (CK) {
            hs.clear(nslots);
            __syncwarp();
            bool ok = true;
            for (int i = lane; i < U; i += 32) ok = hs.insert_cuckoo((uint32_t)keys[i], (uint32_t)i, H, p.ck_iters) && ok;
            ck = __all_sync(kFull, ok);
            __syncwarp();
            if (!ck) {
                hs.clear(nslots);
                __syncwarp();
                for (int i = lane; i < U; i += 32) hs.insert_entry((uint32_t)keys[i], (uint32_t)i);
                __syncwarp();
            }
        }

        // ---- sorted set back to global; nonempty A rows in local order
        int NR = 0, S = 0;
        for (int b0 = 0; b0 < U; b0 += CH * 32) {
            int2 ri[CH];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int i = b0 + c * 32 + lane;
                ri[c] = make_int2(0, 0);
                if (i < U) {
                    const int32_t u = keys[i];
                    tl[i] = u;
                    ri[c] = __ldg(p.a_ri + u);
                }
            }
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (b0 + c * 32 >= U) break;
                const int i = b0 + c * 32 + lane;
                const int deg = ri[c].y;
                const bool ne = deg > 0;
                const unsigned nb = __ballot_sync(kFull, ne);
                const int incl = warp_incl_scan(deg);
                if (ne) {
                    const int qi = NR + __popc(nb & lt);
                    const int st = S + incl - deg;
                    rstart[qi] = st;
                    rinfo[qi] = make_int2(ri[c].x - st, i << 16);
                }
                NR += __popc(nb);
                S += __shfl_sync(kFull, incl, 31);
            }
        }
        if (lane == 0) rstart[NR] = S;
        __syncwarp();

        for (int i = NR + 1 + lane; i <= NR + 32; i += 32) rstart[i] = 0x7fffffff;  // sentinels
        const int nwin = (S + 31) >> 5;
        __syncwarp();

        // ---- induced subgraph: scan the flattened rows in 32-entry windows
        int2* const ed = p.escratch + (p.e_off ? (size_t)p.e_off[r] : (size_t)r * p.e_stride);
        int2* const ed_end = p.e_off ? p.escratch + p.e_off[r + 1] : ed + p.e_stride;
        int2* edc = ed;  // next free edge slot
        // Emit the hits of one window in scan order. CHK is set when the
        // slot might overflow: stores are then bounds-checked, overflow is
        // reported below and the host re-runs the call with larger slots.
        auto emit = [&](int j, int rowsh, int kk, auto chk) {
            const unsigned hb = ballot_nonneg(j);
            int2* dst = edc + __popc(hb & lt);
            if (j >= 0 && (!decltype(chk)::value || dst < ed_end))
                *dst = make_int2(rowsh | j, HAS_GID ? __ldg(p.a_gid + kk) : kk);
            edc += __popc(hb);
        };
// Windows per group: swept on B200 at C2 (G = 2 and 4 double-buffered,
// 5-8 single-buffered): 6 single-buffered groups were best with 16-byte
// bucket probes; with the cuckoo probes 7 is (K2 0.678 vs 0.700 ms; 4: 0.707,
// 5: 0.680, 8: 0.692).
#ifndef HGS_K2_G
#define HGS_K2_G 7
#endif
        constexpr int G = HGS_K2_G;  // windows in flight per group
        int wb = 0;  // first window of the current pass (window info is pass-local)
        auto fetch = [&](int w, int (&rs)[G], int (&kk)[G], uint32_t (&v)[G]) {
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const uint2 wi = winfo[w + u - wb];
                const int own = (int)wi.y + __popc(wi.x & le);
                const int2 ri = rinfo[own];
                kk[u] = ((w + u) << 5) + lane + ri.x;
                rs[u] = ri.y;
            }
#pragma unroll
            for (int u = 0; u < G; ++u) v[u] = (uint32_t)__ldg(p.a_ci + kk[u]);
        };
        // emit for a raw probe result d (the rank on a hit, > rmask on a
        // miss): the hit predicate feeds the vote and the store directly
        auto emit_d = [&](uint32_t d, int rowsh, int kk, auto chk) {
            const bool hit = d <= hs.rmask;
            const unsigned hb = __ballot_sync(kFull, hit);
            int2* dst = edc + __popc(hb & lt);
            if (hit && (!decltype(chk)::value || dst < ed_end))
                *dst = make_int2(rowsh | (int)d, HAS_GID ? __ldg(p.a_gid + kk) : kk);
            edc += __popc(hb);
        };
        // mode: 2 = cuckoo tables, 1 = home bucket only, 0 = bucket chain walk
        auto consume = [&](const int (&rs)[G], const int (&kk)[G], const uint32_t (&v)[G], auto mode) {
            if constexpr (decltype(mode)::value > 0) {
                uint32_t d[G];
#pragma unroll
                for (int u = 0; u < G; ++u)
                    d[u] = decltype(mode)::value == 2 ? hs.probe_cuckoo(v[u], H) : hs.probe_home(v[u]);
                if (edc + 32 * G <= ed_end) {
#pragma unroll
                    for (int u = 0; u < G; ++u) emit_d(d[u], rs[u], kk[u], std::false_type{});
                } else {
#pragma unroll
                    for (int u = 0; u < G; ++u) emit_d(d[u], rs[u], kk[u], std::true_type{});
                }
            } else {
                int j[G];
#pragma unroll
                for (int u = 0; u < G; ++u) j[u] = hs.find_rank(v[u]);
                if (edc + 32 * G <= ed_end) {
#pragma unroll
                    for (int u = 0; u < G; ++u) emit(j[u], rs[u], kk[u], std::false_type{});
                } else {
#pragma unroll
                    for (int u = 0; u < G; ++u) emit(j[u], rs[u], kk[u], std::true_type{});
                }
            }
        };
        // Windows go in passes of win_cap: per pass, the row cursor of each
        // window and a bitmask of row starts inside it (one u32 + one u16 per
        // window, in the dead key array), then the scan.
        for (; wb < nwin; wb += p.win_cap) {
            const int we = min(nwin, wb + p.win_cap);
            for (int w = lane; w < we - wb; w += 32) winfo[w].x = 0u;
            __syncwarp();
            for (int qi = lane; qi < NR; qi += 32) {
                const int s0 = rstart[qi], s1 = rstart[qi + 1];
                const int w0 = s0 >> 5;
                if ((s0 & 31) && w0 >= wb && w0 < we) atomicOr(&winfo[w0 - wb].x, 1u << (s0 & 31));
                for (int w = max((s0 + 31) >> 5, wb); w < we && (w << 5) < s1; ++w) winfo[w - wb].y = (uint32_t)qi;
            }
            __syncwarp();
            // full groups: G windows' column loads in flight together
            const int wfull = min(we, S >> 5);  // windows of the pass with 32 entries
            const int nfg = max(0, wfull - wb) / G;
            int w = wb;
            auto groups = [&](auto mode) {
                for (int gi = 0; gi < nfg; ++gi) {
                    int rsA[G], kkA[G];
                    uint32_t vA[G];
                    fetch(wb + gi * G, rsA, kkA, vA);
                    consume(rsA, kkA, vA, mode);
                }
            };
            if (CK && ck) groups(std::integral_constant<int, 2>{});
            else if (home) groups(std::integral_constant<int, 1>{});
            else groups(std::integral_constant<int, 0>{});
            w = wb + nfg * G;
            for (; w < we; ++w) {  // < G trailing windows, the last one possibly partial
                const int base = w << 5;
                const uint2 wi = winfo[w - wb];
                const int own = min((int)wi.y + __popc(wi.x & le), NR - 1);
                const int2 ri = rinfo[own];
                const int kk = base + lane < S ? base + lane + ri.x : -1;
                if (CK && ck) {
                    const uint32_t d = kk >= 0 ? hs.probe_cuckoo((uint32_t)__ldg(p.a_ci + kk), H) : ~0u;
                    emit_d(d, ri.y, kk, std::true_type{});
                } else {
                    const int j = kk >= 0 ? hs.find_rank((uint32_t)__ldg(p.a_ci + kk)) : -1;
                    emit(j, ri.y, kk, std::true_type{});
                }
            }
            __syncwarp();
        }
        const int count = (int)(edc - ed);
        if (lane == 0) {
            p.root_nv[r] = U;
            p.root_ne[r] = count;
            int rl = -1;
            if (T > 0) {
                if (CK && ck) {
                    const uint32_t d = hs.probe_cuckoo((uint32_t)root, H);
                    rl = d <= hs.rmask ? (int)d : -1;
                } else {
                    rl = hs.find_rank((uint32_t)root);
                }
            }
            p.root_rloc[r] = rl;
            p.root_scan[r] = S;
            if (count > (int)(ed_end - ed)) {
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

// carry: (voff, eoff) at the chunk start, or null for the first chunk
__global__ void k_scan_tiles(int64_t* __restrict__ tile_sums, int32_t tiles, const int32_t* __restrict__ cv,
                             const int32_t* __restrict__ ce, int32_t* __restrict__ ticket) {
    __shared__ int64_t sh[66];
    __shared__ int64_t carry[2];
    if (threadIdx.x == 0) {
        carry[0] = cv ? (int64_t)*cv : 0;
        carry[1] = ce ? (int64_t)*ce : 0;
    }
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

void launch_scan(const int32_t* nv, const int32_t* ne, int32_t r0, int32_t r1, int64_t* tmp, int32_t* voff,
                 int32_t* eoff, int32_t* ticket, cudaStream_t st) {
    const int32_t R = r1 - r0;
    const int tiles = (R + kPairTile - 1) / kPairTile;
    k_scan_reduce<<<tiles, 256, 0, st>>>(nv + r0, ne + r0, R, tmp);
    k_scan_tiles<<<1, 1024, 0, st>>>(tmp, tiles, r0 ? voff + r0 : nullptr, r0 ? eoff + r0 : nullptr, ticket);
    k_scan_apply<<<tiles, 256, 0, st>>>(nv + r0, ne + r0, R, tmp, tiles, voff + r0, eoff + r0);
    HGS_CUDA(cudaGetLastError());
}

int64_t scan_tmp_words(int64_t R) { return 2 * ((R + kPairTile - 1) / kPairTile) + 4; }

// Small calls (R <= kSmallScan, one chunk): the offset scan and the batch
// offsets (k_finalize's work) in one CTA, replacing four launches that each
// cost more than their work at this size.
constexpr int kSmallScanPer = 16;
constexpr int kSmallScan = 1024 * kSmallScanPer;
__global__ void __launch_bounds__(1024) k_scan_small(const int32_t* __restrict__ nv, const int32_t* __restrict__ ne,
                                                     int32_t R, int32_t* __restrict__ voff, int32_t* __restrict__ eoff,
                                                     int32_t* __restrict__ ticket, const int64_t* __restrict__ batch_off,
                                                     int32_t k, int32_t* __restrict__ batch_voff,
                                                     int32_t* __restrict__ batch_eoff, int32_t* __restrict__ comp_off) {
    __shared__ int64_t sh[66];
    constexpr int P = kSmallScanPer;
    const int base = threadIdx.x * P;
    int32_t x[P], y[P];
    int64_t a = 0, b = 0;
    // a thread's P entries are 64 contiguous bytes: 16-byte loads and stores
    // unless the thread straddles R (or a buffer is not 16-byte aligned)
    const bool aligned = ((reinterpret_cast<uintptr_t>(nv) | reinterpret_cast<uintptr_t>(ne) |
                           reinterpret_cast<uintptr_t>(voff) | reinterpret_cast<uintptr_t>(eoff)) & 15) == 0;
    const bool full = aligned && base + P <= R;
    if (full) {
#pragma unroll
        for (int i = 0; i < P; i += 4) {
            const int4 u = *reinterpret_cast<const int4*>(nv + base + i);
            const int4 w = *reinterpret_cast<const int4*>(ne + base + i);
            x[i] = u.x; x[i + 1] = u.y; x[i + 2] = u.z; x[i + 3] = u.w;
            y[i] = w.x; y[i + 1] = w.y; y[i + 2] = w.z; y[i + 3] = w.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < P; ++i) {
            x[i] = base + i < R ? nv[base + i] : 0;
            y[i] = base + i < R ? ne[base + i] : 0;
        }
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
        a += x[i];
        b += y[i];
    }
    int64_t ta, tb;
    block_scan_pair(a, b, sh, ta, tb);
#pragma unroll
    for (int i = 0; i < P; ++i) {  // exclusive offsets in place of the counts
        const int32_t cx = x[i], cy = y[i];
        x[i] = (int32_t)a;
        y[i] = (int32_t)b;
        a += cx;
        b += cy;
    }
    if (full) {
#pragma unroll
        for (int i = 0; i < P; i += 4) {
            *reinterpret_cast<int4*>(voff + base + i) = make_int4(x[i], x[i + 1], x[i + 2], x[i + 3]);
            *reinterpret_cast<int4*>(eoff + base + i) = make_int4(y[i], y[i + 1], y[i + 2], y[i + 3]);
        }
    } else {
#pragma unroll
        for (int i = 0; i < P; ++i)
            if (base + i < R) { voff[base + i] = x[i]; eoff[base + i] = y[i]; }
    }
    if (threadIdx.x == 0) {
        voff[R] = (int32_t)ta;
        eoff[R] = (int32_t)tb;
        if (ta > 0x7fffffff || tb > 0x7fffffff) report(ticket, kErrOverflow, 0, 0);
    }
    __syncthreads();  // the offsets above are visible to the whole CTA
    for (int bi = threadIdx.x; bi <= k; bi += blockDim.x) {
        const int64_t f = batch_off[bi];
        batch_voff[bi] = voff[f];
        batch_eoff[bi] = eoff[f];
        if (bi < k && batch_off[bi + 1] == f) comp_off[f + bi] = 0;  // empty batch
    }
}

bool launch_scan_small(const int32_t* nv, const int32_t* ne, int32_t R, int32_t* voff, int32_t* eoff, int32_t* ticket,
                       const int64_t* batch_off, int32_t k, int32_t* bvoff, int32_t* beoff, int32_t* comp_off,
                       cudaStream_t st) {
    if (R > kSmallScan) return false;
    k_scan_small<<<1, 1024, 0, st>>>(nv, ne, R, voff, eoff, ticket, batch_off, k, bvoff, beoff, comp_off);
    HGS_CUDA(cudaGetLastError());
    return true;
}

// ===========================================================================
// K3
// ===========================================================================

constexpr int kPackSmemBatches = 2048;  // batch offsets staged in shared memory up to this k

__global__ void __launch_bounds__(256) k_pack(PackParams p) {
    const int lane = lane_id();
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    constexpr int U = 8;  // independent loads in flight per lane
    // the batch of each root by binary search over batch_off: staged in
    // shared memory (one load per entry per CTA instead of ~log2(k)
    // dependent global loads per root)
    __shared__ int32_t sbo[kPackSmemBatches + 1];
    const bool staged = p.k <= kPackSmemBatches;
    if (staged)
        for (int i = threadIdx.x; i <= p.k; i += blockDim.x) sbo[i] = (int32_t)p.batch_off[i];
    __syncthreads();
    for (int r = p.r0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < p.R; r += nwarps) {
        int b;
        {
            int lo = 0, hi = p.k;  // largest b with batch_off[b] <= r
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if ((staged ? (int64_t)sbo[mid] : p.batch_off[mid]) <= r) lo = mid; else hi = mid - 1;
            }
            b = lo;
        }
        const int f = (int)p.batch_off[b];
        const int64_t vb = p.root_voff[r], eb = p.root_eoff[r];
        const int Vr = p.root_voff[r + 1] - (int32_t)vb;
        const int Er = p.root_eoff[r + 1] - (int32_t)eb;
        const int ecap = p.e_off ? p.e_off[r + 1] - p.e_off[r] : p.e_stride;
        if (Er > ecap) continue;  // slot overflowed in K2 (reported there): the call is re-run
        if (vb + Vr > p.v_cap || eb + Er > p.e_cap) {
            if (lane == 0) report(p.ticket, kErrCapacity, r, -1);
            continue;
        }
        const int32_t loc = (int32_t)vb - p.root_voff[f];
        if (lane == 0) {
            p.roots_local[r] = loc + p.root_rloc[r];
            p.comp_off[r + b] = loc;
            if (r == p.batch_off[b + 1] - 1) p.comp_off[r + 1 + b] = loc + Vr;
        }
        // local_to_global: the sorted set, as K2 left it in the touched slot
        const int32_t* set = p.touched + (size_t)r * p.stride;
        for (int i0 = 0; i0 < Vr; i0 += 32 * U) {
            int32_t u[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int i = i0 + 32 * k + lane;
                u[k] = i < Vr ? set[i] : 0;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int i = i0 + 32 * k + lane;
                if (i < Vr) __stcs(p.l2g + vb + i, u[k]);
            }
        }
        // COO edges (block_diag rebasing) and edge ids
        const int2* ed = p.escratch + (p.e_off ? (size_t)p.e_off[r] : (size_t)r * p.e_stride);
        for (int t0 = 0; t0 < Er; t0 += 32 * U) {
            int2 e[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int t = t0 + 32 * k + lane;
                e[k] = t < Er ? ed[t] : make_int2(0, 0);
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int t = t0 + 32 * k + lane;
                if (t < Er) {
                    __stcs(p.e_row + eb + t, loc + (e[k].x >> 16));
                    __stcs(p.e_col + eb + t, loc + (e[k].x & 0xffff));
                    __stcs(p.e_gid + eb + t, e[k].y);
                }
            }
        }
    }
}

// K3 fused: pack + gather_features in one pass per root (warp per root).
// The root's outputs are contiguous ranges (its vertices [vb, vb+Vr), edges
// [eb, eb+Er)), so a warp writes them with consecutive lanes on consecutive
// 16-byte pieces: local_to_global and the node rows (read from the L2-resident
// feature table by the set it just read), the COO edges / edge ids and the
// edge rows + labels (one 32-byte record per edge when f_e == 2). One read of
// the sets and edge slots, no re-read of l2g / e_gid, one launch.
#ifndef HGS_K3_U
#define HGS_K3_U 4
#endif
__global__ void __launch_bounds__(256) k_pack_gather(PackParams p, const uint4* __restrict__ erec) {
    const int lane = lane_id();
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    constexpr int U = HGS_K3_U;
    const uint64_t pol = l2_keep_policy();
    for (int r = p.r0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < p.R; r += nwarps) {
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
        const int ecap = p.e_off ? p.e_off[r + 1] - p.e_off[r] : p.e_stride;
        if (Er > ecap) continue;  // slot overflowed in K2 (reported there): the call is re-run
        if (vb + Vr > p.v_cap || eb + Er > p.e_cap) {
            if (lane == 0) report(p.ticket, kErrCapacity, r, -1);
            continue;
        }
        const int32_t loc = (int32_t)vb - p.root_voff[f];
        if (lane == 0) {
            p.roots_local[r] = loc + p.root_rloc[r];
            p.comp_off[r + b] = loc;
            if (r == p.batch_off[b + 1] - 1) p.comp_off[r + 1 + b] = loc + Vr;
        }
        const int32_t* set = p.touched + (size_t)r * p.stride;
        // local_to_global
        for (int i0 = 0; i0 < Vr; i0 += 32 * U) {
            int32_t u[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int i = i0 + 32 * k + lane;
                u[k] = i < Vr ? set[i] : 0;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int i = i0 + 32 * k + lane;
                if (i < Vr) __stcs(p.l2g + vb + i, u[k]);
            }
        }
        // node rows: Vr * f_v/2 sixteen-byte pieces (even f_v), else doubles
        if (p.gather && p.f_v > 0) {
            if ((p.f_v & 1) == 0) {
                const int q2 = p.f_v >> 1;
                const int np = Vr * q2;
                const uint4* src = reinterpret_cast<const uint4*>(p.node_feat);
                uint4* dst = reinterpret_cast<uint4*>(p.xv) + vb * q2;
                for (int e0 = 0; e0 < np; e0 += 32 * U) {
                    uint4 x[U];
#pragma unroll
                    for (int k = 0; k < U; ++k) {
                        const int e = e0 + 32 * k + lane;
                        if (e < np) {
                            const int vi = q2 == 1 ? e : p.fv_magic_local ? (int)__umulhi((unsigned)e, p.fv_magic_local)
                                                                          : e / q2;
                            x[k] = __ldg(src + (int64_t)__ldg(set + vi) * q2 + (e - vi * q2));
                        }
                    }
#pragma unroll
                    for (int k = 0; k < U; ++k) {
                        const int e = e0 + 32 * k + lane;
                        if (e < np) __stcs(dst + e, x[k]);
                    }
                }
            } else {
                const int np = Vr * p.f_v;
                for (int e = lane; e < np; e += 32) {
                    const int vi = e / p.f_v;
                    __stcs(p.xv + vb * p.f_v + e, __ldg(p.node_feat + (int64_t)__ldg(set + vi) * p.f_v + (e - vi * p.f_v)));
                }
            }
        }
        // COO edges (block_diag rebasing), edge ids, edge rows + labels
        const int2* ed = p.escratch + (p.e_off ? (size_t)p.e_off[r] : (size_t)r * p.e_stride);
        for (int t0 = 0; t0 < Er; t0 += 32 * U) {
            int2 e[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int t = t0 + 32 * k + lane;
                e[k] = t < Er ? ed[t] : make_int2(0, 0);
            }
            uint4 fr[U];
            uint32_t lb[U];
            if (p.gather && erec) {
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    if (t0 + 32 * k + lane < Er) {
                        fr[k] = ldg_keep(erec + 2 * (int64_t)e[k].y, pol);
                        lb[k] = ldg_keep(&erec[2 * (int64_t)e[k].y + 1].x, pol);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int t = t0 + 32 * k + lane;
                if (t < Er) {
                    __stcs(p.e_row + eb + t, loc + (e[k].x >> 16));
                    __stcs(p.e_col + eb + t, loc + (e[k].x & 0xffff));
                    __stcs(p.e_gid + eb + t, e[k].y);
                    if (p.gather && erec) {
                        __stcs(reinterpret_cast<uint4*>(p.ye) + eb + t, fr[k]);
                        __stcs(p.lab + eb + t, (uint8_t)lb[k]);
                    }
                }
            }
            if (p.gather && !erec) {  // general f_e: feature by feature
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    const int t = t0 + 32 * k + lane;
                    if (t < Er) {
                        const int64_t g = e[k].y;
                        p.lab[eb + t] = __ldg(p.labels + g);
                        for (int c = 0; c < p.f_e; ++c)
                            __stcs(p.ye + (eb + t) * p.f_e + c, __ldg(p.edge_feat + g * p.f_e + c));
                    }
                }
            }
        }
    }
}

void launch_pack_gather(int grid, const PackParams& pp, const uint4* erec, cudaStream_t st) {
    k_pack_gather<<<grid, 256, 0, st>>>(pp, erec);
    HGS_CUDA(cudaGetLastError());
}

// gather_features (sampler.cpp:211-243) over the packed outputs: node rows
// of l2g, edge rows and labels of the edge ids. Flat grid-stride streams.
// Random rows come from L2 (the event's features are L2-resident), where the
// bound is the number of sector requests, not bytes: node rows are read as
// 16-byte pieces by adjacent threads (one warp instruction touches ~11 rows
// and their shared sectors), and edge features + label come as one 32-byte
// record per edge (DevGraph::erec) instead of two requests.
__global__ void __launch_bounds__(256) k_gather_nodes(const double* __restrict__ node_feat, int32_t f_v,
                                                      uint32_t fv_magic, uint32_t fv_err,
                                                      const int32_t* __restrict__ l2g,
                                                      const int32_t* __restrict__ vb, const int32_t* __restrict__ ve,
                                                      int64_t v_cap, const int32_t* __restrict__ ticket,
                                                      double* __restrict__ xv) {
    if (ticket[1] != 0) return;  // failed call (re-run or reported): l2g may be incomplete
    const int64_t V0 = min((int64_t)*vb, v_cap), V = min((int64_t)*ve, v_cap);  // vertices [V0, V)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
// One piece / edge per thread per grid-stride step: all warps sweep the
// outputs together (U = 2, 4, 8 measured 3-35% slower on B200: writes spread
// over U regions at a time).
#ifndef HGS_GATHER_U
#define HGS_GATHER_U 1
#endif
    constexpr int U = HGS_GATHER_U;
    if ((f_v & 1) == 0) {  // rows as f_v/2 16-byte pieces
        const int q2 = f_v >> 1;
        const int64_t n2 = V * q2;
        // i = floor(e * m / 2^32) with m = ceil(2^32 / q2) is exact while
        // e * (q2 * m - 2^32) < 2^32 (fv_err = q2 * m - 2^32); q2 == 1 needs no
        // division at all (m would be 2^32)
        const bool magic = q2 > 1 && n2 < ((int64_t)1 << 32) && (uint64_t)n2 * fv_err < ((uint64_t)1 << 32);
        const uint4* src = reinterpret_cast<const uint4*>(node_feat);
        uint4* dst = reinterpret_cast<uint4*>(xv);
        for (int64_t e0 = V0 * q2 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < n2; e0 += stride * U) {
            uint4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t e = e0 + stride * u;
                if (e < n2) {
                    const int64_t i = q2 == 1 ? e : magic ? (int64_t)__umulhi((unsigned)e, fv_magic) : e / q2;
                    x[u] = __ldg(src + (int64_t)__ldg(l2g + i) * q2 + (e - i * q2));
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (e0 + stride * u < n2) __stcs(dst + e0 + stride * u, x[u]);
        }
    } else {
        const int64_t n = V * f_v;
        for (int64_t e = V0 * f_v + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
            const int64_t i = e / f_v;
            __stcs(xv + e, __ldg(node_feat + (int64_t)l2g[i] * f_v + (e - i * f_v)));
        }
    }
}

// f_e == 2: erec[2g] = the edge's two features, erec[2g+1].x = its label
__global__ void __launch_bounds__(256) k_gather_edges_rec(const uint4* __restrict__ erec,
                                                          const int32_t* __restrict__ e_gid,
                                                          const int32_t* __restrict__ eb_, const int32_t* __restrict__ ee,
                                                          int64_t e_cap, const int32_t* __restrict__ ticket,
                                                          uint4* __restrict__ ye, uint8_t* __restrict__ lab) {
    if (ticket[1] != 0) return;
    const int64_t E0 = min((int64_t)*eb_, e_cap), E = min((int64_t)*ee, e_cap);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    constexpr int U = HGS_GATHER_U;
    const uint64_t pol = l2_keep_policy();
    for (int64_t t0 = E0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < E; t0 += stride * U) {
        int32_t g[U];
#pragma unroll
        for (int u = 0; u < U; ++u) g[u] = t0 + stride * u < E ? __ldcs(e_gid + t0 + stride * u) : 0;
        uint4 f[U];
        uint32_t lb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (t0 + stride * u < E) {
                f[u] = ldg_keep(erec + 2 * (int64_t)g[u], pol);
                lb[u] = ldg_keep(&erec[2 * (int64_t)g[u] + 1].x, pol);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t t = t0 + stride * u;
            if (t < E) {
                __stcs(ye + t, f[u]);
                __stcs(lab + t, (uint8_t)lb[u]);
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_gather_edges(const double* __restrict__ edge_feat, int32_t f_e,
                                                      const uint8_t* __restrict__ labels,
                                                      const int32_t* __restrict__ e_gid,
                                                      const int32_t* __restrict__ eb_, const int32_t* __restrict__ ee,
                                                      int64_t e_cap, const int32_t* __restrict__ ticket,
                                                      double* __restrict__ ye, uint8_t* __restrict__ lab) {
    if (ticket[1] != 0) return;
    const int64_t E0 = min((int64_t)*eb_, e_cap), E = min((int64_t)*ee, e_cap);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = E0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < E; t += stride) {
        const int64_t g = e_gid[t];
        lab[t] = __ldg(labels + g);
        for (int c = 0; c < f_e; ++c) __stcs(ye + t * f_e + c, __ldg(edge_feat + g * f_e + c));
    }
}

__global__ void k_build_erec(const uint4* __restrict__ edge_feat, const uint8_t* __restrict__ labels,
                             int64_t m, uint4* __restrict__ erec) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        erec[2 * e] = edge_feat[e];
        erec[2 * e + 1] = make_uint4(labels[e], 0u, 0u, 0u);
    }
}

void build_edge_records(DevGraph& g, cudaStream_t st) {
    g.erec.release();
    if (g.f_e != 2 || g.nnz == 0) return;
    g.erec.reserve((size_t)2 * g.nnz);
    k_build_erec<<<1184, 256, 0, st>>>(reinterpret_cast<const uint4*>(g.edge_feat.p), g.labels.p, g.nnz,
                                        g.erec.p);
    HGS_CUDA(cudaGetLastError());
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

void launch_extract(int grid, int warps, size_t smem, const ExtractParams& xp, bool packed, cudaStream_t st) {
    if (xp.gscratch) {  // working sets in global scratch: grid * warps slots of warp_bytes
        auto kern = packed ? (xp.a_gid ? k_extract<true, true, true> : k_extract<true, false, true>)
                           : (xp.a_gid ? k_extract<false, true, true> : k_extract<false, false, true>);
        kern<<<grid, 32 * warps, 0, st>>>(xp);
        HGS_CUDA(cudaGetLastError());
        return;
    }
    auto kern = packed ? (xp.a_gid ? k_extract<true, true, false> : k_extract<true, false, false>)
                       : (xp.a_gid ? k_extract<false, true, false> : k_extract<false, false, false>);
    kern<<<grid, 32 * warps, smem, st>>>(xp);  // shared-memory opt-in: extract_blocks_per_sm
    HGS_CUDA(cudaGetLastError());
}

int prepare_kernel(const void* const* kerns, int n, size_t smem, int warps) {
    struct Entry {
        int dev;
        const void* k0;
        size_t smem;
        int warps, per_sm;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    int dev = 0;
    HGS_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    for (const Entry& e : cache)
        if (e.dev == dev && e.k0 == kerns[0] && e.smem == smem && e.warps == warps) return e.per_sm;
    int best = 1 << 30;
    int optin = 0;
    HGS_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    for (int i = 0; i < n; ++i) {
        // the attribute is one value per kernel: opt in to the device maximum
        // (a per-size value would break a later, larger launch served from the cache)
        HGS_CUDA(cudaFuncSetAttribute(kerns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
        int per_sm = 0;
        HGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kerns[i], 32 * warps, smem));
        best = std::min(best, std::max(per_sm, 1));
    }
    cache.push_back({dev, kerns[0], smem, warps, best});
    return best;
}

int extract_blocks_per_sm(size_t smem, int warps, bool packed) {
    const void* kp[4] = {(const void*)k_extract<true, false, false>, (const void*)k_extract<true, true, false>,
                         (const void*)k_extract<false, false, false>, (const void*)k_extract<false, true, false>};
    return prepare_kernel(packed ? kp : kp + 2, 2, smem, warps);
}

__global__ void k_max_i32(const int32_t* __restrict__ x, int32_t n, int32_t* __restrict__ out) {
    int32_t m = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = max(m, x[i]);
    m = __reduce_max_sync(kFull, m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

void launch_max_i32(const int32_t* x, int32_t n, int32_t* out, cudaStream_t st) {
    HGS_CUDA(cudaMemsetAsync(out, 0, sizeof(int32_t), st));
    k_max_i32<<<std::max(1, std::min(148 * 4, (n + 255) / 256)), 256, 0, st>>>(x, n, out);
    HGS_CUDA(cudaGetLastError());
}

void launch_pack(int grid, const PackParams& pp, cudaStream_t st) {
    k_pack<<<grid, 256, 0, st>>>(pp);
    HGS_CUDA(cudaGetLastError());
}

void launch_gather_packed(int blocks, const PackParams& pp, const uint4* erec, const int32_t* vb,
                          const int32_t* ve, const int32_t* eb, const int32_t* ee, cudaStream_t st) {
    const dim3 grid(blocks), block(256);
    if (pp.f_v > 0)
        k_gather_nodes<<<grid, block, 0, st>>>(pp.node_feat, pp.f_v, pp.fv_magic, pp.fv_err, pp.l2g, vb, ve, pp.v_cap,
                                               pp.ticket, pp.xv);
    if (erec)
        k_gather_edges_rec<<<grid, block, 0, st>>>(erec, pp.e_gid, eb, ee, pp.e_cap, pp.ticket,
                                                   reinterpret_cast<uint4*>(pp.ye), pp.lab);
    else
        k_gather_edges<<<grid, block, 0, st>>>(pp.edge_feat, pp.f_e, pp.labels, pp.e_gid, eb, ee, pp.e_cap,
                                               pp.ticket, pp.ye, pp.lab);
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
