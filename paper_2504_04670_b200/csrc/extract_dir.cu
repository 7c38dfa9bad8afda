// extract_dir.cu — K2, directory variant (opt-in, HGS_K2_DIR=1): dedup, sort and
// induced-subgraph extraction of one root per warp, with the membership
// probe as ONE 4-byte shared-memory load.
//
// sorted_vertex_set (sampler.cpp:48-53): the touched list (duplicates
//   included) is counting-sorted on (v - lo) >> shift buckets over the root's
//   own id range, ranked within its bucket (equal keys by position) and then
//   compacted to the sorted unique set: no hash-set dedup pass.
// The probe structure is a rank directory over the same order: NB buckets
//   b = (v - lo) >> sh (sh = bits(hi - lo) - log2 NB), entry of a nonempty
//   bucket = (low bits of its first key) << 16 | more << 15 | rank of that key.
//   Keys of one bucket are consecutive in sorted order, so a probe of column c
//   reads dir[b(c)] and hits iff the stored low bits equal c's; only a probe
//   that lands in a bucket holding >= 2 keys (more = 1) and misses its first
//   key walks the sorted set (rare: NB ~ 8 x the set size).
// induced_subgraph = S·A·Sᵀ (sparse.cpp:177-191) on the directed edge-id A:
//   the set's nonempty A rows, in local order, are flattened and scanned in
//   32-entry windows (row owner of each lane = per-window cursor + popc of a
//   row-start bitmask), each column probed in the directory; hits are
//   ballot-compacted into the root's edge slot in the reference's CSR order
//   (rows ascending, columns ascending within a row).
//
// Same outputs as k_extract (extract.cu): sorted set written back over the
// touched slot, (V_r, E_r, local id of the root, S_r) per root, edge slots of
// (local i << 16 | j, edge id).
#include <cuda_runtime.h>

#include <type_traits>

#include "kernels.cuh"

namespace hgs {

namespace {

constexpr uint32_t kDirEmpty = 0xffff7fffu;  // low field 0xffff never matches a low <= 0x7fff

}  // namespace

#ifndef HGS_K2D_MINB
#define HGS_K2D_MINB 6  // CTAs of 4 warps per SM the register budget is sized for (4: 0.975 ms, 5: 0.829, 6: 0.774 at C2)
#endif
#ifndef HGS_K2D_G
#define HGS_K2D_G 6  // windows whose column loads are in flight together
#endif

// Per-warp shared memory (bytes; set_cap >= the longest touched list):
//   dir    4 << lnb            sort counters, then the rank directory
//   keys   4 * (set_cap + 4)   touched keys, then the sorted unique set (+ sentinel)
//   tmp    4 * (set_cap + 36)  bucketed keys, then row starts
//   rinfo  8 * set_cap         sorted keys with duplicates, then per nonempty row
//                              (A pos - flat pos, local row << 16)
//   winfo  8 * win_cap         per window of a pass: (row-start mask, cursor)
template <bool HAS_GID>
__global__ void __launch_bounds__(128, HGS_K2D_MINB) k_extract_dir(ExtractParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = lane_id();
    const int warp = threadIdx.x >> 5;
    unsigned char* q = smem_raw + (size_t)warp * p.warp_bytes;
    const int NB = 1 << p.lnb;
    uint32_t* dir = reinterpret_cast<uint32_t*>(q); q += 4 * (size_t)NB;
    int32_t* keys = reinterpret_cast<int32_t*>(q); q += 4 * (size_t)(p.set_cap + 4);
    int32_t* tmp = reinterpret_cast<int32_t*>(q); q += 4 * (size_t)(p.set_cap + 36);
    int2* rinfo = reinterpret_cast<int2*>(q); q += 8 * (size_t)p.set_cap;
    uint2* winfo = reinterpret_cast<uint2*>(q);
    int32_t* sd = reinterpret_cast<int32_t*>(rinfo);
    int32_t* rstart = tmp;
    uint32_t* cnt = dir;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned le = (2u << lane) - 1u;
    constexpr int CH = 4;  // 32-key chunks of loads in flight

    auto next_root = [&]() -> int {
        int r = 0;
        if (lane == 0) r = p.r0 + atomicAdd(p.work, 1);
        return __shfl_sync(kFull, r, 0);
    };
    for (int r = next_root(); r < p.R; r = next_root()) {
        int32_t* tl = p.touched + (size_t)r * p.stride;
        const int T = p.tcount[r];

        // ---- touched keys (duplicates included) into shared memory, id range
        uint32_t lo = 0xffffffffu, hi = 0u;
        for (int b0 = 0; b0 < T; b0 += CH * 32) {
            int32_t v[CH];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int i = b0 + c * 32 + lane;
                v[c] = i < T ? __ldcs(tl + i) : 0;
            }
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int i = b0 + c * 32 + lane;
                if (i < T) {
                    keys[i] = v[c];
                    lo = min(lo, (uint32_t)v[c]);
                    hi = max(hi, (uint32_t)v[c]);
                }
            }
        }
        lo = __reduce_min_sync(kFull, lo);
        hi = __reduce_max_sync(kFull, hi);
        __syncwarp();
        const int32_t root = T > 0 ? keys[0] : -1;  // touched[0] is the root
        const int span_bits = 32 - __clz(hi - lo);  // bits of (hi - lo); 0 for one key

        // ---- counting sort on order-preserving buckets (v - lo) >> shs, ~2T of them
        const int lg = min(p.cnt_lg, max(5, 32 - __clz(max(2 * T - 1, 1))));
        const int shs = max(0, span_bits - lg);
        const int lp = lg - 5;  // counters per lane = 1 << lp
        const uint32_t pm = (1u << lp) - 1u;
        // counter of bucket b at ((b & pm) << 5) | (b >> lp): lane l's
        // consecutive buckets are one bank apart (conflict-free scan)
        auto cidx = [&](uint32_t b) -> int { return (int)(((b & pm) << 5) | (b >> lp)); };
        for (int i = lane; i < (32 << lp); i += 32) cnt[i] = 0u;
        __syncwarp();
        for (int i = lane; i < T; i += 32) atomicAdd(&cnt[cidx(((uint32_t)keys[i] - lo) >> shs)], 1u);
        __syncwarp();
        {
            int s = 0;
            for (int e = 0; e <= (int)pm; ++e) s += (int)cnt[(e << 5) | lane];
            int run = warp_incl_scan(s) - s;
            for (int e = 0; e <= (int)pm; ++e) {
                const int c = (int)cnt[(e << 5) | lane];
                cnt[(e << 5) | lane] = (uint32_t)run;
                run += c;
            }
        }
        __syncwarp();
        for (int i = lane; i < T; i += 32) {  // place (counter becomes the bucket end)
            const uint32_t v = (uint32_t)keys[i];
            tmp[atomicAdd(&cnt[cidx((v - lo) >> shs)], 1u)] = (int32_t)v;
        }
        __syncwarp();
        // position with duplicates = bucket start + smaller keys of the bucket
        // + equal keys placed before it
        for (int i = lane; i < T; i += 32) {
            const uint32_t v = (uint32_t)tmp[i];
            const uint32_t b = (v - lo) >> shs;
            const int e = (int)cnt[cidx(b)];
            const int s = b ? (int)cnt[cidx(b - 1)] : 0;
            int pos = s;
            for (int j = s; j < e; ++j) {
                const uint32_t u = (uint32_t)tmp[j];
                pos += (u < v) || (u == v && j < i);
            }
            sd[pos] = (int32_t)v;
        }
        __syncwarp();
        // ---- unique: sorted set into keys[0, U), sentinel after it
        int U = 0;
        for (int b0 = 0; b0 < T; b0 += 32) {
            const int i = b0 + lane;
            const int32_t v = i < T ? sd[i] : 0;
            int32_t pv = __shfl_up_sync(kFull, v, 1);
            if (lane == 0) pv = b0 > 0 ? sd[b0 - 1] : ~v;
            const bool fresh = i < T && pv != v;
            const unsigned fb = __ballot_sync(kFull, fresh);
            if (fresh) keys[U + __popc(fb & lt)] = v;
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
        if (lane == 0) keys[U] = 0x7fffffff;  // slow-path walks stop here
        // ---- rank directory over the sorted set
        const int sh = max(0, span_bits - p.lnb);
        const uint32_t lowm = (1u << sh) - 1u;
        for (int i = lane; i < NB / 4; i += 32)
            reinterpret_cast<uint4*>(dir)[i] = make_uint4(kDirEmpty, kDirEmpty, kDirEmpty, kDirEmpty);
        __syncwarp();
        for (int b0 = 0; b0 < U; b0 += 32) {
            const int i = b0 + lane;
            const uint32_t d = i < U ? (uint32_t)keys[i] - lo : 0u;
            const uint32_t b = d >> sh;
            uint32_t pb = __shfl_up_sync(kFull, b, 1), nbk = __shfl_down_sync(kFull, b, 1);
            if (lane == 0 && b0 > 0) pb = ((uint32_t)keys[b0 - 1] - lo) >> sh;
            if (lane == 31 && i + 1 < U) nbk = ((uint32_t)keys[i + 1] - lo) >> sh;
            const bool first = i < U && (i == 0 || pb != b);
            const bool more = i + 1 < U && nbk == b;
            if (first) dir[b] = ((d & lowm) << 16) | (more ? 0x8000u : 0u) | (uint32_t)i;
        }
        __syncwarp();
        // Probe, branch-free: local id of column c or -1; *slow is set (and
        // -1 returned) when c misses the first key of a bucket holding >= 2
        // keys, which walk() then resolves (callers test the warp once).
        auto probe = [&](uint32_t c, bool& slow) -> int {
            const uint32_t d = c - lo;
            const uint32_t b = d >> sh;
            const uint32_t e = b < (uint32_t)NB ? dir[b] : kDirEmpty;
            const uint32_t x = e ^ ((d & lowm) << 16);
            const bool hit = x < 0x10000u;
            slow = !hit && (e & 0x8000u);
            return hit ? (int)(x & 0x7fffu) : -1;
        };
        auto walk = [&](uint32_t c) -> int {  // >= 2 keys in c's bucket, c not its first
            const uint32_t e = dir[(c - lo) >> sh];
            for (int k = (int)(e & 0x7fffu) + 1;; ++k) {
                const uint32_t u = (uint32_t)keys[k];
                if (u >= c) return u == c ? k : -1;
            }
        };
        auto find = [&](uint32_t c) -> int {
            bool slow;
            const int j = probe(c, slow);
            return slow ? walk(c) : j;
        };

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
        __syncwarp();
        const int nwin = (S + 31) >> 5;

        // ---- induced subgraph: scan the flattened rows in 32-entry windows
        int2* const ed = p.escratch + (p.e_off ? (size_t)p.e_off[r] : (size_t)r * p.e_stride);
        int2* const ed_end = p.e_off ? p.escratch + p.e_off[r + 1] : ed + p.e_stride;
        int2* edc = ed;  // next free edge slot
        auto emit = [&](int j, int rowsh, int kk, auto chk) {
            const unsigned hb = ballot_nonneg(j);
            int2* dst = edc + __popc(hb & lt);
            if (j >= 0 && (!decltype(chk)::value || dst < ed_end))
                *dst = make_int2(rowsh | j, HAS_GID ? __ldg(p.a_gid + kk) : kk);
            edc += __popc(hb);
        };
        constexpr int G = HGS_K2D_G;
        int wb = 0;
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
        auto consume = [&](const int (&rs)[G], const int (&kk)[G], const uint32_t (&v)[G]) {
            int j[G];
            bool sl[G], any = false;
#pragma unroll
            for (int u = 0; u < G; ++u) {
                j[u] = probe(v[u], sl[u]);
                any |= sl[u];
            }
            if (__any_sync(kFull, any)) {
#pragma unroll
                for (int u = 0; u < G; ++u)
                    if (sl[u]) j[u] = walk(v[u]);
            }
            if (edc + 32 * G <= ed_end) {
#pragma unroll
                for (int u = 0; u < G; ++u) emit(j[u], rs[u], kk[u], std::false_type{});
            } else {
#pragma unroll
                for (int u = 0; u < G; ++u) emit(j[u], rs[u], kk[u], std::true_type{});
            }
        };
        int carry = 0;  // row starts before the pass
        for (; wb < nwin; wb += p.win_cap) {
            const int we = min(nwin, wb + p.win_cap);
            const int nw = we - wb;
            for (int w = lane; w < nw; w += 32) winfo[w].x = 0u;
            __syncwarp();
            for (int qi = lane; qi < NR; qi += 32) {
                const int s0 = rstart[qi];
                const int w0 = (s0 >> 5) - wb;
                if (w0 >= 0 && w0 < nw) atomicOr(&winfo[w0].x, 1u << (s0 & 31));
            }
            __syncwarp();
            // cursor of window w = (row starts before it) - 1: lane l owns a
            // contiguous run of the pass's windows
            {
                const int per = (nw + 31) >> 5;
                const int w0 = lane * per, w1 = min(nw, w0 + per);
                int c = 0;
                for (int w = w0; w < w1; ++w) c += __popc(winfo[w].x);
                const int incl = warp_incl_scan(c);
                int run = carry + incl - c - 1;
                carry += __shfl_sync(kFull, incl, 31);
                for (int w = w0; w < w1; ++w) {
                    const uint32_t m = winfo[w].x;
                    winfo[w].y = (uint32_t)run;
                    run += __popc(m);
                }
            }
            __syncwarp();
            const int wfull = min(we, S >> 5);  // windows of the pass with 32 entries
            const int nfg = max(0, wfull - wb) / G;
            for (int gi = 0; gi < nfg; ++gi) {
                int rsA[G], kkA[G];
                uint32_t vA[G];
                fetch(wb + gi * G, rsA, kkA, vA);
                consume(rsA, kkA, vA);
            }
            for (int w = wb + nfg * G; w < we; ++w) {  // < G trailing windows, the last one possibly partial
                const int base = w << 5;
                const uint2 wi = winfo[w - wb];
                const int own = min((int)wi.y + __popc(wi.x & le), NR - 1);
                const int2 ri = rinfo[max(own, 0)];
                const int kk = base + lane < S ? base + lane + ri.x : -1;
                const int j = kk >= 0 ? find((uint32_t)__ldg(p.a_ci + kk)) : -1;
                emit(j, ri.y, kk, std::true_type{});
            }
            __syncwarp();
        }
        const int count = (int)(edc - ed);
        const int cap = (int)(ed_end - ed);
        const int rloc = T > 0 ? find((uint32_t)root) : -1;
        if (lane == 0) {
            p.root_nv[r] = U;
            p.root_ne[r] = count;
            p.root_rloc[r] = rloc;
            p.root_scan[r] = S;
            if (count > cap) {
                atomicMax(&p.ticket[4], count);
                report(p.ticket, kErrCapacity, r, count);
            }
        }
        __syncwarp();
    }
}

void launch_extract_dir(int grid, int warps, size_t smem, const ExtractParams& xp, cudaStream_t st) {
    auto kern = xp.a_gid ? k_extract_dir<true> : k_extract_dir<false>;
    kern<<<grid, 32 * warps, smem, st>>>(xp);
    HGS_CUDA(cudaGetLastError());
}

int extract_dir_prepare(size_t smem, int warps) {
    // shared-memory opt-in + occupancy query, once per (device, size, warps)
    const void* kerns[2] = {(const void*)k_extract_dir<false>, (const void*)k_extract_dir<true>};
    return prepare_kernel(kerns, 2, smem, warps);
}

}  // namespace hgs
