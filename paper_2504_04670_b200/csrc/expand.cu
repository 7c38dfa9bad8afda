// expand.cu — K1: stacked-Q frontier expansion, one lane per root
// (k_expand; Philox mode with fanouts <= 8: k_expand_group, a few lanes per
// root deciding a level's rows in parallel).
//
// Restates sample_rows + the expansion loop of bulk_shadow
// (sampler.cpp:64-86, 160-184) per root: level by level, every frontier row v
// with deg_walk(v) > 0 makes one choose(deg, min(s, deg)) decision on the
// root's own stream (PerRootChoiceSource resumes the stream across levels,
// rng.hpp:67-82; the Philox source numbers decisions per root), positions come
// back sorted and map to the walk row's ascending columns, children are
// appended in (parent row, position) order. Rows with no support make no
// decision (sampler.cpp:75). The frontier is a multiset: duplicates are
// expanded again (no dedup until the touched set).
//
// Output: per root a touched list (root, then levels 1..d in BFS order) in a
// fixed-stride scratch slot, its length, per-level row counts and the
// draws/decisions consumed. The (row start, degree) pairs of the rows still to
// expand are cached per lane in shared memory, so the next level issues no
// dependent row_ptr loads.
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"

namespace hgs {




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
        return mod_small(v, (uint32_t)m, rc);
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
        return mod_small(v, (uint32_t)m, rc);
    }
};

// Draws of one decision taken from a buffer the group's lane 0 filled from
// the root's xoshiro stream, in order: without rejections (Rng::bounded,
// rng.cpp:43-50, rejects x < 2^64 mod m, probability < m / 2^64) the draw of
// child t of a root is stream draw t - 1, so a decision's draws start at its
// children's offset. A rejection flags the root for the exact serial path.
struct BufStream {
    const uint64_t* b;
    bool rejected = false;
    __device__ __forceinline__ void begin_decision(uint32_t) {}
    __device__ __forceinline__ uint32_t draw(uint32_t i, uint64_t m, uint64_t rc) {
        const uint64_t x = b[i];
        rejected |= hgs::rejected(x, m, rc);
        return mod_small(x, (uint32_t)m, rc);
    }
};

// choose(n, k) of RandomChoiceSource (rng.cpp:105-119) for k <= KCAP without
// materialising the array: step i swaps slots i and j_i = i + bounded(n - i)
// (j_i >= i), so slot i ends holding the value that sat at j_i just before
// step i — the pre-step value of the latest earlier step a with j_a == j_i,
// or j_i itself — and later steps never touch slot i again. The pre-step
// value of slot i is likewise the pre-step value of the latest a with
// j_a == i, or i. O(k^2) register compares, then a 19-comparator network.
template <int KCAP, class Stream>
__device__ __forceinline__ void choose_small(Stream& rs, uint32_t n, uint32_t k,
                                             const uint64_t* recip, uint32_t (&out)[KCAP]) {
    static_assert(KCAP == 4 || KCAP == 6 || KCAP == 8, "sorting networks exist for 4, 6, 8 keys");
    uint32_t jj[KCAP], pre[KCAP];
#pragma unroll
    for (int i = 0; i < KCAP; ++i) {
        out[i] = 0xffffffffu;
        if (i < (int)k) {
            const uint64_t m = n - (uint32_t)i;
            const uint32_t ji = (uint32_t)i + rs.draw((uint32_t)i, m, recip[m]);
            uint32_t pi = (uint32_t)i, vi = ji;
#pragma unroll
            for (int a = 0; a < i; ++a) {  // ascending: the latest match wins
                pi = (jj[a] == (uint32_t)i) ? pre[a] : pi;
                vi = (jj[a] == ji) ? pre[a] : vi;
            }
            jj[i] = ji;
            pre[i] = pi;
            out[i] = vi;
        }
    }
#define HGS_CX(x, y)                                                   \
    {                                                                  \
        const uint32_t lo = min(out[x], out[y]), hi = max(out[x], out[y]); \
        out[x] = lo;                                                   \
        out[y] = hi;                                                   \
    }
    if constexpr (KCAP == 8) {
        HGS_CX(0, 1) HGS_CX(2, 3) HGS_CX(4, 5) HGS_CX(6, 7) HGS_CX(0, 2) HGS_CX(1, 3) HGS_CX(4, 6)
        HGS_CX(5, 7) HGS_CX(1, 2) HGS_CX(5, 6) HGS_CX(0, 4) HGS_CX(3, 7) HGS_CX(1, 5) HGS_CX(2, 6)
        HGS_CX(1, 4) HGS_CX(3, 6) HGS_CX(2, 4) HGS_CX(3, 5) HGS_CX(3, 4)
    } else if constexpr (KCAP == 6) {  // 12 comparators (checked on all 0/1 inputs)
        HGS_CX(1, 2) HGS_CX(4, 5) HGS_CX(0, 2) HGS_CX(3, 5) HGS_CX(0, 1) HGS_CX(3, 4)
        HGS_CX(2, 5) HGS_CX(0, 3) HGS_CX(1, 4) HGS_CX(2, 4) HGS_CX(1, 3) HGS_CX(2, 3)
    } else {
        HGS_CX(0, 1) HGS_CX(2, 3) HGS_CX(0, 2) HGS_CX(1, 3) HGS_CX(1, 2)
    }
#undef HGS_CX
}

// Generic variant for large fanouts: val holds slots [0, k), (dpos, dval)
// the displaced slots >= k (at most k of them). Local-memory arrays for
// k <= kLocalK, else a per-lane slot of global scratch (ChoiceScratch).
template <bool PHILOX>
__device__ void choose_local(RootStream<PHILOX>& rs, uint32_t n, uint32_t k,
                             const uint64_t* __restrict__ recip, uint32_t* val, uint32_t* dpos, uint32_t* dval) {
    int nd = 0;
    for (uint32_t q = 0; q < k; ++q) val[q] = q;
    for (uint32_t i = 0; i < k; ++i) {
        const uint64_t m = n - i;
        const uint32_t j = i + rs.draw(i, m, recip[m]);
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

// Appends one lane's run of touched entries in order: every aligned 4-entry
// block the run fills completely leaves as one 16-byte store, the ragged
// ends of the run (blocks shared with earlier entries or a neighbouring
// root's slot) as single stores. Cuts K1's L1->L2 write requests ~4x.
struct SeqWriter {
    int32_t* ptr;        // next entry (the touched buffer is 16-byte aligned)
    bool clean;          // the current block began inside this run
    int32_t w0, w1, w2;  // its first three entries
    __device__ __forceinline__ void start(int32_t* at) {
        ptr = at;
        clean = false;
        w0 = w1 = w2 = 0;
    }
    __device__ __forceinline__ void put(int32_t v) {
        const uint32_t j = (uint32_t)(reinterpret_cast<uintptr_t>(ptr) >> 2) & 3u;
        clean |= j == 0;
        if (!clean) *ptr = v;  // head block shared with earlier entries
        else if (j == 3) *reinterpret_cast<int4*>(ptr - 3) = make_int4(w0, w1, w2, v);
        w0 = j == 0 ? v : w0;
        w1 = j == 1 ? v : w1;
        w2 = j == 2 ? v : w2;
        ++ptr;
    }
    __device__ __forceinline__ void finish() const {  // the tail block's entries, singly
        const uint32_t j = (uint32_t)(reinterpret_cast<uintptr_t>(ptr) >> 2) & 3u;
        if (clean && j > 0) {
            int32_t* b = ptr - j;
            b[0] = w0;
            if (j > 1) b[1] = w1;
            if (j > 2) b[2] = w2;
        }
    }
};

// Root seed: the uploaded seed, or Rng::derive(seed, {path..., batch_base +
// bi, pos}) (rng.cpp:76-85) from the call's seed spec.
__device__ __forceinline__ uint64_t root_seed(const ExpandParams& p, int r) {
    if (p.seeds) return p.seeds[r];
    int lo = 0, hi = p.k - 1;  // batch of r: largest bi with batch_off[bi] <= r
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(p.batch_off + mid) <= r) lo = mid; else hi = mid - 1;
    }
    uint64_t path[8];
    for (int i = 0; i < 6; ++i) path[i] = p.spec.path[i];
    const int len = p.spec.path_len;
    path[len] = (uint64_t)(p.spec.batch_base + lo);
    path[len + 1] = (uint64_t)(r - __ldg(p.batch_off + lo));
    return derive_seed(p.spec.seed, path, len + 2);
}

// One root, one lane, in the reference's decision order. `cache` (nullable:
// rows are then re-read from the walk CSR) holds (row start, degree) of the
// rows still to expand, entry i of this lane at cache[i * bd + ti].
template <int KCAP, bool PHILOX, bool LOCAL, bool COMBINE = false>
__device__ void expand_root(const ExpandParams& p, int r, int2* cache, int bd, int ti, const uint64_t* recip) {
    const int32_t root = p.roots32 ? p.roots32[r] : (int32_t)p.roots64[r];
    if (root < 0 || root >= p.n) {
        report(p.ticket, kErrRootRange, r, root);
        p.tcount[r] = 0;
        return;
    }
    const uint64_t seed = root_seed(p, r);
    RootStream<PHILOX> rs;
    rs.init(seed, (!PHILOX && p.state) ? p.state + 4 * (size_t)r : nullptr);
    uint32_t ndec = (PHILOX && p.state) ? (uint32_t)p.state[r] : 0u;
    const uint32_t dec0 = ndec;

    int32_t* out = p.touched + (size_t)r * p.stride;
    int32_t* lc = p.level_counts + (size_t)r * (p.depth + 1);
    out[0] = root;
    lc[0] = 1;
    const bool cached = cache != nullptr;
    {
        if (cached) cache[ti] = __ldg(p.w_ri + root);
    }
    int T = 1, lvl_begin = 0, lvl_end = 1;
    bool bad = false;
    // next expandable row of the level (empty rows make no choose call,
    // sampler.cpp:75); false at the end of the level or on a negative row
    auto next_row = [&](int& idx, int2& row, int level) -> bool {
        while (idx < lvl_end) {
            const int i = idx++;
            if (cached) row = cache[(size_t)i * bd + ti];
            else {
                const int32_t v = out[i];
                row = __ldg(p.w_ri + v);
            }
            if (row.y == 0) continue;
            if (p.neg_row && p.neg_row[out[i]]) {
                report(p.ticket, kErrNegative, r, level);
                bad = true;
                return false;
            }
            return true;
        }
        return false;
    };
    auto decide = [&](const int2& row, uint32_t (&pos)[KCAP]) -> uint32_t {
        const uint32_t deg = (uint32_t)row.y;
        const uint32_t k = min((uint32_t)p.fanout, deg);
        rs.begin_decision(ndec);
        ++ndec;
        choose_small<KCAP>(rs, deg, k, recip, pos);
        return k;
    };
    for (int level = 0; level < p.depth; ++level) {
        const bool in_cache = level + 1 < p.depth && cached;
        const int next_begin = T;
        int idx = lvl_begin;
        int2 row;
        if (LOCAL) {
            while (next_row(idx, row, level)) {
                const uint32_t deg = (uint32_t)row.y;
                const uint32_t k = min((uint32_t)p.fanout, deg);
                rs.begin_decision(ndec);
                ++ndec;
                uint32_t lpos[kLocalK], ldp[kLocalK], ldv[kLocalK];
                uint32_t *pos = lpos, *dp = ldp, *dv = ldv;
                if (k > kLocalK) {
                    pos = p.big + (size_t)(r - p.r0) * 3 * p.big_k;
                    dp = pos + p.big_k;
                    dv = dp + p.big_k;
                }
                choose_local<PHILOX>(rs, deg, k, recip, pos, dp, dv);
                for (uint32_t q = 0; q < k; ++q, ++T) {
                    if (in_cache) cache[(size_t)T * bd + ti].x = row.x + (int32_t)pos[q];
                    else out[T] = row.x + (int32_t)pos[q];
                }
            }
        } else if (in_cache) {
            // park the chosen walk positions in the children's cache slots
            while (next_row(idx, row, level)) {
                uint32_t pos[KCAP];
                const uint32_t k = decide(row, pos);
#pragma unroll
                for (int q = 0; q < KCAP; ++q)
                    if (q < (int)k) cache[(size_t)(T + q) * bd + ti].x = row.x + (int32_t)pos[q];
                T += (int)k;
            }
        } else {
            // child loads of decision i are in flight during decision i+1:
            // two register sets, stores of a set one decision late
            int32_t cA[KCAP], cB[KCAP];
            int TA = 0, kA = 0, TB = 0, kB = 0;
            SeqWriter wr;
            wr.start(out + T);
            auto issue = [&](const int2& rw, int32_t (&c)[KCAP], int& Tc, int& kc) {
                uint32_t pos[KCAP];
                kc = (int)decide(rw, pos);
                Tc = T;
#pragma unroll
                for (int q = 0; q < KCAP; ++q) c[q] = q < kc ? __ldg(p.w_ci + rw.x + pos[q]) : 0;
                T += kc;
            };
            auto flush = [&](const int32_t (&c)[KCAP], int Tc, int& kc) {  // in T order
#pragma unroll
                for (int q = 0; q < KCAP; ++q)
                    if (q < kc) {
                        if constexpr (COMBINE) wr.put(c[q]);
                        else out[Tc + q] = c[q];
                    }
                kc = 0;
            };
            for (;;) {
                if (!next_row(idx, row, level)) break;
                issue(row, cA, TA, kA);
                flush(cB, TB, kB);
                if (!next_row(idx, row, level)) break;
                issue(row, cB, TB, kB);
                flush(cA, TA, kA);
            }
            flush(cA, TA, kA);
            flush(cB, TB, kB);
            if constexpr (COMBINE) wr.finish();
        }
        if (bad) {
            p.tcount[r] = T;
            return;
        }
        if (LOCAL || in_cache) {
            // resolve parked walk positions -> vertices (+ next-level rows)
            constexpr int U = 8;
            SeqWriter wr;
            wr.start(out + next_begin);
            for (int t0 = next_begin; t0 < T; t0 += U) {
                int32_t e[U], c[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (t0 + u < T) e[u] = in_cache ? cache[(size_t)(t0 + u) * bd + ti].x : out[t0 + u];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (t0 + u < T) c[u] = __ldg(p.w_ci + e[u]);
                if (in_cache) {
                    int2 ri[U];
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (t0 + u < T) ri[u] = __ldg(p.w_ri + c[u]);
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (t0 + u < T) cache[(size_t)(t0 + u) * bd + ti] = ri[u];
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (t0 + u < T) {
                        if constexpr (COMBINE) wr.put(c[u]);
                        else out[t0 + u] = c[u];
                    }
            }
            if constexpr (COMBINE) wr.finish();
        }
        lc[level + 1] = T - next_begin;
        lvl_begin = next_begin;
        lvl_end = T;
    }
    p.tcount[r] = T;
    p.draws[r] = rs.draws;
    p.decisions[r] = ndec - dec0;
}

template <int KCAP, bool PHILOX, bool LOCAL, bool COMBINE>
__global__ void __launch_bounds__(128, 4) k_expand(ExpandParams p) {
    extern __shared__ int2 cache[];  // [entry][thread]: (row start, degree), then the recip table
    const int r = p.r0 + blockIdx.x * blockDim.x + threadIdx.x;
    // bounded() reciprocals in shared memory when the table is small
    uint64_t* srecip = reinterpret_cast<uint64_t*>(cache + (size_t)p.cache_entries * blockDim.x);
    const uint64_t* recip = p.recip;
    if (p.recip_smem > 0) {
        for (int i = threadIdx.x; i < p.recip_smem; i += blockDim.x) srecip[i] = p.recip[i];
        __syncthreads();
        recip = srecip;
    }
    if (r >= p.R) return;
    expand_root<KCAP, PHILOX, LOCAL, COMBINE>(p, r, p.cache_entries > 0 ? cache : nullptr, blockDim.x, threadIdx.x, recip);
}

// Decision-parallel K1: the rows of one level are independent once each knows
// its decision number (= nonempty rows before it in the root's order) and its
// children's offset (= the sum of the earlier rows' choice counts). A group of
// GL lanes takes a root and walks each level GL rows at a time; segmented
// scans over the group give both numbers.
//   Philox (PhiloxChoiceSource): draws are counter-based, so
//     every lane evaluates its own decisions.
//   xoshiro (PerRootChoiceSource): the stream is sequential, but a decision's
//     draws are the stream draws at its children's offset (one draw per child
//     unless bounded() rejects, probability < 4e-18 per draw at C2): lane 0 of
//     the group generates the chunk's draws into shared memory, each lane
//     consumes its own. A rejection anywhere sends the root to the serial
//     per-root path (expand_root), which reproduces the reference exactly.
// Same outputs as k_expand.
#ifndef HGS_K1_GL
#define HGS_K1_GL 4
#endif
#ifndef HGS_K1X_GL
#define HGS_K1X_GL 4
#endif
template <bool PHILOX>
constexpr int group_lanes() { return PHILOX ? HGS_K1_GL : HGS_K1X_GL; }

template <int KCAP, bool PHILOX>
__global__ void __launch_bounds__(128) k_expand_group(ExpandParams p) {
    extern __shared__ uint64_t smem_g[];  // recip table, then (xoshiro) per-group draw buffers
    constexpr int GL = group_lanes<PHILOX>();
    const uint64_t* recip = p.recip;
    if (p.recip_smem > 0) {
        for (int i = threadIdx.x; i < p.recip_smem; i += blockDim.x) smem_g[i] = p.recip[i];
        __syncthreads();
        recip = smem_g;
    }
    uint64_t* buf = smem_g + ((p.recip_smem + 1) & ~1) + (size_t)(threadIdx.x / GL) * (GL * KCAP);
    const int gl = threadIdx.x & (GL - 1);
    const unsigned gmask = ((1u << GL) - 1u) << (threadIdx.x & 31 & ~(GL - 1));
    const int r = p.r0 + (int)((blockIdx.x * blockDim.x + threadIdx.x) / GL);
    if (r >= p.R) return;  // whole groups leave together
    if (!PHILOX && p.force_serial > 0 && r % p.force_serial == 0) {  // test hook: the exact fallback
        if (gl == 0) expand_root<KCAP, false, false>(p, r, nullptr, 1, 0, recip);
        return;
    }
    const int32_t root = p.roots32 ? p.roots32[r] : (int32_t)p.roots64[r];
    if (root < 0 || root >= p.n) {
        if (gl == 0) {
            report(p.ticket, kErrRootRange, r, root);
            p.tcount[r] = 0;
        }
        return;
    }
    const uint64_t seed = root_seed(p, r);
    RootStream<true> rs;  // Philox
    Xoshiro256 xs{};      // xoshiro: lane 0's copy is the stream
    if constexpr (PHILOX) rs.init(seed, nullptr);
    else if (gl == 0) {
        if (p.state) {
            const uint64_t* st = p.state + 4 * (size_t)r;
            xs.a = st[0]; xs.b = st[1]; xs.c = st[2]; xs.d = st[3];
        } else xs.seed(seed);
    }
    const uint32_t dec0 = (PHILOX && p.state) ? (uint32_t)p.state[r] : 0u;
    uint32_t dec = dec0;
    int32_t* out = p.touched + (size_t)r * p.stride;
    int32_t* lc = p.level_counts + (size_t)r * (p.depth + 1);
    if (gl == 0) {
        out[0] = root;
        lc[0] = 1;
    }
    __syncwarp(gmask);
    int T = 1, lvl_begin = 0, lvl_end = 1;
    bool bad = false, rej = false;
    for (int level = 0; level < p.depth && !bad; ++level) {
        const int next_begin = T;
        // rows of the level's next chunk are loaded one chunk ahead
        auto load_row = [&](int i, int32_t& v, int32_t& b, int32_t& deg) {
            v = 0; b = 0; deg = 0;
            if (i < lvl_end) {
                v = out[i];
                const int2 ri = __ldg(p.w_ri + v);
                b = ri.x;
                deg = ri.y;
            }
        };
        int32_t nv_, nb_, nd_;
        load_row(lvl_begin + gl, nv_, nb_, nd_);
        for (int i0 = lvl_begin; i0 < lvl_end; i0 += GL) {
            const int i = i0 + gl;
            const int32_t v = nv_, b = nb_, deg = nd_;
            if (i0 + GL < lvl_end) load_row(i0 + GL + gl, nv_, nb_, nd_);
            if (i < lvl_end && deg > 0 && p.neg_row && p.neg_row[v]) {
                report(p.ticket, kErrNegative, r, level);
                bad = true;
            }
            if (__any_sync(gmask, bad)) { bad = true; break; }
            const uint32_t k = deg > 0 ? min((uint32_t)p.fanout, (uint32_t)deg) : 0u;
            // group-exclusive prefix of (nonempty rows, choices)
            uint32_t pn = deg > 0 ? 1u : 0u, pk = k;
#pragma unroll
            for (int o = 1; o < GL; o <<= 1) {
                const uint32_t xn = __shfl_up_sync(gmask, pn, o, GL), xk = __shfl_up_sync(gmask, pk, o, GL);
                if (gl >= o) { pn += xn; pk += xk; }
            }
            const uint32_t tn = __shfl_sync(gmask, pn, GL - 1, GL), tk = __shfl_sync(gmask, pk, GL - 1, GL);
            if constexpr (!PHILOX) {
                if (gl == 0)
                    for (uint32_t t = 0; t < tk; ++t) buf[t] = xs.next();
                __syncwarp(gmask);
            }
            if (k > 0) {
                uint32_t pos[KCAP];
                if constexpr (PHILOX) {
                    rs.begin_decision(dec + pn - 1);
                    choose_small<KCAP>(rs, (uint32_t)deg, k, recip, pos);
                } else {
                    BufStream bs{buf + (pk - k)};
                    choose_small<KCAP>(bs, (uint32_t)deg, k, recip, pos);
                    rej |= bs.rejected;
                }
                int32_t c[KCAP];
#pragma unroll
                for (int q = 0; q < KCAP; ++q) c[q] = q < (int)k ? __ldg(p.w_ci + b + pos[q]) : 0;
                int32_t* dst = out + T + (pk - k);
#pragma unroll
                for (int q = 0; q < KCAP; ++q)
                    if (q < (int)k) dst[q] = c[q];
            }
            if constexpr (!PHILOX) __syncwarp(gmask);  // the buffer is refilled by the next chunk
            T += (int)tk;
            dec += tn;
        }
        __syncwarp(gmask);  // this level's children are visible to the whole group
        if (!PHILOX && __any_sync(gmask, rej)) break;
        if (gl == 0 && !bad) lc[level + 1] = T - next_begin;
        lvl_begin = next_begin;
        lvl_end = T;
    }
    if (!PHILOX && __any_sync(gmask, rej)) {  // a rejected draw shifted the stream: redo exactly
        if (gl == 0) expand_root<KCAP, false, false>(p, r, nullptr, 1, 0, recip);
        return;
    }
    uint32_t dr = PHILOX ? rs.draws : 0u;
#pragma unroll
    for (int o = GL / 2; o > 0; o >>= 1) dr += __shfl_down_sync(gmask, dr, o, GL);
    if (gl == 0) {
        p.tcount[r] = T;
        p.draws[r] = PHILOX ? dr : (uint32_t)(T - 1);  // xoshiro: one draw per child
        p.decisions[r] = dec - dec0;
    }
}

// sample_rows (sampler.cpp:64-86): one lane per choice stream, deciding that
// stream's nonempty rows in row order (begin_root(row_streams[r]) then
// choose(|support|, min(s, |support|)), positions -> the row's columns).
template <bool PHILOX>
__global__ void __launch_bounds__(128) k_sample_rows(RowsParams p) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= p.groups) return;
    const int64_t stream = p.sid[g];
    RootStream<PHILOX> rs;
    rs.init(p.seeds[stream], (!PHILOX && p.state) ? p.state + 4 * stream : nullptr);
    uint32_t ndec = (PHILOX && p.state) ? (uint32_t)p.state[stream] : 0u;
    const uint32_t dec0 = ndec;
    for (int64_t i = p.sptr[g]; i < p.sptr[g + 1]; ++i) {
        const int64_t r = p.srows[i];
        const int64_t b = p.row_ptr[r];
        const uint32_t deg = (uint32_t)(p.row_ptr[r + 1] - b);
        const uint32_t k = min((uint32_t)p.fanout, deg);
        rs.begin_decision(ndec);
        ++ndec;
        int64_t* dst = p.out_cols + p.out_off[r];
        if (k <= 8) {
            uint32_t pos[8];
            choose_small<8>(rs, deg, k, p.recip, pos);
            for (uint32_t q = 0; q < k; ++q) dst[q] = p.col[b + pos[q]];
        } else {
            uint32_t lpos[kLocalK], ldp[kLocalK], ldv[kLocalK];
            uint32_t *pos = lpos, *dp = ldp, *dv = ldv;
            if (k > kLocalK) {
                pos = p.big + (size_t)g * 3 * p.big_k;
                dp = pos + p.big_k;
                dv = dp + p.big_k;
            }
            choose_local<PHILOX>(rs, deg, k, p.recip, pos, dp, dv);
            for (uint32_t q = 0; q < k; ++q) dst[q] = p.col[b + pos[q]];
        }
    }
    p.draws[g] = rs.draws;
    p.decisions[g] = ndec - dec0;
}

void launch_sample_rows(const RowsParams& p, bool philox, cudaStream_t st) {
    const unsigned grid = (unsigned)((p.groups + 127) / 128);
    if (grid == 0) return;
    if (philox) k_sample_rows<true><<<grid, 128, 0, st>>>(p);
    else k_sample_rows<false><<<grid, 128, 0, st>>>(p);
    HGS_CUDA(cudaGetLastError());
}

// HGS_K1_GROUPX=1: the decision-parallel kernel for xoshiro streams (see
// HGS_K1X_GROUP); read per call.
static bool getenv_flag_k1_groupx() { return getenv("HGS_K1_GROUPX") != nullptr; }

template <int KCAP, bool PH, bool LOCAL>
static void launch_expand_t(int threads, size_t smem, const ExpandParams& ep, cudaStream_t st) {
    auto kern = ep.combine ? k_expand<KCAP, PH, LOCAL, true> : k_expand<KCAP, PH, LOCAL, false>;
    if (smem > 48 * 1024)
        HGS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = (unsigned)((ep.R - ep.r0 + threads - 1) / threads);
    kern<<<grid, threads, smem, st>>>(ep);
    HGS_CUDA(cudaGetLastError());
}

template <int KCAP, bool PHILOX>
static void launch_expand_group(const ExpandParams& ep, cudaStream_t st) {
    constexpr int GL = group_lanes<PHILOX>();
    const size_t smem = (size_t)((ep.recip_smem + 1) & ~1) * sizeof(uint64_t) +
                        (PHILOX ? 0 : (size_t)128 * KCAP * sizeof(uint64_t));
    auto kern = k_expand_group<KCAP, PHILOX>;
    if (smem > 48 * 1024)
        HGS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t threads = (int64_t)(ep.R - ep.r0) * GL;
    kern<<<(unsigned)((threads + 127) / 128), 128, smem, st>>>(ep);
    HGS_CUDA(cudaGetLastError());
}

#ifndef HGS_K1_GROUP
#define HGS_K1_GROUP 1
#endif
// The decision-parallel xoshiro path is opt-in (HGS_K1X_GROUP=1 at build
// time or HGS_K1_GROUPX=1 at run time): measured on B200 at C2 it takes
// 0.175 ms (4-lane groups; 2: 0.182, 8: 0.243) against 0.166 for one lane
// per root — lane 0's serial stream generation idles the other lanes.
#ifndef HGS_K1X_GROUP
#define HGS_K1X_GROUP 0
#endif

void launch_expand(int threads, size_t smem, int64_t kmax, const ExpandParams& ep, bool philox,
                   cudaStream_t st) {
    // decision-parallel paths for choices of <= 8 (the register network);
    // the xoshiro one needs no uploaded resume state beyond the 4 words
    const bool group = philox ? HGS_K1_GROUP : (HGS_K1X_GROUP || getenv_flag_k1_groupx());
    if (group && kmax <= 8 && ep.R > ep.r0) {
        if (philox) {
            if (kmax > 6) launch_expand_group<8, true>(ep, st);
            else if (kmax > 4) launch_expand_group<6, true>(ep, st);
            else launch_expand_group<4, true>(ep, st);
        } else {
            if (kmax > 6) launch_expand_group<8, false>(ep, st);
            else if (kmax > 4) launch_expand_group<6, false>(ep, st);
            else launch_expand_group<4, false>(ep, st);
        }
        return;
    }
    // register fast path for k <= 8, sized to the call's largest choice
    if (kmax > 8) {
        if (philox) launch_expand_t<8, true, true>(threads, smem, ep, st);
        else launch_expand_t<8, false, true>(threads, smem, ep, st);
    } else if (kmax > 6) {
        if (philox) launch_expand_t<8, true, false>(threads, smem, ep, st);
        else launch_expand_t<8, false, false>(threads, smem, ep, st);
    } else if (kmax > 4) {
        if (philox) launch_expand_t<6, true, false>(threads, smem, ep, st);
        else launch_expand_t<6, false, false>(threads, smem, ep, st);
    } else {
        if (philox) launch_expand_t<4, true, false>(threads, smem, ep, st);
        else launch_expand_t<4, false, false>(threads, smem, ep, st);
    }
}


}  // namespace hgs
