// extract_bm.cu — K2, bitmap-directory variant (opt-in, HGS_K2=bm): dedup,
// sort and induced-subgraph extraction of one root per CTA against a bitmap
// rank directory in shared memory. Parity-green; at C2 it runs as fast as the
// default hash-set kernel (0.78 vs 0.76 ms), see DESIGN.md §4.
//
// The directory covers the whole vertex id range: word w describes ids
// 16w .. 16w+15 as 16 membership bits (low half) and the rank of the word's
// first member (high half). A second-level bitmap marks the nonzero words and
// per-block counters hold the members of each run of 32 words.
//
// sorted_vertex_set (sampler.cpp:48-53) without a sort: the CTA sets the
//   touched list's bits (atomicOr; duplicates collapse); the first setter of
//   each word owns it and, after an exclusive scan of the block counters,
//   computes the word's rank prefix and writes its members into the set —
//   the set comes out ascending, and a vertex's local id is its rank.
// induced_subgraph = S·A·Sᵀ (sparse.cpp:177-191) on the directed edge-id A:
//   A's rows are stored padded to 4-entry quads (DevGraph::a_q, as probe
//   words); the set's nonempty rows, in local order, are flattened in quads
//   and scanned in windows of 32 quads (owner row of each quad from a
//   per-pass u16 owner array), one 16-byte load per lane. Each column is
//   tested with ONE 4-byte shared load of its directory word: member bit and
//   local id (rank prefix + popc of the lower member bits) come out of the
//   same word, no collisions, no slow path. The CTA's warps take consecutive
//   windows in rounds; one barrier per round orders their hits, so they land
//   in the root's edge slot in the reference's CSR order.
// Undo: the set's directory words and second-level bits are zeroed after the
//   root, the block counters cleared, so the directory is never cleared in full.
//
// Outputs as the other K2 kernels: sorted set written back over the touched
// slot, (V_r, E_r, local id of the root, S_r) per root, edge slots of
// (local i << 16 | j, edge id).
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace hgs {

namespace {

// Exclusive block scan of two ints over 32*NW threads; ta/tb = totals.
// sc: 2*NW ints, not reused until the caller's next barrier.
template <int NW>
__device__ __forceinline__ void block_scan2(int& a, int& b, int* sc, int& ta, int& tb) {
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const int ia = warp_incl_scan(a), ib = warp_incl_scan(b);
    if (lane == 31) {
        sc[warp] = ia;
        sc[NW + warp] = ib;
    }
    __syncthreads();
    int pa = 0, pb = 0, sa = 0, sb = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const int x = sc[w], y = sc[NW + w];
        if (w < warp) { pa += x; pb += y; }
        sa += x;
        sb += y;
    }
    a = pa + ia - a;
    b = pb + ib - b;
    ta = sa;
    tb = sb;
}

// 32-bit shared-memory load at a shared-window byte address (keeps the
// probe free of generic-address conversion)
__device__ __forceinline__ uint32_t lds32(uint32_t saddr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
    return v;
}

// probe word of a_q (graph.cu): directory byte offset << 8 | shift of the member bit to bit 15
__device__ __forceinline__ uint32_t probe_word(uint32_t c) { return (((c >> 4) << 2) << 8) | (15u - (c & 15u)); }

// member test + local id of vertex c from its directory word: -1 if absent
__device__ __forceinline__ int dir_rank(uint32_t e, uint32_t c) {
    const uint32_t t = e << (15 - (c & 15));  // c's bit -> bit 15, lower members -> bits < 15
    return (t & 0x8000u) ? (int)((e >> 16) + __popc(t & 0x7fffu)) : -1;
}

}  // namespace

#ifndef HGS_K2M_G
#define HGS_K2M_G 2  // quad windows per warp per round (their loads are in flight together)
#endif

// Shared memory per CTA (ExtractParams::warp_bytes; see plan_extract_bm):
//   tab    4 * tab_n               directory words
//   l2     4 * nw2r                nonzero-word bitmap (nw2r = round4(tab_n / 32))
//   set    4 * (set_cap + 4)       sorted set of the root
//   rinfo  8 * row_cap             per nonempty row (first quad - flat quad, local row << 16)
//   qo     4 * max(qcap/2, nw2r)   per-block member counts, then the owner row (u16)
//                                  of each flat quad of the current pass
//   misc   64 ints                 root indices, S_r, root rank, scan scratch, round counts
template <int NW>
__global__ void __launch_bounds__(32 * NW, 24 / NW) k_extract_bm(ExtractParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int NT = 32 * NW;
    constexpr int G = HGS_K2M_G;
    constexpr int KPT = 512 / NT;  // touched entries per thread (T <= 512)
    constexpr int RPT = 512 / NT;  // set members (rows) per thread (U <= 512)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tab_n = p.tab_n, nw2 = tab_n >> 5, nw2r = (nw2 + 3) & ~3;
    const int qcap = p.win_cap;  // flat quads per pass (multiple of 32)
    const int qw = max(qcap / 2, nw2r);
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* l2 = tab + tab_n;
    int32_t* set = reinterpret_cast<int32_t*>(l2 + nw2r);
    int2* rinfo = reinterpret_cast<int2*>(set + p.set_cap + 4);
    int32_t* c2 = reinterpret_cast<int32_t*>(rinfo + p.row_cap);  // per l2 word: members, then prefix
    uint16_t* qown = reinterpret_cast<uint16_t*>(c2);
    int32_t* misc = c2 + qw;
    int* scB = misc + 4;           // 2*NW: block-count scan
    int* scC = misc + 4 + 2 * NW;  // 2*NW: row scan
    int* rc = misc + 4 + 4 * NW;   // 2*NW: per-round hit counts (double-buffered)
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t tab_s = (uint32_t)__cvta_generic_to_shared(tab);
    const uint32_t pad = probe_word((uint32_t)(p.tab_n << 4) - 1u);  // an id >= n: never a member

    for (int i = tid; i < tab_n + nw2r; i += NT) tab[i] = 0u;
    for (int i = tid; i < qw; i += NT) c2[i] = 0;
    if (tid == 0) misc[0] = p.r0 + atomicAdd(p.work, 1);
    int par = 0, rpar = 0;
    for (;;) {
        __syncthreads();  // root index visible; previous root's undo done
        const int r = misc[rpar];
        if (r >= p.R) break;
        int32_t* tl = p.touched + (size_t)r * p.stride;
        const int T = p.tcount[r];
        const uint32_t root = T > 0 ? (uint32_t)tl[0] : 0u;  // touched[0] is the root
        if (tid == 0) {
            misc[rpar ^ 1] = p.r0 + atomicAdd(p.work, 1);  // next root (read after the next top barrier)
            misc[2] = 0;                                   // S_r
        }
        rpar ^= 1;

        // ---- member bits (duplicates collapse), nonzero-word bitmap and
        // member counts per block of 32 words; each word's first setter owns it
        uint32_t own_w[KPT];
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const int i = tid + u * NT;
            own_w[u] = 0xffffffffu;
            if (i < T) {
                const uint32_t v = (uint32_t)tl[i], e = v >> 4, bit = 1u << (v & 15);
                const uint32_t old = atomicOr(&tab[e], bit);
                if (!(old & bit)) atomicAdd(&c2[e >> 5], 1);
                if (old == 0u) {
                    atomicOr(&l2[e >> 5], 1u << (e & 31));
                    own_w[u] = e;
                }
            }
        }
        __syncthreads();

        // ---- exclusive prefix of the block counts
        int U;
        {
            const int per = (nw2 + NT - 1) / NT;
            const int j0 = tid * per, j1 = min(nw2, j0 + per);
            int cnt = 0;
            for (int j = j0; j < j1; ++j) cnt += c2[j];
            int dummy = 0, td;
            block_scan2<NW>(cnt, dummy, scB, U, td);
            for (int j = j0; j < j1; ++j) {
                const int c = c2[j];
                c2[j] = cnt;
                cnt += c;
            }
        }
        __syncthreads();
        // ---- word owners: rank prefix of the word, its members into the sorted set
        uint32_t own_x[KPT];
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const uint32_t e = own_w[u];
            own_x[u] = 0u;
            if (e != 0xffffffffu) {
                int base = c2[e >> 5];
                uint32_t before = l2[e >> 5] & ((1u << (e & 31)) - 1u);  // earlier nonzero words of the block
                while (before) {
                    base += __popc(tab[(e & ~31u) | (uint32_t)(__ffs(before) - 1)]);
                    before &= before - 1;
                }
                const uint32_t x = tab[e];
                const int v0 = (int)(e << 4);
                int k = base;
                for (uint32_t y = x; y; y &= y - 1) set[k++] = v0 + __ffs(y) - 1;
                own_x[u] = ((uint32_t)base << 16) | x;
            }
        }
        __syncthreads();  // every prefix computed from the low halves; set complete

        // ---- rank prefixes into the directory; rows of the set in local order
        int NR, SQ, qi0, fq0;
        int2 ri[RPT];
        const int q = (U + NT - 1) / NT;
        const int i0 = tid * q;
        {
#pragma unroll
            for (int u = 0; u < KPT; ++u)
                if (own_w[u] != 0xffffffffu) tab[own_w[u]] = own_x[u];
#pragma unroll
            for (int u = 0; u < RPT; ++u)
                ri[u] = (u < q && i0 + u < U) ? __ldg(p.a_rq + set[i0 + u]) : make_int2(0, 0);
            int cn = 0, cs = 0, sd = 0;
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                cn += ri[u].y > 0;
                cs += (ri[u].y + 3) >> 2;
                sd += ri[u].y;
            }
            sd = (int)__reduce_add_sync(kFull, (unsigned)sd);
            if (lane == 0) atomicAdd(&misc[2], sd);
            qi0 = cn;
            fq0 = cs;
            block_scan2<NW>(qi0, fq0, scC, NR, SQ);  // its barrier also publishes the directory words
        }
        if (tid == 0) misc[3] = T > 0 ? dir_rank(tab[root >> 4], root) : -1;
        // rows' info + owners of the first pass's quads
        {
            int qi = qi0, fq = fq0;
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                if (ri[u].y > 0) {
                    const int nq = (ri[u].y + 3) >> 2;
                    rinfo[qi] = make_int2(ri[u].x - fq, (i0 + u) << 16);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (k < nq && fq + k < qcap) qown[fq + k] = (uint16_t)qi;
                    for (int f = fq + 4; f < min(fq + nq, qcap); ++f) qown[f] = (uint16_t)qi;
                    ++qi;
                    fq += nq;
                }
            }
        }
        for (int i = tid; i < U; i += NT) tl[i] = set[i];
        __syncthreads();

        // ---- induced subgraph: quad windows in passes of qcap quads, rounds of NW*G windows
        int2* const ed = p.escratch + (p.e_off ? (size_t)p.e_off[r] : (size_t)r * p.e_stride);
        const int cap = p.e_off ? p.e_off[r + 1] - p.e_off[r] : p.e_stride;
        const int nwin = (SQ + 31) >> 5;
        int run = 0;  // hits so far
        for (int qb = 0; qb < SQ; qb += qcap) {
            if (qb > 0) {  // owners of this pass's quads
                __syncthreads();
                int qi = qi0, fq = fq0;
#pragma unroll
                for (int u = 0; u < RPT; ++u) {
                    if (ri[u].y > 0) {
                        const int nq = (ri[u].y + 3) >> 2;
                        for (int f = max(fq, qb); f < min(fq + nq, qb + qcap); ++f) qown[f - qb] = (uint16_t)qi;
                        ++qi;
                        fq += nq;
                    }
                }
                __syncthreads();
            }
            const int wb = qb >> 5, we = min(nwin, (qb + qcap) >> 5);
            for (int rb = wb; rb < we; rb += NW * G) {
                const int g = min(G, (we - rb + NW - 1) / NW);  // windows per warp this round
                const int w0 = rb + warp * g;
                const int flim = min(SQ, qb + qcap);
                int qq[G], rs[G];
                uint4 cq[G];
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    const int f = ((w0 + u) << 5) + lane;
                    const bool ok = u < g && f < flim;
                    const int own = ok ? qown[f - qb] : 0;
                    const int2 rf = rinfo[own];
                    qq[u] = ok ? f + rf.x : -1;
                    rs[u] = rf.y;
                }
#pragma unroll
                for (int u = 0; u < G; ++u) {  // probe words of the lane's quad; invalid lanes see pads
                    cq[u] = make_uint4(pad, pad, pad, pad);
                    if (qq[u] >= 0) cq[u] = __ldg(reinterpret_cast<const uint4*>(p.a_q) + qq[u]);
                }
                // hit predicates, local ids, hits before the lane's in the round
                int jr[G][4];
                bool hit[G][4];
                int pre[G], tot = 0;
                bool any[G];
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    const uint32_t c[4] = {cq[u].x, cq[u].y, cq[u].z, cq[u].w};
                    unsigned bs[4];
#pragma unroll
                    for (int s4 = 0; s4 < 4; ++s4) {
                        const uint32_t e = lds32(tab_s + (c[s4] >> 8));
                        const uint32_t t = __funnelshift_l(0u, e, c[s4]);  // member bit -> bit 15
                        hit[u][s4] = (t & 0x8000u) != 0u;
                        jr[u][s4] = (int)(e >> 16) + __popc(t & 0x7fffu) + rs[u];  // local row << 16 | local column
                        bs[s4] = __ballot_sync(kFull, hit[u][s4]);
                    }
                    pre[u] = tot + __popc(bs[0] & lt) + __popc(bs[1] & lt) + __popc(bs[2] & lt) + __popc(bs[3] & lt);
                    tot += __popc(bs[0]) + __popc(bs[1]) + __popc(bs[2]) + __popc(bs[3]);
                    any[u] = hit[u][0] | hit[u][1] | hit[u][2] | hit[u][3];
                }
                if (lane == 0) rc[par * NW + warp] = tot;
                __syncthreads();
                int base = run;
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    const int x = rc[par * NW + w];
                    if (w < warp) base += x;
                    run += x;
                }
                par ^= 1;
                const bool fast = run <= cap;  // every hit of the round fits the edge slot
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    int4 id = make_int4(0, 0, 0, 0);
                    if (any[u]) id = __ldg(p.a_qid + qq[u]);
                    const int ids[4] = {id.x, id.y, id.z, id.w};
                    int idx = base + pre[u];
                    int2* dst = ed + idx;
                    if (fast) {
#pragma unroll
                        for (int s4 = 0; s4 < 4; ++s4) {
                            if (hit[u][s4]) *dst = make_int2(jr[u][s4], ids[s4]);
                            dst += hit[u][s4];
                        }
                    } else {
#pragma unroll
                        for (int s4 = 0; s4 < 4; ++s4) {
                            if (hit[u][s4] && idx < cap) ed[idx] = make_int2(jr[u][s4], ids[s4]);
                            idx += hit[u][s4];
                        }
                    }
                }
            }
        }
        if (tid == 0) {
            p.root_nv[r] = U;
            p.root_ne[r] = run;
            p.root_rloc[r] = misc[3];
            p.root_scan[r] = misc[2];
            if (run > cap) {
                atomicMax(&p.ticket[4], run);
                report(p.ticket, kErrCapacity, r, run);
            }
        }
        __syncthreads();  // every probe of this root done
        for (int i = tid; i < U; i += NT) {
            const uint32_t e = (uint32_t)set[i] >> 4;
            tab[e] = 0u;
            l2[e >> 5] = 0u;
        }
        for (int i = tid; i < nw2r; i += NT) c2[i] = 0;  // the quad owners reused this space
    }
}

void launch_extract_bm(int grid, int warps, size_t smem, const ExtractParams& xp, cudaStream_t st) {
    if (warps != HGS_K2M_WARPS) fail(HGS_EINVAL, "hgs: k_extract_bm built for another CTA width");
    auto kern = k_extract_bm<HGS_K2M_WARPS>;
    kern<<<grid, 32 * warps, smem, st>>>(xp);
    HGS_CUDA(cudaGetLastError());
}

int extract_bm_prepare(size_t smem, int warps) {
    const void* kerns[1] = {(const void*)k_extract_bm<HGS_K2M_WARPS>};
    return prepare_kernel(kerns, 1, smem, warps);
}

}  // namespace hgs
