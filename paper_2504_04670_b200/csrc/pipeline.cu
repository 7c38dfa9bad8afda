// pipeline.cu — host orchestration of one bulk_shadow call on the device:
// K1 expand → K2 extract → offset scan → K3 pack/gather → batch offsets, all
// on the sample handle's stream with no host synchronisation in between.
// Capacity guesses (edge slots per root, output edge capacity) are checked
// on the device; on overflow the call is re-run once with exact sizes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace hgs {

namespace {

int64_t tree_bound(int64_t kmax, int64_t upto) {
    // 1 + kmax + ... + kmax^upto, saturating at 2^40
    int64_t total = 0, term = 1;
    const int64_t cap = (int64_t)1 << 40;
    for (int64_t l = 0; l <= upto; ++l) {
        total = std::min(cap, total + term);
        term = std::min(cap, term * std::max<int64_t>(kmax, 1));
    }
    return total;
}

struct CallPlan {
    int64_t kmax, max_t, cache_entries;
    int expand_threads;
    size_t expand_smem;
    int32_t recip_smem;
    int32_t n_buckets, set_cap, row_cap, win_cap, warp_bytes, rank_bits, packed;
    int32_t k2_warps;  // warps per K2 CTA (0: not planned yet)
    bool k2_gmem;      // K2 working sets in global scratch (sets beyond shared memory)
    bool k2_dir;       // K2 = k_extract_dir (rank directory); else the hash-set k_extract
    bool k2_bm;        // K2 = k_extract_bm (one root per CTA, bitmap rank directory)
    int32_t tab_n;     // k_extract_bm: directory words (16 vertex ids each)
    int32_t lnb;       // k_extract_dir: log2 of the directory buckets
};

int ceil_log2(int64_t x) {
    int l = 0;
    while (((int64_t)1 << l) < x) ++l;
    return l;
}

// k_extract_dir per-warp shared memory for touched lists of up to `bound`
// entries (duplicates included): directory of NB = 2^lnb buckets (~8 per
// key, at least the sort's 2*set_cap counters, and fine enough that the low
// bits of a key within its bucket fit 15 bits: n <= NB << 15), keys, bucketed
// keys / row starts, sorted keys / row info, and one pass of window info.
// False when the fast path does not apply (very large sets or id ranges):
// the hash-set kernel then serves the call.
// Opt-in (HGS_K2_DIR=1): measured on B200 at C2 it is no faster than the
// hash-set kernel (0.774 vs 0.752 ms at 24 warps per SM; K2 is bound by its
// per-warp latency chain and occupancy, not by the probe), see DESIGN.md.
bool plan_extract_dir(CallPlan& c, int64_t bound, int64_t n, int32_t max_out_deg) {
    const char* sel = getenv("HGS_K2");
    if (!getenv("HGS_K2_DIR") && !(sel && strcmp(sel, "dir") == 0)) return false;
    if (bound > 2048) return false;
    (void)max_out_deg;
    c.set_cap = (int32_t)std::max<int64_t>(16, (bound + 3) / 4 * 4);
    c.row_cap = c.set_cap;
    c.win_cap = std::max(16, c.set_cap / 2);  // windows per pass (larger rows: several passes)
    const int cnt_lg = 31 - __builtin_clz((unsigned)(2 * c.row_cap));
    int lnb = std::max(cnt_lg, ceil_log2(6 * (int64_t)c.set_cap));
#ifdef HGS_K2D_LNB
    lnb = std::max(cnt_lg, HGS_K2D_LNB);
#endif
    if (const char* e = getenv("HGS_K2D_LNB")) lnb = std::max(cnt_lg, atoi(e));
    lnb = std::max(lnb, ceil_log2(std::max<int64_t>(n, 1)) - 15);
    if (lnb > 14) return false;
    c.lnb = lnb;
    const size_t bytes = 4 * ((size_t)1 << lnb) + 4 * (size_t)(c.set_cap + 4) + 4 * (size_t)(c.set_cap + 36) +
                         8 * (size_t)c.set_cap + 8 * (size_t)c.win_cap;
    c.warp_bytes = (int32_t)((bytes + 15) / 16 * 16);
    const size_t max_block = 232448;
    c.k2_warps = 0;
    for (int w : {4, 2, 1})
        if ((size_t)w * c.warp_bytes <= max_block) { c.k2_warps = w; break; }
    if (c.k2_warps == 0) return false;
    c.k2_dir = true;
    c.k2_gmem = false;
    return true;
}

// K2 per-warp shared memory for sets of up to `bound` vertices: hash set +
// keys + row starts + row info. Entries pack (vertex << rank_bits | rank)
// into 32 bits when vertex ids leave room, else (vertex, rank) pairs. The
// hash (4-slot buckets, any count) takes what is left of a 6-CTA-per-SM
// budget when that still gives >= 2.5 slots per possible key; otherwise 3
// slots per key. Big sets run with 2 or 1 warps per CTA (up to ~227 KB of
// shared memory per warp). False when even one warp cannot hold a set.
bool plan_extract(CallPlan& c, int64_t bound, int64_t n) {
    c.rank_bits = 1;
    while (((int64_t)1 << c.rank_bits) < bound) ++c.rank_bits;
    c.packed = (n + 1 < ((int64_t)1 << (32 - c.rank_bits))) ? 1 : 0;
    c.set_cap = (int32_t)std::max<int64_t>(16, (bound + 3) / 4 * 4);  // >= 16: bucket counters need 32 ints
    c.row_cap = c.set_cap;
    c.win_cap = c.set_cap / 2;  // windows per pass: (u32 mask, u32 cursor) each, in the set array
    const size_t rest = 4 * (size_t)c.set_cap + 4 * (size_t)(c.row_cap + 36) + 8 * (size_t)c.row_cap;
    const size_t bucket_bytes = c.packed ? 16 : 32;
#ifndef HGS_K2_MINB
#define HGS_K2_MINB 6  // K2 CTAs per SM (extract.cu's launch bound)
#endif
    const size_t budget = (233472 / HGS_K2_MINB - 1024) / 4 / 16 * 16;  // per warp, HGS_K2_MINB CTAs of 4 warps
    int64_t nb = budget > rest ? (int64_t)((budget - rest) / bucket_bytes) : 0;
    if (const char* e = getenv("HGS_HASH_SLOTS_PER_KEY")) nb = (atoi(e) * bound + 3) / 4;
    if (4 * nb * 2 < 5 * bound) nb = (3 * bound + 3) / 4;
    const size_t max_block = 232448;  // opt-in dynamic shared memory per CTA (227 KB)
    c.k2_warps = 0;
    for (int spk_min : {3, 2}) {  // very large sets: fall back to 2 slots per key
        if (spk_min == 2) nb = (2 * bound + 3) / 4;
        c.n_buckets = (int32_t)std::max<int64_t>(nb, 2);
        size_t bytes = bucket_bytes * (size_t)c.n_buckets + rest;
        bytes = (bytes + 15) / 16 * 16;
        c.warp_bytes = (int32_t)bytes;
        for (int w : {4, 2, 1})
            if ((size_t)w * bytes <= max_block) { c.k2_warps = w; break; }
        if (c.k2_warps > 0) break;
    }
    c.k2_gmem = false;
    c.k2_dir = false;
    return c.k2_warps > 0;
}

// k_extract_bm (extract_bm.cu): one root per CTA of HGS_K2M_WARPS warps; the
// CTA's shared memory holds the bitmap rank directory of the whole id range
// (one 32-bit word per 16 vertex ids: 16 membership bits + the rank of the
// word's first member) plus the set, row and window arrays of one root.
// Applies to touched lists of <= 512 entries on graphs whose directory leaves
// room for >= 3 CTAs per SM (n up to ~290k ids).
// Opt-in (HGS_K2=bm): measured on B200 at C2 it runs in 0.78 ms against the
// hash-set kernel's 0.76 ms (fewer shared wavefronts, but as many warp
// instructions per root: see DESIGN.md §4).
bool plan_extract_bm(CallPlan& c, int64_t bound, int64_t n) {
    const char* sel = getenv("HGS_K2");
    if (!sel || strcmp(sel, "bm") != 0) return false;
    if (bound > 512 || n <= 0) return false;
    c.tab_n = (int32_t)((n + 1 + 16 * 32 - 1) / (16 * 32) * 32);  // covers the pad id n
    c.set_cap = (int32_t)((bound + 3) / 4 * 4);
    c.row_cap = c.set_cap;
    const int64_t nw2r = (c.tab_n / 32 + 3) & ~3;
    c.win_cap = 1024;  // flat quads per pass (the quad-owner array)
    const int64_t qw = std::max<int64_t>(c.win_cap / 2, nw2r);
    const size_t bytes = 4 * (size_t)c.tab_n + 4 * (size_t)nw2r + 4 * (size_t)(c.set_cap + 4) +
                         8 * (size_t)c.row_cap + 4 * (size_t)qw + 256;
    if (bytes > 72 * 1024) return false;
    c.warp_bytes = (int32_t)((bytes + 127) / 128 * 128);  // per CTA
    c.k2_warps = HGS_K2M_WARPS;
    c.k2_bm = true;
    c.k2_dir = false;
    c.k2_gmem = false;
    return true;
}

bool plan_k2(CallPlan& c, int64_t bound, int64_t n, int32_t max_out_deg) {
    c.k2_bm = false;
    return plan_extract_bm(c, bound, n) || plan_extract_dir(c, bound, n, max_out_deg) || plan_extract(c, bound, n);
}

CallPlan plan_call(int32_t walk_max_deg, int32_t a_max_deg, int64_t n, int64_t depth, int64_t fanout) {
    CallPlan c{};
    c.kmax = std::min<int64_t>(fanout, walk_max_deg);
    if (c.kmax > ((int64_t)1 << 24))
        fail(HGS_ERANGE, "hgs: min(fanout, max degree) > 2^24 is not supported by this build");
    c.max_t = tree_bound(c.kmax, depth);
    // The tree bound only sizes K1's touched slots; the limit that matters is
    // a root's distinct vertex count (16-bit local ids in K2's edge slots),
    // checked by K2 itself (kErrSetRange).
    if (c.max_t > ((int64_t)1 << 30))
        fail(HGS_ERANGE, "hgs: per-root tree bound " + std::to_string(c.max_t) + " is too large; reduce depth/fanout");
    c.cache_entries = tree_bound(c.kmax, depth - 1);
    c.recip_smem = walk_max_deg + 1 <= 4096 ? walk_max_deg + 1 : 0;
    const size_t rbytes = (size_t)c.recip_smem * sizeof(uint64_t);
    // 64-lane blocks: K1's time per SM is linear in its lanes, and finer
    // blocks even out the SMs (C2: 1024 blocks = 6.9 per SM; 128-lane blocks
    // leave 68 SMs with 4 and 80 with 3: 0.173 vs 0.164 ms)
    c.expand_threads = 64;
    c.expand_smem = (size_t)c.cache_entries * c.expand_threads * sizeof(int2) + rbytes;
    if (c.expand_smem > 96 * 1024) {  // deep / wide trees: rows re-read from the walk CSR
        c.cache_entries = 0;
        c.expand_smem = rbytes;
    }
    if (c.max_t > kMaxSet || !plan_k2(c, c.max_t, n, a_max_deg)) c.k2_warps = 0;  // decided after K1 (see sample_enqueue)
    return c;
}

// K3 as pack + two flat gathers (default) or one fused per-root pack+gather
// kernel (HGS_K3_FUSED=1; B200, C2: 0.464 ms against 0.384 — the flat
// kernels sweep the outputs with all warps together, the per-root warps
// write ~9.5k scattered streams)
bool k3_fused() {
    const char* e = getenv("HGS_K3_FUSED");
    return e && e[0] == '1';
}

int sm_count(int device) {
    int n = 0;
    HGS_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    return n;
}

}  // namespace

void sample_enqueue(hgs_sample* s, const hgs_config& cfg, const CallInputs& in, bool rerun) {
    // The graphs of the call: the handle's graph, or one per event of a
    // multi-event call (hgs_sample_run_multi), all on the handle's device.
    const bool multi = in.n_events > 0;
    std::vector<DevGraph*> gs;
    if (multi)
        for (int32_t e = 0; e < in.n_events; ++e) gs.push_back(&in.events[e]->g);
    else
        gs.push_back(&s->graph->g);
    DevGraph& g = *gs[0];
    HGS_CUDA(cudaSetDevice(g.device));
    const bool seq_walk = (cfg.flags & HGS_FLAG_SEQ_WALK) != 0;
    auto walk_of = [&](DevGraph& h) -> DevCsr& {
        return cfg.symmetrize ? h.walk_sym : (seq_walk ? h.full_pattern() : h.a);
    };
    int32_t walk_max = 0, a_max = 0;
    int64_t n_max = 0;
    for (DevGraph* h : gs) {
        if (cfg.symmetrize) graph_build_walk_sym(*h);
        graph_ensure_recip(*h, walk_of(*h).max_deg);
        {
            std::lock_guard<std::recursive_mutex> lk(h->lazy_mu);
            csr_ensure_row_info(walk_of(*h), h->stream);
        }
        if (cfg.gather && !h->has_features) fail(HGS_EINVAL, "gather_features: no features attached to the graph");
        walk_max = std::max(walk_max, walk_of(*h).max_deg);
        a_max = std::max(a_max, h->a.max_deg);
        n_max = std::max<int64_t>(n_max, h->n_rows);
    }
    if (multi)  // K1 stages recip_smem entries of every event's table
        for (DevGraph* h : gs) graph_ensure_recip(*h, walk_max);
    const DevCsr& walk = walk_of(g);
    CallPlan c = plan_call(walk_max, a_max, n_max, cfg.depth, cfg.fanout);
    const int64_t R = in.R, k = in.k;
    if (R * c.max_t >= ((int64_t)1 << 40)) fail(HGS_ERANGE, "hgs: too many roots for one call");
    cudaStream_t st = s->stream;

    s->R = R; s->k = k; s->depth = cfg.depth; s->fanout = cfg.fanout;
    s->gathered = cfg.gather; s->symmetrize = cfg.symmetrize; s->rng = cfg.rng;
    if (!rerun) {
        s->launches = 0;
        s->reruns = 0;
    }
    s->touched_stride = c.max_t;
    const size_t R1 = (size_t)R + 1;
    s->touched.reserve((size_t)std::max<int64_t>(R, 1) * c.max_t);
    s->tcount.reserve(R1);
    s->level_counts.reserve(R1 * (cfg.depth + 1));
    s->draws.reserve(R1);
    s->decisions.reserve(R1);
    s->root_nv.reserve(R1);
    s->root_ne.reserve(R1);
    s->root_rloc.reserve(R1);
    s->root_scan.reserve(R1);
    if (!(rerun && s->exact_slots)) s->escratch.reserve(R1 * s->e_stride);
    s->scan_tmp.reserve(scan_tmp_words(R));
    s->ticket.reserve(8);
    s->root_voff.reserve(R1);
    s->root_eoff.reserve(R1);
    s->roots_local.reserve(R1);
    s->comp_off.reserve((size_t)(R + k) + 1);
    s->batch_voff.reserve((size_t)k + 1);
    s->batch_eoff.reserve((size_t)k + 1);
    // initial output capacity: the tree bound, capped per root (a loose bound
    // would reserve far more than any call produces; a call that needs more
    // grows the capacity once and re-runs, see sample_finish)
    const size_t vneed = (size_t)std::max<int64_t>(1, R * std::min<int64_t>(c.max_t, 4096));
    if (s->v_cap < vneed) s->v_cap = vneed;
    if (s->e_cap == 0) s->e_cap = s->v_cap * 2;
    s->l2g.reserve(s->v_cap);
    s->e_row.reserve(s->e_cap);
    s->e_col.reserve(s->e_cap);
    s->e_gid.reserve(s->e_cap);
    if (cfg.gather) {
        s->xv.reserve(s->v_cap * (size_t)std::max(1, g.f_v));
        s->ye.reserve(s->e_cap * (size_t)std::max(1, g.f_e));
        s->lab.reserve(s->e_cap);
    }
    HGS_CUDA(cudaMemsetAsync(s->ticket.p, 0, 8 * sizeof(int32_t), st));
    if (R == 0) {
        HGS_CUDA(cudaMemsetAsync(s->root_voff.p, 0, sizeof(int32_t), st));
        HGS_CUDA(cudaMemsetAsync(s->root_eoff.p, 0, sizeof(int32_t), st));
    }
    if (!s->ev[0]) for (auto& e : s->ev) HGS_CUDA(cudaEventCreate(&e));
    s->profiled = cfg.profile != 0;
    if (s->profiled) HGS_CUDA(cudaEventRecord(s->ev[0], st));

    ExpandParams ep{};
    ep.w_ri = walk.ri.p; ep.w_ci = walk.ci.p; ep.recip = g.recip.p;
    // The write combiner saves L1->L2 write requests, the bound of large
    // calls (C2: K1 0.148 vs 0.160 ms), but lengthens each lane's chain, the
    // bound of small ones (C1, 16k roots: 0.023 vs 0.020 ms)
    ep.combine = in.R >= 32 * 1024 ? 1 : 0;
    if (const char* e = getenv("HGS_K1_COMBINE")) ep.combine = atoi(e);
    ep.neg_row = (!cfg.symmetrize && !seq_walk && g.has_neg) ? g.neg_row.p : nullptr;
    ep.roots32 = in.roots32; ep.roots64 = in.roots64; ep.seeds = in.seeds; ep.state = in.state;
    ep.batch_off = in.batch_off; ep.k = (int32_t)k;
    if (in.spec) ep.spec = *in.spec;
    ep.depth = (int32_t)cfg.depth;
    ep.fanout = (int32_t)std::min<int64_t>(cfg.fanout, 1 << 30);
    ep.n = (int32_t)g.n_rows; ep.stride = c.max_t; ep.cache_entries = (int32_t)c.cache_entries;
    ep.recip_smem = c.recip_smem;
    ep.touched = s->touched.p; ep.tcount = s->tcount.p; ep.level_counts = s->level_counts.p;
    ep.draws = s->draws.p; ep.decisions = s->decisions.p; ep.ticket = s->ticket.p;
    if (const char* e = getenv("HGS_K1_FORCE_SERIAL")) ep.force_serial = atoi(e);  // test hook

    ExtractParams xp{};
    xp.a_rp = g.a.rp.p; xp.a_ci = g.a.ci.p; xp.a_gid = g.has_gid ? g.a_gid.p : nullptr; xp.a_ri = g.a_ri.p;
    xp.touched = s->touched.p; xp.tcount = s->tcount.p; xp.stride = c.max_t;
    xp.root_nv = s->root_nv.p; xp.root_ne = s->root_ne.p; xp.root_rloc = s->root_rloc.p;
    xp.root_scan = s->root_scan.p; xp.escratch = s->escratch.p; xp.e_stride = s->e_stride;
    xp.e_off = rerun && s->exact_slots ? s->eoff_exact.p : nullptr;
    xp.ck_iters = 64;  // cuckoo chain bound of the hash kernel's scan tables
    if (const char* e = getenv("HGS_K2_CK_ITERS")) xp.ck_iters = atoi(e);  // test hook: 0 forces the fallback
    xp.ticket = s->ticket.p;
    auto set_layout = [&]() {
        xp.n_buckets = c.n_buckets; xp.set_cap = c.set_cap; xp.row_cap = c.row_cap;
        xp.win_cap = c.win_cap; xp.warp_bytes = c.warp_bytes; xp.rank_bits = c.rank_bits;
        xp.cnt_lg = 31 - __builtin_clz((unsigned)(2 * c.row_cap));
        xp.lnb = c.lnb;
        xp.tab_n = c.tab_n;
    };

    PackParams pp{};
    pp.touched = s->touched.p; pp.stride = c.max_t; pp.root_voff = s->root_voff.p;
    pp.root_eoff = s->root_eoff.p; pp.root_rloc = s->root_rloc.p; pp.escratch = s->escratch.p;
    pp.e_stride = s->e_stride; pp.e_off = xp.e_off; pp.batch_off = in.batch_off; pp.k = (int32_t)k;
    pp.l2g = s->l2g.p; pp.roots_local = s->roots_local.p; pp.comp_off = s->comp_off.p;
    pp.e_row = s->e_row.p; pp.e_col = s->e_col.p; pp.e_gid = s->e_gid.p;
    pp.xv = s->xv.p; pp.ye = s->ye.p; pp.lab = s->lab.p;
    pp.node_feat = g.node_feat.p; pp.edge_feat = g.edge_feat.p; pp.labels = g.labels.p;
    pp.f_v = g.f_v; pp.f_e = g.f_e; pp.gather = cfg.gather;
    const uint32_t q2 = (uint32_t)std::max(1, g.f_v / 2);
    {
        const uint64_t m = ((((uint64_t)1 << 32) + q2 - 1) / q2);  // 2^32 for q2 == 1: unused then
        pp.fv_magic = q2 > 1 ? (uint32_t)m : 0u;
        pp.fv_err = q2 > 1 ? (uint32_t)(q2 * m - ((uint64_t)1 << 32)) : 0u;
        // per-root piece indices stay below (kMaxSet + 1) * q2
        pp.fv_magic_local = (q2 > 1 && (uint64_t)(kMaxSet + 1) * q2 * pp.fv_err < ((uint64_t)1 << 32)) ? (uint32_t)m : 0u;
    }
    pp.v_cap = (int64_t)s->v_cap; pp.e_cap = (int64_t)s->e_cap; pp.ticket = s->ticket.p;
    pp.set_cap = c.set_cap;
    const uint4* erec = g.erec.p;
    // point the kernels at one event's graph (multi-event calls rebind per event)
    auto bind = [&](DevGraph& h) {
        const DevCsr& w = walk_of(h);
        ep.w_ri = w.ri.p; ep.w_ci = w.ci.p; ep.recip = h.recip.p;
        ep.neg_row = (!cfg.symmetrize && !seq_walk && h.has_neg) ? h.neg_row.p : nullptr;
        ep.n = (int32_t)h.n_rows;
        xp.a_rp = h.a.rp.p; xp.a_ci = h.a.ci.p; xp.a_gid = h.has_gid ? h.a_gid.p : nullptr; xp.a_ri = h.a_ri.p;
        pp.node_feat = h.node_feat.p; pp.edge_feat = h.edge_feat.p; pp.labels = h.labels.p;
        erec = h.erec.p;
    };
    // the event of each root range: one range per event (multi) or the whole call
    std::vector<int64_t> ev_r0{0, R};
    if (multi) ev_r0.assign(in.ev_r0, in.ev_r0 + in.n_events + 1);

    // Roots go through the stages in chunks: K1 -> K2 -> offset scan of chunk
    // c on the handle's stream, K3 of chunk c on a higher-priority side
    // stream, so the memory-bound packing of chunk c runs on the SMs next to
    // the latency-bound extraction of chunk c+1. A profiled call runs as one
    // serial chunk so each stage can be timed on its own.
    // Off by default: measured on B200 at C2, packing next to extraction
    // slows both (they contend for the LSU pipe), see DESIGN.md.
    int64_t chunk = R;
    if (!s->profiled && !multi)
        if (const char* e = getenv("HGS_CHUNK_ROOTS")) chunk = std::max<int64_t>(32, atoll(e));
    const int64_t nchunks = multi ? in.n_events : (R > 0 ? (R + chunk - 1) / chunk : 0);
    const bool split = !multi && nchunks > 1;  // side-stream packing (opt-in experiment)
    cudaStream_t pst = st;
    if (split) {
        if (!s->aux) {
            int lo = 0, hi = 0;
            HGS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            HGS_CUDA(cudaStreamCreateWithPriority(&s->aux, cudaStreamNonBlocking, hi));
        }
        while ((int64_t)s->chunk_ev.size() < nchunks + 1) {
            cudaEvent_t e;
            HGS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            s->chunk_ev.push_back(e);
        }
        pst = s->aux;
        HGS_CUDA(cudaEventRecord(s->chunk_ev[nchunks], st));  // aux waits for this call's inputs
        HGS_CUDA(cudaStreamWaitEvent(pst, s->chunk_ev[nchunks], 0));
    }
    ep.big = nullptr; ep.big_k = 0;
    if (c.kmax > (int64_t)kLocalK && R > 0) {  // wide choices: a global scratch slot per root
        ep.big_k = (int32_t)c.kmax;
        s->kbig.reserve((size_t)R * 3 * (size_t)c.kmax);
        ep.big = s->kbig.p;
    }
    // K1 over all roots at once (one lane per root, its length is one root's
    // chain); a multi-event call runs it per event, each on its own walk
    for (size_t e = 0; e + 1 < ev_r0.size(); ++e) {
        if (ev_r0[e + 1] <= ev_r0[e]) continue;
        bind(*gs[multi ? e : 0]);
        ep.r0 = (int32_t)ev_r0[e]; ep.R = (int32_t)ev_r0[e + 1];
        launch_expand(c.expand_threads, c.expand_smem, c.kmax, ep, cfg.rng == HGS_RNG_PHILOX, st);
        ++s->launches;
    }
    if (c.k2_warps == 0 && R > 0) {
        // the tree bound is too loose for K2's shared memory: size K2 for the
        // largest touched list K1 actually produced (one host round trip)
        launch_max_i32(s->tcount.p, (int32_t)R, s->ticket.p + 6, st);
        int32_t tmax = 0;
        HGS_CUDA(cudaMemcpyAsync(&tmax, s->ticket.p + 6, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HGS_CUDA(cudaStreamSynchronize(st));
        if (!plan_k2(c, std::max<int32_t>(tmax, 1), n_max, a_max)) {
            // beyond one warp's shared memory: K2 keeps its working sets in
            // a global scratch slot per warp (3 hash slots per key)
            plan_extract(c, 1, n_max);  // rank bits / packing for the real bound below
            c.rank_bits = 1;
            while (((int64_t)1 << c.rank_bits) < tmax) ++c.rank_bits;
            c.packed = (n_max + 1 < ((int64_t)1 << (32 - c.rank_bits))) ? 1 : 0;
            c.set_cap = (tmax + 3) / 4 * 4;
            c.row_cap = c.set_cap;
            c.win_cap = c.set_cap / 2;
            c.n_buckets = (3 * tmax + 3) / 4;
            const size_t bytes = (c.packed ? 16 : 32) * (size_t)c.n_buckets + 4 * (size_t)c.set_cap +
                                 4 * (size_t)(c.row_cap + 36) + 8 * (size_t)c.row_cap;
            c.warp_bytes = (int32_t)((bytes + 15) / 16 * 16);
            c.k2_warps = 4;
            c.k2_gmem = true;
        }
    }
    if (c.k2_warps == 0) plan_k2(c, 1, n_max, a_max);  // R == 0: nothing to extract
    set_layout();
    const size_t xsmem = c.k2_gmem ? 0 : c.k2_bm ? (size_t)c.warp_bytes : (size_t)c.k2_warps * c.warp_bytes;
    const int xper_sm = c.k2_gmem ? 2
                        : c.k2_bm ? extract_bm_prepare(xsmem, c.k2_warps)
                        : c.k2_dir ? extract_dir_prepare(xsmem, c.k2_warps)
                                   : extract_blocks_per_sm(xsmem, c.k2_warps, c.packed != 0);
    xp.gscratch = nullptr;
    if (c.k2_bm)
        for (DevGraph* h : gs) graph_ensure_quads(*h);
    if (c.k2_gmem) {
        const size_t slots = (size_t)xper_sm * sm_count(g.device) * c.k2_warps;
        s->k2g.reserve(slots * (size_t)c.warp_bytes);
        xp.gscratch = s->k2g.p;
    }
    s->frontier_kept = (cfg.flags & HGS_FLAG_KEEP_FRONTIERS) != 0;
    if (s->frontier_kept && R > 0) {  // K2 sorts the touched lists in place
        s->frontier.reserve((size_t)R * c.max_t);
        HGS_CUDA(cudaMemcpyAsync(s->frontier.p, s->touched.p, sizeof(int32_t) * (size_t)R * c.max_t,
                                 cudaMemcpyDeviceToDevice, st));
    }
    if (s->profiled) HGS_CUDA(cudaEventRecord(s->ev[1], st));
    bool small_scan = false;  // scan + batch offsets done by one small launch
    for (int64_t ci = 0; ci < nchunks; ++ci) {
        const int32_t r0 = (int32_t)(multi ? ev_r0[ci] : ci * chunk);
        const int32_t r1 = (int32_t)(multi ? ev_r0[ci + 1] : std::min<int64_t>(R, r0 + chunk));
        if (r1 <= r0) continue;  // an event without roots
        DevGraph& h = *gs[multi ? ci : 0];
        bind(h);
        if (c.k2_bm) {
            xp.a_q = h.a_q.p;
            xp.a_qid = h.a_qid.p;
            xp.a_rq = h.a_rq.p;
        }
        const int64_t Rc = r1 - r0;
        xp.r0 = r0; xp.R = r1;
        const int64_t per_cta = c.k2_bm ? 1 : c.k2_warps;  // roots in flight per CTA
        const int64_t xgrid = (split && !c.k2_gmem)
                                  ? (Rc + per_cta - 1) / per_cta
                                  : std::min<int64_t>((int64_t)xper_sm * sm_count(g.device), (Rc + per_cta - 1) / per_cta);
        xp.work = s->ticket.p + 5;
        HGS_CUDA(cudaMemsetAsync(xp.work, 0, sizeof(int32_t), st));
        if (c.k2_bm) launch_extract_bm((int)std::max<int64_t>(xgrid, 1), c.k2_warps, xsmem, xp, st);
        else if (c.k2_dir) launch_extract_dir((int)std::max<int64_t>(xgrid, 1), c.k2_warps, xsmem, xp, st);
        else launch_extract((int)std::max<int64_t>(xgrid, 1), c.k2_warps, xsmem, xp, c.packed != 0, st);
        ++s->launches;
        if (s->profiled) HGS_CUDA(cudaEventRecord(s->ev[2], st));
        if (nchunks == 1 && launch_scan_small(s->root_nv.p, s->root_ne.p, (int32_t)R, s->root_voff.p, s->root_eoff.p,
                                        s->ticket.p, in.batch_off, (int32_t)k, s->batch_voff.p, s->batch_eoff.p,
                                        s->comp_off.p, st)) {
            small_scan = true;
            s->launches += 1;
        } else {
            launch_scan(s->root_nv.p, s->root_ne.p, r0, r1, s->scan_tmp.p, s->root_voff.p, s->root_eoff.p,
                        s->ticket.p, st);
            s->launches += 3;
        }
        if (s->profiled) HGS_CUDA(cudaEventRecord(s->ev[3], st));
        if (split) {
            HGS_CUDA(cudaEventRecord(s->chunk_ev[ci], st));
            HGS_CUDA(cudaStreamWaitEvent(pst, s->chunk_ev[ci], 0));
        }
        pp.r0 = r0; pp.R = r1;
        const int64_t pgrid = split ? (Rc + 7) / 8 : std::min<int64_t>((int64_t)sm_count(g.device) * 8, (Rc + 7) / 8);
        if (k3_fused()) {  // pack + gathers in one pass per root
            launch_pack_gather((int)std::max<int64_t>(pgrid, 1), pp, erec, pst);
            ++s->launches;
        } else {
        launch_pack((int)std::max<int64_t>(pgrid, 1), pp, pst);
        ++s->launches;
        }
        if (cfg.gather && !k3_fused()) {  // this chunk's vertices / edges
#ifndef HGS_GATHER_BPSM
#define HGS_GATHER_BPSM 8
#endif
            const int gblocks = split ? std::max<int64_t>(1, std::min<int64_t>(sm_count(g.device) * HGS_GATHER_BPSM, Rc * 4))
                                      : sm_count(g.device) * HGS_GATHER_BPSM;
            launch_gather_packed(gblocks, pp, erec, s->root_voff.p + r0, s->root_voff.p + r1,
                                 s->root_eoff.p + r0, s->root_eoff.p + r1, pst);
            s->launches += 2;
        }
    }
    if (s->profiled) HGS_CUDA(cudaEventRecord(s->ev[4], st));
    if (R == 0 && s->profiled)
        for (int i = 2; i <= 3; ++i) HGS_CUDA(cudaEventRecord(s->ev[i], st));
    if (!small_scan) {
        launch_finalize(in.batch_off, (int32_t)k, (int32_t)R, s->root_voff.p, s->root_eoff.p, s->batch_voff.p,
                        s->batch_eoff.p, s->comp_off.p, pst);
        ++s->launches;
    }
    if (split) {  // join: the handle's stream sees the whole call
        HGS_CUDA(cudaEventRecord(s->chunk_ev[nchunks], pst));
        HGS_CUDA(cudaStreamWaitEvent(st, s->chunk_ev[nchunks], 0));
    }
    if (s->profiled) HGS_CUDA(cudaEventRecord(s->ev[5], st));
    if (!s->h_state) HGS_CUDA(cudaMallocHost(&s->h_state, 16 * sizeof(int32_t)));
    HGS_CUDA(cudaMemcpyAsync(s->h_state, s->ticket.p, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaMemcpyAsync(s->h_state + 8, s->batch_voff.p + k, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HGS_CUDA(cudaMemcpyAsync(s->h_state + 9, s->batch_eoff.p + k, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    s->pending = true;
}

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
    if (code == kErrSetRange)
        fail(HGS_ERANGE, "hgs: root ordinal " + std::to_string(s->h_state[2]) + " induces a subgraph of " +
                             std::to_string(s->h_state[3]) + " vertices; this build's per-root limit is " +
                             std::to_string(kMaxSet) + " (reduce depth/fanout)");
    if (code == kErrOverflow)
        fail(HGS_ERANGE, "hgs: more than 2^31-1 sampled vertices/edges in one call; split the call");
    s->V = s->h_state[8];
    s->E = s->h_state[9];
    if (code == kErrCapacity) {
        // An edge slot or the output capacity was too small: grow to the
        // observed need and run the call again (inputs are still resident).
        const int32_t need = s->h_state[4];
        s->exact_slots = false;
        if (need > s->e_stride) {
            // Grow the uniform per-root slot while that stays within a few
            // times the call's own edge count; a few heavy (hub) roots
            // instead get exact slots for the re-run: offsets = the scan of
            // the per-root counts the failed run already produced.
            int64_t es = s->e_stride;
            while (es < need) es *= 2;
            const int64_t uniform = (s->R + 1) * es, budget = std::max<int64_t>(4 * (int64_t)s->E, 1 << 24);
            if (uniform <= budget && es < (1 << 30)) {
                s->e_stride = (int32_t)es;
                s->escratch.release();
            } else {
                s->eoff_exact.reserve((size_t)s->R + 1);
                HGS_CUDA(cudaMemcpyAsync(s->eoff_exact.p, s->root_eoff.p, sizeof(int32_t) * ((size_t)s->R + 1),
                                         cudaMemcpyDeviceToDevice, s->stream));
                s->escratch.reserve((size_t)s->E + 1);
                s->exact_slots = true;
            }
        }
        if ((size_t)s->E > s->e_cap) {
            s->e_cap = (size_t)s->E + (size_t)s->E / 8 + 1024;
            s->e_row.release(); s->e_col.release(); s->e_gid.release(); s->ye.release(); s->lab.release();
        }
        if ((size_t)s->V > s->v_cap) {
            s->v_cap = (size_t)s->V;
            s->l2g.release(); s->xv.release();
        }
        ++s->reruns;
        sample_enqueue(s, cfg, in, true);
        sample_finish(s, cfg, in);
    }
}

void sample_stats(hgs_sample* s, int64_t* out, int n) {
    if (s->depth > 15) fail(HGS_ERANGE, "hgs_sample_stats: depth > 15");
    s->stats_tmp.reserve(19);
    HGS_CUDA(cudaMemsetAsync(s->stats_tmp.p, 0, sizeof(unsigned long long) * 19, s->stream));
    launch_stats(s->level_counts.p, (int32_t)s->depth, s->root_scan.p, s->decisions.p, s->draws.p,
                 (int32_t)s->R, s->stats_tmp.p, s->stream);
    unsigned long long h[19];
    HGS_CUDA(cudaMemcpyAsync(h, s->stats_tmp.p, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
    HGS_CUDA(cudaStreamSynchronize(s->stream));
    std::vector<int64_t> st(10 + 16, 0);
    st[0] = s->R; st[1] = s->k; st[2] = s->V; st[3] = s->E; st[4] = (int64_t)h[0];
    for (int l = 0; l <= s->depth; ++l) {
        if (l < s->depth) st[5] += (int64_t)h[3 + l];
        if (l >= 1) st[6] += (int64_t)h[3 + l];
        st[9 + l] = (int64_t)h[3 + l];
    }
    st[7] = (int64_t)h[1];
    st[8] = (int64_t)h[2];
    for (int i = 0; i < n && i < (int)st.size(); ++i) out[i] = st[i];
}

void gather_rows(DevGraph& g, const int64_t* d_l2g, int64_t V, const int64_t* d_eid, int64_t E,
                 double* d_xv, double* d_ye, uint8_t* d_lab, cudaStream_t st) {
    launch_gather(g, d_l2g, V, d_eid, E, d_xv, d_ye, d_lab, st);
}

}  // namespace hgs
