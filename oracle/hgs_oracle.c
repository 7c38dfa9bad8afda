/*
 * hgs_oracle.c — TEST INFRASTRUCTURE ONLY (see hgs_oracle.h).
 *
 * A plain-C restatement of the reference's bulk ShaDow sampler. Each routine
 * cites the reference lines it restates. The algorithm follows the bulk,
 * level-synchronous formulation of sampler.cpp:123-201 (stacked frontier rows
 * with a row -> root map), not the per-root loop, so its intermediate state
 * (frontier rows per level) mirrors the reference's FrontierObserver data.
 *
 * Exception texts are reproduced verbatim so that the error-path parity tests
 * can compare messages.
 */
#include "hgs_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ===================================================================== */
/* RNG                                                                    */
/* ===================================================================== */

uint64_t or_splitmix64(uint64_t* x) { /* rng.cpp:12-18 */
    uint64_t z = (*x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void or_xoshiro_seed(or_xoshiro* r, uint64_t seed) { /* rng.cpp:26-29 */
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = or_splitmix64(&x);
}

static uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

uint64_t or_xoshiro_next(or_xoshiro* r) { /* rng.cpp:31-41 (xoshiro256**) */
    uint64_t* s = r->s;
    const uint64_t out = rotl64(s[1] * 5u, 7) * 9u;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
}

/* rng.cpp:43-50: reject draws below (2^64 mod n), then reduce. */
static uint64_t bounded_draws(or_xoshiro* r, uint64_t n, int64_t* draws) {
    const uint64_t floor_reject = (0ULL - n) % n;
    for (;;) {
        const uint64_t x = or_xoshiro_next(r);
        if (draws) ++*draws;
        if (x >= floor_reject) return x % n;
    }
}

uint64_t or_xoshiro_bounded(or_xoshiro* r, uint64_t n) { return bounded_draws(r, n, NULL); }

uint64_t or_derive(uint64_t seed, const uint64_t* path, int len) { /* rng.cpp:76-85 */
    uint64_t s = seed;
    uint64_t h = or_splitmix64(&s);
    for (int i = 0; i < len; ++i) {
        s = h ^ (path[i] + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2));
        h = or_splitmix64(&s);
    }
    return h;
}

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

/* Partial Fisher-Yates over a *virtual* identity array [0, n): only the
 * positions the k swaps touch are materialised (a tiny association list), so
 * a choose over a hub row costs O(k^2) instead of the reference's O(n) iota
 * (rng.cpp:105-119). The outcome is identical: slot i receives the value at
 * j = i + bounded(n - i) and slot j receives the old value of slot i. */
typedef struct { uint32_t pos, val; } slot_t;

static uint32_t vget(const slot_t* m, int cnt, uint32_t pos) {
    for (int i = cnt - 1; i >= 0; --i)
        if (m[i].pos == pos) return m[i].val;
    return pos;
}
static int vset(slot_t* m, int cnt, uint32_t pos, uint32_t val) {
    for (int i = cnt - 1; i >= 0; --i)
        if (m[i].pos == pos) { m[i].val = val; return cnt; }
    m[cnt].pos = pos;
    m[cnt].val = val;
    return cnt + 1;
}

typedef uint64_t (*draw_fn)(void* ctx, uint32_t step, uint64_t bound);

static uint32_t choose_with(draw_fn draw, void* ctx, uint32_t n, uint32_t k, uint32_t* out) {
    if (k > n) k = n;
    slot_t* m = (slot_t*)malloc(sizeof(slot_t) * (2 * (size_t)k + 1));
    int cnt = 0;
    for (uint32_t i = 0; i < k; ++i) {
        const uint32_t j = i + (uint32_t)draw(ctx, i, (uint64_t)(n - i));
        const uint32_t vi = vget(m, cnt, i), vj = vget(m, cnt, j);
        cnt = vset(m, cnt, i, vj);
        cnt = vset(m, cnt, j, vi);
    }
    for (uint32_t i = 0; i < k; ++i) out[i] = vget(m, cnt, i);
    free(m);
    qsort(out, k, sizeof(uint32_t), cmp_u32);
    return k;
}

typedef struct { or_xoshiro* rng; int64_t* draws; } xo_ctx;
static uint64_t xo_draw(void* c, uint32_t step, uint64_t bound) {
    (void)step;
    xo_ctx* x = (xo_ctx*)c;
    return bounded_draws(x->rng, bound, x->draws);
}

uint32_t or_choose_xoshiro(or_xoshiro* r, uint32_t n, uint32_t k, uint32_t* out) {
    xo_ctx c = {r, NULL};
    return choose_with(xo_draw, &c, n, k, out);
}

/* Philox4x32-10, Random123 multipliers / Weyl constants. */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c0 = n0; c1 = (uint32_t)p1; c2 = n2; c3 = (uint32_t)p0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

#define OR_PHILOX_TAG 0x43484f53u
typedef struct { uint32_t key[2]; uint32_t decision; int64_t* draws; } ph_ctx;
static uint64_t ph_draw(void* c, uint32_t step, uint64_t bound) {
    ph_ctx* p = (ph_ctx*)c;
    const uint64_t floor_reject = (0ULL - bound) % bound;
    for (uint32_t attempt = 0;; ++attempt) {
        const uint32_t ctr[4] = {p->decision, step, attempt, OR_PHILOX_TAG};
        uint32_t o[4];
        or_philox4x32_10(ctr, p->key, o);
        if (p->draws) ++*p->draws;
        const uint64_t x = ((uint64_t)o[1] << 32) | o[0];
        if (x >= floor_reject) return x % bound;
    }
}

uint32_t or_choose_philox(uint64_t seed, uint32_t decision, uint32_t n, uint32_t k,
                          uint32_t* out) {
    ph_ctx c = {{(uint32_t)seed, (uint32_t)(seed >> 32)}, decision, NULL};
    return choose_with(ph_draw, &c, n, k, out);
}

int64_t or_epoch_root_batches(int64_t n, int64_t b, uint64_t rng_seed, int64_t* perm) {
    /* sampler.cpp:245-263: backwards Fisher-Yates, then full slices of b. */
    or_xoshiro r;
    or_xoshiro_seed(&r, rng_seed);
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    for (int64_t i = n - 1; i > 0; --i) {
        const int64_t j = (int64_t)or_xoshiro_bounded(&r, (uint64_t)i + 1);
        const int64_t t = perm[i];
        perm[i] = perm[j];
        perm[j] = t;
    }
    return n < b ? 1 : n / b;
}

/* ===================================================================== */
/* sparse                                                                  */
/* ===================================================================== */

static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* sparse.cpp:260-272 restated: per row u, merge out-neighbours with
 * in-neighbours (gathered through a counting transpose), sort, unique. */
int64_t or_symmetrize(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* out_rp,
                      int64_t* out_ci) {
    const int64_t nnz = rp[n];
    int64_t* trp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t* tci = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz ? nnz : 1));
    for (int64_t k = 0; k < nnz; ++k) ++trp[ci[k] + 1];
    for (int64_t v = 0; v < n; ++v) trp[v + 1] += trp[v];
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    memcpy(cur, trp, sizeof(int64_t) * (size_t)n);
    for (int64_t u = 0; u < n; ++u)
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k) tci[cur[ci[k]]++] = u;
    int64_t w = 0;
    out_rp[0] = 0;
    for (int64_t u = 0; u < n; ++u) {
        const int64_t start = w;
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k) out_ci[w++] = ci[k];
        for (int64_t k = trp[u]; k < trp[u + 1]; ++k) out_ci[w++] = tci[k];
        qsort(out_ci + start, (size_t)(w - start), sizeof(int64_t), cmp_i64);
        int64_t uniq = start;
        for (int64_t k = start; k < w; ++k)
            if (k == start || out_ci[k] != out_ci[uniq - 1]) out_ci[uniq++] = out_ci[k];
        w = uniq;
        out_rp[u + 1] = w;
    }
    free(trp);
    free(tci);
    free(cur);
    return w;
}

/* ===================================================================== */
/* sampler                                                                 */
/* ===================================================================== */

struct or_result {
    int64_t k, R, V, E, f_v, f_e, gathered, depth;
    int64_t *batch_voff, *batch_eoff, *comp_off, *l2g, *roots_local;
    int64_t *e_row, *e_col, *e_gid;
    double* e_val;
    double *xv, *ye;
    uint8_t* lab;
    int64_t *draws, *decisions, *level_counts, *touched;
    int64_t touched_total;
};

typedef struct { int64_t* p; int64_t n, cap; } vec64;
static void v_push(vec64* v, int64_t x) {
    if (v->n == v->cap) {
        v->cap = v->cap ? v->cap * 2 : 64;
        v->p = (int64_t*)realloc(v->p, sizeof(int64_t) * (size_t)v->cap);
    }
    v->p[v->n++] = x;
}

static void set_err(char* err, int errlen, const char* msg) {
    if (err && errlen > 0) snprintf(err, (size_t)errlen, "%s", msg);
}

static int64_t bsearch_i64(const int64_t* a, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return (lo < n && a[lo] == key) ? lo : -1;
}

void or_result_free(or_result* r) {
    if (!r) return;
    free(r->batch_voff); free(r->batch_eoff); free(r->comp_off); free(r->l2g);
    free(r->roots_local); free(r->e_row); free(r->e_col); free(r->e_gid); free(r->e_val);
    free(r->xv); free(r->ye); free(r->lab); free(r->draws); free(r->decisions);
    free(r->level_counts); free(r->touched);
    free(r);
}

or_result* or_bulk_shadow(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci,
                          const double* values, const int64_t* roots,
                          const int64_t* batch_off, int64_t n_batches,
                          const uint64_t* seeds, int rng_kind, int64_t depth, int64_t fanout,
                          int symmetrize, const double* node_feat, int64_t f_v,
                          const double* edge_feat, int64_t f_e, const uint8_t* labels,
                          char* err, int errlen) {
    return or_bulk_shadow_ex(n_rows, n_cols, rp, ci, values, roots, batch_off, n_batches, seeds,
                             NULL, rng_kind, depth, fanout, symmetrize, 0, node_feat, f_v,
                             edge_feat, f_e, labels, err, errlen);
}

or_result* or_bulk_shadow_ex(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci,
                             const double* values, const int64_t* roots,
                             const int64_t* batch_off, int64_t n_batches,
                             const uint64_t* seeds, const uint64_t* state, int rng_kind,
                             int64_t depth, int64_t fanout, int symmetrize, int flags,
                             const double* node_feat, int64_t f_v, const double* edge_feat,
                             int64_t f_e, const uint8_t* labels, char* err, int errlen) {
    const int seq_walk = (flags & 1) != 0;
    char msg[256];
    /* SamplerConfig::validate (sampler.cpp:57-62) */
    if (depth < 1) { set_err(err, errlen, "SamplerConfig: depth must be >= 1"); return NULL; }
    if (fanout < 1) { set_err(err, errlen, "SamplerConfig: fanout must be >= 1"); return NULL; }
    /* check_roots per batch (sampler.cpp:12-20, called at :128) */
    const int64_t R = batch_off[n_batches];
    {
        char* seen = (char*)calloc((size_t)(n_rows > 0 ? n_rows : 1), 1);
        for (int64_t b = 0; b < n_batches; ++b) {
            for (int64_t i = batch_off[b]; i < batch_off[b + 1]; ++i) {
                const int64_t r = roots[i];
                if (r < 0 || r >= n_rows) {
                    snprintf(msg, sizeof msg, "sampler: root %lld out of range", (long long)r);
                    set_err(err, errlen, msg); free(seen); return NULL;
                }
                if (seen[r]) {
                    snprintf(msg, sizeof msg, "sampler: duplicate root %lld", (long long)r);
                    set_err(err, errlen, msg); free(seen); return NULL;
                }
                seen[r] = 1;
            }
            for (int64_t i = batch_off[b]; i < batch_off[b + 1]; ++i) seen[roots[i]] = 0;
        }
        free(seen);
    }
    /* walk matrix (sampler.cpp:129): symmetrize_pattern checks squareness;
     * the unsymmetrized walk meets the same check inside spgemm(q, walk). */
    if (symmetrize && n_rows != n_cols) {
        set_err(err, errlen, "symmetrize_pattern: matrix must be square"); return NULL;
    }
    if (!symmetrize && n_rows != n_cols) {
        snprintf(msg, sizeof msg, "spgemm: inner dimensions disagree (%lld vs %lld)",
                 (long long)n_cols, (long long)n_rows);
        set_err(err, errlen, msg); return NULL;
    }
    const int64_t n = n_rows, nnz = rp[n];
    int64_t *wrp, *wci;
    const double* wval = NULL; /* only for the unsymmetrized walk */
    if (symmetrize) {
        wrp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
        wci = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * nnz + 1));
        or_symmetrize(n, rp, ci, wrp, wci);
    } else {
        wrp = (int64_t*)rp; wci = (int64_t*)ci; wval = seq_walk ? NULL : values;
    }

    /* Stacked Q: one row per root (sampler.cpp:132-145). Level l's frontier
     * is kept as (lvl_col[l], lvl_root[l]); level 0 holds the roots. */
    or_result* res = (or_result*)calloc(1, sizeof(or_result));
    res->k = n_batches; res->R = R; res->depth = depth;
    res->draws = (int64_t*)calloc((size_t)(R ? R : 1), sizeof(int64_t));
    res->decisions = (int64_t*)calloc((size_t)(R ? R : 1), sizeof(int64_t));
    res->level_counts = (int64_t*)calloc((size_t)(R ? R : 1) * (size_t)(depth + 1), sizeof(int64_t));
    for (int64_t r = 0; r < R; ++r) res->level_counts[r * (depth + 1)] = 1;

    or_xoshiro* streams = NULL;
    if (rng_kind == OR_RNG_XOSHIRO) {
        streams = (or_xoshiro*)malloc(sizeof(or_xoshiro) * (size_t)(R ? R : 1));
        for (int64_t r = 0; r < R; ++r) {
            if (state) memcpy(streams[r].s, state + 4 * r, sizeof(streams[r].s));
            else or_xoshiro_seed(&streams[r], seeds[r]);
        }
    }

    int64_t** lvl_col = (int64_t**)calloc((size_t)depth + 1, sizeof(int64_t*));
    int64_t** lvl_root = (int64_t**)calloc((size_t)depth + 1, sizeof(int64_t*));
    int64_t* lvl_n = (int64_t*)calloc((size_t)depth + 1, sizeof(int64_t));
    lvl_col[0] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(R ? R : 1));
    lvl_root[0] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(R ? R : 1));
    for (int64_t r = 0; r < R; ++r) { lvl_col[0][r] = roots[r]; lvl_root[0][r] = r; }
    lvl_n[0] = R;
    uint32_t* pos = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(fanout + 1));
    int64_t* support = NULL; int64_t sup_cap = 0;

    for (int64_t level = 0; level < depth; ++level) {
        const int64_t* q_col = lvl_col[level];
        const int64_t* q_root = lvl_root[level];
        const int64_t nq = lvl_n[level];
        /* row_normalize's negative check runs over the whole P before any
         * row of this level is sampled (sparse.cpp:193-206 via :161). */
        if (wval) {
            for (int64_t r = 0; r < nq; ++r) {
                const int64_t v = q_col[r];
                for (int64_t k = wrp[v]; k < wrp[v + 1]; ++k)
                    if (wval[k] != 0.0 && wval[k] < 0.0) {
                        snprintf(msg, sizeof msg, "row_normalize: negative value in row %lld",
                                 (long long)r);
                        set_err(err, errlen, msg);
                        goto fail;
                    }
            }
        }
        vec64 ncol = {0}, nroot = {0};
        for (int64_t r = 0; r < nq; ++r) {
            const int64_t v = q_col[r], root = q_root[r];
            /* support of row r of spgemm(q, walk): walk entries whose value
             * survives the zero-drop (sparse.cpp:118-121, 134-137). */
            int64_t deg = 0;
            const int64_t w0 = wrp[v], w1 = wrp[v + 1];
            if (w1 - w0 > sup_cap) {
                sup_cap = w1 - w0;
                support = (int64_t*)realloc(support, sizeof(int64_t) * (size_t)sup_cap);
            }
            for (int64_t k = w0; k < w1; ++k)
                if (!wval || wval[k] != 0.0) support[deg++] = wci[k];
            if (deg == 0) continue; /* sampler.cpp:75 */
            const uint32_t kk = (uint32_t)(deg < fanout ? deg : fanout);
            uint32_t got;
            if (rng_kind == OR_RNG_XOSHIRO) {
                xo_ctx c = {&streams[root], &res->draws[root]};
                got = choose_with(xo_draw, &c, (uint32_t)deg, kk, pos);
            } else {
                ph_ctx c = {{(uint32_t)seeds[root], (uint32_t)(seeds[root] >> 32)},
                            (uint32_t)(res->decisions[root] + (state ? state[root] : 0)),
                            &res->draws[root]};
                got = choose_with(ph_draw, &c, (uint32_t)deg, kk, pos);
            }
            ++res->decisions[root];
            for (uint32_t i = 0; i < got; ++i) { /* sampler.cpp:173-182 */
                v_push(&ncol, support[pos[i]]);
                v_push(&nroot, root);
                ++res->level_counts[root * (depth + 1) + level + 1];
            }
        }
        lvl_col[level + 1] = ncol.p ? ncol.p : (int64_t*)malloc(8);
        lvl_root[level + 1] = nroot.p ? nroot.p : (int64_t*)malloc(8);
        lvl_n[level + 1] = ncol.n;
    }

    /* touched lists per root: root first, then levels in BFS order */
    {
        int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(R + 1));
        start[0] = 0;
        for (int64_t r = 0; r < R; ++r) {
            int64_t t = 0;
            for (int64_t l = 0; l <= depth; ++l) t += res->level_counts[r * (depth + 1) + l];
            start[r + 1] = start[r] + t;
        }
        res->touched_total = start[R];
        res->touched = (int64_t*)malloc(sizeof(int64_t) * (size_t)(start[R] ? start[R] : 1));
        int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(R ? R : 1));
        for (int64_t r = 0; r < R; ++r) { res->touched[start[r]] = roots[r]; fill[r] = start[r] + 1; }
        for (int64_t l = 1; l <= depth; ++l)
            for (int64_t i = 0; i < lvl_n[l]; ++i) res->touched[fill[lvl_root[l][i]]++] = lvl_col[l][i];

        /* sorted_vertex_set + induced_subgraph + block_diag per batch
         * (sampler.cpp:190-200, 26-53; sparse.cpp:177-191, 245-258) */
        vec64 l2g = {0}, erow = {0}, ecol = {0}, egid = {0};
        res->batch_voff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_batches + 1));
        res->batch_eoff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_batches + 1));
        res->comp_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(R + n_batches + 1));
        res->roots_local = (int64_t*)malloc(sizeof(int64_t) * (size_t)(R ? R : 1));
        int64_t* set = (int64_t*)malloc(sizeof(int64_t) * (size_t)(start[R] + 1));
        for (int64_t b = 0; b < n_batches; ++b) {
            res->batch_voff[b] = l2g.n;
            res->batch_eoff[b] = erow.n;
            int64_t comp_base = 0;
            for (int64_t r = batch_off[b]; r < batch_off[b + 1]; ++r) {
                res->comp_off[r + b] = comp_base;
                const int64_t t = start[r + 1] - start[r];
                memcpy(set, res->touched + start[r], sizeof(int64_t) * (size_t)t);
                qsort(set, (size_t)t, sizeof(int64_t), cmp_i64);
                int64_t m = 0;
                for (int64_t i = 0; i < t; ++i)
                    if (i == 0 || set[i] != set[m - 1]) set[m++] = set[i];
                for (int64_t i = 0; i < m; ++i) v_push(&l2g, set[i]);
                res->roots_local[r] = comp_base + bsearch_i64(set, m, roots[r]);
                for (int64_t i = 0; i < m; ++i) {
                    const int64_t u = set[i];
                    for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
                        if (values && values[k] == 0.0) continue; /* zero-drop */
                        const int64_t j = bsearch_i64(set, m, ci[k]);
                        if (j < 0) continue;
                        v_push(&erow, comp_base + i);
                        v_push(&ecol, comp_base + j);
                        v_push(&egid, k);
                    }
                }
                comp_base += m;
            }
            res->comp_off[batch_off[b + 1] + b] = comp_base;
        }
        res->batch_voff[n_batches] = l2g.n;
        res->batch_eoff[n_batches] = erow.n;
        res->V = l2g.n; res->E = erow.n;
        res->l2g = l2g.p; res->e_row = erow.p; res->e_col = ecol.p; res->e_gid = egid.p;
        res->e_val = (double*)malloc(sizeof(double) * (size_t)(res->E ? res->E : 1));
        for (int64_t e = 0; e < res->E; ++e)
            res->e_val[e] = values ? values[res->e_gid[e]] : (double)(res->e_gid[e] + 1);
        free(set); free(fill); free(start);
    }

    /* gather_features (sampler.cpp:211-243) */
    if (node_feat && edge_feat && labels) {
        res->gathered = 1; res->f_v = f_v; res->f_e = f_e;
        for (int64_t i = 0; i < res->V; ++i)
            if (res->l2g[i] < 0 || res->l2g[i] >= n) {
                set_err(err, errlen, "gather_features: batch vertex out of range for event");
                goto fail;
            }
        res->xv = (double*)malloc(sizeof(double) * (size_t)(res->V * f_v + 1));
        for (int64_t i = 0; i < res->V; ++i)
            memcpy(res->xv + i * f_v, node_feat + res->l2g[i] * f_v, sizeof(double) * (size_t)f_v);
        res->ye = (double*)malloc(sizeof(double) * (size_t)(res->E * f_e + 1));
        res->lab = (uint8_t*)malloc((size_t)res->E + 1);
        for (int64_t e = 0; e < res->E; ++e) {
            const int64_t id = (int64_t)llround(res->e_val[e]) - 1;
            if (id < 0 || id >= nnz) {
                set_err(err, errlen,
                        "gather_features: adjacency values do not carry edge ids; "
                        "sample from make_edge_id_matrix(event)");
                goto fail;
            }
            res->e_gid[e] = id;
            res->e_val[e] = 1.0; /* gather_features resets values (sampler.cpp:240) */
            res->lab[e] = labels[id];
            memcpy(res->ye + e * f_e, edge_feat + id * f_e, sizeof(double) * (size_t)f_e);
        }
    }

    for (int64_t l = 0; l <= depth; ++l) { free(lvl_col[l]); free(lvl_root[l]); }
    free(lvl_col); free(lvl_root); free(lvl_n); free(pos); free(support); free(streams);
    if (symmetrize) { free(wrp); free(wci); }
    return res;

fail:
    for (int64_t l = 0; l <= depth; ++l) { free(lvl_col[l]); free(lvl_root[l]); }
    free(lvl_col); free(lvl_root); free(lvl_n);
    or_result_free(res);
    if (symmetrize) { free(wrp); free(wci); }
    free(streams); free(pos); free(support);
    return NULL;
}

void or_result_counts(const or_result* r, int64_t* c) {
    c[0] = r->k; c[1] = r->R; c[2] = r->V; c[3] = r->E;
    c[4] = r->f_v; c[5] = r->f_e; c[6] = r->gathered; c[7] = r->depth;
}

int64_t or_result_touched_total(const or_result* r) { return r->touched_total; }

#define CP(dst, src, cnt, T) do { if (dst && (cnt) > 0) memcpy(dst, src, sizeof(T) * (size_t)(cnt)); } while (0)
void or_result_copy(const or_result* r, int64_t* batch_voff, int64_t* batch_eoff,
                    int64_t* comp_off, int64_t* l2g, int64_t* roots_local, int64_t* e_row,
                    int64_t* e_col, int64_t* e_gid, double* e_val, double* xv, double* ye,
                    uint8_t* lab, int64_t* draws, int64_t* decisions, int64_t* level_counts,
                    int64_t* touched) {
    CP(batch_voff, r->batch_voff, r->k + 1, int64_t);
    CP(batch_eoff, r->batch_eoff, r->k + 1, int64_t);
    CP(comp_off, r->comp_off, r->R + r->k, int64_t);
    CP(l2g, r->l2g, r->V, int64_t);
    CP(roots_local, r->roots_local, r->R, int64_t);
    CP(e_row, r->e_row, r->E, int64_t);
    CP(e_col, r->e_col, r->E, int64_t);
    CP(e_gid, r->e_gid, r->E, int64_t);
    CP(e_val, r->e_val, r->E, double);
    if (r->gathered) {
        CP(xv, r->xv, r->V * r->f_v, double);
        CP(ye, r->ye, r->E * r->f_e, double);
        CP(lab, r->lab, r->E, uint8_t);
    }
    CP(draws, r->draws, r->R, int64_t);
    CP(decisions, r->decisions, r->R, int64_t);
    CP(level_counts, r->level_counts, r->R * (r->depth + 1), int64_t);
    CP(touched, r->touched, r->touched_total, int64_t);
}
