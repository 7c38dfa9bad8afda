/*
 * hgs_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C99) of the reference hot path
 *   hitgnn::bulk_shadow + hitgnn::gather_features
 * (/root/reference/proj/src/sampler.cpp:123-201, 211-243) and of the sparse /
 * RNG semantics it relies on (sparse.cpp, rng.cpp). It is the checker the
 * parity tests compare the CUDA path against; it is never linked into, called
 * by, or measured as the product. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.
 *
 * Parity pinning: validated against (1) the reference itself compiled from
 * /root/reference by oracle/Makefile into oracle/_ref/ (tests/test_oracle.py),
 * (2) the committed golden fixtures in tests/golden/ (generated from
 * oracle/_ref by tests/golden/make_golden.py), (3) the RNG known answers in
 * SURVEY.md Appendix A.6 and the Random123 Philox4x32-10 KATs.
 */
#ifndef HGS_ORACLE_H
#define HGS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG (rng.cpp) ---------------------------------------------------- */
typedef struct { uint64_t s[4]; } or_xoshiro;

uint64_t or_splitmix64(uint64_t* x);                         /* rng.cpp:12-18  */
void     or_xoshiro_seed(or_xoshiro* r, uint64_t seed);      /* rng.cpp:26-29  */
uint64_t or_xoshiro_next(or_xoshiro* r);                     /* rng.cpp:31-41  */
uint64_t or_xoshiro_bounded(or_xoshiro* r, uint64_t n);      /* rng.cpp:43-50  */
uint64_t or_derive(uint64_t seed, const uint64_t* path, int len); /* rng.cpp:76-85 */
/* RandomChoiceSource::choose (rng.cpp:105-119); out gets min(k,n) sorted
 * positions; returns that count. */
uint32_t or_choose_xoshiro(or_xoshiro* r, uint32_t n, uint32_t k, uint32_t* out);

/* Philox4x32-10 (Random123 constants) and the Philox decision stream of
 * SURVEY.md Appendix A.3 (ctr = {decision, draw, attempt, 0x43484f53}). */
void     or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint32_t or_choose_philox(uint64_t seed, uint32_t decision, uint32_t n, uint32_t k,
                          uint32_t* out);

/* Fisher-Yates root batching (sampler.cpp:245-263). Writes n_vertices
 * permuted ids to perm; returns number of full batches (or 1 if n < b). */
int64_t or_epoch_root_batches(int64_t n_vertices, int64_t batch_size, uint64_t rng_seed,
                              int64_t* perm);

/* ---- sparse (sparse.cpp) ---------------------------------------------- */
/* symmetrize_pattern (sparse.cpp:260-272): pattern of A ∪ Aᵀ, per row
 * ascending unique. out_ci needs capacity 2*nnz. Returns walk nnz. */
int64_t or_symmetrize(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* out_rp,
                      int64_t* out_ci);

/* ---- sampler (sampler.cpp) -------------------------------------------- */
enum { OR_RNG_XOSHIRO = 0, OR_RNG_PHILOX = 1 };

typedef struct or_result or_result;

/* bulk_shadow over one CSR graph. values may be NULL (pattern with value
 * k+1 at CSR position k, i.e. make_edge_id_matrix). node_feat/edge_feat/
 * labels may be NULL (no gather). Returns NULL on invalid input with the
 * reference's exception text in err. */
or_result* or_bulk_shadow(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci,
                          const double* values, const int64_t* roots,
                          const int64_t* batch_off, int64_t n_batches,
                          const uint64_t* seeds, int rng_kind, int64_t depth, int64_t fanout,
                          int symmetrize, const double* node_feat, int64_t f_v,
                          const double* edge_feat, int64_t f_e, const uint8_t* labels,
                          char* err, int errlen);

/* Extended form: state (nullable) resumes non-fresh per-root streams —
 * xoshiro: 4 state words per root; philox: decisions already consumed per
 * root. flags & 1 = shadow_reference walk semantics for the unsymmetrized
 * walk (raw rows of A, explicit zeros kept, no negative check;
 * sampler.cpp:104-106) instead of bulk_shadow's spgemm support. */
or_result* or_bulk_shadow_ex(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int64_t* ci,
                             const double* values, const int64_t* roots,
                             const int64_t* batch_off, int64_t n_batches,
                             const uint64_t* seeds, const uint64_t* state, int rng_kind,
                             int64_t depth, int64_t fanout, int symmetrize, int flags,
                             const double* node_feat, int64_t f_v, const double* edge_feat,
                             int64_t f_e, const uint8_t* labels, char* err, int errlen);

/* counts: [0]=n_batches [1]=R [2]=V [3]=E [4]=f_v [5]=f_e [6]=gathered [7]=depth */
void or_result_counts(const or_result* r, int64_t* counts);
/* Any pointer may be NULL. Layout (flat over batches, batch-local indices):
 * batch_voff/eoff[k+1], comp_off[R+k], l2g[V], roots_local[R], e_row/e_col/e_gid[E],
 * e_val[E] (value before gather), xv[V*f_v], ye[E*f_e], lab[E],
 * draws/decisions[R] (per-root consumed RNG draws / choose calls),
 * level_counts[R*(depth+1)] (frontier rows per root per level),
 * touched[sum level_counts] (per root: root, then levels 1..d in BFS order). */
void or_result_copy(const or_result* r, int64_t* batch_voff, int64_t* batch_eoff,
                    int64_t* comp_off, int64_t* l2g, int64_t* roots_local, int64_t* e_row,
                    int64_t* e_col, int64_t* e_gid, double* e_val, double* xv, double* ye,
                    uint8_t* lab, int64_t* draws, int64_t* decisions, int64_t* level_counts,
                    int64_t* touched);
int64_t or_result_touched_total(const or_result* r);
void or_result_free(or_result* r);

#ifdef __cplusplus
}
#endif
#endif
