/*
 * hgs.h — C ABI of the B200 bulk ShaDow sampler ("hitgnn gpu sampler").
 *
 * This is the drop-in boundary for the reference hot path
 *   hitgnn::bulk_shadow      /root/reference/proj/include/hitgnn/sampler.hpp:88-91
 *                            (src/sampler.cpp:123-201)
 *   hitgnn::shadow_reference sampler.hpp:75-76 (sampler.cpp:88-121)
 *   hitgnn::gather_features  sampler.hpp:102   (sampler.cpp:211-243)
 *   hitgnn::symmetrize_pattern sparse.hpp:97   (sparse.cpp:260-272)
 *   hitgnn::Rng::derive      rng.hpp:31-32     (rng.cpp:76-85)
 * Plain pointers and sizes only; no C++ or torch types. Host-side C++
 * (include/hitgnn/*.hpp, libhitgnn_gpu.so) and Python (ctypes) sit above it.
 *
 * Errors: every int-returning call returns HGS_OK (0) or an HGS_E* code; the
 * message is in hgs_last_error() (thread-local). HGS_EINVAL carries the
 * reference's std::invalid_argument text verbatim where one exists (e.g.
 * "sampler: duplicate root 17", sampler.cpp:18).
 *
 * Threading: a graph handle is bound to one CUDA device. A sample handle is
 * a reusable device workspace + output set bound to one graph and one CUDA
 * stream; calls on one sample handle must not overlap. Different sample
 * handles (e.g. one per host thread / GPU) are independent.
 *
 * Device output layout of one call (all int32 unless noted; V, E = totals
 * over all batches of the call; k = n_batches, R = roots):
 *   l2g[V]          local_to_global, components back to back, each sorted
 *   roots_local[R]  batch-local index of each root
 *   comp_off[R+k]   per batch b: its R_b+1 batch-local component offsets
 *   batch_voff[k+1], batch_eoff[k+1]  call-level vertex / edge offsets
 *   e_row[E], e_col[E]  batch-local endpoints (row-major, columns ascending)
 *   e_gid[E]        edge id = CSR position in the input A (make_edge_id_matrix
 *                   value - 1, sampler.cpp:203-209)
 *   root_voff[R+1], root_eoff[R+1]  call-level offsets of every component
 *   xv[V*f_v] (f64), ye[E*f_e] (f64), lab[E] (u8)   when gather != 0
 *   draws[R], decisions[R] (u32) RNG draws / choose() calls consumed per root
 */
#ifndef HGS_H
#define HGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HGS_ABI_VERSION 1

enum {
    HGS_OK = 0,
    HGS_EINVAL = 1,   /* std::invalid_argument in the reference            */
    HGS_ECUDA = 2,    /* CUDA / runtime failure (std::runtime_error)        */
    HGS_ERANGE = 3    /* size limit of this implementation exceeded        */
};

enum {
    HGS_RNG_XOSHIRO = 0, /* PerRootChoiceSource: xoshiro256** per root stream */
    HGS_RNG_PHILOX = 1   /* PhiloxChoiceSource: counter-based per decision     */
};

typedef struct hgs_graph hgs_graph;
typedef struct hgs_sample hgs_sample;

/* SamplerConfig (sampler.hpp:16-24) plus device options. batch_size and
 * bulk_batches are validated like the reference but do not change results. */
typedef struct {
    int64_t depth;        /* d >= 1 */
    int64_t fanout;       /* s >= 1 */
    int64_t batch_size;   /* b >= 1 (validated only) */
    int64_t bulk_batches; /* k >= 1 (validated only) */
    int32_t symmetrize;   /* walk on pattern(A ∪ Aᵀ) */
    int32_t rng;          /* HGS_RNG_* */
    int32_t gather;       /* also gather node/edge features + labels */
    int32_t profile;      /* record per-kernel CUDA event times */
    int32_t flags;        /* HGS_FLAG_* */
} hgs_config;

/* shadow_reference semantics for the unsymmetrized walk: sample over the raw
 * rows of A (explicit zeros included, no negative-value check), as
 * sampler.cpp:104-106 does, instead of bulk_shadow's row_normalize(spgemm(Q, A))
 * support (zeros dropped, negatives rejected; sampler.cpp:161). The two
 * differ only when A stores explicit zeros or negative values. */
#define HGS_FLAG_SEQ_WALK 1
/* Keep a copy of every root's BFS-order touched list (K2 overwrites the
 * working copy with the sorted set) for hgs_sample_copy_frontiers: the
 * FrontierObserver hook of bulk_shadow (sampler.cpp:149-158, 186). */
#define HGS_FLAG_KEEP_FRONTIERS 2

/* Host destinations for hgs_sample_copy_to_host (any pointer may be NULL). */
typedef struct {
    int32_t* batch_voff;  /* k+1 */
    int32_t* batch_eoff;  /* k+1 */
    int32_t* comp_off;    /* R+k */
    int32_t* l2g;         /* V   */
    int32_t* roots_local; /* R   */
    int32_t* e_row;       /* E   */
    int32_t* e_col;       /* E   */
    int32_t* e_gid;       /* E   */
    double* xv;           /* V*f_v */
    double* ye;           /* E*f_e */
    uint8_t* lab;         /* E   */
    uint32_t* draws;      /* R   */
    uint32_t* decisions;  /* R   */
} hgs_host_out;

/* Device pointers of the last call's outputs (valid after hgs_sample_wait,
 * until the next run or destroy on the same sample handle). */
typedef struct {
    const int32_t *batch_voff, *batch_eoff, *comp_off, *l2g, *roots_local;
    const int32_t *e_row, *e_col, *e_gid, *root_voff, *root_eoff;
    const double *xv, *ye;
    const uint8_t* lab;
    const uint32_t *draws, *decisions;
    const int32_t *touched, *touched_count; /* expand scratch: per root, stride touched_stride */
    const int32_t* level_counts;            /* [R][depth+1] frontier rows per level */
    int64_t touched_stride;
} hgs_device_views;

const char* hgs_last_error(void);
int hgs_abi_version(void);
int hgs_device_count(int* count);
/* Page-locked host memory (cudaMallocHost / cudaFreeHost) for staging
 * buffers of host callers that do not link the CUDA runtime themselves. */
int hgs_host_alloc(size_t bytes, void** out);
int hgs_host_free(void* p);
/* The calling thread's current CUDA device (cudaGetDevice): the device the
 * C++ drop-in's reference-signature entry points use. */
int hgs_current_device(int* device);

/* ---- graph store ---------------------------------------------------------
 * A in the reference's CsrMatrix layout (int64 row_ptr[n_rows+1],
 * col_idx[nnz], optional double values[nnz]; NULL values = edge-id matrix).
 * Requires n < 2^31, nnz < 2^31, columns within [0, n_cols). */
int hgs_graph_create(int device, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                     const int64_t* col_idx, const double* values, hgs_graph** out);
/* EventGraph features (data.hpp:17-27): node_feat[n*f_v], edge_feat[nnz*f_e]
 * in canonical edge (= CSR) order, labels[nnz]. */
int hgs_graph_attach_features(hgs_graph* g, const double* node_feat, int64_t f_v,
                              const double* edge_feat, int64_t f_e, const uint8_t* labels);
/* info: [0]=n_rows [1]=n_cols [2]=nnz [3]=walk nnz (sym) [4]=max walk degree (sym)
 *       [5]=max out-degree [6]=f_v [7]=f_e */
int hgs_graph_info(hgs_graph* g, int64_t* info);
/* Copy the device walk CSR (K0 output when symmetrize) to host int64 arrays:
 * row_ptr[n+1], col_idx[walk nnz]. */
int hgs_graph_walk(hgs_graph* g, int32_t symmetrize, int64_t* row_ptr, int64_t* col_idx);
int hgs_graph_destroy(hgs_graph* g);
/* Binary event files (the ingest path; the reference's
 * JSON read_event/write_event, data.cpp:270-368, are its slow twins): a
 * 64-byte-aligned header + sections row_ptr (int64, n+1), col_idx (int64,
 * nnz), values (f64, nnz; optional), node_feat (f64, n*f_v), edge_feat
 * (f64, nnz*f_e), labels (u8, nnz). hgs_graph_load mmaps the file and builds
 * the graph handle (device-side narrowing / validation for edge-id files)
 * with the features attached. info: n_rows, n_cols, nnz, f_v, f_e, flags. */
int hgs_event_save(const char* path, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                   const double* values, const double* node_feat, int64_t f_v, const double* edge_feat, int64_t f_e,
                   const uint8_t* labels);
int hgs_event_info(const char* path, int64_t* info);
int hgs_graph_load(int device, const char* path, hgs_graph** out);
/* gather_features for an arbitrary batch (sampler.cpp:211-243): node rows of
 * l2g[V] and edge rows / labels of edge ids eid[E] (input CSR positions) into
 * host xv[V*f_v], ye[E*f_e], lab[E]. Ids are range-checked (HGS_EINVAL). */
int hgs_graph_gather(hgs_graph* g, const int64_t* l2g, int64_t V, const int64_t* eid, int64_t E,
                     double* xv, double* ye, uint8_t* lab);

/* ---- sampling ------------------------------------------------------------- */
/* stream: a cudaStream_t (NULL = a stream owned by the handle). */
int hgs_sample_create(hgs_graph* g, void* stream, hgs_sample** out);
int hgs_sample_destroy(hgs_sample* s);
/* Re-bind a sample handle (its workspace and stream) to another graph on the
 * same device, e.g. to sample many resident events with a few handles. The
 * last run must have been waited for. */
int hgs_sample_bind(hgs_sample* s, hgs_graph* g);

/* bulk_shadow over batches given as flat roots[batch_off[n_batches]] with
 * batch_off[0] = 0 (host pointers). seeds[R]: per-root stream seeds
 * (PerRootChoiceSource / PhiloxChoiceSource seeds, root ordinal = flat index).
 * rng_state (nullable): resumes non-fresh sources — xoshiro: 4 u64 state
 * words per root; philox: 1 u64 per root = decisions already consumed.
 * Blocks until the results are ready. Limits (HGS_ERANGE): a root whose
 * induced subgraph has more than 32,767 vertices (the message names the
 * root ordinal), min(fanout, walk degree) > 2^24, more than 2^31-1 sampled
 * vertices or edges in one call. */
int hgs_sample_run(hgs_sample* s, const hgs_config* cfg, const int64_t* roots,
                   const int64_t* batch_off, int64_t n_batches, const uint64_t* seeds,
                   const uint64_t* rng_state);
/* One call over minibatches of several resident events (SURVEY.md §8(e),
 * multi-event launches): batch b samples graphs[batch_event[b]] (all graphs
 * on the handle's device; batch_event non-decreasing, so each event's batches
 * are contiguous; equal feature widths when gathering). Roots are checked
 * against their batch's event. Outputs as hgs_sample_run over the
 * concatenated batches; under per-root streams they equal one call per event
 * (the trainer's event loop, trainer.cpp:433-467). Each event's expand,
 * extract and pack kernels run on its own graph; offsets carry across events
 * on the device, so the call synchronises once. Blocks like hgs_sample_run. */
int hgs_sample_run_multi(hgs_sample* s, const hgs_config* cfg, hgs_graph* const* graphs, int32_t n_graphs,
                         const int32_t* batch_event, const int64_t* roots, const int64_t* batch_off,
                         int64_t n_batches, const uint64_t* seeds);
/* Same, with device-resident int32 roots[n_roots], int64 batch_off[n_batches+1]
 * and u64 seeds; enqueued asynchronously on the handle's stream. Roots are
 * range-checked on the device (reported by hgs_sample_wait); per-batch
 * distinctness is the caller's contract on this entry point. */
int hgs_sample_run_device(hgs_sample* s, const hgs_config* cfg, const int32_t* d_roots,
                          const int64_t* d_batch_off, int64_t n_roots, int64_t n_batches,
                          const uint64_t* d_seeds);
/* Per-root stream seeds derived on the device instead of
 * an uploaded seed array: the seed of flat root r, in batch bi at position
 * pos = r - batch_off[bi], is
 *     Rng::derive(seed, {path[0..path_len), batch_base + bi, pos})
 * (rng.cpp:76-85). The trainer's root_stream_seed (trainer.cpp:200-206) is
 * path = {0x73616d706c, epoch, event_ordinal} with batch_base = index of the
 * call's first batch in the epoch; the bench-sampling protocol
 * (cli.cpp:404-408) is path = {0x7374726d, k, rep}, batch_base = 0. */
typedef struct {
    uint64_t seed;
    uint64_t path[6];
    int32_t path_len;   /* 0..6 */
    int64_t batch_base;
} hgs_seed_spec;

/* hgs_sample_run_device with seeds from a hgs_seed_spec (no seed array). */
int hgs_sample_run_device_spec(hgs_sample* s, const hgs_config* cfg, const int32_t* d_roots,
                               const int64_t* d_batch_off, int64_t n_roots, int64_t n_batches,
                               const hgs_seed_spec* spec);
/* The same seeds on the host: out[batch_off[n_batches]] (host arrays). */
int hgs_derive_seeds(const hgs_seed_spec* spec, const int64_t* batch_off, int64_t n_batches, uint64_t* out);

/* Frontiers of the last run made with HGS_FLAG_KEEP_FRONTIERS (host arrays):
 * touched[R*stride] = per root its root then the chosen vertices of levels
 * 1..d in the reference's BFS order (touched[r*stride + i], i < tcount[r]),
 * level_counts[R*(depth+1)] = rows per level. *stride receives the stride. */
int hgs_sample_copy_frontiers(hgs_sample* s, int32_t* touched, int32_t* tcount, int32_t* level_counts,
                              int64_t* stride);

/* Wait for the last run; fills counts[0..3] = R, k, V, E (may be NULL).
 * A run whose edge slots or output buffers proved too small is re-run here
 * with exact sizes (counted by hgs_sample_reruns). For the run_device entry
 * points this means: the device inputs (roots, batch offsets, seeds) must stay
 * unchanged until hgs_sample_wait returns, and the outputs (device views) are
 * valid only after it returns. */
int hgs_sample_wait(hgs_sample* s, int64_t* counts);
int hgs_sample_copy_to_host(hgs_sample* s, const hgs_host_out* out);
int hgs_sample_device_views(hgs_sample* s, hgs_device_views* out);
/* Per-stage times (ms) of the last profiled run, from CUDA events on the
 * handle's stream: [0]=expand (K1) [1]=extract (K2) [2]=offset scan
 * [3]=pack+gather (K3) [4]=finalize [5]=total; HGS_EINVAL if not profiled. */
int hgs_sample_kernel_times(hgs_sample* s, float* ms6);
/* Work counters of the last run, reduced on the device (outside any timed
 * region): [0]=R [1]=k [2]=V [3]=E [4]=S (A entries scanned = sum of
 * out-degrees over all sampled vertices) [5]=sum of expanded frontier rows
 * (levels 0..d-1) [6]=sum of chosen children (levels 1..d) [7]=decisions
 * [8]=draws [9..9+d] = frontier rows per level 0..d. n >= 10 + depth. */
int hgs_sample_stats(hgs_sample* s, int64_t* stats, int32_t n);
/* Number of kernels the last run launched, re-runs included (for
 * gpu_launches accounting). */
int hgs_sample_launches(hgs_sample* s, int64_t* n);
/* Capacity re-runs the last run needed inside hgs_sample_wait (0 once the
 * handle's buffers fit the workload; timed steps must see 0). */
int hgs_sample_reruns(hgs_sample* s, int64_t* n);

/* ---- sample_rows ------------------------------------------------------------
 * hitgnn::sample_rows (sampler.hpp:60-66, sampler.cpp:64-86) on the device,
 * host arrays in and out. P: n_rows x n_cols CSR (values only checked for
 * negatives, as the reference does). For every row with a nonempty support,
 * k = min(s, |support|) distinct positions from choose(|support|, k) on
 * stream row_streams[r] — begin_root(row_streams[r]) is announced only for
 * nonempty rows, like the reference — sorted and mapped to the row's
 * columns. Rows on one stream are decided in row order; streams run in
 * parallel. seeds[n_streams]; rng_state as in hgs_sample_run (nullable).
 * Outputs: out_off[n_rows+1] (offsets of each row's choices), out_cols[...],
 * and per stream the RNG draws / choose calls consumed (nullable). More than
 * 2^24 choices per row is HGS_ERANGE. */
int hgs_sample_rows(int device, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                    const double* values, int64_t s, int32_t rng, const uint64_t* seeds, int64_t n_streams,
                    const uint64_t* rng_state, const int64_t* row_streams, int64_t* out_off, int64_t* out_cols,
                    uint32_t* draws, uint32_t* decisions);

/* ---- consumer --------------------------------------------
 * Device-resident counterparts of what the reference trainer does with a
 * sampled batch: slice_components (trainer.cpp:221-269, the DDP split of a
 * minibatch's components), the IGNN message-passing gathers and scatters
 * (Tape::gather_rows / scatter_add, autodiff.cpp:121-157, used at
 * ignn.cpp:158-164, and their backward passes, autodiff.cpp:260-281) and the
 * reduction step of the coalesced gradient all-reduce (allreduce_coalesced
 * -> InMemoryComm::allreduce_mean, trainer.cpp:84-123, 155-157). Device
 * pointers throughout; fp64 results are bit-identical with the reference
 * (sums in the reference's order, no floating-point atomics). */

/* One slice of a batch of the last run. e_row / e_col / comp_off /
 * roots_local are rebased to the slice (written by a kernel into buffers of
 * the sample handle, valid until its next slice or run); the other pointers
 * are views into the run's outputs (valid until its next run). */
typedef struct {
    int64_t n_vertices, n_edges, n_components, f_v, f_e;
    const int32_t *e_row, *e_col; /* [n_edges] slice-local endpoints, row-major */
    const int32_t* comp_off;      /* [n_components+1], comp_off[0] = 0 */
    const int32_t* roots_local;   /* [n_components] */
    const int32_t* l2g;           /* [n_vertices] */
    const int32_t* e_gid;         /* [n_edges] */
    const double *xv, *ye;        /* [n_vertices*f_v], [n_edges*f_e]; NULL without gather */
    const uint8_t* lab;           /* [n_edges]; NULL without gather */
} hgs_slice_views;

/* slice_components(batch `batch` of the last run, components [begin, end)):
 * HGS_EINVAL "slice_components: bad component range" as the reference.
 * Runs on the handle's stream and returns with the slice complete, so any
 * stream may consume it. */
int hgs_sample_slice(hgs_sample* s, int64_t batch, int64_t begin, int64_t end, hgs_slice_views* out);

/* Tape::gather_rows forward: out[i, :] = x[idx[i], :] for i < m (row-major
 * fp64 with `cols` columns). An index outside [0, n_rows) is HGS_EINVAL
 * "gather_rows: index <value> out of range" (the first in order; checked on
 * the device, so the call synchronizes `stream`). stream: a cudaStream_t. */
int hgs_gather_rows(const double* x, int64_t n_rows, int64_t cols, const int32_t* idx, int64_t m, double* out,
                    void* stream);

/* Tape::scatter_add: out[j, :] = sum of y[i, :] over i ascending with
 * idx[i] == j, rows of out without an index are 0; accumulate != 0 adds onto
 * out's current values in the same order (the backward of gather_rows,
 * autodiff.cpp:260-270). A plan = stable sort of idx + per-row segment
 * offsets, built once per index list (HGS_EINVAL "scatter_add: index
 * <value> out of range") and reused by forward and backward passes. */
typedef struct hgs_scatter_plan hgs_scatter_plan;
int hgs_scatter_plan_create(int device, const int32_t* idx, int64_t m, int64_t n_rows, void* stream,
                            hgs_scatter_plan** out);
int hgs_scatter_add(const hgs_scatter_plan* plan, const double* y, int64_t cols, double* out, int32_t accumulate,
                    void* stream);
int hgs_scatter_plan_destroy(hgs_scatter_plan* plan);
/* gather_rows over a plan's (already validated) index list: no range check,
 * no synchronisation. The index list must outlive the plan; a non-decreasing
 * list (e.g. a batch's rows) is planned without a sort. Plans and their
 * buffers are stream-ordered on the stream they were created on. */
int hgs_gather_rows_planned(const hgs_scatter_plan* plan, const double* x, int64_t n_rows, int64_t cols, double* out,
                            void* stream);

/* The reduction step of InMemoryComm::allreduce_mean: parts[q*n + e] is rank
 * q's element e (q < w); out[e] = (parts[0][e] + ... + parts[w-1][e]) * (1/w)
 * accumulated in rank order. The exchange around it (chunks to their owning
 * rank, reduced chunks back to every rank) is NCCL's. */
int hgs_ordered_mean(const double* parts, int32_t w, int64_t n, double* out, void* stream);

/* ---- RNG helpers (host, no GPU needed) -------------------------------------- */
uint64_t hgs_derive(uint64_t seed, const uint64_t* path, int32_t len);
void hgs_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

#ifdef __cplusplus
}
#endif
#endif
