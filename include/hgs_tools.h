/*
 * hgs_tools.h — C entry points of libhitgnn_gpu.so used by the Python
 * harnesses (bench, tests). Not part of the sampler boundary (hgs.h).
 *
 * hgs_generate_event: the synthetic TrackML-shaped event generator
 * (hitgnn::generate_event; reference data.cpp:124-268) returning the
 * make_edge_id_matrix CSR (sampler.cpp:203-209) and features.
 */
#ifndef HGS_TOOLS_H
#define HGS_TOOLS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct hgs_event hgs_event;

/* Returns 0 on success; message via hgs_tools_last_error(). */
int hgs_generate_event(int64_t n_tracks, int64_t hits_min, int64_t hits_max, int64_t layers,
                       int64_t noise_hits, double false_edge_factor, int64_t f_v, int64_t f_e,
                       uint64_t seed, uint64_t event_id, hgs_event** out);
/* The scalable variant (not in the reference): false-edge candidates from a
 * phi window of half-width phi_window (reference: 0.45), so the work per hit
 * stays constant as layers fill up (~1M hits). */
int hgs_generate_event_windowed(int64_t n_tracks, int64_t hits_min, int64_t hits_max, int64_t layers,
                                int64_t noise_hits, double false_edge_factor, int64_t f_v, int64_t f_e,
                                uint64_t seed, uint64_t event_id, double phi_window, hgs_event** out);
/* sizes: [0]=n [1]=m [2]=f_v [3]=f_e */
void hgs_event_sizes(const hgs_event* ev, int64_t* sizes);
/* row_ptr[n+1], col_idx[m] (make_edge_id_matrix CSR), node_feat[n*f_v],
 * edge_feat[m*f_e], labels[m]; any pointer may be NULL. */
void hgs_event_copy(const hgs_event* ev, int64_t* row_ptr, int64_t* col_idx, double* node_feat,
                    double* edge_feat, uint8_t* labels);
void hgs_event_free(hgs_event* ev);
const char* hgs_tools_last_error(void);

/* End-to-end timing of the C++ drop-in (host arrays in, std::vector<SampledBatch>
 * with gathered features out): mode 0 = gpu::DeviceEvent::bulk_shadow(gather),
 * mode 1 = the reference trainer's bulk_shadow + per-batch gather_features
 * (trainer.cpp:457-458). seconds[reps] wall clock per rep; ve = {V, E}. */
int hgs_dropin_time(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* node_feat,
                    int64_t f_v, const double* edge_feat, int64_t f_e, const uint8_t* labels,
                    const int64_t* roots, const int64_t* batch_off, int64_t n_batches, const uint64_t* seeds,
                    int64_t depth, int64_t fanout, int32_t mode, int32_t warmup, int32_t reps, double* seconds,
                    int64_t* ve);

/* epoch_root_batches (sampler.cpp:245-263) with Rng(rng_seed): writes the
 * shuffled permutation of [0, n) to perm; returns the number of batches. */
int64_t hgs_epoch_root_batches(int64_t n, int64_t batch_size, uint64_t rng_seed, int64_t* perm);
/* seeds[bi*b + pos] = Rng::derive(seed, prefix ++ {bi, pos}) for bi < k, pos < b
 * (bench protocol cli.cpp:401-408, trainer root_stream_seed trainer.cpp:200-206). */
void hgs_derive_grid(uint64_t seed, const uint64_t* prefix, int32_t prefix_len, int64_t k,
                     int64_t b, uint64_t* seeds);

/* The drop-in hitgnn::bulk_shadow (GPU) with a FrontierObserver recording
 * each level's FrontierSet; arrays per level: which = 0 Q col_idx, 1 F
 * row_ptr, 2 F col_idx, 3 P row_ptr, 4 P col_idx (int64), 5 P values (f64).
 * rng: 0 PerRootChoiceSource, 1 PhiloxChoiceSource. values NULL = edge ids. */
typedef struct hgs_frontiers hgs_frontiers;
int hgs_tools_frontiers(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                        const double* values, const int64_t* roots, const int64_t* batch_off, int64_t n_batches,
                        const uint64_t* seeds, int32_t rng, int64_t depth, int64_t fanout, int32_t symmetrize,
                        hgs_frontiers** out);
int64_t hgs_tools_frontiers_levels(const hgs_frontiers* f);
int64_t hgs_tools_frontier_array(const hgs_frontiers* f, int64_t level, int32_t which, void* out);
void hgs_tools_frontiers_free(hgs_frontiers* f);

#ifdef __cplusplus
}
#endif
#endif
