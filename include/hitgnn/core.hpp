// hitgnn/core.hpp — source-compatible drop-in for the reference sampler API,
// backed by the B200 device path (libhgs, include/hgs.h).
//
// Declares, in namespace hitgnn, the types and functions a caller of the
// reference hot path uses (reference headers in /root/reference/proj/include):
//   types.hpp   Index, fail_invalid, fail_state                  (types.hpp:9-17)
//   dense.hpp   DenseMatrix                                       (dense.hpp:12-44)
//   sparse.hpp  CooEntry, CooMatrix, CsrMatrix, coo_to_csr,
//               csr_to_coo, symmetrize_pattern                    (sparse.hpp:11-98)
//   rng.hpp     Rng, ChoiceSource, RandomChoiceSource,
//               PerRootChoiceSource                               (rng.hpp:12-82)
//   data.hpp    EventGraph, GenConfig, generate_event             (data.hpp:17-45)
//   sampler.hpp SamplerConfig, SampledBatch, FrontierSet,
//               FrontierObserver, bulk_shadow, shadow_reference,
//               gather_features, make_edge_id_matrix,
//               epoch_root_batches                                (sampler.hpp:16-102)
// Additions: PhiloxChoiceSource (counter-based streams),
// seed/state accessors on the per-root sources, and hitgnn::gpu::DeviceEvent
// for keeping an event resident on the GPU across calls.
//
// Source-compatible, not ABI-compatible with objects built against the
// reference headers. The per-file headers under hitgnn/ forward here.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <initializer_list>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace hitgnn {

// ---- types -------------------------------------------------------------------
using Index = std::int64_t;
[[noreturn]] inline void fail_invalid(const std::string& m) { throw std::invalid_argument(m); }
[[noreturn]] inline void fail_state(const std::string& m) { throw std::runtime_error(m); }

// ---- dense --------------------------------------------------------------------
struct DenseMatrix {
    Index rows = 0;
    Index cols = 0;
    std::vector<double> data;

    DenseMatrix() = default;
    DenseMatrix(Index r, Index c) : rows(r), cols(c) {
        if (r < 0 || c < 0) fail_invalid("DenseMatrix: negative dimension");
        data.assign(size(), 0.0);
    }
    DenseMatrix(Index r, Index c, std::vector<double> d) : rows(r), cols(c), data(std::move(d)) {
        if (static_cast<std::size_t>(r * c) != data.size())
            fail_invalid("DenseMatrix: data length does not match shape");
    }
    std::size_t size() const { return static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols); }
    double& at(Index i, Index j) { return data[static_cast<std::size_t>(i * cols + j)]; }
    double at(Index i, Index j) const { return data[static_cast<std::size_t>(i * cols + j)]; }
    double* row_ptr(Index i) { return data.data() + i * cols; }
    const double* row_ptr(Index i) const { return data.data() + i * cols; }
    bool all_finite() const {
        for (double v : data)
            if (!std::isfinite(v)) return false;
        return true;
    }
    bool operator==(const DenseMatrix&) const = default;
};

// ---- sparse -------------------------------------------------------------------
struct CooEntry {
    Index row = 0;
    Index col = 0;
    double value = 0.0;
    friend bool operator==(const CooEntry&, const CooEntry&) = default;
};

struct CooMatrix {
    Index n_rows = 0;
    Index n_cols = 0;
    std::vector<CooEntry> entries;
    Index nnz() const { return static_cast<Index>(entries.size()); }
    void canonicalize();
    bool is_canonical() const;
    friend bool operator==(const CooMatrix&, const CooMatrix&) = default;
};

struct CsrMatrix {
    Index n_rows = 0;
    Index n_cols = 0;
    std::vector<Index> row_ptr;
    std::vector<Index> col_idx;
    std::vector<double> values;

    CsrMatrix() : row_ptr(1, 0) {}
    CsrMatrix(Index rows, Index cols)
        : n_rows(rows), n_cols(cols), row_ptr(static_cast<std::size_t>(rows) + 1, 0) {}
    Index nnz() const { return static_cast<Index>(col_idx.size()); }
    Index row_nnz(Index r) const { return row_ptr[r + 1] - row_ptr[r]; }
    std::span<const Index> row_cols(Index r) const {
        return {col_idx.data() + row_ptr[r], static_cast<std::size_t>(row_nnz(r))};
    }
    std::span<const double> row_values(Index r) const {
        return {values.data() + row_ptr[r], static_cast<std::size_t>(row_nnz(r))};
    }
    friend bool operator==(const CsrMatrix&, const CsrMatrix&) = default;
};

CsrMatrix coo_to_csr(const CooMatrix& m);
CooMatrix csr_to_coo(const CsrMatrix& m);
// Pattern of A ∪ Aᵀ with unit values, computed by the device K0 kernels.
CsrMatrix symmetrize_pattern(const CsrMatrix& a);

// ---- rng ------------------------------------------------------------------------
class Rng {
public:
    explicit Rng(std::uint64_t seed);
    std::uint64_t next_u64();
    std::uint64_t bounded(std::uint64_t n);
    double uniform();
    double uniform(double lo, double hi);
    double normal();
    static std::uint64_t derive(std::uint64_t seed, std::initializer_list<std::uint64_t> path);
    // additions: raw xoshiro256** state (4 words)
    const std::uint64_t* state() const { return s_; }

private:
    std::uint64_t s_[4];
    double spare_ = 0.0;
    bool has_spare_ = false;
};

class ChoiceSource {
public:
    virtual ~ChoiceSource() = default;
    virtual std::vector<std::uint32_t> choose(std::uint32_t n_options, std::uint32_t k) = 0;
    virtual void begin_root(std::uint64_t /*root_ordinal*/) {}
};

class RandomChoiceSource final : public ChoiceSource {
public:
    explicit RandomChoiceSource(std::uint64_t seed) : rng_(seed) {}
    explicit RandomChoiceSource(Rng rng) : rng_(rng) {}
    std::vector<std::uint32_t> choose(std::uint32_t n_options, std::uint32_t k) override;
    Rng& rng() { return rng_; }

private:
    Rng rng_;
};

// One xoshiro256** stream per root, resumed across levels (rng.hpp:67-82).
// The device path reads seeds()/states() and writes back consumed draws.
class PerRootChoiceSource final : public ChoiceSource {
public:
    explicit PerRootChoiceSource(std::vector<std::uint64_t> stream_seeds);
    void begin_root(std::uint64_t root_ordinal) override;
    std::vector<std::uint32_t> choose(std::uint32_t n_options, std::uint32_t k) override;

    std::size_t size() const { return seeds_.size(); }
    const std::vector<std::uint64_t>& seeds() const { return seeds_; }
    bool fresh() const { return fresh_; }
    std::size_t current() const { return current_; }
    // 4 state words per root (materialises pending device advances).
    std::vector<std::uint64_t> states();
    // Record that the device consumed draws[r] outputs of every stream r.
    void advance(std::span<const std::uint32_t> draws);

private:
    void settle(std::size_t r);
    std::vector<std::uint64_t> seeds_;
    std::vector<RandomChoiceSource> streams_;
    std::vector<std::uint64_t> pending_;  // device draws not yet replayed on the host
    std::size_t current_ = 0;
    bool fresh_ = true;
};

// Counter-based per-root streams: decision c of root r draws step i, attempt
// a from Philox4x32-10(key = seed_r, ctr = {c, i, a, 0x43484f53}) (SURVEY.md
// Appendix A.3). Decisions are independent, so the device can evaluate them
// in any order; the outcome equals this class's sequential use.
class PhiloxChoiceSource final : public ChoiceSource {
public:
    explicit PhiloxChoiceSource(std::vector<std::uint64_t> stream_seeds);
    void begin_root(std::uint64_t root_ordinal) override;
    std::vector<std::uint32_t> choose(std::uint32_t n_options, std::uint32_t k) override;

    std::size_t size() const { return seeds_.size(); }
    const std::vector<std::uint64_t>& seeds() const { return seeds_; }
    const std::vector<std::uint64_t>& decisions() const { return decisions_; }
    bool fresh() const { return fresh_; }
    std::size_t current() const { return current_; }
    void advance(std::span<const std::uint32_t> decisions);

private:
    std::vector<std::uint64_t> seeds_;
    std::vector<std::uint64_t> decisions_;
    std::size_t current_ = 0;
    bool fresh_ = true;
};

// ---- data -------------------------------------------------------------------------
struct EventGraph {
    std::uint64_t event_id = 0;
    Index n = 0;
    CooMatrix edges;
    DenseMatrix node_features;
    DenseMatrix edge_features;
    std::vector<std::uint8_t> labels;
    Index m() const { return edges.nnz(); }
    void validate() const;
};

struct GenConfig {
    Index n_tracks = 110;
    Index hits_min = 7;
    Index hits_max = 10;
    Index detector_layers = 12;
    Index noise_hits = 65;
    double false_edge_factor = 1.0;
    Index f_v = 6;
    Index f_e = 2;
    std::uint64_t seed = 1;
    void validate() const;
};

// Synthetic TrackML-like event (the reference generator's semantics,
// data.cpp:124-268), with a phi-window sweep instead of the all-pairs
// candidate scan so million-hit events are feasible. Bit-identical output.
EventGraph generate_event(const GenConfig& cfg, std::uint64_t event_id);
// Scalable variant (not in the reference): false-edge candidates from a phi
// window of half-width phi_window (the reference's is 0.45); see eventgen.cpp.
EventGraph generate_event_windowed(const GenConfig& cfg, std::uint64_t event_id, double phi_window);

// ---- sampler ----------------------------------------------------------------------
struct SamplerConfig {
    Index depth = 3;
    Index fanout = 6;
    Index batch_size = 256;
    Index bulk_batches = 1;
    bool symmetrize = true;
    void validate() const;
};

struct SampledBatch {
    CooMatrix adjacency;
    std::vector<Index> component_offsets;
    std::vector<Index> local_to_global;
    std::vector<Index> roots_local;
    DenseMatrix node_features;
    DenseMatrix edge_features;
    std::vector<std::uint8_t> edge_labels;
    std::vector<Index> edge_global_ids;

    Index n_vertices() const { return adjacency.n_rows; }
    Index n_edges() const { return adjacency.nnz(); }
    Index n_components() const { return static_cast<Index>(component_offsets.size()) - 1; }
};

struct FrontierSet {
    CsrMatrix q;
    CsrMatrix f;
    CsrMatrix p;
};
using FrontierObserver = std::function<void(Index level, const FrontierSet&)>;

// Device-path entry points. The ChoiceSource must be a PerRootChoiceSource
// or a PhiloxChoiceSource (anything else: std::invalid_argument — there is
// no host fallback); it is advanced exactly as the reference would.
std::vector<SampledBatch> bulk_shadow(const CsrMatrix& a,
                                      const std::vector<std::vector<Index>>& batches,
                                      const SamplerConfig& cfg, ChoiceSource& choice,
                                      const FrontierObserver& observer = {});
SampledBatch shadow_reference(const CsrMatrix& a, std::span<const Index> roots,
                              const SamplerConfig& cfg, ChoiceSource& choice);
void gather_features(SampledBatch& batch, const EventGraph& event);
CsrMatrix make_edge_id_matrix(const EventGraph& event);
// sample_rows (reference sampler.hpp:60-66) on the GPU (hgs_sample_rows).
std::vector<std::vector<Index>> sample_rows(const CsrMatrix& p, Index s, ChoiceSource& choice,
                                            std::span<const Index> row_streams = {});
std::vector<std::vector<Index>> epoch_root_batches(Index n_vertices, Index batch_size, Rng& rng);

namespace gpu {

// Resident-graph cache behind the reference-signature entry points.
// bulk_shadow / shadow_reference (A) and gather_features (the event's
// features) keep what they upload on the calling thread's current CUDA
// device, so the reference's call pattern (trainer.cpp:457-458: the same
// edge-id matrix and EventGraph every chunk) uploads each event once.
//   A: keyed by device, object address, array pointers, sizes and a full
//      content hash of row_ptr / col_idx / values (checked on every call).
//   event: keyed by device, address, array pointers, sizes and a sampled
//      content fingerprint (4,096 strided elements + both ends of every
//      array); an EventGraph mutated in place at other positions must be
//      released (release_cached) or HGS_DROPIN_VERIFY=full set (full hash).
// Up to 16 entries, least recently used evicted; HGS_DROPIN_CACHE=0 disables
// the cache (upload per call, the pre-cache behaviour).
void release_cached();
std::size_t cached_entries();
// Gather prefetch (the trainer's two lines, trainer.cpp:457-458): once the
// event is resident with its features (after any gather_features call),
// bulk_shadow(edge-id A) gathers on the device as it samples, and the
// following gather_features(batch, event) calls on the same thread take the
// prebuilt features. Returns how many gather_features calls on this thread
// were served that way.
std::size_t prefetched_gathers();

// An event resident on one GPU: A (edge ids), walk, features. Create once per
// event (next to make_edge_id_matrix in Trainer's constructor) and sample
// from it repeatedly; bulk_shadow(..., gather = true) returns batches with
// features already gathered (== bulk_shadow + gather_features).
class DeviceEvent {
public:
    DeviceEvent(const EventGraph& event, int device = 0);
    DeviceEvent(const CsrMatrix& a, int device = 0);  // no features
    ~DeviceEvent();
    DeviceEvent(const DeviceEvent&) = delete;
    DeviceEvent& operator=(const DeviceEvent&) = delete;

    std::vector<SampledBatch> bulk_shadow(const std::vector<std::vector<Index>>& batches,
                                          const SamplerConfig& cfg, ChoiceSource& choice,
                                          bool gather = false,
                                          const FrontierObserver& observer = {});
    Index n() const { return n_; }
    int device() const { return device_; }
    void* handle() const { return graph_; }

private:
    void* graph_ = nullptr;    // hgs_graph*
    void* sampler_ = nullptr;  // hgs_sample*
    Index n_ = 0, nnz_ = 0, f_v_ = 0, f_e_ = 0;
    int device_ = 0;
    std::vector<double> values_;  // non-id values of a general A (may be empty)
    bool ids_ = true;
    std::unique_ptr<CsrMatrix> host_a_;  // host copy of A for FrontierObserver's P
};

}  // namespace gpu
}  // namespace hitgnn
