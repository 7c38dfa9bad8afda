// host_types.cpp — host containers of the drop-in API: canonical COO/CSR
// conversion and the input validators, with the reference's semantics and
// exception texts (sparse.cpp:22-76, data.cpp:92-122, sampler.cpp:57-62).
#include <algorithm>
#include <string>

#include "hitgnn/core.hpp"

namespace hitgnn {

namespace {

std::string coord(Index r, Index c) { return "(" + std::to_string(r) + ", " + std::to_string(c) + ")"; }

bool coord_less(const CooEntry& x, const CooEntry& y) {
    return x.row != y.row ? x.row < y.row : x.col < y.col;
}

}  // namespace

void CooMatrix::canonicalize() {
    for (const CooEntry& e : entries)
        if (e.row < 0 || e.row >= n_rows || e.col < 0 || e.col >= n_cols)
            fail_invalid("CooMatrix: entry " + coord(e.row, e.col) + " out of range for " +
                         std::to_string(n_rows) + "x" + std::to_string(n_cols));
    std::sort(entries.begin(), entries.end(), coord_less);
    // Sum runs of equal coordinates in sorted order, then drop exact zeros.
    std::size_t w = 0;
    for (std::size_t i = 0; i < entries.size();) {
        CooEntry acc = entries[i++];
        while (i < entries.size() && entries[i].row == acc.row && entries[i].col == acc.col)
            acc.value += entries[i++].value;
        if (acc.value != 0.0) entries[w++] = acc;
    }
    entries.resize(w);
}

bool CooMatrix::is_canonical() const {
    const CooEntry* prev = nullptr;
    for (const CooEntry& e : entries) {
        if (e.row < 0 || e.row >= n_rows || e.col < 0 || e.col >= n_cols || e.value == 0.0) return false;
        if (prev && !coord_less(*prev, e)) return false;
        prev = &e;
    }
    return true;
}

CsrMatrix coo_to_csr(const CooMatrix& m) {
    if (!m.is_canonical())
        fail_invalid("coo_to_csr: input must be canonical (sorted, deduplicated, no explicit zeros)");
    CsrMatrix out(m.n_rows, m.n_cols);
    out.col_idx.resize(m.entries.size());
    out.values.resize(m.entries.size());
    std::size_t k = 0;
    for (const CooEntry& e : m.entries) {
        out.row_ptr[static_cast<std::size_t>(e.row) + 1] += 1;
        out.col_idx[k] = e.col;
        out.values[k] = e.value;
        ++k;
    }
    for (Index r = 0; r < m.n_rows; ++r) out.row_ptr[r + 1] += out.row_ptr[r];
    return out;
}

CooMatrix csr_to_coo(const CsrMatrix& m) {
    CooMatrix out{m.n_rows, m.n_cols, {}};
    out.entries.resize(static_cast<std::size_t>(m.nnz()));
    for (Index r = 0; r < m.n_rows; ++r)
        for (Index k = m.row_ptr[r]; k < m.row_ptr[r + 1]; ++k)
            out.entries[static_cast<std::size_t>(k)] = {r, m.col_idx[k], m.values[k]};
    return out;
}

void EventGraph::validate() const {
    if (n < 0) fail_invalid("EventGraph: negative vertex count");
    if (edges.n_rows != n || edges.n_cols != n)
        fail_invalid("EventGraph: adjacency shape does not match vertex count");
    if (!edges.is_canonical()) fail_invalid("EventGraph: edges not canonical");
    for (const CooEntry& e : edges.entries)
        if (e.row == e.col) fail_invalid("EventGraph: self-loop at vertex " + std::to_string(e.row));
    if (node_features.rows != n) fail_invalid("EventGraph: node feature rows != vertex count");
    if (edge_features.rows != m()) fail_invalid("EventGraph: edge feature rows != edge count");
    if (static_cast<Index>(labels.size()) != m()) fail_invalid("EventGraph: label count != edge count");
    if (std::any_of(labels.begin(), labels.end(), [](std::uint8_t l) { return l > 1; }))
        fail_invalid("EventGraph: labels must be 0 or 1");
}

void GenConfig::validate() const {
    if (n_tracks < 1) fail_invalid("GenConfig: n_tracks must be >= 1");
    if (hits_min < 1 || hits_max < hits_min)
        fail_invalid("GenConfig: hits range must satisfy 1 <= min <= max");
    if (hits_max > detector_layers)
        fail_invalid("GenConfig: infeasible geometry, more hits per track (" + std::to_string(hits_max) +
                     ") than detector layers (" + std::to_string(detector_layers) + ")");
    if (noise_hits < 0) fail_invalid("GenConfig: noise_hits must be >= 0");
    if (false_edge_factor < 0.0) fail_invalid("GenConfig: false_edge_factor must be >= 0");
    if (f_v < 3) fail_invalid("GenConfig: f_v must be >= 3 (spatial dims)");
    if (f_e < 1) fail_invalid("GenConfig: f_e must be >= 1");
}

void SamplerConfig::validate() const {
    if (depth < 1) fail_invalid("SamplerConfig: depth must be >= 1");
    if (fanout < 1) fail_invalid("SamplerConfig: fanout must be >= 1");
    if (batch_size < 1) fail_invalid("SamplerConfig: batch_size must be >= 1");
    if (bulk_batches < 1) fail_invalid("SamplerConfig: bulk_batches must be >= 1");
}

}  // namespace hitgnn
