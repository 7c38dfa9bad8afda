// ref_consumer_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper around the UNMODIFIED reference consumer code, compiled
// in place by oracle/Makefile from /root/reference/proj/src/{trainer,ignn,
// tracks,autodiff,...}.cpp with -Dhitgnn=hitgnn_ref (autodiff.cpp against
// oracle/eigen_shim, see there). Every result comes from the reference:
//   slice_components          trainer.cpp:221-269
//   Tape::gather_rows         autodiff.cpp:121-136 (+ backward :260-270)
//   Tape::scatter_add         autodiff.cpp:138-157 (+ backward :271-281)
//   allreduce_coalesced       trainer.cpp:155-157 -> InMemoryComm::allreduce_mean
//                             :84-123 on run_workers threads (:125-153)
// Used by tests/golden/make_consumer_golden.py to pin oracle/consumer.py and
// the device consumer kernels.
#include <algorithm>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "hitgnn/autodiff.hpp"
#include "hitgnn/sampler.hpp"
#include "hitgnn/trainer.hpp"

namespace R = hitgnn_ref;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

R::DenseMatrix dense(const double* p, int64_t r, int64_t c) {
    return R::DenseMatrix(r, c, std::vector<double>(p, p + r * c));
}
}  // namespace

extern "C" {

const char* refc_last_error() { return g_err.c_str(); }

// ---- slice_components over one SampledBatch given as flat arrays ----------
struct refc_batch {
    R::SampledBatch b;
};

// sizes: [0]=V [1]=E [2]=components [3]=f_v [4]=f_e
int refc_slice(int64_t nv, int64_t ne, int64_t nc, const int64_t* comp_off, const int64_t* l2g,
               const int64_t* roots_local, const int64_t* e_row, const int64_t* e_col, const double* e_val,
               const int64_t* e_gid, const double* xv, int64_t f_v, const double* ye, int64_t f_e,
               const uint8_t* lab, int64_t begin, int64_t end, refc_batch** out) {
    return guard([&] {
        R::SampledBatch in;
        in.adjacency.n_rows = in.adjacency.n_cols = nv;
        for (int64_t i = 0; i < ne; ++i) in.adjacency.entries.push_back({e_row[i], e_col[i], e_val[i]});
        in.component_offsets.assign(comp_off, comp_off + nc + 1);
        in.local_to_global.assign(l2g, l2g + nv);
        in.roots_local.assign(roots_local, roots_local + nc);
        if (xv) in.node_features = dense(xv, nv, f_v);
        if (ye) in.edge_features = dense(ye, ne, f_e);
        if (lab) in.edge_labels.assign(lab, lab + ne);
        if (e_gid) in.edge_global_ids.assign(e_gid, e_gid + ne);
        auto* h = new refc_batch{R::slice_components(in, begin, end)};
        *out = h;
    });
}

void refc_batch_sizes(const refc_batch* h, int64_t* s) {
    s[0] = h->b.n_vertices();
    s[1] = h->b.n_edges();
    s[2] = h->b.n_components();
    s[3] = h->b.node_features.cols;
    s[4] = h->b.edge_features.cols;
}

// any pointer may be NULL
void refc_batch_copy(const refc_batch* h, int64_t* comp_off, int64_t* l2g, int64_t* roots_local, int64_t* e_row,
                     int64_t* e_col, double* e_val, int64_t* e_gid, double* xv, double* ye, uint8_t* lab) {
    const R::SampledBatch& b = h->b;
    if (comp_off) std::copy(b.component_offsets.begin(), b.component_offsets.end(), comp_off);
    if (l2g) std::copy(b.local_to_global.begin(), b.local_to_global.end(), l2g);
    if (roots_local) std::copy(b.roots_local.begin(), b.roots_local.end(), roots_local);
    for (size_t i = 0; i < b.adjacency.entries.size(); ++i) {
        if (e_row) e_row[i] = b.adjacency.entries[i].row;
        if (e_col) e_col[i] = b.adjacency.entries[i].col;
        if (e_val) e_val[i] = b.adjacency.entries[i].value;
    }
    if (e_gid) std::copy(b.edge_global_ids.begin(), b.edge_global_ids.end(), e_gid);
    if (xv) std::copy(b.node_features.data.begin(), b.node_features.data.end(), xv);
    if (ye) std::copy(b.edge_features.data.begin(), b.edge_features.data.end(), ye);
    if (lab) std::copy(b.edge_labels.begin(), b.edge_labels.end(), lab);
}

void refc_batch_free(refc_batch* h) { delete h; }

// ---- Tape::gather_rows / scatter_add, forward and backward ----------------
int refc_gather_rows(const double* x, int64_t n, int64_t c, const int64_t* idx, int64_t m, double* out) {
    return guard([&] {
        R::Tape t;
        const R::Tensor g = t.gather_rows(t.input(dense(x, n, c)), std::vector<R::Index>(idx, idx + m));
        const R::DenseMatrix& v = t.value(g);
        std::copy(v.data.begin(), v.data.end(), out);
    });
}

int refc_scatter_add(const double* y, int64_t m, int64_t c, const int64_t* idx, int64_t n, double* out) {
    return guard([&] {
        R::Tape t;
        const R::Tensor s = t.scatter_add(t.input(dense(y, m, c)), std::vector<R::Index>(idx, idx + m), n);
        const R::DenseMatrix& v = t.value(s);
        std::copy(v.data.begin(), v.data.end(), out);
    });
}

// The op's output feeds linear(W[c,1], b) -> bce_with_logits(labels) so that
// each output row receives a different gradient; returns that incoming
// gradient g_out and the op's input gradient g_in, both from the reference tape.
// op 0: x[n,c] -> gather_rows(idx[m]) -> [m,c]; op 1: y[m,c] -> scatter_add(idx[m], n) -> [n,c]
int refc_backward(int32_t op, const double* in, int64_t rows_in, int64_t c, const int64_t* idx, int64_t m, int64_t n,
                  const double* w, const uint8_t* labels, double* g_out, double* g_in) {
    return guard([&] {
        R::Tape t;
        const R::Tensor x = t.input(dense(in, rows_in, c), true);
        const std::vector<R::Index> iv(idx, idx + m);
        const R::Tensor o = op == 0 ? t.gather_rows(x, iv) : t.scatter_add(x, iv, n);
        const int64_t ro = op == 0 ? m : n;
        const R::Tensor wt = t.input(dense(w, c, 1), false);
        const R::Tensor bt = t.input(R::DenseMatrix(1, 1), false);
        const R::Tensor logits = t.linear(o, wt, bt);
        const R::Tensor loss = t.bce_with_logits(logits, std::vector<uint8_t>(labels, labels + ro));
        t.backward(loss);
        const R::DenseMatrix go = t.grad(o), gi = t.grad(x);
        std::copy(go.data.begin(), go.data.end(), g_out);
        std::copy(gi.data.begin(), gi.data.end(), g_in);
    });
}

// ---- allreduce_coalesced over world_size worker threads, in place ----------
int refc_allreduce(int32_t world, double* bufs, int64_t n) {
    return guard([&] {
        R::InMemoryComm comm(world);
        R::run_workers(world, [&](int rank) {
            const R::CommHandle h{&comm, rank};
            R::allreduce_coalesced(std::span<double>(bufs + (size_t)rank * n, (size_t)n), h);
        });
    });
}

}  // extern "C"
