// TEST INFRASTRUCTURE ONLY — C-ABI wrapper around the untouched reference
// headers (/root/reference/proj/include/ttsvd/*.hpp), compiled by
// oracle/Makefile into oracle/_ref/libttsvd_ref.so.  It pins the C restatement
// (oracle/ttsvd_oracle.c) and is the "reference" CPU baseline in bench.py.
// No reference source is copied: this file only #includes the headers where
// they lie.  Signatures mirror the orc_* functions of the restatement.
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "ttsvd/tt_svd.hpp"
#include "oracles.hpp"  // reference tests' input generators (proj/tests/oracles.hpp)

using namespace ttsvd;

namespace {

int code_of(const std::exception& e) {
    if (dynamic_cast<const DimensionError*>(&e)) return 1;
    if (dynamic_cast<const DimensionMismatch*>(&e)) return 2;
    if (dynamic_cast<const ShapeError*>(&e)) return 3;
    if (dynamic_cast<const ConvergenceError*>(&e)) return 4;
    if (dynamic_cast<const AllocationError*>(&e)) return 5;
    if (dynamic_cast<const DegenerateDimension*>(&e)) return 6;
    if (dynamic_cast<const PartitionMismatch*>(&e)) return 7;
    if (dynamic_cast<const IoError*>(&e)) return 9;
    if (dynamic_cast<const LayoutError*>(&e)) return 10;
    return 12;
}

TruncationSpec spec_of(int64_t r_max, double eps) {
    TruncationSpec s;
    s.r_max = r_max;
    s.eps = eps;
    return s;
}

DenseTensor tensor_from(const double* X, const int64_t* dims, int64_t d, int64_t ldx) {
    DenseTensor t{Shape(std::vector<index_t>(dims, dims + d))};
    const index_t rows = t.rows();
    const index_t cols = t.total() / rows;
    for (index_t j = 0; j < cols; ++j) std::memcpy(t.data() + j * t.leading_stride(), X + j * ldx, rows * 8);
    return t;
}

int export_tt(const TensorTrain& tt, int64_t* ranks, double* cores, int64_t cap, int64_t* needed) {
    const auto r = tt.ranks();
    for (std::size_t j = 0; j < r.size(); ++j) ranks[j] = r[j];
    int64_t need = 0;
    for (const auto& c : tt.cores) need += static_cast<int64_t>(c.data.size());
    if (needed) *needed = need;
    if (need > cap) return 11;
    int64_t off = 0;
    for (const auto& c : tt.cores) {
        std::memcpy(cores + off, c.data.data(), c.data.size() * 8);
        off += static_cast<int64_t>(c.data.size());
    }
    return 0;
}

struct StepOut {
    int64_t rows, cols, nsig, rank;
};

void export_steps(const RunRecorder& rec, StepOut* steps) {
    if (!steps) return;
    for (std::size_t i = 0; i < rec.steps.size(); ++i) {
        steps[i].rows = rec.steps[i].rows;
        steps[i].cols = rec.steps[i].cols;
        steps[i].nsig = 0;
        steps[i].rank = rec.steps[i].rank;
    }
}

} // namespace

extern "C" {

void ref_set_budget(int64_t bytes) { memory_budget_bytes().store(bytes); }

int64_t ref_padded_stride(int64_t n) {
    try { return padded_stride(n); } catch (const std::exception&) { return -1; }
}

int64_t ref_block_nb(int64_t m, int64_t budget) { return BlockParams::for_cols(m, budget).n_b; }

int ref_reduce_block(const double* M, int64_t rows, int64_t m, int64_t ldm, const double* R_in, int64_t r_m,
                     double* R_out) {
    try {
        TriangularFactor R(r_m);
        std::memcpy(R.entries.data(), R_in, r_m * r_m * 8);
        BlockParams p;
        p.validate_reflectors = false;
        TriangularFactor o = reduce_block(ConstMatrixView{M, rows, m, ldm}, R, p);
        std::memcpy(R_out, o.entries.data(), m * m * 8);
        return 0;
    } catch (const std::exception& e) { return code_of(e); }
}

int ref_combine_factors(const double* parts, int64_t P, int64_t m, double* R) {
    try {
        std::vector<TriangularFactor> v;
        for (int64_t p = 0; p < P; ++p) {
            TriangularFactor t(m);
            std::memcpy(t.entries.data(), parts + p * m * m, m * m * 8);
            v.push_back(std::move(t));
        }
        BlockParams bp;
        bp.validate_reflectors = false;
        TriangularFactor o = combine_factors(v, bp);
        std::memcpy(R, o.entries.data(), m * m * 8);
        return 0;
    } catch (const std::exception& e) { return code_of(e); }
}

int ref_tsqr(const double* X, int64_t n, int64_t m, int64_t ldx, int64_t n_b, int workers, double* R) {
    try {
        BlockParams p;
        p.n_b = n_b;
        p.validate_reflectors = false;
        TriangularFactor o = tsqr(ConstMatrixView{X, n, m, ldx}, p, workers);
        std::memcpy(R, o.entries.data(), m * m * 8);
        return 0;
    } catch (const std::exception& e) { return code_of(e); }
}

int ref_jacobi_svd(const double* A, int64_t n, int64_t m, int64_t lda, double* sigma, double* U, double* V) {
    try {
        SmallSVD s = jacobi_svd(ConstMatrixView{A, n, m, lda});
        std::memcpy(sigma, s.sigma.data(), m * 8);
        if (U) std::memcpy(U, s.U.data(), n * m * 8);
        std::memcpy(V, s.V.data(), m * m * 8);
        return 0;
    } catch (const std::exception& e) { return code_of(e); }
}

int64_t ref_select_rank(const double* sigma, int64_t m, double delta, int64_t r_max) {
    return select_rank(std::vector<double>(sigma, sigma + m), delta, r_max);
}

int ref_derive_delta(double norm, double eps, int64_t d, double* out) {
    try { *out = derive_delta(norm, eps, d); return 0; } catch (const std::exception& e) { return code_of(e); }
}

int ref_tsmm_reshape(const double* X, int64_t n, int64_t m, int64_t ldx, const double* V, int64_t k, int64_t ldv,
                     double* Y, int64_t out_rows, int64_t out_cols, int64_t ldy, int workers) {
    try {
        PaddedMatrix o = tsmm_reshape(ConstMatrixView{X, n, m, ldx}, ConstMatrixView{V, m, k, ldv}, out_rows,
                                      out_cols, workers);
        if (o.stride() != ldy) return 3;
        std::memcpy(Y, o.data(), o.stride() * out_cols * 8);
        return 0;
    } catch (const std::exception& e) { return code_of(e); }
}

int ref_tt_svd_tsqr(const double* X, const int64_t* dims, int64_t d, int64_t ldx, int64_t r_max, double eps,
                    int workers, int64_t* ranks, double* cores, int64_t cap, int64_t* needed, StepOut* steps) {
    try {
        DenseTensor t = tensor_from(X, dims, d, ldx);
        RunRecorder rec;
        ExecContext ctx;
        ctx.threads = workers;
        ctx.validate_reflectors = false;
        ctx.recorder = &rec;
        TensorTrain tt = tt_svd_tsqr(t, spec_of(r_max, eps), ctx);
        export_steps(rec, steps);
        return export_tt(tt, ranks, cores, cap, needed);
    } catch (const std::exception& e) { return code_of(e); }
}

// The reference's own Alg. 2 steps (tt_svd.hpp:159-199), called one by one
// from this test driver so that every step's singular values can be recorded
// (tt_svd_tsqr does not expose them): detail::svd_of_work, derive_delta,
// detail::choose_rank, detail::core_from_vt, tsmm_reshape, all with
// ctx.threads workers.  tests/test_oracle_pin.py pins it bitwise to
// tt_svd_tsqr.  sigmas: the concatenated sigma of every step (nsig each,
// in execution order; cap doubles), nsig_out: per step.
int ref_tt_svd_tsqr_sigma(const double* X, const int64_t* dims, int64_t d, int64_t ldx, int64_t r_max, double eps,
                          int workers, int64_t* ranks, double* cores, int64_t cap, int64_t* needed, double* sigmas,
                          int64_t sig_cap, int64_t* nsig_out) {
    try {
        if (d < 2) throw DegenerateDimension("tt_svd_tsqr: requires d >= 2");
        DenseTensor t = tensor_from(X, dims, d, ldx);
        ExecContext ctx;
        ctx.threads = workers;
        ctx.validate_reflectors = false;
        TruncationSpec spec = spec_of(r_max, eps);
        std::vector<index_t> dv(dims, dims + d);
        std::vector<TTCore> cs(static_cast<std::size_t>(d));
        PaddedMatrix owned;
        ConstMatrixView cur{t.data(), t.rows(), dims[d - 1], t.leading_stride()};
        index_t r = 1;
        int64_t soff = 0;
        for (index_t i = d - 1; i >= 1; --i) {
            const index_t n_i = dv[static_cast<std::size_t>(i)];
            detail::WorkSVD s = detail::svd_of_work(cur, ctx, nullptr);
            if (!spec.has_delta()) spec.delta = derive_delta(sigma_norm(s.sigma), spec.eps, d);
            const index_t rnew = detail::choose_rank(s, spec, cur.rows);
            nsig_out[d - 1 - i] = s.nsig;
            if (soff + s.nsig <= sig_cap) std::memcpy(sigmas + soff, s.sigma.data(), s.nsig * 8);
            soff += s.nsig;
            cs[static_cast<std::size_t>(i)] = detail::core_from_vt(s, rnew, n_i, r);
            const index_t n_next = dv[static_cast<std::size_t>(i - 1)];
            owned = tsmm_reshape(cur, s.v_view(rnew), cur.rows / n_next, n_next * rnew, ctx.threads, nullptr);
            cur = owned.view();
            r = rnew;
        }
        TTCore first(1, dv[0], r);
        for (index_t l = 0; l < dv[0] * r; ++l) first.data[static_cast<std::size_t>(l)] = cur(l % cur.rows, l / cur.rows);
        cs[0] = std::move(first);
        TensorTrain tt;
        tt.cores = std::move(cs);
        if (soff > sig_cap) return 11;
        return export_tt(tt, ranks, cores, cap, needed);
    } catch (const std::exception& e) { return code_of(e); }
}

// tt_svd.hpp:316-330 and tt_svd.hpp:338 (Alg. 3)
int ref_choose_combined_dims(const int64_t* dims, int64_t d, int64_t m_min, double f1_min, const int64_t* r_tilde,
                             int64_t n_r_tilde, int64_t r_max, int64_t* k_out, int64_t* m_out) {
    try {
        ThickBoundsParams p;
        p.m_min = m_min;
        p.f1_min = f1_min;
        if (r_tilde) p.r_tilde.assign(r_tilde, r_tilde + n_r_tilde);
        const auto km = choose_combined_dims(Shape(std::vector<index_t>(dims, dims + d)), p, r_max);
        *k_out = km.first;
        *m_out = km.second;
        return 0;
    } catch (const std::exception& e) { return code_of(e); }
}

int ref_tt_svd_thick_bounds(const double* X, const int64_t* dims, int64_t d, int64_t ldx, int64_t r_max, double eps,
                            int64_t m_min, double f1_min, const int64_t* r_tilde, int64_t n_r_tilde, int workers,
                            int64_t* ranks, double* cores, int64_t cap, int64_t* needed) {
    try {
        DenseTensor t = tensor_from(X, dims, d, ldx);
        ThickBoundsParams p;
        p.m_min = m_min;
        p.f1_min = f1_min;
        if (r_tilde) p.r_tilde.assign(r_tilde, r_tilde + n_r_tilde);
        ExecContext ctx;
        ctx.threads = workers;
        ctx.validate_reflectors = false;
        TensorTrain tt = tt_svd_thick_bounds(t, spec_of(r_max, eps), p, ctx);
        return export_tt(tt, ranks, cores, cap, needed);
    } catch (const std::exception& e) { return code_of(e); }
}

// tt_svd.hpp:402-512 (Alg. 4) and tsmm.hpp:84-126
int ref_tt_svd_two_sided(const double* X, const int64_t* dims, int64_t d, int64_t ldx, int64_t r_max, double eps,
                         int workers, int64_t* ranks, double* cores, int64_t cap, int64_t* needed) {
    try {
        DenseTensor t = tensor_from(X, dims, d, ldx);
        ExecContext ctx;
        ctx.threads = workers;
        ctx.validate_reflectors = false;
        TensorTrain tt = tt_svd_two_sided(t, spec_of(r_max, eps), ctx);
        return export_tt(tt, ranks, cores, cap, needed);
    } catch (const std::exception& e) { return code_of(e); }
}

int ref_transpose_reorder(const double* W, int64_t n, int64_t m, int64_t ldw, double* Y, int64_t out_rows,
                          int64_t out_cols, int64_t ldy, int workers) {
    try {
        PaddedMatrix o = transpose_reorder(ConstMatrixView{W, n, m, ldw}, out_rows, out_cols, workers);
        if (o.stride() != ldy) return 3;
        std::memcpy(Y, o.data(), o.stride() * out_cols * 8);
        return 0;
    } catch (const std::exception& e) { return code_of(e); }
}

// Timing entry for the CPU baseline: the input is already a reference
// DenseTensor built once by ref_tensor_new, so only tt_svd_tsqr is timed.
void* ref_tensor_new(const double* X, const int64_t* dims, int64_t d, int64_t ldx) {
    try { return new DenseTensor(tensor_from(X, dims, d, ldx)); } catch (...) { return nullptr; }
}
void ref_tensor_free(void* t) { delete static_cast<DenseTensor*>(t); }
int ref_tt_svd_tsqr_tensor(void* t, int64_t r_max, double eps, int workers, int64_t* ranks) {
    try {
        ExecContext ctx;
        ctx.threads = workers;
        ctx.validate_reflectors = false;
        TensorTrain tt = tt_svd_tsqr(*static_cast<DenseTensor*>(t), spec_of(r_max, eps), ctx);
        const auto r = tt.ranks();
        for (std::size_t j = 0; j < r.size(); ++j) ranks[j] = r[j];
        return 0;
    } catch (const std::exception& e) { return code_of(e); }
}

int ref_tt_svd_distributed(const double* const* slabs, int64_t P, const int64_t* ldims, int64_t d_local,
                           int64_t ld_slab, int64_t r_max, double eps, int workers, int64_t* ranks, double* cores,
                           int64_t cap, int64_t* needed) {
    try {
        std::vector<DenseTensor> v;
        for (int64_t p = 0; p < P; ++p) v.push_back(tensor_from(slabs[p], ldims, d_local, ld_slab));
        ExecContext ctx;
        ctx.threads = workers;
        ctx.validate_reflectors = false;
        TensorTrain tt = tt_svd_distributed(v, spec_of(r_max, eps), ctx);
        return export_tt(tt, ranks, cores, cap, needed);
    } catch (const std::exception& e) { return code_of(e); }
}

double ref_tt_error(const double* X, int64_t ldx, const int64_t* dims, int64_t d, const int64_t* ranks,
                    const double* cores) {
    try {
        DenseTensor t = tensor_from(X, dims, d, ldx);
        TensorTrain tt;
        int64_t off = 0;
        for (int64_t j = 0; j < d; ++j) {
            TTCore c(ranks[j], dims[j], ranks[j + 1]);
            std::memcpy(c.data.data(), cores + off, c.data.size() * 8);
            off += static_cast<int64_t>(c.data.size());
            tt.cores.push_back(std::move(c));
        }
        return tt_error(t, tt);
    } catch (const std::exception&) { return -1.0; }
}

// reference test-input generators, used to pin the restated ones
void ref_random_tensor(uint64_t seed, const int64_t* dims, int64_t d, double* out, int64_t ld) {
    DenseTensor t = random_tensor(Shape(std::vector<index_t>(dims, dims + d)), seed);
    const index_t cols = t.total() / t.rows();
    for (index_t j = 0; j < cols; ++j) std::memcpy(out + j * ld, t.data() + j * t.leading_stride(), t.rows() * 8);
}
void ref_gaussian(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    oracles::Dense m = oracles::gaussian(rows, cols, seed);
    std::memcpy(out, m.a.data(), rows * cols * 8);
}
void ref_uniform(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    oracles::Dense m = oracles::uniform(rows, cols, seed);
    std::memcpy(out, m.a.data(), rows * cols * 8);
}

// wire formats (storage.hpp:214-278, tensor_train.hpp:157-191): the
// reference's own writers/readers, for cross-reading files with the package
int ref_save_tt(const char* path, int64_t d, const int64_t* ranks, const int64_t* dims, const double* cores) {
    try {
        TensorTrain tt;
        int64_t off = 0;
        for (int64_t j = 0; j < d; ++j) {
            TTCore c(ranks[j], dims[j], ranks[j + 1]);
            std::memcpy(c.data.data(), cores + off, c.data.size() * 8);
            off += static_cast<int64_t>(c.data.size());
            tt.cores.push_back(std::move(c));
        }
        save_tt(tt, path);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}
int ref_load_tt(const char* path, int64_t* d, int64_t* ranks, int64_t* dims, double* cores, int64_t cap,
                int64_t* needed) {
    try {
        const TensorTrain tt = load_tt(path);
        *d = tt.d();
        for (int64_t j = 0; j < tt.d(); ++j) dims[j] = tt.cores[static_cast<std::size_t>(j)].n;
        return export_tt(tt, ranks, cores, cap, needed);
    } catch (const std::exception& e) {
        return code_of(e);
    }
}
int ref_dump_tensor(const char* path, const double* X, const int64_t* dims, int64_t d, int64_t ldx) {
    try {
        dump_tensor(tensor_from(X, dims, d, ldx), path);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}
// buf: the padded buffer (stride x n_d); cap in doubles
int ref_load_tensor(const char* path, int64_t* d, int64_t* dims, int64_t* ld, double* buf, int64_t cap) {
    try {
        const DenseTensor t = load_tensor(path);
        *d = t.shape().d();
        for (int64_t j = 0; j < *d; ++j) dims[j] = t.shape().dims()[static_cast<std::size_t>(j)];
        *ld = t.leading_stride();
        if (t.buffer_size() > cap) return 11;
        std::memcpy(buf, t.data(), static_cast<std::size_t>(t.buffer_size()) * 8);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

} // extern "C"
