// ttsvd/tt_svd.hpp — the TT-SVD drivers of tt_svd.hpp:19-631 on the B200 path.
//
//   tt_svd_tsqr          tt_svd.hpp:281  (Alg. 2)  -> ttsvd_cu_tt_svd(_host)
//   detail::run_chain    tt_svd.hpp:159            -> ttsvd_cu_run_chain
//   tt_svd_thick_bounds  tt_svd.hpp:338  (Alg. 3)  -> ttsvd_cu_tt_svd_thick
//   tt_svd_two_sided     tt_svd.hpp:402  (Alg. 4)  -> ttsvd_cu_tt_svd_two_sided
//   tt_svd_distributed   tt_svd.hpp:520  (Alg. 5)  -> ttsvd_cu_tt_svd_distributed
//   tt_svd_reference     tt_svd.hpp:215  (Alg. 1)  -> device jacobi_svd per step
//
// Every numeric step runs on the GPU; the host only sequences calls, copies
// cores back and fills the optional RunRecorder / Counters from the device
// step records (phase times are CUDA-event device times while a recorder is
// attached).
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <limits>
#include <utility>
#include <vector>

#include "counters.hpp"
#include "device.hpp"
#include "errors.hpp"
#include "small_svd.hpp"
#include "storage.hpp"
#include "tensor_train.hpp"
#include "threading.hpp"
#include "tsmm.hpp"
#include "tsqr.hpp"

namespace ttsvd {

// tt_svd.hpp:21-37
struct StepRecord {
    index_t step = 0;  // 1-based, execution order
    double t_tsqr = 0, t_small_svd = 0, t_tsmm = 0, t_reorder = 0;  // seconds
    index_t rows = 0, cols = 0, rank = 0;
    double f = 0;  // rank / cols
};

struct RunRecorder {
    std::vector<StepRecord> steps;
    StepRecord& next_step() {
        steps.emplace_back();
        steps.back().step = static_cast<index_t>(steps.size());
        return steps.back();
    }
};

// tt_svd.hpp:39-52; threads / l2 budget / reflector validation have no
// device meaning and are accepted for compatibility
struct ExecContext {
    int threads = 1;
    index_t l2_budget_bytes = 256 * 1024;
    bool validate_reflectors = kDebugBuild;
    Counters* counters = nullptr;
    RunRecorder* recorder = nullptr;
    TsqrStats* tsqr_stats = nullptr;

    BlockParams block_params(index_t m) const {
        BlockParams p = BlockParams::for_cols(m, l2_budget_bytes);
        p.validate_reflectors = validate_reflectors;
        return p;
    }
};

namespace b200 {

// owns a result handle of the C-ABI
class Result {
public:
    Result() = default;
    Result(const Result&) = delete;
    Result& operator=(const Result&) = delete;
    ~Result() {
        if (h_) ttsvd_cu_tt_free(h_);
    }
    ttsvd_cu_tt** out() { return &h_; }
    ttsvd_cu_tt* get() const { return h_; }

    std::vector<index_t> ranks() const {
        std::vector<index_t> r(static_cast<std::size_t>(ttsvd_cu_tt_d(h_) + 1));
        check(ttsvd_cu_tt_ranks(h_, r.data()));
        return r;
    }
    TensorTrain train(const std::vector<index_t>& dims) const {
        const std::vector<index_t> r = ranks();
        TensorTrain tt;
        for (std::size_t j = 0; j < dims.size(); ++j) {
            TTCore c(r[j], dims[j], r[j + 1]);
            check(ttsvd_cu_tt_core(h_, static_cast<index_t>(j), c.data.data()));
            tt.cores.push_back(std::move(c));
        }
        return tt;
    }
    std::vector<ttsvd_cu_step> steps() const {
        std::vector<ttsvd_cu_step> s(static_cast<std::size_t>(std::max<index_t>(ttsvd_cu_tt_nsteps(h_), 0)));
        for (std::size_t i = 0; i < s.size(); ++i) check(ttsvd_cu_tt_step(h_, static_cast<index_t>(i), &s[i]));
        return s;
    }

private:
    ttsvd_cu_tt* h_ = nullptr;
};

// per-phase CUDA-event timing while a recorder listens
class TimingScope {
public:
    TimingScope(ttsvd_cu_ctx* c, bool on) : c_(on ? c : nullptr) {
        if (c_) check(ttsvd_cu_ctx_set_timing(c_, 1));
    }
    ~TimingScope() {
        if (c_) ttsvd_cu_ctx_set_timing(c_, 0);
    }

private:
    ttsvd_cu_ctx* c_;
};

// device step records -> RunRecorder / Counters (the kernels' algorithmic work)
inline void account(const Result& res, const ExecContext& ctx, bool two_sided = false) {
    if (!ctx.recorder && !ctx.counters) return;
    const std::vector<ttsvd_cu_step> steps = res.steps();
    for (std::size_t i = 0; i < steps.size(); ++i) {
        const ttsvd_cu_step& s = steps[i];
        const auto rows = static_cast<std::uint64_t>(s.rows), cols = static_cast<std::uint64_t>(s.cols),
                   k = static_cast<std::uint64_t>(s.rank);
        if (ctx.counters) {
            if (s.rows >= s.cols) ctx.counters->add(2 * rows * cols * cols, 8 * rows * cols);
            ctx.counters->add(2 * rows * cols * k, 8 * rows * (cols + k));
            // the two-sided sweep reorders after every step but a final right one
            if (two_sided && !(i + 1 == steps.size() && i % 2 == 0)) ctx.counters->add(0, 16 * rows * k);
        }
        if (ctx.recorder) {
            StepRecord& r = ctx.recorder->next_step();
            r.t_tsqr = s.t_tsqr_ms * 1e-3;
            r.t_small_svd = s.t_svd_ms * 1e-3;
            r.t_tsmm = s.t_tsmm_ms * 1e-3;
            r.t_reorder = s.t_reorder_ms * 1e-3;
            r.rows = s.rows;
            r.cols = s.cols;
            r.rank = s.rank;
            r.f = s.cols ? static_cast<double>(s.rank) / static_cast<double>(s.cols) : 0.0;
        }
    }
}

}  // namespace b200

namespace detail {

// tt_svd.hpp:62-73
struct WorkSVD {
    std::vector<double> sigma;  // nsig values
    std::vector<double> V;      // cols x nsig, column-major
    index_t cols = 0, nsig = 0;
    ConstMatrixView v_view(index_t r) const { return {V.data(), cols, r, cols}; }
};

// tt_svd.hpp:75-105: tall -> tsqr + small_svd; wide -> Jacobi of W^T (V := U)
inline WorkSVD svd_of_work(ConstMatrixView W, const ExecContext& ctx, StepRecord* = nullptr) {
    WorkSVD out;
    out.cols = W.cols;
    if (W.rows >= W.cols) {
        SmallSVD s = small_svd(tsqr(W, ctx.block_params(W.cols), ctx.threads, ctx.tsqr_stats, ctx.counters));
        out.sigma = std::move(s.sigma);
        out.V = std::move(s.V);
        out.nsig = W.cols;
    } else {
        const PaddedMatrix Wt = transpose_reorder(W);
        SmallSVD s = jacobi_svd(Wt.view());
        out.sigma = std::move(s.sigma);
        out.V = std::move(s.U);
        out.nsig = W.rows;
    }
    return out;
}

// tt_svd.hpp:111-118: the tail rule above the numerical-zero level
inline index_t choose_rank(const WorkSVD& s, const TruncationSpec& spec, index_t rows) {
    const double s1 = s.sigma.empty() ? 0.0 : s.sigma.front();
    const double zero = 32.0 * DBL_EPSILON * s1 * std::sqrt(static_cast<double>(std::max(rows, s.cols)));
    return std::min(select_rank(s.sigma, std::max(spec.delta, zero), spec.r_max), s.nsig);
}

// T(a, x, b) = V[a cols + x + n b] (tt_svd.hpp:121-128)
inline TTCore core_from_vt(const WorkSVD& s, index_t r, index_t n, index_t r_right) {
    TTCore c(r, n, r_right);
    for (index_t b = 0; b < r_right; ++b)
        for (index_t x = 0; x < n; ++x)
            for (index_t a = 0; a < r; ++a) c(a, x, b) = s.V[static_cast<std::size_t>(a * s.cols + x + n * b)];
    return c;
}

// T(a, x, b) = V[b cols + a + r_left x] (tt_svd.hpp:131-138)
inline TTCore core_from_v(const WorkSVD& s, index_t r_left, index_t n, index_t r) {
    TTCore c(r_left, n, r);
    for (index_t b = 0; b < r; ++b)
        for (index_t x = 0; x < n; ++x)
            for (index_t a = 0; a < r_left; ++a) c(a, x, b) = s.V[static_cast<std::size_t>(b * s.cols + a + r_left * x)];
    return c;
}

// flat order of a padded matrix as a core (tt_svd.hpp:140-147)
inline TTCore core_from_padded(const PaddedMatrix& p, index_t r_left, index_t n, index_t r_right) {
    TTCore c(r_left, n, r_right);
    for (index_t l = 0; l < r_left * n * r_right; ++l) c.data[static_cast<std::size_t>(l)] = p(l % p.rows(), l / p.rows());
    return c;
}

// tt_svd.hpp:150-156
struct ChainResult {
    std::vector<TTCore> cores;
    double first_sigma_norm = 0.0;
};

// the Alg. 2 loop (tt_svd.hpp:159-199) on the device; spec.delta is derived
// from the first step when unset and written back, as the reference does
inline ChainResult run_chain(ConstMatrixView W0, const std::vector<index_t>& dims, TruncationSpec& spec,
                             index_t d_for_delta, const ExecContext& ctx) {
    const b200::DeviceBuffer dw = b200::stage(W0);
    ttsvd_cu_ctx* c = b200::context();
    b200::Result res;
    double delta = spec.has_delta() ? spec.delta : -1.0, fsn = 0.0;
    {
        b200::TimingScope t(c, ctx.recorder != nullptr);
        b200::check(ttsvd_cu_run_chain(c, dw.get(), W0.rows, W0.cols, std::max<index_t>(W0.rows, 1), dims.data(),
                                       static_cast<index_t>(dims.size()), spec.r_max, spec.eps, d_for_delta, &delta,
                                       &fsn, res.out()));
    }
    b200::account(res, ctx);
    spec.delta = delta;
    ChainResult out;
    out.cores = res.train(dims).cores;
    out.first_sigma_norm = fsn;
    return out;
}

// tt_svd.hpp:201-210: tsqr, or a zero-padded square block when wide
inline TriangularFactor gram_triangular(ConstMatrixView W, const ExecContext& ctx) {
    if (W.rows >= W.cols) return tsqr(W, ctx.block_params(W.cols), ctx.threads, ctx.tsqr_stats, ctx.counters);
    PaddedMatrix sq(W.cols, W.cols);
    for (index_t j = 0; j < W.cols; ++j)
        for (index_t i = 0; i < W.rows; ++i) sq(i, j) = W(i, j);
    return tsqr(sq.view(), ctx.block_params(W.cols), ctx.threads, ctx.tsqr_stats, ctx.counters);
}

}  // namespace detail

// Alg. 1 (tt_svd.hpp:215-275): the direct truncated SVD of every
// matricization by one-sided Jacobi (device jacobi_svd), W carried as U Sigma
inline TensorTrain tt_svd_reference(const DenseTensor& X, TruncationSpec spec) {
    const index_t d = X.shape().d();
    if (d < 2) throw DegenerateDimension("tt_svd_reference: requires d >= 2");
    const std::vector<index_t>& dims = X.shape().dims();
    spec.delta = derive_delta(frobenius_norm(X), spec.eps, d);
    std::vector<double> w(static_cast<std::size_t>(X.total()));
    for (index_t l = 0; l < X.total(); ++l) w[static_cast<std::size_t>(l)] = X.at_flat(l);
    TensorTrain tt;
    tt.cores.resize(static_cast<std::size_t>(d));
    index_t r = 1, total = X.total();
    for (index_t i = d - 1; i >= 1; --i) {
        const index_t n_i = dims[static_cast<std::size_t>(i)], m = n_i * r, rows = total / m;
        detail::WorkSVD s;
        s.cols = m;
        const bool tall = rows >= m;
        const index_t k = tall ? m : rows;  // columns of U Sigma
        SmallSVD j;
        if (tall) {
            j = jacobi_svd(ConstMatrixView{w.data(), rows, m, rows});
        } else {
            const PaddedMatrix wt = transpose_reorder(ConstMatrixView{w.data(), rows, m, rows});
            j = jacobi_svd(wt.view());
        }
        s.nsig = k;
        s.sigma = j.sigma;
        s.V = tall ? j.V : j.U;
        const std::vector<double>& left = tall ? j.U : j.V;  // rows x k
        const index_t rnew = detail::choose_rank(s, spec, rows);
        tt.cores[static_cast<std::size_t>(i)] = detail::core_from_vt(s, rnew, n_i, r);
        std::vector<double> next(static_cast<std::size_t>(rows * rnew));
        for (index_t c = 0; c < rnew; ++c)
            for (index_t ii = 0; ii < rows; ++ii)
                next[static_cast<std::size_t>(c * rows + ii)] =
                    left[static_cast<std::size_t>(c * rows + ii)] * j.sigma[static_cast<std::size_t>(c)];
        w.swap(next);
        total = rows * rnew;
        r = rnew;
    }
    TTCore first(1, dims[0], r);
    std::copy(w.begin(), w.begin() + static_cast<std::ptrdiff_t>(total), first.data.begin());
    tt.cores[0] = std::move(first);
    tt.validate();
    return tt;
}

// Alg. 2 on a host tensor (H2D inside the call, the reference-facing entry)
inline TensorTrain tt_svd_tsqr(const DenseTensor& X, TruncationSpec spec, const ExecContext& ctx = {}) {
    const index_t d = X.shape().d();
    if (d < 2) throw DegenerateDimension("tt_svd_tsqr: requires d >= 2");
    ttsvd_cu_ctx* c = b200::context();
    b200::Result res;
    {
        b200::TimingScope t(c, ctx.recorder != nullptr);
        b200::check(ttsvd_cu_tt_svd_host(c, X.data(), X.shape().dims().data(), d, X.leading_stride(), spec.r_max,
                                         spec.eps, res.out()));
    }
    b200::account(res, ctx);
    TensorTrain tt = res.train(X.shape().dims());
    tt.validate();
    return tt;
}

// Alg. 2 on a device-resident tensor (padded layout, ld >= N / n_d)
inline TensorTrain tt_svd_tsqr(const double* X_device, const std::vector<index_t>& dims, index_t ld,
                               TruncationSpec spec, const ExecContext& ctx = {}) {
    ttsvd_cu_ctx* c = b200::context();
    b200::Result res;
    {
        b200::TimingScope t(c, ctx.recorder != nullptr);
        b200::check(ttsvd_cu_tt_svd(c, X_device, dims.data(), static_cast<index_t>(dims.size()), ld, spec.r_max,
                                    spec.eps, res.out()));
    }
    b200::account(res, ctx);
    return res.train(dims);
}

// tt_svd.hpp:292-310
struct ThickBoundsParams {
    index_t m_min = 16;
    double f1_min = 0.5;
    std::vector<index_t> r_tilde;  // r~_1..r~_{d-1}; empty = r_max

    index_t estimate_at(index_t pos, const Shape& shape, index_t r_max) const {
        const index_t lead = shape.leading(pos);
        const index_t cap = std::min(lead, shape.total() / lead);
        const index_t rt = r_tilde.empty()
                               ? r_max
                               : r_tilde[static_cast<std::size_t>(
                                     std::min<index_t>(pos - 1, static_cast<index_t>(r_tilde.size()) - 1))];
        return std::min(rt, cap);
    }
};

// tt_svd.hpp:316-330 (host arithmetic of the C-ABI)
inline std::pair<index_t, index_t> choose_combined_dims(const Shape& shape, const ThickBoundsParams& params,
                                                        index_t r_max = std::numeric_limits<index_t>::max()) {
    index_t k = 0, m = 0;
    b200::check(ttsvd_cu_choose_combined_dims(shape.dims().data(), shape.d(), params.m_min, params.f1_min,
                                              params.r_tilde.empty() ? nullptr : params.r_tilde.data(),
                                              static_cast<index_t>(params.r_tilde.size()), r_max, &k, &m));
    return {k, m};
}

// Alg. 3 (tt_svd.hpp:338-400): merge, sweep and recover on the device
inline TensorTrain tt_svd_thick_bounds(const DenseTensor& X, TruncationSpec spec, const ThickBoundsParams& params,
                                       const ExecContext& ctx = {}) {
    const index_t d = X.shape().d();
    if (d < 2) throw DegenerateDimension("tt_svd_thick_bounds: requires d >= 2");
    ttsvd_cu_ctx* c = b200::context();
    b200::Result res;
    {
        // the host-buffer entry: X goes H2D inside the call (in row chunks
        // under the merged first TSQR where its shape allows)
        b200::TimingScope t(c, ctx.recorder != nullptr);
        b200::check(ttsvd_cu_tt_svd_thick_host(c, X.data(), X.shape().dims().data(), d, X.leading_stride(), spec.r_max,
                                               spec.eps, params.m_min, params.f1_min,
                                               params.r_tilde.empty() ? nullptr : params.r_tilde.data(),
                                               static_cast<index_t>(params.r_tilde.size()), res.out()));
    }
    b200::account(res, ctx);
    TensorTrain tt = res.train(X.shape().dims());
    tt.validate();
    return tt;
}

// Alg. 4 (tt_svd.hpp:402-512): alternating ends with transpose_reorder
inline TensorTrain tt_svd_two_sided(const DenseTensor& X, TruncationSpec spec, const ExecContext& ctx = {}) {
    const index_t d = X.shape().d();
    if (d < 2) throw DegenerateDimension("tt_svd_two_sided: requires d >= 2");
    const b200::DeviceBuffer dx = b200::stage(X);
    ttsvd_cu_ctx* c = b200::context();
    b200::Result res;
    {
        b200::TimingScope t(c, ctx.recorder != nullptr);
        b200::check(ttsvd_cu_tt_svd_two_sided(c, dx.get(), X.shape().dims().data(), d, X.leading_stride(),
                                              spec.r_max, spec.eps, res.out()));
    }
    b200::account(res, ctx, true);
    TensorTrain tt = res.train(X.shape().dims());
    tt.validate();
    return tt;
}

// Alg. 5 (tt_svd.hpp:520-631), in-process form: every slab on the current
// device, per-slab TSQR, pinned-order merge of the P triangles, one small SVD
// shared by all partitions.  per_partition[p] is partition p's own train:
// its first core is the (1 x 1 x r) slice p of the global (1 x P x r) core,
// the other cores are the shared ones (tt_svd.hpp:594-628).
inline TensorTrain tt_svd_distributed(const std::vector<DenseTensor>& slabs, TruncationSpec spec,
                                      const ExecContext& ctx = {}, std::vector<TensorTrain>* per_partition = nullptr) {
    if (slabs.empty()) throw PartitionMismatch("tt_svd_distributed: no partitions");
    const Shape& local = slabs.front().shape();
    for (const DenseTensor& s : slabs)
        if (!(s.shape() == local)) throw PartitionMismatch("tt_svd_distributed: slab shapes differ");
    const index_t P = static_cast<index_t>(slabs.size());
    std::vector<b200::DeviceBuffer> bufs;
    std::vector<const double*> ptrs;
    for (const DenseTensor& s : slabs) {
        bufs.push_back(b200::stage(s));
        ptrs.push_back(bufs.back().get());
    }
    ttsvd_cu_ctx* c = b200::context();
    b200::Result res;
    {
        b200::TimingScope t(c, ctx.recorder != nullptr);
        b200::check(ttsvd_cu_tt_svd_distributed(c, ptrs.data(), P, 0, P, local.dims().data(), local.d(),
                                                slabs.front().leading_stride(), spec.r_max, spec.eps, nullptr,
                                                nullptr, res.out()));
    }
    b200::account(res, ctx);
    std::vector<index_t> gdims{P};
    gdims.insert(gdims.end(), local.dims().begin(), local.dims().end());
    TensorTrain tt = res.train(gdims);
    tt.validate();
    if (per_partition) {
        per_partition->assign(static_cast<std::size_t>(P), tt);
        if (P > 1) {
            const TTCore& first = tt.cores.front();
            for (index_t p = 0; p < P; ++p) {
                TTCore own(1, 1, first.r_right);
                for (index_t b = 0; b < first.r_right; ++b) own(0, 0, b) = first(0, p, b);
                (*per_partition)[static_cast<std::size_t>(p)].cores.front() = std::move(own);
            }
        }
    }
    return tt;
}

// Alg. 5 across the GPUs of this process: partition p of P = slabs.size()
// lives on devices[p / (P / D)] (D = devices.size() must divide P); the
// library attaches an NCCL communicator over the devices (ncclCommInitAll)
// and runs one host thread per device, all-gathering the R factors with
// ncclAllGather.  Same result contract as the in-process overload.
inline TensorTrain tt_svd_distributed(const std::vector<DenseTensor>& slabs, const std::vector<int>& devices,
                                      TruncationSpec spec, const ExecContext& ctx = {},
                                      std::vector<TensorTrain>* per_partition = nullptr) {
    if (slabs.empty() || devices.empty()) throw PartitionMismatch("tt_svd_distributed: no partitions or devices");
    const Shape& local = slabs.front().shape();
    for (const DenseTensor& s : slabs)
        if (!(s.shape() == local)) throw PartitionMismatch("tt_svd_distributed: slab shapes differ");
    const int D = static_cast<int>(devices.size());
    const index_t P = static_cast<index_t>(slabs.size());
    if (P % D) throw PartitionMismatch("tt_svd_distributed: the device count must divide the partition count");
    int prev = 0;
    b200::cuda(cudaGetDevice(&prev));
    struct Ctxs {
        std::vector<ttsvd_cu_ctx*> c;
        ~Ctxs() {
            for (ttsvd_cu_ctx* x : c) ttsvd_cu_ctx_destroy(x);
        }
    } ctxs;
    std::vector<b200::DeviceBuffer> bufs;
    std::vector<const double*> ptrs;
    for (index_t p = 0; p < P; ++p) {
        const int dev = devices[static_cast<std::size_t>(p / (P / D))];
        if (p % (P / D) == 0) {
            ttsvd_cu_ctx* c = nullptr;
            b200::check(ttsvd_cu_ctx_create(dev, nullptr, &c));
            ctxs.c.push_back(c);
        }
        b200::cuda(cudaSetDevice(dev));
        bufs.push_back(b200::stage(slabs[static_cast<std::size_t>(p)]));
        ptrs.push_back(bufs.back().get());
    }
    b200::check(ttsvd_cu_ctx_comm_init_all(ctxs.c.data(), D));
    b200::Result res;
    b200::check(ttsvd_cu_tt_svd_distributed_devices(ctxs.c.data(), D, ptrs.data(), P / D, local.dims().data(),
                                                    local.d(), slabs.front().leading_stride(), spec.r_max, spec.eps,
                                                    res.out()));
    b200::cuda(cudaSetDevice(prev));
    b200::account(res, ctx);
    std::vector<index_t> gdims{P};
    gdims.insert(gdims.end(), local.dims().begin(), local.dims().end());
    TensorTrain tt = res.train(gdims);
    tt.validate();
    if (per_partition) {
        per_partition->assign(static_cast<std::size_t>(P), tt);
        const TTCore& first = tt.cores.front();
        for (index_t p = 0; p < P && P > 1; ++p) {
            TTCore own(1, 1, first.r_right);
            for (index_t b = 0; b < first.r_right; ++b) own(0, 0, b) = first(0, p, b);
            (*per_partition)[static_cast<std::size_t>(p)].cores.front() = std::move(own);
        }
    }
    return tt;
}

}  // namespace ttsvd
