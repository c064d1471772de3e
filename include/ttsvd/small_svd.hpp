// ttsvd/small_svd.hpp — small_svd.hpp:14-205 on the B200 path.  jacobi_svd and
// small_svd run the reference's one-sided cyclic Jacobi (same skip rule,
// 30-sweep cap, sort, deterministic completion of U) on the device
// (ttsvd_cu_jacobi_svd); the rank rules are host arithmetic through the ABI.
#pragma once

#include <cmath>
#include <limits>
#include <vector>

#include "device.hpp"
#include "errors.hpp"
#include "tsqr.hpp"

namespace ttsvd {

// A = U diag(sigma) V^T, sigma non-increasing; U n x m, V m x m, column-major
struct SmallSVD {
    index_t n = 0, m = 0;
    std::vector<double> U, sigma, V;
    double u(index_t i, index_t j) const { return U[static_cast<std::size_t>(j * n + i)]; }
    double v(index_t i, index_t j) const { return V[static_cast<std::size_t>(j * m + i)]; }
};

struct TruncationSpec {
    index_t r_max = std::numeric_limits<index_t>::max();
    double eps = 0.0;
    double delta = -1.0;  // < 0: derived from the first step
    bool has_delta() const { return delta >= 0.0; }
};

// eps / sqrt(d - 1) * ||.||_F (small_svd.hpp:41-45)
inline double derive_delta(double norm_source, double eps, index_t d) {
    double out = 0.0;
    b200::check(ttsvd_cu_derive_delta(norm_source, eps, d, &out));
    return out;
}

// tail rule, r = clamp(min(r_max, r_delta), 1, m) (small_svd.hpp:49-63)
inline index_t select_rank(const std::vector<double>& sigma, double delta, index_t r_max) {
    return ttsvd_cu_select_rank_host(sigma.data(), static_cast<index_t>(sigma.size()), delta, r_max);
}

inline double sigma_norm(const std::vector<double>& sigma) {
    double s = 0.0;
    for (double x : sigma) s += x * x;
    return std::sqrt(s);
}

// small_svd.hpp:120: tall A (n >= m)
inline SmallSVD jacobi_svd(ConstMatrixView A) {
    if (A.rows < A.cols) throw DimensionError("jacobi_svd: requires n >= m");
    SmallSVD s;
    s.n = A.rows;
    s.m = A.cols;
    if (A.cols == 0) return s;
    const b200::DeviceBuffer da = b200::stage(A);
    b200::DeviceBuffer ds(static_cast<std::size_t>(A.cols)), dv(static_cast<std::size_t>(A.cols * A.cols)),
        du(static_cast<std::size_t>(A.rows * A.cols));
    b200::check(ttsvd_cu_jacobi_svd(b200::context(), da.get(), A.rows, A.cols, A.rows, ds.get(), dv.get(), du.get()));
    s.sigma.resize(ds.size());
    s.V.resize(dv.size());
    s.U.resize(du.size());
    ds.download(s.sigma.data(), s.sigma.size());
    dv.download(s.V.data(), s.V.size());
    du.download(s.U.data(), s.U.size());
    return s;
}

// small_svd.hpp:196: the SVD of a TSQR factor
inline SmallSVD small_svd(const TriangularFactor& R) {
    if (R.m > 4096) throw DimensionMismatch("small_svd: m exceeds 4096");
    return jacobi_svd(R.view());
}

}  // namespace ttsvd
