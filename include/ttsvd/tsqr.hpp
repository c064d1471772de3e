// ttsvd/tsqr.hpp — the Q-less TSQR entry points of tsqr.hpp:20-292 on the
// B200 path (K_TSQR kernels behind ttsvd_cu_tsqr / _reduce_block /
// _combine_factors).  Same signatures; `workers` and BlockParams are accepted
// and ignored (the device partition is fixed per shape, so results are
// deterministic per shape); R is unique up to the signs of its rows, and the
// device pivots give R(j, j) the sign of the stacked [R; block] pivot.
#pragma once

#include <cfloat>
#include <cstdint>
#include <vector>

#include "counters.hpp"
#include "device.hpp"
#include "errors.hpp"
#include "storage.hpp"

namespace ttsvd {

#ifdef NDEBUG
inline constexpr bool kDebugBuild = false;
#else
inline constexpr bool kDebugBuild = true;
#endif

// m x m upper triangle, column-major, exact zeros below the diagonal
struct TriangularFactor {
    index_t m = 0;
    std::vector<double> entries;

    TriangularFactor() = default;
    explicit TriangularFactor(index_t m_) : m(m_), entries(static_cast<std::size_t>(m_ * m_), 0.0) {}
    double& operator()(index_t i, index_t j) { return entries[static_cast<std::size_t>(j * m + i)]; }
    double operator()(index_t i, index_t j) const { return entries[static_cast<std::size_t>(j * m + i)]; }
    ConstMatrixView view() const { return {entries.data(), m, m, m}; }
};

// CPU blocking knobs (tsqr.hpp:41-55); kept for callers, no device meaning
struct BlockParams {
    index_t n_b = 256;
    double eps_fp = DBL_MIN;
    bool validate_reflectors = kDebugBuild;

    // largest multiple of 8 with (n_b + m) m 8 <= budget, within [16, 4096]
    static BlockParams for_cols(index_t m, index_t l2_budget_bytes = 256 * 1024) {
        BlockParams p;
        const index_t nb = (l2_budget_bytes / 8 / std::max<index_t>(m, 1) - m) / 8 * 8;
        p.n_b = std::min<index_t>(4096, std::max<index_t>(16, nb));
        return p;
    }
};

// tsqr.hpp:58-64.  Not instrumented on the device: the fields stay as the
// caller set them (the device scratch is the per-SM factor stack, bounded by
// the grid, not by n_b).
struct TsqrStats {
    index_t scratch_bytes = 0;
    index_t blocks = 0;
    double max_reflector_dev = 0.0;
};

namespace detail {
// the reference's flop convention for one structured block reduction
// (tsqr.hpp:196-200): short blocks count as zero-padded to m rows
inline std::uint64_t block_flops(index_t rows, index_t m) {
    const std::uint64_t nb = static_cast<std::uint64_t>(std::max(rows, m));
    return 2ull * static_cast<std::uint64_t>(m) * static_cast<std::uint64_t>(m + 1) * (nb + 1);
}

inline TriangularFactor download_triangle(const b200::DeviceBuffer& d, index_t m) {
    TriangularFactor R(m);
    d.download(R.entries.data(), R.entries.size());
    return R;
}
}  // namespace detail

// device-resident X (n x m, ld >= n): one read of X, R^T R = X^T X
inline TriangularFactor tsqr(DeviceMatrixView X, const BlockParams& = {}, int = 1, TsqrStats* = nullptr,
                             Counters* counters = nullptr) {
    if (X.cols < 1) throw DimensionError("tsqr: needs at least one column");
    if (X.rows < X.cols) throw DimensionError("tsqr: requires n >= m");
    b200::DeviceBuffer R(static_cast<std::size_t>(X.cols * X.cols));
    b200::check(ttsvd_cu_tsqr(b200::context(), X.data, X.rows, X.cols, X.stride, R.get()));
    if (counters)
        counters->add(2ull * static_cast<std::uint64_t>(X.rows) * static_cast<std::uint64_t>(X.cols * X.cols),
                      8ull * static_cast<std::uint64_t>(X.rows) * static_cast<std::uint64_t>(X.cols));
    return detail::download_triangle(R, X.cols);
}

// tsqr.hpp:247: the host view is staged to the device first
inline TriangularFactor tsqr(ConstMatrixView X, const BlockParams& params, int workers, TsqrStats* stats = nullptr,
                             Counters* counters = nullptr) {
    if (X.cols < 1) throw DimensionError("tsqr: needs at least one column");
    if (X.rows < X.cols) throw DimensionError("tsqr: requires n >= m");
    const b200::DeviceBuffer d = b200::stage(X);
    return tsqr(DeviceMatrixView{d.get(), X.rows, X.cols, X.rows}, params, workers, stats, counters);
}

// tsqr.hpp:208: R_out^T R_out = M^T M + R^T R
inline TriangularFactor reduce_block(ConstMatrixView M, const TriangularFactor& R, const BlockParams& = {},
                                     TsqrStats* = nullptr, Counters* counters = nullptr) {
    if (R.m != M.cols) throw DimensionMismatch("reduce_block: R.m != M.cols");
    const b200::DeviceBuffer dm = b200::stage(M);
    b200::DeviceBuffer din(R.entries.size()), dout(R.entries.size());
    din.upload(R.entries.data(), R.entries.size());
    b200::check(ttsvd_cu_reduce_block(b200::context(), dm.get(), M.rows, M.cols, std::max<index_t>(M.rows, 1),
                                      din.get(), R.m, dout.get()));
    if (counters) counters->add(detail::block_flops(M.rows, M.cols), 0);
    return detail::download_triangle(dout, R.m);
}

// tsqr.hpp:230: the parts merged in ascending index order on the device
inline TriangularFactor combine_factors(const std::vector<TriangularFactor>& parts, const BlockParams& = {},
                                        TsqrStats* = nullptr, Counters* counters = nullptr) {
    if (parts.empty()) throw DimensionMismatch("combine_factors: empty list");
    const index_t m = parts.front().m;
    for (const TriangularFactor& p : parts)
        if (p.m != m) throw DimensionMismatch("combine_factors: mixed column counts");
    if (parts.size() == 1) return parts.front();
    std::vector<double> stacked;
    stacked.reserve(parts.size() * static_cast<std::size_t>(m * m));
    for (const TriangularFactor& p : parts) stacked.insert(stacked.end(), p.entries.begin(), p.entries.end());
    b200::DeviceBuffer dp(stacked.size()), dout(static_cast<std::size_t>(m * m));
    dp.upload(stacked.data(), stacked.size());
    b200::check(ttsvd_cu_combine_factors(b200::context(), dp.get(), static_cast<index_t>(parts.size()), m, dout.get()));
    if (counters)
        for (std::size_t i = 1; i < parts.size(); ++i) counters->add(detail::block_flops(m, m), 0);
    return detail::download_triangle(dout, m);
}

}  // namespace ttsvd
