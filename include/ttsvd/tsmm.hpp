// ttsvd/tsmm.hpp — tsmm.hpp:14-126 on the B200 path: the fused TSMM + reshape
// (K_TSMM, ttsvd_cu_tsmm_reshape) and the two-sided sweep's transpose +
// reshape (ttsvd_cu_transpose_reorder).  Host views are staged, results come
// back as padded host matrices (the reference's by-value contract).
#pragma once

#include <cstdint>

#include "counters.hpp"
#include "device.hpp"
#include "errors.hpp"
#include "storage.hpp"

namespace ttsvd {

// Y = reshape(X V): product (i, c) at flat position i + n c
inline PaddedMatrix tsmm_reshape(ConstMatrixView X, ConstMatrixView V, index_t out_rows, index_t out_cols,
                                 int = 1, Counters* counters = nullptr) {
    if (V.rows != X.cols) throw ShapeError("tsmm_reshape: V.rows != X.cols");
    if (V.cols > X.cols) throw ShapeError("tsmm_reshape: k > m (kernel only shrinks)");
    if (out_rows < 1 || out_cols < 1 || X.rows * V.cols != out_rows * out_cols)
        throw ShapeError("tsmm_reshape: out shape does not hold n*k elements");
    PaddedMatrix out(out_rows, out_cols);
    const b200::DeviceBuffer dx = b200::stage(X), dv = b200::stage(V);
    b200::DeviceBuffer dy(static_cast<std::size_t>(out.stride() * out_cols));
    b200::check(ttsvd_cu_tsmm_reshape(b200::context(), dx.get(), X.rows, X.cols, std::max<index_t>(X.rows, 1),
                                      dv.get(), V.cols, std::max<index_t>(V.rows, 1), dy.get(), out_rows, out_cols,
                                      out.stride()));
    dy.download(out.data(), dy.size());
    if (counters)
        counters->add(2ull * static_cast<std::uint64_t>(X.rows * X.cols) * static_cast<std::uint64_t>(V.cols),
                      8ull * static_cast<std::uint64_t>(X.rows) * static_cast<std::uint64_t>(X.cols + V.cols));
    return out;
}

inline PaddedMatrix tsmm_reshape(ConstMatrixView X, ConstMatrixView V, int workers = 1, Counters* c = nullptr) {
    return tsmm_reshape(X, V, X.rows, V.cols, workers, c);
}

// flat(W^T) as an (out_rows x out_cols) padded matrix
inline PaddedMatrix transpose_reorder(ConstMatrixView W, index_t out_rows, index_t out_cols, int = 1,
                                      Counters* counters = nullptr) {
    if (out_rows < 1 || out_cols < 1 || out_rows * out_cols != W.rows * W.cols)
        throw ShapeError("transpose_reorder: out shape does not hold n*m elements");
    PaddedMatrix out(out_rows, out_cols);
    const b200::DeviceBuffer dw = b200::stage(W);
    b200::DeviceBuffer dy(static_cast<std::size_t>(out.stride() * out_cols));
    b200::check(ttsvd_cu_transpose_reorder(b200::context(), dw.get(), W.rows, W.cols, std::max<index_t>(W.rows, 1),
                                           dy.get(), out_rows, out_cols, out.stride()));
    dy.download(out.data(), dy.size());
    if (counters) counters->add(0, 16ull * static_cast<std::uint64_t>(W.rows) * static_cast<std::uint64_t>(W.cols));
    return out;
}

// the plain transpose
inline PaddedMatrix transpose_reorder(ConstMatrixView W, int workers = 1, Counters* c = nullptr) {
    return transpose_reorder(W, W.cols, W.rows, workers, c);
}

}  // namespace ttsvd
