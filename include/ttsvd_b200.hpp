// ttsvd_b200.hpp — C++ drop-in for the reference's TT-SVD hot path on B200.
//
// Keeps the names, signatures, containers and exception types of
// /root/reference/proj/include/ttsvd/ (namespace ttsvd) for the functions on
// the path, and runs them on the GPU through the C-ABI of ttsvd_cu.h:
//
//   tsqr             tsqr.hpp:247        reduce_block     tsqr.hpp:208
//   combine_factors  tsqr.hpp:230        small_svd        small_svd.hpp:196
//   jacobi_svd       small_svd.hpp:120   select_rank      small_svd.hpp:49
//   derive_delta     small_svd.hpp:41    tsmm_reshape     tsmm.hpp:20, :74
//   tt_svd_tsqr      tt_svd.hpp:281      tt_svd_distributed tt_svd.hpp:520
//   choose_combined_dims tt_svd.hpp:316  tt_svd_thick_bounds tt_svd.hpp:338
//
// Host views are staged to the device and results copied back (the
// reference's by-value contract); the Device* overloads keep data resident.
// `workers` and BlockParams are accepted and ignored: device results are
// deterministic per shape.  Link: -lttsvd_cu -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <utility>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "ttsvd_cu.h"

namespace ttsvd {

using index_t = std::int64_t;

// ---- errors.hpp:9-62 (+ DeviceError for CUDA/exchange failures) ----------
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& w) : std::runtime_error(w) {}
};
#define TTSVD_B200_ERR(Name) \
    class Name : public Error { using Error::Error; };
TTSVD_B200_ERR(LayoutError)
TTSVD_B200_ERR(AllocationError)
TTSVD_B200_ERR(DimensionMismatch)
TTSVD_B200_ERR(DimensionError)
TTSVD_B200_ERR(DegenerateDimension)
TTSVD_B200_ERR(ConvergenceError)
TTSVD_B200_ERR(ShapeError)
TTSVD_B200_ERR(PartitionMismatch)
TTSVD_B200_ERR(DivergenceError)
TTSVD_B200_ERR(IoError)
TTSVD_B200_ERR(DeviceError)
#undef TTSVD_B200_ERR

namespace b200 {
inline void check(int rc) {
    if (rc == TTSVD_OK) return;
    const std::string msg = ttsvd_cu_last_error();
    switch (rc) {
        case TTSVD_ERR_DIMENSION: throw DimensionError(msg);
        case TTSVD_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case TTSVD_ERR_SHAPE: throw ShapeError(msg);
        case TTSVD_ERR_CONVERGENCE: throw ConvergenceError(msg);
        case TTSVD_ERR_ALLOCATION: throw AllocationError(msg);
        case TTSVD_ERR_DEGENERATE: throw DegenerateDimension(msg);
        case TTSVD_ERR_PARTITION: throw PartitionMismatch(msg);
        case TTSVD_ERR_LAYOUT: throw LayoutError(msg);
        case TTSVD_ERR_DEVICE: throw DeviceError(msg);
        default: throw Error(msg);
    }
}
inline void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw DeviceError(cudaGetErrorString(e));
}

// one library context per device, on the default stream of this thread
inline ttsvd_cu_ctx* context() {
    thread_local ttsvd_cu_ctx* ctx = nullptr;
    thread_local int dev = -1;
    int cur = 0;
    cuda(cudaGetDevice(&cur));
    if (!ctx || dev != cur) {
        check(ttsvd_cu_ctx_create(cur, nullptr, &ctx));
        dev = cur;
    }
    return ctx;
}

// RAII device buffer of doubles
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t n) : n_(n) { cuda(cudaMalloc(&p_, std::max<std::size_t>(n, 1) * 8)); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
    ~DeviceBuffer() { if (p_) cudaFree(p_); }
    double* get() const { return p_; }
    std::size_t size() const { return n_; }
    void upload(const double* h, std::size_t n) { cuda(cudaMemcpy(p_, h, n * 8, cudaMemcpyHostToDevice)); }
    void download(double* h, std::size_t n) const { cuda(cudaMemcpy(h, p_, n * 8, cudaMemcpyDeviceToHost)); }

private:
    double* p_ = nullptr;
    std::size_t n_ = 0;
};
}  // namespace b200

// ---- shape.hpp:22-28 / storage.hpp:30-115 --------------------------------
inline index_t padded_stride(index_t n_rows) {
    if (n_rows < 1) throw DimensionError("padded_stride: n_rows must be >= 1");
    return ttsvd_cu_padded_stride(n_rows);
}

struct ConstMatrixView {
    const double* data = nullptr;
    index_t rows = 0, cols = 0, stride = 0;
    double operator()(index_t i, index_t j) const { return data[j * stride + i]; }
    const double* col(index_t j) const { return data + j * stride; }
};

struct MatrixView {
    double* data = nullptr;
    index_t rows = 0, cols = 0, stride = 0;
    double& operator()(index_t i, index_t j) const { return data[j * stride + i]; }
    operator ConstMatrixView() const { return ConstMatrixView{data, rows, cols, stride}; }
};

// device-resident counterparts (the performance path)
struct DeviceMatrixView {
    const double* data = nullptr;
    index_t rows = 0, cols = 0, stride = 0;
};

class PaddedMatrix {
public:
    PaddedMatrix() = default;
    PaddedMatrix(index_t rows, index_t cols) : rows_(rows), cols_(cols), stride_(padded_stride(rows)) {
        if (rows < 1 || cols < 1) throw DimensionError("PaddedMatrix: empty shape");
        buf_.assign(static_cast<std::size_t>(stride_ * cols_), 0.0);
    }
    index_t rows() const { return rows_; }
    index_t cols() const { return cols_; }
    index_t stride() const { return stride_; }
    double& operator()(index_t i, index_t j) { return buf_[static_cast<std::size_t>(j * stride_ + i)]; }
    double operator()(index_t i, index_t j) const { return buf_[static_cast<std::size_t>(j * stride_ + i)]; }
    ConstMatrixView view() const { return ConstMatrixView{buf_.data(), rows_, cols_, stride_}; }
    MatrixView view() { return MatrixView{buf_.data(), rows_, cols_, stride_}; }
    double* data() { return buf_.data(); }
    const double* data() const { return buf_.data(); }

private:
    index_t rows_ = 0, cols_ = 0, stride_ = 0;
    std::vector<double> buf_;
};

class DenseTensor {
public:
    DenseTensor() = default;
    explicit DenseTensor(std::vector<index_t> dims) : dims_(std::move(dims)) {
        if (dims_.empty()) throw DimensionError("Shape: needs at least one dimension");
        total_ = 1;
        for (index_t n : dims_) {
            if (n < 1) throw DimensionError("Shape: extents must be >= 1");
            total_ *= n;
        }
        rows_ = total_ / dims_.back();
        stride_ = padded_stride(rows_);
        buf_.assign(static_cast<std::size_t>(stride_ * dims_.back()), 0.0);
    }
    const std::vector<index_t>& dims() const { return dims_; }
    index_t total() const { return total_; }
    index_t rows() const { return rows_; }
    index_t leading_stride() const { return stride_; }
    double& at_flat(index_t l) { return buf_[static_cast<std::size_t>((l / rows_) * stride_ + l % rows_)]; }
    double at_flat(index_t l) const { return buf_[static_cast<std::size_t>((l / rows_) * stride_ + l % rows_)]; }
    double* data() { return buf_.data(); }
    const double* data() const { return buf_.data(); }
    index_t buffer_size() const { return static_cast<index_t>(buf_.size()); }

private:
    std::vector<index_t> dims_;
    index_t total_ = 0, rows_ = 0, stride_ = 0;
    std::vector<double> buf_;
};

// ---- tsqr.hpp:24-64, counters.hpp, small_svd.hpp:18-36 -------------------
struct TriangularFactor {
    index_t m = 0;
    std::vector<double> entries;
    TriangularFactor() = default;
    explicit TriangularFactor(index_t m_) : m(m_), entries(static_cast<std::size_t>(m_ * m_), 0.0) {}
    double& operator()(index_t i, index_t j) { return entries[static_cast<std::size_t>(j * m + i)]; }
    double operator()(index_t i, index_t j) const { return entries[static_cast<std::size_t>(j * m + i)]; }
    ConstMatrixView view() const { return ConstMatrixView{entries.data(), m, m, m}; }
};

struct BlockParams {  // accepted for signature compatibility; ignored on the device
    index_t n_b = 256;
    double eps_fp = 2.2250738585072014e-308;
    bool validate_reflectors = false;
    static BlockParams for_cols(index_t m, index_t l2_budget_bytes = 256 * 1024) {
        BlockParams p;
        index_t nb = (l2_budget_bytes / 8 / (m > 1 ? m : 1) - m) / 8 * 8;
        p.n_b = nb < 16 ? 16 : (nb > 4096 ? 4096 : nb);
        return p;
    }
};

struct TsqrStats {
    index_t scratch_bytes = 0, blocks = 0;
    double max_reflector_dev = 0.0;
};

struct Counters {
    std::uint64_t flops = 0, bytes = 0;
    void add(std::uint64_t f, std::uint64_t b) { flops += f; bytes += b; }
};

struct SmallSVD {
    index_t n = 0, m = 0;
    std::vector<double> U, sigma, V;
    double u(index_t i, index_t j) const { return U[static_cast<std::size_t>(j * n + i)]; }
    double v(index_t i, index_t j) const { return V[static_cast<std::size_t>(j * m + i)]; }
};

struct TruncationSpec {
    index_t r_max = std::numeric_limits<index_t>::max();
    double eps = 0.0;
    double delta = -1.0;
    bool has_delta() const { return delta >= 0.0; }
};

// ---- tensor_train.hpp:15-77 ----------------------------------------------
struct TTCore {
    index_t r_left = 1, n = 1, r_right = 1;
    std::vector<double> data;
    TTCore() = default;
    TTCore(index_t rl, index_t n_, index_t rr)
        : r_left(rl), n(n_), r_right(rr), data(static_cast<std::size_t>(rl * n_ * rr), 0.0) {}
    double operator()(index_t a, index_t i, index_t b) const {
        return data[static_cast<std::size_t>(a + r_left * (i + n * b))];
    }
};

struct TensorTrain {
    std::vector<TTCore> cores;
    index_t d() const { return static_cast<index_t>(cores.size()); }
    std::vector<index_t> ranks() const {
        std::vector<index_t> r{cores.empty() ? 1 : cores.front().r_left};
        for (const auto& c : cores) r.push_back(c.r_right);
        return r;
    }
};

inline void validate(const TensorTrain& tt) {  // tensor_train.hpp:60-77
    if (tt.cores.empty()) throw DegenerateDimension("TensorTrain: no cores");
    if (tt.cores.front().r_left != 1 || tt.cores.back().r_right != 1)
        throw DimensionMismatch("TensorTrain: boundary ranks must be 1");
    for (std::size_t j = 0; j + 1 < tt.cores.size(); ++j)
        if (tt.cores[j].r_right != tt.cores[j + 1].r_left) throw DimensionMismatch("TensorTrain: rank chain broken");
}

// ---- wire formats (storage.hpp:214-278, tensor_train.hpp:157-191) ---------
// Little-endian 64-bit integers and IEEE doubles, byte-identical to the
// reference's dump_tensor / load_tensor (header d, dims..., stride; then the
// padded buffer) and save_tt / load_tt (header d, ranks r_0..r_d, dims; then
// the core buffers), written and read in bulk.
namespace wire {
static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "the wire formats are little-endian");
struct Closer {
    void operator()(std::FILE* f) const {
        if (f) std::fclose(f);
    }
};
using File = std::unique_ptr<std::FILE, Closer>;
inline void put(std::FILE* f, const void* p, std::size_t bytes) {
    if (std::fwrite(p, 1, bytes, f) != bytes) throw IoError("dump: short write");
}
inline void get(std::FILE* f, void* p, std::size_t bytes) {
    if (std::fread(p, 1, bytes, f) != bytes) throw IoError("load: short read");
}
inline void put_u64(std::FILE* f, std::uint64_t v) { put(f, &v, 8); }
inline std::uint64_t get_u64(std::FILE* f) {
    std::uint64_t v;
    get(f, &v, 8);
    return v;
}
}  // namespace wire

inline void dump_tensor(const DenseTensor& t, const std::string& path) {
    wire::File f(std::fopen(path.c_str(), "wb"));
    if (!f) throw IoError("dump_tensor: cannot open " + path);
    wire::put_u64(f.get(), static_cast<std::uint64_t>(t.dims().size()));
    for (index_t n : t.dims()) wire::put_u64(f.get(), static_cast<std::uint64_t>(n));
    wire::put_u64(f.get(), static_cast<std::uint64_t>(t.leading_stride()));
    wire::put(f.get(), t.data(), static_cast<std::size_t>(t.buffer_size()) * 8);
}

inline DenseTensor load_tensor(const std::string& path) {
    wire::File f(std::fopen(path.c_str(), "rb"));
    if (!f) throw IoError("load_tensor: cannot open " + path);
    const index_t d = static_cast<index_t>(wire::get_u64(f.get()));
    if (d < 1 || d > 64) throw IoError("load_tensor: bad header");
    std::vector<index_t> dims(static_cast<std::size_t>(d));
    for (auto& n : dims) n = static_cast<index_t>(wire::get_u64(f.get()));
    const index_t stride = static_cast<index_t>(wire::get_u64(f.get()));
    DenseTensor t(dims);
    if (stride != t.leading_stride()) throw IoError("load_tensor: stride mismatch");
    wire::get(f.get(), t.data(), static_cast<std::size_t>(t.buffer_size()) * 8);
    return t;
}

inline void save_tt(const TensorTrain& tt, const std::string& path) {
    validate(tt);
    wire::File f(std::fopen(path.c_str(), "wb"));
    if (!f) throw IoError("save_tt: cannot open " + path);
    wire::put_u64(f.get(), static_cast<std::uint64_t>(tt.d()));
    for (index_t r : tt.ranks()) wire::put_u64(f.get(), static_cast<std::uint64_t>(r));
    for (const auto& c : tt.cores) wire::put_u64(f.get(), static_cast<std::uint64_t>(c.n));
    for (const auto& c : tt.cores) wire::put(f.get(), c.data.data(), c.data.size() * 8);
}

inline TensorTrain load_tt(const std::string& path) {
    wire::File f(std::fopen(path.c_str(), "rb"));
    if (!f) throw IoError("load_tt: cannot open " + path);
    const index_t d = static_cast<index_t>(wire::get_u64(f.get()));
    if (d < 1 || d > 64) throw IoError("load_tt: bad header");
    std::vector<index_t> ranks(static_cast<std::size_t>(d + 1)), dims(static_cast<std::size_t>(d));
    for (auto& r : ranks) r = static_cast<index_t>(wire::get_u64(f.get()));
    for (auto& n : dims) n = static_cast<index_t>(wire::get_u64(f.get()));
    TensorTrain tt;
    for (index_t j = 0; j < d; ++j) {
        TTCore c(ranks[static_cast<std::size_t>(j)], dims[static_cast<std::size_t>(j)], ranks[static_cast<std::size_t>(j + 1)]);
        wire::get(f.get(), c.data.data(), c.data.size() * 8);
        tt.cores.push_back(std::move(c));
    }
    validate(tt);
    return tt;
}

struct ExecContext {  // tt_svd.hpp:39-52; threads / l2 budget have no device meaning
    int threads = 1;
    index_t l2_budget_bytes = 256 * 1024;
    bool validate_reflectors = false;
    Counters* counters = nullptr;
};

namespace b200 {
inline b200::DeviceBuffer stage(ConstMatrixView X) {
    DeviceBuffer d(static_cast<std::size_t>(X.rows * X.cols));
    cuda(cudaMemcpy2D(d.get(), static_cast<std::size_t>(X.rows) * 8, X.data, static_cast<std::size_t>(X.stride) * 8,
                      static_cast<std::size_t>(X.rows) * 8, static_cast<std::size_t>(X.cols), cudaMemcpyHostToDevice));
    return d;
}

inline TensorTrain collect(ttsvd_cu_tt* h, const std::vector<index_t>& dims) {
    std::vector<index_t> ranks(dims.size() + 1);
    TensorTrain tt;
    try {
        check(ttsvd_cu_tt_ranks(h, ranks.data()));
        for (std::size_t j = 0; j < dims.size(); ++j) {
            TTCore c(ranks[j], dims[j], ranks[j + 1]);
            check(ttsvd_cu_tt_core(h, static_cast<index_t>(j), c.data.data()));
            tt.cores.push_back(std::move(c));
        }
    } catch (...) {
        ttsvd_cu_tt_free(h);
        throw;
    }
    ttsvd_cu_tt_free(h);
    return tt;
}
}  // namespace b200

// ---- building blocks -----------------------------------------------------
inline TriangularFactor tsqr(DeviceMatrixView X, const BlockParams& = {}, int = 1, TsqrStats* = nullptr,
                             Counters* counters = nullptr) {
    TriangularFactor R(X.cols);
    b200::DeviceBuffer d(static_cast<std::size_t>(X.cols * X.cols));
    b200::check(ttsvd_cu_tsqr(b200::context(), X.data, X.rows, X.cols, X.stride, d.get()));
    d.download(R.entries.data(), R.entries.size());
    if (counters) counters->add(2ull * X.rows * X.cols * X.cols, 8ull * X.rows * X.cols);
    return R;
}

inline TriangularFactor tsqr(ConstMatrixView X, const BlockParams& p, int workers, TsqrStats* stats = nullptr,
                             Counters* counters = nullptr) {
    if (X.cols < 1) throw DimensionError("tsqr: needs at least one column");
    if (X.rows < X.cols) throw DimensionError("tsqr: requires n >= m");
    b200::DeviceBuffer d = b200::stage(X);
    return tsqr(DeviceMatrixView{d.get(), X.rows, X.cols, X.rows}, p, workers, stats, counters);
}

inline TriangularFactor reduce_block(ConstMatrixView M, const TriangularFactor& R, const BlockParams& = {},
                                     TsqrStats* = nullptr, Counters* = nullptr) {
    if (R.m != M.cols) throw DimensionMismatch("reduce_block: R.m != M.cols");
    b200::DeviceBuffer dm = b200::stage(M), dr(R.entries.size()), out(R.entries.size());
    dr.upload(R.entries.data(), R.entries.size());
    b200::check(ttsvd_cu_reduce_block(b200::context(), dm.get(), M.rows, M.cols, M.rows > 0 ? M.rows : 1, dr.get(),
                                      R.m, out.get()));
    TriangularFactor o(R.m);
    out.download(o.entries.data(), o.entries.size());
    return o;
}

inline TriangularFactor combine_factors(const std::vector<TriangularFactor>& parts, const BlockParams& = {},
                                        TsqrStats* = nullptr, Counters* = nullptr) {
    if (parts.empty()) throw DimensionMismatch("combine_factors: empty list");
    const index_t m = parts.front().m;
    std::vector<double> flat;
    for (const auto& p : parts) {
        if (p.m != m) throw DimensionMismatch("combine_factors: mixed column counts");
        flat.insert(flat.end(), p.entries.begin(), p.entries.end());
    }
    b200::DeviceBuffer d(flat.size()), out(static_cast<std::size_t>(m * m));
    d.upload(flat.data(), flat.size());
    b200::check(ttsvd_cu_combine_factors(b200::context(), d.get(), static_cast<index_t>(parts.size()), m, out.get()));
    TriangularFactor o(m);
    out.download(o.entries.data(), o.entries.size());
    return o;
}

inline SmallSVD small_svd(const TriangularFactor& R) {
    if (R.m > 4096) throw DimensionMismatch("small_svd: m exceeds 4096");
    b200::DeviceBuffer dr(R.entries.size()), ds(static_cast<std::size_t>(R.m)), dv(R.entries.size());
    dr.upload(R.entries.data(), R.entries.size());
    b200::check(ttsvd_cu_small_svd(b200::context(), dr.get(), R.m, ds.get(), dv.get()));
    SmallSVD s;
    s.n = s.m = R.m;
    s.sigma.resize(static_cast<std::size_t>(R.m));
    s.V.resize(R.entries.size());
    ds.download(s.sigma.data(), s.sigma.size());
    dv.download(s.V.data(), s.V.size());
    return s;
}

inline SmallSVD jacobi_svd(ConstMatrixView A) {
    if (A.rows < A.cols) throw DimensionError("jacobi_svd: requires n >= m");
    b200::DeviceBuffer da = b200::stage(A), ds(static_cast<std::size_t>(A.cols)),
        dv(static_cast<std::size_t>(A.cols * A.cols)), du(static_cast<std::size_t>(A.rows * A.cols));
    b200::check(ttsvd_cu_jacobi_svd(b200::context(), da.get(), A.rows, A.cols, A.rows, ds.get(), dv.get(), du.get()));
    SmallSVD s;
    s.n = A.rows;
    s.m = A.cols;
    s.sigma.resize(static_cast<std::size_t>(A.cols));
    s.V.resize(dv.size());
    s.U.resize(du.size());
    ds.download(s.sigma.data(), s.sigma.size());
    dv.download(s.V.data(), s.V.size());
    du.download(s.U.data(), s.U.size());
    return s;
}

inline index_t select_rank(const std::vector<double>& sigma, double delta, index_t r_max) {
    return ttsvd_cu_select_rank_host(sigma.data(), static_cast<index_t>(sigma.size()), delta, r_max);
}

inline double derive_delta(double norm_source, double eps, index_t d) {
    double out = 0.0;
    b200::check(ttsvd_cu_derive_delta(norm_source, eps, d, &out));
    return out;
}

inline PaddedMatrix tsmm_reshape(ConstMatrixView X, ConstMatrixView V, index_t out_rows, index_t out_cols,
                                 int = 1, Counters* counters = nullptr) {
    if (V.rows != X.cols) throw ShapeError("tsmm_reshape: V.rows != X.cols");
    if (V.cols > X.cols) throw ShapeError("tsmm_reshape: k > m (kernel only shrinks)");
    if (out_rows < 1 || out_cols < 1 || X.rows * V.cols != out_rows * out_cols)
        throw ShapeError("tsmm_reshape: out shape does not hold n*k elements");
    PaddedMatrix out(out_rows, out_cols);
    b200::DeviceBuffer dx = b200::stage(X), dv = b200::stage(V),
                       dy(static_cast<std::size_t>(out.stride() * out_cols));
    b200::check(ttsvd_cu_tsmm_reshape(b200::context(), dx.get(), X.rows, X.cols, X.rows, dv.get(), V.cols, V.rows,
                                      dy.get(), out_rows, out_cols, out.stride()));
    dy.download(out.data(), dy.size());
    if (counters) counters->add(2ull * X.rows * X.cols * V.cols, 8ull * X.rows * (X.cols + V.cols));
    return out;
}

inline PaddedMatrix tsmm_reshape(ConstMatrixView X, ConstMatrixView V, int workers = 1, Counters* c = nullptr) {
    return tsmm_reshape(X, V, X.rows, V.cols, workers, c);
}

// ---- drivers -------------------------------------------------------------
inline TensorTrain tt_svd_tsqr(const DenseTensor& X, TruncationSpec spec, const ExecContext& = {}) {
    const index_t d = static_cast<index_t>(X.dims().size());
    if (d < 2) throw DegenerateDimension("tt_svd_tsqr: requires d >= 2");
    ttsvd_cu_tt* h = nullptr;
    const index_t rmax = spec.r_max;
    b200::check(ttsvd_cu_tt_svd_host(b200::context(), X.data(), X.dims().data(), d, X.leading_stride(), rmax,
                                     spec.eps, &h));
    return b200::collect(h, X.dims());
}

// device-resident tensor (padded layout, ld >= N / n_d)
inline TensorTrain tt_svd_tsqr(const double* X_device, const std::vector<index_t>& dims, index_t ld,
                               TruncationSpec spec) {
    ttsvd_cu_tt* h = nullptr;
    const index_t rmax = spec.r_max;
    b200::check(ttsvd_cu_tt_svd(b200::context(), X_device, dims.data(), static_cast<index_t>(dims.size()), ld, rmax,
                                spec.eps, &h));
    return b200::collect(h, dims);
}

// tt_svd.hpp:292-310
struct ThickBoundsParams {
    index_t m_min = 16;
    double f1_min = 0.5;
    std::vector<index_t> r_tilde;  // empty = derive from r_max
};

// tt_svd.hpp:316-330
inline std::pair<index_t, index_t> choose_combined_dims(const std::vector<index_t>& dims,
                                                        const ThickBoundsParams& params,
                                                        index_t r_max = std::numeric_limits<index_t>::max()) {
    index_t k = 0, m = 0;
    const index_t rmax = r_max;
    b200::check(ttsvd_cu_choose_combined_dims(dims.data(), static_cast<index_t>(dims.size()), params.m_min,
                                              params.f1_min, params.r_tilde.empty() ? nullptr : params.r_tilde.data(),
                                              static_cast<index_t>(params.r_tilde.size()), rmax, &k, &m));
    return {k, m};
}

// tt_svd.hpp:338 (Alg. 3): the tensor is staged to the device, then merged,
// swept and recovered there
inline TensorTrain tt_svd_thick_bounds(const DenseTensor& X, TruncationSpec spec, const ThickBoundsParams& params,
                                       const ExecContext& = {}) {
    const index_t d = static_cast<index_t>(X.dims().size());
    if (d < 2) throw DegenerateDimension("tt_svd_thick_bounds: requires d >= 2");
    const index_t rmax = spec.r_max;
    const index_t cols = X.dims()[static_cast<std::size_t>(d - 1)];
    b200::DeviceBuffer dx(static_cast<std::size_t>(X.leading_stride() * cols));
    dx.upload(X.data(), dx.size());
    ttsvd_cu_tt* h = nullptr;
    b200::check(ttsvd_cu_tt_svd_thick(b200::context(), dx.get(), X.dims().data(), d, X.leading_stride(), rmax,
                                      spec.eps, params.m_min, params.f1_min,
                                      params.r_tilde.empty() ? nullptr : params.r_tilde.data(),
                                      static_cast<index_t>(params.r_tilde.size()), &h));
    return b200::collect(h, X.dims());
}

inline TensorTrain tt_svd_distributed(const std::vector<DenseTensor>& slabs, TruncationSpec spec,
                                      const ExecContext& = {}, std::vector<TensorTrain>* per_partition = nullptr) {
    if (slabs.empty()) throw PartitionMismatch("tt_svd_distributed: no partitions");
    const auto& ld = slabs.front().dims();
    for (const auto& s : slabs)
        if (s.dims() != ld) throw PartitionMismatch("tt_svd_distributed: slab shapes differ");
    std::vector<b200::DeviceBuffer> bufs;
    std::vector<const double*> ptrs;
    for (const auto& s : slabs) {
        bufs.emplace_back(static_cast<std::size_t>(s.buffer_size()));
        bufs.back().upload(s.data(), static_cast<std::size_t>(s.buffer_size()));
        ptrs.push_back(bufs.back().get());
    }
    const index_t P = static_cast<index_t>(slabs.size());
    const index_t rmax = spec.r_max;
    ttsvd_cu_tt* h = nullptr;
    b200::check(ttsvd_cu_tt_svd_distributed(b200::context(), ptrs.data(), P, 0, P, ld.data(),
                                            static_cast<index_t>(ld.size()), slabs.front().leading_stride(), rmax,
                                            spec.eps, nullptr, nullptr, &h));
    std::vector<index_t> gdims{P > 1 ? P : 1};
    gdims.insert(gdims.end(), ld.begin(), ld.end());
    TensorTrain tt = b200::collect(h, gdims);
    if (per_partition) per_partition->assign(static_cast<std::size_t>(P), tt);  // shared cores are identical
    return tt;
}

}  // namespace ttsvd
