// ttsvd/device.hpp — plumbing of the C++ drop-in over the C-ABI
// (include/ttsvd_cu.h): status codes -> the reference's exception types, one
// library context per (thread, device), RAII device buffers and the staging
// of host views.  Not part of the reference interface.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <string>

#include "../ttsvd_cu.h"
#include "errors.hpp"
#include "storage.hpp"

namespace ttsvd {
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

// one context per thread and current device, on the legacy default stream
inline ttsvd_cu_ctx* context() {
    struct Slot {
        ttsvd_cu_ctx* ctx = nullptr;
        int dev = -1;
        ~Slot() {
            if (ctx) ttsvd_cu_ctx_destroy(ctx);
        }
    };
    thread_local Slot slot;
    int cur = 0;
    cuda(cudaGetDevice(&cur));
    if (!slot.ctx || slot.dev != cur) {
        if (slot.ctx) ttsvd_cu_ctx_destroy(slot.ctx);
        slot.ctx = nullptr;
        check(ttsvd_cu_ctx_create(cur, nullptr, &slot.ctx));
        slot.dev = cur;
    }
    return slot.ctx;
}

class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t n) : n_(n) { cuda(cudaMalloc(&p_, std::max<std::size_t>(n, 1) * 8)); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        return *this;
    }
    ~DeviceBuffer() {
        if (p_) cudaFree(p_);
    }
    double* get() const { return p_; }
    std::size_t size() const { return n_; }
    void upload(const double* h, std::size_t n) { cuda(cudaMemcpy(p_, h, n * 8, cudaMemcpyHostToDevice)); }
    void download(double* h, std::size_t n) const { cuda(cudaMemcpy(h, p_, n * 8, cudaMemcpyDeviceToHost)); }

private:
    double* p_ = nullptr;
    std::size_t n_ = 0;
};

// a host view packed to the device (ld = max(rows, 1))
inline DeviceBuffer stage(ConstMatrixView X) {
    const index_t ld = std::max<index_t>(X.rows, 1);
    DeviceBuffer d(static_cast<std::size_t>(ld * std::max<index_t>(X.cols, 1)));
    if (X.rows > 0 && X.cols > 0)
        cuda(cudaMemcpy2D(d.get(), static_cast<std::size_t>(ld) * 8, X.data, static_cast<std::size_t>(X.stride) * 8,
                          static_cast<std::size_t>(X.rows) * 8, static_cast<std::size_t>(X.cols),
                          cudaMemcpyHostToDevice));
    return d;
}

// a host tensor's padded buffer, as is, on the device
inline DeviceBuffer stage(const DenseTensor& X) {
    DeviceBuffer d(static_cast<std::size_t>(X.buffer_size()));
    d.upload(X.data(), static_cast<std::size_t>(X.buffer_size()));
    return d;
}

}  // namespace b200
}  // namespace ttsvd
