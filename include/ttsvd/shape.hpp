// ttsvd/shape.hpp — shape.hpp:13-86 on the B200 path: index type, the padded
// leading stride rule (through the C-ABI, so host and device agree) and the
// extent list of a tensor.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <string>
#include <vector>

#include "../ttsvd_cu.h"
#include "errors.hpp"

namespace ttsvd {

using index_t = std::int64_t;

// desk / cluster scale bound on element counts (shape.hpp:16)
inline constexpr index_t kMaxElements = index_t{1} << 40;

// odd multiple of 64 >= n_rows (64 at least): shape.hpp:22-28
inline index_t padded_stride(index_t n_rows) {
    if (n_rows < 1) throw DimensionError("padded_stride: n_rows must be >= 1");
    return ttsvd_cu_padded_stride(n_rows);
}

class Shape {
public:
    Shape() = default;
    Shape(std::initializer_list<index_t> extents) : n_(extents) { check(); }
    explicit Shape(std::vector<index_t> extents) : n_(std::move(extents)) { check(); }

    index_t d() const { return static_cast<index_t>(n_.size()); }
    index_t dim(index_t i) const { return n_[static_cast<std::size_t>(i)]; }
    const std::vector<index_t>& dims() const { return n_; }

    // product of all extents, refused above kMaxElements
    index_t total() const { return product(0, d()); }
    // product of the first k / last k extents
    index_t leading(index_t k) const { return product(0, k); }
    index_t trailing(index_t k) const { return product(d() - k, d()); }

    std::string to_string() const {
        std::string out;
        for (index_t n : n_) out += (out.empty() ? "" : "x") + std::to_string(n);
        return out;
    }
    bool operator==(const Shape& o) const { return n_ == o.n_; }

private:
    index_t product(index_t lo, index_t hi) const {
        index_t p = 1;
        for (index_t i = lo; i < hi; ++i) {
            const index_t n = n_[static_cast<std::size_t>(i)];
            if (p > kMaxElements / n) throw AllocationError("Shape::total: element count exceeds 2^40");
            p *= n;
        }
        return p;
    }
    void check() const {
        if (n_.empty()) throw DimensionError("Shape: needs at least one dimension");
        for (index_t n : n_)
            if (n < 1) throw DimensionError("Shape: extents must be >= 1");
        (void)total();
    }

    std::vector<index_t> n_;
};

}  // namespace ttsvd
