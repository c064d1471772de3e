// ttsvd/counters.hpp — counters.hpp:12-25.  The device drivers tally the
// algorithmic work of every kernel they launch (TSQR 2 n m^2 flops and one
// read of X, TSMM 2 n m k flops and 8 n (m + k) bytes, the reorder 16 n m
// bytes) on the calling thread; the values are exact functions of the shapes.
#pragma once

#include <cstdint>

namespace ttsvd {

struct Counters {
    std::uint64_t flops = 0;
    std::uint64_t bytes = 0;

    void add(std::uint64_t f, std::uint64_t b) {
        flops += f;
        bytes += b;
    }
    Counters& operator+=(const Counters& o) {
        add(o.flops, o.bytes);
        return *this;
    }
};

}  // namespace ttsvd
