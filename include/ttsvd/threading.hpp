// ttsvd/threading.hpp — threading.hpp:14-55.  On the B200 path `workers`
// arguments no longer partition the arithmetic (the device grid does); these
// host helpers stay for callers that size their own host work with them.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <thread>
#include <utility>
#include <vector>

#include "shape.hpp"

namespace ttsvd {

// TTSVD_THREADS, else the logical core count (threading.hpp:14-21)
inline int default_threads() {
    if (const char* env = std::getenv("TTSVD_THREADS")) {
        const int v = std::atoi(env);
        if (v >= 1) return v;
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? static_cast<int>(hw) : 1;
}

// balanced contiguous ranges of [0, n), the first n % w one row longer
inline std::vector<std::pair<index_t, index_t>> partition_rows(index_t n, int workers) {
    const index_t w = std::max<index_t>(1, std::min<index_t>(workers < 1 ? 1 : workers, std::max<index_t>(n, 1)));
    std::vector<std::pair<index_t, index_t>> out;
    index_t at = 0;
    for (index_t i = 0; i < w; ++i) {
        const index_t len = n / w + (i < n % w ? 1 : 0);
        out.emplace_back(at, at + len);
        at += len;
    }
    return out;
}

}  // namespace ttsvd
