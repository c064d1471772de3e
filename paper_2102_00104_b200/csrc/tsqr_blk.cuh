// Shared pieces of the m > 32 TSQR kernels (tsqr_la.cuh, tsqr_t128.cuh):
// job arguments, the DMMA m8n8k4 f64 wrapper, and the packed panel-major
// layout of the running R (row panel p = 32 rows x (M - 32p) columns,
// column-major, ld 32: only the upper triangle is stored and every DMMA
// fragment of R is a contiguous 2 KiB run), plus the layout conversions.
#pragma once

#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kBlkRows = 32;    // tile rows (one per lane in the panel)
constexpr int kBlkLdb = 36;     // smem ld of the tile: fragment loads in 2 wavefronts
constexpr int kTld = 33;        // smem ld of S and T

struct BlkArgs {
    const double* X;        // mode 0: matrix (n x m, ld); mode 1: parts (count x blk_rsize(M))
    int64_t n;              // mode 0: rows; mode 1: number of parts at this level
    int64_t ld;
    double* Rws;            // per-job running R / output (packed panel layout, blk_rsize(M))
    const double* R_init0;  // mode 0 only: starting R (packed panel layout) or nullptr
    int m;                  // logical columns
    int M;                  // padded columns (multiple of 32)
    int mode;
    long long* prof;        // optional per-CTA phase cycle counters (8 per CTA), diagnostics
};

// offset of row panel p in the packed layout, and the packed size
__host__ __device__ __forceinline__ int64_t blk_roff(int p, int M) {
    return 32 * ((int64_t)p * M - 32 * (int64_t)p * (p - 1) / 2);
}
__host__ __device__ __forceinline__ int64_t blk_rsize(int M) { return blk_roff(M / 32, M); }

// packed panel-major M x M factor -> leading m x m block, column-major ld m
__global__ void copy_leading_kernel(const double* Rws, int M, int m, double* R) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += gridDim.x * blockDim.x) {
        const int j = e / m, i = e - j * m;
        const int p = i >> 5;
        R[e] = (i <= j) ? Rws[blk_roff(p, M) + (int64_t)(j - 32 * p) * 32 + (i & 31)] : 0.0;
    }
}

// P parts of m x m (ld m, upper triangular) -> packed panel-major M x M parts
__global__ void pack_parts_kernel(const double* parts, int64_t P, int m, int M, double* out) {
    const int64_t RS = blk_rsize(M);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < P * RS; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = e / RS;
        int64_t o = e - q * RS;
        int p = 0;
        while (p + 1 < M / 32 && blk_roff(p + 1, M) <= o) ++p;
        o -= blk_roff(p, M);
        const int c = 32 * p + (int)(o >> 5), row = 32 * p + (int)(o & 31);
        out[e] = (row < m && c < m && row <= c) ? parts[q * (int64_t)m * m + (int64_t)c * m + row] : 0.0;
    }
}

}  // namespace ttsvd_b200
