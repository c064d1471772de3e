// K_TSQR for small work matrices with 32 < m <= 64 (config 1's m = 64 steps,
// 64..16384 rows): a tree of register-resident tile QRs instead of the
// cooperative grid (gqr: one grid barrier per reflector, ~5 us each even at
// one CTA).
//
//   Level: CTA t factorises rows [t TR, (t+1) TR) of the current matrix
//   (TR = 256 rows, 64 columns in 512 threads) and writes its m x m R into
//   rows [t m, (t+1) m) of a stacked matrix; the stack (4x fewer rows) is
//   the next level's input, until one tile is left (tsqr.hpp:204-240's
//   combine, as a 4-ary tree in index order).
//   Tile: warp w holds rows 32 (w % 8) .. + 31 of column 32 (w / 8) + lane
//   in registers (a column per lane, as t2_panel).  Reflector j: the pivot
//   column (rows > j, zero above) and the pivot row sit in shared memory;
//   every thread forms the dot of the pivot column with its own column over
//   its 32 rows, the eight row blocks' partials meet in shared memory
//   (fixed order), every thread derives the same reflector (LAPACK dlarfg
//   normalisation and the reference's zero rules, tsqr.hpp:120-160, as
//   gqr) and updates its column.  Two CTA barriers per reflector, no
//   shuffles; warps whose columns or rows are all finished skip the work.
#pragma once

#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kSqThreads = 512;
constexpr int kSqRows = 256;  // tile rows (8 row blocks x 2 column halves of 32)
constexpr int64_t kSqMaxRows = 1 << 16;  // beyond: gqr / t128

struct SqArgs {
    const double* X;  // rows x m, ld (column-major)
    int64_t n, ld;
    int m;            // 32 < m <= 64
    int64_t T;        // tiles (CTAs)
    double* out;      // stacked R factors (T m x m, ld ldo), or R (m x m, ld m) when T == 1
    int64_t ldo;
};

__global__ void __launch_bounds__(kSqThreads, 1) tsqr_sq_kernel(SqArgs a) {
    constexpr int RB = 8;  // row blocks
    __shared__ double pv[2][kSqRows];      // pivot column below the pivot (zero at and above it)
    __shared__ double prow[2][64];         // pivot row
    __shared__ double dpart[2][RB][64];    // per-row-block dots
    __shared__ double pu0[2];              // pivot entry
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int h = warp / RB, rb = warp % RB;
    const int col = 32 * h + lane;  // my column
    const int i0 = 32 * rb;         // my first tile row
    const int m = a.m;
    const int64_t r0 = (int64_t)blockIdx.x * kSqRows;
    const int rows = (int)((a.n - r0) < kSqRows ? (a.n - r0) : kSqRows);
    double x[32];
    {
        const double* src = a.X + (int64_t)col * a.ld + r0 + i0;
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = (col < m && i0 + i < rows) ? src[i] : 0.0;
    }
    const int nref = m < rows ? m : rows;
    // Reflectors in blocks of 32: reflector j = 32 blk + jj (jj unrolled, so
    // the pivot's register index is a constant) has its pivot row in row
    // block blk and its pivot column in column half blk.  (A rolled loop
    // with selects or a jump table for x[jj] measured slower: 114 vs 90 us
    // per 256 x 64 tile.)
    for (int blk = 0; 32 * blk < nref; ++blk) {
        const bool hold = rb == blk;       // my warp holds the pivot rows of this block
        const bool pivh = h == blk;        // my warp holds the pivot columns of this block
        // publish reflector 32 blk's pivot column (full rows; the holder
        // block masks at use) and pivot row
        if (pivh && lane == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) pv[0][i0 + i] = x[i];
        }
        if (hold) {
            prow[0][col] = x[0];
            if (pivh && lane == 0) pu0[0] = x[0];
        }
        __syncthreads();
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
            const int j = 32 * blk + jj;
            if (j >= nref) break;
            const int b = jj & 1;
            // warps with a column >= j and a row > j (or the pivot row)
            const bool wact = 32 * h + 31 >= j && i0 + 31 >= j && i0 < rows;
            double d = 0.0;
            if (wact) {
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                if (hold) {
#pragma unroll
                    for (int i = jj + 1; i < 32; ++i) acc[i & 3] = fma(pv[b][i0 + i], x[i], acc[i & 3]);
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i & 3] = fma(pv[b][i0 + i], x[i], acc[i & 3]);
                }
                d = (acc[0] + acc[1]) + (acc[2] + acc[3]);
            }
            dpart[b][rb][col] = d;
            __syncthreads();
            double dv[RB], sv[RB];
#pragma unroll
            for (int q = 0; q < RB; ++q) {
                dv[q] = dpart[b][q][col];
                sv[q] = dpart[b][q][j];
            }
            const double dc = ((dv[0] + dv[1]) + (dv[2] + dv[3])) + ((dv[4] + dv[5]) + (dv[6] + dv[7]));
            const double sp = ((sv[0] + sv[1]) + (sv[2] + sv[3])) + ((sv[4] + sv[5]) + (sv[6] + sv[7]));
            const double u0 = pu0[b];
            const double nrm2 = u0 * u0 + sp;
            const double inv = fast_rsqrt(nrm2);
            const double nr = nrm2 * inv;
            const double au = fabs(u0);
            const double sg = (u0 > 0.0) ? 1.0 : -1.0;
            double alpha = -sg * nr, tj = 1.0 + au * inv, scale = sg * fast_rcp(au + nr);
            if (sp == 0.0 && u0 != 0.0) {  // H = I
                alpha = u0;
                tj = 0.0;
                scale = 0.0;
            }
            if (nrm2 == 0.0) {  // all-zero u
                alpha = sqrt(2.0 * DBL_MIN);
                tj = 2.0;
                scale = 0.0;
            }
            if (wact) {
                // columns > j: x -= f v on the rows > j (v = pivot column x
                // scale), x_jc -= g on the pivot row; the pivot column keeps
                // alpha on its pivot row (its rows below are never read again)
                const bool upd = col > j && col < m;
                const double g = upd ? tj * (prow[b][col] + scale * dc) : 0.0;
                const double f = g * scale;
                if (hold) {
#pragma unroll
                    for (int i = jj + 1; i < 32; ++i) x[i] = fma(-f, pv[b][i0 + i], x[i]);
                    x[jj] = (col == j) ? alpha : x[jj] - g;
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) x[i] = fma(-f, pv[b][i0 + i], x[i]);
                }
            }
            // publish reflector j+1's pivot column and row
            if (jj + 1 < 32 && j + 1 < nref) {
                if (pivh && lane == jj + 1) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) pv[b ^ 1][i0 + i] = x[i];
                }
                if (hold) {
                    prow[b ^ 1][col] = x[(jj + 1) & 31];
                    if (pivh && lane == jj + 1) pu0[b ^ 1] = x[(jj + 1) & 31];
                }
            }
            __syncthreads();
        }
    }
    // R (upper triangle of the first m rows) into the stack
    if (col < m) {
        double* dst = a.out + (int64_t)col * a.ldo + blockIdx.x * (int64_t)m;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (i0 + i < m) dst[i0 + i] = (i0 + i <= col) ? x[i] : 0.0;
    }
}

}  // namespace ttsvd_b200
