// K_TSQR for very narrow work matrices (m <= 8): thread streams.
//
// With m <= 8 a warp stream (tsqr_ws.cuh) leaves most of its lanes idle and
// is FP64-issue bound at ~1 TB/s.  Here every THREAD is a stream: it keeps
// its own R (m x m upper, registers) and folds U rows at a time into it with
// the structured [R; tile] Householder QR (m reflectors per tile, LAPACK
// dlarfg normalisation and the zero rules of tsqr.hpp:120-160, exactly as
// tsqr_ws/la_panel).  Thread s of T takes rows s, s + T, s + 2T, ... so the
// loads of a warp are coalesced.  Each thread writes its R into rows
// [s m, (s+1) m) of a stacked (T m) x m matrix, which the next level factors
// the same way with ~64x fewer threads (the flat-then-tree structure of
// tsqr.hpp:247-292).  Per row the work is ~m^2 + (rsqrt, rcp)/U flops, so the
// kernel streams X at HBM rate.
#pragma once

#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kPtThreads = 256;

struct PtArgs {
    const double* X;
    int64_t n, ld;
    int64_t T;    // thread streams
    double* out;  // stacked factors (T m x m, ld ldo), or R (m x m, ld m) when T == 1
    int64_t ldo;
};

template <int M, int U>
__global__ void __launch_bounds__(kPtThreads) tsqr_pt_kernel(PtArgs a) {
    const int64_t s = (int64_t)blockIdx.x * kPtThreads + threadIdx.x;
    if (s >= a.T) return;
    double R[M][M];
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int c = 0; c < M; ++c) R[i][c] = 0.0;
    const int64_t step = (int64_t)U * a.T;
    for (int64_t r0 = s; r0 < a.n; r0 += step) {
        double x[U][M];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t row = r0 + (int64_t)u * a.T;
#pragma unroll
            for (int c = 0; c < M; ++c) x[u][c] = (row < a.n) ? __ldcs(a.X + (int64_t)c * a.ld + row) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < M; ++j) {
            double sp = 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) sp = fma(x[u][j], x[u][j], sp);
            const double u0 = R[j][j];
            const double nrm2 = u0 * u0 + sp;
            const double inv = rsqrt(nrm2);
            const double nr = nrm2 * inv;
            const double sg = (u0 > 0.0) ? 1.0 : -1.0;
            double alpha = -sg * nr;
            if (sp == 0.0 && u0 != 0.0) alpha = u0;  // H = I
            if (nrm2 == 0.0) alpha = sqrt(2.0 * DBL_MIN);  // all-zero u
            if (j + 1 < M) {
                double tj = 1.0 + fabs(u0) * inv;
                double scale = sg * __drcp_rn(fabs(u0) + nr);
                if (sp == 0.0 && u0 != 0.0) {
                    tj = 0.0;
                    scale = 0.0;
                }
                if (nrm2 == 0.0) {
                    tj = 2.0;
                    scale = 0.0;
                }
#pragma unroll
                for (int c = 1; c < M; ++c) {
                    if (c <= j) continue;
                    double d = 0.0;
#pragma unroll
                    for (int u = 0; u < U; ++u) d = fma(x[u][j], x[u][c], d);
                    const double g = tj * (R[j][c] + scale * d);
                    R[j][c] -= g;
                    const double f = g * scale;
#pragma unroll
                    for (int u = 0; u < U; ++u) x[u][c] = fma(-f, x[u][j], x[u][c]);
                }
            }
            R[j][j] = alpha;
        }
    }
    double* o = a.out + (a.T == 1 ? 0 : s * M);
#pragma unroll
    for (int c = 0; c < M; ++c)
#pragma unroll
        for (int i = 0; i < M; ++i) o[(int64_t)c * a.ldo + i] = (i <= c) ? R[i][c] : 0.0;
}

}  // namespace ttsvd_b200
