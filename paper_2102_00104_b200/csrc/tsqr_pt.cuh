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

#ifndef PT_THREADS
#define PT_THREADS 256
#endif
constexpr int kPtThreads = PT_THREADS;

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
            const double inv = fast_rsqrt(nrm2);
            const double nr = nrm2 * inv;
            const double sg = (u0 > 0.0) ? 1.0 : -1.0;
            double alpha = -sg * nr;
            if (sp == 0.0 && u0 != 0.0) alpha = u0;  // H = I
            if (nrm2 == 0.0) alpha = sqrt(2.0 * DBL_MIN);  // all-zero u
            if (j + 1 < M) {
                double tj = 1.0 + fabs(u0) * inv;
                double scale = sg * fast_rcp(fabs(u0) + nr);
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

namespace ttsvd_b200 {

// K_TSQR for 8 < m <= 32: group streams.  P lanes of a warp share one
// stream: lane q owns columns q, q + P, q + 2P, ... of the U-row fold (and
// those columns of R, registers), so a stream's registers stay ~M^2/(2P).
// Reflector j: the owner lane of column j broadcasts its U pivot values and
// R[j][j] within the group (shuffles of width P); every lane derives the
// reflector redundantly (same bits on every lane) and updates its own
// columns c > j.  Rows are strided as in tsqr_pt_kernel; the warp's lanes
// run the same number of folds (rows past n, and streams past T, fold zeros).
struct GsArgs {
    const double* X;
    int64_t n, ld;
    int m;
    int64_t T;    // streams
    double* out;  // stacked factors (T m x m, ld ldo), or R (m x m, ld m) when T == 1
    int64_t ldo;
    ColSplit cs;  // column layout of X (tsqr_gt_kernel only; q = 0: plain)
    // tsqr_gt_kernel in row chunks (the host entry overlaps the H2D of X with
    // the sweep): this launch folds slices [sl_lo, sl_hi) (sl_lo a multiple of
    // the grid's warp count; sl_hi = 0: all), the streams' running R factors
    // are loaded from `state` first (flag 1) and saved there instead of being
    // written out (flag 2) — bit-identical to one launch over all slices
    int64_t sl_lo, sl_hi;
    double* state;
    int flags;
};

#ifndef GS_MINB
#define GS_MINB 1
#endif
template <int M, int P, int U>
__global__ void __launch_bounds__(kPtThreads, GS_MINB) tsqr_gs_kernel(GsArgs a) {
    constexpr int MC = M / P;
    constexpr int G = 32 / P;
    const int lane = threadIdx.x & 31, q = lane % P;
    const int64_t s0 = (((int64_t)blockIdx.x * kPtThreads + threadIdx.x) >> 5) * G;
    if (s0 >= a.T) return;  // warp-uniform
    const int64_t s = s0 + lane / P;
    const bool live = s < a.T;
    const int m = a.m;
    double R[M][MC];
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int k = 0; k < MC; ++k) R[i][k] = 0.0;
    const int64_t step = (int64_t)U * a.T;
    const int64_t trips = (a.n - s0 + step - 1) / step;
    for (int64_t t = 0; t < trips; ++t) {
        const int64_t r0 = s + t * step;
        double x[U][MC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t row = r0 + (int64_t)u * a.T;
            const bool ok = live && row < a.n;
#pragma unroll
            for (int k = 0; k < MC; ++k) {
                const int c = q + P * k;
                x[u][k] = (ok && c < m) ? __ldcs(a.X + (int64_t)c * a.ld + row) : 0.0;
            }
        }
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const int qj = j % P, kj = j / P;
            double p[U];
            double sp = 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                p[u] = __shfl_sync(kFull, x[u][kj], qj, P);
                sp = fma(p[u], p[u], sp);
            }
            const double u0 = __shfl_sync(kFull, R[j][kj], qj, P);
            const double nrm2 = u0 * u0 + sp;
            const double inv = fast_rsqrt(nrm2);
            const double nr = nrm2 * inv;
            const double sg = (u0 > 0.0) ? 1.0 : -1.0;
            double alpha = -sg * nr;
            if (sp == 0.0 && u0 != 0.0) alpha = u0;        // H = I
            if (nrm2 == 0.0) alpha = sqrt(2.0 * DBL_MIN);  // all-zero u
            if (j + 1 < M) {
                double tj = 1.0 + fabs(u0) * inv;
                double scale = sg * fast_rcp(fabs(u0) + nr);
                if (sp == 0.0 && u0 != 0.0) {
                    tj = 0.0;
                    scale = 0.0;
                }
                if (nrm2 == 0.0) {
                    tj = 2.0;
                    scale = 0.0;
                }
#pragma unroll
                for (int k = 0; k < MC; ++k) {
                    if (k < kj || j > P * k + P - 2) continue;  // no column of this k lies right of j
                    const bool act = q + P * k > j;
                    double d = 0.0;
#pragma unroll
                    for (int u = 0; u < U; ++u) d = fma(p[u], x[u][k], d);
                    const double g = act ? tj * (R[j][k] + scale * d) : 0.0;
                    R[j][k] -= g;
                    const double f = g * scale;
#pragma unroll
                    for (int u = 0; u < U; ++u) x[u][k] = fma(-f, p[u], x[u][k]);
                }
            }
            if (q == qj) R[j][kj] = alpha;
        }
    }
    if (!live) return;
    double* o = a.out + (a.T == 1 ? 0 : s * m);
#pragma unroll
    for (int k = 0; k < MC; ++k) {
        const int c = q + P * k;
        if (c >= m) continue;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            if (i >= m) break;
            double v = 0.0;
            if (i <= P * k + P - 1) v = (i <= c) ? R[i][k] : 0.0;
            o[(int64_t)c * a.ldo + i] = v;
        }
    }
}

}  // namespace ttsvd_b200
