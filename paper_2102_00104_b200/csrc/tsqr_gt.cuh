// K_TSQR for 8 < m <= 32, tall: group streams fed by the bulk-copy engine.
//
// Same fold as tsqr_gs_kernel (P lanes share a stream, lane q owns columns
// q, q + P, ... of the U-row [R; tile] Householder fold, tsqr.hpp:120-164),
// but the rows reach the lanes through shared memory: every warp streams
// contiguous SR = (32 / P) U row slices of X; lane c < m copies column c of a
// slice (SR x 8 bytes) with one cp.async.bulk (TMA, SASS UBLKCP) whose bytes
// are counted on the warp's own mbarrier, kGtStages slices in flight per
// warp.  The threads issue no global loads and never wait on a CTA barrier;
// the next slices land while the warp runs the m reflectors of the current
// one (with the direct loads of tsqr_gs the two resident warps per scheduler
// sat out a full HBM round trip every fold).  Stream g of a warp takes rows
// g, g + G, g + 2G, ... of the slice; the column stride of a stage is SR + G
// doubles so that the 32 lanes of a load hit every bank pair exactly twice.
// Warp w of W takes slices w, w + W, ...; its G streams write their factors
// to rows [(w G + g) m, (w G + g + 1) m) of the stacked matrix the warp-stream
// levels (tsqr_ws.cuh) finish.
// Requires X and ld 16-byte aligned (ld even); the last, partial slice is
// filled by ordinary loads.  Reads split-column views (ColSplit) in place.
#pragma once

#include <cfloat>
#include <cstdint>

#include "tsqr_pt.cuh"

namespace ttsvd_b200 {

constexpr int kGtStages = 2;

// NTH: threads per CTA (8 warps; 12 for m <= 16, where a third warp per
// scheduler gains more than the 168-register cap's spills cost)
template <int M, int P, int U, int ST = kGtStages, int NTH = kPtThreads>
constexpr size_t gt_smem_bytes() {
    return (size_t)(NTH / 32) * ST * M * ((32 / P) * U + 32 / P) * sizeof(double);
}

__device__ __forceinline__ void gt_mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void gt_mbar_expect(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void gt_mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n GT_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra GT_WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void gt_bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

template <int M, int P, int U, int MB = 1, int ST = kGtStages, int NTH = kPtThreads>
__global__ void __launch_bounds__(NTH, MB) tsqr_gt_kernel(GsArgs a) {
    constexpr int kGtWarps = NTH / 32;
    constexpr int MC = M / P;
    constexpr int G = 32 / P;
    constexpr int SR = G * U;   // rows per slice
    constexpr int CS = SR + G;  // column stride of a stage (doubles)
    extern __shared__ __align__(128) double gtsm[];
    __shared__ __align__(8) unsigned long long mbar[kGtWarps][ST];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane % P, g = lane / P;
    const int64_t W = (int64_t)gridDim.x * kGtWarps;
    const int64_t wg = (int64_t)blockIdx.x * kGtWarps + warp;
    const int m = a.m;
    double* xb = gtsm + (size_t)warp * ST * M * CS;
    const int64_t slices = (a.n + SR - 1) / SR;
    auto bar = [&](int s) { return (unsigned)__cvta_generic_to_shared(&mbar[warp][s]); };
    auto full = [&](int64_t sl) { return sl * SR + SR <= a.n; };
    auto issue = [&](int64_t sl, int s) {
        if (!full(sl)) return;  // the partial slice is filled when it is consumed
        if (lane == 0) gt_mbar_expect(bar(s), (unsigned)(m * SR * 8));
        __syncwarp();
        if (lane < m)
            gt_bulk_g2s((unsigned)__cvta_generic_to_shared(xb + ((size_t)s * M + lane) * CS),
                        a.X + col_off(lane, a.ld, a.cs) + sl * SR, (unsigned)(SR * 8), bar(s));
    };
    if (lane == 0)
        for (int s = 0; s < ST; ++s) gt_mbar_init(bar(s), 1);
    // columns m .. M-1 of every stage stay zero (the copies never touch them)
    for (int e = lane; e < ST * M * CS; e += 32)
        if ((e / CS) % M >= m) xb[e] = 0.0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    double R[M][MC];
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int k = 0; k < MC; ++k) R[i][k] = 0.0;
    const int64_t sl_end = a.sl_hi > 0 ? a.sl_hi : slices;
    double* st = a.state + ((size_t)wg * 32 + lane) * (M * MC);
    if (a.flags & 1) {
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int k = 0; k < MC; ++k) R[i][k] = st[i * MC + k];
    }
    int64_t sl = a.sl_lo + wg;
    for (int s = 0; s < ST; ++s)
        if (sl + (int64_t)s * W < sl_end) issue(sl + (int64_t)s * W, s);
    unsigned phase = 0;
    for (int s = 0; sl < sl_end; sl += W) {
        if (full(sl)) {
            gt_mbar_wait(bar(s), phase);
        } else {
            const int64_t r0 = sl * SR;
            for (int e = lane; e < m * SR; e += 32) {
                const int c = e / SR, r = e % SR;
                xb[((size_t)s * M + c) * CS + r] = (r0 + r < a.n) ? __ldcs(a.X + col_off(c, a.ld, a.cs) + r0 + r) : 0.0;
            }
            __syncwarp();
        }
        double x[U][MC];
        {
            const double* xs = xb + (size_t)s * M * CS + g;
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < MC; ++k) x[u][k] = xs[(q + P * k) * CS + G * u];
        }
        __syncwarp();  // the stage has been read: refill it
        if (sl + (int64_t)ST * W < sl_end) issue(sl + (int64_t)ST * W, s);
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
                    const double gm = act ? tj * (R[j][k] + scale * d) : 0.0;
                    R[j][k] -= gm;
                    const double f = gm * scale;
#pragma unroll
                    for (int u = 0; u < U; ++u) x[u][k] = fma(-f, p[u], x[u][k]);
                }
            }
            if (q == qj) R[j][kj] = alpha;
        }
        if (++s == ST) {
            s = 0;
            phase ^= 1;
        }
    }
    if (a.flags & 2) {  // a chunk that is not the last: keep the running factors
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int k = 0; k < MC; ++k) st[i * MC + k] = R[i][k];
        return;
    }
    double* o = a.out + (wg * G + g) * m;
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
