// K_TSMM on the FP64 tensor cores with the rows of X staged by the bulk-copy
// engine (TMA).
//
// Same product and output placement as tsmm_dmma_kernel (each warp computes
// a 32-row x 32-column block of X V with DMMA m8n8k4 and scatters it into the
// next step's padded layout, tsmm.hpp:20-77), but the A fragments come from
// shared memory: a warp's 32 rows of 16 columns of X are one stage (16 bulk
// copies of 256 bytes, cp.async.bulk / UBLKCP, issued by lanes 0..15 and
// counted in bytes on the warp's own mbarrier), four stages (two for m > 256) in flight
// per warp, so ~100 KB per SM are always on their way from HBM and the
// threads spend their issue slots on the fragment loads and the DMMAs.  (With
// fragments loaded straight from X a thread holds at most two k-steps of
// loads, and the kernel sat at 43 % of the FP64 peak while needing 70 % of the
// HBM bandwidth at that peak.)  The stage's column stride is 36 doubles: the
// 32 lanes of a fragment load touch every bank pair exactly twice.
// Requires n % 32 == 0, m % 16 == 0, X and ldx 16-byte aligned (else the
// caller keeps tsmm_dmma_kernel).
#pragma once

#include <cstdint>

#include "tsqr_gt.cuh"

namespace ttsvd_b200 {

constexpr int kDtMt = 8;                 // 8-row tiles per warp block
constexpr int kDtRows = 8 * kDtMt;       // rows per warp block
constexpr int kDtCols = 8;               // columns of X per stage
constexpr int kDtCs = kDtRows + 4;       // column stride of a stage (doubles)

// NT: 8-column tiles of the output chunk a CTA computes (4: k > 16; 2: k <= 16)
inline size_t dt_smem_bytes(int m, int stages, int nt = 4) {
    return ((size_t)m * (8 * nt + 4) + (size_t)8 * stages * kDtCols * kDtCs) * sizeof(double);
}

template <int kDtStages, int NT = 4>
__global__ void __launch_bounds__(256, 1) tsmm_dt_kernel(const double* __restrict__ X, int64_t n, int m, int64_t ldx,
                                                         const double* __restrict__ V, int64_t ldv, int k,
                                                         double* __restrict__ Y, int64_t out_rows, int64_t ldy,
                                                         ColSplit cs) {
    extern __shared__ __align__(128) double dsm[];
    __shared__ __align__(8) unsigned long long mbar[8][kDtStages];
    constexpr int kDtVld = 8 * NT + 4;  // smem ld of the V chunk
    constexpr int KCH = 8 * NT;         // output columns per chunk
    double* Vs = dsm;                   // m x kDtVld
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* xb = dsm + (size_t)m * kDtVld + (size_t)warp * kDtStages * kDtCols * kDtCs;
    const int c0 = blockIdx.y * KCH;
    const int kc = min(KCH, k - c0);
    for (int e = tid; e < m * kDtVld; e += 256) {
        const int j = e / kDtVld, c = e % kDtVld;
        Vs[e] = (c < kc) ? V[(int64_t)(c0 + c) * ldv + j] : 0.0;
    }
    auto bar = [&](int s) { return (unsigned)__cvta_generic_to_shared(&mbar[warp][s]); };
    if (lane == 0)
        for (int s = 0; s < kDtStages; ++s) gt_mbar_init(bar(s), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int r = lane >> 2, q = lane & 3;
    const bool divisible = (n % out_rows) == 0;
    const int64_t n_next = divisible ? n / out_rows : 0;
    const int64_t W = (int64_t)gridDim.x * 8, wg = (int64_t)blockIdx.x * 8 + warp;
    const int64_t blocks = n / kDtRows;
    const int spb = m / kDtCols;  // stages per row block
    // the warp's stream of stages: (row block wg + W t, column group cgp), cgp fastest
    const int64_t my_blocks = wg < blocks ? (blocks - wg + W - 1) / W : 0;
    const int64_t total = my_blocks * spb;
    auto issue = [&](int64_t idx, int s) {
        const int64_t rb = (wg + (idx / spb) * W) * kDtRows;
        const int cg = (int)(idx % spb) * kDtCols;
        if (lane == 0) gt_mbar_expect(bar(s), (unsigned)(kDtCols * kDtRows * 8));
        __syncwarp();
        if (lane < kDtCols)
            gt_bulk_g2s((unsigned)__cvta_generic_to_shared(xb + ((size_t)s * kDtCols + lane) * kDtCs),
                        X + col_off(cg + lane, ldx, cs) + rb, (unsigned)(kDtRows * 8), bar(s));
    };
    for (int s = 0; s < kDtStages; ++s)
        if (s < total) issue(s, s);
    int s = 0;
    unsigned phase = 0;
    int64_t idx = 0;
    for (int64_t t = 0; t < my_blocks; ++t) {
        const int64_t rb = (wg + t * W) * kDtRows;
        double acc[kDtMt][NT][2];
#pragma unroll
        for (int mt = 0; mt < kDtMt; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
        for (int g = 0; g < spb; ++g, ++idx) {
            gt_mbar_wait(bar(s), phase);
            const double* xs = xb + (size_t)s * kDtCols * kDtCs + r;
            const double* vs = Vs + (size_t)(g * kDtCols) * kDtVld + r;
#pragma unroll
            for (int kk = 0; kk < kDtCols / 4; ++kk) {
                const int col = 4 * kk + q;
                double a[kDtMt], b[NT];
#pragma unroll
                for (int mt = 0; mt < kDtMt; ++mt) a[mt] = xs[col * kDtCs + 8 * mt];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) b[nt] = vs[col * kDtVld + 8 * nt];
#pragma unroll
                for (int mt = 0; mt < kDtMt; ++mt)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt], a[mt], b[nt]);
            }
            __syncwarp();  // the stage has been read: refill it
            if (idx + kDtStages < total) issue(idx + kDtStages, s);
            if (++s == kDtStages) {
                s = 0;
                phase ^= 1;
            }
        }
        if (divisible && out_rows >= kDtRows) {
            // one division per row block: the block's rows cross at most one
            // out_rows boundary
            const int64_t b0 = rb / out_rows, i0 = rb - b0 * out_rows;
#pragma unroll
            for (int mt = 0; mt < kDtMt; ++mt) {
                int64_t ii = i0 + 8 * mt + r, b = b0;
                if (ii >= out_rows) {
                    ii -= out_rows;
                    ++b;
                }
                double* yb = Y + (b + n_next * c0) * ldy + ii;
                const int64_t cstep = n_next * ldy;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int c = 8 * nt + 2 * q + e;
                        if (c < kc) yb[c * cstep] = acc[mt][nt][e];
                    }
            }
        } else {
#pragma unroll
            for (int mt = 0; mt < kDtMt; ++mt) {
                const int64_t i = rb + 8 * mt + r;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int c = 8 * nt + 2 * q + e;
                        if (c >= kc) continue;
                        const int64_t p = i + n * (c0 + c);
                        const int64_t cl = p / out_rows;
                        Y[cl * ldy + (p - cl * out_rows)] = acc[mt][nt][e];
                    }
            }
        }
    }
}

}  // namespace ttsvd_b200
