// K_TSQR (m > 32): blocked structured Householder with compact-WY trailing
// updates on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).
//
// Same job structure as tsqr_tile_kernel (per-CTA flat tree over a row range,
// tsqr.hpp:247-292, or one level of the index-ordered merge tree,
// tsqr.hpp:230-240), but each 32-row tile [R; B] is reduced panel by panel:
//
//   1. panel factorisation (warp 0, one panel column per lane): 32 structured
//      reflectors y_j = [e_j; v_j], H_j = I - tau_j y_j y_j^T (LAPACK dlarfg
//      normalisation), alpha_j = -sign(R_jj) ||[R_jj; B(:,j)]||; a zero
//      column under a nonzero pivot is H = I; an all-zero u gives the
//      reference's eps_fp result alpha = sqrt(2 DBL_MIN) (tsqr.hpp:120-126);
//   2. T of the compact WY form H_1..H_32 = I - Y T Y^T from the UT identity
//      T^{-1} = diag(1/tau) + striu(Y^T Y), Y^T Y = I + V^T V;
//   3. trailing update of every 8-column group c (all warps, DMMA):
//        W = R(p, c) + V^T B(:, c);  W = T^T W;  R(p, c) -= W;  B(:, c) -= V W.
//
// R (M x M, ld M, M = m rounded up to 32) lives in the job's global workspace
// (L2 resident); the tile and V live in shared memory.  In merge mode the
// incoming part is upper triangular, so panels left of the tile's first row
// are structurally zero and skipped.
#pragma once

#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kBlkRows = 32;    // tile rows (one per lane in the panel)
constexpr int kBlkLdb = 36;     // smem ld of the tile: fragment loads in 2 wavefronts
constexpr int kBlkThreads = 128;
constexpr int kTld = 33;        // smem ld of S and T

struct BlkArgs {
    const double* X;        // mode 0: matrix (n x m, ld); mode 1: parts (count x M x M)
    int64_t n;              // mode 0: rows; mode 1: number of parts at this level
    int64_t ld;
    double* Rws;            // per-job running R / output (M x M, ld M)
    const double* R_init0;  // mode 0 only: starting R (M x M, ld M) or nullptr
    int m;                  // logical columns
    int M;                  // padded columns (multiple of 32)
    int mode;
};

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

inline size_t blk_smem_bytes(int M) {
    return ((size_t)M * kBlkLdb + 3 * 32 * kTld + 64 + (kBlkThreads / 32) * 32 * 9) * sizeof(double);
}

__global__ void __launch_bounds__(kBlkThreads, 2) tsqr_blk_kernel(BlkArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int M = a.M, m = a.m;
    double* Bt = sm;                          // M columns x 32 rows, ld kBlkLdb
    double* Sm = Bt + (size_t)M * kBlkLdb;    // 32 x 32 (S = V^T V, row-major, ld kTld)
    double* Tm = Sm + 32 * kTld;              // 32 x 32 (T, row-major)
    double* Rp = Tm + 32 * kTld;              // 32 x 32 panel block of R (row-major)
    double* tau = Rp + 32 * kTld;             // 32
    double* ucol = tau + 32;                  // 32: the pivot column being broadcast
    double* Wsc = ucol + 32;                  // per-warp 32 x 8 scratch (ld 9)

    const int64_t job = blockIdx.x;
    const double* X;
    int64_t row0, row1, ld;
    const double* R_init = nullptr;
    double* R = a.Rws + job * (int64_t)M * M;
    if (a.mode == 0) {
        const int64_t G = gridDim.x;
        const int64_t base = a.n / G, rem = a.n % G;
        row0 = job * base + (job < rem ? job : rem);
        row1 = row0 + base + (job < rem ? 1 : 0);
        X = a.X;
        ld = a.ld;
        R_init = a.R_init0;
    } else {
        const int64_t count = a.n;
        R_init = a.X + (2 * job) * (int64_t)M * M;
        if (2 * job + 1 < count) {
            X = a.X + (2 * job + 1) * (int64_t)M * M;
            row0 = 0;
            row1 = M;
        } else {
            X = nullptr;
            row0 = row1 = 0;
        }
        ld = M;
    }
    for (int64_t e = tid; e < (int64_t)M * M; e += kBlkThreads) R[e] = R_init ? R_init[e] : 0.0;
    __syncthreads();

    const int npan = M / 32;
    for (int64_t r0 = row0; r0 < row1; r0 += kBlkRows) {
        const int rows = (int)((row1 - r0) < kBlkRows ? (row1 - r0) : kBlkRows);
        for (int e = tid; e < M * kBlkRows; e += kBlkThreads) {
            const int c = e >> 5, i = e & 31;
            Bt[c * kBlkLdb + i] = (i < rows && c < m) ? X[(int64_t)c * ld + r0 + i] : 0.0;
        }
        __syncthreads();
        const int p_first = a.mode == 1 ? (int)(r0 / 32) : 0;  // structural zeros of a triangular part
        for (int p = p_first; p < npan; ++p) {
            const int c0 = p * 32;
            // ---- 1. panel factorisation: warp 0, lane k owns panel column k ----
            // Column k's 32 tile rows sit in lane k's registers; the pivot
            // column is broadcast by shuffles, so every reflector needs no
            // cross-lane reduction: lanes compute the norm redundantly and
            // their own column's dot product locally.
            if (warp == 0) {
                double x[32];
#pragma unroll
                for (int r = 0; r < 32; ++r) x[r] = Bt[(c0 + lane) * kBlkLdb + r];
                for (int i = 0; i < 32; ++i) Rp[i * kTld + lane] = R[(int64_t)(c0 + lane) * M + c0 + i];
                __syncwarp();
                for (int jj = 0; jj < 32; ++jj) {
                    // pivot column -> shared memory, read back as broadcasts
                    if (lane == jj) {
#pragma unroll
                        for (int r = 0; r < 32; r += 2)
                            *reinterpret_cast<double2*>(ucol + r) = make_double2(x[r], x[r + 1]);
                    }
                    __syncwarp();
                    double s0 = 0.0, s1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
                    for (int r = 0; r < 32; r += 2) {
                        const double2 uu = *reinterpret_cast<const double2*>(ucol + r);
                        s0 += uu.x * uu.x;
                        s1 += uu.y * uu.y;
                        d0 += uu.x * x[r];
                        d1 += uu.y * x[r + 1];
                    }
                    const double s = s0 + s1;
                    const double u0 = Rp[jj * kTld + jj];
                    double alpha, tj, scale;
                    if (s == 0.0 && u0 != 0.0) {
                        alpha = u0;
                        tj = 0.0;
                        scale = 0.0;
                    } else {
                        const double nrm2 = u0 * u0 + s;
                        if (nrm2 == 0.0) {
                            alpha = sqrt(2.0 * DBL_MIN);
                            tj = 2.0;
                            scale = 0.0;
                        } else {
                            const double nr = sqrt(nrm2);
                            alpha = (u0 > 0.0) ? -nr : nr;
                            tj = (alpha - u0) / alpha;
                            scale = 1.0 / (u0 - alpha);
                        }
                    }
                    const double rjk = Rp[jj * kTld + lane];
                    const double g = tj * (rjk + scale * (d0 + d1));
                    const double gs = g * scale;
                    if (lane > jj) {
#pragma unroll
                        for (int r = 0; r < 32; r += 2) {
                            const double2 uu = *reinterpret_cast<const double2*>(ucol + r);
                            x[r] -= gs * uu.x;
                            x[r + 1] -= gs * uu.y;
                        }
                        Rp[jj * kTld + lane] = rjk - g;
                    } else if (lane == jj) {
#pragma unroll
                        for (int r = 0; r < 32; ++r) x[r] *= scale;  // v_j
                        Rp[jj * kTld + jj] = alpha;
                        tau[jj] = tj;
                    }
                    __syncwarp();
                }
#pragma unroll
                for (int r = 0; r < 32; ++r) Bt[(c0 + lane) * kBlkLdb + r] = x[r];
                for (int i = 0; i < 32; ++i) R[(int64_t)(c0 + lane) * M + c0 + i] = Rp[i * kTld + lane];
            }
            __syncthreads();
            if (c0 + 32 >= M) continue;  // no trailing columns: T is not needed
            // ---- 2. S = strict upper part of V^T V, then T = (diag(1/tau) + S)^{-1} ----
            for (int e = tid; e < 32 * 32; e += kBlkThreads) {
                const int i = e >> 5, j = e & 31;
                if (i < j) {
                    const double* vi = Bt + (c0 + i) * kBlkLdb;
                    const double* vj = Bt + (c0 + j) * kBlkLdb;
                    double s = 0.0;
#pragma unroll 8
                    for (int r = 0; r < 32; ++r) s += vi[r] * vj[r];
                    Sm[i * kTld + j] = s;
                }
            }
            __syncthreads();
            if (warp == 0) {
                const int j = lane;  // lane j back-substitutes column j of T
                for (int i = 31; i > j; --i) Tm[i * kTld + j] = 0.0;
                Tm[j * kTld + j] = tau[j];
                for (int i = j - 1; i >= 0; --i) {
                    double acc = 0.0;
                    for (int l = i + 1; l <= j; ++l) acc += Sm[i * kTld + l] * Tm[l * kTld + j];
                    Tm[i * kTld + j] = -tau[i] * acc;
                }
            }
            __syncthreads();
            // ---- 3. trailing update over 8-column groups (DMMA m8n8k4) ----
            double* Ws = Wsc + warp * 32 * 9;
            const int lr = lane >> 2, lc = lane & 3;
            for (int g = c0 + 32 + 8 * warp; g < M; g += 8 * (kBlkThreads / 32)) {
                double acc[4][2], rsav[4][2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        rsav[mt][e] = R[(int64_t)(g + 2 * lc + e) * M + c0 + 8 * mt + lr];
                        acc[mt][e] = rsav[mt][e];
                    }
                // W = R(p, c) + V^T B(:, c):  A = V^T (refl x row), B = tile (row x col)
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const double b = Bt[(g + lr) * kBlkLdb + 4 * kk + lc];
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) dmma884(acc[mt], Bt[(c0 + 8 * mt + lr) * kBlkLdb + 4 * kk + lc], b);
                }
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) Ws[(8 * mt + lr) * 9 + 2 * lc + e] = acc[mt][e];
                __syncwarp();
                // W' = T^T W:  A = T^T (i x k) = T(k, i), B = W (k x col)
                double w2[4][2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) w2[mt][0] = w2[mt][1] = 0.0;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const double b = Ws[(4 * kk + lc) * 9 + lr];
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) dmma884(w2[mt], Tm[(4 * kk + lc) * kTld + 8 * mt + lr], b);
                }
                __syncwarp();
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        R[(int64_t)(g + 2 * lc + e) * M + c0 + 8 * mt + lr] = rsav[mt][e] - w2[mt][e];
                        Ws[(8 * mt + lr) * 9 + 2 * lc + e] = w2[mt][e];
                    }
                __syncwarp();
                // B(:, c) -= V W':  A = -V (row x refl), B = W' (refl x col), C = tile
                double cb[4][2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) cb[mt][e] = Bt[(g + 2 * lc + e) * kBlkLdb + 8 * mt + lr];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const double b = Ws[(4 * kk + lc) * 9 + lr];
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) dmma884(cb[mt], -Bt[(c0 + 4 * kk + lc) * kBlkLdb + 8 * mt + lr], b);
                }
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) Bt[(g + 2 * lc + e) * kBlkLdb + 8 * mt + lr] = cb[mt][e];
                __syncwarp();
            }
            __syncthreads();
        }
    }
}

// leading m x m block of an M x M workspace factor -> R (ld m)
__global__ void copy_leading_kernel(const double* Rws, int M, int m, double* R) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += gridDim.x * blockDim.x) {
        const int j = e / m, i = e - j * m;
        R[e] = Rws[(int64_t)j * M + i];
    }
}

}  // namespace ttsvd_b200
