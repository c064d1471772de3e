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
// R lives in the job's global workspace in a packed panel-major layout (row
// panel p = 32 rows x (M - 32p) columns, column-major, ld 32): only the upper
// triangle is stored, every DMMA fragment of R is a contiguous 2 KiB run, and
// 296 CTAs x M(M+32)/2 doubles stay L2 resident at M = 256.  The tile and V
// live in shared memory.  In merge mode the
// incoming part is upper triangular, so panels left of the tile's first row
// are structurally zero and skipped.
#pragma once

#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kBlkRows = 32;    // tile rows (one per lane in the panel)
constexpr int kBlkLdb = 36;     // smem ld of the tile: fragment loads in 2 wavefronts
constexpr int kBlkThreads = 256;  // 8 lanes per panel column in the panel
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
    int dbg = 0;            // diagnostics only (timing experiments): bit 0 skip trailing, bit 1 skip phase A
};

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// offset of row panel p in the packed layout, and the packed size
__host__ __device__ __forceinline__ int64_t blk_roff(int p, int M) {
    return 32 * ((int64_t)p * M - 32 * (int64_t)p * (p - 1) / 2);
}
__host__ __device__ __forceinline__ int64_t blk_rsize(int M) { return blk_roff(M / 32, M); }

inline size_t blk_smem_bytes(int M) {
    return ((size_t)M * kBlkLdb + 2 * 32 * kTld + 96 + (kBlkThreads / 32) * 32 * 9) * sizeof(double);
}

__global__ void __launch_bounds__(kBlkThreads, 2) tsqr_blk_kernel(BlkArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int M = a.M, m = a.m;
    double* Bt = sm;                          // M columns x 32 rows, ld kBlkLdb
    double* Sm = Bt + (size_t)M * kBlkLdb;    // 32 x 32 (S = V^T V, row-major, ld kTld)
    double* Rp = Sm;                          // 32 x 32 panel block of R: dead before S is formed
    double* Tm = Sm + 32 * kTld;              // 32 x 32 (T, row-major)
    double* tau = Tm + 32 * kTld;             // 32
    double* ucol = tau + 32;                  // 2 x 32: the pivot column being broadcast
    double* Wsc = ucol + 64;                  // per-warp 32 x 8 scratch (ld 9)

    const int64_t job = blockIdx.x;
    const double* X;
    int64_t row0, row1, ld;
    const double* R_init = nullptr;
    const int64_t RS = blk_rsize(M);
    double* R = a.Rws + job * RS;
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
        R_init = a.X + (2 * job) * RS;
        if (2 * job + 1 < count) {
            X = a.X + (2 * job + 1) * RS;
            row0 = 0;
            row1 = M;
        } else {
            X = nullptr;
            row0 = row1 = 0;
        }
        ld = M;
    }
    const uint64_t pol_x = l2_policy_evict_first(), pol_r = l2_policy_evict_last();
    for (int64_t e = tid; e < RS; e += kBlkThreads) st_hint(R + e, R_init ? R_init[e] : 0.0, pol_r);
    __syncthreads();

    long long t_prev = 0, t_acc[6] = {0, 0, 0, 0, 0, 0};
#define TT_PROF(ph)                                  \
    if (a.prof && tid == 0) {                        \
        const long long t_now = clock64();           \
        if (t_prev) t_acc[ph] += t_now - t_prev;     \
        t_prev = t_now;                              \
    }
    TT_PROF(5);
    const int npan = M / 32;
    for (int64_t r0 = row0; r0 < row1; r0 += kBlkRows) {
        const int rows = (int)((row1 - r0) < kBlkRows ? (row1 - r0) : kBlkRows);
        if (a.mode == 0) {
            for (int e = tid; e < M * kBlkRows; e += kBlkThreads) {
                const int c = e >> 5, i = e & 31;
                Bt[c * kBlkLdb + i] = (i < rows && c < m) ? ld_stream_hint(X + (int64_t)c * ld + r0 + i, pol_x) : 0.0;
            }
        } else {
            // row panel t of a packed triangular part: columns < 32t are zero
            const int t = (int)(r0 / 32);
            const double* src = X + blk_roff(t, M) - (int64_t)32 * 32 * t;
            for (int e = tid; e < M * kBlkRows; e += kBlkThreads) {
                const int c = e >> 5, i = e & 31;
                Bt[c * kBlkLdb + i] = (c >= 32 * t) ? src[e] : 0.0;
            }
        }
        __syncthreads();
        TT_PROF(0);
        const int p_first = a.mode == 1 ? (int)(r0 / 32) : 0;  // structural zeros of a triangular part
        for (int p = p_first; p < npan; ++p) {
            const int c0 = p * 32;
            // ---- 1. panel factorisation: warp 0, lane k owns panel column k ----
            // Column k's 32 tile rows sit in lane k's registers; the pivot
            // column is broadcast by shuffles, so every reflector needs no
            // cross-lane reduction: lanes compute the norm redundantly and
            // their own column's dot product locally.
            // ---- 1. panel factorisation: the whole CTA, 8 lanes per panel
            //         column (lane group g holds rows 4g..4g+3), one barrier
            //         per reflector (the pivot column is double buffered) ----
            {
                const int pc = tid >> 3;        // panel column owned by this lane group
                const int rg = (tid & 7) * 4;   // first of this lane's 4 tile rows
                double x[4];
                {
                    const double2 t0 = *reinterpret_cast<const double2*>(Bt + (c0 + pc) * kBlkLdb + rg);
                    const double2 t1 = *reinterpret_cast<const double2*>(Bt + (c0 + pc) * kBlkLdb + rg + 2);
                    x[0] = t0.x; x[1] = t0.y; x[2] = t1.x; x[3] = t1.y;
                }
                {
                    const double* Rpan = R + blk_roff(p, M);  // row panel p: column c0 + k at k*32
                    for (int e = tid; e < 32 * 32; e += kBlkThreads)
                        Rp[(e & 31) * kTld + (e >> 5)] = ld_hint(Rpan + e, pol_r);
                }
                for (int jj = 0; jj < 32; ++jj) {
                    double* ub = ucol + (jj & 1) * 32;
                    if (pc == jj) {
                        *reinterpret_cast<double2*>(ub + rg) = make_double2(x[0], x[1]);
                        *reinterpret_cast<double2*>(ub + rg + 2) = make_double2(x[2], x[3]);
                    }
                    __syncthreads();
                    const double2 u01 = *reinterpret_cast<const double2*>(ub + rg);
                    const double2 u23 = *reinterpret_cast<const double2*>(ub + rg + 2);
                    double sp = u01.x * u01.x + u01.y * u01.y + (u23.x * u23.x + u23.y * u23.y);
                    double dp = u01.x * x[0] + u01.y * x[1] + (u23.x * x[2] + u23.y * x[3]);
#pragma unroll
                    for (int o = 1; o < 8; o <<= 1) {
                        sp += __shfl_xor_sync(0xffffffffu, sp, o);
                        dp += __shfl_xor_sync(0xffffffffu, dp, o);
                    }
                    const double u0 = Rp[jj * kTld + jj];
                    const double nrm2 = u0 * u0 + sp;
                    // alpha = -sign(u0) ||u||, tau = 1 + |u0|/||u||, scale = 1/(u0 - alpha)
                    const double inv = rsqrt(nrm2);
                    const double nr = nrm2 * inv;
                    const double au = fabs(u0);
                    const double sg = (u0 > 0.0) ? 1.0 : -1.0;
                    double alpha = -sg * nr;
                    double tj = 1.0 + au * inv;
                    double scale = sg * __drcp_rn(au + nr);
                    if (sp == 0.0 && u0 != 0.0) {  // H = I
                        alpha = u0;
                        tj = 0.0;
                        scale = 0.0;
                    }
                    if (nrm2 == 0.0) {  // all-zero u: the reference's eps_fp result
                        alpha = sqrt(2.0 * DBL_MIN);
                        tj = 2.0;
                        scale = 0.0;
                    }
                    if (pc > jj) {
                        const double rjk = Rp[jj * kTld + pc];
                        const double g = tj * (rjk + scale * dp);
                        const double f = g * scale;
                        x[0] = fma(-f, u01.x, x[0]);
                        x[1] = fma(-f, u01.y, x[1]);
                        x[2] = fma(-f, u23.x, x[2]);
                        x[3] = fma(-f, u23.y, x[3]);
                        if (rg == 0) Rp[jj * kTld + pc] = rjk - g;
                    } else if (pc == jj) {
                        x[0] = scale * u01.x;  // v_j
                        x[1] = scale * u01.y;
                        x[2] = scale * u23.x;
                        x[3] = scale * u23.y;
                        if (rg == 0) {
                            Rp[jj * kTld + jj] = alpha;
                            tau[jj] = tj;
                        }
                    }
                }
                *reinterpret_cast<double2*>(Bt + (c0 + pc) * kBlkLdb + rg) = make_double2(x[0], x[1]);
                *reinterpret_cast<double2*>(Bt + (c0 + pc) * kBlkLdb + rg + 2) = make_double2(x[2], x[3]);
                __syncthreads();
                {
                    double* Rpan = R + blk_roff(p, M);
                    for (int e = tid; e < 32 * 32; e += kBlkThreads) st_hint(Rpan + e, Rp[(e & 31) * kTld + (e >> 5)], pol_r);
                }
            }
            __syncthreads();
            TT_PROF(1);
            if (c0 + 32 >= M) continue;  // no trailing columns: T is not needed
            // ---- 2. S = V^T V (DMMA, warp w -> reflector columns 8w..8w+7 of 32),
            //         then T = (diag(1/tau) + striu(S))^{-1} blockwise ----
            const int lr = lane >> 2, lc = lane & 3;
            for (int nt = warp; nt < 4; nt += kBlkThreads / 32) {
                double sacc[4][2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) sacc[mt][0] = sacc[mt][1] = 0.0;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const double b = Bt[(c0 + 8 * nt + lr) * kBlkLdb + 4 * kk + lc];
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) dmma884(sacc[mt], Bt[(c0 + 8 * mt + lr) * kBlkLdb + 4 * kk + lc], b);
                }
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) Sm[(8 * mt + lr) * kTld + 8 * nt + 2 * lc + e] = sacc[mt][e];
            }
            __syncthreads();
            TT_PROF(2);
            // T = U^{-1}, U = diag(1/tau) + striu(S), by 8x8 diagonal blocks
            // (lane 8b+j back-substitutes column j of block b) and two levels
            // of the block identity [[A, B], [0, C]]^{-1} = [[A^-1, -A^-1 B C^-1], [0, C^-1]].
            if (warp == 0) {
                const int b0 = 8 * (lane >> 3), j = lane & 7;
                for (int i = 0; i < 32; ++i) Tm[i * kTld + b0 + j] = 0.0;
                Tm[(b0 + j) * kTld + b0 + j] = tau[b0 + j];
                for (int i = j - 1; i >= 0; --i) {
                    double acc = 0.0;
                    for (int l = i + 1; l <= j; ++l) acc += Sm[(b0 + i) * kTld + b0 + l] * Tm[(b0 + l) * kTld + b0 + j];
                    Tm[(b0 + i) * kTld + b0 + j] = -tau[b0 + i] * acc;
                }
            }
            __syncthreads();
            TT_PROF(3);
            for (int lev = 8; lev <= 16; lev *= 2) {
                // blocks [o, o+lev) x [o+lev, o+2lev), o = 0 (and 16 when lev = 8)
                double* Xs = Wsc;  // scratch (>= 16 x 16 used as lev x lev, ld 17)
                const int nblk = 32 / (2 * lev);
                for (int e = tid; e < nblk * lev * lev; e += kBlkThreads) {
                    const int q = e / (lev * lev), i = (e / lev) % lev, j = e % lev;
                    const int o = q * 2 * lev;
                    double acc = 0.0;  // X = S[o.., o+lev..] T[o+lev.., o+lev..]
                    for (int l = 0; l <= j; ++l) acc += Sm[(o + i) * kTld + o + lev + l] * Tm[(o + lev + l) * kTld + o + lev + j];
                    Xs[q * 17 * 17 + i * 17 + j] = acc;
                }
                __syncthreads();
                for (int e = tid; e < nblk * lev * lev; e += kBlkThreads) {
                    const int q = e / (lev * lev), i = (e / lev) % lev, j = e % lev;
                    const int o = q * 2 * lev;
                    double acc = 0.0;  // T[o+i, o+lev+j] = -(T_A X)(i, j)
                    for (int l = i; l < lev; ++l) acc += Tm[(o + i) * kTld + o + l] * Xs[q * 17 * 17 + l * 17 + j];
                    Tm[(o + i) * kTld + o + lev + j] = -acc;
                }
                __syncthreads();
                TT_PROF(3);
            }
            // ---- 3. trailing update over 8-column groups (DMMA m8n8k4) ----
            double* Ws = Wsc + warp * 32 * 9;
            double* Rrow = R + blk_roff(p, M);
            for (int g = c0 + 32 + 8 * warp; g < M; g += 8 * (kBlkThreads / 32)) {
                double acc[4][2], rsav[4][2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        rsav[mt][e] = ld_hint(Rrow + (g + 2 * lc + e - c0) * 32 + 8 * mt + lr, pol_r);
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
                        st_hint(Rrow + (g + 2 * lc + e - c0) * 32 + 8 * mt + lr, rsav[mt][e] - w2[mt][e], pol_r);
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
            TT_PROF(4);
        }
    }
    if (a.prof && tid == 0)
        for (int q = 0; q < 6; ++q) a.prof[blockIdx.x * 8 + q] = t_acc[q];
#undef TT_PROF
}

// ---------------------------------------------------------------------------
// K_TSQR, tall tiles (mode 0, m > 32): the same blocked compact-WY reduction
// with 128-row tiles.  Only the current 32-column panel is staged in shared
// memory; the tile's trailing columns live in a per-CTA scratch in global
// memory (L2 resident: 128 x M doubles per CTA, one CTA per SM), so the
// 32-step reflector chain of a panel — the latency-bound part — is amortised
// over 4x more rows than in tsqr_blk_kernel.  Panel 0 reads the input
// directly (evict-first) and its trailing update writes the scratch.
// ---------------------------------------------------------------------------
constexpr int kTallRows = 128;
constexpr int kTallThreads = 256;
constexpr int kPld = 132;  // smem ld of the panel

struct TallArgs {
    const double* X;
    int64_t n, ld;
    double* Rws;      // per-CTA packed R (blk_rsize(M))
    double* Scr;      // per-CTA tile scratch (kTallRows x M, ld kTallRows)
    int m, M;
    long long* prof;
};

inline size_t tall_smem_bytes() {
    return ((size_t)32 * kPld + 2 * 32 * kTld + 32 + 2 * kTallRows + (kTallThreads / 32) * 32 * 9) * sizeof(double);
}

__global__ void __launch_bounds__(kTallThreads, 1) tsqr_tall_kernel(TallArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int M = a.M, m = a.m;
    double* Pn = sm;                     // 32 panel columns x 128 rows (ld kPld); V after the panel
    double* Sm = Pn + 32 * kPld;         // S = V^T V (row-major, ld kTld); also the panel block Rp
    double* Rp = Sm;
    double* Tm = Sm + 32 * kTld;
    double* tau = Tm + 32 * kTld;
    double* ucol = tau + 32;             // 2 x 128
    double* Wsc = ucol + 2 * kTallRows;  // per-warp 32 x 8 (ld 9)

    const int64_t job = blockIdx.x, G = gridDim.x;
    const int64_t base = a.n / G, rem = a.n % G;
    const int64_t row0 = job * base + (job < rem ? job : rem);
    const int64_t row1 = row0 + base + (job < rem ? 1 : 0);
    const int64_t RS = blk_rsize(M);
    double* R = a.Rws + job * RS;
    double* Scr = a.Scr + job * (int64_t)kTallRows * M;
    const double* X = a.X;
    const int64_t ld = a.ld;
    const uint64_t pol_x = l2_policy_evict_first(), pol_r = l2_policy_evict_last();
    for (int64_t e = tid; e < RS; e += kTallThreads) st_hint(R + e, 0.0, pol_r);
    __syncthreads();

    long long t_prev = 0, t_acc[6] = {0, 0, 0, 0, 0, 0};
#define TT_PROF(ph)                                  \
    if (a.prof && tid == 0) {                        \
        const long long t_now = clock64();           \
        if (t_prev) t_acc[ph] += t_now - t_prev;     \
        t_prev = t_now;                              \
    }
    TT_PROF(5);
    const int npan = M / 32;
    const int lr = lane >> 2, lc = lane & 3;
    for (int64_t r0 = row0; r0 < row1; r0 += kTallRows) {
        const int rows = (int)((row1 - r0) < kTallRows ? (row1 - r0) : kTallRows);
        for (int p = 0; p < npan; ++p) {
            const int c0 = p * 32;
            // ---- stage panel p (input for p = 0, scratch otherwise) and R's panel block ----
            for (int e = tid; e < 32 * kTallRows; e += kTallThreads) {
                const int c = e >> 7, i = e & (kTallRows - 1);
                double v;
                if (p == 0) v = (i < rows && c0 + c < m) ? ld_stream_hint(X + (int64_t)(c0 + c) * ld + r0 + i, pol_x) : 0.0;
                else v = ld_hint(Scr + (int64_t)(c0 + c) * kTallRows + i, pol_r);
                Pn[c * kPld + i] = v;
            }
            {
                const double* Rpan = R + blk_roff(p, M);
                for (int e = tid; e < 32 * 32; e += kTallThreads) Rp[(e & 31) * kTld + (e >> 5)] = ld_hint(Rpan + e, pol_r);
            }
            __syncthreads();
            TT_PROF(0);
            // ---- panel factorisation: 8 lanes per column, 16 rows per lane ----
            {
                const int pc = tid >> 3;
                const int rg = (tid & 7) * 16;
                double x[16];
#pragma unroll
                for (int r = 0; r < 16; r += 2) {
                    const double2 t = *reinterpret_cast<const double2*>(Pn + pc * kPld + rg + r);
                    x[r] = t.x;
                    x[r + 1] = t.y;
                }
                for (int jj = 0; jj < 32; ++jj) {
                    double* ub = ucol + (jj & 1) * kTallRows;
                    if (pc == jj) {
#pragma unroll
                        for (int r = 0; r < 16; r += 2)
                            *reinterpret_cast<double2*>(ub + rg + r) = make_double2(x[r], x[r + 1]);
                    }
                    __syncthreads();
                    double u[16];
                    double s0 = 0.0, s1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
                    for (int r = 0; r < 16; r += 2) {
                        const double2 t = *reinterpret_cast<const double2*>(ub + rg + r);
                        u[r] = t.x;
                        u[r + 1] = t.y;
                        s0 = fma(t.x, t.x, s0);
                        s1 = fma(t.y, t.y, s1);
                        d0 = fma(t.x, x[r], d0);
                        d1 = fma(t.y, x[r + 1], d1);
                    }
                    double sp = s0 + s1, dp = d0 + d1;
#pragma unroll
                    for (int o = 1; o < 8; o <<= 1) {
                        sp += __shfl_xor_sync(0xffffffffu, sp, o);
                        dp += __shfl_xor_sync(0xffffffffu, dp, o);
                    }
                    const double u0 = Rp[jj * kTld + jj];
                    const double nrm2 = u0 * u0 + sp;
                    const double inv = rsqrt(nrm2);
                    const double nr = nrm2 * inv;
                    const double au = fabs(u0);
                    const double sg = (u0 > 0.0) ? 1.0 : -1.0;
                    double alpha = -sg * nr;
                    double tj = 1.0 + au * inv;
                    double scale = sg * __drcp_rn(au + nr);
                    if (sp == 0.0 && u0 != 0.0) {
                        alpha = u0;
                        tj = 0.0;
                        scale = 0.0;
                    }
                    if (nrm2 == 0.0) {
                        alpha = sqrt(2.0 * DBL_MIN);
                        tj = 2.0;
                        scale = 0.0;
                    }
                    if (pc > jj) {
                        const double rjk = Rp[jj * kTld + pc];
                        const double g = tj * (rjk + scale * dp);
                        const double f = g * scale;
#pragma unroll
                        for (int r = 0; r < 16; ++r) x[r] = fma(-f, u[r], x[r]);
                        if (rg == 0) Rp[jj * kTld + pc] = rjk - g;
                    } else if (pc == jj) {
#pragma unroll
                        for (int r = 0; r < 16; ++r) x[r] = scale * u[r];
                        if (rg == 0) {
                            Rp[jj * kTld + jj] = alpha;
                            tau[jj] = tj;
                        }
                    }
                }
#pragma unroll
                for (int r = 0; r < 16; r += 2)
                    *reinterpret_cast<double2*>(Pn + pc * kPld + rg + r) = make_double2(x[r], x[r + 1]);
                __syncthreads();
                double* Rpan = R + blk_roff(p, M);
                for (int e = tid; e < 32 * 32; e += kTallThreads) st_hint(Rpan + e, Rp[(e & 31) * kTld + (e >> 5)], pol_r);
            }
            __syncthreads();
            TT_PROF(1);
            if (c0 + 32 >= M) continue;
            // ---- S = V^T V (DMMA, K = 128 rows), T = (diag(1/tau) + striu(S))^{-1} ----
            if (warp < 4) {
                const int nt = warp;
                double sacc[4][2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) sacc[mt][0] = sacc[mt][1] = 0.0;
#pragma unroll 8
                for (int kk = 0; kk < kTallRows / 4; ++kk) {
                    const double b = Pn[(8 * nt + lr) * kPld + 4 * kk + lc];
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) dmma884(sacc[mt], Pn[(8 * mt + lr) * kPld + 4 * kk + lc], b);
                }
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) Sm[(8 * mt + lr) * kTld + 8 * nt + 2 * lc + e] = sacc[mt][e];
            }
            __syncthreads();
            TT_PROF(2);
            if (warp == 0) {
                const int b0 = 8 * (lane >> 3), j = lane & 7;
                for (int i = 0; i < 32; ++i) Tm[i * kTld + b0 + j] = 0.0;
                Tm[(b0 + j) * kTld + b0 + j] = tau[b0 + j];
                for (int i = j - 1; i >= 0; --i) {
                    double acc = 0.0;
                    for (int l = i + 1; l <= j; ++l) acc += Sm[(b0 + i) * kTld + b0 + l] * Tm[(b0 + l) * kTld + b0 + j];
                    Tm[(b0 + i) * kTld + b0 + j] = -tau[b0 + i] * acc;
                }
            }
            __syncthreads();
            for (int lev = 8; lev <= 16; lev *= 2) {
                double* Xs = Wsc;
                const int nblk = 32 / (2 * lev);
                for (int e = tid; e < nblk * lev * lev; e += kTallThreads) {
                    const int q = e / (lev * lev), i = (e / lev) % lev, j = e % lev;
                    const int o = q * 2 * lev;
                    double acc = 0.0;
                    for (int l = 0; l <= j; ++l) acc += Sm[(o + i) * kTld + o + lev + l] * Tm[(o + lev + l) * kTld + o + lev + j];
                    Xs[q * 17 * 17 + i * 17 + j] = acc;
                }
                __syncthreads();
                for (int e = tid; e < nblk * lev * lev; e += kTallThreads) {
                    const int q = e / (lev * lev), i = (e / lev) % lev, j = e % lev;
                    const int o = q * 2 * lev;
                    double acc = 0.0;
                    for (int l = i; l < lev; ++l) acc += Tm[(o + i) * kTld + o + l] * Xs[q * 17 * 17 + l * 17 + j];
                    Tm[(o + i) * kTld + o + lev + j] = -acc;
                }
                __syncthreads();
            }
            TT_PROF(3);
            // ---- trailing update of the 8-column groups right of the panel ----
            double* Ws = Wsc + warp * 32 * 9;
            double* Rrow = R + blk_roff(p, M);
            for (int g = c0 + 32 + 8 * warp; g < M; g += 8 * (kTallThreads / 32)) {
                // B(:, g..g+7): fragment view b[kk] = B(row 4kk + lc, col g + lr)
                double bf[kTallRows / 4];
                if (p == 0) {
                    const bool colok = g + lr < m;
#pragma unroll
                    for (int kk = 0; kk < kTallRows / 4; ++kk) {
                        const int row = 4 * kk + lc;
                        bf[kk] = (colok && row < rows) ? ld_stream_hint(X + (int64_t)(g + lr) * ld + r0 + row, pol_x) : 0.0;
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < kTallRows / 4; ++kk)
                        bf[kk] = ld_hint(Scr + (int64_t)(g + lr) * kTallRows + 4 * kk + lc, pol_r);
                }
                double acc[4][2], rsav[4][2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        rsav[mt][e] = ld_hint(Rrow + (g + 2 * lc + e - c0) * 32 + 8 * mt + lr, pol_r);
                        acc[mt][e] = rsav[mt][e];
                    }
#pragma unroll
                for (int kk = 0; kk < kTallRows / 4; ++kk)
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) dmma884(acc[mt], Pn[(8 * mt + lr) * kPld + 4 * kk + lc], bf[kk]);
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) Ws[(8 * mt + lr) * 9 + 2 * lc + e] = acc[mt][e];
                __syncwarp();
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
                        st_hint(Rrow + (g + 2 * lc + e - c0) * 32 + 8 * mt + lr, rsav[mt][e] - w2[mt][e], pol_r);
                        Ws[(8 * mt + lr) * 9 + 2 * lc + e] = w2[mt][e];
                    }
                __syncwarp();
                // B(:, g..g+7) -= V W'  (C layout: rows 8mt + lr, cols g + 2lc + e)
                double wf[8];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) wf[kk] = Ws[(4 * kk + lc) * 9 + lr];
                double cb[kTallRows / 8][2];
#pragma unroll
                for (int mt = 0; mt < kTallRows / 8; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = g + 2 * lc + e, row = 8 * mt + lr;
                        if (p == 0)
                            cb[mt][e] = (col < m && row < rows) ? ld_stream_hint(X + (int64_t)col * ld + r0 + row, pol_x) : 0.0;
                        else
                            cb[mt][e] = ld_hint(Scr + (int64_t)col * kTallRows + row, pol_r);
                    }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
#pragma unroll
                    for (int mt = 0; mt < kTallRows / 8; ++mt) dmma884(cb[mt], -Pn[(4 * kk + lc) * kPld + 8 * mt + lr], wf[kk]);
#pragma unroll
                for (int mt = 0; mt < kTallRows / 8; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        st_hint(Scr + (int64_t)(g + 2 * lc + e) * kTallRows + 8 * mt + lr, cb[mt][e], pol_r);
                __syncwarp();
            }
            __syncthreads();
            TT_PROF(4);
        }
    }
    if (a.prof && tid == 0)
        for (int q = 0; q < 6; ++q) a.prof[blockIdx.x * 8 + q] = t_acc[q];
#undef TT_PROF
}

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
