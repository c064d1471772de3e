// K_TSQR (m > 32), 128-row tiles, one CTA (16 warps) per SM.
//
// Same job structure and packed R workspace as tsqr_la_kernel, but each tile
// [R; B] has 128 rows, so the serial reflector chain of a panel is paid once
// per 128 rows instead of once per 32:
//   * warps 0..3 (one per SM sub-partition) factor the panel together: warp k
//     keeps tile rows 32k..32k+31 of the 32 panel columns in registers (lane =
//     column); per reflector the four partial dot products meet through
//     shared memory and one 128-thread named barrier; every panel warp then
//     derives the same reflector (LAPACK dlarfg normalisation and the
//     reference's zero rules, tsqr.hpp:120-160) and updates its rows;
//   * warps 4..7 first apply panel p's block reflector to panel p+1's columns
//     ("phase A", DMMA, result straight into the next panel buffer), then all
//     eight update warps apply it to the remaining columns while warps 0..3
//     factor panel p+1;
//   * the tile's trailing columns live in a per-CTA scratch in global memory
//     (L2 resident, 128 x M doubles); panel 0 and the first trailing update of
//     a tile read the input directly.
// T of the compact WY form is built from S = V^T V, which falls out of the
// panel's dot products, by the four panel warps (t2_build_t).
#pragma once

#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kT2Rows = 128;     // rows per tile of the 128-row variant
constexpr int kT2Threads = 512;  // ROWS / 32 panel warps + the rest update warps
constexpr int kT2Pld = 132;  // smem ld of a panel buffer (128 rows + 4)
// smem ld of a panel buffer of a ROWS-row tile
__host__ __device__ constexpr int t2_pld(int rows) { return rows + 4; }

struct T2Args {
    const double* X;
    int64_t n, ld;
    double* Rws;  // per-CTA packed R (blk_rsize(M))
    double* Scr;  // per-CTA tile scratch (kT2Rows x M, ld kT2Rows)
    int m, M;
    long long* prof;  // optional per-CTA phase cycle counters (8 per CTA), diagnostics
    ColSplit cs;      // column layout of X (q = 0: plain)
    // row chunks (the thick-bounds host entry folds X as it arrives): this
    // launch factors rows [n_lo, n_hi) (n_hi = 0: all rows), split over the
    // CTAs as usual; keep != 0: the per-CTA factors continue from the previous
    // launch instead of starting at zero
    int64_t n_lo, n_hi;
    int keep;
};

inline size_t t2_smem_bytes(int rows = kT2Rows) {
    const int pw = rows / 32;
    return ((size_t)2 * 32 * t2_pld(rows) + 32 * kLaRld + 32 * kTld + 2 * 32 * kLaTld + 32 + pw * 32 + 2 * pw * 32) *
           sizeof(double);
}

template <int PW, int ID = 2>
__device__ __forceinline__ void t2_bar_panel() {
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(PW * 32) : "memory");
}
// T build: four warps (the panel warps 0..3 of a stream)
template <int ID = 3>
__device__ __forceinline__ void t2_bar_t() { asm volatile("bar.sync %0, 128;" ::"n"(ID) : "memory"); }

// panel warps: factor the (32 PW) x 32 panel in P (ld 32 PW + 4) against the
// diagonal R block Rp; leaves V in P, the new block in Rp, tau, striu(S) in Sm.
// Register tile: lane (rq, cg) = rq + 8 cg of warp w keeps rows
// 32 w + rq + 8 r (r < 4) of columns 8 cg + c (c < 8).  Reflector j: the four
// lanes of column j's group broadcast its rows (4 shuffles), each lane forms
// its eight column dots over its four rows and a transpose-reduce over the 8
// row lanes leaves column `lane`'s warp partial in lane `lane` (7 shuffles);
// the PW partials meet in shared memory (one named barrier) and lane c derives
// column c's scalars as before (it "owns" column c); the f of its 8 register
// columns come back through a per-warp shared row.  (A column per lane with
// 32 rows needed the pivot lane to store its 32 values every reflector: ~400
// of ~1.7 k cycles per reflector.)
template <int PW, int BAR = 2>
__device__ __forceinline__ void t2_panel(double* P, double* Rp, double* tau, double* pvall, double* dpart, double* Sm,
                                         int warp, int lane) {
    constexpr int Pld = 32 * PW + 4;
    const int rq = lane & 7, cg = lane >> 3;
    double* fb = pvall + 32 * warp;  // per-warp f of the 32 columns
    double x[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[r][c] = P[(8 * cg + c) * Pld + 32 * warp + rq + 8 * r];
    const unsigned s_fb = (unsigned)__cvta_generic_to_shared(fb);
    const unsigned s_rcol = (unsigned)__cvta_generic_to_shared(Rp + lane * kLaRld);
    const unsigned s_scol = (unsigned)__cvta_generic_to_shared(Sm + lane * kTld);
    const unsigned s_dp = (unsigned)__cvta_generic_to_shared(dpart);
    const unsigned s_rp = (unsigned)__cvta_generic_to_shared(Rp);
    const unsigned s_tau = (unsigned)__cvta_generic_to_shared(tau);
    const bool w0 = (warp == 0);
    double my_scale = 1.0;  // scale of the reflector of column `lane`
    // warp 0 writes row j of the R block one reflector late (the other panel
    // warps may still be reading it)
    double pend_r = 0.0, pend_alpha = 0.0, pend_tau = 0.0;
    bool pend_upd = false;
    int pend_j = -1;
#pragma unroll 1
    for (int cgj = 0; cgj < 4; ++cgj) {
#pragma unroll
        for (int cj = 0; cj < 8; ++cj) {
            const int j = 8 * cgj + cj;
            const int par = j & 1;
            // pivot column j on my four rows
            double pr[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) pr[r] = __shfl_sync(0xffffffffu, x[r][cj], rq + 8 * cgj);
            double a[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                a[c] = pr[0] * x[0][c];
#pragma unroll
                for (int r = 1; r < 4; ++r) a[c] = fma(pr[r], x[r][c], a[c]);
            }
            // transpose-reduce over the row lanes (bits 2, 1, 0 of the lane):
            // lane ends with column 8 cg + rq = lane
#pragma unroll
            for (int o = 4; o >= 1; o >>= 1) {
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int t = 0; t < o; ++t) {
                    const double send = up ? a[t] : a[t + o];
                    const double keep = up ? a[t + o] : a[t];
                    a[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            sts1_if(true, s_dp + 8 * (par * 32 * PW + warp * 32 + lane), a[0]);
            t2_bar_panel<PW, BAR>();
            if (w0 && pend_j >= 0) {  // everyone is past reflector j-1: publish its R row
                sts1_if(pend_upd, s_rcol + 8 * pend_j, pend_r);
                sts1_if(lane == pend_j, s_rp + 8 * pend_j * (kLaRld + 1), pend_alpha);
                sts1_if(lane == pend_j, s_tau + 8 * pend_j, pend_tau);
            }
            double dv[PW], sv[PW];
#pragma unroll
            for (int w = 0; w < PW; ++w) {
                dv[w] = lds1(s_dp + 8 * (par * 32 * PW + 32 * w + lane));
                sv[w] = lds1(s_dp + 8 * (par * 32 * PW + 32 * w + j));
            }
            if constexpr ((PW & (PW - 1)) == 0) {
#pragma unroll
                for (int h = PW / 2; h >= 1; h >>= 1)
#pragma unroll
                    for (int w = 0; w < h; ++w) {
                        dv[w] = dv[w] + dv[w + h];
                        sv[w] = sv[w] + sv[w + h];
                    }
            } else {
#pragma unroll
                for (int w = 1; w < PW; ++w) {
                    dv[0] += dv[w];
                    sv[0] += sv[w];
                }
            }
            const double d = dv[0], sp = sv[0];
            const double u0 = lds1(s_rp + 8 * j * (kLaRld + 1));
            const double rjc = lds1(s_rcol + 8 * j);
            const double nrm2 = u0 * u0 + sp;
            const double inv = fast_rsqrt(nrm2);
            const double nr = nrm2 * inv;
            const double au = fabs(u0);
            const double sg = (u0 > 0.0) ? 1.0 : -1.0;
            double alpha = -sg * nr;
            double tj = 1.0 + au * inv;
            double scale = sg * fast_rcp(au + nr);
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
            const bool upd = lane > j;
            const double g = tj * (rjc + scale * d);
            const double f = upd ? g * scale : 0.0;
            my_scale = (lane == j) ? scale : my_scale;
            if (w0) {
                sts1_if(lane < j, s_scol + 8 * j, my_scale * scale * d);  // S(c, j) = v_c . v_j
                pend_r = rjc - g;
                pend_upd = upd;
                pend_alpha = alpha;
                pend_tau = tj;
                pend_j = j;
            }
            // f of column `lane` to the lanes holding it
            sts1_if(true, s_fb + 8 * lane, f);
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 8; c += 2) {
                const double2 t = lds2(s_fb + 8 * (8 * cg + c));
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    x[r][c] = fma(-t.x, pr[r], x[r][c]);
                    x[r][c + 1] = fma(-t.y, pr[r], x[r][c + 1]);
                }
            }
            __syncwarp();
        }
    }
    t2_bar_panel<PW, BAR>();
    if (w0) {
        sts1_if(pend_upd, s_rcol + 8 * pend_j, pend_r);
        sts1_if(lane == pend_j, s_rp + 8 * pend_j * (kLaRld + 1), pend_alpha);
        sts1_if(lane == pend_j, s_tau + 8 * pend_j, pend_tau);
    }
    // V = scale_c x (the scale of column c's reflector lives in lane c)
    sts1_if(true, s_fb + 8 * lane, my_scale);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const double sc = lds1(s_fb + 8 * (8 * cg + c));
#pragma unroll
        for (int r = 0; r < 4; ++r) P[(8 * cg + c) * Pld + 32 * warp + rq + 8 * r] = sc * x[r][c];
    }
    t2_bar_panel<PW, BAR>();
}

// panel warps 0..3: T = (diag(1/tau) + striu(S))^{-1} (row-major, ld kLaTld)
// by 8 x 8 diagonal blocks (warp k back-substitutes block k, lane j < 8 one
// column) and two levels of [[A, B], [0, C]]^{-1} = [[A^-1, -A^-1 B C^-1],
// [0, C^-1]]; X (16 x 16 scratch) holds the B C^-1 products.
template <int BAR = 3>
__device__ __forceinline__ void t2_build_t(const double* Sm, const double* tau, double* Tm, double* X, int warp,
                                           int lane) {
    {
        const int b0 = 8 * warp, j = lane & 7;
        double t[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) t[i] = (i == j) ? tau[b0 + j] : 0.0;
#pragma unroll
        for (int i = 6; i >= 0; --i) {
            double acc = 0.0;
#pragma unroll
            for (int l = i + 1; l < 8; ++l) acc = fma(Sm[(b0 + i) * kTld + b0 + l], t[l], acc);
            if (i < j) t[i] = -tau[b0 + i] * acc;
        }
        if (lane < 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i) Tm[(b0 + i) * kLaTld + b0 + j] = t[i];
            // the strictly lower blocks of this block row
            for (int c = 0; c < b0; ++c)
#pragma unroll
                for (int i = 0; i < 8; ++i) Tm[(b0 + i) * kLaTld + c] = 0.0;
        }
    }
    t2_bar_t<BAR>();
    // level 1: blocks (0,1) by warp 0, (2,3) by warp 1: T_ab = -T_aa (S_ab T_bb)
    if (warp < 2) {
        const int a0 = 16 * warp, b0 = a0 + 8;
        double* Xw = X + warp * 64;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = lane + 32 * h, i = e >> 3, j = e & 7;
            double acc = 0.0;
#pragma unroll
            for (int l = 0; l < 8; ++l) acc = fma(Sm[(a0 + i) * kTld + b0 + l], Tm[(b0 + l) * kLaTld + b0 + j], acc);
            Xw[i * 8 + j] = acc;
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = lane + 32 * h, i = e >> 3, j = e & 7;
            double acc = 0.0;
#pragma unroll
            for (int l = 0; l < 8; ++l) acc = fma(Tm[(a0 + i) * kLaTld + a0 + l], Xw[l * 8 + j], acc);
            Tm[(a0 + i) * kLaTld + b0 + j] = -acc;
        }
    }
    t2_bar_t<BAR>();
    // level 2: T[0:16, 16:32] = -T[0:16, 0:16] (S[0:16, 16:32] T[16:32, 16:32])
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int e = 64 * warp + lane + 32 * h, i = e >> 4, j = e & 15;
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < 16; ++l) acc = fma(Sm[i * kTld + 16 + l], Tm[(16 + l) * kLaTld + 16 + j], acc);
        X[i * 16 + j] = acc;
    }
    t2_bar_t<BAR>();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int e = 64 * warp + lane + 32 * h, i = e >> 4, j = e & 15;
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < 16; ++l) acc = fma(Tm[i * kLaTld + l], X[l * 16 + j], acc);
        Tm[i * kLaTld + 16 + j] = -acc;
    }
    t2_bar_t<BAR>();
}

// one warp: apply panel p's block reflector (V: 128 x 32 in smem, ld kT2Pld;
// T) to tile columns g..g+7 (source: input X or the scratch; destination:
// scratch or a panel buffer) and to R(p, g..g+7).
//   W^T = R(p, c)^T + B(:, c)^T V;  W'^T = W^T T;  R(p, c) -= W';  B(:, c) -= V W'.
template <bool SRC_X, bool DST_SMEM, int ROWS, bool SRC_SMEM = false>
__device__ __forceinline__ void t2_group(const double* src, int64_t lds, int rows, int mcols, double* dst, int64_t ldd,
                                         const double* V, const double* Tm, double* Rrow, int c0, int g, int gd,
                                         int lane, uint64_t pol_x, uint64_t pol_r, ColSplit cs = ColSplit{0, 0}) {
    const int r = lane >> 2, q = lane & 3;
    double* Rc = Rrow + (int64_t)(g + r - c0) * 32;
    double acc[4][2], rsav[4][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
        rsav[nt][0] = ld_hint(Rc + 8 * nt + 2 * q, pol_r);
        rsav[nt][1] = ld_hint(Rc + 8 * nt + 2 * q + 1, pol_r);
        acc[nt][0] = rsav[nt][0];
        acc[nt][1] = rsav[nt][1];
    }
    const double* scol = src + (SRC_X ? col_off(g + r, lds, cs) : (int64_t)(g + r) * lds);
#pragma unroll
    for (int kc = 0; kc < ROWS / 4; kc += 8) {
        double av[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int row = 4 * (kc + u) + q;
            if (SRC_X) av[u] = (row < rows && g + r < mcols) ? ld_hint(scol + row, pol_x) : 0.0;
            else if (SRC_SMEM) av[u] = scol[row];
            else av[u] = __ldcg(scol + row);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
                dmma884(acc[nt], av[u], V[(8 * nt + r) * t2_pld(ROWS) + 4 * (kc + u) + q]);
    }
    double w2[4][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) w2[nt][0] = w2[nt][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const int sl = r * 4 + 2 * (kk & 1) + (q >> 1);
        const double s0 = __shfl_sync(kFull, acc[kk >> 1][0], sl);
        const double s1 = __shfl_sync(kFull, acc[kk >> 1][1], sl);
        const double av = (q & 1) ? s1 : s0;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(w2[nt], av, Tm[(4 * kk + q) * kLaTld + 8 * nt + r]);
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
        st_hint(Rc + 8 * nt + 2 * q, rsav[nt][0] - w2[nt][0], pol_r);
        st_hint(Rc + 8 * nt + 2 * q + 1, rsav[nt][1] - w2[nt][1], pol_r);
    }
    double bv[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const int sl = r * 4 + 2 * (kk & 1) + (q >> 1);
        const double s0 = __shfl_sync(kFull, w2[kk >> 1][0], sl);
        const double s1 = __shfl_sync(kFull, w2[kk >> 1][1], sl);
        bv[kk] = (q & 1) ? s1 : s0;  // W'[4kk + q][r]
    }
    const double* s0c = src + (SRC_X ? col_off(g + 2 * q, lds, cs) : (int64_t)(g + 2 * q) * lds);
    const int64_t s1o = SRC_X ? col_off(g + 2 * q + 1, lds, cs) - col_off(g + 2 * q, lds, cs) : lds;  // to the odd column
#pragma unroll 2
    for (int mc = 0; mc < ROWS / 8; mc += 4) {
        double cb[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = 8 * (mc + u) + r;
                if (SRC_X)
                    cb[u][e] = (row < rows && g + 2 * q + e < mcols) ? ld_stream_hint(s0c + e * s1o + row, pol_x) : 0.0;
                else if (SRC_SMEM) cb[u][e] = s0c[e * lds + row];
                else cb[u][e] = __ldcg(s0c + e * lds + row);
            }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
#pragma unroll
            for (int u = 0; u < 4; ++u) dmma884(cb[u], -V[(4 * kk + q) * t2_pld(ROWS) + 8 * (mc + u) + r], bv[kk]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = 8 * (mc + u) + r;
                if (DST_SMEM) dst[(int64_t)(gd + 2 * q + e) * ldd + row] = cb[u][e];
                else __stcg(dst + (int64_t)(gd + 2 * q + e) * ldd + row, cb[u][e]);
            }
    }
}

template <int ROWS>
__global__ void __launch_bounds__(kT2Threads, 1) tsqr_t128_kernel(T2Args a) {
    constexpr int PW = ROWS / 32, Pld = t2_pld(ROWS), NUW = kT2Threads / 32 - PW;
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int M = a.M, m = a.m;
    double* Pb = sm;                           // 2 panel buffers, 32 columns x 128 rows (ld Pld)
    double* Rp = Pb + 2 * 32 * Pld;         // diagonal R block (ld kLaRld)
    double* Sm = Rp + 32 * kLaRld;             // striu(V^T V) (ld kTld)
    double* Tm0 = Sm + 32 * kTld;              // 2 x T (ld kLaTld)
    double* tau = Tm0 + 2 * 32 * kLaTld;       // 32
    double* pvall = tau + 32;                  // 4 x 32 pivot parts
    double* dpart = pvall + PW * 32;           // 2 x PW x 32 partial dots

    const int64_t job = blockIdx.x, G = gridDim.x;
    const int64_t n_end = a.n_hi > 0 ? a.n_hi : a.n, n_len = n_end - a.n_lo;
    const int64_t base = n_len / G, rem = n_len % G;
    const int64_t row0 = a.n_lo + job * base + (job < rem ? job : rem);
    const int64_t row1 = row0 + base + (job < rem ? 1 : 0);
    const int64_t RS = blk_rsize(M);
    double* R = a.Rws + job * RS;
    double* Scr = a.Scr + job * (int64_t)ROWS * M;
    const uint64_t pol_x = l2_policy_evict_first(), pol_r = l2_policy_evict_last();
    if (!a.keep)
        for (int64_t e = tid; e < RS; e += kT2Threads) st_hint(R + e, 0.0, pol_r);
    __syncthreads();
    const int npan = M / 32;
    const bool panel_warp = warp < PW;
#ifdef TTSVD_T2_PROF
    // diagnostics builds: per-CTA phase cycles of thread 0
    long long t_prev = 0, t_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define T2_PROF(ph)                                   \
    if (a.prof && tid == 0) {                         \
        const long long t_now = clock64();            \
        if (t_prev) t_acc[ph] += t_now - t_prev;      \
        t_prev = t_now;                               \
    }
#else
#define T2_PROF(ph)
#endif
    T2_PROF(7);
    const int uw = warp - PW;  // update warp index
    for (int64_t r0 = row0; r0 < row1; r0 += ROWS) {
        const int rows = (int)((row1 - r0) < ROWS ? (row1 - r0) : ROWS);
        const double* Xt = a.X + r0;  // column c at Xt + c * ld
        // panel 0 of the tile straight from the input
        if (warp == 0) la_fetch_rdiag(Rp, R, lane);
        // (and panel 1's raw columns into the second buffer, for phase A of
        // p = 0 from shared memory; all loads of both panels in flight at once)
        const int c_first = npan > 1 ? 64 : 32;
        // (cp.async: every thread's loads in flight at once — a load followed
        // by its shared-memory store serialised 32 HBM round trips per thread
        // and tile)
        for (int e = tid; e < c_first * ROWS; e += kT2Threads) {
            const int c = e / ROWS, i = e % ROWS;
            double* dst = &Pb[(c >> 5) * 32 * Pld + (c & 31) * Pld + i];
            if (i < rows && c < m) cp_async8_hint(dst, Xt + col_off(c, a.ld, a.cs) + i, pol_x);
            else *dst = 0.0;
        }
        cp_async_wait_all();
        __syncthreads();
        T2_PROF(0);
        if (panel_warp) {
            t2_panel<PW>(Pb, Rp, tau, pvall, dpart, Sm, warp, lane);
            if (warp == 0) la_store_rdiag(Rp, R, lane, pol_r);
            if (npan > 1 && warp < 4) t2_build_t(Sm, tau, Tm0, dpart, warp, lane);
        }
        __syncthreads();
        T2_PROF(0);
        for (int p = 0; p + 1 < npan; ++p) {
            const int c0 = 32 * p, nxt = c0 + 32;
            const double* V = Pb + (p & 1) * 32 * Pld;
            double* Pn = Pb + ((p + 1) & 1) * 32 * Pld;
            const double* Tp = Tm0 + (p & 1) * 32 * kLaTld;
            double* Rrow = R + blk_roff(p, M);
            if (warp == 0) la_fetch_rdiag(Rp, R + blk_roff(p + 1, M), lane);
            if (p > 0) {
                // panel p+1's columns from the scratch into the next panel
                // buffer (cp.async, all threads), so phase A runs from shared
                // memory instead of waiting on L2 round trips
                for (int e = tid; e < 32 * (ROWS / 2); e += kT2Threads) {
                    const int c = e / (ROWS / 2), i2 = 2 * (e % (ROWS / 2));
                    cp_async16(Pn + c * Pld + i2, Scr + (int64_t)(nxt + c) * ROWS + i2);
                }
                cp_async_wait_all();
                __syncthreads();
            }
            // phase A: panel p+1's columns, alone on the tensor pipes
            if (uw >= 0 && uw < 4) {
                if (p == 0)
                    t2_group<false, true, ROWS, true>(Pn - (int64_t)nxt * Pld, Pld, rows, m, Pn, Pld, V, Tp, Rrow, c0,
                                                      nxt + 8 * uw, 8 * uw, lane, pol_x, pol_r);
                else
                    t2_group<false, true, ROWS, true>(Pn - (int64_t)nxt * Pld, Pld, rows, m, Pn, Pld, V, Tp, Rrow, c0,
                                                      nxt + 8 * uw, 8 * uw, lane, pol_x, pol_r);
            }
            T2_PROF(5);
            if (warp == 0) cp_async_wait_all();
            T2_PROF(6);
            __syncthreads();
            T2_PROF(1);
            if (panel_warp) {
                t2_panel<PW>(Pn, Rp, tau, pvall, dpart, Sm, warp, lane);
                T2_PROF(2);
                if (warp == 0) la_store_rdiag(Rp, R + blk_roff(p + 1, M), lane, pol_r);
                if (p + 2 < npan && warp < 4) t2_build_t(Sm, tau, Tm0 + ((p + 1) & 1) * 32 * kLaTld, dpart, warp, lane);
                T2_PROF(3);
            } else {
                for (int g = nxt + 32 + 8 * uw; g < M; g += 8 * NUW) {
                    if (p == 0)
                        t2_group<true, false, ROWS>(Xt, a.ld, rows, m, Scr, ROWS, V, Tp, Rrow, c0, g, g, lane, pol_x, pol_r,
                                                    a.cs);
                    else
                        t2_group<false, false, ROWS>(Scr, ROWS, rows, m, Scr, ROWS, V, Tp, Rrow, c0, g, g, lane, pol_x,
                                               pol_r);
                }
            }
            __syncthreads();
            T2_PROF(4);
        }
    }
#ifdef TTSVD_T2_PROF
    if (a.prof && tid == 0)
        for (int q = 0; q < 8; ++q) a.prof[blockIdx.x * 8 + q] = t_acc[q];
#endif
#undef T2_PROF
}

}  // namespace ttsvd_b200
