// K_TSQR for short-fat work matrices: communication-avoiding QR (CAQR, R
// only) on one cooperative grid.  Replaces gqr.cuh's one grid barrier per
// reflector (config 2 steps 3-4: ~11.5 k cycles per reflector, of which ~5 k
// are the barrier and the fixed-order sums) by a TSQR per 32-column panel:
//
//   CTA c owns the contiguous rows [r0_c, r1_c) (<= 512).
//   Panel p (32 columns [32p, 32p + 32)):
//     stage 0  every CTA factors ITS rows of the panel in shared memory (32
//              reflectors, one CTA barrier each, no grid barrier): local
//              Y_c, T_c, R_c, and applies (I - Y_c T_c Y_c^T)^T to its rows of
//              the trailing columns;
//     stage 1  the CTAs form groups of 16: every member stacks the group's
//              R_c (16 x 32 = 512 rows) and factors the stack (redundantly —
//              identical bits on every member), then member s applies it to
//              the members' 32 "top" rows (the rows that carry R_c) for the
//              trailing column groups g = s (mod members);
//     stage 2  every CTA stacks the group factors R_g (<= 16 x 32 rows),
//              factors them and applies that to the group leaders' top rows,
//              column groups split over all CTAs.
//   The panel's rows of R are R_p (the last stage's triangle) and the final
//   top rows of slot 0 (right of the diagonal block); slot 0 retires those
//   32 rows.  Slot 0 rotates with p, so every CTA retires at most once
//   (G >= panels).  Three grid barriers per panel instead of 32+; every
//   reduction has a fixed order, so the result is bitwise deterministic.
//   Reflectors: LAPACK normalisation computed through the reference's
//   DBL_MIN-shifted quantities (tsqr.hpp:120-142, see caqr_qr); a zero column
//   under a nonzero pivot is H = I.  X is only read (panel 0 reads it; the
//   trailing updates write the work copy A): no copy pass.
//
// The panel QR keeps the block in shared memory, two columns per warp: per
// reflector the owner warp forms v (one warp reduction), one CTA barrier,
// then every warp updates its own columns (one warp reduction each) — no
// second barrier, since the next pivot column belongs to a single warp.
// The trailing updates run in teams of RB warps (32 rows each, RB covering
// the block), one 8-column group per team at a time: partial W = Y^T C per
// warp (DMMA), the team's partials summed in a fixed order and W' = T^T W
// formed by the team's first warp, C -= Y W' (DMMA).
#pragma once

#include <cooperative_groups.h>
#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kCaqrThreads = 512;
constexpr int kCaqrWarps = kCaqrThreads / 32;
constexpr int kCaqrLdy = 516;  // smem ld of the block (rows <= 512): conflict-free DMMA fragment loads
constexpr int kCaqrGroup = 16;

struct CaqrArgs {
    const double* X;  // input n x m (ld ldx), read by panel 0 only
    int64_t ldx;
    double* A;        // work copy n x M (ld lda): trailing columns after every panel
    int64_t lda;
    int64_t n;
    int m, M;
    double* S1;       // G x 1024: local factors R_c (32 x 32, column-major)
    double* S2;       // 16 x 1024: group factors R_g
    double* R;        // output m x m (ld ldr), zeroed by the caller
    int64_t ldr;
};

inline size_t caqr_smem_bytes() {
    // block, S, T, tau, per-warp partial W (8 x 32), per-team W' (32 x 9), row bases
    return ((size_t)32 * kCaqrLdy + 2 * 32 * 33 + 32 + kCaqrWarps * 256 + kCaqrWarps * 288 + 16) * sizeof(double);
}

__device__ __forceinline__ int64_t caqr_r0(int q, int64_t n, int G) {
    const int64_t base = n / G, rem = n % G;
    return q * base + (q < rem ? q : rem);
}

__device__ __forceinline__ void caqr_team_bar(int team, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(nthreads) : "memory");
}

// column ck <- H_j ck (v = column j of the block, unit pivot)
__device__ __forceinline__ void caqr_update1(const double* v, double tj, double* ck, int j, int rows, int lane) {
    double d = 0.0, e = 0.0;
    int i = j + 1 + lane;
#pragma unroll 4
    for (; i + 32 < rows; i += 64) {
        d = fma(v[i], ck[i], d);
        e = fma(v[i + 32], ck[i + 32], e);
    }
    if (i < rows) d = fma(v[i], ck[i], d);
    d = warp_sum(d + e);
    const double g = tj * (ck[j] + d);
#pragma unroll 4
    for (int r = j + 1 + lane; r < rows; r += 32) ck[r] = fma(-g, v[r], ck[r]);
    __syncwarp();
    if (lane == 0) ck[j] -= g;
    __syncwarp();
}

// both columns c1, c2 <- H_j (one pass, two interleaved butterflies)
__device__ __forceinline__ void caqr_update2(const double* v, double tj, double* c1, double* c2, int j, int rows,
                                             int lane) {
    double d1 = 0.0, d2 = 0.0, e1 = 0.0, e2 = 0.0;
    int i = j + 1 + lane;
#pragma unroll 4
    for (; i + 32 < rows; i += 64) {
        const double v0 = v[i], v1 = v[i + 32];
        d1 = fma(v0, c1[i], d1);
        d2 = fma(v0, c2[i], d2);
        e1 = fma(v1, c1[i + 32], e1);
        e2 = fma(v1, c2[i + 32], e2);
    }
    if (i < rows) {
        const double v0 = v[i];
        d1 = fma(v0, c1[i], d1);
        d2 = fma(v0, c2[i], d2);
    }
    d1 += e1;
    d2 += e2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        d1 += __shfl_xor_sync(0xffffffffu, d1, o);
        d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    }
    const double g1 = tj * (c1[j] + d1), g2 = tj * (c2[j] + d2);
#pragma unroll 4
    for (int r = j + 1 + lane; r < rows; r += 32) {
        const double vr = v[r];
        c1[r] = fma(-g1, vr, c1[r]);
        c2[r] = fma(-g2, vr, c2[r]);
    }
    __syncwarp();
    if (lane == 0) {
        c1[j] -= g1;
        c2[j] -= g2;
    }
    __syncwarp();
}

// The critical path of caqr_qr between two barriers: the owner of column
// j + 1 applies H_j to it and forms reflector j + 1 from the result, with the
// column held in registers (16 rows per lane, one smem read and one write).
__device__ __forceinline__ void caqr_owner_step(const double* v, double tj, double* cn, int j, int rows, int lane,
                                                double* tau) {
    double x[16], y[16];
    double d = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int r = lane + 32 * q;
        const bool in = r >= j && r < rows;
        y[q] = in ? cn[r] : 0.0;
        x[q] = (r > j && r < rows) ? v[r] : (r == j ? 1.0 : 0.0);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) d = fma(x[q], y[q], d);
    d = warp_sum(d);
    const double g = tj * d;  // H_j = I - tau v v^T, v = [1; v_below]
    double sp = 0.0, u0l = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int r = lane + 32 * q;
        y[q] = fma(-g, x[q], y[q]);
        if (r > j + 1 && r < rows) sp = fma(y[q], y[q], sp);
        if (r == j + 1) u0l = y[q];
    }
    sp = warp_sum(sp);
    const double u0 = __shfl_sync(0xffffffffu, u0l, (j + 1) & 31);
    // LAPACK normalisation (v = [1; x / (u0 - alpha)]) through the reference's
    // DBL_MIN-shifted quantities: t = DBL_MIN + ||u||^2, alpha = -sign(u0)
    // sqrt(t + DBL_MIN), tau = (u0 - alpha)^2 / (t - alpha u0).  Equal to the
    // plain formulas for normal columns; when a rank-deficient block's residue
    // decays into the subnormal range (each further reflector is built from
    // ~eps times the previous residue), the shift keeps tau ||v||^2 = 2 to
    // rounding.  An all-zero u gives alpha = sqrt(2 DBL_MIN), tau = 2, v = e_1
    // (tsqr.hpp:120).
    const double nrm2 = u0 * u0 + sp;
    const double sg = (u0 > 0.0) ? 1.0 : -1.0;
    const double t1 = DBL_MIN + nrm2;
    const double a2 = t1 + DBL_MIN;
    double alpha = -sg * (a2 * fast_rsqrt(a2));
    const double dd = u0 - alpha;
    double tn = dd * dd * fast_rcp(t1 - alpha * u0), scale = fast_rcp(dd);
    if (sp == 0.0 && u0 != 0.0) {  // nothing below the pivot: H = I
        alpha = u0;
        tn = 0.0;
        scale = 0.0;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int r = lane + 32 * q;
        if (r >= j && r < rows) cn[r] = r == j + 1 ? alpha : (r > j + 1 ? y[q] * scale : y[q]);
    }
    if (lane == 0) tau[j + 1] = tn;
    __syncwarp();
}

// The first reflector (column 0, no update before it).
__device__ __forceinline__ void caqr_first(double* c0, int rows, int lane, double* tau) {
    caqr_owner_step(c0, 0.0, c0, -1, rows, lane, tau);
}

// QR of the rows x 32 block in shared memory (column k at B + k * kCaqrLdy,
// 32 <= rows <= 512).  Afterwards the upper triangle holds R, the entries
// below the diagonal the reflectors v (unit diagonal implied), tau[32] the
// scalars.  Warp w owns columns w and w + 16.  One CTA barrier per
// reflector; the owner of the next pivot column updates it and forms the next
// reflector at once (caqr_owner_step), and applies H_j to its other column
// after the next barrier (a deferred update, in order).
__device__ __forceinline__ void caqr_qr(double* B, int rows, double* tau) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k1 = warp, k2 = warp + kCaqrWarps;
    double* c1 = B + k1 * kCaqrLdy;
    double* c2 = B + k2 * kCaqrLdy;
    if (warp == 0) caqr_first(B, rows, lane, tau);
    int pend = -1;  // a reflector still owed to column k2
    for (int j = 0; j < 32; ++j) {
        __syncthreads();
        if (pend >= 0) {
            caqr_update1(B + pend * kCaqrLdy, tau[pend], c2, pend, rows, lane);
            pend = -1;
        }
        const double* v = B + j * kCaqrLdy;
        const double tj = tau[j];
        if (j + 1 < 32 && warp == ((j + 1) & (kCaqrWarps - 1))) {
            caqr_owner_step(v, tj, B + (j + 1) * kCaqrLdy, j, rows, lane, tau);
            if (k1 == j + 1) pend = j;  // k2 = j + 17 still needs H_j
        } else if (k1 > j) {
            caqr_update2(v, tj, c1, c2, j, rows, lane);
        } else if (k2 > j) {
            caqr_update1(v, tj, c2, j, rows, lane);
        }
    }
    __syncthreads();
}

// The block after caqr_qr becomes Y (unit lower trapezoid, zero rows up to
// rows8); S = Y^T Y (DMMA, 4 warps); T from T^{-1} = diag(1/tau) + striu(S)
// by back substitution, one lane per column.  The caller has copied R out.
__device__ __forceinline__ void caqr_form_t(double* B, int rows, double* Sm, double* Tm, const double* tau) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lr = lane >> 2, lc = lane & 3;
    const int rows8 = (rows + 7) & ~7;
    for (int e = tid; e < 32 * 32; e += kCaqrThreads) {
        const int k = e >> 5, i = e & 31;
        if (i <= k) B[k * kCaqrLdy + i] = i == k ? 1.0 : 0.0;
    }
    for (int e = rows + tid; e < rows8; e += kCaqrThreads)
#pragma unroll
        for (int k = 0; k < 32; ++k) B[k * kCaqrLdy + e] = 0.0;
    __syncthreads();
    if (warp < 4) {
        const int nt = warp;
        double sacc[4][2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) sacc[mt][0] = sacc[mt][1] = 0.0;
        for (int kk = 0; kk < rows8 / 4; ++kk) {
            const double b = B[(8 * nt + lr) * kCaqrLdy + 4 * kk + lc];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) dmma884(sacc[mt], B[(8 * mt + lr) * kCaqrLdy + 4 * kk + lc], b);
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int e = 0; e < 2; ++e) Sm[(8 * mt + lr) * 33 + 8 * nt + 2 * lc + e] = sacc[mt][e];
    }
    __syncthreads();
    if (warp == 0) {
        // (D^{-1} + striu(S)) T = I: T(i, j) = tau_i (delta_ij - sum_{l>i} S(i, l) T(l, j))
        const int j = lane;
        double t[32];
#pragma unroll
        for (int i = 31; i >= 0; --i) {
            double s = 0.0;
#pragma unroll
            for (int l = i + 1; l < 32; ++l) s = fma(Sm[i * 33 + l], t[l], s);
            t[i] = (i > j) ? 0.0 : (i == j ? tau[j] : -tau[i] * s);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) Tm[i * 33 + j] = t[i];
    }
    __syncthreads();
}

// C <- (I - Y T Y^T)^T C on `rows` rows: row k of C is row rowbase[k >> 5] +
// (k & 31) of the column-major src (ld lds; columns >= src_cols read as zero),
// written to dst (ld ldd).  Column groups (8 columns at cb + 8 gi) gi =
// g0, g0 + gs, ... < ngr.
__device__ __forceinline__ void caqr_apply(const double* src, int64_t lds, int64_t src_cols, double* dst,
                                           int64_t ldd, const int64_t* rowbase, int rows, int64_t cb, int ngr,
                                           int g0, int gs, const double* B, const double* Tm, double* Wp,
                                           double* Wt) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lr = lane >> 2, lc = lane & 3;
    const int RB = rows <= 64 ? 2 : rows <= 128 ? 4 : rows <= 256 ? 8 : 16;
    const int NTm = kCaqrWarps / RB;  // <= 8 teams: named barriers 1..8
    const int team = warp / RB, r = warp % RB, row0 = 32 * r;
    double* wp = Wp + warp * 256;
    double* wt = Wt + team * 288;
    (void)tid;
    for (int gi = g0 + team * gs; gi < ngr; gi += NTm * gs) {
        const int64_t g = cb + 8 * gi;
        // my 32 rows of the group: B fragments (W = Y^T C) and C fragments
        // (the update), all 16 loads in flight
        double cbf[8], ccf[4][2];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const int row = row0 + 4 * kk + lc;
            cbf[kk] = (row < rows && g + lr < src_cols) ? __ldcg(src + (g + lr) * lds + rowbase[row >> 5] + (row & 31))
                                                        : 0.0;
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = row0 + 8 * mt + lr;
                const int64_t col = g + 2 * lc + e;
                ccf[mt][e] = (row < rows && col < src_cols)
                                 ? __ldcg(src + col * lds + rowbase[row >> 5] + (row & 31))
                                 : 0.0;
            }
        double acc[4][2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
                dmma884(acc[mt], B[(8 * mt + lr) * kCaqrLdy + row0 + 4 * kk + lc], cbf[kk]);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int e = 0; e < 2; ++e) wp[(8 * mt + lr) * 8 + 2 * lc + e] = acc[mt][e];
        caqr_team_bar(team, RB * 32);
        if (r == 0) {
            // W = the team's partials in a fixed order (B-fragment layout), W' = T^T W
            double w[8];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                double s = 0.0;
                for (int q = 0; q < RB; ++q) s += Wp[(team * RB + q) * 256 + (4 * kk + lc) * 8 + lr];
                w[kk] = s;
            }
            double accp[4][2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) accp[mt][0] = accp[mt][1] = 0.0;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) dmma884(accp[mt], Tm[(4 * kk + lc) * 33 + 8 * mt + lr], w[kk]);
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int e = 0; e < 2; ++e) wt[(8 * mt + lr) * 9 + 2 * lc + e] = accp[mt][e];
        }
        caqr_team_bar(team, RB * 32);
        double wf[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) wf[kk] = wt[(4 * kk + lc) * 9 + lr];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
                dmma884(ccf[mt], -B[(4 * kk + lc) * kCaqrLdy + row0 + 8 * mt + lr], wf[kk]);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = row0 + 8 * mt + lr;
                if (row < rows) dst[(g + 2 * lc + e) * ldd + rowbase[row >> 5] + (row & 31)] = ccf[mt][e];
            }
    }
    __syncthreads();
}

#ifdef CAQR_PROF  // diagnostics builds only (tools/caqr_debug.cu)
__device__ long long* g_caqr_prof;
#define CAQR_MARK(k_)                                                                   \
    if (tid == 0 && c == (p % G) && g_caqr_prof) {                                     \
        long long t_;                                                                  \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
        g_caqr_prof[p * 24 + (k_)] = t_;                                               \
    }
#else
#define CAQR_MARK(k_)
#endif

__global__ void __launch_bounds__(kCaqrThreads, 1) caqr_kernel(CaqrArgs ca) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) double sm[];
    double* Bs = sm;                          // 32 x kCaqrLdy: the stage's block
    double* Sm = Bs + 32 * kCaqrLdy;          // 32 x 33
    double* Tm = Sm + 32 * 33;                // 32 x 33
    double* tau = Tm + 32 * 33;               // 32
    double* Wp = tau + 32;                    // warps x 256
    double* Wt = Wp + kCaqrWarps * 256;       // teams x 288
    int64_t* rowbase = reinterpret_cast<int64_t*>(Wt + kCaqrWarps * 288);  // 16
    const int tid = threadIdx.x;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t n = ca.n;
    const int m = ca.m, M = ca.M, npan = M / 32;
    const int Gg = (G + kCaqrGroup - 1) / kCaqrGroup;
    const int64_t r1 = caqr_r0(c + 1, n, G);
    for (int p = 0; p < npan; ++p) {
        const int64_t c0 = 32 * (int64_t)p, t0 = c0 + 32;
        const int ngr = (int)((M - t0) / 8);
        const int o = p % G;  // slot 0 of this panel (retires its top rows)
        const int slot = (c - o + G) % G;
        const int grp = slot / kCaqrGroup, mem = slot % kCaqrGroup;
        const int nmem = min(kCaqrGroup, G - kCaqrGroup * grp);
        // first active row of CTA q: CTA q retired 32 rows at panel q (G >= panels)
        auto a0_of = [&](int q) { return caqr_r0(q, n, G) + (q < p ? 32 : 0); };
        const double* src = p == 0 ? ca.X : ca.A;
        const int64_t lds = p == 0 ? ca.ldx : ca.lda;
        const int64_t srcc = p == 0 ? m : M;
        for (int stage = 0; stage < 3; ++stage) {
            if (stage == 2 && Gg == 1) break;
            const bool final_stage = (stage == 2) || (stage == 1 && Gg == 1);
            const int rows = stage == 0 ? (int)(r1 - a0_of(c)) : (stage == 1 ? 32 * nmem : 32 * Gg);
            // this stage's rows of the work matrix, in 32-row blocks
            if (tid < 16) {
                int64_t b = 0;
                if (stage == 0) b = a0_of(c) + 32 * tid;
                else if (stage == 1) b = a0_of((o + kCaqrGroup * grp + tid) % G);
                else b = a0_of((o + kCaqrGroup * tid) % G);
                rowbase[tid] = b;
            }
            CAQR_MARK(stage * 6 + 0);
            // the block: my rows of the panel, or the stacked triangles
            if (stage == 0) {
                const int64_t a0 = a0_of(c);
                for (int e = tid; e < 32 * rows; e += kCaqrThreads) {
                    const int k = e / rows, i = e - k * rows;
                    Bs[k * kCaqrLdy + i] = (c0 + k < srcc) ? __ldcg(src + (c0 + k) * lds + a0 + i) : 0.0;
                }
            } else {
                for (int e = tid; e < 32 * rows; e += kCaqrThreads) {
                    const int k = e / rows, i = e - k * rows;
                    const int s = i >> 5;
                    const double* S = stage == 1 ? ca.S1 + (int64_t)((o + kCaqrGroup * grp + s) % G) * 1024
                                                 : ca.S2 + (int64_t)s * 1024;
                    Bs[k * kCaqrLdy + i] = __ldcg(S + k * 32 + (i & 31));
                }
            }
            __syncthreads();
            CAQR_MARK(stage * 6 + 1);
            caqr_qr(Bs, rows, tau);
            CAQR_MARK(stage * 6 + 2);
            // the stage's triangle: to the next stage, or the panel's rows of R
            {
                const bool writer =
                    stage == 0 || (stage == 1 && mem == 0 && !final_stage) || (final_stage && slot == 0);
                if (writer)
                    for (int e = tid; e < 1024; e += kCaqrThreads) {
                        const int k = e >> 5, i = e & 31;
                        const double v = i <= k ? Bs[k * kCaqrLdy + i] : 0.0;
                        if (!final_stage) {
                            double* dstS = stage == 0 ? ca.S1 + (int64_t)c * 1024 : ca.S2 + (int64_t)grp * 1024;
                            dstS[e] = v;
                        } else if (i <= k && c0 + k < m && c0 + i < m) {
                            ca.R[(c0 + k) * ca.ldr + c0 + i] = v;
                        }
                    }
            }
            __syncthreads();
            caqr_form_t(Bs, rows, Sm, Tm, tau);
            CAQR_MARK(stage * 6 + 3);
            // trailing update: my rows (stage 0, all column groups) or the
            // stacked top rows (stages 1, 2: the column groups split over the
            // CTAs that share the stage)
            const int g0 = stage == 0 ? 0 : (stage == 1 ? mem : slot);
            const int gs = stage == 0 ? 1 : (stage == 1 ? nmem : G);
            if (ngr > 0) {
                if (stage == 0)
                    caqr_apply(src, lds, srcc, ca.A, ca.lda, rowbase, rows, t0, ngr, g0, gs, Bs, Tm, Wp, Wt);
                else
                    caqr_apply(ca.A, ca.lda, M, ca.A, ca.lda, rowbase, rows, t0, ngr, g0, gs, Bs, Tm, Wp, Wt);
            }
            CAQR_MARK(stage * 6 + 4);
            if (final_stage) {
                // slot 0's top rows are the panel's rows of R right of its
                // diagonal block: the column groups this CTA just updated
                const int64_t top = rowbase[0];
                for (int gi = g0; gi < ngr; gi += gs)
                    for (int e = tid; e < 256; e += kCaqrThreads) {
                        const int i = e & 31;
                        const int64_t col = t0 + 8 * gi + (e >> 5);
                        if (col < m && c0 + i < m) ca.R[col * ca.ldr + c0 + i] = __ldcg(ca.A + col * ca.lda + top + i);
                    }
            }
            __threadfence();
            cg::this_grid().sync();
            CAQR_MARK(stage * 6 + 5);
        }
    }
}

}  // namespace ttsvd_b200
