// K_TSQR (m > 32), look-ahead variant of tsqr_blk_kernel: same jobs, same
// packed panel-major R workspace (blk_roff), same reflector definitions and
// zero rules, but the serial panel chain no longer stalls the CTA.
//
// Per 32-row tile [R; B] and row panel p:
//   * warp 0 factors panel p+1 — lane c owns panel column c (32 doubles in
//     registers), the pivot column is broadcast through shared memory, so a
//     reflector costs no CTA barrier and S = V^T V falls out of the same dot
//     products; then T (lane j back-substitutes column j of
//     (diag(1/tau) + striu(S))^{-1});
//   * meanwhile warps 1..7 apply panel p's compact-WY block reflector to the
//     trailing columns beyond panel p+1 (DMMA; W^T, W^T T and V W' are
//     chained through register shuffles, no shared scratch);
//   * panel p+1's own 32 columns are updated first (warps 0..3, "phase A"),
//     the only part of the trailing update on the critical path.
// The diagonal block of R's row panel p+1 is fetched with cp.async while
// phase A runs.  T is double buffered by panel parity.
#pragma once

#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kLaThreads = 256;
constexpr int kLaRld = 34;  // column-major ld of the panel's diagonal R block (16-byte aligned columns)
constexpr int kLaTld = 36;  // row-major ld of T (conflict-free B fragments)
constexpr unsigned kFull = 0xffffffffu;

inline size_t la_smem_bytes(int M) {
    return ((size_t)M * kBlkLdb + 32 * kLaRld + 32 * kTld + 2 * 32 * kLaTld + 64) * sizeof(double);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
// 8-byte asynchronous copy with an L2 eviction policy (streamed input rows)
__device__ __forceinline__ void cp_async8_hint(void* smem_dst, const void* gsrc, uint64_t pol) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(s), "l"(gsrc), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// warp: the 32 x 32 diagonal block of a row panel (packed layout: column k at
// k * 32) -> Rp (column-major, ld kLaRld), asynchronously
__device__ __forceinline__ void la_fetch_rdiag(double* Rp, const double* Rpan, int lane) {
#pragma unroll 4
    for (int e = lane; e < 32 * 16; e += 32) {
        const int col = e >> 4, ch = e & 15;
        cp_async16(Rp + col * kLaRld + 2 * ch, Rpan + col * 32 + 2 * ch);
    }
}

// warp 0: structured Householder QR of panel [Rp; Bt(:, c0..c0+31)]; lane c
// owns panel column c (its 32 tile rows in registers).  Reflector j (LAPACK
// dlarfg normalisation, tsqr.hpp:120-160): alpha = -sign(u0) ||[u0; x_j]||,
// tau = 1 + |u0| / ||u||, v = x_j / (u0 - alpha); zero column under a nonzero
// pivot: H = I; all-zero u: alpha = sqrt(2 DBL_MIN), tau = 2 (the reference's
// eps_fp result).  Per reflector the pivot lane publishes its column in
// shared memory (pv); every lane takes its dot product with it — for c > j
// that is the update's v^T x_c, for c < j (finished columns) it is entry
// (c, j) of S = V^T V up to the two scales — and lanes c > j update their
// column.  Columns stay unscaled until the panel ends (v_c = scale_c x_c).
// Leaves V in Bt, the updated block in Rp, tau, and striu(S) in Sm (ld kTld).
__device__ __forceinline__ double2 lds2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds1(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts2_if(bool p, unsigned a, double x, double y) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.v2.f64 [%1], {%2, %3}; }" ::"r"((unsigned)p), "r"(a),
                 "d"(x), "d"(y)
                 : "memory");
}
__device__ __forceinline__ void sts1_if(bool p, unsigned a, double x) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.f64 [%1], %2; }" ::"r"((unsigned)p), "r"(a), "d"(x)
                 : "memory");
}

__device__ __forceinline__ void la_panel(double* Bt, int c0, double* Rp, double* tau, double* pv, double* Sm,
                                         int lane) {
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
        const double2 t = *reinterpret_cast<const double2*>(Bt + (c0 + lane) * kBlkLdb + i);
        x[i] = t.x;
        x[i + 1] = t.y;
    }
    // shared-space addresses, fixed for the whole panel
    const unsigned s_pv = (unsigned)__cvta_generic_to_shared(pv);
    const unsigned s_rcol = (unsigned)__cvta_generic_to_shared(Rp + lane * kLaRld);  // R(., lane): + 8 j
    const unsigned s_scol = (unsigned)__cvta_generic_to_shared(Sm + lane * kTld);    // S(lane, .): + 8 j
    const unsigned s_tau = (unsigned)__cvta_generic_to_shared(tau);
    double my_scale = 1.0;
#pragma unroll 1
    for (int j = 0; j < 32; ++j) {
        const bool piv = (lane == j);
#pragma unroll
        for (int i = 0; i < 32; i += 2) sts2_if(piv, s_pv + 8 * i, x[i], x[i + 1]);
        __syncwarp();
        double a[8];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            const double2 p0 = lds2(s_pv + 8 * i);
            if (i < 16) {
                a[i / 2] = p0.x * x[i];
                a[i / 2] = fma(p0.y, x[i + 1], a[i / 2]);
            } else {
                a[(i - 16) / 2] = fma(p0.x, x[i], a[(i - 16) / 2]);
                a[(i - 16) / 2] = fma(p0.y, x[i + 1], a[(i - 16) / 2]);
            }
        }
        const double d = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
        const double sp = __shfl_sync(kFull, d, j);
        const unsigned s_rjj = (unsigned)__cvta_generic_to_shared(Rp + j * (kLaRld + 1));
        const double u0 = lds1(s_rjj);
        const double rjc = lds1(s_rcol + 8 * j);  // R(j, lane): meaningful for lane > j
        const double nrm2 = u0 * u0 + sp;
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
        if (nrm2 == 0.0) {  // all-zero u
            alpha = sqrt(2.0 * DBL_MIN);
            tj = 2.0;
            scale = 0.0;
        }
        const bool upd = lane > j;
        const double g = tj * (rjc + scale * d);
        const double f = upd ? g * scale : 0.0;
        my_scale = piv ? scale : my_scale;
        __syncwarp();
        sts1_if(upd, s_rcol + 8 * j, rjc - g);
        sts1_if(lane < j, s_scol + 8 * j, my_scale * scale * d);  // S(c, j) = v_c . v_j
        sts1_if(piv, s_rjj, alpha);
        sts1_if(piv, s_tau + 8 * j, tj);
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            const double2 p0 = lds2(s_pv + 8 * i);
            x[i] = fma(-f, p0.x, x[i]);
            x[i + 1] = fma(-f, p0.y, x[i + 1]);
        }
        __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < 32; i += 2)
        *reinterpret_cast<double2*>(Bt + (c0 + lane) * kBlkLdb + i) = make_double2(my_scale * x[i], my_scale * x[i + 1]);
    __syncwarp();
}

// warp 0: T = (diag(1/tau) + striu(S))^{-1} (lane j back-substitutes column j)
// into Tm (row-major, ld kLaTld); S comes from la_panel.
__device__ __forceinline__ void la_build_t(const double* Sm, const double* tau, double* Tm, int lane) {
    double t[32];
    const double tl = tau[lane];
#pragma unroll
    for (int i = 0; i < 32; ++i) t[i] = (i == lane) ? tl : 0.0;
#pragma unroll
    for (int i = 30; i >= 0; --i) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int l = i + 1; l < 32; l += 2) {
            a0 = fma(Sm[i * kTld + l], t[l], a0);
            if (l + 1 < 32) a1 = fma(Sm[i * kTld + l + 1], t[l + 1], a1);
        }
        if (i < lane) t[i] = -tau[i] * (a0 + a1);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) Tm[i * kLaTld + lane] = t[i];
}

// one warp: apply panel p's block reflector (V in Bt columns c0.., T) to the
// 8 tile columns g..g+7 and to R(p, g..g+7):
//   W = R(p, c) + V^T B(:, c);  W' = T^T W;  R(p, c) -= W';  B(:, c) -= V W'.
// Computed transposed (W^T, W'^T = W^T T) so the C fragments of one product
// become the A/B fragments of the next through 2 shuffles per k-step.
__device__ __forceinline__ void la_group(double* Bt, int c0, int g, const double* Tm, double* Rrow, int lane,
                                         uint64_t pol_r) {
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
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const double av = Bt[(g + r) * kBlkLdb + 4 * kk + q];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[nt], av, Bt[(c0 + 8 * nt + r) * kBlkLdb + 4 * kk + q]);
    }
    double w2[4][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) w2[nt][0] = w2[nt][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const int src = r * 4 + 2 * (kk & 1) + (q >> 1);
        const double s0 = __shfl_sync(kFull, acc[kk >> 1][0], src);
        const double s1 = __shfl_sync(kFull, acc[kk >> 1][1], src);
        const double av = (q & 1) ? s1 : s0;  // W^T[r][4kk + q]
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(w2[nt], av, Tm[(4 * kk + q) * kLaTld + 8 * nt + r]);
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
        st_hint(Rc + 8 * nt + 2 * q, rsav[nt][0] - w2[nt][0], pol_r);
        st_hint(Rc + 8 * nt + 2 * q + 1, rsav[nt][1] - w2[nt][1], pol_r);
    }
    double cb[4][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int e = 0; e < 2; ++e) cb[mt][e] = Bt[(g + 2 * q + e) * kBlkLdb + 8 * mt + r];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const int src = r * 4 + 2 * (kk & 1) + (q >> 1);
        const double s0 = __shfl_sync(kFull, w2[kk >> 1][0], src);
        const double s1 = __shfl_sync(kFull, w2[kk >> 1][1], src);
        const double bv = (q & 1) ? s1 : s0;  // W'[4kk + q][r]
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) dmma884(cb[mt], -Bt[(c0 + 4 * kk + q) * kBlkLdb + 8 * mt + r], bv);
    }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int e = 0; e < 2; ++e) Bt[(g + 2 * q + e) * kBlkLdb + 8 * mt + r] = cb[mt][e];
}

__device__ __forceinline__ void la_store_rdiag(const double* Rp, double* Rpan, int lane, uint64_t pol_r) {
    for (int e = lane; e < 32 * 32; e += 32) st_hint(Rpan + e, Rp[(e >> 5) * kLaRld + (e & 31)], pol_r);
}

__global__ void __launch_bounds__(kLaThreads, 2) tsqr_la_kernel(BlkArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int M = a.M, m = a.m;
    double* Bt = sm;                          // M columns x 32 rows, ld kBlkLdb
    double* Rp = Bt + (size_t)M * kBlkLdb;    // panel diagonal block of R (ld kLaRld)
    double* Sm = Rp + 32 * kLaRld;            // striu(V^T V) of the last panel (ld kTld)
    double* Tm0 = Sm + 32 * kTld;             // 2 x (32 x kLaTld)
    double* tau = Tm0 + 2 * 32 * kLaTld;      // 32
    double* pv = tau + 32;                    // 32: the panel's pivot column (16-byte aligned)

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
    for (int64_t e = tid; e < RS; e += kLaThreads) st_hint(R + e, R_init ? R_init[e] : 0.0, pol_r);
    // Roles.  The panel warp must not share its SM sub-partition (hardware
    // warp slot % 4) with another busy warp, including the panel warp of the
    // other CTA on the SM: pick sub-partition (slot of warp 0) / 8 mod 4 (the
    // co-resident CTA's slots start 8 further on), leave the second warp on
    // it idle, and run the block updates on the other six.
    __shared__ int slot_of[8], roles[2];
    if (lane == 0) {
        unsigned wid;
        asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
        slot_of[warp] = (int)wid;
    }
    __syncthreads();
    if (tid == 0) {
        const int want = (slot_of[0] / 8) & 3;
        int pw = 0, iw = 4;
        for (int w = 0; w < 8; ++w)
            if ((slot_of[w] & 3) == want) {
                pw = w;
                break;
            }
        for (int w = 0; w < 8; ++w)
            if (w != pw && (slot_of[w] & 3) == (slot_of[pw] & 3)) {
                iw = w;
                break;
            }
        if (iw == pw) iw = (pw + 4) & 7;
        roles[0] = pw;
        roles[1] = iw;
    }
    __syncthreads();
    const int pwarp = roles[0], iwarp = roles[1];
    const bool is_panel = (warp == pwarp), is_idle = (warp == iwarp);
    // rank among the six update warps
    const int wi = warp - (warp > pwarp) - (warp > iwarp);

    long long t_prev = 0, t_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define TT_PROF(ph)                                  \
    if (a.prof && lane == 0 && is_panel) {           \
        const long long t_now = clock64();           \
        if (t_prev) t_acc[ph] += t_now - t_prev;     \
        t_prev = t_now;                              \
    }
    TT_PROF(5);
    const int npan = M / 32;
    for (int64_t r0 = row0; r0 < row1; r0 += kBlkRows) {
        const int rows = (int)((row1 - r0) < kBlkRows ? (row1 - r0) : kBlkRows);
        const int p_first = a.mode == 1 ? (int)(r0 / 32) : 0;  // structural zeros of a triangular part
        if (is_panel) la_fetch_rdiag(Rp, R + blk_roff(p_first, M), lane);
        if (a.mode == 0) {
            for (int e = tid; e < M * kBlkRows; e += kLaThreads) {
                const int c = e >> 5, i = e & 31;
                Bt[c * kBlkLdb + i] = (i < rows && c < m) ? ld_stream_hint(X + (int64_t)c * ld + r0 + i, pol_x) : 0.0;
            }
        } else {
            const int t = (int)(r0 / 32);
            const double* src = X + blk_roff(t, M) - (int64_t)32 * 32 * t;
            for (int e = tid; e < M * kBlkRows; e += kLaThreads) {
                const int c = e >> 5, i = e & 31;
                Bt[c * kBlkLdb + i] = (c >= 32 * t) ? src[e] : 0.0;
            }
        }
        if (is_panel) cp_async_wait_all();
        __syncthreads();
        TT_PROF(0);
        if (is_panel) {
            la_panel(Bt, 32 * p_first, Rp, tau, pv, Sm, lane);
            la_store_rdiag(Rp, R + blk_roff(p_first, M), lane, pol_r);
            __syncwarp();
            TT_PROF(6);
            if (p_first + 1 < npan) la_build_t(Sm, tau, Tm0 + (p_first & 1) * 32 * kLaTld, lane);
            TT_PROF(7);
        }
        __syncthreads();
        TT_PROF(5);
        for (int p = p_first; p + 1 < npan; ++p) {
            const int c0 = 32 * p, nxt = c0 + 32;
            const double* Tp = Tm0 + (p & 1) * 32 * kLaTld;
            double* Rrow = R + blk_roff(p, M);
            if (is_panel) la_fetch_rdiag(Rp, R + blk_roff(p + 1, M), lane);
            if (!is_panel && !is_idle && wi < 4) {
                // phase A: the next panel's columns
                la_group(Bt, c0, nxt + 8 * wi, Tp, Rrow, lane, pol_r);
                __threadfence_block();
                asm volatile("bar.arrive 1, 160;" ::: "memory");
            }
            if (is_panel) {
                TT_PROF(5);
                asm volatile("bar.sync 1, 160;" ::: "memory");
                cp_async_wait_all();
                __syncwarp();
                TT_PROF(1);
                la_panel(Bt, nxt, Rp, tau, pv, Sm, lane);
                la_store_rdiag(Rp, R + blk_roff(p + 1, M), lane, pol_r);
                __syncwarp();
                TT_PROF(2);
                if (p + 2 < npan) la_build_t(Sm, tau, Tm0 + ((p + 1) & 1) * 32 * kLaTld, lane);
                TT_PROF(3);
            } else if (!is_idle) {
                const int idx = (wi + 2) % 6;  // the two warps without phase A work first
                for (int g = nxt + 32 + 8 * idx; g < M; g += 8 * 6) la_group(Bt, c0, g, Tp, Rrow, lane, pol_r);
            }
            __syncthreads();
            TT_PROF(4);
        }
    }
    if (a.prof && lane == 0 && is_panel)
        for (int q = 0; q < 8; ++q) a.prof[blockIdx.x * 8 + q] = t_acc[q];
#undef TT_PROF
}

}  // namespace ttsvd_b200
