// K_TSQR for short-fat work matrices (n / m <= 256, m > 32): one cooperative
// grid factorises the whole n x M matrix with blocked Householder QR (R only)
// instead of per-CTA flat trees + a merge tree.  For n / m ~ 8..128 the merge
// tree of the per-CTA path costs log2(G) sequential M-column structured QRs
// on single CTAs (config 2 step 3: ~26 of 31.6 ms); here every panel is
// shared by the whole GPU.
//
//   CTA c owns rows [c n/G, (c+1) n/G) for the whole factorisation.
//   Panel p (32 columns): the CTA's rows of the panel sit in shared memory;
//   reflector j needs the squared norm of column j below the pivot and the
//   dots with the panel columns right of it — per-CTA partials, one grid
//   barrier, then every CTA sums the partials in the same fixed order (so all
//   CTAs compute identical alpha/tau/gamma, deterministically) and updates
//   its rows.  LAPACK dlarfg normalisation; a zero column under a nonzero
//   pivot is H = I; an all-zero u gives alpha = sqrt(2 DBL_MIN) (tsqr.hpp:120).
//   Then T = (diag(1/tau) + striu(Y^T Y))^{-1}, W = Y^T A(:, trail) by split-K
//   DMMA over the CTAs' rows, W' = T^T W reduced column-chunk-wise, and every
//   CTA updates its rows A -= Y W' on DMMA.
//   A is a private copy of the work matrix (the TSMM still needs the original).
#pragma once

#include <cooperative_groups.h>
#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kGqrThreads = 256;  // threads of the 256-thread variant (rows per CTA <= 256)
constexpr int kGqrMaxRows = 512;  // rows per CTA (panel rows in shared memory)
constexpr int kGqrCluster = 16;   // CTAs of the cluster variant

struct GqrArgs {
    double* A;       // n x M, ld lda (column-major), factorised in place
    int64_t n, lda;
    int m, M;
    double* part;    // reduction partials: 2 x G x 33 (reflectors), G x 32 x 32 (S), G x 32 x M (W)
    double* piv;     // 2 x 32: the pivot row of the current reflector
    double* Wfin;    // 32 x M: W' = T^T W of the current panel
    double* Sfin;    // 1024: S = Y^T Y of the current panel
    long long* prof; // optional (diagnostics): CTA 0 cycle sums [stage, reflectors, writeback+S+T, W partial, W reduce, update]
};

__device__ __forceinline__ long long gqr_clock() {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}

// 32 per-lane values -> lane k holds the warp sum of value k (butterfly
// reduce-scatter: 16 + 8 + 4 + 2 + 1 shuffles)
__device__ __forceinline__ double warp_reduce_scatter32(double (&v)[32], int lane) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2, b0 = lane & 1;
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = (b4 ? v[k + 16] : v[k]) + __shfl_xor_sync(0xffffffffu, b4 ? v[k] : v[k + 16], 16);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (b3 ? v[k + 8] : v[k]) + __shfl_xor_sync(0xffffffffu, b3 ? v[k] : v[k + 8], 8);
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (b2 ? v[k + 4] : v[k]) + __shfl_xor_sync(0xffffffffu, b2 ? v[k] : v[k + 4], 4);
#pragma unroll
    for (int k = 0; k < 2; ++k) v[k] = (b1 ? v[k + 2] : v[k]) + __shfl_xor_sync(0xffffffffu, b1 ? v[k] : v[k + 2], 2);
    return (b0 ? v[1] : v[0]) + __shfl_xor_sync(0xffffffffu, b0 ? v[0] : v[1], 1);
}

__device__ __forceinline__ double gqr_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// sum over q = first, first + step, ... < G of base[q * qstride] (L2 reads,
// data of other CTAs) in a fixed association order, so every CTA computes
// bit-identical totals; CH loads in flight per chunk (one L2 round trip per
// chunk)
template <int CH>
__device__ __forceinline__ double gqr_sum_inflight(const double* base, int64_t qstride, int G, int first, int step) {
    double s = 0.0;
    for (int q0 = first; q0 < G; q0 += CH * step) {
        double v[CH];
#pragma unroll
        for (int u = 0; u < CH; ++u) {
            const int q = q0 + u * step;
            v[u] = q < G ? __ldcg(base + (int64_t)q * qstride) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < CH; ++u) s += v[u];
    }
    return s;
}

__host__ __device__ inline int gqr_ldy(int rows) { return ((((rows + 3) & ~3) + 7) & ~7) + 4; }

inline size_t gqr_smem_bytes(int rows_max, int nt = kGqrThreads) {
    const int ldy = gqr_ldy(rows_max);
    return ((size_t)32 * ldy + 2 * 32 * 33 + 32 + 2 * (nt / 32) * 33 + (nt / 32) * 32 * 9 + 40) * sizeof(double);
}

// CL = false: one cooperative grid (grid.sync); CL = true: the grid is one
// thread-block cluster (<= 16 CTAs) and every grid barrier is a cluster
// barrier (arrive.release / wait.acquire orders the global-memory partials
// at cluster scope) — ~0.2 us instead of ~2 us per barrier for the short
// steps (n <= 16 x 512)
template <bool CL, int NT>
__global__ void __launch_bounds__(NT, 1) gqr_kernel(GqrArgs a) {
    namespace cg = cooperative_groups;
    auto gsync = [&]() {
        if constexpr (CL) {
            asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else {
            cg::this_grid().sync();
        }
    };
    // the explicit fences of the grid path (the per-reflector barrier relies
    // on grid.sync's own fence); the cluster barrier's release covers them
    auto gfence = [&]() {
        if constexpr (!CL) __threadfence();
    };
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t n = a.n, lda = a.lda;
    const int M = a.M;
    const int64_t base = n / G, rem = n % G;
    const int64_t r0 = c * base + (c < rem ? c : rem);
    const int rows = (int)(base + (c < rem ? 1 : 0));
    const int rows4 = (rows + 3) & ~3;      // K extent for DMMA (zero padded)
    const int ldy = gqr_ldy(rows);           // smem ld of the panel rows
    double* Ys = sm;                         // 32 columns x ldy
    double* Sm = Ys + 32 * ldy;              // 32 x 33
    double* Tm = Sm + 32 * 33;               // 32 x 33
    double* tau = Tm + 32 * 33;              // 32
    double* red = tau + 32;                  // 2 NW x 33 (warp totals, then slice totals)
    double* Wsc = red + 2 * (NT / 32) * 33;  // per-warp 32 x 8 (ld 9)
    double* gsm = Wsc + (NT / 32) * 32 * 9;  // 32 gamma + scale, alpha
    double* part = a.part;
    double* A = a.A;
    const int lr = lane >> 2, lc = lane & 3;

    const bool pf = a.prof && c == 0 && tid == 0;
    long long tpv = pf ? gqr_clock() : 0;
#define GQR_PROF(ph)                          \
    if (pf) {                                 \
        const long long tn = gqr_clock();     \
        a.prof[ph] += tn - tpv;               \
        tpv = tn;                             \
    }
    for (int p = 0; p < M / 32; ++p) {
        const int64_t c0 = 32 * (int64_t)p;
        // ---- stage my rows of the panel (8-byte cp.async: all loads in flight) ----
        for (int k = warp; k < 32; k += NT / 32) {
            const double* src = A + (c0 + k) * lda + r0;
            double* dst = Ys + k * ldy;
            for (int i = lane; i < ldy; i += 32) {
                if (i < rows) {
                    const unsigned sd = (unsigned)__cvta_generic_to_shared(dst + i);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sd), "l"(src + i) : "memory");
                } else {
                    dst[i] = 0.0;
                }
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        // ---- 32 reflectors, one grid barrier each ----
        GQR_PROF(0);
        // The CTA's rows of the panel live in registers for the 32 reflectors
        // (warp w: rows 32 w .. 32 w + 31 as 4-row x 8-column tiles, lane
        // rq + 8 cg: rows 32 w + rq + 8 r, columns 8 cg + c — the layout of
        // tsqr_t128's panel): the pivot column reaches the other column groups
        // by 4 shuffles, a 7-shuffle transpose-reduce leaves column `lane`'s
        // warp dot in lane `lane`, and the rank-1 update is 32 register FMAs
        // per lane.  (With the panel in shared memory the update was two
        // shared-memory accesses per FMA: ~3 k of the ~10.5 k cycles per
        // reflector, and the dots another 1.4 k.)  Rows above the pivot are
        // zero in the registers (their panel entries stay in Ys); a pivot row
        // is written to Ys and zeroed as soon as its reflector has been applied.
        constexpr int NW = NT / 32;
        const int rq = lane & 7, cg = lane >> 3;
        double* dpart = Wsc;  // 2 x NW x 32 warp partials (Wsc is free until the blocked update)
        double x[4][8];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = 32 * warp + rq + 8 * r;
            const bool live = i < rows && r0 + i >= c0;
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) x[r][cc] = live ? Ys[(8 * cg + cc) * ldy + i] : 0.0;
        }
#pragma unroll 1
        for (int cgj = 0; cgj < 4; ++cgj) {
#pragma unroll
            for (int cj = 0; cj < 8; ++cj) {
                const int jj = 8 * cgj + cj;
                const int64_t j = c0 + jj;
                const int buf = jj & 1;
                long long tr0 = pf ? gqr_clock() : 0;
                const int li = (int)(j - r0);  // the pivot's row among mine (if 0 <= li < rows)
                const bool mine = li >= 0 && li < rows && (li >> 5) == warp && (li & 7) == rq;  // my rows hold it
                const int rp = (li >> 3) & 3;
                double pr[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) pr[r] = __shfl_sync(0xffffffffu, x[r][cj], rq + 8 * cgj);
                if (mine) {  // pivot row -> broadcast slot
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        const double v = rp == 0 ? x[0][cc] : (rp == 1 ? x[1][cc] : (rp == 2 ? x[2][cc] : x[3][cc]));
                        a.piv[buf * 32 + 8 * cg + cc] = v;
                    }
                }
                // dots over the rows below the pivot: value 0 = sum x_j^2, value k = sum x_j x_k
                double acc[8];
#pragma unroll
                for (int r = 0; r < 4; ++r) pr[r] = (mine && r == rp) ? 0.0 : pr[r];  // the pivot row stays out
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    acc[cc] = pr[0] * x[0][cc];
#pragma unroll
                    for (int r = 1; r < 4; ++r) acc[cc] = fma(pr[r], x[r][cc], acc[cc]);
                }
                // transpose-reduce over the row lanes: lane ends with column 8 cg + rq = lane
#pragma unroll
                for (int o = 4; o >= 1; o >>= 1) {
                    const bool up = (lane & o) != 0;
#pragma unroll
                    for (int t = 0; t < o; ++t) {
                        const double send = up ? acc[t] : acc[t + o];
                        const double keep = up ? acc[t + o] : acc[t];
                        acc[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                    }
                }
                dpart[(buf * NW + warp) * 32 + lane] = acc[0];
                __syncthreads();
                if (tid < 32) {
                    double t = 0.0;
#pragma unroll
                    for (int w = 0; w < NW; ++w) t += dpart[(buf * NW + w) * 32 + tid];
                    const double tj = __shfl_sync(0xffffffffu, t, jj);
                    part[((int64_t)buf * G + c) * 33 + tid] = tid == 0 ? tj : (tid > jj ? t : 0.0);
                }
                long long tq0 = pf ? gqr_clock() : 0;
                if (pf) a.prof[6] += tq0 - tr0;
                // grid.sync orders the partials: its barrier is preceded by a
                // device-scope fence on behalf of the whole CTA
                gsync();
                // totals in a fixed order (identical on every CTA): value k = tid & 31,
                // slice s = tid >> 5 sums CTAs q = s, s + 8, ...; then the 8 slices
                {
                    const int k = tid & 31, sl = tid >> 5;
                    const double pv = (sl == 0) ? __ldcg(&a.piv[buf * 32 + k]) : 0.0;  // in flight with the sums
                    // (columns 1 .. jj carry no value: no loads for them)
                    red[(NT / 32) * 33 + sl * 33 + k] =
                        (k == 0 || k > jj) ? gqr_sum_inflight<20>(part + (int64_t)buf * G * 33 + k, 33, G, sl, NT / 32)
                                           : 0.0;
                    if (sl == 0) red[33 + k] = pv;
                }
                __syncthreads();
                // warp 0: the totals, the reflector (every CTA derives the same
                // bits) and gamma_k = tau (A(j,k) + scale d_k) for the columns
                // k > jj, once per CTA instead of once per thread
                if (tid < 32) {
                    double t = 0.0;
#pragma unroll
                    for (int sl = 0; sl < NT / 32; ++sl) t += red[(NT / 32) * 33 + sl * 33 + tid];
                    const double pk = red[33 + tid];
                    const double sp = __shfl_sync(0xffffffffu, t, 0);
                    const double u0 = __shfl_sync(0xffffffffu, pk, jj);
                    const double nrm2 = u0 * u0 + sp;
                    const double inv = fast_rsqrt(nrm2);
                    const double nr = nrm2 * inv;
                    const double au = fabs(u0);
                    const double sg = (u0 > 0.0) ? 1.0 : -1.0;
                    double alpha = -sg * nr, tj = 1.0 + au * inv, scale = sg * fast_rcp(au + nr);
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
                    gsm[tid] = (tid > jj) ? tj * (pk + scale * t) : 0.0;
                    if (tid == 0) {
                        gsm[32] = scale;
                        gsm[33] = alpha;
                        tau[jj] = tj;
                    }
                }
                __syncthreads();
                if (pf) {
                    const long long tq1 = gqr_clock();
                    a.prof[7] += tq1 - tq0;
                }
                // rank-1 update of my rows in registers: x_k -= gamma_k f with
                // f = x_j scale (the pivot row: f = 1); column j keeps v = f
                // (the pivot row: alpha).  gamma_k = 0 for k <= jj.
                {
                    const double scale = gsm[32], alpha = gsm[33];
                    double f[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) f[r] = (mine && r == rp) ? 1.0 : pr[r] * scale;
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        const double gk = gsm[8 * cg + cc];
#pragma unroll
                        for (int r = 0; r < 4; ++r) x[r][cc] = fma(-gk, f[r], x[r][cc]);
                    }
                    if (cg == cgj) {
#pragma unroll
                        for (int r = 0; r < 4; ++r) x[r][cj] = (mine && r == rp) ? alpha : f[r];
                    }
                    if (mine) {  // the pivot row is final: to Ys, and out of the later dots and updates
#pragma unroll
                        for (int cc = 0; cc < 8; ++cc) {
                            const double v = rp == 0 ? x[0][cc] : (rp == 1 ? x[1][cc] : (rp == 2 ? x[2][cc] : x[3][cc]));
                            Ys[(8 * cg + cc) * ldy + li] = v;
                        }
#pragma unroll
                        for (int r = 0; r < 4; ++r)
                            if (r == rp) {
#pragma unroll
                                for (int cc = 0; cc < 8; ++cc) x[r][cc] = 0.0;
                            }
                    }
                }
            }
        }
        // the rows below the panel's last pivot (v of all 32 reflectors) back to Ys
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = 32 * warp + rq + 8 * r;
            if (i < rows && r0 + i >= c0 + 32) {
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) Ys[(8 * cg + cc) * ldy + i] = x[r][cc];
            }
        }
        __syncthreads();
        GQR_PROF(1);
        // ---- write back the panel (R rows and v), then the structured Y in smem ----
        for (int e = tid; e < 32 * ldy; e += NT) {
            const int k = e / ldy, i = e - k * ldy;
            if (i < rows) {
                A[(c0 + k) * lda + r0 + i] = Ys[e];
                const int64_t gi = r0 + i;
                Ys[e] = gi > c0 + k ? Ys[e] : (gi == c0 + k ? 1.0 : 0.0);
            }
        }
        __syncthreads();
        if (c0 + 32 >= M) break;
        // ---- S = Y^T Y partial (DMMA over my rows), reduce, T ----
        if (warp < 4) {
            const int nt = warp;
            double sacc[4][2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) sacc[mt][0] = sacc[mt][1] = 0.0;
            for (int kk = 0; kk < rows4 / 4; ++kk) {
                const double b = Ys[(8 * nt + lr) * ldy + 4 * kk + lc];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) dmma884(sacc[mt], Ys[(8 * mt + lr) * ldy + 4 * kk + lc], b);
            }
            double* ps = part + (int64_t)2 * G * 33 + (int64_t)c * 1024;
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int e = 0; e < 2; ++e) ps[(8 * mt + lr) * 32 + 8 * nt + 2 * lc + e] = sacc[mt][e];
        }
        gfence();
        gsync();
        // S = sum of the G partials, distributed: CTA c reduces entries
        // [c E, (c+1) E) (warp per entry, lanes over the CTAs, fixed butterfly
        // order), one grid barrier, then every CTA reads the 1024 totals
        {
            const int E = (1024 + G - 1) / G;
            const double* ps = part + (int64_t)2 * G * 33;
            for (int el = warp; el < E; el += NT / 32) {
                const int e = c * E + el;
                if (e < 1024) {
                    double s = gqr_sum_inflight<8>(ps + e, 1024, G, lane, 32);
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    if (lane == 0) a.Sfin[e] = s;
                }
            }
        }
        gfence();
        gsync();
        {
            double sv[1024 / NT];
#pragma unroll
            for (int r = 0; r < 1024 / NT; ++r) sv[r] = __ldcg(a.Sfin + tid + r * NT);
#pragma unroll
            for (int r = 0; r < 1024 / NT; ++r) {
                const int e = tid + r * NT;
                Sm[(e >> 5) * 33 + (e & 31)] = sv[r];
            }
        }
        __syncthreads();
        if (warp == 0) {
            const int b0 = 8 * (lane >> 3), jx = lane & 7;
            for (int i = 0; i < 32; ++i) Tm[i * 33 + b0 + jx] = 0.0;
            Tm[(b0 + jx) * 33 + b0 + jx] = tau[b0 + jx];
            for (int i = jx - 1; i >= 0; --i) {
                double acc = 0.0;
                for (int l = i + 1; l <= jx; ++l) acc += Sm[(b0 + i) * 33 + b0 + l] * Tm[(b0 + l) * 33 + b0 + jx];
                Tm[(b0 + i) * 33 + b0 + jx] = -tau[b0 + i] * acc;
            }
        }
        __syncthreads();
        for (int lev = 8; lev <= 16; lev *= 2) {
            double* Xs = Wsc;
            const int nblk = 32 / (2 * lev);
            for (int e = tid; e < nblk * lev * lev; e += NT) {
                const int q = e / (lev * lev), i = (e / lev) % lev, jx = e % lev;
                const int o = q * 2 * lev;
                double acc = 0.0;
                for (int l = 0; l <= jx; ++l) acc += Sm[(o + i) * 33 + o + lev + l] * Tm[(o + lev + l) * 33 + o + lev + jx];
                Xs[q * 17 * 17 + i * 17 + jx] = acc;
            }
            __syncthreads();
            for (int e = tid; e < nblk * lev * lev; e += NT) {
                const int q = e / (lev * lev), i = (e / lev) % lev, jx = e % lev;
                const int o = q * 2 * lev;
                double acc = 0.0;
                for (int l = i; l < lev; ++l) acc += Tm[(o + i) * 33 + o + l] * Xs[q * 17 * 17 + l * 17 + jx];
                Tm[(o + i) * 33 + o + lev + jx] = -acc;
            }
            __syncthreads();
        }
        GQR_PROF(2);
        // ---- W partial = Y_c^T A(rows_c, trail): DMMA, K = my rows ----
        const int64_t t0 = c0 + 32;
        const int ngr = (int)((M - t0) / 8);
        double* pw = part + (int64_t)2 * G * 33 + (int64_t)G * 1024;  // G x 32 x M (cols t0..M used)
        for (int gq = warp; gq < ngr; gq += NT / 32) {
            const int64_t g = t0 + 8 * gq;
            double acc[4][2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
            const double* colp = A + (g + lr) * lda + r0;
            for (int k0 = 0; k0 < rows4 / 4; k0 += 8) {
                double bv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int row = 4 * (k0 + u) + lc;
                    bv[u] = (k0 + u < rows4 / 4 && row < rows) ? colp[row] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (k0 + u < rows4 / 4) {
#pragma unroll
                        for (int mt = 0; mt < 4; ++mt)
                            dmma884(acc[mt], Ys[(8 * mt + lr) * ldy + 4 * (k0 + u) + lc], bv[u]);
                    }
                }
            }
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int e = 0; e < 2; ++e) pw[((int64_t)c * 32 + 8 * mt + lr) * M + g + 2 * lc + e] = acc[mt][e];
        }
        gfence();
        gsync();
        GQR_PROF(3);
        // ---- reduce W over the CTAs (column chunks), W' = T^T W -> Wfin ----
        {
            const int64_t ncols = M - t0;
            const int64_t chunk = (ncols + G - 1) / G;
            const int64_t ca = t0 + c * chunk, cb = (ca + chunk < M) ? ca + chunk : M;
            // per column: thread (k = lane, slice = warp) sums CTAs q = warp,
            // warp + 8, ... (loads in flight), then warp 0 adds the 8 slices
            // in order and forms W'(:, col) = T^T W(:, col)
            double* wsl = Wsc;  // 8 x 33
            for (int64_t col = ca; col < cb; ++col) {
                wsl[warp * 33 + lane] = gqr_sum_inflight<20>(pw + (int64_t)lane * M + col, (int64_t)32 * M, G, warp, NT / 32);
                __syncthreads();
                if (warp == 0) {
                    double w = 0.0;
#pragma unroll
                    for (int sl = 0; sl < NT / 32; ++sl) w += wsl[sl * 33 + lane];
                    double wp = 0.0;
                    for (int k = 0; k < 32; ++k) wp = fma(Tm[k * 33 + lane], __shfl_sync(0xffffffffu, w, k), wp);
                    a.Wfin[(int64_t)lane * M + col] = wp;
                }
                __syncthreads();
            }
        }
        gfence();
        gsync();
        GQR_PROF(4);
        // ---- A(rows_c, trail) -= Y_c W': DMMA per 8-column group, 64-row chunks ----
        for (int gq = warp; gq < ngr; gq += NT / 32) {
            const int64_t g = t0 + 8 * gq;
            double* Ws = Wsc + warp * 32 * 9;
            for (int e = lane; e < 256; e += 32) Ws[(e >> 3) * 9 + (e & 7)] = __ldcg(&a.Wfin[(int64_t)(e >> 3) * M + g + (e & 7)]);
            __syncwarp();
            double wf[8];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) wf[kk] = Ws[(4 * kk + lc) * 9 + lr];
            for (int rb = 0; rb < rows4; rb += 64) {
                double cbv[8][2];
#pragma unroll
                for (int mt = 0; mt < 8; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int row = rb + 8 * mt + lr;
                        cbv[mt][e] = row < rows ? A[(g + 2 * lc + e) * lda + r0 + row] : 0.0;
                    }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
#pragma unroll
                    for (int mt = 0; mt < 8; ++mt) {
                        const int row = rb + 8 * mt + lr;
                        const double y = row < ldy ? Ys[(4 * kk + lc) * ldy + row] : 0.0;
                        dmma884(cbv[mt], -y, wf[kk]);
                    }
#pragma unroll
                for (int mt = 0; mt < 8; ++mt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int row = rb + 8 * mt + lr;
                        if (row < rows) A[(g + 2 * lc + e) * lda + r0 + row] = cbv[mt][e];
                    }
            }
            __syncwarp();
        }
        gfence();
        gsync();
        GQR_PROF(5);
    }
#undef GQR_PROF
}

// count packed panel-major factors (blk_rsize(M) each) -> the dense stacked
// matrix S (count*M x M, ld count*M): rows [q M, (q+1) M) hold factor q
// (zeros below its diagonal)
__global__ void stack_packed_kernel(const double* parts, int64_t count, int M, double* S) {
    const int64_t RS = blk_rsize(M), ld = count * M;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ld * M; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t col = e / ld, row = e - col * ld;
        const int64_t q = row / M;
        const int i = (int)(row - q * M), j = (int)col;
        const int p = i >> 5;
        S[e] = (i <= j) ? parts[q * RS + blk_roff(p, M) + (int64_t)(j - 32 * p) * 32 + (i & 31)] : 0.0;
    }
}

// upper triangle of A(0:m, 0:m) (ld lda) -> R (m x m, ld m)
__global__ void gqr_extract_kernel(const double* A, int64_t lda, int m, double* R) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += gridDim.x * blockDim.x) {
        const int j = e / m, i = e - j * m;
        R[e] = i <= j ? A[(int64_t)j * lda + i] : 0.0;
    }
}

}  // namespace ttsvd_b200
