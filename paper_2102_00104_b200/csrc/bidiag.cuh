// K_SVD for the TT-SVD driver (no rotation accumulation): sigma and the
// leading left singular vectors of the n x m work matrix A (n >= m; A = R^T
// of a tall step or W^T of a wide step, so A's left singular vectors are the
// right singular vectors of the step's matrix) by Householder
// bidiagonalisation, bisection and inverse iteration — in place of the
// one-sided Jacobi sweeps, whose ~13 sweeps x 127 rounds are latency bound.
//
//   1. bd_kernel (one thread-block cluster, A in the CTAs' shared memory,
//      `cpc` columns per CTA): A = U_B B V_B^T, B upper bidiagonal (d, e).
//      Step k: the left reflector of column k (owner CTA; LAPACK dlarfg
//      normalisation, beta = -sign(alpha) ||x||), broadcast through
//      distributed shared memory and applied by every CTA to its columns;
//      then the right reflector of row k (row norm: one partial per CTA,
//      summed in CTA order so every CTA derives the same reflector), its
//      product z = A v reduce-scattered and all-gathered through DSMEM, and
//      the rank-1 update.  Four cluster barriers per step.  Column k keeps
//      the left reflector u_k below the diagonal (u_k[k] = 1).
//   2. bd_bisect_kernel: every sigma of B (descending) by 32-way
//      multisection per warp on the Golub-Kahan tridiagonal T (zero
//      diagonal, off-diagonals d1 e1 d2 ... dm; Sturm counts of T - s I).
//   3. bd_vectors_kernel: the left singular vectors x of B for the leading
//      r sigmas by inverse iteration on T (the x entries of T's eigenvector
//      (y1 x1 y2 x2 ...)); sigmas closer than 1e-3 ||T|| form a cluster that
//      one thread iterates with modified Gram-Schmidt against its earlier
//      members (LAPACK dstein's scheme).
//   4. bd_back_kernel: V = U_B [x; 0] by the stored left reflectors.
//
// sigma is accurate to ~eps ||A|| absolute (backward stable
// bidiagonalisation; bisection to 1e-18 ||T||), vector i to
// ~eps ||A|| / gap_i, the same orders as the Jacobi path's normalised
// columns.
#pragma once

#include <cfloat>
#include <cstdint>

namespace ttsvd_b200 {

constexpr int kBdThreads = 512;

struct BdArgs {
    double* A;  // n x m (ld n), overwritten below the diagonal with the left reflectors
    int n, m, cpc;
    double* d;     // m
    double* e;     // m - 1
    double* tauL;  // m
    double* xg;    // exchange (global, L2): u_k (2 x (n + 1), by step parity), partial z (16 x n),
                   // row-norm partials + A[k][k+1] (2 x 2C, by step parity)
    long long* prof;  // optional (diagnostics): CTA 0 cycle sums per phase
};

inline size_t bd_smem_bytes(int n, int cpc) { return ((size_t)cpc * n + 3 * (size_t)n + 3 * (size_t)cpc + 8) * sizeof(double); }

// split cluster barrier (arrive.release / wait.acquire)
__device__ __forceinline__ void bd_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void bd_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// sum over the CTA (every thread gets the same value; fixed order)
__device__ __forceinline__ double bd_block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kBdThreads / 32; ++w) s += red[w];
    return s;
}

__device__ __forceinline__ double bd_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int kBdCluster = 16;

// CPC: compile-time columns per CTA (the row passes keep a row's CPC entries
// in registers); a.cpc <= CPC
template <int CPC>
__global__ void __launch_bounds__(kBdThreads, 1) bd_kernel(BdArgs a) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[32];
    __shared__ double pub[4];  // [k & 1] tau_L (owner of column k; two slots: the last steps have no
                               // barrier between a read and the next write), [2] row-norm partial, [3] A[k][k+1]
    __shared__ double rs[2];   // row reflector inputs, CTA-local copies
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int C = kBdCluster;
    const int rank = (int)cl.block_rank();
    const int n = a.n, m = a.m, cpc = CPC;
    double* As = sm;          // cpc columns, ld n
    double* ub = As + (size_t)cpc * n;
    double* zp = ub + n;      // partial z over my columns
    double* zf = zp + n;      // full z
    double* vl = zf + n;      // right reflector, my columns
    double* wl = vl + cpc;    // left-reflector products w_j
    double* rk = wl + cpc;    // row k after the left update
    const int c0 = rank * cpc;
    double* ug = a.xg;
    double* zg = a.xg + 2 * (size_t)(n + 1);
    for (int e = tid; e < cpc * n; e += kBdThreads) {
        const int j = e / n, i = e - j * n, gj = c0 + j;
        As[e] = gj < m ? a.A[(int64_t)gj * n + i] : 0.0;
    }
    __syncthreads();
    cl.sync();
    long long* pf = (a.prof && rank == C - 1 && tid == 0) ? a.prof : nullptr;  // the last CTA: active to the end
    long long tp = pf ? bj_clock() : 0;
#define BD_MARK(i)                           \
    if (pf) {                                \
        const long long tq = bj_clock();     \
        pf[i] += tq - tp;                    \
        tp = tq;                             \
    }
    // the owner of column k computes its left reflector at the end of step
    // k-1 (after updating that one column), arrives at the cluster barrier and
    // only then updates its other columns; step 0's reflector is computed here
    auto left_reflector = [&](int k) {
        double* col = As + (size_t)(k - c0) * n;
        double s = 0.0;
        for (int i = k + 1 + tid; i < n; i += kBdThreads) s = fma(col[i], col[i], s);
        s = bd_block_sum(s, red);
        const double alpha = col[k];
        double tau = 0.0, beta = alpha, scale = 0.0;
        if (s != 0.0) {
            const double nr = sqrt(fma(alpha, alpha, s));
            beta = alpha >= 0.0 ? -nr : nr;
            tau = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        double* ug_k = ug + (size_t)(k & 1) * (n + 1);
        for (int i = k + 1 + tid; i < n; i += kBdThreads) {
            const double u = col[i] * scale;
            col[i] = u;
            __stcg(ug_k + i, u);
        }
        if (tid == 0) {
            col[k] = 1.0;
            __stcg(ug_k + k, 1.0);
            __stcg(ug_k + n, tau);
            a.d[k] = beta;
            a.tauL[k] = tau;
        }
        __syncthreads();
    };
    if (rank == 0) left_reflector(0);
    bd_arrive();
    for (int k = 0; k < m; ++k) {
        const int lj0 = max(0, k + 1 - c0);  // first local column right of k
        const int lj1 = min(cpc, m - c0);     // past the last real column
        bd_wait();  // B1: u_k published
        BD_MARK(0)
        {
            // u_k through L2 (16 readers of one SM's shared memory would
            // serialise on its DSMEM port)
            const double* ug_k = ug + (size_t)(k & 1) * (n + 1);
            for (int i = k + tid; i < n; i += kBdThreads) ub[i] = __ldcg(ug_k + i);
            if (tid == 0) rs[0] = __ldcg(ug_k + n);
        }
        __syncthreads();
        BD_MARK(1)
        const double tauL = rs[0];
        // ---- pass 1: w_j = tau_L u^T a_j (warp per column); row k after the
        // left update: a_kj - w_j (u_k = 1) ----
        for (int la = lj0 + warp; la < lj1; la += 2 * (kBdThreads / 32)) {
            const int lb = la + kBdThreads / 32;  // second column of this warp (if any)
            const bool hb = lb < lj1;
            const double* ca = As + (size_t)la * n;
            const double* cb = As + (size_t)(hb ? lb : la) * n;
            double da0 = 0.0, da1 = 0.0, db0 = 0.0, db1 = 0.0;
            int i = k + lane;
            for (; i + 32 < n; i += 64) {
                const double u0 = ub[i], u1 = ub[i + 32];
                da0 = fma(u0, ca[i], da0);
                da1 = fma(u1, ca[i + 32], da1);
                db0 = fma(u0, cb[i], db0);
                db1 = fma(u1, cb[i + 32], db1);
            }
            if (i < n) {
                da0 = fma(ub[i], ca[i], da0);
                db0 = fma(ub[i], cb[i], db0);
            }
            const double wa = tauL * bd_warp_sum(da0 + da1);
            const double wb = tauL * bd_warp_sum(db0 + db1);
            if (lane == 0) {
                wl[la] = wa;
                rk[la] = ca[k] - wa;
                if (hb) {
                    wl[lb] = wb;
                    rk[lb] = cb[k] - wb;
                }
            }
        }
        __syncthreads();
        BD_MARK(2)
        if (k + 2 < m) {
            // ---- right reflector of row k (columns k+1 ..) ----
            if (warp == 0) {
                double s = 0.0;
                for (int lj = max(lj0, k + 2 - c0) + lane; lj < lj1; lj += 32) s = fma(rk[lj], rk[lj], s);
                s = bd_warp_sum(s);
                if (lane == 0) {
                    pub[2] = s;
                    if ((k + 1) / cpc == rank) pub[3] = rk[k + 1 - c0];
                }
            }
            __syncthreads();
            cl.sync();  // B2
            BD_MARK(3)
            if (warp == 0) {
                double p = lane < C ? *cl.map_shared_rank(&pub[2], lane) : 0.0;
                p = bd_warp_sum(p);
                if (lane == 0) {
                    rs[0] = p;
                    rs[1] = *cl.map_shared_rank(&pub[3], (k + 1) / cpc);
                }
            }
            __syncthreads();
            const double st = rs[0], y0 = rs[1];
            double tauR = 0.0, gamma = y0, scaleR = 0.0;
            if (st != 0.0) {
                const double nr = sqrt(fma(y0, y0, st));
                gamma = y0 >= 0.0 ? -nr : nr;
                tauR = (gamma - y0) / gamma;
                scaleR = 1.0 / (y0 - gamma);
            }
            if (rank == 0 && tid == 0) a.e[k] = gamma;
            for (int lj = lj0 + tid; lj < lj1; lj += kBdThreads) vl[lj] = (c0 + lj == k + 1) ? 1.0 : rk[lj] * scaleR;
            __syncthreads();
            // ---- pass 2 (thread per row): left update, z partial ----
            for (int i = k + 1 + tid; i < n; i += kBdThreads) {
                const double ui = ub[i];
                double z = 0.0;
                for (int lj = lj0; lj < lj1; ++lj) {
                    double* pa = As + (size_t)lj * n + i;
                    const double x = fma(-wl[lj], ui, *pa);
                    *pa = x;
                    z = fma(x, vl[lj], z);
                }
                zg[(size_t)rank * n + i] = z;
            }
            BD_MARK(4)
            cl.sync();  // B3
            BD_MARK(5)
            // ---- z = tau_R sum of the partials (same order on every CTA),
            // right update; the owner of column k+1 updates it first and
            // publishes the next left reflector before the others ----
            const int on = (k + 1) / cpc;
            if (lj0 < lj1) {
                for (int i = k + 1 + tid; i < n; i += kBdThreads) {
                    double p[C];
#pragma unroll
                    for (int t = 0; t < C; ++t) p[t] = __ldcg(zg + (size_t)t * n + i);
                    double z = 0.0;
#pragma unroll
                    for (int t = 0; t < C; ++t) z += p[t];
                    zf[i] = tauR * z;
                }
            }
            __syncthreads();
            BD_MARK(6)
            if (rank == on) {
                double* col = As + (size_t)(k + 1 - c0) * n;
                for (int i = k + 1 + tid; i < n; i += kBdThreads) col[i] = fma(-zf[i], 1.0, col[i]);
                __syncthreads();
                left_reflector(k + 1);
            }
            bd_arrive();
            {
                const int skip = (rank == on) ? k + 1 - c0 : -1;  // the owner's column k+1 is done
                for (int i = k + 1 + tid; i < n; i += kBdThreads) {
                    const double z = zf[i];
                    for (int lj = lj0; lj < lj1; ++lj)
                        if (lj != skip) As[(size_t)lj * n + i] = fma(-z, vl[lj], As[(size_t)lj * n + i]);
                }
            }
            __syncthreads();
            BD_MARK(7)
        } else {
            // last two steps: left update only (no right reflector)
            for (int i = k + 1 + tid; i < n; i += kBdThreads) {
                const double ui = ub[i];
                for (int lj = lj0; lj < lj1; ++lj) As[(size_t)lj * n + i] = fma(-wl[lj], ui, As[(size_t)lj * n + i]);
            }
            if (k + 2 == m && (k + 1) / cpc == rank && tid == 0) a.e[k] = rk[k + 1 - c0];
            __syncthreads();
            if (k + 1 < m && (k + 1) / cpc == rank) left_reflector(k + 1);
            bd_arrive();
        }
    }
    bd_wait();
#undef BD_MARK
    for (int e = tid; e < cpc * n; e += kBdThreads) {
        const int j = e / n, i = e - j * n, gj = c0 + j;
        if (gj < m) a.A[(int64_t)gj * n + i] = As[e];
    }
}

// Register-resident variant (n <= kBdThreads): thread i keeps row i of the
// CTA's CPC columns in registers, so the rank-1 updates and z = A v never
// touch shared memory; the column products w = u^T A are a transpose-reduce
// of CPC values inside each warp (lane L ends with column L) plus a 16-way
// sum over the warps.  Inactive columns (j <= k) carry w_j = v_j = 0 and
// inactive rows u_i = z_i = 0, so every thread runs the same unrolled code.
// The exchange (u_k, partial z) goes through L2 as in bd_kernel.
// mbarrier + st.async: a point-to-point exchange inside the cluster (the
// receiver's mbarrier counts the bytes that landed in its shared memory), in
// place of a cluster barrier whose release has to drain the remote stores
__device__ __forceinline__ unsigned bd_smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bd_mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void bd_mbar_expect(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bd_mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n BD_WAIT_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra BD_WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ unsigned bd_mapa(unsigned addr, int rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void bd_st_async(unsigned raddr, double v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}

// fixed-order pairwise sum of N values (N a power of two): log2(N) dependent
// adds instead of N - 1
template <int N>
__device__ __forceinline__ double bd_tree_sum(double (&v)[N]) {
#pragma unroll
    for (int h = N / 2; h >= 1; h >>= 1)
#pragma unroll
        for (int t = 0; t < h; ++t) v[t] += v[t + h];
    return v[0];
}

template <int CPC>
__device__ __forceinline__ double bd_transpose_reduce(double (&p)[CPC], int lane) {
#pragma unroll
    for (int o = 16; o >= CPC; o >>= 1)
#pragma unroll
        for (int t = 0; t < CPC; ++t) p[t] += __shfl_xor_sync(0xffffffffu, p[t], o);
#pragma unroll
    for (int o = CPC / 2; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int t = 0; t < o; ++t) {
            const double send = up ? p[t] : p[t + o];
            const double keep = up ? p[t + o] : p[t];
            p[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return p[0];  // column lane % CPC
}

// Register-resident kernel's exchanges: point-to-point st.async into the
// receivers' shared memory, each receiver counting the bytes on an mbarrier
// (no cluster barrier, no L2 round trip).  Per step k (right reflector):
//   EN  at the end of reflect(k) every CTA sends its row-k norm partial (and
//       the owner of column k+1 A[k][k+1]) to every CTA;
//   E1  every CTA sends, for each row i > k, its partial
//       T_i = sum_j x_ij rowk_j (and the owner's x_i,k+1) to the row's
//       reducer, CTA i / S (a reduce-scatter over S-row slices);
//   E2  the reducer sums its slice, forms z_i = tauR (scaleR T_i + x_i,k+1)
//       and sends (z_i, x_i,k+1 - z_i) for every row of the slice to every
//       CTA (the all-gather).
// Buffers alternate by step parity; a CTA can only reach step k + 2 of an
// exchange after every CTA has consumed step k (each E1/EN follows the
// previous E2 from every reducer, each E2 the E1 from every CTA).
// Measured and dropped: the exchanges as cp.async.bulk copies of staged
// warp chunks (m = 512: 3.2-3.5 vs 2.74 ms).
__device__ __forceinline__ void bd_st_async2(unsigned raddr, double v0, double v1, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "l"(__double_as_longlong(v0)), "l"(__double_as_longlong(v1)), "r"(rbar)
                 : "memory");
}

// Register tile: thread (warp w, lane rq + 8 cg) keeps rows 32 w + rq + 8 r
// (r < 4) of the CTA's columns cg CC .. cg CC + CC - 1 (CC = CPC / 4).
// Column sums (w = u^T A) add the four rows inside the thread and reduce
// over the 8 row lanes; row sums (T = A rowk) add the CC columns inside the
// thread and reduce over the 4 column lanes, which leaves row 32 w + lane's
// sum in that lane.  13 64-bit shuffles per warp and step at CPC = 32
// instead of 36 with a row per thread — the SM issues one 32-bit shuffle
// per cycle (tools/tput_probe.cu), which bound the row-per-thread layout.
template <int CC>
__device__ __forceinline__ double bd_colsum(double (&p)[CC], int lane) {
#pragma unroll
    for (int o = 4; o >= CC; o >>= 1)
#pragma unroll
        for (int t = 0; t < CC; ++t) p[t] += __shfl_xor_sync(0xffffffffu, p[t], o);
#pragma unroll
    for (int o = CC / 2; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int t = 0; t < o; ++t) {
            const double send = up ? p[t] : p[t + o];
            const double keep = up ? p[t + o] : p[t];
            p[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return p[0];  // column lane & (CC - 1) of the lane's group
}

__device__ __forceinline__ double bd_rowsum4(double (&t)[4], int lane) {
    const bool u4 = (lane & 16) != 0, u3 = (lane & 8) != 0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const double send = u4 ? t[q] : t[q + 2];
        const double keep = u4 ? t[q + 2] : t[q];
        t[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    const double send = u3 ? t[0] : t[1];
    const double keep = u3 ? t[1] : t[0];
    return keep + __shfl_xor_sync(0xffffffffu, send, 8);  // row r = lane >> 3
}

template <int CPC, int C = kBdCluster>
__global__ void __launch_bounds__(kBdThreads, 1) bd_reg_kernel(BdArgs a) {
    cg::cluster_group cl = cg::this_cluster();
    constexpr int W = kBdThreads / 32;
    constexpr int S = kBdThreads / C;  // rows per reduction slice
    constexpr int CC = CPC / 4;        // columns per thread
    __shared__ double wred[W][CPC], sred[W];
    __shared__ double wl[CPC], rowa[CPC], rowk[CPC];
    __shared__ double pnorm[2][C + 1];                // EN: row-norm partials of all CTAs + A[k][k+1]
    // E1: T partials of my slice from every CTA; [.][1] of the owner of
    // column k+1 carries its x_i,k+1 (one 16-byte message)
    __shared__ __align__(16) double rsb[2][C][S][2];
    __shared__ __align__(16) double agb[2][kBdThreads][2];  // E2: (z_i, column k+1 after the update)
    __shared__ double rs[2];
    __shared__ __align__(8) unsigned long long mbar[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rq = lane & 7, cgp = lane >> 3;
    const int rank = (int)cl.block_rank();
    const int n = a.n, m = a.m;
    const int c0 = rank * CPC;
    const int jc0 = cgp * CC;          // my first column (CTA-local)
    const int w0 = 32 * warp;          // my warp's first row
    const int si = tid / S, so = tid % S;  // reducer CTA and slot of row tid (the row whose sums this lane sends)
    int row[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) row[r] = w0 + rq + 8 * r;
    double x[4][CC];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < CC; ++c)
            x[r][c] = (row[r] < n && c0 + jc0 + c < m) ? a.A[(int64_t)(c0 + jc0 + c) * n + row[r]] : 0.0;
#ifdef TTSVD_BD_PROF
    // diagnostics builds (tools/bd_prof.cu): per-phase cycles of one thread
    // per CTA, kept in registers and written once at the end
    long long pacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tp = bj_clock();
#define BD_MARK(q)                           \
    {                                        \
        const long long tq = bj_clock();     \
        pacc[q] += tq - tp;                  \
        tp = tq;                             \
    }
#else
#define BD_MARK(q)
#endif
#ifdef TTSVD_BD_TRACE
    // diagnostics builds: globaltimer of events ev of steps [K0, K0 + 8) for
    // thread TTSVD_BD_TRACE of every CTA: prof[((rank * 8 + ev) * 8 + k - K0]
#ifdef TTSVD_BD_TRACE_WARPS
    // lane 0 of every warp of CTA TTSVD_BD_TRACE_WARPS (indexed by warp)
#define BD_TR(ev, kk)                                                                          \
    if (a.prof && rank == TTSVD_BD_TRACE_WARPS && lane == 0 && (kk) >= TTSVD_BD_K0 && (kk) < TTSVD_BD_K0 + 8) { \
        unsigned long long g_;                                                                 \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_)::"memory");                       \
        a.prof[(warp * 8 + (ev)) * 8 + (kk) - TTSVD_BD_K0] = (long long)g_;                     \
    }
#else
#define BD_TR(ev, kk)                                                                          \
    if (a.prof && tid == TTSVD_BD_TRACE && (kk) >= TTSVD_BD_K0 && (kk) < TTSVD_BD_K0 + 8) {     \
        unsigned long long g_;                                                                 \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_)::"memory");                       \
        a.prof[(rank * 8 + (ev)) * 8 + (kk) - TTSVD_BD_K0] = (long long)g_;                     \
    }
#endif
#else
#define BD_TR(ev, kk)
#endif
    // EN needs one mbarrier per step parity: a CTA with no rows left to
    // reduce is not on the E1 -> E2 path that orders the other exchanges
    const unsigned mbn0 = bd_smem_addr(&mbar[0]), mb1 = bd_smem_addr(&mbar[2]), mb2 = bd_smem_addr(&mbar[3]);
    if (tid == 0) {
        bd_mbar_init(mbn0, 1);
        bd_mbar_init(mbn0 + 8, 1);
        bd_mbar_init(mb1, 1);
        bd_mbar_init(mb2, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const unsigned r_mb1 = bd_mapa(mb1, si);
    const int s_lo = S * rank, s_hi = min(S * rank + S, n);  // my slice
    // Left reflector of column k from its entries ck (every CTA computes it
    // from the same bits) fused with the next products w_j = tau u^T x_j:
    // one reduction of (ck^2, ck x_ij) over the rows below k; u_k = 1 adds
    // row k.  Warps whose rows all lie above k contribute zeros without
    // computing.  Also row k after the left update (rowk = rowa - wl, the
    // right reflector's row) and, when step k has a right reflector, its
    // norm partial to every CTA (EN).  u gets u_i of my rows; the owner keeps
    // u in its column.
    auto reflect = [&](int k, const double (&ck)[4], double (&u)[4]) {
        if (w0 + 31 >= k && w0 < n) {
            double cb[4], ssp = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                cb[r] = (row[r] > k && row[r] < n) ? ck[r] : 0.0;
                ssp = fma(cb[r], cb[r], ssp);
            }
            double p[CC];
#pragma unroll
            for (int c = 0; c < CC; ++c) {
                p[c] = cb[0] * x[0][c];
#pragma unroll
                for (int r = 1; r < 4; ++r) p[c] = fma(cb[r], x[r][c], p[c]);
            }
            const double cs = bd_colsum<CC>(p, lane);
#pragma unroll
            for (int o = 1; o <= 4; o <<= 1) ssp += __shfl_xor_sync(0xffffffffu, ssp, o);
            if (rq < CC) wred[warp][jc0 + rq] = cs;
            if (lane == 0) sred[warp] = ssp;
            if ((k >> 5) == warp && rq == (k & 7)) {  // the four lanes holding row k (predicated stores)
                const int rk = (k >> 3) & 3;
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if (r == rk) {
#pragma unroll
                        for (int c = 0; c < CC; ++c) rowa[jc0 + c] = x[r][c];
                        if (cgp == 0) rs[0] = ck[r];
                    }
            }
        } else {
            if (lane < CPC) wred[warp][lane] = 0.0;
            if (lane == 0) sred[warp] = 0.0;
        }
        BD_MARK(3)
        BD_TR(0, k)
        __syncthreads();
        double sv[W];
#pragma unroll
        for (int q = 0; q < W; ++q) sv[q] = sred[q];
        const double s = bd_tree_sum<W>(sv);
        const double alpha = rs[0];
        double tau = 0.0, beta = alpha, scale = 0.0;
        if (s != 0.0) {
            const double x2 = fma(alpha, alpha, s), inv = fast_rsqrt(x2), nr = x2 * inv;
            beta = alpha >= 0.0 ? -nr : nr;
            tau = 1.0 + fabs(alpha) * inv;  // (beta - alpha) / beta
            scale = fast_rcp(alpha - beta);
        }
        double rk = 0.0, yk = 0.0;  // warp 0: row k after the left update, A[k][k+1]
        if (tid < CPC) {
            double wv[W];
#pragma unroll
            for (int q = 0; q < W; ++q) wv[q] = wred[q][tid];
            const double sj = bd_tree_sum<W>(wv);
            const int gj = c0 + tid;
            const double w = (gj > k && gj < m) ? tau * fma(scale, sj, rowa[tid]) : 0.0;
            wl[tid] = w;
            const double rr = rowa[tid] - w;
            rk = (gj >= k + 2 && gj < m) ? rr : 0.0;
            yk = gj == k + 1 ? rr : 0.0;
            rowk[tid] = rk;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) u[r] = (row[r] > k && row[r] < n) ? ck[r] * scale : (row[r] == k ? 1.0 : 0.0);
        if (rank == 0 && tid == 0) {
            a.d[k] = beta;
            a.tauL[k] = tau;
        }
        BD_MARK(10)
        __syncthreads();  // wl / rowk visible; rs / rowa / wred free
        BD_MARK(11)
        BD_TR(1, k)
        if (warp == 0 && k + 2 < m) {
            // EN: lane t sends the row-norm partial (and A[k][k+1]) to CTA t
            const double sn = bd_warp_sum(rk * rk);
            const double y = bd_warp_sum(yk);
            if (lane < C) {
                double* pn = pnorm[k & 1];
                const unsigned rb = bd_mapa(mbn0 + 8 * (k & 1), lane);
                bd_st_async(bd_mapa(bd_smem_addr(pn + rank), lane), sn, rb);
                if (rank == (k + 1) / CPC) bd_st_async(bd_mapa(bd_smem_addr(pn + C), lane), y, rb);
            }
        }
    };
    // column k of the result takes u on rows >= k: straight to global memory
    // (no later step reads the column; the final store skips it), by the
    // owner while it waits for E2; lane (rq, cg) stores row tid = its row cg
    auto store_u = [&](int k, const double (&u)[4]) {
        if (k / CPC == rank && tid >= k && tid < n)
            a.A[(int64_t)k * n + tid] = cgp == 0 ? u[0] : (cgp == 1 ? u[1] : (cgp == 2 ? u[2] : u[3]));
    };
    // every CTA reads column 0 itself (before the barrier: step 0 stores u_0
    // over it); the barrier publishes the mbarrier inits
    double ui[4], ck[4], xpre[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < 4; ++r) ck[r] = row[r] < n ? a.A[row[r]] : 0.0;
    if (rank == 0 && cgp == 1 / CC) {  // column 1 for step 0
#pragma unroll
        for (int r = 0; r < 4; ++r) xpre[r] = x[r][1 % CC];
    }
    bd_arrive();
    bd_wait();
    if (tid == 0 && 2 < m) bd_mbar_expect(mbn0, (unsigned)(C + 1) * 8);
    reflect(0, ck, ui);
    for (int k = 0; k < m; ++k) {
        BD_MARK(0)
        const int b = k & 1;
        const unsigned par = (unsigned)(k & 1);
        const int on = (k + 1) / CPC;  // owner of column k+1
        const int lk1 = k + 1 - c0;    // its local index (owner)
        const bool live = tid > k && tid < n;  // row tid takes part in step k's right update
        double T = 0.0;
        if (w0 + 31 >= k && w0 < n) {
            // left update (rows >= k) fused with T_i = sum_j x_ij rowk_j
            double T4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int c = 0; c < CC; ++c) {
                const double wc = wl[jc0 + c], rc = rowk[jc0 + c];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    x[r][c] = fma(-wc, ui[r], x[r][c]);
                    T4[r] = fma(x[r][c], rc, T4[r]);
                }
            }
            T = bd_rowsum4(T4, lane);
        }
        if (k + 1 >= m) {
            store_u(k, ui);
            break;
        }
        // the owner's column k+1 on my rows (lanes of its column group): the
        // left update of xpre, picked out of x during the previous step's
        // wait for E2 (a select chain off the critical path)
        const bool hold1 = rank == on && lk1 / CC == cgp;
        double xk1[4];
        {
            const double w1 = wl[hold1 ? lk1 : 0];
#pragma unroll
            for (int r = 0; r < 4; ++r) xk1[r] = hold1 ? fma(-w1, ui[r], xpre[r]) : 0.0;
        }
        BD_MARK(7)
        double zt[4] = {0.0, 0.0, 0.0, 0.0};
        if (k + 2 < m) {
            const int cr = max(0, s_hi - max(s_lo, k + 1));  // my slice's rows in (k, n)
            if (tid == 0) {
                bd_mbar_expect(mb1, (unsigned)(C + 1) * (unsigned)cr * 8);
                bd_mbar_expect(mb2, (unsigned)(n - k - 1) * 16);
                if (k + 3 < m) bd_mbar_expect(mbn0 + 8 * ((k + 1) & 1), (unsigned)(C + 1) * 8);  // EN of step k + 1
            }
            // ---- E1 (reduce-scatter): T_i (and the owner's x_i,k+1) to the row's reducer ----
            if (rank == on) {
                // x_i,k+1 of row tid from the lane of column k+1's group
                // holding it (its row cg of this lane's rq)
                const int src = rq + 8 * (lk1 / CC);
                double v[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) v[r] = __shfl_sync(0xffffffffu, xk1[r], src);
                const double xv = cgp == 0 ? v[0] : (cgp == 1 ? v[1] : (cgp == 2 ? v[2] : v[3]));
                if (live) bd_st_async2(bd_mapa(bd_smem_addr(&rsb[b][rank][so][0]), si), T, xv, r_mb1);
            } else if (live) {
                bd_st_async(bd_mapa(bd_smem_addr(&rsb[b][rank][so][0]), si), T, r_mb1);
            }
            BD_MARK(1)
            BD_TR(2, k)
            // the right reflector from EN (sent at the end of reflect(k))
            bd_mbar_wait(mbn0 + 8 * b, (unsigned)((k >> 1) & 1));
            BD_MARK(8)
            BD_TR(3, k)
            const double* pn = pnorm[b];
            double pv[C];
#pragma unroll
            for (int t = 0; t < C; ++t) pv[t] = pn[t];
            const double st = bd_tree_sum<C>(pv);
            const double y0 = pn[C];
            double tauR = 0.0, gamma = y0, scaleR = 0.0;
            if (st != 0.0) {
                const double x2 = fma(y0, y0, st), inv = fast_rsqrt(x2), nr = x2 * inv;
                gamma = y0 >= 0.0 ? -nr : nr;
                tauR = 1.0 + fabs(y0) * inv;  // (gamma - y0) / gamma
                scaleR = fast_rcp(y0 - gamma);
            }
            if (rank == 0 && tid == 0) a.e[k] = gamma;
            BD_MARK(9)
            // ---- E2 (all-gather): the reducer's rows (z_i, x_i,k+1 - z_i) to every CTA ----
            if (live && si == rank) {
                bd_mbar_wait(mb1, par);
                BD_TR(4, k)
                double q[C];
#pragma unroll
                for (int t = 0; t < C; ++t) q[t] = rsb[b][t][so][0];
                const double xr = rsb[b][(k + 1) / CPC][so][1];
                const double z = tauR * fma(scaleR, bd_tree_sum<C>(q), xr);
                const unsigned la = bd_smem_addr(&agb[b][tid][0]);
#pragma unroll
                for (int t = 0; t < C; ++t) bd_st_async2(bd_mapa(la, t), z, xr - z, bd_mapa(mb2, t));
            }
            BD_MARK(2)
            BD_TR(5, k)
            store_u(k, ui);
            // column k+2 before this step's right update, for step k+1
            const int lk2 = k + 2 - c0;
            const bool hold2 = rank == (k + 2) / CPC && lk2 / CC == cgp;
            if (hold2) {
                const int c2 = lk2 % CC;
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < CC; ++c)
                        if (c == c2) xpre[r] = x[r][c];
            }
            bd_mbar_wait(mb2, par);
            BD_MARK(4)
            BD_TR(6, k)
            if (w0 + 31 > k && w0 < n) {
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if (row[r] > k && row[r] < n) {
                        const double2 v = *reinterpret_cast<const double2*>(&agb[b][row[r]][0]);
                        zt[r] = v.x;
                        ck[r] = v.y;
                    } else {
                        ck[r] = 0.0;
                    }
                // right update of the columns > k+1 (column k+1 takes the next
                // left reflector in reflect(k+1); rowk is zero there)
                double zs[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) zs[r] = zt[r] * scaleR;
#pragma unroll
                for (int c = 0; c < CC; ++c) {
                    const double rc = rowk[jc0 + c];
#pragma unroll
                    for (int r = 0; r < 4; ++r) x[r][c] = fma(-zs[r], rc, x[r][c]);
                }
                if (hold2) {
                    const double rc = rowk[hold2 ? lk2 : 0];
#pragma unroll
                    for (int r = 0; r < 4; ++r) xpre[r] = fma(-zs[r], rc, xpre[r]);
                }
            } else {
#pragma unroll
                for (int r = 0; r < 4; ++r) ck[r] = 0.0;
            }
            BD_MARK(5)
        } else {
            // k = m-2: no right reflector; e_k = A[k][k+1]; column k+1 from its owner to every CTA
            if (tid == 0) bd_mbar_expect(mb2, (unsigned)(n - k - 1) * 16);
            store_u(k, ui);
            if (hold1) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (row[r] == k) a.e[k] = xk1[r];
                    if (row[r] > k && row[r] < n) {
                        const unsigned la = bd_smem_addr(&agb[b][row[r]][0]);
#pragma unroll
                        for (int t = 0; t < C; ++t) bd_st_async2(bd_mapa(la, t), 0.0, xk1[r], bd_mapa(mb2, t));
                    }
                }
            }
            bd_mbar_wait(mb2, par);
#pragma unroll
            for (int r = 0; r < 4; ++r) ck[r] = (row[r] > k && row[r] < n) ? agb[b][row[r]][1] : 0.0;
        }
        reflect(k + 1, ck, ui);
        BD_MARK(6)
    }
#undef BD_MARK
#undef BD_TR
#ifdef TTSVD_BD_PROF
    if (a.prof && tid == TTSVD_BD_PROF_TID)
        for (int q = 0; q < 12; ++q) a.prof[rank * 12 + q] = pacc[q];
#endif
    // rows above the diagonal (the rows >= j of column j hold u_j already)
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < CC; ++c)
            if (row[r] < c0 + jc0 + c && c0 + jc0 + c < m) a.A[(int64_t)(c0 + jc0 + c) * n + row[r]] = x[r][c];
}

// off-diagonal t (0..2m-2) of the Golub-Kahan tridiagonal: d0 e0 d1 e1 ... d_{m-1}
__device__ __forceinline__ double bd_tgk(const double* d, const double* e, int t) {
    return (t & 1) ? e[t >> 1] : d[t >> 1];
}

constexpr int kBisThreads = 256;

// Sturm count: eigenvalues of T (zero diagonal, squared off-diagonals b2,
// 2m x 2m) below s
__device__ __forceinline__ int bd_sturm(const double* b2, int N, double s, double pivmin) {
    double q = -s;
    if (fabs(q) < pivmin) q = -pivmin;
    int c = q < 0.0;
    for (int t = 1; t < N; ++t) {
        q = -s - b2[t - 1] * fast_rcp(q);
        if (fabs(q) < pivmin) q = -pivmin;
        c += q < 0.0;
    }
    return c;
}

// warp per sigma (descending index); every CTA stages T's squared
// off-diagonals and the Gershgorin bound
__global__ void __launch_bounds__(kBisThreads) bd_bisect_kernel(const double* d, const double* e, int m, double* sigma) {
    extern __shared__ double b2[];  // 2m - 1
    __shared__ double red[kBisThreads / 32][2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = 2 * m;
    double bmax = 0.0, b2max = 0.0;
    for (int t = tid; t < N - 1; t += kBisThreads) {
        const double b = bd_tgk(d, e, t);
        b2[t] = b * b;
        const double g = fabs(b) + (t > 0 ? fabs(bd_tgk(d, e, t - 1)) : 0.0);
        const double g2 = fabs(b) + (t + 1 < N - 1 ? fabs(bd_tgk(d, e, t + 1)) : 0.0);
        bmax = fmax(bmax, fmax(g, g2));
        b2max = fmax(b2max, b * b);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        bmax = fmax(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
        b2max = fmax(b2max, __shfl_xor_sync(0xffffffffu, b2max, o));
    }
    if (lane == 0) {
        red[warp][0] = bmax;
        red[warp][1] = b2max;
    }
    __syncthreads();
    bmax = 0.0;
    b2max = 0.0;
    for (int w = 0; w < kBisThreads / 32; ++w) {
        bmax = fmax(bmax, red[w][0]);
        b2max = fmax(b2max, red[w][1]);
    }
    const int i = blockIdx.x * (kBisThreads / 32) + warp;
    if (i >= m) return;
    if (N == 2) {  // 1 x 1: sigma = |d0|
        if (lane == 0) sigma[0] = fabs(d[0]);
        return;
    }
    const double pivmin = DBL_MIN * fmax(1.0, b2max);
    const int j = m - 1 - i;  // ascending index
    double lo = 0.0, hi = bmax * (1.0 + 4.0 * DBL_EPSILON) + pivmin;
    const double floor_tol = 1e-18 * hi;
    // 16-way multisection; each shift's inertia from a twisted factorisation
    // split in the middle (Sylvester): the even lane of a pair runs the
    // forward recurrence over the first half, the odd lane the backward one
    // over the second half, so a count costs N/2 dependent steps instead of N.
    // #{eigenvalues < s} = #{d+_t < 0, t < h} + #{d-_t < 0, t > h} + [gamma_h < 0],
    // gamma_h = d+_h + d-_h - (T_hh - s) (T_hh = 0 on the Golub-Kahan form).
    const int h = N / 2;
    const int pi = lane >> 1;
    const bool fwd = (lane & 1) == 0;
    for (int it = 0; it < 60; ++it) {
        if (hi - lo <= fmax(2.0 * DBL_EPSILON * hi, floor_tol)) break;
        const double sft = lo + (hi - lo) * (double)(pi + 1) * (1.0 / 17.0);
        double q = -sft;
        if (fabs(q) < pivmin) q = -pivmin;
        int c = 0;
        // one instruction stream for both lanes (no divergence): step u uses
        // b2[u-1] forward (d+_u from d+_{u-1}) and b2[N-1-u] backward (d-_{N-1-u}
        // from d-_{N-u}); the backward half is one step shorter
        for (int u = 1; u < h; ++u) {
            c += q < 0.0;
            q = -sft - b2[fwd ? u - 1 : N - 1 - u] * fast_rcp(q);
            if (fabs(q) < pivmin) q = -pivmin;
        }
        if (fwd) {
            c += q < 0.0;
            q = -sft - b2[h - 1] * fast_rcp(q);
            if (fabs(q) < pivmin) q = -pivmin;
        }
        const double qo = __shfl_xor_sync(0xffffffffu, q, 1);
        const int co = __shfl_xor_sync(0xffffffffu, c, 1);
        double gam = q + qo + sft;
        if (fabs(gam) < pivmin) gam = -pivmin;
        const int cnt = c + co + (gam < 0.0) - m;
        const unsigned above = __ballot_sync(0xffffffffu, cnt > j) & 0x55555555u;  // one lane per shift
        const int f2 = above ? (__ffs(above) - 1) >> 1 : 16;  // first shift index with count > j
        const double s_f = __shfl_sync(0xffffffffu, sft, 2 * min(f2, 15));
        const double s_b = __shfl_sync(0xffffffffu, sft, 2 * max(f2 - 1, 0));
        if (f2 < 16) {
            hi = s_f;
            if (f2 > 0) lo = s_b;
        } else {
            lo = s_f;
        }
    }
    if (lane == 0) sigma[i] = 0.5 * (lo + hi);
}

// inverse iteration on T - sigma I for the leading r sigmas; thread per
// cluster leader.  Scratch per thread: 5 * 2m doubles + 2m ints (global).
// sigmas closer than kBdOrtol ||T|| are a cluster (bd_vectors_kernel)
constexpr double kBdOrtol = 1e-6;

struct BdVecArgs {
    const double* d;
    const double* e;
    const double* sigma;
    int m, r;
    double* scratch;  // r * 7 * 2m doubles
    double* X;        // m x r (ld m): left singular vectors of B
};

__device__ void bd_solve(const double* dl, const double* dg, const double* du, const double* du2, const int* ip, int N,
                         double* z) {
    // L: forward with row interchanges (dgttrs)
    for (int t = 0; t < N - 1; ++t) {
        if (ip[t]) {
            const double tmp = z[t];
            z[t] = z[t + 1];
            z[t + 1] = tmp - dl[t] * z[t];
        } else {
            z[t + 1] -= dl[t] * z[t];
        }
    }
    // U: backward (diagonal dg, super du, second super du2)
    z[N - 1] /= dg[N - 1];
    if (N > 1) z[N - 2] = (z[N - 2] - du[N - 2] * z[N - 1]) / dg[N - 2];
    for (int t = N - 3; t >= 0; --t) z[t] = (z[t] - du[t] * z[t + 1] - du2[t] * z[t + 2]) / dg[t];
}

// One CTA, a thread per leading sigma.  Members of a cluster (sigmas within
// kBdOrtol ||T|| of a neighbour) factor T - sigma I and run the inverse
// iteration solves in parallel, a thread each; between the solves a warp per
// cluster orthonormalises its members in index order (modified Gram-Schmidt,
// lanes over the 2m entries).  (A thread per cluster — members in sequence —
// took 5 ms on the 32-fold sigma = 1 cluster of thick-bounds' recovery step,
// whose work matrix has orthonormal rows by construction.)
__global__ void __launch_bounds__(1024) bd_vectors_kernel(BdVecArgs a) {
    const int i = threadIdx.x;
    const int lane = i & 31, warp = i >> 5, nwarps = blockDim.x >> 5;
    const int m = a.m, r = a.r, N = 2 * m;
    // Gershgorin bound of T (scale of the cluster tolerance and pivot floor)
    double tn = 0.0;
    for (int t = 0; t < N - 1; ++t) tn = fmax(tn, fabs(bd_tgk(a.d, a.e, t)) + (t > 0 ? fabs(bd_tgk(a.d, a.e, t - 1)) : 0.0));
    tn = fmax(tn, N > 1 ? fabs(bd_tgk(a.d, a.e, N - 2)) : 0.0);
    const double ortol = kBdOrtol * tn;
    const double tiny = DBL_EPSILON * tn + DBL_MIN;
    const bool member = i < r && ((i > 0 && a.sigma[i - 1] - a.sigma[i] <= ortol) ||
                                  (i + 1 < r && a.sigma[i] - a.sigma[i + 1] <= ortol));
    if (!__syncthreads_or(member)) return;  // no cluster: bd_twisted_kernel's vectors stand
    double* base = a.scratch + (size_t)(i < r ? i : 0) * 7 * N;
    double* dl = base;
    double* dg = dl + N;
    double* du = dg + N;
    double* du2 = du + N;
    double* z = base + 4 * N;  // member i's eigenvector of T
    int* ip = reinterpret_cast<int*>(du2 + 2 * N);
    if (member) {
        const double s = a.sigma[i];
        // factor T - s I (dgttrf: partial pivoting)
        for (int t = 0; t < N; ++t) dg[t] = -s;
        for (int t = 0; t < N - 1; ++t) {
            du[t] = bd_tgk(a.d, a.e, t);
            dl[t] = du[t];
        }
        for (int t = 0; t < N - 2; ++t) du2[t] = 0.0;
        for (int t = 0; t < N - 1; ++t) {
            if (fabs(dg[t]) >= fabs(dl[t])) {
                ip[t] = 0;
                if (dg[t] == 0.0) dg[t] = tiny;
                const double f = dl[t] / dg[t];
                dl[t] = f;
                dg[t + 1] -= f * du[t];
            } else {
                ip[t] = 1;
                const double f = dg[t] / dl[t];
                dg[t] = dl[t];
                dl[t] = f;
                const double tmp = du[t];
                du[t] = dg[t + 1];
                dg[t + 1] = tmp - f * dg[t + 1];
                if (t < N - 2) {
                    du2[t] = du[t + 1];
                    du[t + 1] = -f * du[t + 1];
                }
            }
        }
        if (dg[N - 1] == 0.0) dg[N - 1] = tiny;
        for (int t = 0; t < N - 1; ++t)
            if (dg[t] == 0.0) dg[t] = tiny;
        // start: a fixed pseudo-random vector
        unsigned h = 0x9e3779b9u * (unsigned)(i + 1);
        for (int t = 0; t < N; ++t) {
            h ^= h << 13;
            h ^= h >> 17;
            h ^= h << 5;
            z[t] = 0.5 + (double)(h & 0xffffu) * (1.0 / 65536.0);
        }
    }
    for (int it = 0; it < 3; ++it) {
        if (member) bd_solve(dl, dg, du, du2, ip, N, z);
        __syncthreads();
        // warp w orthonormalises the clusters whose leader index is w, w + nwarps, ...
        for (int ld = warp; ld < r; ld += nwarps) {
            if (ld > 0 && a.sigma[ld - 1] - a.sigma[ld] <= ortol) continue;  // not a leader
            int last = ld;
            while (last + 1 < r && a.sigma[last] - a.sigma[last + 1] <= ortol) ++last;
            if (last == ld) continue;  // isolated
            for (int v = ld; v <= last; ++v) {
                double* zv = a.scratch + (size_t)v * 7 * N + 4 * N;
                for (int w = ld; w < v; ++w) {
                    const double* zw = a.scratch + (size_t)w * 7 * N + 4 * N;
                    double dt = 0.0;
                    for (int t = lane; t < N; t += 32) dt = fma(zw[t], zv[t], dt);
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) dt += __shfl_xor_sync(0xffffffffu, dt, o);
                    for (int t = lane; t < N; t += 32) zv[t] = fma(-dt, zw[t], zv[t]);
                }
                double nr = 0.0;
                for (int t = lane; t < N; t += 32) nr = fma(zv[t], zv[t], nr);
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) nr += __shfl_xor_sync(0xffffffffu, nr, o);
                const double inv = 1.0 / sqrt(nr);
                for (int t = lane; t < N; t += 32) zv[t] *= inv;
                __syncwarp();
            }
        }
        __syncthreads();
    }
    if (member) {
        // x entries (odd positions), normalised
        double nx = 0.0;
        for (int k = 0; k < m; ++k) nx = fma(z[2 * k + 1], z[2 * k + 1], nx);
        const double ix = nx > 0.0 ? 1.0 / sqrt(nx) : 0.0;
        for (int k = 0; k < m; ++k) a.X[(size_t)i * m + k] = z[2 * k + 1] * ix;
    }
}

// Fast path of the vectors: one twisted factorisation per sigma (warp per
// vector; lanes 0 / 1 run the top-down LDL^T and bottom-up UDU^T of T - sI
// concurrently, the twist index minimises |gamma_k|, and the eigenvector
// follows from z_k = 1 by products only) — one inverse-iteration step from
// the optimal start vector e_k.  Vectors whose sigma lies within kBdOrtol
// ||T|| of a neighbour are redone by bd_vectors_kernel (clusters).
constexpr int kTwWarps = 4;

__global__ void __launch_bounds__(kTwWarps * 32) bd_twisted_kernel(BdVecArgs a) {
    extern __shared__ double tw[];  // per warp: D+ (N), D- (N)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int v = blockIdx.x * kTwWarps + warp;
    const int m = a.m, N = 2 * m;
    if (v >= a.r) return;
    double* dp = tw + (size_t)warp * 2 * N;
    double* dm = dp + N;
    double tn = 0.0, b2max = 0.0;
    for (int t = lane; t < N - 1; t += 32) {
        const double b = fabs(bd_tgk(a.d, a.e, t));
        tn = fmax(tn, b + (t > 0 ? fabs(bd_tgk(a.d, a.e, t - 1)) : 0.0));
        tn = fmax(tn, b + (t + 1 < N - 1 ? fabs(bd_tgk(a.d, a.e, t + 1)) : 0.0));
        b2max = fmax(b2max, b * b);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        tn = fmax(tn, __shfl_xor_sync(0xffffffffu, tn, o));
        b2max = fmax(b2max, __shfl_xor_sync(0xffffffffu, b2max, o));
    }
    const double s = a.sigma[v];
    const double pivmin = DBL_MIN * fmax(1.0, b2max);
    // T - sI = L D+ L^T (top-down, lane 0) = U D- U^T (bottom-up, lane 1)
    if (lane == 0) {
        double q = -s;
        if (fabs(q) < pivmin) q = -pivmin;
        dp[0] = q;
        for (int t = 1; t < N; ++t) {
            const double b = bd_tgk(a.d, a.e, t - 1);
            q = -s - b * b * fast_rcp(q);
            if (fabs(q) < pivmin) q = -pivmin;
            dp[t] = q;
        }
    } else if (lane == 1) {
        double q = -s;
        if (fabs(q) < pivmin) q = -pivmin;
        dm[N - 1] = q;
        for (int t = N - 2; t >= 0; --t) {
            const double b = bd_tgk(a.d, a.e, t);
            q = -s - b * b * fast_rcp(q);
            if (fabs(q) < pivmin) q = -pivmin;
            dm[t] = q;
        }
    }
    __syncwarp();
    // twist: gamma_k = D+_k + D-_k - (T - sI)_kk = D+_k + D-_k + s
    double best = DBL_MAX;
    int kb = 0;
    for (int t = lane; t < N; t += 32) {
        const double g = fabs(dp[t] + dm[t] + s);
        if (g < best) {
            best = g;
            kb = t;
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ok = __shfl_xor_sync(0xffffffffu, kb, o);
        if (ob < best || (ob == best && ok < kb)) {
            best = ob;
            kb = ok;
        }
    }
    // z_k = 1; upward z_t = -(b_t / D+_t) z_{t+1} (lane 0), downward
    // z_{t+1} = -(b_t / D-_{t+1}) z_t (lane 1); z overwrites dp / dm
    if (lane == 0) {
        double z = 1.0;
        for (int t = kb - 1; t >= 0; --t) {
            z = -bd_tgk(a.d, a.e, t) * fast_rcp(dp[t]) * z;
            dp[t] = z;
        }
    } else if (lane == 1) {
        double z = 1.0;
        for (int t = kb; t < N - 1; ++t) {
            z = -bd_tgk(a.d, a.e, t) * fast_rcp(dm[t + 1]) * z;
            dm[t + 1] = z;
        }
    }
    __syncwarp();
    // x entries: odd positions (z_t from dp for t < kb, 1 at kb, dm for t > kb)
    double nx = 0.0;
    for (int k = lane; k < m; k += 32) {
        const int t = 2 * k + 1;
        const double z = t < kb ? dp[t] : (t == kb ? 1.0 : dm[t]);
        nx = fma(z, z, nx);
    }
    nx = bd_warp_sum(nx);
    const double ix = nx > 0.0 ? 1.0 / sqrt(nx) : 0.0;
    for (int k = lane; k < m; k += 32) {
        const int t = 2 * k + 1;
        const double z = t < kb ? dp[t] : (t == kb ? 1.0 : dm[t]);
        a.X[(size_t)v * m + k] = z * ix;
    }
}

// V = U_B [X; 0] for n <= 32 NPL: a warp applies the reflectors to 4
// vectors at once (lane: rows lane + 32 q), the next reflector's entries are
// loaded while the current one is applied
constexpr int kBack4Warps = 4;

template <int NPL>
__global__ void __launch_bounds__(kBack4Warps * 32) bd_back4_kernel(const double* A, const double* tauL, int n, int m,
                                                                    const double* X, int r, double* V) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int v0 = (blockIdx.x * kBack4Warps + warp) * 4;
    if (v0 >= r) return;
    double x[4][NPL];
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int row = lane + 32 * q;
            x[v][q] = (v0 + v < r && row < m) ? X[(size_t)(v0 + v) * m + row] : 0.0;
        }
    double un[NPL];
    auto load = [&](int k) {
        const double* u = A + (size_t)k * n;
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int row = lane + 32 * q;
            un[q] = (row > k && row < n) ? __ldg(u + row) : (row == k ? 1.0 : 0.0);
        }
    };
    load(m - 1);
    for (int k = m - 1; k >= 0; --k) {
        double u[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) u[q] = un[q];
        if (k > 0) load(k - 1);
        const double tau = tauL[k];
        double d[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < NPL; ++q)
#pragma unroll
            for (int v = 0; v < 4; ++v) d[v] = fma(u[q], x[v][q], d[v]);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
            for (int v = 0; v < 4; ++v) d[v] += __shfl_xor_sync(0xffffffffu, d[v], o);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const double w = tau * d[v];
#pragma unroll
            for (int q = 0; q < NPL; ++q) x[v][q] = fma(-w, u[q], x[v][q]);
        }
    }
#pragma unroll
    for (int v = 0; v < 4; ++v)
        if (v0 + v < r)
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int row = lane + 32 * q;
                if (row < n) V[(size_t)(v0 + v) * n + row] = x[v][q];
            }
}

// bd_back4_kernel with the reflectors staged in shared memory: chunks of
// kB4sChunk columns of A are copied by cp.async (double buffered, all threads)
// while the previous chunk is applied, so a reflector costs its arithmetic
// and reductions instead of an L2 round trip (the register prefetch of
// bd_back4_kernel looks one reflector ahead, less than the L2 latency).
constexpr int kB4sChunk = 16;
constexpr int kB4sWarps = 4;  // warps per CTA: 8 CTAs for r = 32 (m = 512 SVD 2.21 -> 2.12 ms; 16 warps: 2 CTAs, 2 warps: 2.14)
constexpr int kB4sVpw = 1;    // vectors per warp

__device__ __forceinline__ void bd_cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned sd = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sd), "l"(gsrc) : "memory");
}

inline size_t bd_back4s_smem(int npl) { return (size_t)2 * kB4sChunk * 32 * npl * sizeof(double); }

template <int NPL>
__global__ void __launch_bounds__(kB4sWarps * 32) bd_back4s_kernel(const double* A, const double* tauL, int n, int m,
                                                                     const double* X, int r, double* V) {
    extern __shared__ __align__(16) double us[];  // 2 x kB4sChunk x (32 NPL): raw columns k of A
    __shared__ double taus[2 * kB4sChunk];
    constexpr int LD = 32 * NPL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int v0 = (blockIdx.x * kB4sWarps + warp) * kB4sVpw;
    const int nchunks = (m + kB4sChunk - 1) / kB4sChunk;
    // chunk c: reflectors k = m-1-c*CH down to max(0, m-CH-c*CH)
    auto stage = [&](int c) {
        double* dst = us + (c & 1) * kB4sChunk * LD;
        const int khi = m - 1 - c * kB4sChunk;
        const int cnt = min(kB4sChunk, khi + 1);
        if (tid < cnt) taus[(c & 1) * kB4sChunk + tid] = tauL[khi - tid];
        // warp per column, lane per 16-byte pair (no index division)
        for (int kk = warp; kk < cnt; kk += kB4sWarps) {
            const double* src = A + (size_t)(khi - kk) * n;
            double* d = dst + kk * LD;
            if ((n & 1) == 0) {
                for (int p2 = 2 * lane; p2 < n; p2 += 64) bd_cp_async16(d + p2, src + p2);
            } else {  // odd n: columns are not 16-byte aligned
                for (int i = lane; i < n; i += 32) d[i] = src[i];
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double x[kB4sVpw][NPL];
#pragma unroll
    for (int v = 0; v < kB4sVpw; ++v)
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int row = lane + 32 * q;
            x[v][q] = (v0 + v < r && row < m) ? X[(size_t)(v0 + v) * m + row] : 0.0;
        }
    stage(0);
    for (int c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) {
            stage(c + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double* ub = us + (c & 1) * kB4sChunk * LD;
        const int khi = m - 1 - c * kB4sChunk;
        const int cnt = min(kB4sChunk, khi + 1);
        for (int kk = 0; kk < cnt; ++kk) {
            const int k = khi - kk;
            double u[NPL];
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int row = lane + 32 * q;
                u[q] = (row > k && row < n) ? ub[kk * LD + row] : (row == k ? 1.0 : 0.0);
            }
            const double tau = taus[(c & 1) * kB4sChunk + kk];
            double d[kB4sVpw][2];
#pragma unroll
            for (int v = 0; v < kB4sVpw; ++v) d[v][0] = d[v][1] = 0.0;
#pragma unroll
            for (int q = 0; q < NPL; ++q)
#pragma unroll
                for (int v = 0; v < kB4sVpw; ++v) d[v][q & 1] = fma(u[q], x[v][q], d[v][q & 1]);
            double dd[kB4sVpw];
#pragma unroll
            for (int v = 0; v < kB4sVpw; ++v) dd[v] = d[v][0] + d[v][1];
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
                for (int v = 0; v < kB4sVpw; ++v) dd[v] += __shfl_xor_sync(0xffffffffu, dd[v], o);
#pragma unroll
            for (int v = 0; v < kB4sVpw; ++v) {
                const double w = tau * dd[v];
#pragma unroll
                for (int q = 0; q < NPL; ++q) x[v][q] = fma(-w, u[q], x[v][q]);
            }
        }
        __syncthreads();  // the buffer is restaged two chunks later
    }
    if (v0 >= r) return;
#pragma unroll
    for (int v = 0; v < kB4sVpw; ++v)
        if (v0 + v < r)
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int row = lane + 32 * q;
                if (row < n) V[(size_t)(v0 + v) * n + row] = x[v][q];
            }
}

// V (n x r, ld n) = U_B [X; 0]: the left reflectors of bd_kernel applied in
// reverse; warp per vector
constexpr int kBackWarps = 4;

__global__ void __launch_bounds__(kBackWarps * 32) bd_back_kernel(const double* A, const double* tauL, int n, int m,
                                                                  const double* X, int r, double* V) {
    extern __shared__ double xs[];  // kBackWarps x n
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int v = blockIdx.x * kBackWarps + warp;
    if (v >= r) return;
    double* x = xs + (size_t)warp * n;
    for (int i = lane; i < n; i += 32) x[i] = i < m ? X[(size_t)v * m + i] : 0.0;
    __syncwarp();
    for (int k = m - 1; k >= 0; --k) {
        const double tau = tauL[k];
        if (tau == 0.0) continue;
        const double* u = A + (size_t)k * n;
        double dot = 0.0;
        for (int i = k + 1 + lane; i < n; i += 32) dot = fma(u[i], x[i], dot);
        dot = bd_warp_sum(dot) + x[k];
        const double w = tau * dot;
        __syncwarp();
        if (lane == 0) x[k] -= w;
        for (int i = k + 1 + lane; i < n; i += 32) x[i] = fma(-w, u[i], x[i]);
        __syncwarp();
    }
    for (int i = lane; i < n; i += 32) V[(size_t)v * n + i] = x[i];
}

}  // namespace ttsvd_b200
