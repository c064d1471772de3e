// sm_100a kernels of the TT-SVD hot path (arXiv 2102.00104, Alg. 2/5/6).
//
//   K_TSQR   tsqr_tile_kernel      Q-less structured Householder over row tiles,
//                                  per-CTA flat tree (tsqr.hpp:247-292) and the
//                                  index-ordered merge tree (tsqr.hpp:230-240)
//   K_SVD    jacobi_kernel         one-sided Jacobi (small_svd.hpp:72-114) in a
//                                  parallel round-robin order; single CTA with
//                                  the matrix in shared memory, or a cooperative
//                                  grid with the matrix in L2
//            jacobi_finalize       norms, stable descending sort, normalisation
//                                  and the deterministic completion
//                                  (small_svd.hpp:133-191)
//   K_TSMM   tsmm_kernel           Y = reshape(X V) written straight into the
//                                  next step's padded layout (tsmm.hpp:20-71)
//
// All arithmetic is fp64.  Everything here is deterministic for a fixed launch
// shape: no floating-point atomics, fixed reduction trees.
#pragma once

#include <cooperative_groups.h>
#include <cstdint>
#include <cfloat>

namespace ttsvd_b200 {

namespace cg = cooperative_groups;

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// D += A B on the FP64 tensor cores (mma.sync m8n8k4 f64).  Fragments: lane l
// holds A[l/4][l%4], B[l%4][l/4] and C/D[l/4][2(l%4) + e].
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// A work matrix whose columns are not uniformly strided: column c starts at
// (c / q) ld + (c mod q) ld_lo (q = 0: the plain c ld).  Thick-bounds' merged
// matricization (n_1 .. n_{d-k}) x (n_{d-k+1} .. n_d) is such a view of the
// caller's padded X (q = m / n_d, ld_lo = its row count), so K_TSQR and K_TSMM
// read it in place instead of through copy_logical's copy (tt_svd.hpp:347-348,
// storage.hpp:158-172).
struct ColSplit {
    int q;
    int64_t ld_lo;
};
__host__ __device__ __forceinline__ int64_t col_off(int c, int64_t ld, ColSplit cs) {
    return cs.q ? (int64_t)(c / cs.q) * ld + (int64_t)(c % cs.q) * cs.ld_lo : (int64_t)c * ld;
}

// 1/sqrt(x) and 1/x for reflector / rotation scalars without the libdevice slow-path
// calls (a call site inside the unrolled reflector loop pins every live value
// across it): the SFU seed (measured max relative error 2^-20,
// tools/approx_probe.cu) and one cubic Newton step (error ~2^-60, below the
// final rounding).
// x > 0; zero and the all-zero rules are handled by the caller.
__device__ __forceinline__ double fast_rsqrt(double x) {
    // subnormal squared norms (entries ~1e-155) would flush to zero in the
    // seed: scale by an exact power of two instead
    const bool tiny = x < 0x1p-1000;
    const double xs = tiny ? x * 0x1p1000 : x;
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(xs));
    const double e = fma(-xs, y * y, 1.0);
    y = fma(fma(0.375, e, 0.5), e * y, y);
    return tiny ? y * 0x1p500 : y;
}

__device__ __forceinline__ double fast_rcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x, y, 1.0);
    return fma(fma(e, e, e), y, y);
}

__device__ __forceinline__ double ldg_stream(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// L2 eviction-priority hints: the streamed input is evict-first so that the
// per-CTA R factors (re-read for every tile) stay L2 resident.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_stream_hint(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
    return v;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// ---------------------------------------------------------------------------
// Synthetic input: counter-based uniform[-1,1) (restated in oracle/ttsvd_oracle.c
// orc_gen_uniform; both steps are exact in fp64 so host and device agree).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void gen_uniform_kernel(uint64_t seed, int64_t total, int64_t rows, int64_t ld, double* X) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < total; l += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t z = splitmix64(seed + (uint64_t)(l + 1) * 0x9E3779B97F4A7C15ULL);
        const double u = (double)(z >> 11) * 0x1.0p-53;
        const int64_t j = l / rows;
        X[j * ld + (l - j * rows)] = 2.0 * u - 1.0;
    }
}

// partition `part` of `nparts`: local flat l is global part + nparts*l.
// kind 0: uniform[-1,1) (as gen_uniform); kind 1: += scale * N(0,1) from
// Box-Muller on two counter draws of the global index
__global__ void gen_partition_kernel(uint64_t seed, int kind, double scale, int64_t total, int64_t rows, int64_t ld,
                                     int64_t nparts, int64_t part, double* X) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < total; l += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t g = (uint64_t)(part + nparts * l);
        const int64_t j = l / rows;
        double* x = X + j * ld + (l - j * rows);
        if (kind == 0) {
            const uint64_t z = splitmix64(seed + (g + 1) * 0x9E3779B97F4A7C15ULL);
            *x = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
        } else {
            const uint64_t z1 = splitmix64(seed + (2 * g + 1) * 0x9E3779B97F4A7C15ULL);
            const uint64_t z2 = splitmix64(seed + (2 * g + 2) * 0x9E3779B97F4A7C15ULL);
            const double u1 = ((double)(z1 >> 11) + 0.5) * 0x1.0p-53, u2 = (double)(z2 >> 11) * 0x1.0p-53;
            *x += scale * sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
        }
    }
}

// ---------------------------------------------------------------------------
// K_TSQR — structured Householder reduction of [R; B] over row tiles.
//
// One CTA owns a job: a contiguous row range of a column-major matrix and a
// running m x m upper-triangular R.  Each tile of `bt` rows is staged in shared
// memory and folded into R column by column.  Reflector j spans R(j,j) and
// the tile's column j (R's rows above j are final, rows below are zero), the
// reference's eps_fp trick (tsqr.hpp:120-142) keeps it branch-free:
//     t = eps + ||u||^2, alpha = -sign(u0) sqrt(t + eps), t -= alpha u0,
//     beta = 1/sqrt(t), v = beta (u - alpha e1), ||v||^2 = 2;
// a zero block column under a nonzero pivot leaves R's row untouched (H = I).
// The trailing columns are updated by warps (one column per warp at a time,
// lanes over rows, shuffle reduction).  Two modes:
//   mode 0 (sweep):  job g = rows [g*n/G, (g+1)*n/G) of X, R starts at 0;
//   mode 1 (merge):  job i stacks part 2i+1 (m x m, ld m) under part 2i —
//                    one level of the fixed index-ordered merge tree.
// ---------------------------------------------------------------------------
struct TsqrArgs {
    const double* X;   // mode 0: matrix; mode 1: parts base (count * m*m)
    int64_t n;         // mode 0: rows; mode 1: number of parts at this level
    int64_t ld;        // mode 0: leading dimension
    double* R_out;     // job outputs, m*m each (ld m)
    int m;
    int bt;            // tile rows
    int ldb;           // tile leading dimension in shared memory
    int mode;
    int r_in_smem;
    const double* R_init0;  // mode 0 only, grid 1: start from this R (reduce_block)
};

template <int NT>
__global__ void __launch_bounds__(NT) tsqr_tile_kernel(TsqrArgs a) {
    extern __shared__ __align__(16) double smem[];
    constexpr int NW = NT / kWarp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = a.m;
    const int64_t job = blockIdx.x;

    const double* X;
    int64_t row0, row1, ld;
    const double* R_init = nullptr;
    double* R_out = a.R_out + job * (int64_t)m * m;
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
        R_init = a.X + (2 * job) * (int64_t)m * m;
        if (2 * job + 1 < count) {
            X = a.X + (2 * job + 1) * (int64_t)m * m;
            row0 = 0;
            row1 = m;
        } else {
            X = nullptr;
            row0 = row1 = 0;
        }
        ld = m;
    }

    double* R = a.r_in_smem ? smem : R_out;
    double* B = smem + (a.r_in_smem ? m * m : 0);
    double* red = B + (int64_t)a.ldb * m;  // NW + 4 doubles

    for (int e = tid; e < m * m; e += NT) R[e] = R_init ? R_init[e] : 0.0;
    __syncthreads();

    const double eps = DBL_MIN;
    for (int64_t r0 = row0; r0 < row1; r0 += a.bt) {
        const int rows = (int)((row1 - r0) < (int64_t)a.bt ? (row1 - r0) : (int64_t)a.bt);
        for (int j = 0; j < m; ++j) {
            const double* src = X + j * ld + r0;
            double* dst = B + j * a.ldb;
            for (int i = tid; i < rows; i += NT) dst[i] = src[i];
        }
        __syncthreads();
        for (int j = 0; j < m; ++j) {
            const double* bj = B + j * a.ldb;
            double s = 0.0;
            for (int i = tid; i < rows; i += NT) s += bj[i] * bj[i];
            s = warp_sum(s);
            if (lane == 0) red[warp] = s;
            __syncthreads();
            if (tid == 0) {
                double tot = 0.0;
                for (int w = 0; w < NW; ++w) tot += red[w];
                const double u0 = R[j * m + j];
                if (tot == 0.0 && u0 != 0.0) {
                    // nothing below a nonzero pivot: H = I (LAPACK dlarfg
                    // convention), R(j,:) stays bitwise as it is.  An all-zero
                    // u still takes the eps_fp path below, which yields the
                    // reference's alpha = sqrt(2 DBL_MIN) (tsqr.hpp:120-126).
                    red[NW + 0] = u0;
                    red[NW + 1] = 0.0;
                    red[NW + 2] = 0.0;
                } else {
                    double t = eps + (u0 * u0 + tot);
                    double alpha = sqrt(t + eps);
                    alpha = (u0 > 0.0) ? -alpha : alpha;
                    t -= alpha * u0;
                    const double beta = 1.0 / sqrt(t);
                    red[NW + 0] = alpha;
                    red[NW + 1] = beta;
                    red[NW + 2] = (u0 - alpha) * beta;
                }
            }
            __syncthreads();
            const double alpha = red[NW + 0], beta = red[NW + 1], v0 = red[NW + 2];
            for (int k = j + 1 + warp; k < m; k += NW) {
                double* bk = B + k * a.ldb;
                double p = 0.0;
                for (int i = lane; i < rows; i += kWarp) p += bj[i] * bk[i];
                p = warp_sum(p);
                const double rjk = R[k * m + j];
                const double g = v0 * rjk + beta * p;
                const double gb = g * beta;
                for (int i = lane; i < rows; i += kWarp) bk[i] -= gb * bj[i];
                if (lane == 0) R[k * m + j] = rjk - g * v0;
            }
            __syncthreads();
            if (tid == 0) R[j * m + j] = alpha;
        }
        __syncthreads();
    }
    if (a.r_in_smem) {
        for (int e = tid; e < m * m; e += NT) R_out[e] = R[e];
    }
}

// ---------------------------------------------------------------------------
// K_SVD — one-sided Jacobi on the columns of A (n x m, ld n).
//
// Pairs follow the circle method: in round r (0 <= r < mp-1, mp = m rounded
// up to even) pair i is (r, mp-1) for i = 0 and ((r+i) mod (mp-1),
// (r-i) mod (mp-1)) otherwise; every unordered pair meets once per sweep, and
// the mp/2 pairs of a round are independent.  The rotation and the skip rule
// are the reference's (small_svd.hpp:84-108): skip if |gamma| <= 1e2 eps
// sqrt(alpha beta); converged after a sweep without rotations; at most 30
// sweeps.  With `acc` the rotations are also applied to Vacc (m x m) — that
// gives jacobi_svd()'s V.  Without it the orthogonalised columns themselves
// are the wanted singular vectors (the driver runs this on R^T or W^T).
// ---------------------------------------------------------------------------
struct JacobiArgs {
    double* A;     // n x m, ld n (global)
    double* Vacc;  // m x m or nullptr
    int n, m;
    int* sweep_flags;  // >= max_sweeps ints, zeroed (cooperative mode)
    int* status;       // out: sweeps used, or -1 if not converged
    int max_sweeps;
};

__device__ __forceinline__ void circle_pair(int r, int i, int mp, int& p, int& q) {
    const int M1 = mp - 1;
    if (i == 0) {
        p = r;
        q = M1;
    } else {
        p = (r + i) % M1;
        q = (r - i + M1) % M1;
    }
    if (p > q) {
        const int t = p;
        p = q;
        q = t;
    }
}

// One rotation of columns (ap, aq) of length n (and optionally vp, vq of
// length m).  Columns are pulled into registers in CH-wide chunks so that all
// loads of a chunk are in flight together (the pair is latency-bound).
template <int CH>
__device__ __forceinline__ void rotate_cols(double* x, double* y, int n, int lane, double c, double s) {
    for (int base = 0; base < n; base += CH * kWarp) {
        double a[CH], b[CH];
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            const int i = base + t * kWarp + lane;
            a[t] = i < n ? x[i] : 0.0;
            b[t] = i < n ? y[i] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            const int i = base + t * kWarp + lane;
            if (i < n) {
                x[i] = c * a[t] - s * b[t];
                y[i] = s * a[t] + c * b[t];
            }
        }
    }
}

__device__ __forceinline__ bool jacobi_pair(double* ap, double* aq, int n, double* vp, double* vq, int m, int lane) {
    constexpr int CH = 16;  // n <= 512: every load of the pair in flight at once
    double al = 0.0, be = 0.0, ga = 0.0;
    for (int base = 0; base < n; base += CH * kWarp) {
        double a[CH], b[CH];
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            const int i = base + t * kWarp + lane;
            a[t] = i < n ? ap[i] : 0.0;
            b[t] = i < n ? aq[i] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            al += a[t] * a[t];
            be += b[t] * b[t];
            ga += a[t] * b[t];
        }
    }
    al = warp_sum(al);
    be = warp_sum(be);
    ga = warp_sum(ga);
    const double tol = 1e2 * DBL_EPSILON;
    if (fabs(ga) <= tol * sqrt(al * be)) return false;
    // the reference's rotation (small_svd.hpp:92-96) with correctly rounded
    // reciprocals / rsqrt instead of divisions (<= 1 ulp apart)
    const double zeta = (be - al) * __drcp_rn(2.0 * ga);
    const double t = ((zeta >= 0.0) ? 1.0 : -1.0) * __drcp_rn(fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
    const double c = rsqrt(fma(t, t, 1.0));
    const double s = c * t;
    rotate_cols<CH>(ap, aq, n, lane, c, s);
    if (vp) rotate_cols<CH>(vp, vq, m, lane, c, s);
    return true;
}

// single CTA, A (and Vacc) resident in shared memory
template <int NT>
__global__ void __launch_bounds__(NT) jacobi_smem_kernel(JacobiArgs a) {
    extern __shared__ __align__(16) double smem[];
    constexpr int NW = NT / kWarp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = a.n, m = a.m, mp = (m + 1) & ~1;
    double* A = smem;
    double* V = a.Vacc ? smem + (int64_t)n * m : nullptr;
    for (int64_t e = tid; e < (int64_t)n * m; e += NT) A[e] = a.A[e];
    if (V)
        for (int e = tid; e < m * m; e += NT) V[e] = (e % (m + 1) == 0) ? 1.0 : 0.0;
    __syncthreads();
    int sweep = 0;
    bool converged = (m < 2);
    for (; sweep < a.max_sweeps && !converged; ++sweep) {
        int rotated = 0;
        for (int r = 0; r < mp - 1; ++r) {
            for (int i = warp; i < mp / 2; i += NW) {
                int p, q;
                circle_pair(r, i, mp, p, q);
                if (q >= m) continue;
                if (jacobi_pair(A + (int64_t)p * n, A + (int64_t)q * n, n, V ? V + p * m : nullptr,
                                V ? V + q * m : nullptr, m, lane))
                    rotated = 1;
            }
            __syncthreads();
        }
        converged = __syncthreads_or(rotated) == 0;
    }
    for (int64_t e = tid; e < (int64_t)n * m; e += NT) a.A[e] = A[e];
    if (V)
        for (int e = tid; e < m * m; e += NT) a.Vacc[e] = V[e];
    if (tid == 0) *a.status = converged ? sweep : -1;
}

// cooperative grid, A (and Vacc) in global memory (L2 resident); grid.sync per round
template <int NT>
__global__ void __launch_bounds__(NT) jacobi_coop_kernel(JacobiArgs a) {
    cg::grid_group grid = cg::this_grid();
    constexpr int NW = NT / kWarp;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * NW + (threadIdx.x >> 5);
    const int tw = gridDim.x * NW;
    const int n = a.n, m = a.m, mp = (m + 1) & ~1;
    double* A = a.A;
    double* V = a.Vacc;
    if (V) {
        for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < (int64_t)m * m; e += (int64_t)gridDim.x * NT)
            V[e] = (e % (m + 1) == 0) ? 1.0 : 0.0;
        grid.sync();
    }
    int sweep = 0;
    bool converged = (m < 2);
    for (; sweep < a.max_sweeps && !converged; ++sweep) {
        int rotated = 0;
        for (int r = 0; r < mp - 1; ++r) {
            for (int i = gw; i < mp / 2; i += tw) {
                int p, q;
                circle_pair(r, i, mp, p, q);
                if (q >= m) continue;
                if (jacobi_pair(A + (int64_t)p * n, A + (int64_t)q * n, n, V ? V + (int64_t)p * m : nullptr,
                                V ? V + (int64_t)q * m : nullptr, m, lane))
                    rotated = 1;
            }
            grid.sync();
        }
        if (rotated && lane == 0) atomicAdd(&a.sweep_flags[sweep], 1);
        grid.sync();
        converged = *((volatile int*)&a.sweep_flags[sweep]) == 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.status = converged ? sweep : -1;
}

// Column norms, stable descending order, sigma, normalised columns -> Uout
// (n x m) with the reference's canonical completion for sigma <= n eps sigma_1
// (small_svd.hpp:133-191), and Vacc permuted -> Vout (m x m) when given.
// One CTA.  smem: norms[m], pos[m] (as double), deficient flags.
template <int NT>
__global__ void __launch_bounds__(NT) jacobi_finalize_kernel(const double* A, int n, int m, const double* Vacc,
                                                             double* sigma, double* Uout, double* Vout) {
    extern __shared__ __align__(16) double smem[];
    constexpr int NW = NT / kWarp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* norms = smem;
    int* pos = reinterpret_cast<int*>(norms + m);
    int* src_of = pos + m;
    double* red = reinterpret_cast<double*>(src_of + m);  // 2m ints keep 8-byte alignment
    for (int j = warp; j < m; j += NW) {
        double s = 0.0;
        const double* c = A + (int64_t)j * n;
        for (int i = lane; i < n; i += kWarp) s += c[i] * c[i];
        s = warp_sum(s);
        if (lane == 0) norms[j] = sqrt(s);
    }
    __syncthreads();
    for (int j = tid; j < m; j += NT) {
        const double x = norms[j];
        int p = 0;
        for (int i = 0; i < m; ++i) {
            const double y = norms[i];
            p += (y > x) || (y == x && i < j);
        }
        pos[j] = p;
        src_of[p] = j;
    }
    __syncthreads();
    const double sigma1 = m > 0 ? norms[src_of[0]] : 0.0;
    const double cutoff = sigma1 * (double)n * DBL_EPSILON;
    for (int j = tid; j < m; j += NT) sigma[pos[j]] = norms[j];
    for (int jj = warp; jj < m; jj += NW) {
        const int src = src_of[jj];
        const double s = norms[src];
        double* u = Uout + (int64_t)jj * n;
        const double* c = A + (int64_t)src * n;
        if (s > cutoff) {
            const double inv = 1.0 / s;
            for (int i = lane; i < n; i += kWarp) u[i] = c[i] * inv;
        } else {
            for (int i = lane; i < n; i += kWarp) u[i] = 0.0;
        }
        if (Vout) {
            const double* vs = Vacc + (int64_t)src * m;
            double* vd = Vout + (int64_t)jj * m;
            for (int i = lane; i < m; i += kWarp) vd[i] = vs[i];
        }
    }
    __syncthreads();
    __threadfence_block();
    // deterministic completion of the deficient columns (rare; sequential over
    // columns and axes, the CTA cooperates on each dot product)
    int next_axis = 0;
    for (int j = 0; j < m; ++j) {
        if (norms[src_of[j]] > cutoff) continue;
        double* uj = Uout + (int64_t)j * n;
        for (; next_axis < n; ++next_axis) {
            for (int i = tid; i < n; i += NT) uj[i] = (i == next_axis) ? 1.0 : 0.0;
            __syncthreads();
            for (int pass = 0; pass < 2; ++pass) {
                for (int k = 0; k < m; ++k) {
                    if (k == j) continue;
                    const double* uk = Uout + (int64_t)k * n;
                    double s = 0.0;
                    for (int i = tid; i < n; i += NT) s += uk[i] * uj[i];
                    s = warp_sum(s);
                    if (lane == 0) red[warp] = s;
                    __syncthreads();
                    double dot = 0.0;
                    for (int w = 0; w < NW; ++w) dot += red[w];
                    for (int i = tid; i < n; i += NT) uj[i] -= dot * uk[i];
                    __syncthreads();
                }
            }
            double s = 0.0;
            for (int i = tid; i < n; i += NT) s += uj[i] * uj[i];
            s = warp_sum(s);
            if (lane == 0) red[warp] = s;
            __syncthreads();
            double nrm = 0.0;
            for (int w = 0; w < NW; ++w) nrm += red[w];
            nrm = sqrt(nrm);
            __syncthreads();
            if (nrm > 0.5) {
                for (int i = tid; i < n; i += NT) uj[i] /= nrm;
                __syncthreads();
                ++next_axis;
                break;
            }
        }
    }
}

// dst (cols x rows, ld cols) = src^T, src rows x cols with ld_src
__global__ void transpose_kernel(const double* src, int64_t rows, int64_t cols, int64_t ld_src, double* dst) {
    __shared__ double tile[32][33];
    const int64_t bx = blockIdx.x * 32, by = blockIdx.y * 32;  // bx over cols, by over rows
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t r = by + threadIdx.x, c = bx + k;
        if (r < rows && c < cols) tile[k][threadIdx.x] = src[c * ld_src + r];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t c = bx + threadIdx.x, r = by + k;
        if (r < rows && c < cols) dst[r * cols + c] = tile[threadIdx.x][k];
    }
}

// ---------------------------------------------------------------------------
// K_TSMM — Y = reshape(X V[:, c0:c0+KC]).  One thread per row i; the V chunk
// sits in shared memory as [j][c] so every FMA reads a broadcast; the KC
// results of row i go to flat positions p = i + n*c, i.e. Y(p mod out_rows,
// p div out_rows) (tsmm.hpp:14-19).  When out_rows divides n (every TT step)
// the destination is column (i div out_rows) + n_next*c, row i mod out_rows,
// so consecutive threads write consecutive addresses.
// ---------------------------------------------------------------------------
template <int KC>
__global__ void __launch_bounds__(256) tsmm_kernel(const double* __restrict__ X, int64_t n, int m, int64_t ldx,
                                                   const double* __restrict__ V, int64_t ldv, int k,
                                                   double* __restrict__ Y, int64_t out_rows, int64_t ldy) {
    extern __shared__ __align__(16) double Vs[];
    const int c0 = blockIdx.y * KC;
    const int kc = min(KC, k - c0);
    for (int e = threadIdx.x; e < m * KC; e += blockDim.x) {
        const int j = e / KC, c = e % KC;
        Vs[e] = (c < kc) ? V[(int64_t)(c0 + c) * ldv + j] : 0.0;
    }
    __syncthreads();
    const bool divisible = (n % out_rows) == 0;
    const int64_t n_next = divisible ? n / out_rows : 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double acc[KC];
#pragma unroll
        for (int c = 0; c < KC; ++c) acc[c] = 0.0;
        const double* xi = X + i;
#pragma unroll 4
        for (int j = 0; j < m; ++j) {
            const double x = ldg_stream(xi + (int64_t)j * ldx);
            const double* vj = Vs + j * KC;
#pragma unroll
            for (int c = 0; c < KC; ++c) acc[c] = fma(vj[c], x, acc[c]);
        }
        if (divisible) {
            const int64_t b = i / out_rows, ii = i - b * out_rows;
#pragma unroll
            for (int c = 0; c < KC; ++c)
                if (c < kc) Y[(b + n_next * (c0 + c)) * ldy + ii] = acc[c];
        } else {
#pragma unroll
            for (int c = 0; c < KC; ++c)
                if (c < kc) {
                    const int64_t p = i + n * (c0 + c);
                    const int64_t col = p / out_rows;
                    Y[col * ldy + (p - col * out_rows)] = acc[c];
                }
        }
    }
}

// K_TSMM for short X (n <= 2^14 rows: the last steps of a chain, where the
// row-per-thread kernel leaves one to sixteen CTAs walking all m columns with
// four loads in flight each).  CTA (b, y) owns 32 rows and KC output columns;
// its eight warps split the contraction index (warp w: columns
// [w jw, (w+1) jw) of X, lane = row), the eight partial sums meet in shared
// memory and are added in warp order.  Output placement as tsmm_kernel.
template <int KC>
__global__ void __launch_bounds__(256) tsmm_small_kernel(const double* __restrict__ X, int64_t n, int m, int64_t ldx,
                                                         const double* __restrict__ V, int64_t ldv, int k,
                                                         double* __restrict__ Y, int64_t out_rows, int64_t ldy) {
    static_assert(KC <= 8, "one finishing thread per (column, row)");
    extern __shared__ __align__(16) double Vs[];
    double* red = Vs + m * KC;  // 8 x KC x 32
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c0 = blockIdx.y * KC;
    const int kc = min(KC, k - c0);
    for (int e = tid; e < m * KC; e += 256) {
        const int j = e / KC, c = e % KC;
        Vs[e] = (c < kc) ? V[(int64_t)(c0 + c) * ldv + j] : 0.0;
    }
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * 32 + lane;
    const int jw = (m + 7) / 8;
    const int j0 = warp * jw, j1 = min(m, j0 + jw);
    double acc[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) acc[c] = 0.0;
    if (i < n) {
        const double* xi = X + i;
#pragma unroll 8
        for (int j = j0; j < j1; ++j) {
            const double x = __ldg(xi + (int64_t)j * ldx);
            const double* vj = Vs + j * KC;
#pragma unroll
            for (int c = 0; c < KC; ++c) acc[c] = fma(vj[c], x, acc[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < KC; ++c) red[(warp * KC + c) * 32 + lane] = acc[c];
    __syncthreads();
    const int c = warp;  // finishing thread: column c0 + warp, row `lane`
    if (c < kc && i < n) {
        double t = red[c * 32 + lane];
#pragma unroll
        for (int w = 1; w < 8; ++w) t += red[(w * KC + c) * 32 + lane];
        const int64_t p = i + n * (int64_t)(c0 + c);
        const int64_t col = p / out_rows;
        Y[col * ldy + (p - col * out_rows)] = t;
    }
}

// K_TSMM for narrow X (m <= 32) and few output columns: the streamed rows are
// staged in shared memory by cp.async (each thread copies its own row's m
// values, 8 bytes apiece, one chunk of 256 rows ahead), so the bytes in
// flight per SM are bounded by shared memory instead of registers; a thread
// only reads the row it copied itself, so cp.async.wait_group is the only
// synchronisation.  Same arithmetic and output placement as tsmm_kernel.
template <int KC>
__global__ void __launch_bounds__(256) tsmm_async_kernel(const double* __restrict__ X, int64_t n, int m, int64_t ldx,
                                                         const double* __restrict__ V, int64_t ldv, int k,
                                                         double* __restrict__ Y, int64_t out_rows, int64_t ldy) {
    extern __shared__ __align__(16) double tsm[];
    double* Vs = tsm;                         // m x KC
    double* xb = tsm + ((m * KC + 1) & ~1);   // 2 x m x 256
    const int tid = threadIdx.x;
    const int c0 = blockIdx.y * KC;
    const int kc = min(KC, k - c0);
    for (int e = tid; e < m * KC; e += blockDim.x) {
        const int j = e / KC, c = e % KC;
        Vs[e] = (c < kc) ? V[(int64_t)(c0 + c) * ldv + j] : 0.0;
    }
    __syncthreads();
    const bool divisible = (n % out_rows) == 0;
    const int64_t n_next = divisible ? n / out_rows : 0;
    const int64_t chunks = (n + 255) / 256;
    auto stage = [&](int64_t ch, int buf) {
        const int64_t row = ch * 256 + tid;
        double* dst = xb + (size_t)buf * m * 256 + tid;
        if (row < n) {
            for (int j = 0; j < m; ++j) {
                const unsigned sd = (unsigned)__cvta_generic_to_shared(dst + j * 256);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sd), "l"(X + (int64_t)j * ldx + row)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int buf = 0;
    int64_t ch = blockIdx.x;
    if (ch < chunks) stage(ch, 0);
    for (; ch < chunks; ch += gridDim.x) {
        const int64_t nx = ch + gridDim.x;
        if (nx < chunks) {
            stage(nx, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        const int64_t i = ch * 256 + tid;
        if (i < n) {
            const double* xr = xb + (size_t)buf * m * 256 + tid;
            double acc[KC];
#pragma unroll
            for (int c = 0; c < KC; ++c) acc[c] = 0.0;
#pragma unroll 4
            for (int j = 0; j < m; ++j) {
                const double x = xr[j * 256];
                const double* vj = Vs + j * KC;
#pragma unroll
                for (int c = 0; c < KC; ++c) acc[c] = fma(vj[c], x, acc[c]);
            }
            if (divisible) {
                const int64_t b = i / out_rows, ii = i - b * out_rows;
#pragma unroll
                for (int c = 0; c < KC; ++c)
                    if (c < kc) Y[(b + n_next * (c0 + c)) * ldy + ii] = acc[c];
            } else {
#pragma unroll
                for (int c = 0; c < KC; ++c)
                    if (c < kc) {
                        const int64_t p = i + n * (c0 + c);
                        const int64_t col = p / out_rows;
                        Y[col * ldy + (p - col * out_rows)] = acc[c];
                    }
            }
        }
        buf ^= 1;
    }
}

// tsmm_async_kernel for wider X (m > 32): the row chunk is streamed in
// blocks of 32 columns (one cp.async stage per (chunk, column block), double
// buffered across the flattened sequence), the KC accumulators persist over a
// chunk's blocks.  V (m x KC) stays in shared memory.
template <int KC>
__global__ void __launch_bounds__(256) tsmm_async_wide_kernel(const double* __restrict__ X, int64_t n, int m,
                                                              int64_t ldx, const double* __restrict__ V, int64_t ldv,
                                                              int k, double* __restrict__ Y, int64_t out_rows,
                                                              int64_t ldy) {
    extern __shared__ __align__(16) double tsm[];
    constexpr int MB = 32;
    double* Vs = tsm;                        // m x KC
    double* xb = tsm + ((m * KC + 1) & ~1);  // 2 x MB x 256
    const int tid = threadIdx.x;
    const int c0 = blockIdx.y * KC;
    const int kc = min(KC, k - c0);
    for (int e = tid; e < m * KC; e += blockDim.x) {
        const int j = e / KC, c = e % KC;
        Vs[e] = (c < kc) ? V[(int64_t)(c0 + c) * ldv + j] : 0.0;
    }
    __syncthreads();
    const bool divisible = (n % out_rows) == 0;
    const int64_t n_next = divisible ? n / out_rows : 0;
    const int64_t chunks = (n + 255) / 256;
    const int nb = (m + MB - 1) / MB;
    const int64_t my_chunks = (chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;  // chunks of this CTA
    const int64_t seq = blockIdx.x < chunks ? my_chunks * nb : 0;
    auto stage = [&](int64_t sidx, int buf) {
        const int64_t ch = blockIdx.x + (sidx / nb) * gridDim.x;
        const int b = (int)(sidx % nb);
        const int64_t row = ch * 256 + tid;
        double* dst = xb + (size_t)buf * MB * 256 + tid;
        const int jn = min(MB, m - b * MB);
        if (row < n) {
            for (int jj = 0; jj < jn; ++jj) {
                const unsigned sd = (unsigned)__cvta_generic_to_shared(dst + jj * 256);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sd),
                             "l"(X + (int64_t)(b * MB + jj) * ldx + row)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) acc[c] = 0.0;
    if (seq > 0) stage(0, 0);
    for (int64_t sidx = 0; sidx < seq; ++sidx) {
        const int buf = (int)(sidx & 1);
        if (sidx + 1 < seq) {
            stage(sidx + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        const int64_t ch = blockIdx.x + (sidx / nb) * gridDim.x;
        const int b = (int)(sidx % nb);
        const int64_t i = ch * 256 + tid;
        const int jn = min(MB, m - b * MB);
        const double* xr = xb + (size_t)buf * MB * 256 + tid;
        const double* vb = Vs + (size_t)b * MB * KC;
        if (i < n) {
#pragma unroll 4
            for (int jj = 0; jj < jn; ++jj) {
                const double x = xr[jj * 256];
                const double* vj = vb + jj * KC;
#pragma unroll
                for (int c = 0; c < KC; ++c) acc[c] = fma(vj[c], x, acc[c]);
            }
        }
        if (b == nb - 1) {
            if (i < n) {
                if (divisible) {
                    const int64_t bb = i / out_rows, ii = i - bb * out_rows;
#pragma unroll
                    for (int c = 0; c < KC; ++c)
                        if (c < kc) Y[(bb + n_next * (c0 + c)) * ldy + ii] = acc[c];
                } else {
#pragma unroll
                    for (int c = 0; c < KC; ++c)
                        if (c < kc) {
                            const int64_t p = i + n * (c0 + c);
                            const int64_t col = p / out_rows;
                            Y[col * ldy + (p - col * out_rows)] = acc[c];
                        }
                }
            }
#pragma unroll
            for (int c = 0; c < KC; ++c) acc[c] = 0.0;
        }
    }
}

// K_TSMM on the FP64 tensor cores: each warp computes a 32-row x 8NT-column
// block of X V with DMMA m8n8k4 (A fragments loaded straight from X — for a
// fixed fragment column the 8 rows are one contiguous 64-byte run — B
// fragments from the chunk of V staged in shared memory), then scatters it
// into the next step's padded layout exactly as tsmm_kernel (element (i, c)
// at flat position i + n c).  Output columns c0 .. c0 + 8NT - 1 (grid.y
// chunks).  The product of a unit column of V is exact (column selection).
__host__ __device__ inline int tsmm_vld(int nt) { return ((8 * nt + 15) / 16) * 16 + 4; }

template <int NT>
__global__ void __launch_bounds__(256) tsmm_dmma_kernel(const double* __restrict__ X, int64_t n, int m, int64_t ldx,
                                                        const double* __restrict__ V, int64_t ldv, int k,
                                                        double* __restrict__ Y, int64_t out_rows, int64_t ldy) {
    extern __shared__ __align__(16) double Vs[];  // (m rounded to 4) x tsmm_vld(NT)
    constexpr int VLD = ((8 * NT + 15) / 16) * 16 + 4;
    const int c0 = blockIdx.y * 8 * NT;
    const int kc = min(8 * NT, k - c0);
    const int m4 = (m + 3) & ~3;
    for (int e = threadIdx.x; e < m4 * VLD; e += blockDim.x) {
        const int j = e / VLD, c = e % VLD;
        Vs[e] = (j < m && c < kc) ? V[(int64_t)(c0 + c) * ldv + j] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = lane >> 2, q = lane & 3;
    const bool divisible = (n % out_rows) == 0;
    const int64_t n_next = divisible ? n / out_rows : 0;
    const int64_t stride = (int64_t)gridDim.x * (blockDim.x / 32) * 32;
    for (int64_t rb = ((int64_t)blockIdx.x * (blockDim.x / 32) + warp) * 32; rb < n; rb += stride) {
        double acc[4][NT][2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
        const bool full = rb + 32 <= n;
#pragma unroll 2
        for (int kk = 0; kk < m4 / 4; ++kk) {
            const int col = 4 * kk + q;
            const double* xc = X + (int64_t)col * ldx + rb + r;
            double a[4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
                a[mt] = (col < m && (full || rb + 8 * mt + r < n)) ? ldg_stream(xc + 8 * mt) : 0.0;
            double b[NT];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) b[nt] = Vs[col * VLD + 8 * nt + r];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt], a[mt], b[nt]);
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int64_t i = rb + 8 * mt + r;
            if (i >= n) continue;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = 8 * nt + 2 * q + e;
                    if (c >= kc) continue;
                    if (divisible) {
                        const int64_t b = i / out_rows, ii = i - b * out_rows;
                        Y[(b + n_next * (c0 + c)) * ldy + ii] = acc[mt][nt][e];
                    } else {
                        const int64_t p = i + n * (c0 + c);
                        const int64_t cl = p / out_rows;
                        Y[cl * ldy + (p - cl * out_rows)] = acc[mt][nt][e];
                    }
                }
        }
    }
}

// ---------------------------------------------------------------------------
// transpose_reorder (tsmm.hpp:84-126, the two-sided sweep's reorder): W (n x m,
// ld ldw) is flattened as W^T, i.e. W(i, j) goes to flat position p = m i + j,
// which is Y(p mod out_rows, p div out_rows).  A pure permutation, HBM-bound
// (16 n m bytes).  A 32 x 32 tile is read along W's columns (coalesced) into
// shared memory and written along W's rows: for a fixed i the 32 values of
// j are 32 consecutive flat positions, i.e. a contiguous run of Y (split at
// most once where it crosses an out_rows boundary).  Grid-stride over tiles.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) transpose_reorder_kernel(const double* __restrict__ W, int64_t n, int64_t m,
                                                                int64_t ldw, double* __restrict__ Y,
                                                                int64_t out_rows, int64_t ldy) {
    __shared__ double tile[32][33];
    const int64_t ti = (n + 31) / 32, tj = (m + 31) / 32;
    for (int64_t t = blockIdx.x; t < ti * tj; t += gridDim.x) {
        const int64_t i0 = (t % ti) * 32, j0 = (t / ti) * 32;
        for (int k = threadIdx.y; k < 32; k += blockDim.y) {
            const int64_t i = i0 + threadIdx.x, j = j0 + k;
            if (i < n && j < m) tile[k][threadIdx.x] = W[j * ldw + i];
        }
        __syncthreads();
        for (int k = threadIdx.y; k < 32; k += blockDim.y) {
            const int64_t i = i0 + k, j = j0 + threadIdx.x;
            if (i < n && j < m) {
                const int64_t p = m * i + j;
                Y[(p / out_rows) * ldy + p % out_rows] = tile[threadIdx.x][k];
            }
        }
        __syncthreads();
    }
}

// zero rows [out_rows, ldy) of every column of Y (the padded slots, storage.hpp:57)
__global__ void zero_padding_kernel(double* Y, int64_t out_rows, int64_t ldy, int64_t cols) {
    const int64_t pad = ldy - out_rows;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < pad * cols; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / pad;
        Y[c * ldy + out_rows + (e - c * pad)] = 0.0;
    }
}

}  // namespace ttsvd_b200
