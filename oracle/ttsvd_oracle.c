/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the TT-SVD hot path.
 *
 * A plain-C restatement of the reference algorithm in
 * /root/reference/proj/include/ttsvd/ (the .hpp headers) (arXiv 2102.00104, Alg. 2 / Alg. 5 /
 * Alg. 6).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load this library, and only as the checker.  The product path
 * (paper_2102_00104_b200/) never links, loads or calls it.
 *
 * Parity pin: every function here is checked against the reference itself
 * (oracle/_ref/libttsvd_ref.so, compiled from the untouched reference headers by
 * oracle/Makefile) and against the reference tests' known answers — see
 * tests/test_oracle_pin.py.  The arithmetic follows the reference operation by
 * operation (same summation order, same 4-way partial dot products, same
 * reflector formula), so the two agree bitwise when both are built with
 * -ffp-contract=off.
 *
 * Status codes are the ones in include/ttsvd_cu.h (TTSVD_OK, TTSVD_ERR_*).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_DIMENSION 1          /* DimensionError */
#define ORC_ERR_DIMENSION_MISMATCH 2 /* DimensionMismatch */
#define ORC_ERR_SHAPE 3              /* ShapeError */
#define ORC_ERR_CONVERGENCE 4        /* ConvergenceError */
#define ORC_ERR_ALLOCATION 5         /* AllocationError */
#define ORC_ERR_DEGENERATE 6         /* DegenerateDimension */
#define ORC_ERR_PARTITION 7          /* PartitionMismatch */
#define ORC_ERR_INVALID 9
#define ORC_ERR_CAPACITY 11

typedef int64_t idx;

static idx imax(idx a, idx b) { return a > b ? a : b; }
static idx imin(idx a, idx b) { return a < b ? a : b; }

/* shape.hpp:22-28 — smallest odd multiple of 64 that is >= n (64 for n <= 64). */
idx orc_padded_stride(idx n_rows) {
    if (n_rows < 1) return -1;
    if (n_rows <= 64) return 64;
    idx q = (n_rows + 63) / 64;
    if (q % 2 == 0) ++q;
    return 64 * q;
}

/* tsqr.hpp:48-56 — BlockParams::for_cols: largest multiple of 8 with
 * (n_b + m) * m * 8 <= budget, clamped to [16, 4096]. */
idx orc_block_nb(idx m, idx l2_budget_bytes) {
    const idx cap = l2_budget_bytes / 8;
    idx nb = (cap / imax(m, 1) - m) / 8 * 8;
    if (nb < 16) nb = 16;
    if (nb > 4096) nb = 4096;
    return nb;
}

/* threading.hpp:23-36 — contiguous balanced partition, depends only on (n, workers). */
int orc_partition_rows(idx n, int workers, idx* begins, idx* ends) {
    if (workers < 1) workers = 1;
    const idx w = imin(workers, imax(n, 1));
    const idx base = n / w, rem = n % w;
    idx b = 0;
    for (idx i = 0; i < w; ++i) {
        const idx len = base + (i < rem ? 1 : 0);
        begins[i] = b;
        ends[i] = b + len;
        b += len;
    }
    return (int)w;
}

/* tsqr.hpp:145-157 — four independent partial sums, then the sequential tail. */
static double dot4(const double* a, const double* b, idx len) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    idx i = 0;
    for (; i + 4 <= len; i += 4) {
        s0 += a[i] * b[i];
        s1 += a[i + 1] * b[i + 1];
        s2 += a[i + 2] * b[i + 2];
        s3 += a[i + 3] * b[i + 3];
    }
    double s = (s0 + s1) + (s2 + s3);
    for (; i < len; ++i) s += a[i] * b[i];
    return s;
}

/*
 * tsqr.hpp:176-194 (reduce_into) + tsqr.hpp:90-170 (BlockReducer, Alg. 6).
 * Staircase W = [M zero-padded to n_b = max(rows, m) rows; R], ld = n_b + m.
 * Reflector j spans rows j..j+n_b of column j (n_b + 1 entries).  The
 * reference's recursive column split (tsqr.hpp:105-118) is a pure reordering
 * of the plain j-loop — every column k still receives apply(0..k-1, k) in
 * increasing order before form_reflector(k) — so the plain loop is bitwise
 * identical.  w/v are caller scratch of (n_b+m)*m and (n_b+1)*m doubles.
 */
static void reduce_into(const double* M, idx rows, idx m, idx ldm, double* R, double* w, double* v) {
    const double eps = DBL_MIN; /* BlockParams::eps_fp, tsqr.hpp:43 */
    const idx n_b = imax(rows, m);
    const idx ldw = n_b + m;
    for (idx j = 0; j < m; ++j) {
        double* wj = w + j * ldw;
        memcpy(wj, M + j * ldm, (size_t)rows * sizeof(double));
        for (idx i = rows; i < n_b; ++i) wj[i] = 0.0;
        memcpy(wj + n_b, R + j * m, (size_t)m * sizeof(double));
    }
    for (idx j = 0; j < m; ++j) {
        /* form_reflector(j), tsqr.hpp:120-142 */
        double* wj = w + j * ldw;
        double* u = wj + j;
        double t = eps + dot4(u, u, n_b + 1);
        double alpha = sqrt(t + eps);
        alpha = (u[0] > 0.0) ? -alpha : alpha;
        t -= alpha * u[0];
        const double beta = 1.0 / sqrt(t);
        double* vj = v + j * (n_b + 1);
        vj[0] = (u[0] - alpha) * beta;
        for (idx i = 1; i <= n_b; ++i) vj[i] = u[i] * beta;
        for (idx i = 0; i < j; ++i) wj[n_b + i] = wj[i];
        wj[n_b + j] = alpha;
        /* apply(j, k), tsqr.hpp:159-164 */
        for (idx k = j + 1; k < m; ++k) {
            double* wk = w + k * ldw + j;
            const double gamma = dot4(vj, wk, n_b + 1);
            for (idx i = 0; i <= n_b; ++i) wk[i] -= gamma * vj[i];
        }
    }
    for (idx j = 0; j < m; ++j) memcpy(R + j * m, w + j * ldw + n_b, (size_t)m * sizeof(double));
}

/* tsqr.hpp:208-224 — Rbar with Rbar^T Rbar = M^T M + R^T R. */
int orc_reduce_block(const double* M, idx rows, idx m, idx ldm, const double* R_in, idx r_m, double* R_out) {
    if (r_m != m) return ORC_ERR_DIMENSION_MISMATCH;
    if (m < 1 || rows < 0) return ORC_ERR_INVALID;
    const idx n_b = imax(rows, m);
    double* w = (double*)malloc((size_t)((n_b + m) * m + (n_b + 1) * m) * sizeof(double));
    if (!w) return ORC_ERR_ALLOCATION;
    memcpy(R_out, R_in, (size_t)(m * m) * sizeof(double));
    reduce_into(M, rows, m, ldm, R_out, w, w + (n_b + m) * m);
    free(w);
    return ORC_OK;
}

/* tsqr.hpp:230-240 — pinned left-to-right merge; the accumulated triangle stays
 * the R operand, each new part enters as M. */
int orc_combine_factors(const double* parts, idx P, idx m, double* R) {
    if (P < 1) return ORC_ERR_DIMENSION_MISMATCH;
    memcpy(R, parts, (size_t)(m * m) * sizeof(double));
    double* w = (double*)malloc((size_t)(2 * m * m + (m + 1) * m) * sizeof(double));
    if (!w) return ORC_ERR_ALLOCATION;
    for (idx p = 1; p < P; ++p) reduce_into(parts + p * m * m, m, m, m, R, w, w + 2 * m * m);
    free(w);
    return ORC_OK;
}

/* tsqr.hpp:247-292 — per-worker flat tree over contiguous row ranges in blocks
 * of n_b rows, then combine_factors in ascending worker order.  Workers run
 * sequentially here; the result depends only on (n, workers, n_b). */
int orc_tsqr(const double* X, idx n, idx m, idx ldx, idx n_b, int workers, double* R) {
    if (m < 1) return ORC_ERR_DIMENSION;
    if (n < m) return ORC_ERR_DIMENSION;
    if (n_b < 1) return ORC_ERR_INVALID;
    if (workers < 1) workers = 1;
    idx* b = (idx*)malloc(sizeof(idx) * 2 * (size_t)workers);
    const int nw = orc_partition_rows(n, workers, b, b + workers);
    const idx nbm = imax(n_b, m);
    double* parts = (double*)calloc((size_t)(nw * m * m), sizeof(double));
    double* w = (double*)malloc((size_t)((nbm + m) * m + (nbm + 1) * m) * sizeof(double));
    if (!parts || !w) {
        free(b); free(parts); free(w);
        return ORC_ERR_ALLOCATION;
    }
    for (int q = 0; q < nw; ++q) {
        double* Rq = parts + (idx)q * m * m;
        for (idx r0 = b[q]; r0 < b[workers + q]; r0 += n_b) {
            const idx rows = imin(n_b, b[workers + q] - r0);
            reduce_into(X + r0, rows, m, ldx, Rq, w, w + (imax(rows, m) + m) * m);
        }
    }
    int rc = ORC_OK;
    if (nw == 1) memcpy(R, parts, (size_t)(m * m) * sizeof(double));
    else rc = orc_combine_factors(parts, nw, m, R);
    free(b); free(parts); free(w);
    return rc;
}

/* small_svd.hpp:72-114 — cyclic one-sided Jacobi, rotations accumulated into V. */
static int jacobi_orthogonalize(double* a, idx n, idx m, double* v) {
    for (idx i = 0; i < m * m; ++i) v[i] = 0.0;
    for (idx j = 0; j < m; ++j) v[j * m + j] = 1.0;
    const double tol = 1e2 * DBL_EPSILON;
    for (int sweep = 0; sweep < 30; ++sweep) {
        int rotated = 0;
        for (idx p = 0; p < m - 1; ++p) {
            for (idx q = p + 1; q < m; ++q) {
                double* ap = a + p * n;
                double* aq = a + q * n;
                double alpha = 0.0, beta = 0.0, gamma = 0.0;
                for (idx i = 0; i < n; ++i) {
                    alpha += ap[i] * ap[i];
                    beta += aq[i] * aq[i];
                    gamma += ap[i] * aq[i];
                }
                if (fabs(gamma) <= tol * sqrt(alpha * beta)) continue;
                rotated = 1;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = ((zeta >= 0.0) ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double s = c * t;
                for (idx i = 0; i < n; ++i) {
                    const double x = ap[i], y = aq[i];
                    ap[i] = c * x - s * y;
                    aq[i] = s * x + c * y;
                }
                double* vp = v + p * m;
                double* vq = v + q * m;
                for (idx i = 0; i < m; ++i) {
                    const double x = vp[i], y = vq[i];
                    vp[i] = c * x - s * y;
                    vq[i] = s * x + c * y;
                }
            }
        }
        if (!rotated) return ORC_OK;
    }
    return ORC_ERR_CONVERGENCE;
}

/* small_svd.hpp:120-193 — jacobi_svd of a tall n x m matrix: sigma sorted
 * non-increasing (stable), V permuted to match, U = a/sigma with the
 * deterministic canonical-basis completion for sigma <= n*eps*sigma_1.
 * U may be NULL (the TT-SVD drivers only consume V; tt_svd.hpp:88-90). */
int orc_jacobi_svd(const double* A, idx n, idx m, idx lda, double* sigma, double* U, double* V) {
    if (n < m) return ORC_ERR_DIMENSION;
    double* a = (double*)malloc((size_t)(n * m + m * m + m) * sizeof(double));
    idx* order = (idx*)malloc((size_t)(m > 0 ? m : 1) * sizeof(idx));
    if (!a || !order) {
        free(a); free(order);
        return ORC_ERR_ALLOCATION;
    }
    double* v = a + n * m;
    double* norms = v + m * m;
    for (idx j = 0; j < m; ++j)
        for (idx i = 0; i < n; ++i) a[j * n + i] = A[j * lda + i];
    int rc = jacobi_orthogonalize(a, n, m, v);
    if (rc != ORC_OK) {
        free(a); free(order);
        return rc;
    }
    for (idx j = 0; j < m; ++j) {
        double s = 0.0;
        const double* c = a + j * n;
        for (idx i = 0; i < n; ++i) s += c[i] * c[i];
        norms[j] = sqrt(s);
    }
    /* std::stable_sort descending by norm == insertion sort with strict '>' */
    for (idx j = 0; j < m; ++j) order[j] = j;
    for (idx j = 1; j < m; ++j) {
        const idx key = order[j];
        idx i = j - 1;
        while (i >= 0 && norms[key] > norms[order[i]]) {
            order[i + 1] = order[i];
            --i;
        }
        order[i + 1] = key;
    }
    const double sigma1 = m > 0 ? norms[order[0]] : 0.0;
    const double cutoff = sigma1 * (double)n * DBL_EPSILON;
    if (U) for (idx i = 0; i < n * m; ++i) U[i] = 0.0;
    for (idx j = 0; j < m; ++j) {
        const idx src = order[j];
        const double s = norms[src];
        sigma[j] = s;
        for (idx i = 0; i < m; ++i) V[j * m + i] = v[src * m + i];
        if (U && s > cutoff) {
            const double inv = 1.0 / s;
            for (idx i = 0; i < n; ++i) U[j * n + i] = a[src * n + i] * inv;
        }
    }
    if (U) {
        idx next_axis = 0;
        for (idx j = 0; j < m; ++j) {
            if (sigma[j] > cutoff) continue;
            double* uj = U + j * n;
            for (; next_axis < n; ++next_axis) {
                for (idx i = 0; i < n; ++i) uj[i] = 0.0;
                uj[next_axis] = 1.0;
                for (int pass = 0; pass < 2; ++pass) {
                    for (idx k = 0; k < m; ++k) {
                        if (k == j) continue;
                        const double* uk = U + k * n;
                        double dot = 0.0;
                        for (idx i = 0; i < n; ++i) dot += uk[i] * uj[i];
                        for (idx i = 0; i < n; ++i) uj[i] -= dot * uk[i];
                    }
                }
                double nrm = 0.0;
                for (idx i = 0; i < n; ++i) nrm += uj[i] * uj[i];
                nrm = sqrt(nrm);
                if (nrm > 0.5) {
                    for (idx i = 0; i < n; ++i) uj[i] /= nrm;
                    ++next_axis;
                    break;
                }
            }
        }
    }
    free(a); free(order);
    return ORC_OK;
}

/* small_svd.hpp:196-199 */
int orc_small_svd(const double* R, idx m, double* sigma, double* U, double* V) {
    if (m > 4096) return ORC_ERR_DIMENSION_MISMATCH;
    return orc_jacobi_svd(R, m, m, m, sigma, U, V);
}

/* small_svd.hpp:49-63 — tail-sum rank rule, clamped to [1, m]. */
idx orc_select_rank(const double* sigma, idx m, double delta, idx r_max) {
    double tail = 0.0;
    idx r_delta = m;
    for (idx j = m; j-- > 0;) {
        tail += sigma[j] * sigma[j];
        if (tail <= delta * delta) r_delta = j;
        else break;
    }
    idx r = imin(r_max, r_delta);
    if (r < 1) r = 1;
    return imin(r, imax(m, 1));
}

/* small_svd.hpp:41-44 */
int orc_derive_delta(double norm_source, double eps, idx d, double* out) {
    if (d < 2) return ORC_ERR_DEGENERATE;
    *out = eps / sqrt((double)(d - 1)) * norm_source;
    return ORC_OK;
}

/* small_svd.hpp:201-205 */
double orc_sigma_norm(const double* sigma, idx m) {
    double s = 0.0;
    for (idx j = 0; j < m; ++j) s += sigma[j] * sigma[j];
    return sqrt(s);
}

/* tt_svd.hpp:111-118 — tail rule with the numerical-zero floor. */
idx orc_choose_rank(const double* sigma, idx len, idx cols, idx nsig, double delta, idx r_max, idx rows) {
    const double sigma1 = len > 0 ? sigma[0] : 0.0;
    const double zero_level = 32.0 * DBL_EPSILON * sigma1 * sqrt((double)imax(rows, cols));
    const double delta_eff = delta > zero_level ? delta : zero_level;
    return imin(orc_select_rank(sigma, len, delta_eff, r_max), nsig);
}

/* tsmm.hpp:20-71 — Y = reshape(X V): product element (i,c) lands at flat
 * position p = i + n*c of the (out_rows x out_cols) padded output.  Per
 * element the accumulation order is j = 0..m-1 starting from 0.  Y's padding
 * is left untouched (the caller zero-fills, as PaddedMatrix does). */
int orc_tsmm_reshape(const double* X, idx n, idx m, idx ldx, const double* V, idx k, idx ldv, double* Y,
                     idx out_rows, idx out_cols, idx ldy) {
    if (k > m) return ORC_ERR_SHAPE;
    if (out_rows < 1 || out_cols < 1 || n * k != out_rows * out_cols) return ORC_ERR_SHAPE;
    double* acc = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    if (!acc) return ORC_ERR_ALLOCATION;
    for (idx c = 0; c < k; ++c) {
        for (idx i = 0; i < n; ++i) acc[i] = 0.0;
        for (idx j = 0; j < m; ++j) {
            const double vjc = V[c * ldv + j];
            const double* xj = X + j * ldx;
            for (idx i = 0; i < n; ++i) acc[i] += vjc * xj[i];
        }
        for (idx i = 0; i < n; ++i) {
            const idx p = i + n * c;
            Y[(p / out_rows) * ldy + p % out_rows] = acc[i];
        }
    }
    free(acc);
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * Drivers: run_chain / tt_svd_tsqr (tt_svd.hpp:159-199, 281-290) and
 * tt_svd_distributed (tt_svd.hpp:520-631).
 * Output: ranks[0..d], cores concatenated (core j is r_j x n_j x r_{j+1},
 * index a + r_j*(x + n_j*b)), per-step records and singular values.
 * ------------------------------------------------------------------------- */

typedef struct {
    idx rows, cols, nsig, rank;
} orc_step;

typedef struct {
    const double* data;
    idx rows, cols, ld;
} view_t;

/* svd_of_work, tt_svd.hpp:75-105: sigma (len nsig) and V (cols x nsig, ld cols). */
static int svd_of_work(view_t W, idx n_b_budget, int workers, double* sigma, double* V, idx* nsig) {
    int rc;
    if (W.rows >= W.cols) {
        const idx m = W.cols;
        double* R = (double*)malloc((size_t)(m * m) * sizeof(double));
        rc = orc_tsqr(W.data, W.rows, m, W.ld, orc_block_nb(m, n_b_budget), workers, R);
        if (rc == ORC_OK) rc = orc_small_svd(R, m, sigma, NULL, V);
        free(R);
        *nsig = m;
    } else {
        const idx rows = W.rows, cols = W.cols;
        double* wt = (double*)malloc((size_t)(rows * cols) * sizeof(double));
        for (idx j = 0; j < cols; ++j)
            for (idx i = 0; i < rows; ++i) wt[i * cols + j] = W.data[j * W.ld + i];
        double* vv = (double*)malloc((size_t)(rows * rows) * sizeof(double));
        rc = orc_jacobi_svd(wt, cols, rows, cols, sigma, V /* = U of W^T */, vv);
        free(vv);
        free(wt);
        *nsig = rows;
    }
    return rc;
}

static idx core_size(const idx* ranks, const idx* dims, idx j) { return ranks[j] * dims[j] * ranks[j + 1]; }

int orc_tt_svd_tsqr(const double* X, const idx* dims, idx d, idx ldx, idx r_max, double eps, int workers,
                    idx* ranks, double* cores, idx cores_cap, idx* cores_needed, orc_step* steps,
                    double* sigmas, idx sig_cap) {
    if (d < 2) return ORC_ERR_DEGENERATE;
    idx total = 1;
    for (idx i = 0; i < d; ++i) total *= dims[i];
    const idx n_d = dims[d - 1];
    view_t cur = {X, total / n_d, n_d, ldx};
    double delta = -1.0;
    idx r = 1;
    double* owned = NULL;
    /* per-core storage until the rank chain is known */
    double** cbuf = (double**)calloc((size_t)d, sizeof(double*));
    idx* cr = (idx*)calloc((size_t)(d + 1), sizeof(idx));
    cr[d] = 1;
    idx sig_used = 0;
    int rc = ORC_OK;
    for (idx i = d - 1; i >= 1; --i) {
        const idx n_i = dims[i];
        const idx m = n_i * r;
        const idx nsig_max = imin(cur.rows, cur.cols);
        double* sigma = (double*)malloc((size_t)imax(cur.cols, 1) * sizeof(double));
        double* V = (double*)malloc((size_t)(cur.cols * imax(nsig_max, 1)) * sizeof(double));
        idx nsig = 0;
        rc = svd_of_work(cur, 256 * 1024, workers, sigma, V, &nsig);
        if (rc != ORC_OK) {
            free(sigma); free(V);
            break;
        }
        if (delta < 0.0) {
            rc = orc_derive_delta(orc_sigma_norm(sigma, nsig), eps, d, &delta);
            if (rc != ORC_OK) { free(sigma); free(V); break; }
        }
        const idx rnew = orc_choose_rank(sigma, nsig, cur.cols, nsig, delta, r_max, cur.rows);
        if (steps) {
            steps[d - 1 - i].rows = cur.rows;
            steps[d - 1 - i].cols = m;
            steps[d - 1 - i].nsig = nsig;
            steps[d - 1 - i].rank = rnew;
        }
        if (sigmas) {
            for (idx q = 0; q < nsig && sig_used < sig_cap; ++q) sigmas[sig_used++] = sigma[q];
        }
        /* core_from_vt, tt_svd.hpp:121-128 */
        double* core = (double*)malloc((size_t)(rnew * n_i * r) * sizeof(double));
        for (idx b = 0; b < r; ++b)
            for (idx x = 0; x < n_i; ++x)
                for (idx a = 0; a < rnew; ++a) core[a + rnew * (x + n_i * b)] = V[a * cur.cols + (x + n_i * b)];
        cbuf[i] = core;
        cr[i] = rnew;
        const idx n_next = dims[i - 1];
        const idx out_rows = cur.rows / n_next;
        const idx out_cols = n_next * rnew;
        const idx ldy = orc_padded_stride(out_rows);
        double* next = (double*)calloc((size_t)(ldy * out_cols), sizeof(double));
        rc = orc_tsmm_reshape(cur.data, cur.rows, cur.cols, cur.ld, V, rnew, cur.cols, next, out_rows, out_cols, ldy);
        free(sigma); free(V);
        free(owned);
        owned = next;
        cur.data = next;
        cur.rows = out_rows;
        cur.cols = out_cols;
        cur.ld = ldy;
        r = rnew;
        if (rc != ORC_OK) break;
    }
    if (rc == ORC_OK) {
        /* T^(1): the final 1 x (n_1 r_1) work matrix, tt_svd.hpp:193-197 */
        double* first = (double*)malloc((size_t)(dims[0] * r) * sizeof(double));
        for (idx l = 0; l < dims[0] * r; ++l) first[l] = cur.data[(l / cur.rows) * cur.ld + l % cur.rows];
        cbuf[0] = first;
        cr[0] = 1;
        cr[1] = r;
        idx need = 0;
        for (idx j = 0; j < d; ++j) need += core_size(cr, dims, j);
        if (cores_needed) *cores_needed = need;
        for (idx j = 0; j <= d; ++j) ranks[j] = cr[j];
        if (need > cores_cap) rc = ORC_ERR_CAPACITY;
        else {
            idx off = 0;
            for (idx j = 0; j < d; ++j) {
                const idx sz = core_size(cr, dims, j);
                memcpy(cores + off, cbuf[j], (size_t)sz * sizeof(double));
                off += sz;
            }
        }
    }
    for (idx j = 0; j < d; ++j) free(cbuf[j]);
    free(cbuf); free(cr); free(owned);
    return rc;
}

/*
 * tt_svd.hpp:520-631 — in-process Alg. 5.  P slabs of identical local shape
 * (ldims[0..d_local-1], each stored in its own padded Fortran layout with
 * leading stride ld_slab); global tensor (P, ldims...), first core (1, P, r).
 * P == 1 degenerates to tt_svd_tsqr on the (1, ldims...) tensor (same buffer).
 */
int orc_tt_svd_distributed(const double* const* slabs, idx P, const idx* ldims, idx d_local, idx ld_slab, idx r_max,
                           double eps, int workers, idx* ranks, double* cores, idx cores_cap, idx* cores_needed,
                           orc_step* steps, double* sigmas, idx sig_cap) {
    if (P < 1) return ORC_ERR_PARTITION;
    const idx d = d_local + 1;
    idx* gdims = (idx*)malloc((size_t)d * sizeof(idx));
    gdims[0] = P;
    for (idx i = 0; i < d_local; ++i) gdims[i + 1] = ldims[i];
    if (P == 1) {
        gdims[0] = 1;
        const int rc = orc_tt_svd_tsqr(slabs[0], gdims, d, ld_slab, r_max, eps, workers, ranks, cores, cores_cap,
                                       cores_needed, steps, sigmas, sig_cap);
        free(gdims);
        return rc;
    }
    idx total = 1;
    for (idx i = 0; i < d_local; ++i) total *= ldims[i];
    view_t* cur = (view_t*)malloc((size_t)P * sizeof(view_t));
    double** owned = (double**)calloc((size_t)P, sizeof(double*));
    for (idx p = 0; p < P; ++p) {
        if (d_local == 1) {
            cur[p].data = slabs[p]; cur[p].rows = 1; cur[p].cols = ldims[0]; cur[p].ld = ld_slab;
        } else {
            cur[p].data = slabs[p]; cur[p].rows = total / ldims[d_local - 1];
            cur[p].cols = ldims[d_local - 1]; cur[p].ld = ld_slab;
        }
    }
    double** cbuf = (double**)calloc((size_t)d, sizeof(double*));
    idx* cr = (idx*)calloc((size_t)(d + 1), sizeof(idx));
    cr[d] = 1;
    double delta = -1.0;
    idx r = 1, sig_used = 0;
    int rc = ORC_OK;
    for (idx i = d_local - 1; i >= 0 && rc == ORC_OK; --i) {
        const idx n_i = ldims[i];
        const idx m = n_i * r;
        double* parts = (double*)calloc((size_t)(P * m * m), sizeof(double));
        idx global_rows = 0;
        for (idx p = 0; p < P && rc == ORC_OK; ++p) {
            global_rows += cur[p].rows;
            /* gram_triangular, tt_svd.hpp:204-210 */
            if (cur[p].rows >= cur[p].cols) {
                rc = orc_tsqr(cur[p].data, cur[p].rows, m, cur[p].ld, orc_block_nb(m, 256 * 1024), workers,
                              parts + p * m * m);
            } else {
                const idx ldq = orc_padded_stride(m);
                double* sq = (double*)calloc((size_t)(ldq * m), sizeof(double));
                for (idx j = 0; j < m; ++j)
                    for (idx q = 0; q < cur[p].rows; ++q) sq[j * ldq + q] = cur[p].data[j * cur[p].ld + q];
                rc = orc_tsqr(sq, m, m, ldq, orc_block_nb(m, 256 * 1024), workers, parts + p * m * m);
                free(sq);
            }
        }
        double* R = (double*)malloc((size_t)(m * m) * sizeof(double));
        if (rc == ORC_OK) rc = orc_combine_factors(parts, P, m, R);
        free(parts);
        double* sigma = (double*)malloc((size_t)m * sizeof(double));
        double* V = (double*)malloc((size_t)(m * m) * sizeof(double));
        if (rc == ORC_OK) rc = orc_small_svd(R, m, sigma, NULL, V);
        free(R);
        if (rc != ORC_OK) { free(sigma); free(V); break; }
        const idx nsig = imin(m, global_rows);
        if (delta < 0.0) orc_derive_delta(orc_sigma_norm(sigma, m), eps, d, &delta);
        const idx rnew = orc_choose_rank(sigma, m, m, nsig, delta, r_max, global_rows);
        if (steps) {
            steps[d_local - 1 - i].rows = global_rows;
            steps[d_local - 1 - i].cols = m;
            steps[d_local - 1 - i].nsig = nsig;
            steps[d_local - 1 - i].rank = rnew;
        }
        if (sigmas)
            for (idx q = 0; q < m && sig_used < sig_cap; ++q) sigmas[sig_used++] = sigma[q];
        double* core = (double*)malloc((size_t)(rnew * n_i * r) * sizeof(double));
        for (idx b = 0; b < r; ++b)
            for (idx x = 0; x < n_i; ++x)
                for (idx a = 0; a < rnew; ++a) core[a + rnew * (x + n_i * b)] = V[a * m + (x + n_i * b)];
        cbuf[i + 1] = core;
        cr[i + 1] = rnew;
        for (idx p = 0; p < P && rc == ORC_OK; ++p) {
            const idx out_rows = i >= 1 ? cur[p].rows / ldims[i - 1] : 1;
            const idx out_cols = i >= 1 ? ldims[i - 1] * rnew : rnew;
            const idx ldy = orc_padded_stride(out_rows);
            double* next = (double*)calloc((size_t)(ldy * out_cols), sizeof(double));
            rc = orc_tsmm_reshape(cur[p].data, cur[p].rows, cur[p].cols, cur[p].ld, V, rnew, m, next, out_rows,
                                  out_cols, ldy);
            free(owned[p]);
            owned[p] = next;
            cur[p].data = next; cur[p].rows = out_rows; cur[p].cols = out_cols; cur[p].ld = ldy;
        }
        free(sigma); free(V);
        r = rnew;
    }
    if (rc == ORC_OK) {
        double* first = (double*)malloc((size_t)(P * r) * sizeof(double));
        for (idx p = 0; p < P; ++p)
            for (idx b = 0; b < r; ++b) first[p + P * b] = cur[p].data[b * cur[p].ld];
        cbuf[0] = first;
        cr[0] = 1;
        idx need = 0;
        for (idx j = 0; j < d; ++j) need += core_size(cr, gdims, j);
        if (cores_needed) *cores_needed = need;
        for (idx j = 0; j <= d; ++j) ranks[j] = cr[j];
        if (need > cores_cap) rc = ORC_ERR_CAPACITY;
        else {
            idx off = 0;
            for (idx j = 0; j < d; ++j) {
                const idx sz = core_size(cr, gdims, j);
                memcpy(cores + off, cbuf[j], (size_t)sz * sizeof(double));
                off += sz;
            }
        }
    }
    for (idx j = 0; j < d; ++j) free(cbuf[j]);
    for (idx p = 0; p < P; ++p) free(owned[p]);
    free(cbuf); free(cr); free(owned); free(cur); free(gdims);
    return rc;
}

/* tensor_train.hpp:80-110 — left-to-right contraction into a flat
 * (unpadded, column-major) buffer of prod(dims) entries. */
int orc_tt_reconstruct(const idx* dims, idx d, const idx* ranks, const double* cores, double* out) {
    if (d < 1 || ranks[0] != 1 || ranks[d] != 1) return ORC_ERR_DIMENSION_MISMATCH;
    idx total = 1;
    for (idx j = 0; j < d; ++j) total *= dims[j];
    /* M: N x r col-major; starts as core 0 (1 x n_0 x r_1 == n_0 x r_1) */
    idx N = dims[0];
    idx off = core_size(ranks, dims, 0);
    double* M = (double*)malloc((size_t)(N * ranks[1]) * sizeof(double));
    memcpy(M, cores, (size_t)(N * ranks[1]) * sizeof(double));
    for (idx j = 1; j < d; ++j) {
        const double* c = cores + off;
        const idx rl = ranks[j], n = dims[j], rr = ranks[j + 1];
        const idx nc = n * rr; /* horizontal unfolding rl x (n*rr), ld rl */
        double* next = (double*)calloc((size_t)(N * nc), sizeof(double));
        for (idx cc = 0; cc < nc; ++cc) {
            double* dst = next + cc * N;
            for (idx l = 0; l < rl; ++l) {
                const double h = c[cc * rl + l];
                if (h == 0.0) continue;
                const double* src = M + l * N;
                for (idx i = 0; i < N; ++i) dst[i] += h * src[i];
            }
        }
        free(M);
        M = next;
        N *= n;
        off += core_size(ranks, dims, j);
    }
    memcpy(out, M, (size_t)total * sizeof(double));
    free(M);
    return ORC_OK;
}

/* tensor_train.hpp:113-124 — ||X - TT|| / ||X||, X in its padded layout
 * (rows = total / n_d, leading stride ldx). */
double orc_tt_error(const double* X, idx ldx, const idx* dims, idx d, const idx* ranks, const double* cores) {
    idx total = 1;
    for (idx j = 0; j < d; ++j) total *= dims[j];
    const idx rows = total / dims[d - 1];
    double* Y = (double*)malloc((size_t)total * sizeof(double));
    if (orc_tt_reconstruct(dims, d, ranks, cores, Y) != ORC_OK) {
        free(Y);
        return -1.0;
    }
    double diff = 0.0, nrm = 0.0;
    for (idx l = 0; l < total; ++l) {
        const double x = X[(l / rows) * ldx + l % rows];
        const double e = x - Y[l];
        diff += e * e;
        nrm += x * x;
    }
    free(Y);
    return sqrt(diff) / sqrt(nrm);
}

/* Restatement of the counter-based input generator of the device path
 * (paper_2102_00104_b200/csrc/ttsvd_kernels.cuh, gen_uniform): entry l of a
 * seeded stream is (splitmix64(seed + (l+1)*golden) >> 11) * 2^-53 mapped to
 * 2u-1 in [-1, 1); both steps are exact in fp64, so host and device agree
 * bitwise.  The flat index l is the Fortran (column-major) order; the buffer
 * is written in the padded layout (rows, ld). */
static uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void orc_gen_uniform(uint64_t seed, idx total, idx rows, idx ld, double* out) {
    for (idx l = 0; l < total; ++l) {
        const uint64_t z = splitmix64(seed + (uint64_t)(l + 1) * 0x9E3779B97F4A7C15ULL);
        const double u = (double)(z >> 11) * 0x1.0p-53;
        out[(l / rows) * ld + l % rows] = 2.0 * u - 1.0;
    }
}

/* ---------------------------------------------------------------------------
 * Test-input generators of the reference, restated so the reference tests'
 * exact inputs can be regenerated without the reference present:
 *   std::mt19937_64 (the C++ standard's published parameters),
 *   random_tensor       storage.hpp:202-212  ((eng() >> 11) * 2^-53 in [0,1))
 *   oracles::gaussian   tests/oracles.hpp:75-83 (Box-Muller on (x+0.5)*2^-53)
 *   oracles::uniform    tests/oracles.hpp:85-90
 *   oracles::random_tt  tests/oracles.hpp:144-154 (entries in [-0.5, 0.5))
 * ------------------------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64_t;

static void mt64_seed(mt64_t* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64_t* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* random_tensor: Fortran flat order into the padded layout (rows, ld) */
void orc_random_tensor(uint64_t seed, idx total, idx rows, idx ld, double* out) {
    mt64_t g;
    mt64_seed(&g, seed);
    for (idx l = 0; l < total; ++l) out[(l / rows) * ld + l % rows] = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
}

void orc_mt_gaussian(uint64_t seed, idx count, double* out) {
    mt64_t g;
    mt64_seed(&g, seed);
    for (idx i = 0; i < count; ++i) {
        const double u1 = ((double)(mt64_next(&g) >> 11) + 0.5) * 0x1.0p-53;
        const double u2 = ((double)(mt64_next(&g) >> 11) + 0.5) * 0x1.0p-53;
        out[i] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    }
}

void orc_mt_uniform(uint64_t seed, idx count, double shift, double* out) {
    mt64_t g;
    mt64_seed(&g, seed);
    for (idx i = 0; i < count; ++i) out[i] = (double)(mt64_next(&g) >> 11) * 0x1.0p-53 + shift;
}

/* Diagnostics: sweeps the cyclic one-sided Jacobi needs on A (n x m). */
int orc_jacobi_sweeps(const double* A, idx n, idx m, idx lda) {
    double* a = (double*)malloc((size_t)(n * m + m * m) * sizeof(double));
    for (idx j = 0; j < m; ++j)
        for (idx i = 0; i < n; ++i) a[j * n + i] = A[j * lda + i];
    double* v = a + n * m;
    for (idx i = 0; i < m * m; ++i) v[i] = 0.0;
    const double tol = 1e2 * DBL_EPSILON;
    int sweep = 0;
    for (; sweep < 60; ++sweep) {
        int rotated = 0;
        for (idx p = 0; p < m - 1; ++p)
            for (idx q = p + 1; q < m; ++q) {
                double* ap = a + p * n;
                double* aq = a + q * n;
                double al = 0, be = 0, ga = 0;
                for (idx i = 0; i < n; ++i) { al += ap[i] * ap[i]; be += aq[i] * aq[i]; ga += ap[i] * aq[i]; }
                if (fabs(ga) <= tol * sqrt(al * be)) continue;
                rotated = 1;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = ((zeta >= 0.0) ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (idx i = 0; i < n; ++i) { const double x = ap[i], y = aq[i]; ap[i] = c * x - s * y; aq[i] = s * x + c * y; }
            }
        if (!rotated) break;
    }
    free(a);
    return sweep;
}
