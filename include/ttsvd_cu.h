/*
 * ttsvd_cu.h — the drop-in C-ABI of the B200-native TT-SVD hot path.
 *
 * Reference: arXiv 2102.00104, /root/reference/proj/include/ttsvd/ (the .hpp headers) (a
 * header-only C++20 CPU library).  Each entry point below replaces one
 * reference function; the citation names the function it stands in for.  The
 * C++ host mirror (include/ttsvd_b200.hpp) keeps the reference's own names
 * and signatures on top of this ABI, and INTEGRATION.md shows how a
 * maintainer binds it.
 *
 * Conventions (the reference's layout contract, storage.hpp:28-45):
 *   - matrices are column-major, element (i,j) at data[j*ld + i];
 *   - a DenseTensor of shape (n_1..n_d) is stored as its (N/n_d) x n_d
 *     matricization with ld = padded_stride(N/n_d) (shape.hpp:22-28,
 *     storage.hpp:82-115);
 *   - all double* arguments are DEVICE pointers unless the name ends in _host;
 *   - every call is stream-ordered on the context's stream and returns a
 *     status code; nothing throws across the boundary.  Calls that return
 *     host-visible results (ranks, cores, rank, ...) synchronise first.
 *   - `workers` and `BlockParams` of the reference have no meaning on the
 *     GPU; results are deterministic for a fixed (shape, device) instead.
 */
#ifndef TTSVD_CU_H
#define TTSVD_CU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the C++ mirror maps them onto the errors.hpp:9-62 tree. */
enum {
    TTSVD_OK = 0,
    TTSVD_ERR_DIMENSION = 1,          /* DimensionError      (tsqr.hpp:250-251)  */
    TTSVD_ERR_DIMENSION_MISMATCH = 2, /* DimensionMismatch   (tsqr.hpp:213,233)  */
    TTSVD_ERR_SHAPE = 3,              /* ShapeError          (tsmm.hpp:23-26)    */
    TTSVD_ERR_CONVERGENCE = 4,        /* ConvergenceError    (small_svd.hpp:113) */
    TTSVD_ERR_ALLOCATION = 5,         /* AllocationError     (storage.hpp:22-26) */
    TTSVD_ERR_DEGENERATE = 6,         /* DegenerateDimension (tt_svd.hpp:283)    */
    TTSVD_ERR_PARTITION = 7,          /* PartitionMismatch   (tt_svd.hpp:523-526)*/
    TTSVD_ERR_DEVICE = 8,             /* CUDA / exchange failure (new)          */
    TTSVD_ERR_INVALID = 9,            /* null pointer / bad argument            */
    TTSVD_ERR_LAYOUT = 10             /* LayoutError         (storage.hpp:134)   */
};

typedef struct ttsvd_cu_ctx ttsvd_cu_ctx; /* device, stream, workspace, counters */
typedef struct ttsvd_cu_tt ttsvd_cu_tt;   /* a TensorTrain result (tensor_train.hpp:42-77) */

/* Per-step record, the counterpart of StepRecord (tt_svd.hpp:21-26). */
typedef struct {
    int64_t rows, cols, nsig, rank;
    double t_tsqr_ms, t_svd_ms, t_tsmm_ms; /* device time, CUDA events */
    double t_tsqr_sweep_ms;                /* the TSQR's main sweep kernel alone (no merge) */
    int32_t tsqr_kernel;                   /* which: TTSVD_K_* below */
    int32_t svd_sweeps;                    /* Jacobi sweeps of the step's small SVD */
    double t_reorder_ms;                   /* two-sided sweep: transpose_reorder (StepRecord::t_reorder) */
} ttsvd_cu_step;

/* tsqr_kernel values (diagnostics) */
enum {
    TTSVD_K_NONE = 0,
    TTSVD_K_WS = 1,    /* warp streams, m <= 32 */
    TTSVD_K_V1 = 2,    /* block-per-job tiles, m <= 32 */
    TTSVD_K_LA = 3,    /* 32-row look-ahead tiles */
    TTSVD_K_T128 = 4,  /* 128-row tiles, one CTA per SM */
    TTSVD_K_GQR = 5,   /* cooperative whole-grid QR */
    TTSVD_K_PT = 6,    /* thread streams, m <= 8 */
    TTSVD_K_GS = 7,    /* lane-group streams, 8 < m <= 32 */
    TTSVD_K_SQ = 8,    /* levels of single 256-row tiles (tsqr_t128_kernel), 32 < m <= 64, small n */
    TTSVD_K_GT = 9     /* lane-group streams fed by TMA bulk copies, 8 < m <= 32, tall */
};

/* All-gather over the ranks of a distributed run (replaces the in-process
 * combine over partitions at tt_svd.hpp:568-575; Alg. 5's MPI_Allreduce,
 * PAPER.md:389-392).  recv receives count doubles from every rank, in rank
 * order.  Called stream-ordered on `stream`; returns 0 on success. */
typedef int (*ttsvd_cu_exchange_fn)(void* user, const double* send, double* recv, int64_t count, void* stream);

/* ---- context ----------------------------------------------------------- */
const char* ttsvd_cu_version(void);
const char* ttsvd_cu_last_error(void); /* message of the last failing call on this thread */
int ttsvd_cu_ctx_create(int device, void* stream, ttsvd_cu_ctx** out);
int ttsvd_cu_ctx_destroy(ttsvd_cu_ctx* ctx);
int ttsvd_cu_ctx_set_stream(ttsvd_cu_ctx* ctx, void* stream);
int ttsvd_cu_synchronize(ttsvd_cu_ctx* ctx);
/* number of kernels this context has launched since creation */
int64_t ttsvd_cu_ctx_launches(const ttsvd_cu_ctx* ctx);
/* enable per-phase CUDA-event timing in ttsvd_cu_step (off by default) */
int ttsvd_cu_ctx_set_timing(ttsvd_cu_ctx* ctx, int on);

/* shape.hpp:22-28 */
int64_t ttsvd_cu_padded_stride(int64_t n_rows);

/* ---- building blocks (device pointers) --------------------------------- */
/* tsqr.hpp:247 tsqr(): R (m x m, ld m, exact-zero strict lower triangle) with
 * R^T R = X^T X; X (n x m, ld ldx) is read exactly once, Q is never formed. */
int ttsvd_cu_tsqr(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int64_t m, int64_t ldx, double* R);
/* tsqr.hpp:208 reduce_block(): R_out^T R_out = M^T M + R_in^T R_in. */
int ttsvd_cu_reduce_block(ttsvd_cu_ctx* ctx, const double* M, int64_t rows, int64_t m, int64_t ldm,
                          const double* R_in, int64_t r_m, double* R_out);
/* tsqr.hpp:230 combine_factors(): P triangles (P*m*m, each ld m), merged in a
 * fixed index-ordered tree. */
int ttsvd_cu_combine_factors(ttsvd_cu_ctx* ctx, const double* parts, int64_t P, int64_t m, double* R);
/* small_svd.hpp:196 small_svd(): sigma[m] non-increasing, V (m x m, ld m). */
int ttsvd_cu_small_svd(ttsvd_cu_ctx* ctx, const double* R, int64_t m, double* sigma, double* V);
/* small_svd.hpp:120 jacobi_svd() of A (n x m, n >= m): sigma[m], V (m x m)
 * and, if U != NULL, U (n x m, ld n) with the reference's deterministic
 * completion for sigma <= n*eps*sigma_1. */
int ttsvd_cu_jacobi_svd(ttsvd_cu_ctx* ctx, const double* A, int64_t n, int64_t m, int64_t lda, double* sigma,
                        double* V, double* U);
/* The TT-SVD driver's SVD of a work matrix A (n x m, n >= m, device, ld lda;
 * tt_svd.hpp:85-110 calls small_svd on R / W and keeps the leading r right
 * singular vectors): sigma (m, non-increasing) and the leading r left
 * singular vectors of A (V: n x r, ld n).  Bidiagonalisation + bisection +
 * twisted factorisation when A fits a 16-CTA cluster (64 <= m), else block
 * Jacobi.  *path_out (optional): 1 bidiagonal, 0 Jacobi. */
int ttsvd_cu_driver_svd(ttsvd_cu_ctx* ctx, const double* A, int64_t n, int64_t m, int64_t lda, int64_t r,
                        double* sigma, double* V, int32_t* path_out);
/* small_svd.hpp:49 select_rank() on a device sigma; the rank is returned on the host. */
int ttsvd_cu_select_rank(ttsvd_cu_ctx* ctx, const double* sigma, int64_t m, double delta, int64_t r_max,
                         int64_t* rank_host);
/* small_svd.hpp:49 select_rank() on a host sigma (pure host arithmetic). */
int64_t ttsvd_cu_select_rank_host(const double* sigma_host, int64_t m, double delta, int64_t r_max);
/* small_svd.hpp:41 derive_delta() (host arithmetic, kept for completeness). */
int ttsvd_cu_derive_delta(double norm_source, double eps, int64_t d, double* delta_host);
/* tsmm.hpp:20 tsmm_reshape(): Y (out_rows x out_cols, ld ldy >= out_rows)
 * receives reshape(X V[:, :k]); product element (i,c) lands at flat position
 * i + n*c.  Padding rows out_rows..ldy-1 are zeroed. */
int ttsvd_cu_tsmm_reshape(ttsvd_cu_ctx* ctx, const double* X, int64_t n, int64_t m, int64_t ldx, const double* V,
                          int64_t k, int64_t ldv, double* Y, int64_t out_rows, int64_t out_cols, int64_t ldy);

/* ---- drivers ----------------------------------------------------------- */
/* tt_svd.hpp:281 tt_svd_tsqr() (Alg. 2): X is the device tensor in the padded
 * layout (ldx = padded_stride(N/n_d) or larger).  r_max is the reference's
 * TruncationSpec::r_max: INT64_MAX is uncapped, r_max < 1 clamps every rank to 1
 * (select_rank, small_svd.hpp:49-63). */
int ttsvd_cu_tt_svd(ttsvd_cu_ctx* ctx, const double* X, const int64_t* dims, int64_t d, int64_t ldx, int64_t r_max,
                    double eps, ttsvd_cu_tt** out);
/* tt_svd.hpp:159-199 detail::run_chain(): the Alg. 2 loop on a work matrix W
 * (rows x cols, device, ld ldw) that is the last-mode matricization of a
 * tensor with extents dims[0..d-1].  *delta_io < 0 derives the truncation
 * parameter from the first step's sigma with d_for_delta modes and writes it
 * back (run_chain takes the TruncationSpec by reference, tt_svd.hpp:160);
 * first_sigma_norm_out (optional) receives ChainResult::first_sigma_norm. */
int ttsvd_cu_run_chain(ttsvd_cu_ctx* ctx, const double* W, int64_t rows, int64_t cols, int64_t ldw, const int64_t* dims,
                       int64_t d, int64_t r_max, double eps, int64_t d_for_delta, double* delta_io,
                       double* first_sigma_norm_out, ttsvd_cu_tt** out);
/* tt_svd.hpp:402-512 tt_svd_two_sided() (Alg. 4): alternating right / left
 * steps with a transpose_reorder between them; same arguments as
 * ttsvd_cu_tt_svd. */
int ttsvd_cu_tt_svd_two_sided(ttsvd_cu_ctx* ctx, const double* X, const int64_t* dims, int64_t d, int64_t ldx,
                              int64_t r_max, double eps, ttsvd_cu_tt** out);
/* tsmm.hpp:84-126 transpose_reorder(): Y (out_rows x out_cols, ld ldy) holds
 * the column-major flat order of W^T (W: n x m, ld ldw), i.e. W(i, j) lands at
 * flat position m*i + j; padding rows out_rows..ldy-1 are zeroed. */
int ttsvd_cu_transpose_reorder(ttsvd_cu_ctx* ctx, const double* W, int64_t n, int64_t m, int64_t ldw, double* Y,
                               int64_t out_rows, int64_t out_cols, int64_t ldy);
/* tt_svd.hpp:316-330 choose_combined_dims() with ThickBoundsParams
 * (tt_svd.hpp:292-310): k trailing modes merged into one of extent m.
 * r_tilde may be NULL (n_r_tilde = 0): the estimates default to r_max
 * (INT64_MAX: uncapped). */
int ttsvd_cu_choose_combined_dims(const int64_t* dims, int64_t d, int64_t m_min, double f1_min, const int64_t* r_tilde,
                                  int64_t n_r_tilde, int64_t r_max, int64_t* k_out, int64_t* m_out);
/* tt_svd.hpp:338 tt_svd_thick_bounds() (Alg. 3): merge the k trailing modes,
 * run the TSQR sweep on the merged tensor, recover the k boundary cores from
 * the combined core with the rescaled delta.  k == 1 is the plain driver. */
int ttsvd_cu_tt_svd_thick(ttsvd_cu_ctx* ctx, const double* X, const int64_t* dims, int64_t d, int64_t ldx,
                          int64_t r_max, double eps, int64_t m_min, double f1_min, const int64_t* r_tilde,
                          int64_t n_r_tilde, ttsvd_cu_tt** out);
/* ttsvd_cu_tt_svd from a HOST buffer (pinned or pageable, the same padded
 * layout): the H2D copy is part of the call — this is the reference-facing
 * end-to-end entry (tt_svd_tsqr(const DenseTensor&), tt_svd.hpp:281-290).
 * When the first step runs on the TMA-staged stream kernel, X is copied in
 * row chunks on a second stream and every chunk is folded as soon as it has
 * landed, so the first TSQR runs under the transfer; the result is
 * bit-identical to ttsvd_cu_tt_svd on the uploaded tensor. */
int ttsvd_cu_tt_svd_host(ttsvd_cu_ctx* ctx, const double* X_host, const int64_t* dims, int64_t d, int64_t ldx,
                         int64_t r_max, double eps, ttsvd_cu_tt** out);
/* ttsvd_cu_tt_svd_thick from a HOST buffer (tt_svd_thick_bounds(const
 * DenseTensor&), tt_svd.hpp:338).  When the merged first step runs on the
 * tall-tile kernel, X arrives in row chunks of the merged matricization and
 * each chunk is folded as it lands (per-CTA factors carried between the
 * launches): the dominant TSQR of Alg. 3 runs under the H2D.  Same algorithm
 * as the device entry with other tile boundaries: equal within rounding, not
 * bit for bit. */
int ttsvd_cu_tt_svd_thick_host(ttsvd_cu_ctx* ctx, const double* X_host, const int64_t* dims, int64_t d, int64_t ldx,
                               int64_t r_max, double eps, int64_t m_min, double f1_min, const int64_t* r_tilde,
                               int64_t n_r_tilde, ttsvd_cu_tt** out);
/* tt_svd.hpp:520 tt_svd_distributed() (Alg. 5).  This process owns n_slabs
 * slabs (device pointers, each the padded layout of the local shape ldims,
 * leading stride ld_slab) which are global partitions part0 .. part0+n_slabs-1
 * of P_total.  With n_slabs == P_total no exchange is needed (exchange may be
 * NULL, the reference's in-process form); otherwise `exchange` all-gathers the
 * per-process R factors.  The global tensor is (P_total, ldims...) with the
 * partition index fastest; the result's first core is (1, P_total, r). */
int ttsvd_cu_tt_svd_distributed(ttsvd_cu_ctx* ctx, const double* const* slabs, int64_t n_slabs, int64_t part0,
                                int64_t P_total, const int64_t* ldims, int64_t d_local, int64_t ld_slab,
                                int64_t r_max, double eps, ttsvd_cu_exchange_fn exchange, void* user,
                                ttsvd_cu_tt** out);

/* ---- multi-GPU: NCCL inside the library --------------------------------- */
/* Replaces the in-process combine of tt_svd.hpp:568-575 across GPUs (Alg. 5's
 * MPI_Allreduce, becomes an all-gather of the R factors +
 * the pinned-order merge).  libnccl.so.2 is loaded on first use. */
#define TTSVD_COMM_ID_BYTES 128
/* a fresh NCCL unique id (128 bytes) — create on one rank, broadcast it */
int ttsvd_cu_comm_unique_id(void* id_out);
/* one process per GPU: attach an NCCL communicator (nranks, rank) to ctx.
 * ttsvd_cu_tt_svd_distributed with exchange == NULL then all-gathers over it
 * on the context's stream; rank k must own partitions k*n_slabs .. */
int ttsvd_cu_ctx_comm_init(ttsvd_cu_ctx* ctx, const void* unique_id, int nranks, int rank);
/* one process driving ndev GPUs (one context per device): ncclCommInitAll */
int ttsvd_cu_ctx_comm_init_all(ttsvd_cu_ctx* const* ctxs, int ndev);
/* Alg. 5 over ndev GPUs of this process, one host thread per device: device i
 * owns slabs[i*slabs_per_device ..] (device pointers on that device, each the
 * padded layout of ldims with leading stride ld_slab).  Needs
 * ttsvd_cu_ctx_comm_init_all on ctxs.  Result as ttsvd_cu_tt_svd_distributed
 * (first core (1, P, r), P = ndev * slabs_per_device). */
int ttsvd_cu_tt_svd_distributed_devices(ttsvd_cu_ctx* const* ctxs, int ndev, const double* const* slabs,
                                        int64_t slabs_per_device, const int64_t* ldims, int64_t d_local,
                                        int64_t ld_slab, int64_t r_max, double eps, ttsvd_cu_tt** out);

/* ---- results ----------------------------------------------------------- */
int64_t ttsvd_cu_tt_d(const ttsvd_cu_tt* tt);
int ttsvd_cu_tt_ranks(const ttsvd_cu_tt* tt, int64_t* ranks /* d+1 */);
/* core j as r_j x n_j x r_{j+1}, index a + r_j*(x + n_j*b) (tensor_train.hpp:24-29) */
int ttsvd_cu_tt_core(const ttsvd_cu_tt* tt, int64_t j, double* dst_host);
int64_t ttsvd_cu_tt_nsteps(const ttsvd_cu_tt* tt);
int ttsvd_cu_tt_step(const ttsvd_cu_tt* tt, int64_t s, ttsvd_cu_step* out);
/* singular values of step s (nsig of them) */
int ttsvd_cu_tt_sigma(const ttsvd_cu_tt* tt, int64_t s, double* dst_host);
void ttsvd_cu_tt_free(ttsvd_cu_tt* tt);

/* ---- synthetic inputs (off the timed path) ------------------------------ */
/* Counter-based uniform[-1,1) tensor (restated bit-exactly in the oracle). */
int ttsvd_cu_gen_uniform(ttsvd_cu_ctx* ctx, uint64_t seed, int64_t total, int64_t rows, int64_t ld, double* X);
/* Partition `part` of `nparts` of a counter-based tensor: local flat entry l
 * is global entry part + nparts*l (split_first_dim, ttsvd_bench.cpp:72-86), so
 * every partition count generates the same global tensor.  kind 0: X = 2u-1
 * (gen_uniform when nparts == 1); kind 1: X += scale * N(0,1) (Box-Muller). */
int ttsvd_cu_gen_partition(ttsvd_cu_ctx* ctx, uint64_t seed, int kind, double scale, int64_t total_local,
                           int64_t rows, int64_t ld, int64_t nparts, int64_t part, double* X);

#ifdef __cplusplus
}
#endif
#endif /* TTSVD_CU_H */
