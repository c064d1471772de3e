"""GPU parity of the building blocks through the C-ABI, against the oracle.

Mirrors /root/reference/proj/tests/test_tsqr.cpp, test_small_svd.cpp,
test_tsmm.cpp and acceptance C04/C05.  Tolerances (north_star): Gram residual
<= 1e-12 relative (C04), singular values |dsigma| <= 1e-10 sigma_1 (C05),
TSMM <= 1e-13 ||Y|| (test_tsmm.cpp:40-49), column selection bit-exact.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2102_00104_b200 as tt
    return tt


def host(T):
    return T.detach().cpu().numpy()


def gram_resid(X, R):
    gx = X.T @ X
    return float(np.linalg.norm(R.T @ R - gx) / np.linalg.norm(gx))


# ------------------------------------------------------------------ tsqr ----
def test_reduce_block_hand_householder(tt):
    # test_tsqr.cpp:28-36 — M = [3;4], R = [0] -> |Rbar| = 5.  The reference
    # pivots on M's row (u1 = 3 > 0 gives -5); the device kernel pivots on the
    # R diagonal of the stacked [R; M] (0 gives +5).  R is unique up to row
    # signs, and every consumer (small SVD, TT cores) is sign-gauge invariant.
    rb = host(tt.reduce_block(np.array([[3.0], [4.0]]), np.zeros((1, 1))))
    assert abs(abs(rb[0, 0]) - 5.0) <= 1e-14


def test_reduce_block_zero_block_keeps_triangle(tt):
    # test_tsqr.cpp:38-44
    rb = host(tt.reduce_block(np.zeros((5, 1)), np.array([[2.0]])))
    assert rb[0, 0] == 2.0


def test_reduce_block_gram_preservation(tt):
    # test_tsqr.cpp:46-63
    from oracle.oracle import gaussian
    m = gaussian(8, 3, 42)
    rt = gaussian(3, 3, 43)
    r = np.triu(rt)
    rb = host(tt.reduce_block(m, r))
    expect = m.T @ m + r.T @ r
    assert np.linalg.norm(rb.T @ rb - expect) <= 1e-13 * np.linalg.norm(expect)
    assert np.all(np.tril(rb, -1) == 0.0)


def test_reduce_block_dimension_mismatch(tt):
    with pytest.raises(tt.DimensionMismatch):
        tt.reduce_block(np.zeros((4, 3)), np.zeros((2, 2)))


def test_tsqr_embedded_identity(tt):
    # test_tsqr.cpp:71-79
    x = np.zeros((100, 4))
    x[:4, :4] = np.eye(4)
    r = host(tt.tsqr(x))
    assert np.allclose(np.abs(np.diag(r)), 1.0, atol=1e-14)
    assert np.all(np.abs(np.triu(r, 1)) <= 1e-15)


@pytest.mark.parametrize("n,m", [(100000, 8), (1000, 1), (64, 64), (65, 64), (3000, 17), (20000, 32), (5000, 100),
                                 (4096, 256), (700, 512)])
def test_tsqr_gram_property(tt, n, m):
    from oracle.oracle import gaussian
    X = gaussian(n, m, 7 + m)
    R = host(tt.tsqr(X))
    assert np.all(np.isfinite(R))
    assert np.all(np.tril(R, -1) == 0.0)
    assert gram_resid(X, R) <= 1e-12


# The wide-factor kernels: 32-row look-ahead tiles (tsqr_la_kernel, n below
# 4 x 128 rows per SM) and 128-row tiles (tsqr_t128_kernel), including partial
# tiles, m not a multiple of 32, zero and duplicated columns and low rank.
# (40000, 150) and (50000, 200): the cooperative short-fat kernel with more
# than 256 rows per CTA (512 threads, a row each).
@pytest.mark.parametrize("n,m,kind", [(40000, 96, "dense"), (30011, 45, "dup"), (80000, 64, "dense"),
                                      (90001, 45, "dup"), (77777, 130, "lowrank"), (160000, 256, "dense"),
                                      (40000, 150, "dense"), (40000, 150, "dup"), (50000, 200, "lowrank")])
def test_tsqr_wide_kernels(tt, n, m, kind):
    from oracle.oracle import gaussian
    X = gaussian(n, m, 31 + m).copy(order="F")
    if kind == "dup":
        X[:, m - 1] = X[:, 0]
        X[:, m // 2] = 0.0
    if kind == "lowrank":
        X = np.asfortranarray(gaussian(n, 7, 5) @ gaussian(7, m, 6))
    R = host(tt.tsqr(X))
    assert np.all(np.isfinite(R))
    assert np.all(np.tril(R, -1) == 0.0)
    assert gram_resid(X, R) <= 1e-12
    s_r = np.linalg.svd(R, compute_uv=False)
    s_x = np.linalg.svd(X, compute_uv=False)
    assert np.max(np.abs(s_r - s_x)) <= 1e-10 * s_x[0]
    if kind != "dense":
        rank = 7 if kind == "lowrank" else m - 2
        assert s_r[rank] <= 1e-13 * s_r[0]
    # the same bytes give the same R (fixed reduction orders; a race in the
    # register-panel exchanges would show here)
    assert np.array_equal(host(tt.tsqr(X)), R)


# The register tile levels (tsqr_t128_kernel with one tile per CTA, 32 < m <= 64, n <= 2^16: 256-row
# tile QRs, their stacked factors the next level's rows): partial tiles, one to five levels, zero / duplicated columns, low
# rank and subnormal squares.
@pytest.mark.parametrize("n,m,kind", [(40, 33, "dense"), (64, 64, "dense"), (65, 33, "dup"), (256, 64, "dense"),
                                      (257, 48, "lowrank"), (1000, 64, "tiny"), (4096, 64, "dup"),
                                      (16384, 64, "dense"), (65536, 40, "dense"), (50001, 63, "dup")])
def test_tsqr_register_tiles(tt, n, m, kind):
    from oracle.oracle import gaussian
    X = gaussian(n, m, 51 + m).copy(order="F")
    if kind == "dup":
        X[:, m - 1] = X[:, 0]
        X[:, 1] = 0.0
    if kind == "lowrank":
        X = np.asfortranarray(gaussian(n, 3, 5) @ gaussian(3, m, 6))
    if kind == "tiny":
        X[:, 3] *= 1e-156
        X[:, 40] = 0.0
    R = host(tt.tsqr(X))
    assert np.all(np.isfinite(R))
    assert np.all(np.tril(R, -1) == 0.0)
    assert gram_resid(X, R) <= 1e-12
    s_r = np.linalg.svd(R, compute_uv=False)
    s_x = np.linalg.svd(X, compute_uv=False)
    assert np.max(np.abs(s_r - s_x)) <= 1e-10 * s_x[0]
    if kind in ("dup", "lowrank"):
        rank = 3 if kind == "lowrank" else m - 2
        assert s_r[rank] <= 1e-13 * s_r[0]
    cn_r, cn_x = np.linalg.norm(R, axis=0), np.linalg.norm(X, axis=0)
    assert np.allclose(cn_r, cn_x, rtol=1e-6 if kind == "tiny" else 1e-12, atol=1e-150)
    assert np.array_equal(host(tt.tsqr(X)), R)


# The thread-stream kernel (tsqr_pt_kernel, m <= 8, n >= 4096: every thread
# folds 8 strided rows at a time into its own R) and the lane-group kernel
# (tsqr_gs_kernel, 8 < m <= 32: 4 or 8 lanes share a stream by columns);
# ragged row counts, zero / duplicated columns, low rank and a column whose
# squared norms are subnormal.
@pytest.mark.parametrize("n,m,kind", [(100003, 1, "dense"), (50000, 2, "dense"), (70001, 3, "dup"),
                                      (1 << 20, 4, "dense"), (65537, 5, "lowrank"), (200000, 8, "dup"),
                                      (4096, 8, "dense"), (300001, 6, "dense"), (4099, 7, "dup"),
                                      (4096, 16, "dense"), (100003, 12, "dup"), (1 << 20, 16, "dense"),
                                      (65537, 20, "lowrank"), (300001, 32, "dup"), (8191, 25, "dense"),
                                      (200000, 9, "tiny")])
def test_tsqr_thread_streams(tt, n, m, kind):
    _check_streams(tt, n, m, kind)


# The bulk-copy (TMA) staged group streams (tsqr_gt_kernel, 8 < m <= 32 and
# n >= 4 slices per warp of the grid): full and partial last slices, m below
# the padded width, zero / duplicated columns, low rank, subnormal squares.
@pytest.mark.parametrize("n,m,kind", [(400003, 12, "dup"), (1 << 19, 32, "dense"), (303200, 20, "lowrank"),
                                      (500001, 9, "tiny"), (350000, 27, "dup"), (1 << 21, 16, "dense"),
                                      (303104, 17, "dense")])
def test_tsqr_bulk_staged_streams(tt, n, m, kind):
    _check_streams(tt, n, m, kind)


def _check_streams(tt, n, m, kind):
    from oracle.oracle import gaussian
    X = gaussian(n, m, 41 + m).copy(order="F")
    if kind == "dup" and m >= 3:
        X[:, m - 1] = X[:, 0]
        X[:, 1] = 0.0
    if kind == "lowrank":
        X = np.asfortranarray(gaussian(n, 2, 5) @ gaussian(2, m, 6))
    if kind == "tiny":
        X[:, 3] *= 1e-156
        X[:, 5] = 0.0
    R = host(tt.tsqr(X))
    assert np.all(np.isfinite(R))
    assert np.all(np.tril(R, -1) == 0.0)
    assert gram_resid(X, R) <= 1e-12
    s_r = np.linalg.svd(R, compute_uv=False)
    s_x = np.linalg.svd(X, compute_uv=False)
    assert np.max(np.abs(s_r - s_x)) <= 1e-10 * s_x[0]
    if kind in ("dup", "lowrank"):
        rank = 2 if kind == "lowrank" else m - 2
        assert s_r[rank] <= 1e-13 * s_r[0]
    # orthogonal transforms keep column norms: ||R e_c|| = ||X e_c||, also for
    # the 1e-156 column whose squares are subnormal (no flush to zero)
    cn_r, cn_x = np.linalg.norm(R, axis=0), np.linalg.norm(X, axis=0)
    assert np.allclose(cn_r, cn_x, rtol=1e-6 if kind == "tiny" else 1e-12, atol=1e-150)
    # the same bytes give the same R (fixed reduction order)
    assert np.array_equal(host(tt.tsqr(X)), R)


def test_tsqr_rank_deficient_duplicate_column(tt, orc):
    # test_tsqr.cpp:88-97
    from oracle.oracle import gaussian
    d = gaussian(10000, 5, 9).copy(order="F")
    d[:, 2] = d[:, 0]
    R = host(tt.tsqr(d))
    assert np.all(np.isfinite(R))
    s, _, _ = orc.jacobi_svd(R, want_u=False)
    assert s[4] / s[0] <= 1e-14
    assert gram_resid(d, R) <= 1e-12


def test_tsqr_zero_and_short(tt):
    # test_tsqr.cpp:99-107
    R = host(tt.tsqr(np.zeros((1000, 3))))
    assert np.all(np.isfinite(R)) and np.linalg.norm(R) <= 1e-150
    with pytest.raises(tt.DimensionError):
        tt.tsqr(np.zeros((2, 3)))


def test_tsqr_tiny_column(tt):
    # test_tsqr.cpp:149-159 (1e-200 column, zero column)
    from oracle.oracle import gaussian
    d = gaussian(10000, 4, 12).copy(order="F")
    d[:, 1] = 0.0
    d[:, 3] = 1e-200 * d[:, 0]
    R = host(tt.tsqr(d))
    assert np.all(np.isfinite(R))
    assert gram_resid(d, R) <= 1e-12


def test_tsqr_randomized_sweep_c04(tt):
    # acceptance_test.cpp:140-179 (C04), reduced trial count
    rng = np.random.default_rng(99)
    from oracle.oracle import gaussian
    worst = 0.0
    for trial in range(40):
        if trial % 10 == 0:
            n, m = 200000, (32 if trial % 20 == 0 else 8)
        elif trial % 5 == 0:
            n, m = int(10000 + rng.integers(20000)), int(16 + rng.integers(17))
        else:
            n, m = int(100 + rng.integers(4000)), int(1 + rng.integers(16))
        d = gaussian(n, m, 4000 + trial).copy(order="F")
        if trial % 3 == 1 and m > 1:
            d[:, m - 1] = 0.0
        if trial % 3 == 2 and m > 2:
            d[:, m - 1] = d[:, 0]
        R = host(tt.tsqr(d))
        assert np.all(np.isfinite(R))
        worst = max(worst, gram_resid(d, R))
    assert worst <= 1e-12


def test_tsqr_deterministic_bitwise(tt):
    # test_tsqr.cpp:127-133 and acceptance C10
    from oracle.oracle import gaussian
    X = gaussian(50000, 6, 5)
    a, b = host(tt.tsqr(X)), host(tt.tsqr(X))
    assert np.array_equal(a, b)


def test_tsqr_singular_values_c05(tt, orc):
    # acceptance_test.cpp:181-208 — QR-trick sigma vs Jacobi on X, kappa <= 1e6
    from oracle.oracle import with_singular_values
    rng = np.random.default_rng(55)
    worst = 0.0
    for trial in range(12):
        n = int(500 + rng.integers(3000))
        m = int(2 + rng.integers(23))
        kappa = 10.0 ** (1 + trial % 6)
        sv = [kappa ** (-j / (m - 1)) for j in range(m)]
        d = with_singular_values(n, m, sv, 6000 + trial)
        R = host(tt.tsqr(d))
        s_gpu = host(tt.small_svd(R).sigma)
        s_dir, _, _ = orc.jacobi_svd(d, want_u=False)
        worst = max(worst, float(np.max(np.abs(s_gpu - s_dir)) / s_dir[0]))
    assert worst <= 1e-10


def test_combine_factors(tt):
    # test_tsqr.cpp:161-192
    a = np.eye(2)
    single = host(tt.combine_factors([a]))
    assert np.array_equal(single, a)
    c = host(tt.combine_factors([a, a]))
    g = c.T @ c
    assert abs(g[0, 0] - 2) <= 1e-15 and abs(g[1, 1] - 2) <= 1e-15 and abs(g[0, 1]) <= 1e-15
    from oracle.oracle import gaussian
    parts, expect = [], np.zeros((4, 4))
    for p in range(7):
        r = np.triu(gaussian(4, 4, 100 + p))
        expect += r.T @ r
        parts.append(r)
    c = host(tt.combine_factors(parts))
    assert np.linalg.norm(c.T @ c - expect) <= 1e-13 * np.linalg.norm(expect)
    with pytest.raises(tt.DimensionMismatch):
        tt.combine_factors(parts + [np.zeros((3, 3))])


# ------------------------------------------------------------- small svd ----
def test_small_svd_diagonal(tt):
    # test_small_svd.cpp:39-54
    s = tt.small_svd(np.diag([3.0, 2.0, 1.0]))
    assert np.allclose(host(s.sigma), [3, 2, 1], atol=1e-14)
    assert np.allclose(np.abs(host(s.V)), np.eye(3), atol=1e-14)


def test_small_svd_golden_ratio(tt):
    # test_small_svd.cpp:56-71
    s = host(tt.small_svd(np.array([[1.0, 1.0], [0.0, 1.0]])).sigma)
    phi = (1 + math.sqrt(5)) / 2
    assert abs(s[0] - phi) <= 1e-14 and abs(s[1] - 1 / phi) <= 1e-14
    for sv in s:
        x = sv * sv
        assert abs(x * x - 3 * x + 1) <= 1e-13


@pytest.mark.parametrize("m", [16, 64, 130, 256])
def test_small_svd_random_triangular(tt, orc, m):
    # test_small_svd.cpp:73-83 invariants + sigma parity with the oracle.
    # Random triangular factors are badly conditioned for large m, so only
    # gauge-free quantities are compared: sigma, V^T V = I, ||R v_j|| = sigma_j.
    from oracle.oracle import gaussian
    r = np.triu(gaussian(m, m, 21))
    s = tt.small_svd(r)
    sig, V = host(s.sigma), host(s.V)
    assert np.all(np.diff(sig) <= 0)
    ref_s, _, ref_V = orc.jacobi_svd(r, want_u=False)
    assert np.max(np.abs(sig - ref_s)) <= 1e-10 * ref_s[0]
    assert np.linalg.norm(V.T @ V - np.eye(m)) <= 1e-12 * m
    assert np.max(np.abs(np.linalg.norm(r @ V, axis=0) - sig)) <= 1e-10 * sig[0]


@pytest.mark.parametrize("m", [8, 64, 128, 256])
def test_small_svd_of_tsqr_factor_vectors(tt, orc, m):
    # the TT-SVD use: R of a well-conditioned tall matrix; singular vectors
    # agree with the oracle's up to sign (distinct sigma)
    from oracle.oracle import gaussian
    X = gaussian(4 * m, m, 500 + m)
    R = orc.tsqr(X)
    s = tt.small_svd(R)
    sig, V = host(s.sigma), host(s.V)
    ref_s, _, ref_V = orc.jacobi_svd(R, want_u=False)
    assert np.max(np.abs(sig - ref_s)) <= 1e-12 * ref_s[0]
    dots = np.abs(np.sum(V * ref_V, axis=0))
    assert np.max(np.abs(dots - 1.0)) <= 1e-9


def test_small_svd_rank_deficient(tt):
    # test_small_svd.cpp:85-95
    r = np.zeros((4, 4))
    r[0, 0] = 2
    r[0, 2] = 1
    s = tt.small_svd(r)
    sig, V = host(s.sigma), host(s.V)
    assert abs(sig[0] - math.sqrt(5)) <= 1e-14 and abs(sig[2]) <= 1e-14 and abs(sig[3]) <= 1e-14
    assert np.linalg.norm(V.T @ V - np.eye(4)) <= 1e-12 * 4


def test_jacobi_svd_tall(tt, orc):
    # test_small_svd.cpp:129-134 + U/V against the oracle
    from oracle.oracle import gaussian
    a = gaussian(200, 5, 3)
    s = tt.jacobi_svd(a)
    sig, U, V = host(s.sigma), host(s.U), host(s.V)
    assert abs(np.sum(sig ** 2) - np.linalg.norm(a) ** 2) <= 1e-10 * np.sum(sig ** 2)
    assert np.linalg.norm(U.T @ U - np.eye(5)) <= 1e-12 * 5
    rs, rU, rV = orc.jacobi_svd(a)
    assert np.max(np.abs(sig - rs)) <= 1e-12 * rs[0]
    assert np.allclose(np.abs(np.sum(V * rV, axis=0)), 1.0, atol=1e-12)


def test_jacobi_svd_zero_completion(tt, orc):
    # small_svd.hpp:165-191: zero input -> canonical completion of U
    s = tt.jacobi_svd(np.zeros((6, 3)))
    rs, rU, rV = orc.jacobi_svd(np.zeros((6, 3)))
    assert np.array_equal(host(s.U), rU)
    assert np.array_equal(host(s.V), rV)
    assert np.all(host(s.sigma) == 0)


def test_select_rank_and_delta(tt):
    # test_small_svd.cpp:97-124
    assert tt.select_rank([2, 1, 0.5, 0.1], 0.2, 10) == 3
    assert tt.select_rank([2, 1, 0.5], 0.0, 2) == 2
    assert tt.select_rank([5], 10.0, 3) == 1
    assert tt.derive_delta(123.0, 0.0, 7) == 0.0
    assert abs(tt.derive_delta(2.0, 0.1, 5) - 0.1) <= 1e-15
    with pytest.raises(tt.DegenerateDimension):
        tt.derive_delta(1.0, 0.1, 1)


# ------------------------------------------------------------------ tsmm ----
def _relabel(prod, out_rows, out_cols):
    n, k = prod.shape
    out = np.zeros((out_rows, out_cols))
    for c in range(k):
        p = np.arange(n) + n * c
        out[p % out_rows, p // out_rows] = prod[:, c]
    return out


def test_tsmm_identity_keeps_content(tt):
    from oracle.oracle import uniform
    x = uniform(64, 5, 1)
    y = host(tt.tsmm_reshape(x, np.eye(5), 64, 5))
    assert np.array_equal(y, x)


def test_tsmm_matches_naive_oracle(tt, orc):
    from oracle.oracle import gaussian
    x = gaussian(100, 6, 2)
    v = gaussian(6, 3, 3)
    y = host(tt.tsmm_reshape(x, v, 50, 6))
    expect = _relabel(x @ v, 50, 6)
    assert np.max(np.abs(y - expect)) <= 1e-13 * np.linalg.norm(expect)
    yo = orc.tsmm_reshape(x, v, 50, 6)[:50]
    assert np.max(np.abs(y - yo)) <= 1e-13 * np.linalg.norm(expect)


def test_tsmm_column_selection_is_exact(tt):
    from oracle.oracle import uniform
    n = 1 << 16
    x = uniform(n, 8, 4)
    sel = np.zeros((8, 4))
    sel[np.arange(4), np.arange(4)] = 1.0
    y = host(tt.tsmm_reshape(x, sel, n // 2, 8))
    flat = x[:, :4].reshape(-1, order="F")
    assert np.array_equal(y.reshape(-1, order="F"), flat)


def test_tsmm_dt_non_dividing_reshape(tt, orc):
    # tsmm_dt_kernel with out_rows that does not divide n (per-element placement)
    from oracle.oracle import gaussian
    n, m, k = 1 << 16, 48, 24
    x = gaussian(n, m, 5)
    v = np.linalg.qr(gaussian(m, k, 6))[0]
    out_rows, out_cols = 3 << 14, 32
    y = host(tt.tsmm_reshape(x, v, out_rows, out_cols))
    yo = orc.tsmm_reshape(x, v, out_rows, out_cols)[:out_rows]
    assert np.max(np.abs(y - yo)) <= 1e-13 * np.linalg.norm(yo)


def test_tsmm_guards(tt):
    with pytest.raises(tt.ShapeError):
        tt.tsmm_reshape(np.zeros((10, 4)), np.zeros((4, 2)), 7, 3)
    with pytest.raises(tt.ShapeError):
        tt.tsmm_reshape(np.zeros((10, 4)), np.zeros((4, 6)), 10, 6)


def test_tsmm_frobenius_and_padding(tt):
    from oracle.oracle import gaussian, orthonormal
    x = gaussian(512, 7, 8)
    v = orthonormal(7, 3, 9)
    Y = tt.tsmm_reshape(x, v, 256, 6)
    y = host(Y)
    prod = x @ v
    assert abs(np.linalg.norm(y) - np.linalg.norm(prod)) <= 1e-13 * np.linalg.norm(prod)
    assert np.linalg.norm(y) <= np.linalg.norm(x) * (1 + 1e-12)
    assert Y.stride(1) == tt.padded_stride(256)
    buf = Y.as_strided((Y.stride(1), 6), (1, Y.stride(1)))
    assert bool((buf[256:] == 0).all())


@pytest.mark.parametrize("n,m,k,nn", [(1 << 20, 16, 16, 16), (1 << 16, 256, 32, 16), (4096, 512, 32, 16),
                                      (30000, 50, 40, 10), (1000, 3, 2, 1),
                                      # short X (tsmm_small_kernel): partial row blocks and column chunks,
                                      # m not a multiple of the warp split, a non-dividing reshape
                                      (256, 512, 32, 16), (16, 512, 16, 16), (16384, 64, 16, 4), (1000, 77, 13, 10),
                                      (33, 40, 9, 3), (4097, 100, 5, 17),
                                      # TMA-staged DMMA kernel (tsmm_dt_kernel): n % 64 == 0, m % 8 == 0, k > 16,
                                      # two column chunks, two stages (m > 256)
                                      (1 << 18, 64, 24, 4), (1 << 16, 40, 32, 2), (262208, 96, 20, 16),
                                      (1 << 16, 264, 40, 8), (1 << 16, 512, 32, 16)])
def test_tsmm_shapes_vs_oracle(tt, orc, n, m, k, nn):
    from oracle.oracle import gaussian, orthonormal
    x = gaussian(n, m, n + m)
    v = orthonormal(m, k, 103) if m <= 64 else np.linalg.qr(gaussian(m, k, 103))[0]
    out_rows, out_cols = n // nn, nn * k
    y = host(tt.tsmm_reshape(x, v, out_rows, out_cols))
    yo = orc.tsmm_reshape(x, v, out_rows, out_cols)[:out_rows]
    assert np.max(np.abs(y - yo)) <= 1e-13 * max(np.linalg.norm(yo), 1.0)
    assert np.array_equal(host(tt.tsmm_reshape(x, v, out_rows, out_cols)), y)
