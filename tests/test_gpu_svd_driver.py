"""GPU parity of the TT-SVD driver's SVD (tt_svd.hpp:85-110: the small SVD of
R / W whose leading r right singular vectors become the core) through the
C-ABI ttsvd_cu_driver_svd: the bidiagonal path (Householder
bidiagonalisation in a 16-CTA cluster, bisection, twisted factorisation /
clustered inverse iteration) and the Jacobi path it replaces, against numpy's
LAPACK SVD on the same matrices.

Tolerances (north_star): sigma |dsigma| <= 1e-10 sigma_1 (we hold 1e-12);
vectors compared up to gauge by the largest principal angle of the leading
r-dimensional subspace (sin <= 1e-10 when the r / r+1 gap is >= 1e-3 sigma_1),
orthonormality ||V^T V - I|| <= 1e-12.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2102_00104_b200 as tt
    return tt


def host(T):
    return T.detach().cpu().numpy()


def subspace_sin(U, V):
    """sin of the largest principal angle between span(U) and span(V) (orthonormal columns)."""
    resid = V - U @ (U.T @ V)
    return float(np.linalg.norm(resid, 2)) if resid.size else 0.0


def with_sigma(n, m, sig, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, m)))
    W, _ = np.linalg.qr(rng.standard_normal((m, m)))
    return np.asfortranarray((U * sig) @ W.T), U


def check(tt, A, r, path="bidiag", sig_tol=1e-12, ang_tol=1e-10):
    s, V, p = tt.driver_svd(A, r)
    s, V = host(s), host(V)
    assert p == path
    s_ref = np.linalg.svd(A, compute_uv=False)
    assert np.all(np.diff(s) <= 0.0)
    assert np.max(np.abs(s - s_ref)) <= sig_tol * s_ref[0]
    if r:
        assert np.linalg.norm(V.T @ V - np.eye(r)) <= 1e-12
        U_ref = np.linalg.svd(A, full_matrices=False)[0][:, :r]
        assert subspace_sin(U_ref, V) <= ang_tol
    return s, V


@pytest.mark.parametrize("n,m,r", [(64, 64, 16), (100, 100, 32), (512, 512, 32), (512, 256, 16), (300, 257, 40),
                                   (900, 200, 8), (1024, 129, 1)])
def test_driver_svd_random(tt, n, m, r):
    # Gaussian singular spectrum: the leading gaps are ~1e-2 sigma_1
    rng = np.random.default_rng(n * 7 + m)
    A = np.asfortranarray(rng.standard_normal((n, m)))
    check(tt, A, r, ang_tol=1e-9)


# the register-tile bidiagonalisation at every (columns per CTA, cluster)
# instantiation and at row counts that leave warps, lanes or whole reducer
# slices empty (the DSMEM exchanges count only the live rows)
@pytest.mark.parametrize("n,m,r", [(33, 33, 8), (129, 129, 16), (250, 250, 32), (257, 257, 32), (511, 511, 32),
                                   (512, 300, 32), (400, 400, 64), (480, 17, 17), (96, 65, 20)])
def test_driver_svd_tile_shapes(tt, n, m, r):
    rng = np.random.default_rng(n * 13 + m)
    A = np.asfortranarray(rng.standard_normal((n, m)))
    check(tt, A, r, ang_tol=1e-9)


def test_driver_svd_config2_like(tt):
    # exact rank 32 + 1e-8 relative noise (the config-2 work matrices)
    rng = np.random.default_rng(3)
    n = m = 512
    A = rng.standard_normal((n, 32)) @ rng.standard_normal((32, m))
    A += 1e-8 * np.linalg.norm(A) / np.sqrt(n * m) * rng.standard_normal((n, m))
    check(tt, np.asfortranarray(A), 32)


def test_driver_svd_graded_and_zero(tt):
    # graded spectrum 1 .. 1e-14 with 40 exact zeros: sigmas are absolutely
    # accurate, the leading vectors (well separated) are accurate
    n, m = 400, 300
    sig = np.concatenate([np.logspace(0, -14, m - 40), np.zeros(40)])
    A, _ = with_sigma(n, m, sig, 5)
    check(tt, A, 20)


def test_driver_svd_clusters(tt):
    # a triple cluster (1e-12 apart) and an exact double inside the leading 12:
    # the clustered members go through inverse iteration with Gram-Schmidt;
    # the subspace of each cluster and the whole leading 12 are exact
    n, m = 256, 200
    sig = np.linspace(1.0, 0.01, m)
    sig[3:6] = 0.7 + np.array([0.0, 1e-12, 2e-12])
    sig[8:10] = 0.5
    sig = np.sort(sig)[::-1]
    A, U = with_sigma(n, m, sig, 9)
    s, V = check(tt, A, 12)
    # each cluster's subspace individually
    order = np.argsort(-sig)
    for lo, hi in [(3, 6), (8, 10)]:
        Uc = U[:, order[lo:hi]]
        assert subspace_sin(Uc, V[:, lo:hi]) <= 1e-9


def test_driver_svd_wide_work_matrix(tt):
    # the wide step's W^T: n = 512 > m = 256 (config-2 step 5 shape)
    rng = np.random.default_rng(11)
    W = rng.standard_normal((256, 32)) @ rng.standard_normal((32, 512))
    W += 1e-8 * rng.standard_normal(W.shape)
    check(tt, np.asfortranarray(W.T), 32)


def test_driver_svd_small_uses_jacobi(tt):
    # below the bidiagonal threshold (m < 16) the Jacobi path runs; same contract
    rng = np.random.default_rng(2)
    A = np.asfortranarray(rng.standard_normal((80, 12)))
    check(tt, A, 6, path="jacobi", ang_tol=1e-9)


@pytest.mark.parametrize("n,m,r", [(80, 40, 10), (16, 16, 16), (512, 16, 16), (300, 17, 5)])
def test_driver_svd_narrow_bidiag(tt, n, m, r):
    # from m = 16 the bidiagonal path runs (config 2 steps 1 and 6 have m = 16)
    rng = np.random.default_rng(n + m)
    A = np.asfortranarray(rng.standard_normal((n, m)))
    check(tt, A, r, path="bidiag", ang_tol=1e-9)


def test_driver_svd_matches_reference_jacobi(tt):
    # the reference's algorithm (small_svd.hpp: one-sided Jacobi, ttsvd_cu_jacobi_svd)
    # and the bidiagonal path agree on sigma and on the leading subspace
    rng = np.random.default_rng(4)
    A = np.asfortranarray(rng.standard_normal((384, 384)) * np.logspace(0, -6, 384)[None, :])
    s, V, p = tt.driver_svd(A, 24)
    assert p == "bidiag"
    ref = tt.jacobi_svd(A)
    s_j, U_j = host(ref.sigma), host(ref.U)
    assert np.max(np.abs(host(s) - s_j)) <= 1e-12 * s_j[0]
    assert subspace_sin(U_j[:, :24], host(V)) <= 1e-9


def test_driver_svd_rejects_bad_shapes(tt):
    with pytest.raises(tt.Error):
        tt.driver_svd(np.zeros((10, 20)), 2)
    with pytest.raises(tt.Error):
        tt.driver_svd(np.ones((80, 70)), 71)
