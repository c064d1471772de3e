"""GPU parity of the thick-bounds driver (Alg. 3, tt_svd.hpp:292-400) through
the C-ABI against the reference's own tt_svd_thick_bounds (oracle/_ref) on the
same inputs.  Thick-bounds is not parity-equal to the plain driver (SURVEY
§4, C01), so the reference for these cases is tt_svd_thick_bounds itself.
Tolerances as the plain driver's: ranks identical, relative reconstruction
error within 1e-10 of the reference's, cores equal up to gauge (principal
angles of the right frames <= 1e-8 rad).
"""
import numpy as np
import pytest

from helpers import frame_angles, rel_error

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2102_00104_b200 as tt
    return tt


def run_thick(tt, ref, X, dims, r_max, eps=0.0, m_min=16, f1_min=0.5, r_tilde=()):
    import torch
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    rows = int(np.prod(dims)) // dims[-1]
    T = tt.tt_svd_thick_bounds(Xd[:rows], dims, tt.TruncationSpec(r_max=r_max, eps=eps),
                               tt.ThickBoundsParams(m_min=m_min, f1_min=f1_min, r_tilde=list(r_tilde)))
    r, cores = ref.tt_svd_thick_bounds(X, dims, X.shape[0], r_max, eps, m_min, f1_min, r_tilde)
    return T, r, cores


def check(ref, X, dims, T, r, cores, err_tol=1e-10, angle_tol=1e-8):
    assert T.ranks() == r
    gpu_cores = [c.data for c in T.cores]
    for c, n in zip(gpu_cores, dims):
        assert c.shape[1] == n
    e_gpu = rel_error(X, dims, gpu_cores)
    e_ref = ref.tt_error(X, X.shape[0], dims, r, cores)
    assert abs(e_gpu - e_ref) <= err_tol
    assert max(frame_angles(gpu_cores, cores)) <= angle_tol
    return e_gpu, e_ref


def test_config1_thick(tt, orc, ref):
    # BASELINE config 1 (4^10 uniform[-1,1], seed 1, r_max 16): k = 3, m = 64
    dims = [4] * 10
    X = orc.gen_uniform(1, dims)
    assert tt.choose_combined_dims(dims, tt.ThickBoundsParams(), 16) == (3, 64)
    T, r, cores = run_thick(tt, ref, X, dims, 16)
    check(ref, X, dims, T, r, cores)


def test_exact_tt_thick(tt, ref):
    # exact TT of rank 8 plus 1e-8 noise (the config-2 recipe at 16^5): lossless recovery
    from oracle.oracle import random_tt, tt_reconstruct
    dims = [16] * 5
    ranks = [1] + [8] * 4 + [1]
    X = tt_reconstruct(random_tt(dims, ranks, 71), dims)
    rng = np.random.default_rng(72)
    X = X + 1e-8 * np.linalg.norm(X) / np.sqrt(X.size) * rng.standard_normal(X.shape)
    X = np.asfortranarray(X)
    T, r, cores = run_thick(tt, ref, X, dims, 8)
    assert r == ranks
    e_gpu, _ = check(ref, X, dims, T, r, cores, err_tol=1e-8)
    assert e_gpu <= 1e-7


@pytest.mark.parametrize("dims,r_max,eps,m_min,f1_min", [
    ([2] * 14, 6, 0.0, 16, 0.5),      # k = 4 merged binary modes
    ([3, 5, 4, 6, 2, 7], 10, 0.0, 16, 0.5),
    ([2] * 12, 64, 0.05, 8, 0.5),     # tolerance-driven ranks, rescaled recovery delta
    ([8, 8, 8, 8], 4, 0.0, 4, 1.0),   # k = 1: the plain driver
])
def test_thick_shapes(tt, ref, dims, r_max, eps, m_min, f1_min):
    from oracle.oracle import random_tensor
    X = random_tensor(91 + len(dims), dims)
    T, r, cores = run_thick(tt, ref, X, dims, r_max, eps, m_min, f1_min)
    check(ref, X, dims, T, r, cores, err_tol=1e-9)


def test_rank_one_boundary(tt, ref):
    # rank-1 tensor: r_b = 1 and a rank-1 recovery -> the captured scalar moves
    # to the first core (tt_svd.hpp:380-387)
    from oracle.oracle import random_tt, tt_reconstruct
    dims = [3] * 8
    X = np.asfortranarray(tt_reconstruct(random_tt(dims, [1] * 9, 73), dims))
    T, r, cores = run_thick(tt, ref, X, dims, 4)
    assert all(v == 1 for v in r)
    e_gpu, _ = check(ref, X, dims, T, r, cores)
    assert e_gpu <= 1e-13
    # the boundary core is right-orthonormal: the norm sits in core 0
    b = T.cores[-1].data
    assert abs(np.linalg.norm(b) - 1.0) <= 1e-12


# The merged matricization read in place (ColSplit view of the caller's padded
# X; tt_svd.hpp:347-348's copy_logical avoided): tall-tile TSQR + TMA-staged
# TSMM (m = 64), TMA-staged streams + TSMM (m = 32), and a rank (6 <= 8) that
# leaves the view-reading TSMM kernel, so the view is materialised for that one
# product.  Same parity bar as the copied layout.
@pytest.mark.parametrize("dims,r_max,m_min,expect_km,tt_rank", [
    ([4] * 12, 16, 16, (3, 64), 0),     # uniform[-1,1] in the padded layout
    ([2] * 24, 12, 32, (5, 32), 12),    # exact TT (rank <= 12) + 1e-8 noise: well separated frames
    ([2] * 24, 6, 16, (4, 16), 6),
])
def test_thick_view_in_place(tt, orc, ref, dims, r_max, m_min, expect_km, tt_rank):
    import torch
    if tt_rank:
        from oracle.oracle import random_tt, tt_reconstruct
        d = len(dims)
        ranks = [min(tt_rank, 2 ** min(j, d - j)) for j in range(d + 1)]
        X = tt_reconstruct(random_tt(dims, ranks, 77), dims)
        rng = np.random.default_rng(78)
        X = np.asfortranarray(X + 1e-8 * np.linalg.norm(X) / np.sqrt(X.size) * rng.standard_normal(X.shape))
    else:
        X = orc.gen_uniform(5, dims)
    p = tt.ThickBoundsParams(m_min=m_min)
    assert tt.choose_combined_dims(dims, p, r_max) == expect_km
    free0 = torch.cuda.mem_get_info()[0]
    T, r, cores = run_thick(tt, ref, X, dims, r_max, 0.0, m_min)
    free1 = torch.cuda.mem_get_info()[0]
    check(ref, X, dims, T, r, cores, err_tol=1e-8 if tt_rank else 1e-10)
    if r_max > 8:
        # no copy of X (8 prod(dims) bytes) was allocated next to it (the
        # device copy of X itself is; the work buffers are a fraction of it)
        assert free0 - free1 < 2 * 8 * int(np.prod(dims)) - (8 * int(np.prod(dims))) // 4


def test_thick_host_entry_chunked_h2d(tt, ref):
    # host buffer in: X arrives in row chunks of the merged matricization
    # (2^19 x 64) and tsqr_t128 folds each chunk as it lands; same parity bar
    # against the reference's tt_svd_thick_bounds, and agreement with the
    # device entry within rounding (other tile boundaries, not bit for bit)
    import torch
    from oracle.oracle import random_tt, tt_reconstruct
    dims = [2] * 25
    d = len(dims)
    ranks = [min(12, 2 ** min(j, d - j)) for j in range(d + 1)]
    X = tt_reconstruct(random_tt(dims, ranks, 81), dims)
    rng = np.random.default_rng(82)
    X = np.asfortranarray(X + 1e-8 * np.linalg.norm(X) / np.sqrt(X.size) * rng.standard_normal(X.shape))
    p = tt.ThickBoundsParams(m_min=64)
    assert tt.choose_combined_dims(dims, p, 12) == (6, 64)
    Th = tt.tt_svd_thick_bounds(X, dims, tt.TruncationSpec(r_max=12), p)          # host entry
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    rows = int(np.prod(dims)) // dims[-1]
    Td = tt.tt_svd_thick_bounds(Xd[:rows], dims, tt.TruncationSpec(r_max=12), p)  # device entry
    r, cores = ref.tt_svd_thick_bounds(X, dims, X.shape[0], 12, 0.0, 64, 0.5, ())
    check(ref, X, dims, Th, r, cores, err_tol=1e-8)
    assert Th.ranks() == Td.ranks()
    for sh, sd in zip(Th.sigmas, Td.sigmas):
        assert np.max(np.abs(sh - sd)) <= 1e-10 * sd[0]
    assert max(frame_angles([c.data for c in Th.cores], [c.data for c in Td.cores])) <= 1e-8
