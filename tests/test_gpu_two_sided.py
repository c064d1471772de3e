"""§8 f-4: the two-sided sweep (Alg. 4, tt_svd.hpp:402-512) and
transpose_reorder (tsmm.hpp:84-126) on the device, against the reference
itself (oracle/_ref: the reference headers compiled) on the same inputs.

* transpose_reorder is a pure permutation: bit-exact, padding zero.
* tt_svd_two_sided: ranks identical to the reference's two-sided run,
  relative reconstruction error within 1e-10 of the reference's, and the
  orthonormality of every core but the middle one at the reference's level
  (test_tt_svd.cpp:190-230 shapes: rank one, odd / even d, 3^d for d = 2..7,
  cap-bound and uncapped runs).
"""
import numpy as np
import pytest

from helpers import rel_error

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2102_00104_b200 as tt
    return tt


@pytest.mark.parametrize("n,m,out_rows", [(1, 1, 1), (4, 2, 2), (6, 2, 4), (1024, 8, 8), (1024, 8, 2048),
                                          (777, 13, 13), (4096, 64, 512), (100, 300, 300), (65536, 5, 327680)])
def test_transpose_reorder_bit_exact(tt, ref, n, m, out_rows):
    import torch
    g = np.random.default_rng(n * 31 + m)
    W = np.asfortranarray(g.standard_normal((n, m)))
    out_cols = n * m // out_rows
    Y = tt.transpose_reorder(torch.from_numpy(W.T.copy()).cuda().t(), out_rows, out_cols)
    ldy = tt.padded_stride(out_rows)
    Yfull = Y.as_strided((ldy, out_cols), (1, ldy)).cpu().numpy()
    Yr = ref.transpose_reorder(W, out_rows, out_cols)
    assert np.array_equal(Yfull, Yr)


def two_sided_both(tt, ref, X, dims, r_max, eps=0.0):
    import torch
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    rows = int(np.prod(dims)) // dims[-1]
    T = tt.tt_svd_two_sided(Xd[:rows], dims, tt.TruncationSpec(r_max=r_max, eps=eps))
    r, cores = ref.tt_svd_two_sided(X, dims, X.shape[0], r_max, eps)
    return T, r, cores


def orthonormality(cores, excluded):
    worst = 0.0
    for j, c in enumerate(cores):
        if j == excluded:
            continue
        rl, n, rr = c.shape
        if j < excluded:
            V = np.asfortranarray(c).reshape(rl * n, rr, order="F")
            g = V.T @ V
        else:
            H = np.asfortranarray(c).reshape(rl, n * rr, order="F")
            g = H @ H.T
        worst = max(worst, float(np.linalg.norm(g - np.eye(g.shape[0]))))
    return worst


CASES = [("rank1", [4, 4, 4, 4], 8, 0.0), ("odd", [8, 8, 8], 8, 0.0), ("cap", [2] * 10, 4, 0.0),
         ("uncapped", [4, 4, 4, 4], 2 ** 63 - 1, 0.0), ("eps", [2] * 12, 2 ** 63 - 1, 1e-1),
         ("mixed", [2, 3, 4, 5, 6], 5, 0.0)] + [(f"3^{d}", [3] * d, 27, 0.0) for d in range(2, 8)]


@pytest.mark.parametrize("name,dims,r_max,eps", CASES, ids=[c[0] for c in CASES])
def test_two_sided_vs_reference(tt, ref, name, dims, r_max, eps):
    from oracle.oracle import random_tensor, random_tt, tt_reconstruct
    if name == "rank1":
        X = tt_reconstruct(random_tt(dims, [1] * (len(dims) + 1), 89), dims)
    else:
        X = random_tensor(97 + len(dims), dims)
    T, r, cores = two_sided_both(tt, ref, X, dims, r_max, eps)
    assert T.ranks() == r
    e_gpu = rel_error(X, dims, [c.data for c in T.cores])
    e_ref = rel_error(X, dims, cores)
    assert abs(e_gpu - e_ref) <= 1e-10, (e_gpu, e_ref)
    d = len(dims)
    mid = d // 2
    excl = mid - 1 if d % 2 == 0 else mid
    o_gpu = orthonormality([c.data for c in T.cores], excl)
    o_ref = orthonormality(cores, excl)
    assert o_gpu <= max(10 * o_ref, 1e-11 * max(T.ranks())), (o_gpu, o_ref)


def test_two_sided_step_records(tt):
    # steps alternate right / left; the reorder is timed on every step but a
    # final right one (StepRecord::t_reorder)
    X = tt.gen_uniform(7, [4] * 6)
    ctx = tt.context()
    ctx.set_timing(True)
    try:
        T = tt.tt_svd_two_sided(X, [4] * 6, tt.TruncationSpec(r_max=8))
    finally:
        ctx.set_timing(False)
    assert len(T.steps) == 5
    assert all(s.t_reorder > 0 for s in T.steps[:-1])
