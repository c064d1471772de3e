"""GPU parity of the TT-SVD drivers (tt_svd_tsqr, tt_svd_distributed) through
the C-ABI against the CPU reference / oracle on the same seeded inputs.

Mirrors /root/reference/proj/tests/test_tt_svd.cpp and acceptance C01-C03,
C07, C08, C10.  Tolerances (north_star): ranks identical; per-step singular
values |dsigma| <= 1e-10 sigma_1; relative reconstruction error within 1e-8 of
the reference's (1e-10 where the reference test pins it); cores compared up
to gauge via the principal angles of the right frames (<= 1e-8 rad).
"""
import numpy as np
import pytest

from helpers import frame_angles, rel_error, split_slabs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2102_00104_b200 as tt
    return tt


def cores_of(T):
    return [c.data for c in T.cores]


def run_both(tt, orc, X, dims, r_max, eps=0.0):
    import torch
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()  # (ld x n_d) Fortran view
    rows = int(np.prod(dims)) // dims[-1]
    T = tt.tt_svd_tsqr(Xd[:rows], dims, tt.TruncationSpec(r_max=r_max, eps=eps))
    r, cores, steps, sig = orc.tt_svd_tsqr(X, dims, X.shape[0], r_max, eps, with_sigma=True)
    return T, (r, cores, steps, sig)


def assert_parity(tt, orc, X, dims, T, ref, err_tol=1e-10):
    r, cores, steps, sig = ref
    assert T.ranks() == r
    for s_gpu, s_ref in zip(T.sigmas, sig):
        assert len(s_gpu) == len(s_ref)
        assert np.max(np.abs(s_gpu - s_ref)) <= 1e-10 * s_ref[0]
    e_gpu = rel_error(X, dims, cores_of(T))
    e_ref = orc.tt_error(X, X.shape[0], dims, r, cores)
    assert abs(e_gpu - e_ref) <= err_tol
    assert max(frame_angles(cores_of(T), cores)) <= 1e-8
    return e_gpu, e_ref


def test_config1_4pow10(tt, orc):
    # BASELINE config 1: 4^10 uniform[-1,1] (seed 1), r_max = 16, no tolerance
    dims = [4] * 10
    X = orc.gen_uniform(1, dims)
    T, ref = run_both(tt, orc, X, dims, 16)
    assert T.ranks() == [1, 4, 16, 16, 16, 16, 16, 16, 16, 4, 1]
    assert_parity(tt, orc, X, dims, T, ref, err_tol=1e-10)


def test_reference_inputs_match(tt, orc, ref):
    # test_tt_svd.cpp:59-65 — the reference's own random_tensor input (seed 43)
    from oracle.oracle import random_tensor
    dims = [2] * 12
    X = random_tensor(43, dims)
    T, o = run_both(tt, orc, X, dims, 4)
    assert_parity(tt, orc, X, dims, T, o)
    rr, rc, _ = ref.tt_svd_tsqr(X, dims, X.shape[0], 4)[:3]
    assert rr == T.ranks()


def test_rank_one_and_synthetic_recovery(tt, orc):
    # test_tt_svd.cpp:67-77 and acceptance C03
    from oracle.oracle import random_tt, tt_reconstruct
    dims = [2] * 12
    X = tt_reconstruct(random_tt(dims, [1] * 13, 47), dims)
    T, o = run_both(tt, orc, X, dims, 8)
    assert all(r == 1 for r in T.ranks())
    assert rel_error(X, dims, cores_of(T)) <= 1e-13
    dims = [4] * 6
    ranks = [1, 2, 3, 3, 2, 1, 1]
    Y = tt_reconstruct(random_tt(dims, ranks, 53), dims)
    T, o = run_both(tt, orc, Y, dims, 3)
    assert T.ranks() == ranks
    assert rel_error(Y, dims, cores_of(T)) <= 1e-12


def test_table2_reproduction_c07(tt, orc):
    # acceptance_test.cpp:282-309: 2^16 random (seed 4242), r_max = 5
    from oracle.oracle import random_tensor
    dims = [2] * 16
    X = random_tensor(4242, dims)
    T, o = run_both(tt, orc, X, dims, 5)
    r = T.ranks()
    assert r[-2] == 2 and r[-3] == 4 and r[-4] == 5 and r[-5] == 5
    f = [s.f for s in T.steps]
    assert f[0] == 1.0 and f[1] == 1.0 and f[2] == 5.0 / 8.0 and f[3] == 0.5
    assert_parity(tt, orc, X, dims, T, o)


@pytest.mark.parametrize("t", range(8))
def test_oracle_equivalence_c01_plain(tt, orc, t):
    # acceptance_test.cpp:44-91, plain-TSQR cells (the only variant C01 holds for)
    from oracle.oracle import random_tensor
    shapes = [[2] * 12, [4] * 6, [8] * 4, [2, 3, 4, 5, 6]]
    configs = [(1, 0.0), (4, 0.0), (8, 1e-2), (2 ** 62, 1e-1)]
    dims = shapes[t % 4]
    X = random_tensor(5000 + t, dims)
    for r_max, eps in configs:
        T, o = run_both(tt, orc, X, dims, r_max, eps)
        assert_parity(tt, orc, X, dims, T, o)


def test_error_budget_c02(tt, orc):
    from oracle.oracle import random_tensor
    for eps in (1e-1, 1e-3, 1e-8):
        dims = [2] * 12
        X = random_tensor(61, dims)
        T, o = run_both(tt, orc, X, dims, 2 ** 62, eps)
        assert rel_error(X, dims, cores_of(T)) <= eps + 1e-10
        assert T.ranks() == o[0]


def test_work_matrix_shrinkage(tt, orc):
    # test_tt_svd.cpp:102-116
    from oracle.oracle import random_tensor
    dims = [2] * 10
    X = random_tensor(67, dims)
    T, _ = run_both(tt, orc, X, dims, 4)
    assert len(T.steps) == 9
    size = float(np.prod(dims))
    for s in T.steps:
        assert s.f <= 1.0
        assert abs(s.rows * s.cols - size) <= 0.5
        size *= s.f


def test_determinism_c10(tt):
    from oracle.oracle import random_tensor
    import torch
    dims = [2] * 14
    X = random_tensor(888, dims)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()[: 2 ** 13]
    a = tt.tt_svd_tsqr(Xd, dims, (6, 1e-3))
    b = tt.tt_svd_tsqr(Xd, dims, (6, 1e-3))
    for ca, cb in zip(a.cores, b.cores):
        assert np.array_equal(ca.data, cb.data)


def test_speculative_chain_matches_stepwise(tt, orc):
    # eps = 0: the chain runs on predicted ranks with the rank rule on the
    # device (K6, choose_rank: small_svd.hpp:49-63, tt_svd.hpp:111-118) and one
    # synchronisation at its end; a timed context runs step by step with the
    # host rule.  Same bytes either way — also when a prediction fails (exact
    # low rank below r_max) and the chain is run again.
    from oracle.oracle import random_tensor, random_tt, tt_reconstruct
    import torch
    ctx = tt.context()
    for X, dims, r_max in ((random_tensor(77, [4] * 8), [4] * 8, 16),
                           (tt_reconstruct(random_tt([4] * 6, [1, 2, 3, 3, 2, 1, 1], 53), [4] * 6), [4] * 6, 3),
                           (tt_reconstruct(random_tt([3] * 7, [1, 2, 2, 2, 2, 2, 2, 1], 5), [3] * 7), [3] * 7, 9)):
        Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
        rows = int(np.prod(dims)) // dims[-1]
        a = tt.tt_svd_tsqr(Xd[:rows], dims, tt.TruncationSpec(r_max=r_max))
        ctx.set_timing(True)
        try:
            b = tt.tt_svd_tsqr(Xd[:rows], dims, tt.TruncationSpec(r_max=r_max))
        finally:
            ctx.set_timing(False)
        assert a.ranks() == b.ranks()
        r, cores, steps, sig = orc.tt_svd_tsqr(X, dims, X.shape[0], r_max, 0.0, with_sigma=True)
        assert a.ranks() == r
        for ca, cb in zip(a.cores, b.cores):
            assert np.array_equal(ca.data, cb.data)
        for sa, sb in zip(a.sigmas, b.sigmas):
            assert np.array_equal(sa, sb)
        assert [s.rank for s in a.steps] == [s.rank for s in b.steps]


def test_host_entry_matches_device_entry(tt, orc):
    # the reference-facing host-buffer path (H2D inside the call) == device path
    dims = [4] * 8
    X = orc.gen_uniform(11, dims)
    a = tt.tt_svd_tsqr(X, dims, (16, 0.0))
    T, _ = run_both(tt, orc, X, dims, 16)
    for ca, cb in zip(a.cores, T.cores):
        assert np.array_equal(ca.data, cb.data)


def test_host_entry_chunked_h2d_matches_device_entry(tt, orc):
    # a first step on the TMA-staged stream kernel (2^20 x 16): the host entry
    # copies X in row chunks under the first TSQR (running factors carried
    # between the chunk launches) — same bytes out as the device entry
    import torch
    dims = [16] * 6
    X = orc.gen_uniform(13, dims)
    a = tt.tt_svd_tsqr(X, dims, (8, 0.0))
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    rows = int(np.prod(dims)) // dims[-1]
    b = tt.tt_svd_tsqr(Xd[:rows], dims, tt.TruncationSpec(r_max=8))
    assert a.ranks() == b.ranks()
    for ca, cb in zip(a.cores, b.cores):
        assert np.array_equal(ca.data, cb.data)
    for sa, sb in zip(a.sigmas, b.sigmas):
        assert np.array_equal(sa, sb)
    # and again (the chunk state buffer is reused)
    c = tt.tt_svd_tsqr(X, dims, (8, 0.0))
    for ca, cc in zip(a.cores, c.cores):
        assert np.array_equal(ca.data, cc.data)


def test_zero_tensor(tt, orc):
    dims = [3, 4, 5]
    X = np.zeros((64, 5), order="F")
    T, o = run_both(tt, orc, X, dims, 4)
    assert T.ranks() == o[0]
    for c in T.cores:
        assert np.all(np.isfinite(c.data))


def test_degenerate_dimension(tt):
    with pytest.raises(tt.DegenerateDimension):
        tt.tt_svd_tsqr(np.zeros((64, 5), order="F"), [5], (1, 0.0))


def test_wide_steps_and_odd_shapes(tt, orc):
    # rows < cols steps at the chain end (tt_svd.hpp:91-103), odd extents
    from oracle.oracle import random_tensor
    dims = [3, 5, 7, 2, 9]
    X = random_tensor(113, dims)
    for r_max in (1, 2, 5, 2 ** 62):
        T, o = run_both(tt, orc, X, dims, r_max)
        assert_parity(tt, orc, X, dims, T, o)


# Steps that reach every small-SVD kernel: the cluster block Jacobi for
# m >= 96 (tall steps on R^T and wide steps on W^T, m and n not multiples of
# 4 or 8), the single-CTA shared-memory kernel, and the cooperative kernel
# for a wide W^T too large for one CTA's shared memory.
@pytest.mark.parametrize("dims,r_max", [([6, 7, 9, 13, 11], 400), ([2] * 16, 200), ([4] * 9, 130),
                                        ([7, 11, 13, 17], 300)])
def test_svd_kernel_shapes(tt, orc, dims, r_max):
    from oracle.oracle import random_tensor
    X = random_tensor(211 + len(dims), dims)
    T, o = run_both(tt, orc, X, dims, r_max)
    assert_parity(tt, orc, X, dims, T, o, err_tol=1e-9)


def test_exact_tt_rank32_scaled_config2(tt, orc):
    # config 2's structure at a reduced size: 16^5, exact TT rank 8 + 1e-8 noise
    rng = np.random.default_rng(2)
    dims = [16] * 5
    ranks = [1, 8, 8, 8, 8, 1]
    cores = [rng.standard_normal((ranks[j], 16, ranks[j + 1])) for j in range(5)]
    from oracle.oracle import tt_reconstruct
    X = tt_reconstruct([np.asfortranarray(c) for c in cores], dims)
    rows = 16 ** 4
    nrm = np.linalg.norm(X[:rows])
    X[:rows] += rng.standard_normal((rows, 16)) * (1e-8 * nrm / np.sqrt(16 ** 5))
    T, o = run_both(tt, orc, X, dims, 8)
    assert T.ranks() == ranks
    e_gpu, e_ref = assert_parity(tt, orc, X, dims, T, o, err_tol=1e-8)
    assert e_gpu <= 1e-7


# ----------------------------------------------------------- distributed ----
def test_distributed_matches_unsplit_c08(tt, orc, ref):
    # acceptance_test.cpp:311-340: (4, 2^12) split over 4 partitions
    import torch
    from oracle.oracle import random_tensor
    gdims = [4] + [2] * 12
    glob = random_tensor(2718, gdims)
    slabs, ldims, ld = split_slabs(glob, gdims, 4)
    rows = int(np.prod(ldims)) // ldims[-1]
    dev = [torch.from_numpy(np.ascontiguousarray(s.T)).cuda().t()[:rows] for s in slabs]
    T = tt.tt_svd_distributed(dev, ldims, (4, 0.0))
    rr, rcores = ref.tt_svd_distributed(slabs, ldims, ld, 4)
    assert T.ranks() == rr
    e_gpu = rel_error(glob, gdims, cores_of(T))
    e_ref = orc.tt_error(glob, glob.shape[0], gdims, rr, rcores)
    assert abs(e_gpu - e_ref) <= 1e-10
    assert max(frame_angles(cores_of(T), rcores)) <= 1e-8
    # every partition sees the same combined R -> shared cores identical
    T2 = tt.tt_svd_distributed(dev, ldims, (4, 0.0))
    for a, b in zip(T.cores, T2.cores):
        assert np.array_equal(a.data, b.data)


def test_distributed_single_partition(tt, orc):
    # test_tt_svd.cpp:237-251: one partition == tt_svd_tsqr on (1, dims)
    import torch
    from oracle.oracle import random_tensor
    dims = [2] * 8
    X = random_tensor(107, dims)
    rows = 2 ** 7
    dev = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()[:rows]
    a = tt.tt_svd_distributed([dev], dims, (3, 0.0))
    b = tt.tt_svd_tsqr(dev, [1] + dims, (3, 0.0))
    assert a.ranks() == b.ranks()
    for ca, cb in zip(a.cores, b.cores):
        assert np.array_equal(ca.data, cb.data)


def test_distributed_partition_mismatch(tt):
    import torch
    a = torch.zeros((5, 64), dtype=torch.float64, device="cuda").t()[:2]
    b = torch.zeros((6, 64), dtype=torch.float64, device="cuda").t()[:2]
    with pytest.raises(tt.PartitionMismatch):
        tt.tt_svd_distributed([a, b], [2, 5], (2, 0.0))


# ------------------------------------------------- committed golden fixtures ----
GOLD = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.abspath(__file__)), "golden",
                                  "reference_golden.npz")


@pytest.mark.parametrize("name,seed,dims,rmax,eps", [("tt_2pow12_seed43_r4", 43, [2] * 12, 4, 0.0),
                                                     ("tt_2pow16_seed4242_r5", 4242, [2] * 16, 5, 0.0),
                                                     ("tt_2x3x4x5x6_seed113_r5", 113, [2, 3, 4, 5, 6], 5, 0.0),
                                                     ("tt_4pow6_seed5001_r8_eps1e-2", 5001, [4] * 6, 8, 1e-2)])
def test_gpu_vs_reference_golden(tt, name, seed, dims, rmax, eps):
    """GPU result vs outputs the reference itself produced (tests/golden/)."""
    import torch
    from oracle.oracle import random_tensor, split_cores
    g = np.load(GOLD)
    X = random_tensor(seed, dims)
    rows = int(np.prod(dims)) // dims[-1]
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()[:rows]
    T = tt.tt_svd_tsqr(Xd, dims, (rmax, eps))
    ranks = g[f"{name}_ranks"].tolist()
    assert T.ranks() == ranks
    ref_cores = split_cores(g[f"{name}_cores"], dims, ranks)
    assert abs(rel_error(X, dims, cores_of(T)) - float(g[f"{name}_error"])) <= 1e-10
    assert max(frame_angles(cores_of(T), ref_cores)) <= 1e-8


def test_gpu_config1_vs_reference_golden(tt, orc):
    import torch
    from oracle.oracle import split_cores
    g = np.load(GOLD)
    dims = [4] * 10
    X = orc.gen_uniform(1, dims)
    Xd = tt.gen_uniform(1, dims)  # the device generator must give the same bytes
    full = Xd.as_strided((Xd.stride(1), dims[-1]), (1, Xd.stride(1))).cpu().numpy()
    assert np.array_equal(full, X)
    T = tt.tt_svd_tsqr(Xd, dims, (16, 0.0))
    ranks = g["cfg1_ranks"].tolist()
    assert T.ranks() == ranks
    sig = np.concatenate(T.sigmas)
    assert np.max(np.abs(sig - g["cfg1_sigma"])) <= 1e-10 * np.max(g["cfg1_sigma"])
    assert abs(rel_error(X, dims, cores_of(T)) - float(g["cfg1_error"])) <= 1e-10
    assert max(frame_angles(cores_of(T), split_cores(g["cfg1_cores"], dims, ranks))) <= 1e-8


def test_distributed_exchange_callback_path(tt):
    """The multi-process code path of ttsvd_cu_tt_svd_distributed (exchange
    callback through ctypes, device pointers wrapped as torch tensors) on one
    GPU: a callback that plays four ranks holding identical slabs must give
    the in-process four-slab result bitwise (which test_distributed_* pin to
    the reference)."""
    import torch
    from oracle.oracle import padded_stride
    # global (2, 4, 4, 4): both partitions equal -> slab s twice
    from oracle.oracle import random_tensor
    ldims = [4, 4, 4]
    s = random_tensor(31, ldims)
    rows = 16
    dev = torch.from_numpy(np.ascontiguousarray(s.T)).cuda().t()[:rows]
    calls = []

    def dup(send, recv):  # rank-ordered all-gather of four identical ranks
        calls.append(send.numel())
        for q in range(4):
            recv[q * send.numel():(q + 1) * send.numel()].copy_(send)

    a = tt.tt_svd_distributed([dev], ldims, (4, 0.0), P_total=4, exchange=dup)
    b = tt.tt_svd_distributed([dev] * 4, ldims, (4, 0.0))
    assert len(calls) == len(ldims) + 1  # one R exchange per step + the final gather
    assert a.ranks() == b.ranks()
    for ca, cb in zip(a.cores, b.cores):
        assert np.array_equal(ca.data, cb.data)
