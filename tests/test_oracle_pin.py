"""Pin the oracle before trusting it (CPU, no GPU).

1. The C restatement (oracle/ttsvd_oracle.c) is BITWISE equal to the
   reference itself (oracle/_ref, compiled from /root/reference) on every
   building block and driver, and on the reference tests' input generators.
2. It reproduces the committed golden fixtures (tests/golden/, made by the
   reference through tests/golden/make_golden.py) — this leg also runs where
   /root/reference is absent.
3. It reproduces the known answers of the reference's own tests
   (test_tsqr.cpp, test_small_svd.cpp, test_tsmm.cpp, test_tt_svd.cpp,
   acceptance_test.cpp).
"""
import math
import os

import numpy as np
import pytest

from oracle.oracle import gaussian, padded_stride, random_tensor, random_tt, split_cores, tt_reconstruct, uniform

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


# ------------------------------------------------------- restated == ref ----
@pytest.mark.parametrize("n,m,w", [(1000, 3, 1), (5000, 6, 3), (100, 100, 1), (3000, 17, 4), (777, 64, 2),
                                   (4097, 1, 3), (50, 50, 2)])
def test_tsqr_bitwise_vs_reference(orc, ref, n, m, w):
    X = gaussian(n, m, n + m)
    assert np.array_equal(orc.tsqr(X, workers=w), ref.tsqr(X, workers=w))


def test_blocks_bitwise_vs_reference(orc, ref):
    m, r = gaussian(8, 3, 42), np.triu(gaussian(3, 3, 43))
    assert np.array_equal(orc.reduce_block(m, r), ref.reduce_block(m, r))
    parts = [np.triu(gaussian(5, 5, 7 + p)) for p in range(5)]
    assert np.array_equal(orc.combine_factors(parts), ref.combine_factors(parts))
    A = gaussian(40, 12, 1)
    for a, b in zip(orc.jacobi_svd(A), ref.jacobi_svd(A)):
        assert np.array_equal(a, b)
    A0 = np.zeros((6, 3))
    for a, b in zip(orc.jacobi_svd(A0), ref.jacobi_svd(A0)):
        assert np.array_equal(a, b)
    x, v = gaussian(300, 7, 2), gaussian(7, 4, 3)
    assert np.array_equal(orc.tsmm_reshape(x, v, 150, 8), ref.tsmm_reshape(x, v, 150, 8))
    for sig, delta, rmax in [([2, 1, .5, .1], .2, 10), ([2, 1, .5], 0., 2), ([5], 10., 3), ([3, 1e-17], 0., 9)]:
        assert orc.select_rank(sig, delta, rmax) == ref.select_rank(sig, delta, rmax)
    for n in (1, 63, 64, 65, 128, 192, 1000, 262144, 1 << 24):
        assert orc.padded_stride(n) == ref.padded_stride(n) == padded_stride(n)
    for m_ in (1, 7, 8, 16, 32, 64, 100, 128, 170, 256, 512, 4096):
        assert orc.block_nb(m_) == ref.block_nb(m_)


@pytest.mark.parametrize("dims,rmax,eps,seed", [([2] * 12, 4, 0.0, 43), ([4] * 6, 8, 1e-2, 5001),
                                                ([2, 3, 4, 5, 6], 5, 0.0, 113), ([8] * 4, 2 ** 62, 1e-1, 5002),
                                                ([3, 4, 5], 4, 0.0, 7)])
def test_drivers_bitwise_vs_reference(orc, ref, dims, rmax, eps, seed):
    X = random_tensor(seed, dims)
    for w in (1, 3):
        ra, ca, sa, _ = orc.tt_svd_tsqr(X, dims, X.shape[0], rmax, eps, workers=w)
        rb, cb, sb, _ = ref.tt_svd_tsqr(X, dims, X.shape[0], rmax, eps, workers=w)
        assert ra == rb
        assert all(np.array_equal(a, b) for a, b in zip(ca, cb))
        assert [s[3] for s in sa] == [s[3] for s in sb]
        # the step-by-step reference driver (the GPU parity tests' sigma
        # source) is the reference's tt_svd_tsqr, bitwise, and its sigmas are
        # the restatement's
        rc, cc, sc = ref.tt_svd_tsqr_sigma(X, dims, X.shape[0], rmax, eps, workers=w)
        assert rc == rb and all(np.array_equal(a, b) for a, b in zip(cc, cb))
        _, _, _, so = orc.tt_svd_tsqr(X, dims, X.shape[0], rmax, eps, workers=w, with_sigma=True)
        assert len(sc) == len(so) and all(np.array_equal(a, b) for a, b in zip(sc, so))


def test_distributed_bitwise_vs_reference(orc, ref):
    from helpers import split_slabs
    gd = [4] + [2] * 10
    glob = random_tensor(109, gd)
    slabs, ldims, ld = split_slabs(glob, gd, 4)
    ra, ca = orc.tt_svd_distributed(slabs, ldims, ld, 4)
    rb, cb = ref.tt_svd_distributed(slabs, ldims, ld, 4)
    assert ra == rb and all(np.array_equal(a, b) for a, b in zip(ca, cb))
    # one partition: the reference's (1, dims) degenerate path
    ra, ca = orc.tt_svd_distributed([slabs[0]], ldims, ld, 3)
    rb, cb = ref.tt_svd_distributed([slabs[0]], ldims, ld, 3)
    assert ra == rb and all(np.array_equal(a, b) for a, b in zip(ca, cb))


def test_generators_bitwise_vs_reference(ref):
    import ctypes as C
    dp = C.POINTER(C.c_double)
    a = np.zeros(999)
    ref.lib.ref_gaussian.argtypes = [C.c_int64, C.c_int64, C.c_uint64, dp]
    ref.lib.ref_gaussian(999, 1, 42, a.ctypes.data_as(dp))
    assert np.array_equal(gaussian(999, 1, 42).ravel(), a)
    ref.lib.ref_uniform.argtypes = [C.c_int64, C.c_int64, C.c_uint64, dp]
    ref.lib.ref_uniform(999, 1, 7, a.ctypes.data_as(dp))
    assert np.array_equal(uniform(999, 1, 7).ravel(), a)
    dims = np.array([2] * 10, dtype=np.int64)
    b = np.zeros((padded_stride(512), 2), order="F")
    ref.lib.ref_random_tensor.argtypes = [C.c_uint64, C.POINTER(C.c_int64), C.c_int64, dp, C.c_int64]
    ref.lib.ref_random_tensor(43, dims.ctypes.data_as(C.POINTER(C.c_int64)), 10, b.ctypes.data_as(dp), b.shape[0])
    assert np.array_equal(random_tensor(43, [2] * 10), b)


# ------------------------------------------------------- golden fixtures ----
def test_golden_building_blocks(orc, gold):
    X = gaussian(5000, 6, 5)
    assert np.array_equal(orc.tsqr(X, workers=1), gold["tsqr_5000x6_seed5_w1"])
    assert np.array_equal(orc.tsqr(X, workers=3), gold["tsqr_5000x6_seed5_w3"])
    assert np.array_equal(orc.reduce_block(gaussian(8, 3, 42), np.triu(gaussian(3, 3, 43))), gold["reduce_block_8x3"])
    parts = [np.triu(gaussian(4, 4, 100 + p)) for p in range(4)]
    assert np.array_equal(orc.combine_factors(parts), gold["combine_4x4_x4"])
    s, U, V = orc.jacobi_svd(gaussian(200, 5, 3))
    assert np.array_equal(s, gold["jacobi_200x5_sigma"]) and np.array_equal(U, gold["jacobi_200x5_U"])
    assert np.array_equal(V, gold["jacobi_200x5_V"])
    Y = orc.tsmm_reshape(gaussian(100, 6, 2), gaussian(6, 3, 3), 50, 6)
    assert np.array_equal(Y, gold["tsmm_100x6_6x3_50x6"])


@pytest.mark.parametrize("name,seed,dims,rmax,eps", [("tt_2pow12_seed43_r4", 43, [2] * 12, 4, 0.0),
                                                     ("tt_2pow16_seed4242_r5", 4242, [2] * 16, 5, 0.0),
                                                     ("tt_2x3x4x5x6_seed113_r5", 113, [2, 3, 4, 5, 6], 5, 0.0),
                                                     ("tt_4pow6_seed5001_r8_eps1e-2", 5001, [4] * 6, 8, 1e-2)])
def test_golden_drivers(orc, gold, name, seed, dims, rmax, eps):
    X = random_tensor(seed, dims)
    ranks, cores, _, _ = orc.tt_svd_tsqr(X, dims, X.shape[0], rmax, eps)
    assert ranks == gold[f"{name}_ranks"].tolist()
    flat = np.concatenate([c.reshape(-1, order="F") for c in cores])
    assert np.array_equal(flat, gold[f"{name}_cores"])
    assert orc.tt_error(X, X.shape[0], dims, ranks, cores) == float(gold[f"{name}_error"])


def test_golden_config1(orc, gold):
    dims = [4] * 10
    X = orc.gen_uniform(1, dims)
    ranks, cores, _, sig = orc.tt_svd_tsqr(X, dims, X.shape[0], 16, with_sigma=True)
    assert ranks == gold["cfg1_ranks"].tolist() == [1, 4, 16, 16, 16, 16, 16, 16, 16, 4, 1]
    assert np.array_equal(np.concatenate([c.reshape(-1, order="F") for c in cores]), gold["cfg1_cores"])
    assert np.array_equal(np.concatenate(sig), gold["cfg1_sigma"])


# ------------------------------------------- reference tests' known answers ----
def test_known_answers_tsqr(orc):
    # test_tsqr.cpp:28-44
    assert orc.reduce_block(np.array([[3.0], [4.0]]), np.zeros((1, 1)))[0, 0] == pytest.approx(-5.0, abs=1e-14)
    assert orc.reduce_block(np.zeros((5, 1)), np.array([[2.0]]))[0, 0] == 2.0
    # 71-79 embedded identity
    x = np.zeros((100, 4))
    x[:4, :4] = np.eye(4)
    r = orc.tsqr(x)
    assert np.allclose(np.abs(np.diag(r)), 1, atol=1e-14) and np.all(np.abs(np.triu(r, 1)) <= 1e-15)
    # 99-107 zero input, short input
    r = orc.tsqr(np.zeros((1000, 3)), workers=2)
    assert np.all(np.isfinite(r)) and np.linalg.norm(r) <= 1e-150
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        orc.tsqr(np.zeros((2, 3)))
    # 194-203 block sizing rule
    assert orc.block_nb(1) == 4096 and orc.block_nb(16) == 2032
    nb = orc.block_nb(100)
    assert (nb + 100) * 100 * 8 <= 256 * 1024 < (nb + 8 + 100) * 100 * 8


def test_known_answers_small_svd(orc):
    s, U, V = orc.jacobi_svd(np.diag([3.0, 2.0, 1.0]))
    assert np.allclose(s, [3, 2, 1], atol=1e-14)
    s, _, _ = orc.jacobi_svd(np.array([[1.0, 1.0], [0.0, 1.0]]))
    phi = (1 + math.sqrt(5)) / 2
    assert abs(s[0] - phi) <= 1e-14 and abs(s[1] - 1 / phi) <= 1e-14
    assert orc.select_rank([2, 1, 0.5, 0.1], 0.2, 10) == 3
    assert orc.select_rank([2, 1, 0.5], 0.0, 2) == 2
    assert orc.select_rank([5], 10.0, 3) == 1
    assert orc.derive_delta(123.0, 0.0, 7) == 0.0
    assert abs(orc.derive_delta(2.0, 0.1, 5) - 0.1) <= 1e-15


def test_known_answers_tsmm(orc):
    n = 1 << 12
    x = uniform(n, 8, 4)
    sel = np.zeros((8, 4))
    sel[np.arange(4), np.arange(4)] = 1.0
    y = orc.tsmm_reshape(x, sel, n // 2, 8)[: n // 2]
    assert np.array_equal(y.reshape(-1, order="F"), x[:, :4].reshape(-1, order="F"))


def test_known_answers_drivers(orc):
    # acceptance C07 (Table 2): 2^16, r_max 5 -> ranks end ..., 5, 5, 4, 2 and f = (1, 1, 5/8, 1/2)
    dims = [2] * 16
    X = random_tensor(4242, dims)
    ranks, cores, steps, _ = orc.tt_svd_tsqr(X, dims, X.shape[0], 5)
    assert ranks[-5:-1] == [5, 5, 4, 2]
    f = [s[3] / s[1] for s in steps]
    assert f[:4] == [1.0, 1.0, 5 / 8, 0.5]
    # C03 constructive recovery: TT (1,2,3,3,2,1,1) on 4^6
    d6 = [4] * 6
    Y = tt_reconstruct(random_tt(d6, [1, 2, 3, 3, 2, 1, 1], 777), d6)
    ranks, cores, _, _ = orc.tt_svd_tsqr(Y, d6, Y.shape[0], 3)
    assert ranks == [1, 2, 3, 3, 2, 1, 1]
    assert orc.tt_error(Y, Y.shape[0], d6, ranks, cores) <= 1e-12
    # test_tt_svd.cpp:290-303 rank caps
    d5 = [2, 3, 4, 5, 6]
    X = random_tensor(113, d5)
    for rmax in (1, 2, 5):
        r = orc.tt_svd_tsqr(X, d5, X.shape[0], rmax)[0]
        for i in range(1, len(r) - 1):
            assert r[i] <= min(rmax, int(np.prod(d5[:i])), int(np.prod(d5[i:])))


def test_split_cores_roundtrip():
    cores = random_tt([3, 4], [1, 2, 1], 1)
    flat = np.concatenate([c.reshape(-1, order="F") for c in cores])
    back = split_cores(flat, [3, 4], [1, 2, 1])
    assert all(np.array_equal(a, b) for a, b in zip(cores, back))
