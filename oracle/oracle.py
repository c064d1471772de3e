"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* ``Oracle("restated")`` loads oracle/_build/libttsvd_oracle.so, the plain-C
  restatement of the reference path (oracle/ttsvd_oracle.c);
* ``Oracle("reference")`` loads oracle/_ref/libttsvd_ref.so, the reference
  headers themselves compiled by oracle/Makefile (oracle/ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  The product package
(paper_2102_00104_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restated": os.path.join(HERE, "_build", "libttsvd_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "libttsvd_ref.so"),
}

i64 = C.c_int64
dptr = C.POINTER(C.c_double)
i64ptr = C.POINTER(C.c_int64)


class Step(C.Structure):
    _fields_ = [("rows", i64), ("cols", i64), ("nsig", i64), ("rank", i64)]


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a: np.ndarray):
    return a.ctypes.data_as(dptr)


def _pi(a: np.ndarray):
    return a.ctypes.data_as(i64ptr)


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: status {code}")
        self.code = code


def padded_stride(n: int) -> int:
    """shape.hpp:22-28, restated for the tests' own layout bookkeeping."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if n <= 64:
        return 64
    q = (n + 63) // 64
    if q % 2 == 0:
        q += 1
    return 64 * q


class Oracle:
    def __init__(self, kind: str = "restated"):
        path = LIBS[kind]
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.kind = kind
        self.pre = "orc_" if kind == "restated" else "ref_"
        self.lib = C.CDLL(path)
        L = self.lib
        f = self._f
        f("padded_stride").restype = i64
        f("padded_stride").argtypes = [i64]
        f("block_nb").restype = i64
        f("block_nb").argtypes = [i64, i64]
        f("reduce_block").argtypes = [dptr, i64, i64, i64, dptr, i64, dptr]
        f("combine_factors").argtypes = [dptr, i64, i64, dptr]
        f("tsqr").argtypes = [dptr, i64, i64, i64, i64, C.c_int, dptr]
        f("jacobi_svd").argtypes = [dptr, i64, i64, i64, dptr, dptr, dptr]
        f("select_rank").restype = i64
        f("select_rank").argtypes = [dptr, i64, C.c_double, i64]
        f("derive_delta").argtypes = [C.c_double, C.c_double, i64, dptr]
        f("tt_error").restype = C.c_double
        f("tt_error").argtypes = [dptr, i64, i64ptr, i64, i64ptr, dptr]
        if kind == "restated":
            f("tsmm_reshape").argtypes = [dptr, i64, i64, i64, dptr, i64, i64, dptr, i64, i64, i64]
            f("tt_svd_tsqr").argtypes = [dptr, i64ptr, i64, i64, i64, C.c_double, C.c_int, i64ptr, dptr, i64,
                                         i64ptr, C.POINTER(Step), dptr, i64]
            f("tt_svd_distributed").argtypes = [C.POINTER(dptr), i64, i64ptr, i64, i64, i64, C.c_double, C.c_int,
                                                i64ptr, dptr, i64, i64ptr, C.POINTER(Step), dptr, i64]
            f("gen_uniform").argtypes = [C.c_uint64, i64, i64, i64, dptr]
            f("choose_rank").restype = i64
            f("choose_rank").argtypes = [dptr, i64, i64, i64, C.c_double, i64, i64]
            f("tt_reconstruct").argtypes = [i64ptr, i64, i64ptr, dptr, dptr]
            f("random_tensor").argtypes = [C.c_uint64, i64, i64, i64, dptr]
            f("mt_gaussian").argtypes = [C.c_uint64, i64, dptr]
            f("mt_uniform").argtypes = [C.c_uint64, i64, C.c_double, dptr]
        else:
            f("tsmm_reshape").argtypes = [dptr, i64, i64, i64, dptr, i64, i64, dptr, i64, i64, i64, C.c_int]
            f("tt_svd_tsqr").argtypes = [dptr, i64ptr, i64, i64, i64, C.c_double, C.c_int, i64ptr, dptr, i64,
                                         i64ptr, C.POINTER(Step)]
            f("tt_svd_tsqr_sigma").argtypes = [dptr, i64ptr, i64, i64, i64, C.c_double, C.c_int, i64ptr, dptr, i64,
                                               i64ptr, dptr, i64, i64ptr]
            f("tt_svd_distributed").argtypes = [C.POINTER(dptr), i64, i64ptr, i64, i64, i64, C.c_double, C.c_int,
                                                i64ptr, dptr, i64, i64ptr]
            f("set_budget").argtypes = [i64]
            f("tensor_new").restype = C.c_void_p
            f("tensor_new").argtypes = [dptr, i64ptr, i64, i64]
            f("tensor_free").argtypes = [C.c_void_p]
            f("tt_svd_tsqr_tensor").argtypes = [C.c_void_p, i64, C.c_double, C.c_int, i64ptr]
            f("choose_combined_dims").argtypes = [i64ptr, i64, i64, C.c_double, C.c_void_p, i64, i64, i64ptr, i64ptr]
            f("tt_svd_thick_bounds").argtypes = [dptr, i64ptr, i64, i64, i64, C.c_double, i64, C.c_double,
                                                 C.c_void_p, i64, C.c_int, i64ptr, dptr, i64, i64ptr]
            f("tt_svd_two_sided").argtypes = [dptr, i64ptr, i64, i64, i64, C.c_double, C.c_int, i64ptr, dptr, i64,
                                              i64ptr]
            f("transpose_reorder").argtypes = [dptr, i64, i64, i64, dptr, i64, i64, i64, C.c_int]
            L.ref_set_budget(1 << 40)

    def _f(self, name):
        return getattr(self.lib, self.pre + name)

    @staticmethod
    def _check(rc: int, where: str):
        if rc != 0:
            raise OracleError(rc, where)

    # ---- building blocks -------------------------------------------------
    def padded_stride(self, n: int) -> int:
        return int(self._f("padded_stride")(n))

    def block_nb(self, m: int, budget: int = 256 * 1024) -> int:
        return int(self._f("block_nb")(m, budget))

    def reduce_block(self, M: np.ndarray, R: np.ndarray) -> np.ndarray:
        M = np.asfortranarray(M, dtype=np.float64)
        R = np.asfortranarray(R, dtype=np.float64)
        out = np.zeros((M.shape[1], M.shape[1]), order="F")
        self._check(self._f("reduce_block")(_p(M), M.shape[0], M.shape[1], max(M.shape[0], 1), _p(R), R.shape[0],
                                            _p(out)), "reduce_block")
        return out

    def combine_factors(self, parts: list[np.ndarray]) -> np.ndarray:
        m = parts[0].shape[0]
        buf = np.concatenate([np.asfortranarray(p).reshape(-1, order="F") for p in parts])
        out = np.zeros((m, m), order="F")
        self._check(self._f("combine_factors")(_p(buf), len(parts), m, _p(out)), "combine_factors")
        return out

    def tsqr(self, X: np.ndarray, ld: int | None = None, n_b: int | None = None, workers: int = 1,
             n: int | None = None, m: int | None = None) -> np.ndarray:
        """X is either a Fortran (n x m) array or a padded buffer with (n, m, ld)."""
        if ld is None:
            X = np.asfortranarray(X, dtype=np.float64)
            n, m = X.shape
            ld = max(n, 1)
        if n_b is None:
            n_b = self.block_nb(m)
        out = np.zeros((m, m), order="F")
        self._check(self._f("tsqr")(_p(X), n, m, ld, n_b, workers, _p(out)), "tsqr")
        return out

    def jacobi_svd(self, A: np.ndarray, want_u: bool = True):
        A = np.asfortranarray(A, dtype=np.float64)
        n, m = A.shape
        sigma = np.zeros(m)
        U = np.zeros((n, m), order="F") if want_u else None
        V = np.zeros((m, m), order="F")
        self._check(self._f("jacobi_svd")(_p(A), n, m, max(n, 1), _p(sigma), _p(U) if want_u else None, _p(V)),
                    "jacobi_svd")
        return sigma, U, V

    def select_rank(self, sigma, delta: float, r_max: int) -> int:
        s = np.ascontiguousarray(sigma, dtype=np.float64)
        return int(self._f("select_rank")(_p(s), len(s), delta, r_max))

    def derive_delta(self, norm: float, eps: float, d: int) -> float:
        out = C.c_double()
        self._check(self._f("derive_delta")(norm, eps, d, C.byref(out)), "derive_delta")
        return out.value

    def tsmm_reshape(self, X: np.ndarray, V: np.ndarray, out_rows: int, out_cols: int, workers: int = 1,
                     n: int | None = None, ld: int | None = None) -> np.ndarray:
        """Returns the padded (ld x out_cols) output buffer, Fortran order.
        With n and ld, X is a padded (ld x m) Fortran buffer holding n rows."""
        V = np.asfortranarray(V, dtype=np.float64)
        if ld is None:
            X = np.asfortranarray(X, dtype=np.float64)
            n, m = X.shape
            ld = max(n, 1)
        else:
            assert X.flags.f_contiguous and X.shape[0] == ld
            m = X.shape[1]
        k = V.shape[1]
        ldy = padded_stride(out_rows)
        Y = np.zeros((ldy, out_cols), order="F")
        if self.kind == "restated":
            rc = self._f("tsmm_reshape")(_p(X), n, m, ld, _p(V), k, max(V.shape[0], 1), _p(Y), out_rows,
                                         out_cols, ldy)
        else:
            rc = self._f("tsmm_reshape")(_p(X), n, m, ld, _p(V), k, max(V.shape[0], 1), _p(Y), out_rows,
                                         out_cols, ldy, workers)
        self._check(rc, "tsmm_reshape")
        return Y

    # ---- drivers ---------------------------------------------------------
    def tt_svd_tsqr(self, X: np.ndarray, dims, ld: int, r_max: int, eps: float = 0.0, workers: int = 1,
                    with_sigma: bool = False):
        """X: padded Fortran buffer (ld x n_d) of the tensor with shape dims.
        Returns (ranks, cores list, steps, sigmas-per-step or None)."""
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        d = len(dims)
        ranks = np.zeros(d + 1, dtype=np.int64)
        need = np.zeros(1, dtype=np.int64)
        steps = (Step * max(d - 1, 1))()
        total = int(np.prod(dims))
        cap = max(1, min(total, 1 << 22))
        sig_cap = 1 << 20
        while True:
            cores = np.zeros(cap)
            if self.kind == "restated":
                sig = np.zeros(max(sig_cap, 1) if with_sigma else 1)
                rc = self._f("tt_svd_tsqr")(_p(X), _pi(dims), d, ld, r_max, eps, workers, _pi(ranks), _p(cores),
                                            cap, _pi(need), steps, _p(sig) if with_sigma else None,
                                            sig_cap if with_sigma else 0)
            else:
                sig = None
                rc = self._f("tt_svd_tsqr")(_p(X), _pi(dims), d, ld, r_max, eps, workers, _pi(ranks), _p(cores),
                                            cap, _pi(need), steps)
            if rc == 11:
                cap = int(need[0])
                continue
            self._check(rc, "tt_svd_tsqr")
            break
        core_list = split_cores(cores, dims, ranks)
        step_list = [(s.rows, s.cols, s.nsig, s.rank) for s in steps][: d - 1]
        sig_list = None
        if with_sigma and sig is not None:
            sig_list, off = [], 0
            for (_, _, nsig, _) in step_list:
                sig_list.append(sig[off:off + nsig].copy())
                off += nsig
        return ranks.tolist(), core_list, step_list, sig_list

    def tt_svd_tsqr_sigma(self, X: np.ndarray, dims, ld: int, r_max: int, eps: float = 0.0, workers: int = 1):
        """The reference's Alg. 2 run step by step from its own functions
        (ref_shim.cpp ref_tt_svd_tsqr_sigma) with `workers` host threads:
        (ranks, cores, sigmas per step).  Reference library only."""
        assert self.kind == "reference"
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        d = len(dims)
        ranks = np.zeros(d + 1, dtype=np.int64)
        need = np.zeros(1, dtype=np.int64)
        nsig = np.zeros(max(d - 1, 1), dtype=np.int64)
        total = int(np.prod(dims))
        cap = max(1, min(total, 1 << 22))
        sig_cap = 1 << 20
        while True:
            cores = np.zeros(cap)
            sig = np.zeros(sig_cap)
            rc = self._f("tt_svd_tsqr_sigma")(_p(X), _pi(dims), d, ld, r_max, eps, workers, _pi(ranks), _p(cores),
                                              cap, _pi(need), _p(sig), sig_cap, _pi(nsig))
            if rc == 11:
                cap = max(cap, int(need[0]))
                sig_cap = max(sig_cap, int(nsig.sum()))
                continue
            self._check(rc, "tt_svd_tsqr_sigma")
            break
        sig_list, off = [], 0
        for k in nsig[: d - 1]:
            sig_list.append(sig[off:off + int(k)].copy())
            off += int(k)
        return ranks.tolist(), split_cores(cores, dims, ranks), sig_list

    def tt_svd_distributed(self, slabs: list[np.ndarray], ldims, ld: int, r_max: int, eps: float = 0.0,
                           workers: int = 1):
        ldims = np.ascontiguousarray(ldims, dtype=np.int64)
        P = len(slabs)
        d = len(ldims) + 1
        ranks = np.zeros(d + 1, dtype=np.int64)
        need = np.zeros(1, dtype=np.int64)
        arr = (dptr * P)(*[_p(s) for s in slabs])
        cap = 1 << 16
        gdims = np.concatenate([[P], ldims]).astype(np.int64)
        while True:
            cores = np.zeros(cap)
            if self.kind == "restated":
                rc = self._f("tt_svd_distributed")(arr, P, _pi(ldims), len(ldims), ld, r_max, eps, workers,
                                                   _pi(ranks), _p(cores), cap, _pi(need), None, None, 0)
            else:
                rc = self._f("tt_svd_distributed")(arr, P, _pi(ldims), len(ldims), ld, r_max, eps, workers,
                                                   _pi(ranks), _p(cores), cap, _pi(need))
            if rc == 11:
                cap = int(need[0])
                continue
            self._check(rc, "tt_svd_distributed")
            break
        if P == 1:
            gdims[0] = 1
        return ranks.tolist(), split_cores(cores, gdims, ranks)

    def choose_combined_dims(self, dims, m_min: int = 16, f1_min: float = 0.5, r_tilde=(), r_max: int = 2 ** 62):
        """Reference only (tt_svd.hpp:316-330)."""
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        rt = np.ascontiguousarray(r_tilde, dtype=np.int64)
        k, m = np.zeros(1, dtype=np.int64), np.zeros(1, dtype=np.int64)
        self._check(self._f("choose_combined_dims")(_pi(dims), len(dims), m_min, f1_min,
                                                    rt.ctypes.data if len(rt) else None, len(rt), r_max, _pi(k),
                                                    _pi(m)), "choose_combined_dims")
        return int(k[0]), int(m[0])

    def tt_svd_thick_bounds(self, X: np.ndarray, dims, ld: int, r_max: int, eps: float = 0.0, m_min: int = 16,
                            f1_min: float = 0.5, r_tilde=(), workers: int = 1):
        """Reference only (tt_svd.hpp:338, Alg. 3).  Returns (ranks, cores)."""
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        rt = np.ascontiguousarray(r_tilde, dtype=np.int64)
        d = len(dims)
        ranks = np.zeros(d + 1, dtype=np.int64)
        need = np.zeros(1, dtype=np.int64)
        cap = max(1, min(int(np.prod(dims)), 1 << 22))
        while True:
            cores = np.zeros(cap)
            rc = self._f("tt_svd_thick_bounds")(_p(X), _pi(dims), d, ld, r_max, eps, m_min, f1_min,
                                                rt.ctypes.data if len(rt) else None, len(rt), workers, _pi(ranks),
                                                _p(cores), cap, _pi(need))
            if rc == 11:
                cap = int(need[0])
                continue
            self._check(rc, "tt_svd_thick_bounds")
            break
        return ranks.tolist(), split_cores(cores, dims, ranks)

    def tt_svd_two_sided(self, X: np.ndarray, dims, ld: int, r_max: int, eps: float = 0.0, workers: int = 1):
        """Reference only (tt_svd.hpp:402-512, Alg. 4).  Returns (ranks, cores)."""
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        d = len(dims)
        ranks = np.zeros(d + 1, dtype=np.int64)
        need = np.zeros(1, dtype=np.int64)
        cap = max(1, min(int(np.prod(dims)), 1 << 22))
        while True:
            cores = np.zeros(cap)
            rc = self._f("tt_svd_two_sided")(_p(X), _pi(dims), d, ld, r_max, eps, workers, _pi(ranks), _p(cores),
                                             cap, _pi(need))
            if rc == 11:
                cap = int(need[0])
                continue
            self._check(rc, "tt_svd_two_sided")
            break
        return ranks.tolist(), split_cores(cores, dims, ranks)

    def transpose_reorder(self, W: np.ndarray, out_rows: int, out_cols: int, workers: int = 1) -> np.ndarray:
        """Reference only (tsmm.hpp:84-126): the padded (ld x out_cols) output."""
        W = np.asfortranarray(W, dtype=np.float64)
        n, m = W.shape
        ldy = padded_stride(out_rows)
        Y = np.zeros((ldy, out_cols), order="F")
        self._check(self._f("transpose_reorder")(_p(W), n, m, max(n, 1), _p(Y), out_rows, out_cols, ldy, workers),
                    "transpose_reorder")
        return Y

    def tt_error(self, X: np.ndarray, ld: int, dims, ranks, cores: list[np.ndarray]) -> float:
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        ranks = np.ascontiguousarray(ranks, dtype=np.int64)
        flat = np.concatenate([np.asarray(c, dtype=np.float64).reshape(-1, order="F") for c in cores])
        return float(self._f("tt_error")(_p(X), ld, _pi(dims), len(dims), _pi(ranks), _p(flat)))

    def gen_uniform(self, seed: int, dims, ld: int | None = None) -> np.ndarray:
        dims = [int(x) for x in dims]
        total = int(np.prod(dims))
        rows = total // dims[-1]
        ld = ld or padded_stride(rows)
        out = np.zeros((ld, dims[-1]), order="F")
        self._f("gen_uniform")(seed, total, rows, ld, _p(out))
        return out


# ---- reference test-input generators (restated; pinned in test_oracle_pin) ----
def _orc() -> "Oracle":
    global _ORC
    try:
        return _ORC
    except NameError:
        _ORC = Oracle("restated")
        return _ORC


def random_tensor(seed: int, dims, ld: int | None = None) -> np.ndarray:
    """storage.hpp:202-212 — padded (ld x n_d) Fortran buffer, entries in [0,1)."""
    dims = [int(x) for x in dims]
    total = int(np.prod(dims))
    rows = total // dims[-1]
    ld = ld or padded_stride(rows)
    out = np.zeros((ld, dims[-1]), order="F")
    _orc().lib.orc_random_tensor(seed, total, rows, ld, _p(out))
    return out


def gaussian(rows: int, cols: int, seed: int) -> np.ndarray:
    """tests/oracles.hpp:75-83"""
    out = np.zeros(rows * cols)
    _orc().lib.orc_mt_gaussian(seed, rows * cols, _p(out))
    return out.reshape((rows, cols), order="F")


def uniform(rows: int, cols: int, seed: int) -> np.ndarray:
    """tests/oracles.hpp:85-90"""
    out = np.zeros(rows * cols)
    _orc().lib.orc_mt_uniform(seed, rows * cols, 0.0, _p(out))
    return out.reshape((rows, cols), order="F")


def orthonormal(rows: int, cols: int, seed: int) -> np.ndarray:
    """tests/oracles.hpp:93-110 — two-pass MGS of gaussian(rows, cols, seed)."""
    q = gaussian(rows, cols, seed).copy(order="F")
    for j in range(cols):
        for _ in range(2):
            for k in range(j):
                dot = 0.0
                for i in range(rows):
                    dot += q[i, k] * q[i, j]
                q[:, j] -= dot * q[:, k]
        nrm = float(np.sqrt(sum(float(x) * float(x) for x in q[:, j])))
        q[:, j] /= nrm
    return q


def with_singular_values(rows: int, cols: int, sv, seed: int) -> np.ndarray:
    """tests/oracles.hpp:113-126"""
    u = orthonormal(rows, cols, seed)
    v = orthonormal(cols, cols, seed + 1)
    return np.asfortranarray((u * np.asarray(sv)[None, :]) @ v.T)


def random_tt(dims, ranks, seed: int) -> list[np.ndarray]:
    """tests/oracles.hpp:144-154 — cores with entries in [-0.5, 0.5)."""
    total = sum(int(ranks[j]) * int(n) * int(ranks[j + 1]) for j, n in enumerate(dims))
    flat = np.zeros(total)
    _orc().lib.orc_mt_uniform(seed, total, -0.5, _p(flat))
    return split_cores(flat, dims, ranks)


def tt_reconstruct(cores, dims, ld: int | None = None) -> np.ndarray:
    """tensor_train.hpp:80-110, returned in the padded tensor layout."""
    dims = np.ascontiguousarray(dims, dtype=np.int64)
    ranks = np.asarray([1] + [c.shape[2] for c in cores], dtype=np.int64)
    total = int(np.prod(dims))
    flat = np.zeros(total)
    buf = np.concatenate([np.asarray(c, dtype=np.float64).reshape(-1, order="F") for c in cores])
    rc = _orc().lib.orc_tt_reconstruct(_pi(dims), len(dims), _pi(ranks), _p(buf), _p(flat))
    if rc != 0:
        raise OracleError(rc, "tt_reconstruct")
    rows = total // int(dims[-1])
    ld = ld or padded_stride(rows)
    out = np.zeros((ld, int(dims[-1])), order="F")
    out[:rows, :] = flat.reshape((rows, int(dims[-1])), order="F")
    return out


def split_cores(flat: np.ndarray, dims, ranks) -> list[np.ndarray]:
    """Core j as a Fortran (r_j, n_j, r_{j+1}) array (tensor_train.hpp:24-29)."""
    out, off = [], 0
    for j, n in enumerate(dims):
        rl, rr = int(ranks[j]), int(ranks[j + 1])
        sz = rl * int(n) * rr
        out.append(flat[off:off + sz].reshape((rl, int(n), rr), order="F").copy())
        off += sz
    return out


# ---- wire formats through the reference's own writers/readers ---------------
class RefWire:
    """save_tt / load_tt / dump_tensor / load_tensor of the compiled reference
    (storage.hpp:214-278, tensor_train.hpp:157-191), for cross-reading files
    written by the package."""

    def __init__(self):
        path = LIBS["reference"]
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_save_tt.argtypes = [C.c_char_p, i64, i64ptr, i64ptr, dptr]
        L.ref_load_tt.argtypes = [C.c_char_p, i64ptr, i64ptr, i64ptr, dptr, i64, i64ptr]
        L.ref_dump_tensor.argtypes = [C.c_char_p, dptr, i64ptr, i64, i64]
        L.ref_load_tensor.argtypes = [C.c_char_p, i64ptr, i64ptr, i64ptr, dptr, i64]

    def save_tt(self, path: str, cores: list) -> None:
        d = len(cores)
        ranks = np.array([cores[0].shape[0]] + [c.shape[2] for c in cores], dtype=np.int64)
        dims = np.array([c.shape[1] for c in cores], dtype=np.int64)
        flat = np.concatenate([np.asarray(c).reshape(-1, order="F") for c in cores])
        rc = self.lib.ref_save_tt(path.encode(), d, _pi(ranks), _pi(dims), _p(flat))
        if rc:
            raise OracleError(rc, "ref_save_tt")

    def load_tt(self, path: str) -> list:
        d = np.zeros(1, dtype=np.int64)
        ranks = np.zeros(65, dtype=np.int64)
        dims = np.zeros(64, dtype=np.int64)
        need = np.zeros(1, dtype=np.int64)
        buf = np.zeros(1)
        rc = self.lib.ref_load_tt(path.encode(), _pi(d), _pi(ranks), _pi(dims), _p(buf), 0, _pi(need))
        if rc not in (0, 11):
            raise OracleError(rc, "ref_load_tt")
        buf = np.zeros(int(need[0]))
        rc = self.lib.ref_load_tt(path.encode(), _pi(d), _pi(ranks), _pi(dims), _p(buf), buf.size, _pi(need))
        if rc:
            raise OracleError(rc, "ref_load_tt")
        cores, off = [], 0
        for j in range(int(d[0])):
            rl, n, rr = int(ranks[j]), int(dims[j]), int(ranks[j + 1])
            cores.append(buf[off:off + rl * n * rr].reshape((rl, n, rr), order="F"))
            off += rl * n * rr
        return cores

    def dump_tensor(self, path: str, X: np.ndarray, dims, ld: int) -> None:
        dv = np.asarray(dims, dtype=np.int64)
        Xf = np.asfortranarray(X)
        rc = self.lib.ref_dump_tensor(path.encode(), _p(Xf), _pi(dv), dv.size, ld)
        if rc:
            raise OracleError(rc, "ref_dump_tensor")

    def load_tensor(self, path: str):
        """-> (padded buffer as a Fortran (ld x n_d) array, dims)"""
        d = np.zeros(1, dtype=np.int64)
        dims = np.zeros(64, dtype=np.int64)
        ld = np.zeros(1, dtype=np.int64)
        cap = os.path.getsize(path) // 8
        buf = np.zeros(cap)
        rc = self.lib.ref_load_tensor(path.encode(), _pi(d), _pi(dims), _pi(ld), _p(buf), cap)
        if rc:
            raise OracleError(rc, "ref_load_tensor")
        dd = [int(x) for x in dims[:int(d[0])]]
        return buf[:int(ld[0]) * dd[-1]].reshape((int(ld[0]), dd[-1]), order="F"), dd
