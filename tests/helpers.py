"""Shared comparison helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np


def gram_residual(X: np.ndarray, R: np.ndarray) -> float:
    """||R^T R - X^T X||_F / ||X^T X||_F (test_tsqr.cpp:20-24, acceptance C04)."""
    gx = X.T @ X
    gr = R.T @ R
    return float(np.linalg.norm(gr - gx) / np.linalg.norm(gx))


def right_frames(cores: list[np.ndarray]) -> list[np.ndarray]:
    """F_i (r_{i-1} x n_i...n_d): contraction of cores i..d-1 (0-based), the
    gauge-invariant right interface of a TT-SVD (rows orthonormal)."""
    F = [None] * len(cores)
    nxt = np.ones((1, 1))
    for i in range(len(cores) - 1, 0, -1):
        c = cores[i]
        rl, n, rr = c.shape
        # F[a, x + n*L] = sum_b c[a, x, b] nxt[b, L]
        t = np.tensordot(c, nxt, axes=([2], [0]))  # rl x n x L
        F[i] = t.reshape(rl, n * nxt.shape[1], order="F")
        nxt = F[i]
    return F


def max_principal_angle(A: np.ndarray, B: np.ndarray) -> float:
    """Largest principal angle between the row spaces of A and B."""
    qa, _ = np.linalg.qr(A.T)
    qb, _ = np.linalg.qr(B.T)
    # sin of the largest angle = ||(I - Qa Qa^T) Qb||_2 (well conditioned near 0)
    resid = qb - qa @ (qa.T @ qb)
    s = np.linalg.norm(resid, 2) if resid.size else 0.0
    return float(np.arcsin(np.clip(s, 0.0, 1.0)))


def frame_angles(cores_a, cores_b) -> list[float]:
    fa, fb = right_frames(cores_a), right_frames(cores_b)
    return [max_principal_angle(fa[i], fb[i]) for i in range(1, len(cores_a))]


def column_angle(Va: np.ndarray, Vb: np.ndarray) -> float:
    """Largest principal angle between the column spaces of Va and Vb."""
    return max_principal_angle(Va.T, Vb.T)


def tt_full(cores: list[np.ndarray]) -> np.ndarray:
    """Flat (Fortran order) contraction of a train."""
    M = cores[0].reshape(cores[0].shape[1], cores[0].shape[2], order="F")  # n0 x r1
    for c in cores[1:]:
        M = _step(M, c)
    return M.reshape(-1, order="F")


def _step(M: np.ndarray, c: np.ndarray) -> np.ndarray:
    # M: N x rl ; result (N*n) x rr with row index i + N*x
    rl, n, rr = c.shape
    N = M.shape[0]
    out = np.einsum("ia,axb->ixb", M, c).reshape(N * n, rr, order="F")
    return out


def padded_to_flat(X: np.ndarray, dims) -> np.ndarray:
    total = int(np.prod(dims))
    rows = total // int(dims[-1])
    return np.asfortranarray(X[:rows, :]).reshape(-1, order="F")


def rel_error(X: np.ndarray, dims, cores) -> float:
    x = padded_to_flat(X, dims)
    y = tt_full(cores)
    return float(np.linalg.norm(x - y) / np.linalg.norm(x))


def split_slabs(glob: np.ndarray, gdims, P: int):
    """split_first_dim (ttsvd_bench.cpp:72-86): slab p holds global flat
    entries l -> p + P*l, each stored in its own padded layout."""
    from oracle.oracle import padded_stride
    ldims = list(gdims[1:])
    rest = int(np.prod(gdims)) // P
    rows = rest // ldims[-1]
    ld = padded_stride(rows)
    grows = int(np.prod(gdims)) // gdims[-1]
    flat = glob[:grows].reshape(-1, order="F")
    out = []
    for p in range(P):
        s = np.zeros((ld, ldims[-1]), order="F")
        s[:rows] = flat[p::P].reshape((rows, ldims[-1]), order="F")
        out.append(s)
    return out, ldims, ld
