"""Device-side verification of a TT-SVD result (SURVEY §8 f, rank 2): the
reconstruction error and the core orthonormality of tensor_train.hpp:79-155,
computed on the GPU so that full-size inputs (BASELINE configs 2, 4, 5) are
checked without a host copy of X.

Off the timed path: the contraction uses device GEMMs through torch
(cuBLAS DGEMM), which SURVEY §8 f allows for verification.  Nothing here is
part of the decomposition itself.
"""
from __future__ import annotations

import numpy as np
import torch

from .inputs import tt_contract_flat
from .ttsvd import TensorTrain


def _cores_on(tt: TensorTrain, device) -> list[torch.Tensor]:
    return [torch.from_numpy(np.ascontiguousarray(c.data)).to(device) for c in tt.cores]


def tt_reconstruct_flat(tt: TensorTrain, device=0) -> torch.Tensor:
    """tt_reconstruct (tensor_train.hpp:79-107): the flat Fortran-order tensor
    (N doubles) on the device."""
    tt.validate()
    return tt_contract_flat(_cores_on(tt, torch.device("cuda", device) if isinstance(device, int) else device))


def tt_error(X: torch.Tensor, dims, tt: TensorTrain, chunk_cols: int = 1) -> float:
    """||X - reconstruct(tt)||_F / ||X||_F (tensor_train.hpp:110-122) with X the
    device tensor in the reference's padded layout (rows = N / n_d, column
    stride padded_stride(rows)).  Sums in fp64 on the device."""
    dims = [int(x) for x in dims]
    if tt.dims() != dims:
        raise ValueError("tt_error: dims mismatch")
    N = int(np.prod(dims))
    rows, nd = N // dims[-1], dims[-1]
    Y = tt_reconstruct_flat(tt, X.device).view(nd, rows)
    diff = torch.zeros((), dtype=torch.float64, device=X.device)
    nrm = torch.zeros((), dtype=torch.float64, device=X.device)
    for j in range(0, nd, chunk_cols):
        xs = X[:rows, j:j + chunk_cols]
        ys = Y[j:j + chunk_cols].t()
        diff += torch.sum((xs - ys) ** 2)
        nrm += torch.sum(xs * xs)
    del Y
    return float(torch.sqrt(diff) / torch.sqrt(nrm))


def check_orthonormality(tt: TensorTrain, excluded: int = 0, device=0) -> float:
    """check_orthonormality (tensor_train.hpp:127-155): the largest
    ||G^T G - I||_F (cores left of `excluded`, vertical unfolding) or
    ||G G^T - I||_F (cores right of it, horizontal unfolding).  The Alg. 2
    chain leaves cores 2..d right-orthonormal, so excluded = 0."""
    dev = torch.device("cuda", device) if isinstance(device, int) else device
    worst = 0.0
    for j, c in enumerate(tt.cores):
        if j == excluded:
            continue
        rl, n, rr = c.data.shape
        G = torch.from_numpy(np.asfortranarray(c.data)).to(dev)
        if j < excluded:
            V = G.permute(2, 1, 0).reshape(rr, n * rl).t()  # vertical: (rl*n) x rr, row a + rl*x
            g = V.t() @ V
        else:
            H = G.permute(0, 2, 1).reshape(rl, rr * n)  # horizontal: rl x (n*rr), col x + n*b (any order)
            g = H @ H.t()
        dev2 = torch.linalg.matrix_norm(g - torch.eye(g.shape[0], dtype=g.dtype, device=dev))
        worst = max(worst, float(dev2))
    return worst
