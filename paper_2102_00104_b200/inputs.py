"""Seeded synthetic inputs of the BASELINE configs, generated on the device in
the reference's padded tensor layout (storage.hpp:82-115).  Off the timed
path; torch is used here only as plumbing for the contractions.

    config 1  4^10 uniform[-1,1]                    (counter-based, gen_uniform)
    config 2  16^7 exact TT rank 32 + 1e-8 noise    (N(0,1) cores, seed 2/102)
    config 3  n x k uniform[-1,1], n*k = 2^30       (seed 3)
    config 4  2^32 as d=32, n=2, TT rank <= 64 + 1e-10 noise (seed 4/104)
    config 5  8^11 uniform + rank-50 TT signal of 100x the noise norm (seed 5/105)
"""
from __future__ import annotations

import numpy as np
import torch

from .ttsvd import fortran_empty, gen_uniform, padded_stride


def tt_contract_flat(cores: list[torch.Tensor]) -> torch.Tensor:
    """Flat Fortran-order contraction of TT cores (each (r_l, n, r_r), float64,
    on the device) — tensor_train.hpp:80-110 done with device GEMMs."""
    M = cores[0][0].t().contiguous()  # (r1, n1): M[a, L]
    for c in cores[1:]:
        rl, n, rr = c.shape
        Gp = c.permute(2, 1, 0).reshape(rr * n, rl)  # row b*n + x
        T = Gp @ M  # (rr*n, N): row (b, x), col L
        M = T.reshape(rr, n * M.shape[1])  # col x*N + L  == Fortran index of (L, x)
    return M.reshape(-1)


def to_padded(flat: torch.Tensor, dims) -> torch.Tensor:
    dims = [int(x) for x in dims]
    rows = int(np.prod(dims)) // dims[-1]
    X = fortran_empty(rows, dims[-1], ld=padded_stride(rows), device=flat.device.index, zero=True)
    X.copy_(flat.view(dims[-1], rows).t())
    return X


def config1(seed: int = 1):
    dims = [4] * 10
    return gen_uniform(seed, dims), dims, 16, 0.0


def exact_tt(dims, ranks, seed: int, noise_rel: float, noise_seed: int, device: int = 0):
    rng = np.random.default_rng(seed)
    cores = [torch.from_numpy(rng.standard_normal((ranks[j], dims[j], ranks[j + 1]))).to(f"cuda:{device}")
             for j in range(len(dims))]
    flat = tt_contract_flat(cores)
    del cores
    if noise_rel > 0:
        g = torch.Generator(device=flat.device)
        g.manual_seed(noise_seed)
        sigma = noise_rel * float(torch.linalg.vector_norm(flat)) / np.sqrt(flat.numel())
        flat.add_(torch.randn(flat.numel(), dtype=torch.float64, device=flat.device, generator=g), alpha=sigma)
    X = to_padded(flat, dims)
    del flat
    torch.cuda.empty_cache()
    return X


def config2(scale_modes: int = 7, device: int = 0):
    """16^7 (2^28 entries, 2 GiB) exact TT with rank 32 + N(0, 1e-8 ||X|| / sqrt(N))."""
    d = scale_modes
    dims = [16] * d
    ranks = [1] + [32] * (d - 1) + [1]  # G_1: 1x16x32, G_2..G_{d-1}: 32x16x32, G_d: 32x16x1
    return exact_tt(dims, ranks, 2, 1e-8, 102, device), dims, 32, 0.0


def config3_matrix(k: int, device: int = 0, total: int = 1 << 30):
    n = total // k
    return gen_uniform(3, [n, k]), n, k
