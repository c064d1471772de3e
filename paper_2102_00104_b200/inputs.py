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
    on the device) — tensor_train.hpp:80-110 done with device GEMMs.  The
    running factor is kept row-major as (N, r): rows x*N .. x*N + N - 1 of the
    next factor are M @ G[:, x, :], so every GEMM has leading dimension r and
    row chunks below 2^31 (cuBLAS int32 dimensions; config 4 has N = 2^32)."""
    M = cores[0][0].contiguous()  # (n1, r1): M[L, a]
    chunk = 1 << 30
    for c in cores[1:]:
        rl, n, rr = c.shape
        N = M.shape[0]
        out = torch.empty((n * N, rr), dtype=M.dtype, device=M.device)
        if rr == 1:  # last core: out (n x N, row-major) = G[:, :, 0]^T M^T, one GEMM per chunk
            Gt = c[:, :, 0].t().contiguous()  # n x rl
            o2 = out.view(n, N)
            ck = 1 << 27  # the (n x ck) product is staged: o2's row stride N may exceed int32
            for c0 in range(0, N, ck):
                c1 = min(N, c0 + ck)
                o2[:, c0:c1].copy_(Gt @ M[c0:c1].t())
            del M
            M = out
            continue
        for x in range(n):
            Gx = c[:, x, :].contiguous()  # rl x rr
            for c0 in range(0, N, chunk):
                c1 = min(N, c0 + chunk)
                torch.matmul(M[c0:c1], Gx, out=out[x * N + c0:x * N + c1])
        del M
        M = out
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


def gaussian_cores(dims, ranks, seed: int, device: int = 0) -> list[torch.Tensor]:
    """N(0,1) TT cores r_{j-1} x n_j x r_j from one seeded host stream (SURVEY
    §8 d: Gaussian cores on the host, then copied to the device)."""
    rng = np.random.default_rng(seed)
    return [torch.from_numpy(rng.standard_normal((ranks[j], dims[j], ranks[j + 1]))).to(f"cuda:{device}")
            for j in range(len(dims))]


def _add_noise(flat: torch.Tensor, sigma: float, noise_seed: int, chunk: int = 1 << 27) -> None:
    """flat += sigma N(0,1), generated chunk-wise (no N-sized temporary)."""
    g = torch.Generator(device=flat.device)
    g.manual_seed(noise_seed)
    for c0 in range(0, flat.numel(), chunk):
        n = min(chunk, flat.numel() - c0)
        flat[c0:c0 + n].add_(torch.randn(n, dtype=torch.float64, device=flat.device, generator=g), alpha=sigma)


def exact_tt(dims, ranks, seed: int, noise_rel: float, noise_seed: int, device: int = 0):
    flat = tt_contract_flat(gaussian_cores(dims, ranks, seed, device))
    if noise_rel > 0:
        sigma = noise_rel * float(torch.linalg.vector_norm(flat)) / np.sqrt(flat.numel())
        _add_noise(flat, sigma, noise_seed)
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


def config4(d: int = 32, device: int = 0):
    """2^d entries as d modes of 2 (d = 32: 2^32, 32 GiB), exact TT with
    r_j = min(64, 2^j, 2^(d-j)), N(0,1) cores (seed 4), plus N(0, s^2) noise
    with s = 1e-10 ||X|| / sqrt(N) (seed 104); TT-SVD r_max = 64, eps = 0."""
    dims = [2] * d
    ranks = [min(64, 2 ** j, 2 ** (d - j)) for j in range(d + 1)]
    return exact_tt(dims, ranks, 4, 1e-10, 104, device), dims, 64, 0.0


def config5(d: int = 11, device: int = 0):
    """8^d entries (d = 11: 2^33, 64 GiB): E uniform[-1,1] (seed 5) plus a TT
    signal S with N(0,1) cores, r_j = min(50, 8^j, 8^(d-j)) (seed 105), scaled
    so ||S|| = 100 ||E||; TT-SVD r_max = 50, eps = 1e-4."""
    dims = [8] * d
    ranks = [min(50, 8 ** j, 8 ** (d - j)) for j in range(d + 1)]
    X = gen_uniform(5, dims)
    rows = int(np.prod(dims)) // dims[-1]
    S = tt_contract_flat(gaussian_cores(dims, ranks, 105, device)).view(dims[-1], rows).t()
    e2 = float(sum(torch.sum(X[:rows, j] ** 2) for j in range(dims[-1])))
    s2 = float(sum(torch.sum(S[:, j] ** 2) for j in range(dims[-1])))
    X[:rows].add_(S, alpha=100.0 * np.sqrt(e2 / s2))
    del S
    torch.cuda.empty_cache()
    return X, dims, 50, 1e-4
