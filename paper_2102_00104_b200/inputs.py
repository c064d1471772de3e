"""Seeded synthetic inputs of the BASELINE configs, generated on the device in
the reference's padded tensor layout (storage.hpp:82-115).  Off the timed
path; torch is used here only as plumbing for the contractions.

    config 1  4^10 uniform[-1,1]                    (counter-based, gen_uniform)
    config 2  16^7 exact TT rank 32 + 1e-8 noise    (N(0,1) cores, seed 2/102)
    config 3  n x k uniform[-1,1], n*k = 2^30       (seed 3)
    config 4  2^32 as d=32, n=2, TT rank <= 64 + 1e-10 noise (seed 4/104)
    config 5  8^11 uniform + rank-50 TT signal of 100x the noise norm (seed 5/105)

Configs 4 and 5 are also generated per partition (config4_slab,
config5_slab): partition p of P holds the global entries l = p + P * l_local
(split_first_dim, ttsvd_bench.cpp:72-86) — for config 4 the leading log2(P)
modes are merged into the partition index, for config 5 mode 1 (extent 8) is
split as (P, 8/P) with P fastest.  The exact-TT part of a slab is itself a TT
(the merged modes contracted into the first local core), the noise and the
uniform part are counter-based on the GLOBAL index, and the norms that scale
them are global (analytic for the TT, an all-reduce for the uniform part), so
every P generates the same global tensor.
"""
from __future__ import annotations

import numpy as np
import torch

from .ttsvd import fortran_empty, gen_partition, gen_uniform, padded_stride


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


def tt_norm(cores: list[torch.Tensor]) -> float:
    """||TT||_F from the chain of core Gram matrices (no contraction)."""
    G = torch.ones((1, 1), dtype=torch.float64, device=cores[0].device)
    for c in cores:
        G = torch.einsum("ab,axc,bxd->cd", G, c, c)
    return float(G[0, 0].clamp(min=0).sqrt())


def _merge_leading(cores: list[torch.Tensor], digits: list[int]) -> list[torch.Tensor]:
    """Fix the leading modes at `digits` and fold them into the next core."""
    v = torch.ones((1, 1), dtype=torch.float64, device=cores[0].device)
    for j, x in enumerate(digits):
        v = v @ cores[j][:, x, :]
    rest = cores[len(digits):]
    return [torch.einsum("a,axb->xb", v[0], rest[0]).unsqueeze(0)] + list(rest[1:])


def config4_slab(P: int, p: int, d: int = 32, device: int = 0):
    """Partition p of P of config 4 (P a power of two): the slab of the
    global 2^d tensor whose leading log2(P) modes index p; local dims
    [2] * (d - log2 P).  P = 1 is the whole tensor."""
    q = int(P).bit_length() - 1
    if P < 1 or (1 << q) != P or q >= d:
        raise ValueError("config 4 partitions: P must be a power of two below 2^d")
    dims = [2] * d
    ranks = [min(64, 2 ** j, 2 ** (d - j)) for j in range(d + 1)]
    cores = gaussian_cores(dims, ranks, 4, device)
    sigma = 1e-10 * tt_norm(cores) / np.sqrt(2.0 ** d)
    local = _merge_leading(cores, [(p >> j) & 1 for j in range(q)]) if q else cores
    ldims = dims[q:]
    X = to_padded(tt_contract_flat(local), ldims)
    gen_partition(104, 1, X, 2 ** (d - q), P, p, scale=sigma)
    torch.cuda.empty_cache()
    return X, ldims, 64, 0.0


def config4(d: int = 32, device: int = 0):
    """2^d entries as d modes of 2 (d = 32: 2^32, 32 GiB), exact TT with
    r_j = min(64, 2^j, 2^(d-j)), N(0,1) cores (seed 4), plus N(0, s^2) noise
    with s = 1e-10 ||X|| / sqrt(N) (counter-based, seed 104); TT-SVD
    r_max = 64, eps = 0."""
    return config4_slab(1, 0, d, device)


def config5_slab(P: int, p: int, d: int = 11, device: int = 0, allreduce=None):
    """Partition p of P (P | 8) of config 5: mode 1 split as (P, 8/P), P
    fastest, so the slab holds j_1 = p (mod P); local dims [8/P, 8, ...]
    ([8] * (d-1) at P = 8).  ``allreduce(float) -> float`` sums ||E_p||^2
    over the partitions (torch.distributed); without it P must be 1."""
    if 8 % P or P < 1:
        raise ValueError("config 5 partitions: P must divide 8")
    dims = [8] * d
    ranks = [min(50, 8 ** j, 8 ** (d - j)) for j in range(d + 1)]
    cores = gaussian_cores(dims, ranks, 105, device)
    s_norm = tt_norm(cores)
    if P == 8:
        local, ldims = _merge_leading(cores, [p]), dims[1:]
    else:
        local, ldims = [cores[0][:, p::P, :].contiguous()] + cores[1:], [8 // P] + dims[1:]
    total = int(np.prod(ldims))
    rows = total // ldims[-1]
    X = fortran_empty(rows, ldims[-1], ld=padded_stride(rows), device=device, zero=True)
    gen_partition(5, 0, X, total, P, p)
    e2 = float(sum(torch.sum(X[:, j] ** 2) for j in range(ldims[-1])))
    if allreduce is not None:
        e2 = allreduce(e2)
    elif P != 1:
        raise ValueError("config5_slab: pass allreduce for P > 1")
    S = tt_contract_flat(local).view(ldims[-1], rows).t()
    X.add_(S, alpha=100.0 * np.sqrt(e2) / s_norm)
    del S
    torch.cuda.empty_cache()
    return X, ldims, 50, 1e-4


def config5(d: int = 11, device: int = 0):
    """8^d entries (d = 11: 2^33, 64 GiB): E uniform[-1,1] (seed 5) plus a TT
    signal S with N(0,1) cores, r_j = min(50, 8^j, 8^(d-j)) (seed 105), scaled
    so ||S|| = 100 ||E||; TT-SVD r_max = 50, eps = 1e-4."""
    return config5_slab(1, 0, d, device)
