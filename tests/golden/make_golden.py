"""Generate the golden fixtures of tests/golden/ from the REFERENCE itself.

Runs oracle/_ref/libttsvd_ref.so — the untouched reference headers
(/root/reference/proj/include/ttsvd) compiled by oracle/Makefile — on the
reference tests' own inputs (regenerated bit-exactly by the restated
generators, which test_oracle_pin.py pins against the reference's) and on
BASELINE config 1.  Inputs that are cheap to regenerate are stored as seeds;
outputs are stored in full.

    python tests/golden/make_golden.py        (needs /root/reference; run here)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle.oracle import Oracle, gaussian, random_tensor  # noqa: E402


def main():
    ref = Oracle("reference")
    out = {}
    # --- tsqr / reduce_block / combine on the reference tests' inputs ---
    X = gaussian(5000, 6, 5)  # test_tsqr.cpp:127-133
    for w in (1, 3):
        out[f"tsqr_5000x6_seed5_w{w}"] = ref.tsqr(X, workers=w)
    m8 = gaussian(8, 3, 42)  # test_tsqr.cpp:46-63
    r3 = np.triu(gaussian(3, 3, 43))
    out["reduce_block_8x3"] = ref.reduce_block(m8, r3)
    out["reduce_block_hand"] = ref.reduce_block(np.array([[3.0], [4.0]]), np.zeros((1, 1)))
    parts = [np.triu(gaussian(4, 4, 100 + p)) for p in range(4)]  # test_tsqr.cpp:175-192
    out["combine_4x4_x4"] = ref.combine_factors(parts)
    # --- jacobi_svd (test_small_svd.cpp:129-134) ---
    s, U, V = ref.jacobi_svd(gaussian(200, 5, 3))
    out["jacobi_200x5_sigma"], out["jacobi_200x5_U"], out["jacobi_200x5_V"] = s, U, V
    s, U, V = ref.jacobi_svd(np.triu(gaussian(16, 16, 21)))
    out["small_svd_16_sigma"], out["small_svd_16_V"] = s, V
    # --- tsmm_reshape (test_tsmm.cpp:40-49) ---
    out["tsmm_100x6_6x3_50x6"] = ref.tsmm_reshape(gaussian(100, 6, 2), gaussian(6, 3, 3), 50, 6)
    # --- drivers ---
    for name, seed, dims, rmax, eps in [("tt_2pow12_seed43_r4", 43, [2] * 12, 4, 0.0),
                                         ("tt_2pow16_seed4242_r5", 4242, [2] * 16, 5, 0.0),
                                         ("tt_2x3x4x5x6_seed113_r5", 113, [2, 3, 4, 5, 6], 5, 0.0),
                                         ("tt_4pow6_seed5001_r8_eps1e-2", 5001, [4] * 6, 8, 1e-2)]:
        Xt = random_tensor(seed, dims)
        ranks, cores, steps = ref.tt_svd_tsqr(Xt, dims, Xt.shape[0], rmax, eps)[:3]
        out[f"{name}_ranks"] = np.asarray(ranks)
        out[f"{name}_cores"] = np.concatenate([c.reshape(-1, order="F") for c in cores])
        out[f"{name}_error"] = np.asarray(ref.tt_error(Xt, Xt.shape[0], dims, ranks, cores))
    # BASELINE config 1: 4^10 counter-based uniform[-1,1] (seed 1), r_max = 16
    orc = Oracle("restated")
    dims = [4] * 10
    X1 = orc.gen_uniform(1, dims)
    ranks, cores, steps = ref.tt_svd_tsqr(X1, dims, X1.shape[0], 16, 0.0)[:3]
    _, _, _, sig = orc.tt_svd_tsqr(X1, dims, X1.shape[0], 16, 0.0, with_sigma=True)
    out["cfg1_ranks"] = np.asarray(ranks)
    out["cfg1_cores"] = np.concatenate([c.reshape(-1, order="F") for c in cores])
    out["cfg1_error"] = np.asarray(ref.tt_error(X1, X1.shape[0], dims, ranks, cores))
    out["cfg1_sigma"] = np.concatenate(sig)
    out["cfg1_sigma_len"] = np.asarray([len(x) for x in sig])
    # distributed (acceptance_test.cpp:311-340 input, 4 partitions)
    gd = [4] + [2] * 12
    glob = random_tensor(2718, gd)
    from helpers import split_slabs  # noqa: E402
    slabs, ld_, ld = split_slabs(glob, gd, 4)
    rr, rc = ref.tt_svd_distributed(slabs, ld_, ld, 4)
    out["dist_4x2pow12_ranks"] = np.asarray(rr)
    out["dist_4x2pow12_cores"] = np.concatenate([c.reshape(-1, order="F") for c in rc])
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
