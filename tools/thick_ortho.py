"""Config 5's reduced instance (8^7, eps 1e-4, r_max 50) through thick-bounds:
check_orthonormality of the device result and of the reference's own
tt_svd_thick_bounds on the same bytes (tests/test_gpu_parity_full.py asserts
the comparison; this prints the numbers)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2102_00104_b200 as tt
from paper_2102_00104_b200 import inputs
from oracle.oracle import Oracle
from test_gpu_parity_full import host_copy, orthonormality
from helpers import rel_error
ref = Oracle("reference")
X, dims, r_max, eps = inputs.config5(7)
for variant in ("thick", "plain"):
    if variant == "thick":
        T = tt.tt_svd_thick_bounds(X, dims, tt.TruncationSpec(r_max=r_max, eps=eps), tt.ThickBoundsParams())
        Xh = host_copy(X, dims)
        r, cores = ref.tt_svd_thick_bounds(Xh, dims, Xh.shape[0], r_max, eps, 16, 0.5, ())
    else:
        T = tt.tt_svd_tsqr(X, dims, tt.TruncationSpec(r_max=r_max, eps=eps))
        r, cores = ref.tt_svd_tsqr(Xh, dims, Xh.shape[0], r_max, eps)[:2]
    print(json.dumps({"variant": variant, "ranks_equal": T.ranks() == r,
                      "orthonormality_gpu": orthonormality([c.data for c in T.cores]),
                      "orthonormality_ref": orthonormality(cores),
                      "error_gpu": rel_error(Xh, dims, [c.data for c in T.cores]),
                      "error_ref": rel_error(Xh, dims, cores)}))
