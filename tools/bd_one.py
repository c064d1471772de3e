"""Diagnostics: one driver SVD of a config-2-like 512 x 512 work matrix (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2102_00104_b200 as tt
rng = np.random.default_rng(3)
n = m = int(sys.argv[1]) if len(sys.argv) > 1 else 512
A = rng.standard_normal((n, 32)) @ rng.standard_normal((32, m))
A += 1e-8 * np.linalg.norm(A) / np.sqrt(n * m) * rng.standard_normal((n, m))
Ad = tt.to_device_matrix(np.asfortranarray(A))
for _ in range(2):
    s, V, p = tt.driver_svd(Ad, 32)
torch.cuda.synchronize()
print(p, float(s[0]))
