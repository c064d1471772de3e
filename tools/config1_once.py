"""One config-1 decomposition after warm-up (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2102_00104_b200 as tt
from paper_2102_00104_b200 import inputs

X, dims, r_max, eps = inputs.config1()
for _ in range(3):
    T = tt.tt_svd_tsqr(X, dims, tt.TruncationSpec(r_max=r_max))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
T = tt.tt_svd_tsqr(X, dims, tt.TruncationSpec(r_max=r_max))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(T.ranks())
