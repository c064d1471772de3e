"""Time the device small SVD on R factors like config 2's (diagnostics)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2102_00104_b200 as tt
for m, rank in [(64, 64), (128, 128), (256, 32), (512, 32), (512, 512)]:
    g = torch.Generator(device="cuda").manual_seed(m)
    A = torch.randn(4 * m, rank, dtype=torch.float64, device="cuda", generator=g) @ torch.randn(rank, m, dtype=torch.float64, device="cuda", generator=g)
    A += 1e-8 * torch.randn(4 * m, m, dtype=torch.float64, device="cuda", generator=g)
    X = tt.to_device_matrix(A.t().contiguous().t())
    R = tt.tsqr(X)
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        s = tt.small_svd(R)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    print(f"m={m} rank={rank}: small_svd {1e3*(t1-t0):.2f} ms", flush=True)
