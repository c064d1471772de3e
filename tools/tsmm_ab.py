"""A/B timing of the config-2 step-1 TSMM (2^24 x 16 times 16 x 16 -> 2^20 x 256)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2102_00104_b200 as tt
n, m, k = 1 << 24, 16, 16
X = tt.gen_uniform(3, [n, m], ld=n + 64)
V = torch.linalg.qr(torch.randn(m, k, dtype=torch.float64, device="cuda"))[0].t().contiguous().t()
for _ in range(3):
    Y = tt.tsmm_reshape(X, V, n // 16, 16 * k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    Y = tt.tsmm_reshape(X, V, n // 16, 16 * k)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(os.environ.get("TTSVD_LIB_VARIANT", "default"), f"{ms:.4f} ms", f"{8 * n * (m + k) / ms / 1e9:.0f} GB/s")
