"""BASELINE config 1 (4^10, r_max 16) on one B200: device time per
decomposition (CUDA events, mean of 20 after warm-up) — the latency-bound
small case (79 kernels, one host round trip per step for the rank)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2102_00104_b200 as tt
from paper_2102_00104_b200 import inputs

X, dims, r_max, eps = inputs.config1()
for _ in range(3):
    T = tt.tt_svd_tsqr(X, dims, tt.TruncationSpec(r_max=r_max))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    T = tt.tt_svd_tsqr(X, dims, tt.TruncationSpec(r_max=r_max))
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"config": 1, "ms": round(ms, 3), "gbs": round(8 * 4 ** 10 / ms / 1e6, 2), "ranks": T.ranks()}),
      flush=True)

ctx = tt.context()
ctx.set_timing(True)
T = tt.tt_svd_tsqr(X, dims, tt.TruncationSpec(r_max=r_max))
torch.cuda.synchronize()
ctx.set_timing(False)
for s in T.steps:
    print(f"step {s.step}: {s.rows}x{s.cols} r={s.rank} tsqr {s.t_tsqr*1e3:.3f} ({s.tsqr_kernel}) svd {s.t_small_svd*1e3:.3f} tsmm {s.t_tsmm*1e3:.3f} ms")
