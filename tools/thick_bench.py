"""Time tt_svd_thick_bounds vs tt_svd_tsqr on config 2 (diagnostics)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2102_00104_b200 as tt
from paper_2102_00104_b200 import inputs
X, dims, r_max, eps = inputs.config2(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
spec = tt.TruncationSpec(r_max=r_max, eps=eps)
print("k, m =", tt.choose_combined_dims(dims, tt.ThickBoundsParams(), r_max))
for name, f in (("plain", lambda: tt.tt_svd_tsqr(X, dims, spec)),
                ("thick", lambda: tt.tt_svd_thick_bounds(X, dims, spec, tt.ThickBoundsParams()))):
    for _ in range(2):
        T = f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        T = f()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    print(f"{name}: {ms:.2f} ms  {8 * X.shape[0] * X.shape[1] / ms / 1e6:.2f} GB/s  ranks {T.ranks()}", flush=True)

ctx = tt.context()
ctx.set_timing(True)
T = tt.tt_svd_thick_bounds(X, dims, spec, tt.ThickBoundsParams())
torch.cuda.synchronize()
ctx.set_timing(False)
for s in T.steps:
    print(f"thick step {s.step}: {s.rows}x{s.cols} r={s.rank} tsqr {s.t_tsqr*1e3:.3f} ({s.tsqr_kernel}) svd {s.t_small_svd*1e3:.3f} tsmm {s.t_tsmm*1e3:.3f} ms")
