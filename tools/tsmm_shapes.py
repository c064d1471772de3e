"""Diagnostics: time and check tsmm_reshape on given shapes (n x m times m x k,
reshaped to (n / nn) x (nn k)); arguments n,m,k,nn ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2102_00104_b200 as tt

shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or \
    [(1 << 20, 256, 32, 16), (1 << 25, 32, 32, 2), (1 << 24, 64, 32, 2), (1 << 23, 128, 32, 2), (1 << 16, 512, 32, 16)]
for n, m, k, nn in shapes:
    X = tt.gen_uniform(3, [n, m], ld=n + 64)
    V = torch.linalg.qr(torch.randn(m, k, dtype=torch.float64, device="cuda"))[0].t().contiguous().t()
    for _ in range(3):
        Y = tt.tsmm_reshape(X, V, n // nn, nn * k)
    torch.cuda.synchronize()
    reps = 15
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    evs[0].record()
    for i in range(reps):
        Y = tt.tsmm_reshape(X, V, n // nn, nn * k)
        evs[i + 1].record()
    torch.cuda.synchronize()
    ms = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(reps))[reps // 2]  # median call
    # element (i, c) of X V sits at flat position i + n c of the reshaped output
    idx = torch.randint(0, n, (4096,), device="cuda")
    ref = X[idx] @ V
    err = 0.0
    for c in range(0, k, max(1, k // 4)):
        p_ = idx + n * c
        got = Y[p_ % (n // nn), p_ // (n // nn)]
        err = max(err, float((ref[:, c] - got).abs().max()))
    t_roof = max(8.0 * n * (m + k) / 6.5e12, 2.0 * n * m * k / 37.1e12) * 1e3
    print(f"{n}x{m} k={k}: {ms:.4f} ms  roof {t_roof:.4f} ms  frac {t_roof / ms:.3f}  max err {err:.2e}", flush=True)
