"""Diagnostics: Gram residual of the TSQR (ttsvd_cu_tsqr) on assorted
shapes, and its time (CUDA events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2102_00104_b200 as tt

shapes = [(int(a), int(b)) for a, b in (s.split("x") for s in sys.argv[1:])] or \
    [(2048, 32), (4096, 64), (8192, 64), (40000, 96), (4096, 512), (65536, 512), (37888, 256), (16384, 64)]
for n, m in shapes:
    g = torch.Generator(device="cuda").manual_seed(n + m)
    X = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g).t()
    R = tt.tsqr(X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        R = tt.tsqr(X)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    Xh = X.cpu().numpy()
    Rh = R.cpu().numpy()
    gx = Xh.T @ Xh
    res = np.linalg.norm(Rh.T @ Rh - gx) / np.linalg.norm(gx)
    # per panel diagnosis: first column block where R^T R deviates
    d = np.abs(Rh.T @ Rh - gx) / np.linalg.norm(gx)
    bad = np.argwhere(d > 1e-12)
    first = (int(bad[0][0]), int(bad[0][1])) if len(bad) else None
    print(f"{n}x{m}: resid {res:.3e} first bad entry {first} tril0 {np.all(np.tril(Rh, -1) == 0)} {ms:.3f} ms", flush=True)
