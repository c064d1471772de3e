"""Diagnostics: time the driver SVD (sigma + leading r vectors) on n x m shapes: n,m,r ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2102_00104_b200 as tt

shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or \
    [(256, 32, 32), (512, 16, 16), (64, 64, 16), (512, 256, 32), (512, 512, 32), (256, 256, 32), (128, 32, 16)]
for n, m, r in shapes:
    g = torch.Generator(device="cuda").manual_seed(n + m)
    A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g).t()
    for _ in range(3):
        s, V, path = tt.driver_svd(A, r)
    torch.cuda.synchronize()
    reps = 10
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    evs[0].record()
    for i in range(reps):
        s, V, path = tt.driver_svd(A, r)
        evs[i + 1].record()
    torch.cuda.synchronize()
    ms = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(reps))[reps // 2]
    print(f"{n}x{m} r={r}: {ms:.3f} ms ({path})", flush=True)
