"""Time tt.tsqr on config-2 step shapes (diagnostics)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2102_00104_b200 as tt
shapes = [(1 << 20, 256), (65536, 512), (4096, 512)] if len(sys.argv) < 2 else [tuple(map(int, a.split("x"))) for a in sys.argv[1:]]
for n, m in shapes:
    g = torch.Generator(device="cuda").manual_seed(1)
    X = torch.rand(m, n, dtype=torch.float64, device="cuda", generator=g).t()
    best = 1e9
    for i in range(3):
        torch.cuda.synchronize(); t = time.perf_counter(); R = tt.tsqr(X); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"tsqr {n}x{m}: {1e3*best:.2f} ms", flush=True)
