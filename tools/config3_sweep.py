"""BASELINE config 3: building-block sweep (diagnostics / evidence).
TSQR of n x k (n*k = 2^30 fp64, uniform[-1,1], stride n+64) and TSMM of the
same X with a k x r orthonormal V, output reshaped to (n/2, 2r); device
time by CUDA events, GB/s and roofline fraction per (k, r) (SURVEY 8 d)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2102_00104_b200 as tt

try:  # GB/s, the driver-written MEASURED_PEAKS.json (copy bandwidth)
    _pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
    HBM = float(_pk.get("hbm_copy_gbs") or _pk.get("hbm_gbs") or 6461.2)
except Exception:
    HBM = 6461.2
FP64 = 37.1   # TF/s, DMMA probe


def timed(f, reps=3):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = []
log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for k in (1, 2, 4, 8, 16, 32, 64, 128):
    n = (1 << log2) // k
    X = tt.gen_uniform(3, [n, k], ld=n + 64)  # seeded counter-based uniform[-1,1], stride n + 64
    ms = timed(lambda: tt.tsqr(X))
    byts, flops = 8.0 * n * k, 2.0 * n * k * k
    t_roof = max(byts / HBM / 1e9, flops / FP64 / 1e12) * 1e3
    row = {"kernel": "tsqr", "k": k, "ms": round(ms, 4), "GBps": round(byts / ms / 1e6, 1),
           "roofline_ms": round(t_roof, 4), "frac": round(t_roof / ms, 3)}
    print(json.dumps(row), flush=True)
    out.append(row)
    g = torch.Generator(device="cuda").manual_seed(103)
    for r in (1, 4, 16, 32):
        if r > k:
            continue
        V = torch.linalg.qr(torch.randn(k, r, dtype=torch.float64, device="cuda", generator=g))[0]
        Vf = V.t().contiguous().t()
        out_rows, out_cols = n // 2, 2 * r
        ms = timed(lambda: tt.tsmm_reshape(X, Vf, out_rows, out_cols))
        byts, flops = 8.0 * n * (k + r), 2.0 * n * k * r
        t_roof = max(byts / HBM / 1e9, flops / FP64 / 1e12) * 1e3
        row = {"kernel": "tsmm", "k": k, "r": r, "ms": round(ms, 4), "GBps": round(byts / ms / 1e6, 1),
               "roofline_ms": round(t_roof, 4), "frac": round(t_roof / ms, 3)}
        print(json.dumps(row), flush=True)
        out.append(row)
    del X
    torch.cuda.empty_cache()
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                                 "config3_sweep.json"), "w"), indent=1)
