"""BASELINE configs 4 and 5 on ONE B200 (they fit in its HBM): seeded device
generation, TT-SVD timed with CUDA events, device verification (reconstruction
error, core orthonormality).  Usage:
    python tools/big_configs.py --config 4 --d 32      # full config 4 (2^32, 32 GiB)
    python tools/big_configs.py --config 5 --d 10      # config 5's 8 GiB per-GPU slab size
Prints one JSON line per run."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--d", type=int, default=32)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--thick", action="store_true")
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2102_00104_b200 as tt
    from paper_2102_00104_b200 import inputs, verify
    torch.cuda.set_device(0)
    t0 = time.time()
    gen = inputs.config4 if a.config == 4 else inputs.config5
    X, dims, r_max, eps = gen(a.d)
    torch.cuda.synchronize()
    t_gen = time.time() - t0
    nbytes = 8 * int(np.prod(dims))
    run = (lambda: tt.tt_svd_thick_bounds(X, dims, tt.TruncationSpec(r_max=r_max, eps=eps))) if a.thick else \
        (lambda: tt.tt_svd_tsqr(X, dims, tt.TruncationSpec(r_max=r_max, eps=eps)))
    T = run()  # warm-up (workspaces)
    torch.cuda.synchronize()
    times = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        T = run()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    err = verify.tt_error(X, dims, T)
    ortho = verify.check_orthonormality(T)
    ms = min(times)
    out = {"config": a.config, "dims": f"{dims[0]}^{len(dims)}", "tensor_bytes": nbytes, "r_max": r_max, "eps": eps,
           "variant": "thick" if a.thick else "plain", "ranks": T.ranks(), "ms": round(ms, 3),
           "gbs": round(nbytes / ms / 1e6, 2), "rel_error": err, "orthonormality": ortho,
           "gen_s": round(t_gen, 1), "peak_mem_gib": round(torch.cuda.max_memory_allocated() / 2 ** 30, 1),
           "steps": [[s.rows, s.cols, s.rank, s.tsqr_kernel] for s in T.steps]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
