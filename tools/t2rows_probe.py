import sys, os, json
sys.path.insert(0, '/root/repo')
import torch
import paper_2102_00104_b200 as tt
def timed(f, reps=2):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for k in (32, 64, 128):
    n = (1 << 30) // k
    X = tt.gen_uniform(3, [n, k], ld=n + 64)
    print(os.environ.get("TTSVD_T2ROWS"), os.environ.get("TTSVD_TSQR"), k, round(timed(lambda: tt.tsqr(X)), 3), flush=True)
    del X; torch.cuda.empty_cache()
