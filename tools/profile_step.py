"""Run TT-SVD steps on BASELINE config 2 for profiling (ncu / nsys-less launch
lists).  Usage: python tools/profile_step.py [--modes 7] [--steps 1] [--warm 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", type=int, default=7)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warm", type=int, default=1)
    a = ap.parse_args()
    import torch
    import paper_2102_00104_b200 as tt
    from paper_2102_00104_b200 import inputs
    X, dims, r_max, eps = inputs.config2(a.modes)
    torch.cuda.synchronize()
    for _ in range(a.warm + a.steps):
        T = tt.tt_svd_tsqr(X, dims, (r_max, eps))
    torch.cuda.synchronize()
    print("ranks", T.ranks(), "launches", tt.context().launches)


if __name__ == "__main__":
    main()
