#!/usr/bin/env python
"""Run one W6Ax linear shape a few times (profiling target for ncu).

    ncu --set full -k regex:gemm_tc -s 2 -c 1 -o out python tools/prof_one.py --n 13824 --k 5120 --m 64
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=13824)
    ap.add_argument("--k", type=int, default=5120)
    ap.add_argument("--m", type=int, default=64)
    ap.add_argument("--q", type=int, default=6)
    ap.add_argument("--iters", type=int, default=4)
    args = ap.parse_args()
    import torch

    from paper_2508_04405_b200 import FlexQLinear

    w = torch.randn((args.n, args.k), device="cuda", dtype=torch.float16)
    lay = FlexQLinear(w, 6, args.q, 128)
    x = torch.randn((args.m, args.k), device="cuda", dtype=torch.float16)
    out = torch.empty((args.m, args.n), device="cuda", dtype=torch.float16)
    for _ in range(args.iters):
        lay.forward(x, out=out)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
