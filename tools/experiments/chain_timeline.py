"""Per-CTA phase timeline of one FlexQChain launch (FLEXQ_CHAIN_TIMELINE=1, debug build path).

    FLEXQ_CHAIN_TIMELINE=1 python tools/chain_timeline.py [--model llama2-70b] [--m 1]

For every link: when the CTAs reach grid barrier A (previous link done), leave it, leave
barrier B (operand quantized) and finish their unit ranges (slowest warp of the CTA), in us
from the kernel's first CTA start (min / median / max over CTAs).
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama2-70b")
    ap.add_argument("--m", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-dep", action="store_true")
    args = ap.parse_args()
    os.environ["FLEXQ_CHAIN_TIMELINE"] = "1"
    import torch

    import paper_2508_04405_b200 as fq
    from paper_2508_04405_b200 import _lib
    from paper_2508_04405_b200.shapes import MODELS, WORKLOADS

    shapes = WORKLOADS.get(args.model, None) or MODELS[args.model]
    if args.model == "config1":
        shapes = shapes * 16
    g = torch.Generator(device="cuda").manual_seed(0)
    layers = [fq.FlexQLinear(torch.randn((s.n, s.k), generator=g, device="cuda").half(),
                             activation_bits=s.act_bits) for s in shapes]
    xs = [torch.randn((args.m, s.k), generator=g, device="cuda").half() for s in shapes]
    chain = fq.FlexQChain(layers, depends_on_prev=not args.no_dep)
    L = _lib.lib()
    L.flexq_debug_chain_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
    per = 1 + 4 * 16
    buf = np.zeros(148 * 16 * per, np.int64)
    for rep in range(args.reps):
        chain(xs)
        torch.cuda.synchronize()
    n = L.flexq_debug_chain_timeline(buf.ctypes.data, buf.size)
    tl = buf[: n * per].reshape(n, per).astype(np.float64)
    t0 = tl[:, 0].min()
    rel = (tl - t0) / 1e3
    print(f"{n} CTAs; kernel start spread {rel[:, 0].max():.2f} us")
    for j, s in enumerate(shapes):
        cols = [1 + 4 * j, 2 + 4 * j, 3 + 4 * j, 4 + 4 * j]
        a_in, a_out, b_out, done = (rel[:, c] for c in cols)
        def st(v):
            return f"{v.min():7.2f} {np.median(v):7.2f} {v.max():7.2f}"
        print(f"link {j} {s.name:10s} A in {st(a_in)} | A out {st(a_out)} | B out {st(b_out)} | "
              f"done {st(done)}")


if __name__ == "__main__":
    main()
