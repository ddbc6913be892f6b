#!/usr/bin/env python
"""Debug: per-warp globaltimer spans of one GEMV launch (FLEXQ_GEMV_TIMELINE=1)."""
import ctypes
import os
import sys

os.environ["FLEXQ_GEMV_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2508_04405_b200 import FlexQLinear, _lib

    n, k, m = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 1)))
    lay = FlexQLinear(torch.randn((n, k), device="cuda", dtype=torch.float16), 6, 6, 128)
    x = torch.randn((m, k), device="cuda", dtype=torch.float16)
    out = torch.empty((m, n), device="cuda", dtype=torch.float16)
    for _ in range(3):
        lay.forward(x, out=out)
    torch.cuda.synchronize()
    lay.gemm_only(m, out)
    nall = 148 * 16 * 8
    buf = (ctypes.c_longlong * nall)()
    fn = _lib.lib().flexq_debug_gemv_timeline
    fn.restype = ctypes.c_int
    fn(buf, nall)
    a = np.frombuffer(buf, dtype=np.int64).reshape(-1, 8)
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    d = (a - t0) / 1e3
    print(f"{n}x{k} m={m}: warps {len(a)}")
    for i, name in enumerate(["start", "init_done", "prologue", "pdl_done", "first_data",
                              "loop_done", "-", "end"]):
        if name == "-":
            continue
        print(f"  {name:10s} min {d[:, i].min():7.2f}  median {np.median(d[:, i]):7.2f}  max {d[:, i].max():7.2f} us")
    per_cta(a)



def per_cta(a, warps_per_cta=4):
    import numpy as np
    dur = (a[:, 5] - a[:, 4]) / 1e3
    n = len(dur) // warps_per_cta * warps_per_cta
    c = dur[:n].reshape(-1, warps_per_cta).mean(1)
    print("  per-CTA loop us: " + " ".join(f"{v:.1f}" for v in c[:48]))
    print(f"  corr(cta index, dur) = {np.corrcoef(np.arange(len(c)), c)[0, 1]:.2f}; "
          f"odd/even CTA mean {c[1::2].mean():.2f}/{c[0::2].mean():.2f}")


if __name__ == "__main__":
    main()
