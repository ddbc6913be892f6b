#!/usr/bin/env python
"""Debug: clock64 role timeline of CTA 0 of the kind::f16 batched kernel (gemm_tc16.cu).

    FLEXQ_TC_TIMELINE=1 python tools/tc16_timeline.py M N K
Per role the median period (cycles per k-block) and the median gaps between its marks.
"""
import ctypes
import os
import sys

os.environ["FLEXQ_TC_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2508_04405_b200 import FlexQLinear, _lib

    m, n, k = [int(v) for v in sys.argv[1:4]] if len(sys.argv) >= 4 else (64, 28672, 8192)
    lay = FlexQLinear(torch.randn((n, k), device="cuda", dtype=torch.float16), 6, 6, 128)
    x = torch.randn((m, k), device="cuda", dtype=torch.float16)
    for _ in range(3):
        lay(x)
    torch.cuda.synchronize()
    L = _lib.lib()
    fn = L.flexq_debug_tc16_timeline
    fn.restype = ctypes.c_int
    buf = (ctypes.c_longlong * (4 * 64 * 4))()
    fn(buf, 4 * 64 * 4)
    a = np.frombuffer(buf, dtype=np.int64).reshape(4, 64, 4)
    names = ["conv(start,wfull,aempty,done)", "mma(start,dempty,afull,issued)",
             "wprod(start,wempty,-,-)", "bprod(start,aempty,-,-)"]
    for r, nm in enumerate(names):
        rows = a[r, 8:]
        rows = rows[rows[:, 0] > 0]
        if len(rows) < 3:
            continue
        per = np.median(np.diff(rows[:, 0]))
        gaps = [np.median(rows[:, e + 1] - rows[:, e]) for e in range(3) if (rows[:, e + 1] > 0).all()]
        print(f"{nm:40s} period {per:7.0f}  gaps " + " ".join(f"{g:7.0f}" for g in gaps))


if __name__ == "__main__":
    main()
