#!/usr/bin/env python
"""Debug: clock64 timeline of CTA 0 of the tcgen05 GEMM (FLEXQ_TC_TIMELINE=1)."""
import ctypes
import os
import sys

os.environ["FLEXQ_TC_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2508_04405_b200 import FlexQLinear, _lib

    m = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    n, k = 13824, 5120
    w = torch.randn((n, k), device="cuda", dtype=torch.float16)
    lay = FlexQLinear(w, 6, 6, 128)
    x = torch.randn((m, k), device="cuda", dtype=torch.float16)
    for _ in range(3):
        y = lay(x)
    torch.cuda.synchronize()
    L = _lib.lib()
    buf = (ctypes.c_longlong * (4 * 64 * 4))()
    fn = L.flexq_debug_tc_timeline
    fn.restype = ctypes.c_int
    cnt = fn(buf, 4 * 64 * 4)
    a = np.frombuffer(buf, dtype=np.int64).reshape(4, 64, 4)
    t0 = a[a > 0].min()
    names = ["conv(start,wfull,aempty,done)", "mma(start,dempty,bfull,afull)",
             "epi(sfull_ok,table_loaded,ld_done,chunk0_done)", "epi(start,dfull_ok,arrived)"]
    for r in range(4):
        print(names[r])
        for i in range(64):
            row = a[r, i]
            if row.max() == 0:
                continue
            print(f"  u{i:2d} " + " ".join(f"{(v - t0) if v else -1:8d}" for v in row))


if __name__ == "__main__":
    main()
