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
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 13824
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 5120
    w = torch.randn((n, k), device="cuda", dtype=torch.float16)
    lay = FlexQLinear(w, 6, 6, 128)
    x = torch.randn((m, k), device="cuda", dtype=torch.float16)
    for _ in range(3):
        y = lay(x)
    torch.cuda.synchronize()
    L = _lib.lib()
    R = 6
    nall = R * 64 * 4 + 4 * 1024
    buf = (ctypes.c_longlong * nall)()
    fn = L.flexq_debug_tc_timeline
    fn.restype = ctypes.c_int
    cnt = fn(buf, nall)
    allv = np.frombuffer(buf, dtype=np.int64)
    a = allv[:R * 64 * 4].reshape(R, 64, 4)
    cm = allv[R * 64 * 4:].reshape(1024, 4)
    cm = cm[cm[:, 0] > 0]
    t0g = cm[:, 0].min()
    print(f"CTAs {len(cm)}: start spread {(cm[:,0].max()-t0g)/1e3:.2f} us; mma done "
          f"min {(cm[:,1].min()-t0g)/1e3:.2f} max {(cm[:,1].max()-t0g)/1e3:.2f} us; end min "
          f"{(cm[:,2].min()-t0g)/1e3:.2f} max {(cm[:,2].max()-t0g)/1e3:.2f} us; units {cm[:,3].min()}-{cm[:,3].max()}")
    order = np.argsort(cm[:, 2])[-5:]
    for i in order:
        print(f"  slow cta: start {(cm[i,0]-t0g)/1e3:.2f} mma_done {(cm[i,1]-t0g)/1e3:.2f} end {(cm[i,2]-t0g)/1e3:.2f}")
    t0 = a[a > 0].min()
    names = ["conv(start,wfull,aempty,done)", "mma(start,afull_ok,mma_issued,commit_done)",
             "epi(sfull_ok,table_loaded,ld_done,chunk0_done)", "epi(start,dfull_ok,arrived)",
             "wprod(start,wempty_ok,issued,-)", "bprod(start,aempty_ok,B_issued,slots_issued)"]
    for r in range(R):
        print(names[r])
        for i in range(64):
            row = a[r, i]
            if row.max() == 0:
                continue
            print(f"  u{i:2d} " + " ".join(f"{(v - t0) if v else -1:8d}" for v in row))
    summarize(a, names)


def summarize(a, names):
    import numpy as np
    print("per-role medians over units 8..63 (cycles): period of event 0, and event gaps")
    for r, nm in enumerate(names):
        rows = a[r, 8:]
        rows = rows[rows[:, 0] > 0]
        if len(rows) < 3:
            continue
        per = np.median(np.diff(rows[:, 0]))
        gaps = [np.median(rows[:, e + 1] - rows[:, e]) for e in range(3) if (rows[:, e + 1] > 0).all()]
        print(f"  {nm:48s} period {per:7.0f}  gaps " + " ".join(f"{g:7.0f}" for g in gaps))


if __name__ == "__main__":
    main()
