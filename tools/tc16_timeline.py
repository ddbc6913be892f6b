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
    buf = (ctypes.c_longlong * (32 + 1024 + 4 * 1024))()
    if fn(buf, 32 + 1024 + 4 * 1024) == 0:
        print("no profile: build with -DFLEXQ_TC16_TIMELINE=1 (tools/build_debug.sh) and set FLEXQ_LIB")
        return
    allv = np.frombuffer(buf, dtype=np.int64)
    a = allv[:32].reshape(4, 8)
    per = allv[32:32 + 1024]
    per = per[per > 0]
    if len(per):
        print(f"MMA loop cycles over {len(per)} CTAs: min {per.min()} median {int(np.median(per))} "
              f"max {per.max()} (CTA 0: {per[0]})")
    marks = allv[32 + 1024:].reshape(1024, 4)
    marks = marks[marks[:, 0] > 0]
    if len(marks):
        t0 = marks[:, 0].min()
        q = lambda a: f"min {a.min() / 1e3:6.2f} med {np.median(a) / 1e3:6.2f} max {a.max() / 1e3:6.2f} us"
        print(f"{len(marks)} CTAs (globaltimer): entry after first entry {q(marks[:, 0] - t0)}")
        print(f"  entry -> MMA loop start {q(marks[:, 1] - marks[:, 0])}")
        print(f"  MMA loop                {q(marks[:, 2] - marks[:, 1])}")
        print(f"  loop end -> CTA exit    {q(marks[:, 3] - marks[:, 2])}")
        print(f"  last exit after first entry {(marks[:, 3].max() - t0) / 1e3:.2f} us")
    roles = [("converter w0", ["wait raw", "wait A/B stage", "convert", "store+arrive"]),
             ("weight producer", ["wait free raw", "issue"]),
             ("B producer", ["wait free stage", "issue"]),
             ("MMA", ["wait TMEM acc", "wait operands", "issue+commit"])]
    for r, (name, phases) in enumerate(roles):
        units = max(int(a[r, 4]), 1)
        tot = sum(a[r, :len(phases)])
        print(f"{name:16s} {units} units, {tot / units:7.0f} cyc/unit: " +
              ", ".join(f"{ph} {a[r, i] / units:6.0f}" for i, ph in enumerate(phases)))


if __name__ == "__main__":
    main()
