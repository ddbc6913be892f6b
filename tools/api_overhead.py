#!/usr/bin/env python
"""Host-side cost of one FlexQLinear.forward (Python + ctypes + launch), the part of bench.py's
e2e number that the device-timed value does not see.

    python tools/api_overhead.py [calls]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2508_04405_b200 import FlexQLinear  # noqa: E402


def main():
    calls = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    lay = FlexQLinear(torch.randn((256, 1024), device="cuda", dtype=torch.float16), 6, 8, 128)
    x = torch.randn((1, 1024), device="cuda", dtype=torch.float16)
    out = torch.empty((1, 256), device="cuda", dtype=torch.float16)
    for _ in range(50):
        lay(x, out=out)
    torch.cuda.synchronize()
    for label, kw in (("forward(x)", {}), ("forward(x, out=out)", {"out": out})):
        t0 = time.perf_counter()
        for _ in range(calls):
            lay(x, **kw)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{label:22s} host {1e6 * (t1 - t0) / calls:6.2f} us/call, "
              f"with drain {1e6 * (t2 - t0) / calls:6.2f} us/call")
    t0 = time.perf_counter()
    for _ in range(calls * 10):
        torch.cuda.current_stream().cuda_stream
    print(f"torch.cuda.current_stream().cuda_stream {1e6 * (time.perf_counter() - t0) / calls / 10:.2f} us")


if __name__ == "__main__":
    main()
