#!/usr/bin/env python
"""Run FlexQLinear.forward a few times on one shape (for ncu captures):
    python tools/run_linear.py M N K [abits] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2508_04405_b200 import FlexQLinear  # noqa: E402

m, n, k = (int(v) for v in sys.argv[1:4])
abits = int(sys.argv[4]) if len(sys.argv) > 4 else 6
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 3
lay = FlexQLinear(torch.randn((n, k), device="cuda", dtype=torch.float16), 6, abits, 128)
x = torch.randn((m, k), device="cuda", dtype=torch.float16)
for _ in range(iters):
    lay(x)
torch.cuda.synchronize()
print("ok", m, n, k)
