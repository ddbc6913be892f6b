#!/usr/bin/env python
"""Latency of the activation quantizer alone (flexq_quantize -> act operand), graph replay."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2508_04405_b200 import _lib

    L = _lib.lib()
    for m, k, bits in [(1, 8192, 6), (1, 28672, 8), (8, 8192, 6), (1, 4096, 6)]:
        x = torch.randn((m, k), device="cuda").half()
        m_pad = L.flexq_act_m_pad(m)
        frag = torch.zeros(L.flexq_act_frag_bytes(m_pad, k, 128) // 4, dtype=torch.int32, device="cuda")
        xs = torch.zeros((k // 128, m_pad), dtype=torch.float32, device="cuda")
        corr = torch.zeros((k // 128, m_pad), dtype=torch.int32, device="cuda")
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")

        def q():
            _lib.check(L.flexq_quantize(_lib.ptr(x), 0, m, k, bits, 128, 1, None, None, _lib.ptr(frag),
                                        _lib.ptr(xs), _lib.ptr(corr), m_pad, _lib.ptr(flag),
                                        _lib.stream()))
        q()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                q()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"quantize m={m} k={k} bits={bits}: {e0.elapsed_time(e1) / 200 * 1e3:.2f} us/launch")


if __name__ == "__main__":
    main()
