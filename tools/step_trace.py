#!/usr/bin/env python
"""Debug: lay one bench step (quantizer + GEMV per linear) out on one time axis.

    python tools/step_trace.py [M] [model]

Runs the bench.py step of the given model (default llama2-70b) as a CUDA graph with
FLEXQ_TRACE=1; every instrumented kernel appends globaltimer records (quantizer: per
warp [start, after griddepcontrol.wait, end]; GEMV: per warp [start, first data, end]).
Prints, per launch, when its first CTA started, when its data phase began, when its last
warp ended, and the gap to the previous launch's end -- the serialisation the graph pays.
"""
import ctypes
import os
import sys

os.environ["FLEXQ_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2508_04405_b200 import FlexQLinear, _lib
    from paper_2508_04405_b200.shapes import MODELS, policy_kind

    m = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    model = sys.argv[2] if len(sys.argv) > 2 else "llama2-70b"
    shapes = MODELS[model]
    layers, xs, outs = [], [], []
    for s in shapes:
        w = torch.randn((s.n, s.k), device="cuda", dtype=torch.float16)
        layers.append(FlexQLinear(w, 6, s.act_bits, 128, layer_kind=policy_kind(s.name)))
        xs.append(torch.randn((m, s.k), device="cuda", dtype=torch.float16))
        outs.append(torch.empty((m, s.n), device="cuda", dtype=torch.float16))

    def step():
        for lay, x, o in zip(layers, xs, outs):
            lay.forward(x, out=o)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    fn = _lib.lib().flexq_debug_trace
    fn.restype = ctypes.c_int
    cap = 1 << 16
    buf = (ctypes.c_longlong * (4 * cap))()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    fn(buf, cap)  # drop warm-up records
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    n = fn(buf, cap)
    rec = np.frombuffer(buf, dtype=np.int64)[:4 * n].reshape(n, 4)
    t0 = rec[:, 1].min()
    warp_of = rec[:, 0] >> 40  # GEMV records carry the warp index above bit 40
    rec = rec.copy()
    rec[:, 0] &= (1 << 40) - 1
    names = {1: "quantize", 2: "gemv", 3: "fused_quant", 4: "gemm_tc"}
    print(f"{model} M={m}: graph step {e0.elapsed_time(e1) * 1e3:.1f} us (events), "
          f"{(rec[:, 3].max() - t0) / 1e3:.1f} us first-start..last-end (globaltimer)")
    print(f"{'launch':>8} {'kind':>11} {'recs':>5} {'start0':>8} {'start50':>8} {'mid0':>8} "
          f"{'mid50':>8} {'end50':>8} {'end100':>8} {'gap':>7} {'late':>5}")
    prev_end = None
    for tag in sorted(set(rec[:, 0].tolist())):
        r = rec[rec[:, 0] == tag]
        d = (r[:, 1:] - t0) / 1e3
        kind = names.get(tag & 0xFF, str(tag & 0xFF))
        gap = d[:, 0].min() - prev_end if prev_end is not None else 0.0
        print(f"{tag >> 8:>8} {kind:>11} {len(r):>5} {d[:, 0].min():8.2f} {np.median(d[:, 0]):8.2f} "
              f"{d[:, 1].min():8.2f} {np.median(d[:, 1]):8.2f} {np.median(d[:, 2]):8.2f} "
              f"{d[:, 2].max():8.2f} {gap:7.2f} {int((d[:, 0] > d[:, 0].min() + 5).sum()):>5}")
        prev_end = d[:, 2].max()
    np.save(os.path.join("gpurun_out", f"step_trace_{model}_m{m}.npy"),
            np.hstack([rec, warp_of[:, None]]))


if __name__ == "__main__":
    main()
