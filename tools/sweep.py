#!/usr/bin/env python
"""M sweep of the W6Ax linear on one B200 (BASELINE configs 2-4: the GEMV-to-GEMM
crossover on LLaMA-2 7B/13B/70B layer shapes).

For every (layer shape, M) it times, with CUDA-graph replay and CUDA events:
  gemm    the T6 GEMM alone on already-quantized activations (the kernel the roofline
          is about: gemv_stream for M <= 16, gemm_tc (tcgen05) above),
  fwd     the full online call FlexQLinear.forward (quantizer + GEMM, fp16 in/out),
  mma     (M > 16) the same GEMM forced onto the mma.sync kernel (ksplit=-1), the
          unpack-to-INT8 IMMA baseline the tcgen05 kernel replaces.
Every timed graph cycles through enough distinct copies of the layer's packed
weights (>= 2x the 126 MB L2) that each launch streams its weights from HBM.

    python tools/sweep.py --model llama2-13b --ms 1,2,4,8,16,32,64,128,256 > out.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 2**20


_KERNELS = {0: "gemv_stream", 1: "gemm_tc", 2: "gemm_tc16", 3: "gemm_t6"}


def kernel_name(m, n, k):
    """The kernel flexq_linear_forward routes this shape to at group 128, fp16 scales
    (flexq_linear_kernel: csrc/capi.cu)."""
    from paper_2508_04405_b200 import _lib

    return _KERNELS.get(_lib.load().flexq_linear_kernel(m, n, k, 128, 1), "?")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama2-13b")
    ap.add_argument("--ms", default="1,2,4,8,16,32,64,128,256")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--no-mma", action="store_true")
    ap.add_argument("--tc16-route", type=int, default=-1, choices=[-1, 0, 1],
                    help="flexq_set_tc16_route for the run: -1 auto, 0 never, 1 always (M > 16)")
    ap.add_argument("--no-cublas", action="store_true",
                    help="skip the cuBLAS fp16 (W16A16) and cuBLASLt int8 (W8A8) comparators")
    args = ap.parse_args()

    import torch

    from paper_2508_04405_b200 import FlexQLinear, _lib
    from paper_2508_04405_b200.shapes import MODELS, gemm_bytes, policy_kind, unfused

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    if args.tc16_route != -1:
        L.flexq_set_tc16_route(args.tc16_route)
    shapes = MODELS[args.model]
    if args.model != "llama2-70b":
        shapes = unfused(shapes)
    ms = [int(v) for v in args.ms.split(",")]

    def timed(fn, reps):
        fn()  # eager warm-up (library handles, workspaces) before the capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    for s in shapes:
        gen = torch.Generator(device=dev)
        gen.manual_seed(s.n + s.k)
        w = torch.randn((s.n, s.k), generator=gen, device=dev, dtype=torch.float16)
        base = FlexQLinear(w, 6, s.act_bits, 128, fp16_scales=True, layer_kind=policy_kind(s.name))
        del w
        copies = max(1, -(-2 * L2_BYTES // base.weight_bytes))
        lays = [base]
        for _ in range(copies - 1):  # distinct weight buffers, same values
            c = object.__new__(FlexQLinear)
            c.__dict__.update(base.__dict__)
            c.t6, c.wscale, c._bufs = base.t6.clone(), base.wscale.clone(), {}
            c._f16_ready = set()
            c.flag = torch.zeros(1, dtype=torch.int32, device=dev)
            lays.append(c)
        for m in ms:
            x = torch.randn((m, s.k), device=dev, dtype=torch.float16)
            outs = [torch.empty((m, s.n), dtype=torch.float16, device=dev) for _ in lays]
            for lay, o in zip(lays, outs):
                lay.forward(x, out=o)
            torch.cuda.synchronize()

            def fwd():
                for lay, o in zip(lays, outs):
                    lay.forward(x, out=o)

            def gemm():
                for lay, o in zip(lays, outs):
                    lay.gemm_only(m, o)

            t_fwd = timed(fwd, args.reps) / len(lays)
            t_gemm = timed(gemm, args.reps) / len(lays)
            row = {"model": args.model, "layer": s.name, "m": m, "n": s.n, "k": s.k,
                   "q": s.act_bits, "kernel": kernel_name(m, s.n, s.k),
                   "us_gemm": t_gemm * 1e3, "us_fwd": t_fwd * 1e3}
            def forced(ksplit, reps):  # the GEMM alone on a forced kernel route
                wsb = L.flexq_gemm_workspace_bytes(m, s.n, s.k, 128, ksplit)
                wss = [torch.zeros(wsb, dtype=torch.uint8, device=dev) for _ in lays]

                def run():
                    for lay, o, wsx in zip(lays, outs, wss):
                        frag, xs, corr, m_pad = lay._act_views(m)
                        _lib.check(L.flexq_gemm_t6(
                            _lib.ptr(lay.t6), _lib.ptr(lay.wscale), 1, frag, xs, corr, m, m_pad,
                            s.n, s.k, 128, None, _lib.ptr(o), _lib.OUT_F16, _lib.ptr(wsx), ksplit,
                            _lib.stream()))

                return timed(run, reps) / len(lays) * 1e3

            if 16 < m <= 32:  # the tcgen05 kernel the streaming GEMV replaced here
                row["us_tc"] = forced(-2, args.reps)
            if m > 16 and not args.no_mma:
                row["us_mma_sync"] = forced(-1, max(3, args.reps // 4))
            b = gemm_bytes(m, s.n, s.k)
            row["gbs_gemm"] = b / (t_gemm * 1e-3) / 1e9
            row["frac_hbm"] = row["gbs_gemm"] / peak
            row["tops_gemm"] = 2 * m * s.n * s.k / (t_gemm * 1e-3) / 1e12
            row["tops_fwd"] = 2 * m * s.n * s.k / (t_fwd * 1e-3) / 1e12
            if "us_mma_sync" in row:
                row["tops_mma_sync"] = 2 * m * s.n * s.k / (row["us_mma_sync"] * 1e-6) / 1e12
            print(json.dumps(row), flush=True)
        del lays, base
        torch.cuda.empty_cache()
        if args.no_cublas:
            continue
        # external comparators on the same layer (the paper's baseline is cuBLAS W8A8,
        # PAPER.md:498,511): torch.matmul fp16 -> cuBLAS, torch._int_mm int8 -> cuBLASLt,
        # weights rotated over >= 2x L2 like ours; activations already in the GEMM's dtype
        w16 = [torch.randn((s.n, s.k), device=dev, dtype=torch.float16)
               for _ in range(max(1, -(-2 * L2_BYTES // (s.n * s.k * 2))))]
        w8 = [torch.randint(-127, 128, (s.k, s.n), device=dev, dtype=torch.int8).t().contiguous().t()
              for _ in range(max(1, -(-2 * L2_BYTES // (s.n * s.k))))]
        for m in ms:
            row = {"model": args.model, "layer": s.name, "m": m, "n": s.n, "k": s.k,
                   "comparator": "cuBLAS"}
            x16 = torch.randn((m, s.k), device=dev, dtype=torch.float16)
            o16 = [torch.empty((m, s.n), device=dev, dtype=torch.float16) for _ in w16]

            def f16():
                for w_, o_ in zip(w16, o16):
                    torch.matmul(x16, w_.t(), out=o_)

            row["us_cublas_f16"] = timed(f16, args.reps) / len(w16) * 1e3
            if m > 16 and m % 8 == 0:  # torch._int_mm: M > 16, multiples of 8
                x8 = torch.randint(-127, 128, (m, s.k), device=dev, dtype=torch.int8)
                o8 = [torch.empty((m, s.n), device=dev, dtype=torch.int32) for _ in w8]

                def i8():
                    for w_, o_ in zip(w8, o8):
                        torch._int_mm(x8, w_, out=o_)

                try:
                    row["us_cublas_i8"] = timed(i8, args.reps) / len(w8) * 1e3
                except Exception as e:  # pragma: no cover
                    row["us_cublas_i8_error"] = str(e)[:80]
            print(json.dumps(row), flush=True)
        del w16, w8
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
