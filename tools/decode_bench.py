#!/usr/bin/env python
"""LLaMA-2 random-init greedy decode on FlexQ linears: tokens/s at batch 1-8 (BASELINE config 5).

Every linear is a FlexQLinear (W6A6; down_proj W6A8 under the reference's default
policy).  One decode step = one CUDA-graph replay; context grows 1 -> steps.  Prints one
JSON line per batch size.

    python tools/decode_bench.py --model 7b --batches 1,2,4,8 --steps 128 --warmup 32
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b", choices=["7b", "13b", "tiny"])
    ap.add_argument("--batches", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=32)
    ap.add_argument("--layers", type=int, default=0, help="override layer count (0 = model's)")
    ap.add_argument("--policy", default="sensitivity", choices=["sensitivity", "default"],
                    help="A8 layer kinds: chosen by rank_layers on layer 0 (budget 1), or the "
                         "reference DEFAULT_POLICY (down_proj)")
    args = ap.parse_args()
    import dataclasses

    import torch

    from paper_2508_04405_b200.llama import LLAMA2_7B, LLAMA2_13B, FlexQLlamaDecoder, LlamaConfig

    cfg = {"7b": LLAMA2_7B, "13b": LLAMA2_13B,
           "tiny": LlamaConfig(hidden=512, heads=4, ffn=1408, layers=2, vocab=1000)}[args.model]
    if args.layers:
        cfg = dataclasses.replace(cfg, layers=args.layers)
    max_len = args.warmup + args.steps + 8
    base = None
    sens = None
    for b in [int(v) for v in args.batches.split(",")]:
        dec = FlexQLlamaDecoder(cfg, batch=b, max_len=max_len, weights_from=base)
        if base is None and args.policy == "sensitivity":
            from paper_2508_04405_b200.sensitivity import calibrate_decoder

            calib = FlexQLlamaDecoder(cfg, batch=8, max_len=16, weights_from=dec)
            calib.reset()
            report, policy = calibrate_decoder(calib, steps=4, layers=1, budget_k=1)
            sens = {"ranking": list(report.ranking),
                    "sqnr_db": {m.layer_kind: round(m.sqnr_db, 3) for m in report.metrics},
                    "a8_kinds": [k for k, v in policy.activation_bits_by_layer.items() if v == 8]}
            del calib
        base = base or dec
        if sens is not None:
            from paper_2508_04405_b200.quantize import BitPolicy  # noqa: F401

            dec.apply_policy(policy)
        dec.reset()
        dec.capture()
        for _ in range(args.warmup):
            dec.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            dec.step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        dec.check_errors()
        print(json.dumps({
            "metric": f"LLaMA-2-{args.model} random-init greedy decode tokens/s (FlexQ W6, A8 on the sensitivity-selected layer kinds, A6 elsewhere)",
            "batch": b, "tokens_per_s": b / (ms * 1e-3), "ms_per_step": ms,
            "context": [args.warmup, args.warmup + args.steps], "layers": cfg.layers,
            "weight_GB_per_step": dec.weight_bytes / 1e9,
            "weight_GBps": dec.weight_bytes / (ms * 1e-3) / 1e9,
            "activation_bits": dec.policy_table(), "sensitivity": sens,
            "timing": "CUDA-graph replay per step, CUDA events",
        }), flush=True)
        del dec


if __name__ == "__main__":
    main()
