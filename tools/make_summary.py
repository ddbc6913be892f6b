#!/usr/bin/env python
"""Collect a round's measurement files (gpurun_out/<R>_*) into profiles/.

    python tools/make_summary.py r01

Copies the bench lines, sweeps and decode lines into profiles/ and writes
profiles/<R>_summary.md (tables quoted by DESIGN.md sec. 8).
"""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_jsonl(path):
    if not os.path.exists(path):
        return []
    return [json.loads(l) for l in open(path) if l.strip().startswith("{")]


def main(tag):
    src, dst = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
    out = [f"# Measurements {tag} (B200, one GPU; raw lines beside this file)", ""]
    # bench lines
    out += ["## bench.py (LLaMA-2-70B decoder-layer linears, CUDA-graph step)", "",
            "| M | value (TOPS) | us/step | GEMM GB/s | roofline frac (of measured HBM) | e2e TOPS | CPU baseline TOPS (cores) | SM MHz |",
            "|---|---|---|---|---|---|---|---|"]
    for m in ("m1", "m8", "m32", "m64", "m128", "m256"):
        p = os.path.join(src, f"{tag}_bench_{m}.json")
        if not os.path.exists(p):
            continue
        shutil.copy(p, os.path.join(dst, f"{tag}_bench_{m}.json"))
        d = json.loads(open(p).read().strip().splitlines()[-1])
        r, cb = d["roofline"], d.get("cpu_baseline") or {}
        out.append(f"| {d['config']['batch']} | {d['value']:.2f} | {d['ms_per_step'] * 1e3:.1f} | "
                   f"{r['achieved']:.0f} | {r['frac']:.3f} | {d['e2e']['value']:.2f} | "
                   f"{cb.get('value', float('nan')):.2e} ({cb.get('cores', '-')}) | {d['clocks']['sm_mhz']} |")
    p = os.path.join(src, f"{tag}_bench_ref.json")
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, f"{tag}_bench_reference.json"))
        d = json.loads(open(p).read().strip().splitlines()[-1])
        out += ["", f"Reference arm (`--impl reference`, the reference's CPU path on "
                    f"{d['cpu_baseline']['cores']} host cores): {d['value']:.2e} TOPS "
                    f"({d['ms_per_step']:.0f} ms per sampled step; {d['cpu_baseline']['sample']})."]
    # sweeps
    for mdl in ("llama2-7b", "llama2-13b", "llama2-70b"):
        p = os.path.join(src, f"{tag}_sweep_{mdl}.jsonl")
        rows = load_jsonl(p)
        if not rows:
            continue
        shutil.copy(p, os.path.join(dst, f"{tag}_sweep_{mdl}.jsonl"))
        out += ["", f"## M sweep, {mdl} (tools/sweep.py; GEMM alone on quantized inputs, "
                    "weights rotated over > 2x L2)", "",
                "| layer | N x K | M | kernel | GEMM us | fwd us | GB/s | frac HBM | TOPS | tcgen05 us (forced) | mma.sync us |",
                "|---|---|---|---|---|---|---|---|---|---|---|"]
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from sweep import kernel_name
        comp = {(r["layer"], r["m"]): r for r in rows if r.get("comparator")}
        rows = [r for r in rows if not r.get("comparator")]
        for r in rows:
            r["kernel"] = kernel_name(r["m"], r["n"], r["k"])
            out.append(f"| {r['layer']} | {r['n']}x{r['k']} | {r['m']} | {r['kernel']} | "
                       f"{r['us_gemm']:.1f} | {r['us_fwd']:.1f} | {r['gbs_gemm']:.0f} | "
                       f"{r['frac_hbm']:.2f} | {r['tops_gemm']:.1f} | "
                       f"{r.get('us_tc', float('nan')):.1f} | "
                       f"{r.get('us_mma_sync', float('nan')):.1f} |")
        if comp:
            out += ["", f"cuBLAS comparators, {mdl} (same layers, weights rotated over > 2x L2; "
                        "W16A16 `torch.matmul`, W8A8 `torch._int_mm` int32 out -- no dequant, "
                        "M > 16 only):", "",
                    "| layer | M | this repo GEMM us | this repo fwd us | cuBLAS fp16 us | cuBLASLt int8 us |",
                    "|---|---|---|---|---|---|"]
            for r in rows:
                c = comp.get((r["layer"], r["m"]))
                if c:
                    i8 = c.get("us_cublas_i8")
                    out.append(f"| {r['layer']} | {r['m']} | {r['us_gemm']:.1f} | {r['us_fwd']:.1f} | "
                               f"{c['us_cublas_f16']:.1f} | {'-' if i8 is None else f'{i8:.1f}'} |")
    # decode
    p = os.path.join(src, f"{tag}_decode_7b.jsonl")
    rows = load_jsonl(p)
    if rows:
        shutil.copy(p, os.path.join(dst, f"{tag}_decode_7b.jsonl"))
        out += ["", "## LLaMA-2-7B random-init greedy decode (tools/decode_bench.py, config 5)", "",
                "| batch | tokens/s | ms/step | weight GB/s | A8 kinds |", "|---|---|---|---|---|"]
        for d in rows:
            a8 = [k for k, v in (d.get("activation_bits") or {}).items() if v == 8]
            out.append(f"| {d['batch']} | {d['tokens_per_s']:.0f} | {d['ms_per_step']:.3f} | "
                       f"{d['weight_GBps']:.0f} | {','.join(a8) or '-'} |")
        s = rows[0].get("sensitivity")
        if s:
            out += ["", f"Sensitivity selection (layer 0, budget 1): ranking {s['ranking']}, "
                        f"SQNR dB {s['sqnr_db']}."]
    for f in (f"{tag}_launches_m1.csv", f"{tag}_gpu.txt"):
        if os.path.exists(os.path.join(src, f)):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    with open(os.path.join(dst, f"{tag}_summary.md"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    print("\n".join(out[:40]))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
