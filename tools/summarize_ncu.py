"""Turn a round's ncu captures (gpurun_out/) into committed summaries under profiles/.

    python tools/summarize_ncu.py r01 [--model llama2-70b]

Reads gpurun_out/<R>_gemm_m{1,8,128}.ncu-rep (--set full, one launch per layer of one
step: the GEMV for M <= 16, the tcgen05 GEMM above) and gpurun_out/<R>_launches_m1.csv
(launch list), writes
profiles/<R>_ncu.md (human summary) and updates profiles/ncu_summary.json
(per-step DRAM traffic of the GEMM kernel, read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KEYS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__cycles_active.avg", "SM active cyc (avg)"),
    ("sm__cycles_elapsed.avg", "elapsed cyc"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
]


_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw_rows(rep: str):
    """Rows of `ncu --page raw` (from a report, or its exported _raw.csv), bytes in bytes."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        for h, u in zip(hdr, units):
            if u in _SCALE and num(d.get(h)) is not None:
                d[h] = num(d[h]) * _SCALE[u]
        res.append(d)
    return res


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except Exception:
        return None


def summarize(tag: str, model: str):
    from paper_2508_04405_b200.shapes import MODELS

    shapes = MODELS[model]
    lines = [f"# ncu summary {tag} ({model} decoder-layer linears)", ""]
    summary_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    summary.setdefault("gemm_traffic_bytes_per_step", {})
    for m in (1, 8, 32, 64, 128, 256):
        rep = os.path.join(ROOT, "gpurun_out", f"{tag}_gemm_m{m}_raw.csv")
        if not os.path.exists(rep):
            rep = os.path.join(ROOT, "gpurun_out", f"{tag}_gemm_m{m}.ncu-rep")
        if not os.path.exists(rep):
            continue
        rows = raw_rows(rep)
        names = sorted({(r.get("Kernel Name") or "?").split("(")[0] for r in rows})
        kname = " / ".join(names) + {"gemm_tc_kernel": " (tcgen05.mma kind::i8)",
                                     "flexq::gemm_tc16_kernel": " (tcgen05.mma kind::f16)"}.get(
                                         names[0].split("<")[0] if len(names) == 1 else "", "")
        lines += [f"## M={m}: `ncu --set full` on the {len(rows)} {kname} launches of one step", "",
                  "| layer | " + " | ".join(lbl for _, lbl in KEYS) + " |",
                  "|---" * (len(KEYS) + 1) + "|"]
        traffic = 0.0
        for s, r in zip(shapes, rows):
            vals = []
            for key, _ in KEYS:
                v = num(r.get(key))
                if key.startswith("dram__bytes") and v is not None:
                    v = v / 1e6  # bytes -> MB
                vals.append("-" if v is None else f"{v:.4g}")
            rd, wr = num(r.get("dram__bytes_read.sum")) or 0, num(r.get("dram__bytes_write.sum")) or 0
            traffic += rd + wr
            lines.append(f"| {s.name} {s.n}x{s.k} | " + " | ".join(vals) + " |")
        lines.append("")
        summary["gemm_traffic_bytes_per_step"][f"{model}_m{m}"] = traffic
    launches = os.path.join(ROOT, "gpurun_out", f"{tag}_launches_m1.csv")
    if os.path.exists(launches):
        from tools.ncu_table import load

        d = load(launches)
        items = list(d.values())[-2 * len(shapes):]
        lines += ["## M=1 launch list, last step (cold-cache, serialised: compare shares)", "",
                  "| kernel | grid | duration (ns) | DRAM read | share |", "|---|---|---|---|---|"]
        tot = sum(num(e.get("gpu__time_duration.sum")) or 0 for e in items)
        for e in items:
            t = num(e.get("gpu__time_duration.sum")) or 0
            lines.append(f"| {e['kernel'][:60]} | {e['grid']} | {t:.0f} | "
                         f"{e.get('dram__bytes_read.sum')} | {100 * t / tot:.1f}% |")
        lines.append("")
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu.md"), "w") as f:
        f.write("\n".join(lines))
    with open(summary_path, "w") as f:
        json.dump(summary, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    model = sys.argv[sys.argv.index("--model") + 1] if "--model" in sys.argv else "llama2-70b"
    summarize(tag, model)
