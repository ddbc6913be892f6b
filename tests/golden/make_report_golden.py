"""Freeze JSON documents written by the REAL reference CLI (bitserial.cli).

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_report_golden.py

Writes tests/golden/reports/*.json: a bench report (sweep suite, one repeat), the
manifests of quantize/gemm/bench runs and a sensitivity report, all produced by
the reference's own commands (cli.py:91-316).  tests/test_reports.py checks that
reports.validate_json accepts every one of them and rejects mutations the way the
reference's jsonschema validation does, so documents from either CLI are
interchangeable.
"""
from __future__ import annotations

import json
import os
import shutil
import tempfile

import numpy as np

from bitserial import fileio
from bitserial.cli import main

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reports")


def main_() -> None:
    os.makedirs(OUT, exist_ok=True)
    work = tempfile.mkdtemp()
    cwd = os.getcwd()
    os.chdir(work)
    try:
        rng = np.random.default_rng(42)
        fileio.write_float("w.flxq", rng.standard_normal((32, 384)))
        fileio.write_float("x.flxq", rng.standard_normal((4, 384)))
        assert main(["quantize", "w.flxq", "-o", "wq.flxq"]) == 0
        assert main(["gemm", "w.flxq", "x.flxq", "-o", "y.flxq", "--oracle"]) == 0
        assert main(["bench", "--suite", "sweep", "--repeat", "1", "-o", "bench.json"]) == 0
        entries = []
        for kind in ("gate_proj", "down_proj", "up_proj"):
            acts = rng.standard_normal((8, 256))
            if kind == "down_proj":
                acts[:, 3] *= 100
            fileio.write_float(f"{kind}_w.flxq", rng.standard_normal((16, 256)))
            fileio.write_float(f"{kind}_x.flxq", acts)
            entries.append({"layer_name": f"blk.0.{kind}", "kind": kind,
                            "weight_file": f"{kind}_w.flxq", "act_file": f"{kind}_x.flxq"})
        json.dump(entries, open("layers.json", "w"))
        assert main(["sensitivity", "layers.json", "-o", "report.json"]) == 0
        for src, dst in (("wq.flxq.manifest.json", "manifest_quantize.json"),
                         ("y.flxq.manifest.json", "manifest_gemm.json"),
                         ("bench.json", "bench_sweep.json"),
                         ("bench.json.manifest.json", "manifest_bench.json"),
                         ("layers.json", "sensitivity_manifest.json"),
                         ("report.json", "sensitivity_report.json")):
            shutil.copy(src, os.path.join(OUT, dst))
    finally:
        os.chdir(cwd)
        shutil.rmtree(work)
    print(sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main_()
