"""The fp32 quantization steps of the production quantizer (csrc/quant_math.cuh:
group_scale_h, quant_one_h) are bit-identical to the reference's float64 steps
(quantize.py:29-36, 99-148) for fp16 inputs and fp16 scales: exhaustive over every
(finite fp16 value, positive fp16 scale) pair and every fp16 group peak (tools/check_f32_quant.c,
plain C on the host -- no GPU)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_f32_quantization_is_exact(tmp_path):
    exe = str(tmp_path / "check_f32_quant")
    subprocess.run(["gcc", "-O2", "-o", exe, os.path.join(ROOT, "tools", "check_f32_quant.c"), "-lm"],
                   check=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True, timeout=600).stdout
    assert "codes: pairs 2015299584 mismatches 0" in out
    assert "scales: cases 222201 mismatches 0" in out
