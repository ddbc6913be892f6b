"""Freeze FLXQ containers written by the REAL reference (bitserial.fileio).

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_flxq_golden.py

Writes tests/golden/flxq/*.flxq (each produced by the reference's own writers,
fileio.py:85-111, from the reference's quantize/pack) and
tests/golden/flxq/expect.npz with the arrays each container must decode to plus
the reference's quantized_linear output (engine.py:487-513) for the weight
containers (the reference engine run on the stored weights with FlexQLinear's
activation quantizer mode, fp16-rounded scales), so the GPU tests can check that a
reference-quantized weight file loaded into FlexQLinear serves the same y.  The GPU box reads only these files.
"""
from __future__ import annotations

import os

import numpy as np

from bitserial import fileio
from bitserial.bitplane import decompose
from bitserial.engine import GemmConfig, group_matmul_fused, quantized_linear
from bitserial.packing import activation_pack_config, pack, weight_pack_config
from bitserial.quantize import quantize

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "flxq")


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20250806)
    exp = {}

    def path(name):
        return os.path.join(OUT, name + ".flxq")

    # kind 0: float tensors in three payload dtypes
    f = rng.standard_normal((5, 33))
    for dt, tag in (("<f8", "f8"), ("<f4", "f4"), ("<f2", "f2")):
        fileio.write_float(path(f"float_{tag}"), f, dtype=dt)
        exp[f"float_{tag}"] = f.astype(np.dtype(dt)).astype(np.float64)

    # weights for the serving tests: fp16-valued [N, K] with a ragged last group
    n, k, m = 72, 320, 5
    w = rng.standard_normal((n, k)).astype(np.float16).astype(np.float64)
    x = rng.standard_normal((m, k))
    x[:, 9] *= 40.0  # outlier channel
    x = x.astype(np.float16).astype(np.float64)
    exp["weight"], exp["x"] = w.astype(np.float16), x.astype(np.float16)
    fileio.write_float(path("weight_f2"), w, dtype="<f2")

    # kind 1: W6 g128 with f8 scales, W6 g64 with fp16 scales, A8 per-token
    for name, bits, gs, fp16 in (("wq6_g128_f8", 6, 128, False), ("wq6_g64_f2", 6, 64, True)):
        q = quantize(w, bits, gs, fp16_scales=fp16)
        fileio.write_quant(path(name), q, scale_dtype="<f2" if fp16 else "<f8")
        exp[name + "_values"], exp[name + "_scales"] = q.values, q.scales
        for a_bits in (6, 8):
            # the reference engine on these stored weights with FlexQLinear's activation
            # quantizer mode (fp16-rounded per-token scales, quantize.py:118-148)
            xq = quantize(x, a_bits, gs, fp16_scales=True)
            cfg = GemmConfig(m=m, n=n, k=k, weight_bits=bits, activation_bits=a_bits, group_size=gs)
            exp[f"{name}_y_a{a_bits}"] = group_matmul_fused(
                pack(decompose(q), weight_pack_config()), pack(decompose(xq), activation_pack_config(m)),
                q.scales, xq.scales, cfg).data
            if not fp16:  # and the reference's one-call path (f8 scales throughout)
                exp[f"{name}_ql_a{a_bits}"] = quantized_linear(w, x, bits, a_bits, gs).data
    qa = quantize(x, 8, 4096)
    fileio.write_quant(path("xq8_pertoken"), qa)
    exp["xq8_pertoken_values"], exp["xq8_pertoken_scales"] = qa.values, qa.scales

    # kind 2: FLXQ-P weights (64-bit words, 8-row chunks) and activations (32-bit words)
    wq = quantize(w, 6, 128)
    wp = pack(decompose(wq), weight_pack_config(64))
    fileio.write_packed(path("wp6_w64"), wp)
    exp["wp6_w64_words"] = wp.words
    xq = quantize(x[:3, :200], 6, 128)
    xp = pack(decompose(xq), activation_pack_config(3, 32))
    fileio.write_packed(path("xp6_w32"), xp)
    exp["xp6_w32_words"], exp["xp6_w32_values"] = xp.words, xq.values

    np.savez_compressed(os.path.join(OUT, "expect.npz"), **exp)
    for fn in sorted(os.listdir(OUT)):
        print(fn, os.path.getsize(os.path.join(OUT, fn)), fileio.file_digest(os.path.join(OUT, fn))[:16])


if __name__ == "__main__":
    main()
