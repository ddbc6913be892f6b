"""Freeze golden vectors from the REAL reference package (bitserial).

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  The fixtures pin both the CPU oracle
(oracle/np_oracle.py, oracle/flexq_oracle.c) and the CUDA path: codes,
scales, FLXQ-P packed words, exact per-group INT partials, float64 outputs
and bmma pass counts, all produced by the reference's own functions
(quantize.py:118, packing.py:132, engine.py:290/337/487).  The GPU box never
reads /root/reference; it only reads the committed .npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

from bitserial.bitplane import decompose
from bitserial.engine import GemmConfig, group_matmul_fused, int_matmul_reference, quantized_linear
from bitserial.packing import activation_pack_config, pack, weight_pack_config
from bitserial.quantize import quantize
from bitserial.verify import random_quant

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main() -> None:
    g = {}
    # ---- quantizer known-answer tests (test_quantize.py:42-45, 87-91) + random
    qcases = [
        ("kat_unit_pair", np.array([[1.0, -1.0]]), 6, 2, False),
        ("kat_half_away", np.array([[2.5, -2.5, 31.0]]), 6, 3, False),
        ("kat_zeros", np.zeros((3, 8)), 6, 4, False),
    ]
    rng = np.random.default_rng(424242)
    for bits in (6, 8):
        for gs in (128, 32, 999):
            for fp16 in (False, True):
                x = rng.standard_normal((5, 300)) * rng.uniform(1e-2, 1e2, size=(5, 1))
                if fp16:  # fp16-valued inputs, the B200 activation dtype
                    x = x.astype(np.float16).astype(np.float64)
                qcases.append((f"rand_b{bits}_g{gs}_f{int(fp16)}", x, bits, gs, fp16))
    # outlier channel (sensitivity.py:189-190 style), fp16 values, per-token (g >= K)
    x = rng.standard_normal((4, 512)); x[:, 7] *= 100.0
    qcases.append(("outlier_pertoken_b8", x.astype(np.float16).astype(np.float64), 8, 4096, True))
    names = []
    for name, x, bits, gs, fp16 in qcases:
        q = quantize(x, bits, gs, fp16_scales=fp16)
        g[f"q/{name}/x"] = x
        g[f"q/{name}/meta"] = np.array([bits, gs, int(fp16)])
        g[f"q/{name}/values"] = q.values
        g[f"q/{name}/scales"] = q.scales
        names.append(name)
    g["q/names"] = np.array(names)

    # ---- packing (test_packing.py:44-56, 88-97)
    pcases = [(8, 256, 6, "w"), (1, 512, 6, "a"), (9, 300, 3, "a"), (17, 1000, 6, "a"),
              (3, 200, 6, "w"), (20, 384, 8, "a"), (24, 640, 6, "w")]
    pnames = []
    for i, (rows, cols, bits, kind) in enumerate(pcases):
        q = random_quant(rng, rows, cols, bits, 128)
        cfg = weight_pack_config() if kind == "w" else activation_pack_config(rows)
        p = pack(decompose(q), cfg)
        name = f"p{i}"
        g[f"p/{name}/values"] = q.values
        g[f"p/{name}/meta"] = np.array([rows, cols, bits, cfg.chunk_m])
        g[f"p/{name}/words"] = p.words
        pnames.append(name)
    g["p/names"] = np.array(pnames)

    # ---- GEMM (test_engine.py:108-161, test_acceptance.py:32-63)
    gcases = []
    for pq in ((6, 6), (6, 8)):
        for (m, n, k) in ((1, 8, 128), (4, 8, 512), (8, 24, 384), (16, 40, 1024), (1, 64, 4096), (3, 17, 300)):
            gcases.append((m, n, k, pq[0], pq[1], 128))
    for gs in (32, 64, 96, 256, 999):
        gcases.append((4, 8, 384, 6, 6, gs))
    for p in (2, 4, 8):
        for q in (3, 6, 8):
            gcases.append((3, 5, 192, p, q, 64))
    gcases.append((5, 16, 256, 6, 8, 4096))  # per-channel / per-token (g >= K)
    gnames = []
    for i, (m, n, k, p, q, gs) in enumerate(gcases):
        wq = random_quant(rng, n, k, p, gs)
        xq = random_quant(rng, m, k, q, gs)
        cfg = GemmConfig(m=m, n=n, k=k, weight_bits=p, activation_bits=q, group_size=gs)
        wp = pack(decompose(wq), weight_pack_config())
        xp = pack(decompose(xq), activation_pack_config(m))
        fused = group_matmul_fused(wp, xp, wq.scales, xq.scales, cfg, trace=True)
        ref = int_matmul_reference(wq, xq, cfg, trace=True)
        assert np.array_equal(fused.data, ref.data)
        assert np.abs(ref.group_partials).max() < 2**31
        name = f"g{i}"
        g[f"g/{name}/meta"] = np.array([m, n, k, p, q, gs, fused.bmma_passes])
        g[f"g/{name}/wv"] = wq.values
        g[f"g/{name}/ws"] = wq.scales
        g[f"g/{name}/xv"] = xq.values
        g[f"g/{name}/xs"] = xq.scales
        g[f"g/{name}/y"] = fused.data
        g[f"g/{name}/partials"] = fused.group_partials.astype(np.int32)
        gnames.append(name)
    g["g/names"] = np.array(gnames)

    # ---- quantized_linear from float inputs (engine.py:487-513), incl. KATs (test_engine.py:171-176)
    lcases = [("ones_1x256", np.ones((1, 256)), np.ones((1, 256)), 6, 6, 128)]
    for (m, n, k, q) in ((1, 32, 2048, 6), (4, 16, 640, 8), (8, 40, 1024, 6)):
        w = rng.standard_normal((n, k))
        x = rng.standard_normal((m, k)) * 3
        lcases.append((f"lin_m{m}_n{n}_k{k}_q{q}", w, x, 6, q, 128))
    lnames = []
    for name, w, x, p, q, gs in lcases:
        out = quantized_linear(w, x, p, q, gs, trace=True)
        g[f"l/{name}/w"] = w
        g[f"l/{name}/x"] = x
        g[f"l/{name}/meta"] = np.array([p, q, gs, out.bmma_passes])
        g[f"l/{name}/y"] = out.data
        g[f"l/{name}/partials"] = out.group_partials.astype(np.int32)
        lnames.append(name)
    g["l/names"] = np.array(lnames)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {os.path.getsize(OUT) / 1e6:.2f} MB, {len(g)} arrays")


if __name__ == "__main__":
    if "bitserial" not in sys.modules and not os.path.isdir("/root/reference/pkg/src"):
        raise SystemExit("needs the reference: PYTHONPATH=/root/reference/pkg/src")
    main()
