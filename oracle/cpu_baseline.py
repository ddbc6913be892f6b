"""Timed CPU baseline: the reference's online path, restated (oracle port).

TEST/BENCH INFRASTRUCTURE ONLY (bench.py's cpu_baseline and ``--impl
reference`` legs).  Per linear layer it times exactly what the reference does
online: quantize(x) (quantize.py:118-148) ->
pack(decompose(xq)) (bitplane.py:55-84, packing.py:132-147) ->
group_matmul_fused over pre-packed weights (engine.py:290-334), using the
numpy restatement in np_oracle.py.  Weight quantize+pack is offline and
excluded, as in the reference's own benchmark (bench.py:70-117).

Work is a bounded sample: the first ``rows`` output rows of every layer
(cost is linear in N, so throughput scales exactly), split across threads by
row shards (numpy's bitwise ufuncs release the GIL).
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import c_oracle, np_oracle


class SampledLayer:
    def __init__(self, n_rows: int, k: int, q: int, rng, group_size: int = 128, threads: int = 1):
        self.k, self.q, self.gs = k, q, group_size
        self.rows = n_rows
        w = rng.standard_normal((n_rows, k)).astype(np.float16)
        # offline: quantize + pack the sampled weight rows (fp16 scales, as the GPU path)
        wc, self.ws = c_oracle.quantize(w, 6, group_size, True)
        self.shards = []
        per = -(-n_rows // threads)
        per = -(-per // 8) * 8
        for r0 in range(0, n_rows, per):
            r1 = min(n_rows, r0 + per)
            words = np_oracle.pack_planes(np_oracle.bit_planes(wc[r0:r1], 6), 8)
            self.shards.append((r0, r1, words))

    def run(self, x: np.ndarray, pool: ThreadPoolExecutor | None):
        m = x.shape[0]
        xc, xs = np_oracle.quantize(x, self.q, self.gs, fp16_scales=True)
        xw = np_oracle.pack_planes(np_oracle.bit_planes(xc, self.q), np_oracle.activation_chunk_m(m))

        def shard(t):
            r0, r1, words = t
            y, _, _ = np_oracle.bitserial_matmul(words, xw, self.ws[r0:r1], xs, m, r1 - r0, self.k,
                                                 6, self.q, self.gs)
            return y

        parts = list(pool.map(shard, self.shards)) if pool else [shard(t) for t in self.shards]
        return np.concatenate(parts, axis=1)


class CpuBaseline:
    """The 7-layer workload, sampled to `rows_per_layer` output rows per layer."""

    def __init__(self, shapes, m: int, rows_per_layer: int, threads: int | None = None, seed: int = 0):
        self.threads = threads or os.cpu_count() or 1
        rng = np.random.default_rng(seed)
        self.m = m
        self.layers = [(s, SampledLayer(min(rows_per_layer, s.n), s.k, s.act_bits, rng,
                                        threads=self.threads)) for s in shapes]
        self.inputs = {s.k: rng.standard_normal((m, s.k)).astype(np.float16) for s in shapes}
        self.pool = ThreadPoolExecutor(self.threads) if self.threads > 1 else None

    @property
    def flops(self) -> int:
        return sum(2 * self.m * lay.rows * s.k for s, lay in self.layers)

    def step(self) -> float:
        t0 = time.perf_counter()
        for s, lay in self.layers:
            lay.run(self.inputs[s.k], self.pool)
        return time.perf_counter() - t0

    def describe(self) -> str:
        rows = sorted({lay.rows for _, lay in self.layers})
        return (f"first {rows} output rows of each of {len(self.layers)} layers, M={self.m}; "
                f"online quantize+pack+bit-serial GEMM (np_oracle restatement of "
                f"quantize.py:118 / packing.py:132 / engine.py:290), weights pre-packed")


def calibrate_rows(shapes, m: int, budget_s: float, threads: int | None = None, probe_rows: int = 16):
    """Rows per layer so one sampled step takes about `budget_s` seconds."""
    probe = CpuBaseline(shapes, m, probe_rows, threads)
    probe.step()  # warm
    t = probe.step()
    rows = int(probe_rows * budget_s / max(t, 1e-6))
    rows = max(8, min(rows, max(s.n for s in shapes)))
    return -(-rows // 8) * 8
