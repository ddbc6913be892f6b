"""Timed CPU baseline through the REAL reference (`bitserial` installed in baseline/_ref/).

BENCH INFRASTRUCTURE ONLY (bench.py's cpu_baseline and ``--impl reference`` legs).  Where
oracle/cpu_baseline.py times the numpy restatement, this imports the unmodified reference
package (tools/install_reference.sh) and times its own online path per linear layer, as
its bench does (/root/reference/pkg/src/bitserial/bench.py:70-117) but with the weights
pre-packed (offline, excluded):

    xq = quantize(x, q, 128, fp16_scales=True)               quantize.py:118-148
    xp = pack(decompose(xq), activation_pack_config(M))      bitplane.py:82, packing.py:132
    group_matmul_fused(wp, xp, wq.scales, xq.scales, cfg)    engine.py:290-334

Work is a bounded sample: the first ``rows`` output rows of every layer (cost is linear
in N), split into row shards (multiples of the 8-row weight chunk) run concurrently on a
thread pool -- numpy's AND/popcount/einsum release the GIL, so this is the reference's
fastest use of the host's cores (its execute_tiled worker pool is GIL-bound and slower,
README.md:124-126).
"""
from __future__ import annotations

import os
import platform
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "bitserial"))


def _bitserial():
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import bitserial

    return bitserial


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class RefLayer:
    def __init__(self, rows: int, k: int, q: int, rng, threads: int, group_size: int = 128):
        bs = _bitserial()
        self.k, self.q, self.gs, self.rows = k, q, group_size, rows
        w = rng.standard_normal((rows, k)).astype(np.float16).astype(np.float64)
        per = -(-rows // threads)
        per = -(-per // 8) * 8
        self.shards = []
        for r0 in range(0, rows, per):  # offline: quantize + pack each weight shard
            r1 = min(rows, r0 + per)
            wq = bs.quantize(w[r0:r1], 6, group_size, fp16_scales=True)
            wp = bs.pack(bs.decompose(wq), bs.weight_pack_config())
            self.shards.append((r1 - r0, wq, wp))

    def run(self, x: np.ndarray, pool):
        bs = _bitserial()
        m = x.shape[0]
        xq = bs.quantize(x, self.q, self.gs, fp16_scales=True)
        xp = bs.pack(bs.decompose(xq), bs.activation_pack_config(m))

        def shard(t):
            n, wq, wp = t
            cfg = bs.GemmConfig(m=m, n=n, k=self.k, weight_bits=6, activation_bits=self.q,
                                group_size=self.gs)
            return bs.group_matmul_fused(wp, xp, wq.scales, xq.scales, cfg).data

        parts = list(pool.map(shard, self.shards)) if pool else [shard(t) for t in self.shards]
        return np.concatenate(parts, axis=1)


class RefBaseline:
    """The decoder-layer workload through the reference, sampled to `rows` rows per layer."""

    kind = "reference"

    def __init__(self, shapes, m: int, rows_per_layer: int, threads: int | None = None,
                 seed: int = 0):
        self.threads = threads or os.cpu_count() or 1
        rng = np.random.default_rng(seed)
        self.m = m
        self.layers = [(s, RefLayer(min(rows_per_layer, s.n), s.k, s.act_bits, rng, self.threads))
                       for s in shapes]
        self.inputs = {s.k: rng.standard_normal((m, s.k)).astype(np.float16).astype(np.float64)
                       for s in shapes}
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
        return (f"first {rows} output rows of each of {len(self.layers)} layers, M={self.m}; the "
                f"reference package itself (baseline/_ref bitserial: quantize -> pack(decompose) -> "
                f"group_matmul_fused, quantize.py:118 / packing.py:132 / engine.py:290), weights "
                f"pre-packed, row shards on {self.threads} threads; CPU: {cpu_model()}")


def calibrate_rows(shapes, m: int, budget_s: float, threads: int | None = None,
                   probe_rows: int = 16) -> int:
    """Rows per layer so one sampled step takes about `budget_s` seconds."""
    threads = threads or os.cpu_count() or 1
    probe = RefBaseline(shapes, m, max(probe_rows, 8 * threads), threads)
    probe.step()  # warm
    t = probe.step()
    rows = int(max(probe_rows, 8 * threads) * budget_s / max(t, 1e-6))
    rows = max(8 * threads, min(rows, max(s.n for s in shapes)))
    return -(-rows // 8) * 8
