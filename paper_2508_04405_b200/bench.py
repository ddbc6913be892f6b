"""GEMM benchmark suites on the B200 (drop-in for bitserial.bench, bench.py:1-167).

Same cases, same report (schemas/bench_report.schema.json, restated in
reports.py), so ``bench --suite llama-shapes`` output from the reference's CPU
engine and from this GPU build can be diffed field by field.  ``wall_ns`` keeps
the reference's meaning -- host wall time of one numpy-in / numpy-out GEMM call,
best of ``repeat`` -- which on the GPU includes the H2D of the scales and the D2H
of the float64 result.  (Device-only kernel times are what the repo-root bench.py
and tools/sweep.py report.)

``engine`` picks the GPU kernel behind the call: ``"bitserial"`` runs
``execute_tiled`` over FLXQ-P operands (the reference's algorithm: AND+popcount
plane products, csrc/bitserial.cu), ``"t6"`` runs ``int_matmul_reference``
(the production T6 tensor-core GEMV/GEMM with the exact float64 epilogue).  Both
return bit-identical results.  The tile knobs are validated like the reference's
and recorded in the report, but the kernels choose their own CTA tiling, so the
"sweep" suite measures noise around one configuration; the B200 counterpart of
the reference's tile search is tools/sweep.py's kernel/M sweep.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .bitplane import decompose
from .engine import GemmConfig, execute_tiled, int_matmul_reference
from .errors import ConfigError
from .packing import activation_pack_config, pack, weight_pack_config
from .verify import random_quant

ENGINES = ("bitserial", "t6")


@dataclass(frozen=True)
class BenchCase:
    name: str
    m: int
    n: int
    k: int
    p: int = 6
    q: int = 6


@dataclass
class BenchResult:
    name: str
    shape: tuple[int, int, int]
    p: int
    q: int
    group_size: int
    stages: int
    workers: int
    tile: tuple[int, int, int]
    wall_ns: int
    bmma_passes: int
    effective_gops: float

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k in ("name", "shape", "p", "q", "group_size", "stages",
                                           "workers", "tile", "wall_ns", "bmma_passes")}
        d["shape"], d["tile"] = list(self.shape), list(self.tile)
        d["effective_GOPS"] = self.effective_gops
        return d


def _fit(v: int, extent: int, chunk: int) -> int:
    """Clamp a tile dim to the chunk-padded problem extent, at least one chunk."""
    return max(min(v, -(-extent // chunk) * chunk), chunk)


def run_case(case: BenchCase, group_size: int = 128, bm: int = 8, bn: int = 64, bk: int = 512,
             stages: int = 2, workers: int = 4, repeat: int = 3, seed: int = 0,
             engine: str = "bitserial") -> BenchResult:
    """Best-of-``repeat`` wall time of one GEMM shape (bench.py:68-117)."""
    if engine not in ENGINES:
        raise ConfigError(f"engine must be one of {ENGINES}, got {engine!r}")
    rng = np.random.default_rng(seed)
    wq = random_quant(rng, case.n, case.k, case.p, group_size)
    xq = random_quant(rng, case.m, case.k, case.q, group_size)
    wp = pack(decompose(wq), weight_pack_config())
    xp = pack(decompose(xq), activation_pack_config(case.m))
    cm, cn, ck = xp.config.chunk_m, wp.config.chunk_m, xp.config.chunk_k
    cfg = GemmConfig(m=case.m, n=case.n, k=case.k, weight_bits=case.p, activation_bits=case.q,
                     group_size=group_size, bm=_fit(bm, case.m, cm), bn=_fit(bn, case.n, cn),
                     bk=_fit(bk, case.k, ck), pipeline_stages=stages, worker_count=workers)
    if engine == "bitserial":
        def call():
            return execute_tiled(wp, xp, wq.scales, xq.scales, cfg)
    else:
        def call():
            return int_matmul_reference(wq, xq, cfg)
    call()  # first call uploads the operands and loads the kernels; not timed
    times, passes = [], 0
    for _ in range(repeat):
        t0 = time.perf_counter_ns()
        out = call()
        times.append(time.perf_counter_ns() - t0)
        passes = out.bmma_passes
    best = min(times)
    return BenchResult(name=case.name, shape=(case.m, case.n, case.k), p=case.p, q=case.q,
                       group_size=group_size, stages=stages, workers=workers,
                       tile=(cfg.bm, cfg.bn, cfg.bk), wall_ns=best, bmma_passes=passes,
                       effective_gops=2 * case.m * case.n * case.k / best)


def llama_shape_cases(scale: int = 8) -> list[BenchCase]:
    """Decoder linear shapes at batch 1/4/8 (bench.py:120-137): the 4096x4096 attention GEMM
    unscaled, the 7B and 70B FFN down projections (W6A8) divided by ``scale``."""
    classes = (("attn_4k", 4096, 4096, 6, 1), ("ffn_down_7b", 11008, 4096, 8, scale),
               ("ffn_down_70b", 28672, 8192, 8, scale))
    return [BenchCase(name=f"{name}_b{m}", m=m, n=n // div, k=k // div, p=6, q=q)
            for m in (1, 4, 8) for name, k, n, q, div in classes]


def run_llama_suite(scale: int = 8, repeat: int = 3, stages: int = 2, workers: int = 4,
                    engine: str = "bitserial") -> dict:
    return {"suite": "llama-shapes",
            "results": [run_case(c, repeat=repeat, stages=stages, workers=workers,
                                 engine=engine).to_dict() for c in llama_shape_cases(scale)]}


def run_sweep(m: int = 8, n: int = 256, k: int = 1024, p: int = 6, q: int = 6, repeat: int = 3,
              stages: int = 2, workers: int = 4, engine: str = "bitserial") -> dict:
    """Every (bm, bn, bk) of the reference grid (bench.py:146-167); the winner is the fastest,
    exact ties broken toward the smallest tile."""
    case = BenchCase(name="sweep", m=m, n=n, k=k, p=p, q=q)
    results = [run_case(case, bm=8, bn=bn, bk=bk, repeat=repeat, stages=stages, workers=workers,
                        engine=engine)
               for bn in (8, 16, 32, 64, 128) for bk in (128, 256, 512, 1024)]
    best = min(results, key=lambda r: (-r.effective_gops, r.tile))
    return {"suite": "sweep", "results": [r.to_dict() for r in results], "best": best.to_dict()}
