#!/usr/bin/env python
"""Benchmark: W6A6/W6A8 LLaMA-2-70B decoder-layer linears on B200.

One step = the 5 linear layers of one LLaMA-2-70B decoder layer (fused
qkv_proj, o/gate/up W6A6, down W6A8; group 128, fp16 scales) at batch M (default
1, decode GEMV), each the full online path: fused activation quantizer + T6
tensor-core GEMM/GEMV + fused dequant, fp16 in/out.  Weights are random-init
INT6 of the real shapes, inputs synthetic fp16; the 642 MB of packed weights
per step exceed the 126 MB L2, so every step streams from HBM.

    python bench.py [--gpus N --steps K --warmup W --batch M]
    torchrun --nproc-per-node N bench.py --gpus N ...   (column shards + NCCL all-gather)
    python bench.py --impl reference ...                (the reference's CPU path, oracle port)

Prints ONE JSON line (rank 0).  See DESIGN.md sec. 5 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "W6Ax linear effective TOPS (2*M*N*K / latency), LLaMA-2-70B decoder-layer linears"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--batch", type=int, default=1, help="tokens M per linear call")
    ap.add_argument("--model", default="llama2-70b",
                    help="llama2-7b / llama2-13b / llama2-70b decoder-layer linears, or config1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--cpu-budget", type=float, default=2.0,
                    help="seconds of CPU work per sampled cpu_baseline step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bitserial", action="store_true",
                    help="skip timing the BTC-equivalent AND+popcount kernel (the north star's "
                         "bit-serial vs unpack-to-INT8 decision, extra key 'bitserial')")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the M=8 and config-1 companion measurements")
    return ap.parse_args()


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---- clocks sampler (NVML, during the timed region) ------------------------------------------
class ClockSampler:
    def __init__(self, index: int, period: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self._stop = period, threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    _REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
                0x2: "applications_clocks_setting", 0x1: "gpu_idle", 0x10: "sync_boost"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---- CPU baseline: the reference package itself when installed (baseline/_ref), else the port
def cpu_baseline_impl():
    from oracle import ref_baseline

    if ref_baseline.available():
        return ref_baseline.RefBaseline, ref_baseline.calibrate_rows, "reference"
    from oracle.cpu_baseline import CpuBaseline, calibrate_rows

    return CpuBaseline, calibrate_rows, "port"


def reference_config1():
    """BASELINE config 1 at full size through the reference's own call: 4096x4096 W6A8, M=1,
    quantize + pack + group_matmul_fused (engine.py:290-334), one core (numpy), best of 3."""
    import numpy as np

    from oracle import ref_baseline

    if not ref_baseline.available():
        return None
    lay = ref_baseline.RefLayer(4096, 4096, 8, np.random.default_rng(7), threads=1)
    x = np.random.default_rng(8).standard_normal((1, 4096)).astype(np.float16).astype(np.float64)
    best = min((time.perf_counter(), lay.run(x, None), time.perf_counter()) for _ in range(3))
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        lay.run(x, None)
        ts.append(time.perf_counter() - t0)
    del best
    t = min(ts)
    return {"workload": "config 1: single W6A8 4096x4096 linear, M=1, full size", "s_per_call": t,
            "TOPS": 2 * 4096 * 4096 / t / 1e12, "cores": 1,
            "path": "bitserial.quantize -> pack(decompose) -> group_matmul_fused (baseline/_ref)"}


# ---- reference arm: the reference's CPU path on host cores --------------------------------------
def run_reference(args, shapes, rank):
    if rank != 0:
        return
    Impl, calibrate_rows, kind = cpu_baseline_impl()
    threads = os.cpu_count() or 1
    budget = max(0.2, min(3.0, 120.0 / max(1, args.steps + args.warmup)))
    rows = calibrate_rows(shapes, args.batch, budget, threads)
    cb = Impl(shapes, args.batch, rows, threads)
    for _ in range(args.warmup):
        cb.step()
    t = sum(cb.step() for _ in range(args.steps))
    tops = cb.flops * args.steps / t / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": tops, "unit": "TOPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u1 planes (AND+popcount), int64 accum, f64 epilogue",
        "data": "synthetic fp16 N(0,1) weights/activations",
        "config": {"workload": f"{args.model} decoder-layer linears, M={args.batch}, sampled rows",
                   "batch": args.batch, "group_size": 128},
        "cpu_baseline": {"value": tops, "unit": "TOPS", "cores": threads, "kind": kind,
                         "sample": cb.describe()},
        "e2e": {"value": tops, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_extra:
        line["config1"] = reference_config1()
    print(json.dumps(line), flush=True)


# ---- our arm ---------------------------------------------------------------------------------------
class Step:
    """One bench step over `layers` at batch M: per linear the fused activation quantizer +
    the T6 GEMV/GEMM (FlexQLinear.forward), then the shard-boundary collective under
    torchrun; captured once in a CUDA graph.  `gemm` replays only the GEMM launches (the
    dominant kernel, for the roofline)."""

    def __init__(self, torch, dist, layers, M, world, rank, dev):
        self.torch, self.dist, self.layers, self.M, self.world = torch, dist, layers, M, world
        self.dev = dev
        self.inputs, self.x_loc, self.outs, self.gathered = {}, [], [], []
        for s, lay in layers:
            if s.k not in self.inputs:
                gx = torch.Generator(device=dev)
                gx.manual_seed(99 + s.k + 7919 * M)  # same activations on every rank
                self.inputs[s.k] = torch.randn((M, s.k), generator=gx, device=dev, dtype=torch.float16)
            kl = lay.k
            self.x_loc.append(self.inputs[s.k][:, rank * kl:(rank + 1) * kl].contiguous()
                              if lay.mode == "row" else self.inputs[s.k])
            self.outs.append(torch.empty((M, lay.n), device=dev, dtype=torch.float32
                                         if lay.mode == "row" else torch.float16))
            self.gathered.append(torch.empty((world, M, lay.n), dtype=torch.float16, device=dev)
                                 if world > 1 and lay.mode == "column" else None)
        for _ in range(3):  # eager warm-up: allocates the per-M buffers
            self.eager()
        torch.cuda.synchronize()
        self.graph, self.ggraph = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(self.graph):
                self.eager()
            with torch.cuda.graph(self.ggraph):
                self.gemm_eager()
            self.run, self.gemm = self.graph.replay, self.ggraph.replay
        except Exception as e:  # e.g. NCCL capture unsupported: time eager launches instead
            print(f"[bench] graph capture failed ({e}); timing eager launches", file=sys.stderr)
            self.run, self.gemm = self.eager, self.gemm_eager

    def eager(self):
        for i, (s, lay) in enumerate(self.layers):
            lay.forward(self.x_loc[i], out=self.outs[i])
            if self.world > 1:
                if lay.mode == "row":
                    self.dist.all_reduce(self.outs[i], op=self.dist.ReduceOp.SUM)
                else:
                    self.dist.all_gather_into_tensor(self.gathered[i], self.outs[i])

    def gemm_eager(self):
        for i, (s, lay) in enumerate(self.layers):
            lay.gemm_only(self.M, self.outs[i])

    def timed(self, fn, reps):
        torch, dist, world = self.torch, self.dist, self.world
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1) / reps
        if world > 1:
            t = torch.tensor([ms], device=self.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def summary(self, shapes, ms_step, ms_gemm):
        from paper_2508_04405_b200.shapes import gemm_bytes

        M = self.M
        flops = sum(2 * M * s.n * s.k for s in shapes)
        gb = sum(gemm_bytes(M, lay.n, lay.k) for _, lay in self.layers)
        peak, _ = hbm_peak()
        return {"ms_per_step": ms_step, "value": flops / (ms_step * 1e-3) / 1e12, "unit": "TOPS",
                "gemm_us_per_step": ms_gemm * 1e3,
                "roofline_frac": gb / (ms_gemm * 1e-3) / 1e9 / peak,
                "step_frac": gb / (ms_step * 1e-3) / 1e9 / peak}


def build_layers(torch, FlexQLinear, shapes, world, rank, dev, seed=1234):
    """Random-init INT6 layers of the real shapes.  Megatron pairing under torchrun (SURVEY.md
    sec. 8(e), sharding.py): qkv/gate/up are column shards (rank r owns N/world output rows;
    replicated x; NCCL all-gather of the fp16 y shards), o/down are row shards (rank r owns
    K/world input columns on group boundaries; fp32 partial y; NCCL all-reduce)."""
    from paper_2508_04405_b200.shapes import policy_kind

    g = torch.Generator(device=dev)
    g.manual_seed(seed + rank)
    layers = []
    for s in shapes:
        mode = "row" if (world > 1 and s.name in ("o_proj", "down_proj")) else "column"
        n_loc, k_loc = (s.n, s.k // world) if mode == "row" else (s.n // world, s.k)
        w = torch.randn((n_loc, k_loc), generator=g, device=dev, dtype=torch.float16)
        lay = FlexQLinear(w, 6, s.act_bits, 128, fp16_scales=True, layer_kind=policy_kind(s.name))
        lay.mode = mode
        del w
        layers.append((s, lay))
    torch.cuda.synchronize()
    return layers


def main():
    args = parse()
    import torch

    from paper_2508_04405_b200.shapes import MODELS, WORKLOADS, layer_bytes

    shapes = WORKLOADS.get(args.model) or MODELS[args.model]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, shapes, rank)
        return

    import torch.distributed as dist

    from paper_2508_04405_b200 import FlexQLinear, _lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    M = args.batch
    layers = build_layers(torch, FlexQLinear, shapes, world, rank, dev)
    st = Step(torch, dist, layers, M, world, rank, dev)
    for _ in range(args.warmup):
        st.run()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms_step = st.timed(st.run, args.steps)
    ms_gemm = st.timed(st.gemm, max(args.steps // 2, 10))

    # ---- e2e through the public API: pinned host x -> device, one forward per layer, y -> pinned host
    inputs = st.inputs
    host_in = {k: v.cpu().pin_memory() for k, v in inputs.items()}
    dev_in = {k: torch.empty_like(v) for k, v in inputs.items()}
    host_out = [torch.empty((M, s.n), dtype=torch.float16).pin_memory() for s, _ in layers]
    h2d = sum(v.numel() * 2 for v in host_in.values())
    d2h = sum(o.numel() * 2 for o in host_out)

    # single GPU: the step's inputs travel in one pinned buffer (one H2D copy) and the
    # layers write into views of one device output buffer read back by one D2H copy
    in_sizes = {k_: v.numel() for k_, v in inputs.items()}
    host_in_all = torch.empty(sum(in_sizes.values()), dtype=torch.float16).pin_memory()
    dev_in_all = torch.empty_like(host_in_all, device=dev)
    in_views, off = {}, 0
    for k_, v in inputs.items():
        host_in_all[off:off + in_sizes[k_]].copy_(host_in[k_].reshape(-1))
        in_views[k_] = dev_in_all[off:off + in_sizes[k_]].view(v.shape)
        off += in_sizes[k_]
    out_sizes = [M * lay.n for _, lay in layers]
    dev_out_all = torch.empty(sum(out_sizes), dtype=torch.float16, device=dev)
    host_out_all = torch.empty(sum(out_sizes), dtype=torch.float16).pin_memory()
    out_views, off = [], 0
    for (_, lay), sz in zip(layers, out_sizes):
        out_views.append(dev_out_all[off:off + sz].view(M, lay.n))
        off += sz

    def e2e_step():
        if world == 1:
            dev_in_all.copy_(host_in_all, non_blocking=True)
            for i, (s, lay) in enumerate(layers):
                lay(in_views[s.k], out=out_views[i])
            host_out_all.copy_(dev_out_all, non_blocking=True)
            return
        for k_, hv in host_in.items():
            dev_in[k_].copy_(hv, non_blocking=True)
        for i, (s, lay) in enumerate(layers):
            if lay.mode == "row":
                kl = lay.k
                y = lay(dev_in[s.k][:, rank * kl:(rank + 1) * kl].contiguous(),
                        out_dtype=torch.float32)
                dist.all_reduce(y, op=dist.ReduceOp.SUM)
                y = y.half()
            else:
                y = lay(dev_in[s.k])
                dist.all_gather_into_tensor(st.gathered[i], y)
                y = st.gathered[i].permute(1, 0, 2).reshape(M, -1)
            host_out[i].copy_(y, non_blocking=True)

    for _ in range(5):
        e2e_step()
    ms_e2e = st.timed(e2e_step, args.e2e_steps)

    def eager_step():  # diagnostic: the same eager forwards without the host copies
        for i, (s, lay) in enumerate(layers):
            lay(in_views[s.k] if world == 1 else dev_in[s.k], out=out_views[i] if world == 1 else None)

    ms_eager = st.timed(eager_step, args.e2e_steps) if world == 1 else None

    from paper_2508_04405_b200.shapes import gemm_bytes

    flops_total = sum(2 * M * s.n * s.k for s in shapes)  # whole job (all ranks)
    tops = flops_total / (ms_step * 1e-3) / 1e12
    gbytes_loc = sum(gemm_bytes(M, lay.n, lay.k) for s, lay in layers)
    layer_b = sum(layer_bytes(M, s.n, s.k) for s in shapes)
    peak, peak_kind = hbm_peak()
    achieved = gbytes_loc / (ms_gemm * 1e-3) / 1e9
    traffic = None
    try:
        with open(PROFILE_SUMMARY) as f:
            prof = json.load(f)
        key = f"{args.model}_m{M}"
        if key in prof.get("gemm_traffic_bytes_per_step", {}):
            traffic = prof["gemm_traffic_bytes_per_step"][key] / len(shapes)
    except Exception:
        pass
    launches_per_fwd = 2  # fused activation quantizer + one GEMV/GEMM kernel per linear
    # the kernel flexq_linear_forward routes each layer to (flexq_linear_kernel)
    names = {_lib.KERNEL_GEMV: ("flexq::gemv_t6_stream_kernel", "int8 IMMA mma.sync (u6 offset-binary W x s8 A), int32 accum, fp32 epilogue"),
             _lib.KERNEL_TC_I8: ("flexq::gemm_tc_kernel (tcgen05.mma kind::i8)", "int8 tcgen05.mma kind::i8 (u6 offset-binary W x s8 A), int32 accum, fp32 epilogue"),
             _lib.KERNEL_TC16: ("flexq::gemm_tc16_kernel (tcgen05.mma kind::f16)", "tcgen05.mma kind::f16 over fp16(w*ws) x fp16(code*xs) (INT6/INT8 codes, fp16 scales), fp32 accum"),
             _lib.KERNEL_MMA_SYNC: ("flexq::gemm_t6_kernel (mma.sync)", "int8 IMMA mma.sync, int32 accum")}
    kinds = sorted({_lib.lib().flexq_linear_kernel(M, lay.n, lay.k, 128, 1) for _, lay in layers})
    kernel_label = " + ".join(names[k_][0] for k_ in kinds)
    dtype_label = " + ".join(names[k_][1] for k_ in kinds)
    desc = (f"{args.model} decoder-layer linears qkv,o,gate,up (W6A6) + down (W6A8), M={M}"
            if args.model in MODELS else WORKLOAD_DESC.get(args.model, args.model) + f", M={M}")
    wbytes = sum(lay.weight_bytes for _, lay in layers) * world
    line = {
        "metric": METRIC, "value": tops, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": dtype_label + ", fp16 out",
        "data": "synthetic: random-init INT6 weights of the real shapes (fp16 N(0,1) quantized), fp16 N(0,1) activations",
        "config": {"workload": desc, "batch": M, "group_size": 128, "scales": "fp16",
                   "parallelism": (f"tp{world}: qkv/gate/up column shards + NCCL all-gather, "
                                   f"o/down row shards (fp32 partials) + NCCL all-reduce")
                                  if world > 1 else "single GPU",
                   "l2": (f"weights {wbytes / 1e6:.0f} MB/step > 126 MB L2 (no flush needed)"
                          if wbytes > 2 * 126e6 else
                          f"weights {wbytes / 1e6:.0f} MB/step: L2 flushed between steps"),
                   "timing": "CUDA-graph replay of the whole step, CUDA events, max over ranks"},
        "latency_us_per_step": ms_step * 1e3,
        "weight_GBps": wbytes / (ms_step * 1e-3) / 1e9,
        "hbm_GBps_algorithmic": layer_b / (ms_step * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": kernel_label
                               + f" ({len(shapes)} launches/step, per-launch bytes in DESIGN.md sec. 4)",
                     "peak_source": peak_kind, "gemm_us_per_step": ms_gemm * 1e3,
                     "step_frac": gbytes_loc / (ms_step * 1e-3) / 1e9 / peak},
        "clocks": clk.summary(),
        "e2e": {"value": flops_total / (ms_e2e * 1e-3) / 1e12, "unit": "TOPS",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": ms_e2e, "ms_per_step_eager_no_copies": ms_eager,
                "path": "FlexQLinear.__call__ (public API); per step one H2D of the inputs from pinned host memory and one D2H of all outputs"},
        "gpu_launches": args.steps * len(shapes) * launches_per_fwd,
        "tuning": _lib.lib().flexq_tuning().decode(),
    }
    if world == 1 and not args.no_extra:
        line["extra"] = extra_lines(torch, dist, FlexQLinear, layers, shapes, args, dev)
    if not args.no_bitserial and world == 1:
        line["bitserial"] = time_bitserial(layers, M, shapes)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Impl, calibrate_rows, kind = cpu_baseline_impl()
        threads = os.cpu_count() or 1
        rows = calibrate_rows(shapes, M, args.cpu_budget, threads)
        cb = Impl(shapes, M, rows, threads)
        cb.step()
        reps = 3
        tcpu = sum(cb.step() for _ in range(reps)) / reps
        line["cpu_baseline"] = {"value": cb.flops / tcpu / 1e12, "unit": "TOPS", "cores": threads,
                                "kind": kind, "sample": cb.describe()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


WORKLOAD_DESC = {"config1": "BASELINE config 1: single W6A8 4096x4096 linear (GEMV)"}


def extra_lines(torch, dist, FlexQLinear, layers, shapes, args, dev):
    """Driver-run companions of the headline (same process, same clocks): the same 70B step
    at M=8 (the top of the north star's batch 1-8 band) and BASELINE config 1 (one W6A8
    4096x4096 linear at M=1; 12.6 MB of weights < L2, so 16 distinct copies are cycled to
    stream from HBM)."""
    from paper_2508_04405_b200.shapes import WORKLOADS

    out = {}
    if args.batch != 8 and args.model == "llama2-70b":
        st = Step(torch, dist, layers, 8, 1, 0, dev)
        for _ in range(20):
            st.run()
        out["llama2-70b_m8"] = st.summary(shapes, st.timed(st.run, 1000), st.timed(st.gemm, 500))
        del st
    c1 = WORKLOADS["config1"]
    copies = [build_layers(torch, FlexQLinear, c1, 1, 0, dev, seed=4321 + i) for i in range(16)]
    st = Step(torch, dist, [l for c in copies for l in c], 1, 1, 0, dev)  # 16 layers per replay
    for _ in range(20):
        st.run()
    s16 = st.summary(c1 * 16, st.timed(st.run, 500), st.timed(st.gemm, 500))
    s16["us_per_linear"] = s16["ms_per_step"] * 1e3 / 16
    s16["gemm_us_per_linear"] = s16["gemm_us_per_step"] / 16
    s16["note"] = "one replay = 16 distinct 4096x4096 W6A8 layers back to back (>2x L2 of weights)"
    out["config1_w6a8_4096_m1"] = s16
    return out


def time_bitserial(layers, M, shapes):
    """BTC-equivalent AND+popcount kernel over FLXQ-P planes, same step (extra key)."""
    import torch

    from paper_2508_04405_b200 import _lib, pack, weight_pack_config, activation_pack_config
    from paper_2508_04405_b200.bitplane import BitPlaneSet, plane_coeffs

    L = _lib.lib()
    runs = []
    for s, lay in layers:
        codes, scales = lay.qweight.device_tensors()
        wp = pack(BitPlaneSet(None, plane_coeffs(6), 6, True, _codes=codes.to(torch.int16),
                              _numpy=False), weight_pack_config())
        xc = torch.randint(-31, 32, (M, s.k), dtype=torch.int16, device=codes.device)
        xp = pack(BitPlaneSet(None, plane_coeffs(s.act_bits), s.act_bits, True, _codes=xc,
                              _numpy=False), activation_pack_config(M))
        ng = -(-s.k // 128)
        wsf = scales.float().contiguous()
        xsf = torch.ones((M, ng), dtype=torch.float32, device=codes.device)
        y = torch.empty((M, lay.n), dtype=torch.float16, device=codes.device)
        wsp = torch.zeros(max(L.flexq_gemm_workspace_bytes(M, lay.n, s.k, 128, 0), 16),
                          dtype=torch.uint8, device=codes.device)
        runs.append((s, lay, wp, xp, wsf, xsf, y, wsp))

    def go():
        for s, lay, wp, xp, wsf, xsf, y, wsp in runs:
            _lib.check(L.flexq_gemm_bitserial(
                _lib.ptr(wp.device_bytes()), _lib.ptr(xp.device_bytes()), _lib.ptr(wsf),
                _lib.ptr(xsf), M, lay.n, s.k, 6, s.act_bits, 128, 8, min(M, 8), None,
                _lib.ptr(y), _lib.OUT_F16, _lib.ptr(wsp), 0, _lib.stream()))

    go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        go()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = sum(2 * M * s.n * s.k for s in shapes)
    wbytes = sum(s.n * s.k * 6 // 8 for s in shapes)
    return {"ms_per_step": ms, "TOPS": flops / (ms * 1e-3) / 1e12,
            "weight_GBps": wbytes / (ms * 1e-3) / 1e9}


if __name__ == "__main__":
    main()
