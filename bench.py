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
    ap.add_argument("--model", default="llama2-70b")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--cpu-budget", type=float, default=2.0,
                    help="seconds of CPU work per sampled cpu_baseline step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--bitserial", action="store_true",
                    help="also time the BTC-equivalent bit-serial kernel (extra key)")
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


# ---- reference arm: the reference's CPU path (oracle port) on host cores -------------------
def run_reference(args, shapes, rank):
    if rank != 0:
        return
    from oracle.cpu_baseline import CpuBaseline, calibrate_rows

    threads = os.cpu_count() or 1
    budget = max(0.2, min(3.0, 120.0 / max(1, args.steps + args.warmup)))
    rows = calibrate_rows(shapes, args.batch, budget, threads)
    cb = CpuBaseline(shapes, args.batch, rows, threads)
    for _ in range(args.warmup):
        cb.step()
    t = sum(cb.step() for _ in range(args.steps))
    tops = cb.flops * args.steps / t / 1e12
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": tops, "unit": "TOPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u1 planes (AND+popcount), int64 accum, f64 epilogue",
        "data": "synthetic fp16 N(0,1) weights/activations",
        "config": {"workload": f"{args.model} decoder-layer linears, M={args.batch}, sampled rows",
                   "batch": args.batch, "group_size": 128},
        "cpu_baseline": {"value": tops, "unit": "TOPS", "cores": threads, "kind": "port",
                         "sample": cb.describe()},
        "e2e": {"value": tops, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---- our arm ---------------------------------------------------------------------------------------
def main():
    args = parse()
    import torch

    from paper_2508_04405_b200.shapes import MODELS, gemm_bytes, layer_bytes, policy_kind

    shapes = MODELS[args.model]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, shapes, rank)
        return

    import torch.distributed as dist

    from paper_2508_04405_b200 import FlexQLinear

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    M = args.batch
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)

    # Megatron pairing under torchrun (sharding.py): qkv/gate/up are
    # column shards (rank r owns N/world output rows; replicated x; NCCL all-gather of the
    # fp16 y shards), o/down are row shards (rank r owns K/world input columns on group
    # boundaries; fp32 partial y; NCCL all-reduce).  world = 1: plain layers, no collective.
    ROW_SHARDED = ("o_proj", "down_proj")
    layers, inputs, outs, gathered, x_loc = [], {}, [], [], []
    for s in shapes:
        mode = "row" if (world > 1 and s.name in ROW_SHARDED) else "column"
        n_loc, k_loc = (s.n, s.k // world) if mode == "row" else (s.n // world, s.k)
        w = torch.randn((n_loc, k_loc), generator=g, device=dev, dtype=torch.float16)
        lay = FlexQLinear(w, 6, s.act_bits, 128, fp16_scales=True, layer_kind=policy_kind(s.name))
        lay.mode = mode
        del w
        layers.append((s, lay))
        if s.k not in inputs:
            gx = torch.Generator(device=dev)
            gx.manual_seed(99 + s.k)  # same activations on every rank (replicated X)
            inputs[s.k] = torch.randn((M, s.k), generator=gx, device=dev, dtype=torch.float16)
        x_loc.append(inputs[s.k][:, rank * k_loc:(rank + 1) * k_loc].contiguous()
                     if mode == "row" else inputs[s.k])
        outs.append(torch.empty((M, n_loc), device=dev,
                                dtype=torch.float32 if mode == "row" else torch.float16))
        gathered.append(torch.empty((world, M, n_loc), dtype=torch.float16, device=dev)
                        if world > 1 and mode == "column" else None)
    torch.cuda.synchronize()

    def collective(i, y):
        if world == 1:
            return
        if layers[i][1].mode == "row":
            dist.all_reduce(y, op=dist.ReduceOp.SUM)
        else:
            dist.all_gather_into_tensor(gathered[i], y)

    def step():
        for i, (s, lay) in enumerate(layers):
            lay.forward(x_loc[i], out=outs[i])
            collective(i, outs[i])

    def gemm_step():
        for i, (s, lay) in enumerate(layers):
            lay.gemm_only(M, outs[i])

    for _ in range(3):  # eager warm-up: allocates per-M buffers
        step()
    torch.cuda.synchronize()
    graph, ggraph = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    use_graph = True
    try:
        with torch.cuda.graph(graph):
            step()
        with torch.cuda.graph(ggraph):
            gemm_step()
    except Exception as e:  # e.g. NCCL capture unsupported: time eager launches instead
        print(f"[bench] graph capture failed ({e}); timing eager launches", file=sys.stderr)
        use_graph = False
    run = graph.replay if use_graph else step
    run_gemm = ggraph.replay if use_graph else gemm_step

    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()

    def timed(fn, reps):
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
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    with ClockSampler(local) as clk:
        ms_step = timed(run, args.steps)
    ms_gemm = timed(run_gemm, max(args.steps // 2, 10))

    # ---- e2e through the public API: pinned host x -> device, one forward per layer, y -> pinned host
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
                kl = s.k // world
                y = lay(dev_in[s.k][:, rank * kl:(rank + 1) * kl].contiguous(),
                        out_dtype=torch.float32)
                dist.all_reduce(y, op=dist.ReduceOp.SUM)
                y = y.half()
            else:
                y = lay(dev_in[s.k])
                dist.all_gather_into_tensor(gathered[i], y)
                y = gathered[i].permute(1, 0, 2).reshape(M, -1)
            host_out[i].copy_(y, non_blocking=True)

    for _ in range(5):
        e2e_step()
    ms_e2e = timed(e2e_step, args.e2e_steps)

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
    # the automatic route (csrc/gemm_t6.cu): streaming GEMV for M <= 16, and for M <= 32 on
    # layers of >= 8192 units (64 rows x 128 k); tcgen05 otherwise
    streamed = [M <= 16 or (M <= 32 and -(-lay.n // 64) * -(-lay.k // 128) >= 8192) for _, lay in layers]
    kern_gemv = "flexq::gemv_t6_stream_kernel"
    kern_tc = "flexq::gemm_tc_kernel (tcgen05.mma kind::i8)"
    kernel_label = kern_gemv if all(streamed) else kern_tc if not any(streamed) else \
        f"{kern_gemv} + {kern_tc}"
    dtype_label = ("int8 IMMA mma.sync" if all(streamed) else "int8 tcgen05.mma kind::i8"
                   if not any(streamed) else "int8 IMMA mma.sync + tcgen05.mma kind::i8")
    line = {
        "metric": METRIC, "value": tops, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": dtype_label + " (u6 offset-binary W x s8 A), int32 accum, fp32 epilogue, fp16 out",
        "data": "synthetic: random-init INT6 weights of the real shapes (fp16 N(0,1) quantized), fp16 N(0,1) activations",
        "config": {"workload": f"{args.model} decoder-layer linears qkv,o,gate,up (W6A6) + down (W6A8), M={M}",
                   "batch": M, "group_size": 128, "scales": "fp16",
                   "parallelism": (f"tp{world}: qkv/gate/up column shards + NCCL all-gather, "
                                   f"o/down row shards (fp32 partials) + NCCL all-reduce")
                                  if world > 1 else "single GPU",
                   "l2": "weights 642 MB/step > 126 MB L2 (no flush needed)",
                   "timing": "CUDA-graph replay of the whole step, CUDA events, max over ranks"},
        "latency_us_per_step": ms_step * 1e3,
        "weight_GBps": sum(lay.weight_bytes for _, lay in layers) * world / (ms_step * 1e-3) / 1e9,
        "hbm_GBps_algorithmic": layer_b / (ms_step * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": kernel_label
                               + f" ({len(shapes)} launches/step, per-launch bytes in DESIGN.md sec. 4)",
                     "peak_source": peak_kind, "gemm_us_per_step": ms_gemm * 1e3},
        "clocks": clk.summary(),
        "e2e": {"value": flops_total / (ms_e2e * 1e-3) / 1e12, "unit": "TOPS",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": ms_e2e, "path": "FlexQLinear.__call__ (public API); per step one H2D of the inputs from pinned host memory and one D2H of all outputs"},
        "gpu_launches": args.steps * len(shapes) * launches_per_fwd,
    }
    if args.bitserial and world == 1:
        line["bitserial"] = time_bitserial(layers, M, shapes)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle.cpu_baseline import CpuBaseline, calibrate_rows

        threads = os.cpu_count() or 1
        rows = calibrate_rows(shapes, M, args.cpu_budget, threads)
        cb = CpuBaseline(shapes, M, rows, threads)
        cb.step()
        reps = 3
        tcpu = sum(cb.step() for _ in range(reps)) / reps
        line["cpu_baseline"] = {"value": cb.flops / tcpu / 1e12, "unit": "TOPS", "cores": threads,
                                "kind": "port", "sample": cb.describe()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
