"""Multi-process (gloo, world_size 2, CPU) test of the tensor-parallel host logic:
column shards + all-gather and row shards + all-reduce around the per-rank
compute.  The per-rank compute here is the CPU oracle (injected), so the test
checks partitioning and collectives; the GPU kernels are covered by -m gpu."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import c_oracle
from paper_2508_04405_b200.errors import ConfigError, ShapeError
from paper_2508_04405_b200.sharding import ShardedLinear, ShardSpec, shard_weight

M, N, K, GS = 3, 96, 512, 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def oracle_linear(w, q, gs):
    """Per-rank stand-in: oracle quantize both operands + exact int GEMM (f64)."""
    wc, ws = c_oracle.quantize(w, 6, gs, True)

    def f(x):
        xc, xs = c_oracle.quantize(x.numpy(), q, gs, True)
        y, _ = c_oracle.int_matmul(wc, xc, ws, xs, gs, threads=1)
        return torch.from_numpy(y)
    return f


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    w = rng.standard_normal((N, K)).astype(np.float16)
    x = torch.from_numpy(rng.standard_normal((M, K)).astype(np.float16))
    res = {}
    for mode in ("column", "row"):
        spec = ShardSpec(mode, world, rank, N, K, GS)
        lin = ShardedLinear(w, spec, local=oracle_linear(shard_weight(w, spec), 8, GS))
        res[mode] = lin(x).numpy()
    if rank == 0:
        out_q.put(res)
    dist.barrier()
    dist.destroy_process_group()


_RESULTS = {}


def _run(mode, world=2):
    if not _RESULTS:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
        for p in procs:
            p.start()
        _RESULTS.update(q.get(timeout=300))
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
    return _RESULTS[mode]


def _reference_y():
    rng = np.random.default_rng(0)
    w = rng.standard_normal((N, K)).astype(np.float16)
    x = rng.standard_normal((M, K)).astype(np.float16)
    return oracle_linear(w, 8, GS)(torch.from_numpy(x)).numpy()


def test_column_shards_allgather_bit_identical():
    y = _run("column")
    assert np.array_equal(y, _reference_y())


def test_row_shards_allreduce_matches():
    y = _run("row")
    ref = _reference_y()
    # exact integer group partials; only the float64 sum order across ranks differs
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_shard_spec_validation():
    with pytest.raises(ShapeError):
        ShardSpec("column", 3, 0, 100, 256, 128)
    with pytest.raises(ConfigError):
        ShardSpec("row", 2, 0, 64, 384, 128)  # 192-wide shards split a 128-group
    with pytest.raises(ConfigError):
        ShardSpec("diag", 2, 0, 64, 256, 128)
    s = ShardSpec("row", 4, 3, 8192, 28672, 128)
    assert (s.cols.start, s.cols.stop) == (21504, 28672)
    s = ShardSpec("column", 8, 7, 28672, 8192, 128)
    assert (s.rows.start, s.rows.stop) == (25088, 28672)
