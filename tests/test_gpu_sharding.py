"""ShardedLinear with its default per-rank compute (FlexQLinear on the GPU), world size 2.

Both ranks run on cuda:0 (gpurun gives one GPU) and talk over gloo, host-staged by
ShardedLinear.  Column shards + all-gather and row shards + all-reduce of fp32 partials
(the reference's disjoint output tiles, engine.py:442-483, and
group-independent integer partials, engine.py:277-286) are checked against the float64
oracle (int_matmul_reference, engine.py:337-365) within the fp16 tolerance, and the
gathered column result against each rank's shard computed alone (bit-identical).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import c_oracle  # noqa: E402

FP16_TOL = 1e-3
CASES = [(3, 1024, 2048, 6), (8, 768, 4096, 8), (40, 512, 2048, 6)]  # (M, N, K, q)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(m, n, k, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((n, k)).astype(np.float16)
    x = rng.standard_normal((m, k)).astype(np.float16)
    return w, x


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_04405_b200 import FlexQLinear
    from paper_2508_04405_b200.sharding import ShardedLinear, ShardSpec, shard_weight

    res = {}
    for ci, (m, n, k, q) in enumerate(CASES):
        w, x = _inputs(m, n, k, ci)
        xd = torch.from_numpy(x).cuda()
        for mode in ("column", "row"):
            spec = ShardSpec(mode, world, rank, n, k, 128)
            y = ShardedLinear(w, spec, activation_bits=q)(xd)
            alone = None
            if mode == "column":  # this rank's shard through a plain FlexQLinear
                alone = FlexQLinear(np.ascontiguousarray(shard_weight(w, spec)),
                                    activation_bits=q)(xd).cpu().numpy()
            res[(ci, mode, rank)] = (y.cpu().numpy(), str(y.dtype), str(y.device), alone)
    out_q.put(res)
    dist.barrier()
    dist.destroy_process_group()


_RESULTS = {}


def _results(world=2):
    if not _RESULTS:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
        for p in procs:
            p.start()
        for _ in range(world):
            _RESULTS.update(q.get(timeout=600))
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
    return _RESULTS


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_sharded_linear_default_compute(ci):
    m, n, k, q = CASES[ci]
    w, x = _inputs(m, n, k, ci)
    wc, ws = c_oracle.quantize(w, 6, 128, True)
    xc, xs = c_oracle.quantize(x, q, 128, True)
    y_ref, _ = c_oracle.int_matmul(wc, xc, ws, xs, 128)
    res = _results()
    scale = np.abs(y_ref).max()
    for rank in range(2):
        y, dtype, dev, _ = res[(ci, "column", rank)]
        assert dtype == "torch.float16" and dev.startswith("cuda")
        assert np.abs(y.astype(np.float64) - y_ref).max() <= FP16_TOL * scale
        # the gather assembles the ranks' shards unchanged
        for r in range(2):
            shard = res[(ci, "column", r)][3]
            assert np.array_equal(y[:, r * n // 2:(r + 1) * n // 2], shard)
        y, dtype, dev, _ = res[(ci, "row", rank)]
        # fp32 partials summed across ranks, never rounded to fp16 on the way
        assert dtype == "torch.float32" and dev.startswith("cuda")
        assert np.abs(y.astype(np.float64) - y_ref).max() <= FP16_TOL * scale
    assert np.array_equal(res[(ci, "row", 0)][0], res[(ci, "row", 1)][0])
