"""Tensor-parallel sharding of W6Ax linear layers across the GPUs of one node.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  The
reference has no distributed code; this follows the
north-star plan:

* column (N) sharding -- rank r owns output rows [r*N/P, (r+1)*N/P).  X is
  replicated, every rank quantizes it identically, computes its y shard, and
  one all-gather assembles y.  Every output element is computed by exactly one
  rank, so the gather is exact.  Used for qkv/gate/up.
* row (K) sharding -- rank r owns the K range [r*K/P, (r+1)*K/P), which must
  fall on scale-group boundaries so INT32 group partials stay exact.  Each
  rank quantizes its slice of x (groups are local), computes an fp32 partial
  y over its K range, and an all-reduce (sum) combines them.  Partials per
  group are exact; only the float sum order differs from P = 1 (within the
  fp16 tolerance).  Used for o_proj and down_proj, which consume the column-
  sharded outputs of qkv/attention and gate/up (the Megatron pairing).

The collective sits only at the shard boundary.  ``local`` is the per-rank
compute (FlexQLinear on the GPU; row shards ask it for an unrounded fp32 y, so
nothing is rounded to fp16 before the sum); tests also inject the CPU oracle to
exercise the partitioning and collectives with gloo on CPU.  Over gloo, CUDA
results are staged through host memory for the collective (NCCL needs none).
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError, ShapeError


@dataclass(frozen=True)
class ShardSpec:
    mode: str      # "column" or "row"
    world: int
    rank: int
    n: int
    k: int
    group_size: int

    def __post_init__(self):
        if self.mode not in ("column", "row"):
            raise ConfigError(f"shard mode must be 'column' or 'row', got {self.mode!r}")
        if not 0 <= self.rank < self.world:
            raise ConfigError(f"rank {self.rank} outside world of {self.world}")
        if self.mode == "column" and self.n % self.world:
            raise ShapeError(f"N={self.n} is not divisible by {self.world} column shards")
        if self.mode == "row":
            if self.k % self.world:
                raise ShapeError(f"K={self.k} is not divisible by {self.world} row shards")
            if (self.k // self.world) % self.group_size:
                raise ConfigError(
                    f"row shard K/{self.world}={self.k // self.world} must hold whole scale "
                    f"groups (group_size={self.group_size}) so INT32 group partials stay exact")

    @property
    def rows(self) -> slice:
        if self.mode == "row":
            return slice(0, self.n)
        step = self.n // self.world
        return slice(self.rank * step, (self.rank + 1) * step)

    @property
    def cols(self) -> slice:
        if self.mode == "column":
            return slice(0, self.k)
        step = self.k // self.world
        return slice(self.rank * step, (self.rank + 1) * step)


def shard_weight(weight, spec: ShardSpec):
    """This rank's block of the [N, K] weight."""
    if tuple(weight.shape) != (spec.n, spec.k):
        raise ShapeError(f"weight shape {tuple(weight.shape)} != {(spec.n, spec.k)}")
    return weight[spec.rows, spec.cols]


class ShardedLinear:
    """A W6Ax linear layer split over a process group.

    local(x_local) -> y_local must return this rank's [M, N_local] (column) or
    fp32 partial [M, N] (row) result.  By default it is a FlexQLinear built from
    the rank's weight shard.
    """

    def __init__(self, weight, spec: ShardSpec, activation_bits: int = 6, group=None,
                 local=None, fp16_scales: bool = True):
        self.spec = spec
        self.group = group
        if local is None:
            from .linear import FlexQLinear

            w = shard_weight(weight, spec)
            lin = FlexQLinear(w.contiguous() if hasattr(w, "contiguous") else w, 6,
                              activation_bits, spec.group_size, fp16_scales=fp16_scales)
            import torch

            # row shards: fp32 partial y straight from the GEMM epilogue (no fp16 rounding
            # before the cross-rank sum); column shards: the final fp16 y
            out_dtype = torch.float32 if spec.mode == "row" else torch.float16
            local = (lambda x, _lin=lin, _dt=out_dtype: _lin(x, out_dtype=_dt))
        self.local = local

    def __call__(self, x):
        import torch
        import torch.distributed as dist

        s = self.spec
        x_loc = x[:, s.cols].contiguous() if s.mode == "row" else x
        y = self.local(x_loc)
        if s.world == 1:
            return y
        dev = y.device
        stage = y.is_cuda and dist.get_backend(self.group) == "gloo"
        if stage:
            y = y.cpu()
        if s.mode == "column":
            m, n_loc = y.shape
            buf = torch.empty((s.world * m, n_loc), dtype=y.dtype, device=y.device)
            dist.all_gather_into_tensor(buf, y.contiguous(), group=self.group)
            y = buf.view(s.world, m, n_loc).permute(1, 0, 2).reshape(m, s.world * n_loc)
        else:
            y = y.contiguous()
            dist.all_reduce(y, op=dist.ReduceOp.SUM, group=self.group)
        return y.to(dev) if stage else y
