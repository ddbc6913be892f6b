"""LLaMA-2 linear-layer shapes used by the benchmark and the parity suite.

N = output features, K = input features (W is [N, K], engine.py:3).  The
activation width follows the FlexQ policy: A8 for down_proj, A6 elsewhere
(quantize.py:172-198, sec. 4.1.2).  BASELINE.json's "8192x28672" /
"28672x8192" are (K, N) in the paper's notation.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class LinearShape:
    name: str   # layer kind (policy key)
    n: int
    k: int
    bits: int = 0  # activation bits; 0 = the FlexQ policy for the layer kind

    @property
    def act_bits(self) -> int:
        if self.bits:
            return self.bits
        return 8 if self.name == "down_proj" else 6


def _decoder(hidden: int, ffn: int, kv: int) -> list[LinearShape]:
    """One decoder layer's linears, q/k/v fused as the reference's ``qkv_proj``
    layer kind (quantize.py:26)."""
    return [
        LinearShape("qkv_proj", hidden + 2 * kv, hidden),
        LinearShape("o_proj", hidden, hidden),
        LinearShape("gate_proj", ffn, hidden),
        LinearShape("up_proj", ffn, hidden),
        LinearShape("down_proj", hidden, ffn),
    ]


MODELS = {
    "llama2-7b": _decoder(4096, 11008, 4096),
    "llama2-13b": _decoder(5120, 13824, 5120),
    "llama2-70b": _decoder(8192, 28672, 1024),  # GQA: 8 kv heads x 128
}


# single-linear workloads of BASELINE.json's config list
WORKLOADS = {
    "config1": [LinearShape("linear", 4096, 4096, bits=8)],  # config 1: W6A8 4096x4096, M=1
}


def policy_kind(name: str) -> str:
    """Map a projection name onto the policy's layer kinds (quantize.py:26)."""
    return {"q_proj": "qkv_proj", "k_proj": "qkv_proj", "v_proj": "qkv_proj"}.get(name, name)


def unfused(shapes: list[LinearShape]) -> list[LinearShape]:
    """Split a fused qkv_proj back into q/k/v (for per-projection parity cases)."""
    out = []
    for s in shapes:
        if s.name == "qkv_proj":
            kv = (s.n - s.k) // 2
            out += [LinearShape("q_proj", s.k, s.k), LinearShape("k_proj", kv, s.k),
                    LinearShape("v_proj", kv, s.k)]
        else:
            out.append(s)
    return out


def gemm_bytes(m: int, n: int, k: int, group_size: int = 128, wbits: int = 6) -> int:
    """Algorithmic HBM bytes of one T6 GEMM launch:
    packed weights + fp16 weight scales + int8 activation codes + fp32 scale and
    int32 correction per (token, group) + fp16 output."""
    g = -(-k // group_size)
    return n * k * wbits // 8 + 2 * n * g + m * k + 8 * m * g + 2 * m * n


def layer_bytes(m: int, n: int, k: int, group_size: int = 128, wbits: int = 6) -> int:
    """Algorithmic bytes of one whole linear call from fp16 x to fp16 y
    (SURVEY.md sec. 8(d)): weights + fp16 scales + fp16 x + fp16 y."""
    g = -(-k // group_size)
    return n * k * wbits // 8 + 2 * n * g + 2 * m * k + 2 * m * n
