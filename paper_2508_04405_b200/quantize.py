"""Symmetric group quantization on the GPU (drop-in for bitserial.quantize).

Public names, signatures, error classes and messages follow the reference's
quantize.py; the arithmetic runs in libflexq_sm100a (csrc/quantize.cu), which
reproduces quantize.py:118-148 bit for bit (float64 divide, half-away
rounding, optional fp16 scale rounding).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from types import MappingProxyType
from typing import Any, Mapping

import numpy as np

from . import _dev, _lib
from .errors import InvalidInputError, PolicyMissError

DEFAULT_GROUP_SIZE = 128

LAYER_KINDS = ("qkv_proj", "o_proj", "gate_proj", "up_proj", "down_proj", "generic")


def qmax(bits: int) -> int:
    """2^(b-1) - 1, the symmetric range limit (quantize.py:34-36)."""
    return (1 << (bits - 1)) - 1


def _n_groups(cols: int, group_size: int) -> int:
    return -(-cols // group_size)


@dataclass(frozen=True)
class QuantTensor:
    """Group-quantized tensor (quantize.py:39-83).

    values: int8 [rows, cols] in [-qmax, qmax]; scales: float64 [rows, G] > 0.
    Either numpy arrays or torch CUDA tensors; a device copy is cached so the
    GPU packers never re-upload.
    """

    values: Any
    scales: Any
    bits: int
    group_size: int
    group_axis: int = 1
    _device: Any = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        vshape = tuple(self.values.shape)
        if len(vshape) != 2:
            raise InvalidInputError(f"values must be 2-D, got shape {vshape}")
        if self.group_axis != 1:
            raise InvalidInputError("groups must run along axis 1 (K)")
        if not 2 <= self.bits <= 8:
            raise InvalidInputError(f"bits must be in 2..8, got {self.bits}")
        if self.group_size < 1:
            raise InvalidInputError(f"group_size must be >= 1, got {self.group_size}")
        rows, cols = vshape
        expected = (rows, _n_groups(cols, self.group_size))
        if tuple(self.scales.shape) != expected:
            raise InvalidInputError(f"scales shape {tuple(self.scales.shape)} != expected {expected}")
        lim = qmax(self.bits)
        if _dev.is_torch(self.values):
            ok_scales = bool((self.scales > 0).all()) if self.scales.numel() else True
            ok_vals = (bool((self.values.to(_dev.torch().int64).abs() <= lim).all())
                       if self.values.numel() else True)  # widen first: abs(int8 -128) wraps
        else:
            ok_scales = bool(np.all(np.asarray(self.scales) > 0))
            ok_vals = not np.any(np.abs(np.asarray(self.values).astype(np.int64)) > lim)
        if not ok_scales:
            raise InvalidInputError("all scales must be strictly positive")
        if not ok_vals:
            raise InvalidInputError(f"values exceed symmetric {self.bits}-bit range +/-{lim}")

    @property
    def shape(self) -> tuple[int, int]:
        return tuple(self.values.shape)

    @property
    def n_groups(self) -> int:
        return int(self.scales.shape[1])

    def device_tensors(self):
        """(values int8, scales float64) as torch CUDA tensors (cached)."""
        if self._device is None:
            t = _dev.torch()
            object.__setattr__(self, "_device", (_dev.to_device(self.values, t.int8),
                                                 _dev.to_device(self.scales, t.float64)))
        return self._device


def _check_flag(flag) -> None:
    bits = int(flag.item())
    if bits & _lib.FLAG_NONFINITE:
        raise InvalidInputError("input contains non-finite values")
    if bits & _lib.FLAG_NONPOS_SCALE:
        raise InvalidInputError("all scales must be strictly positive")


def quantize_device(x, bits: int, group_size: int, fp16_scales: bool):
    """Device-level quantize: torch CUDA float tensor -> (codes int8, scales f64)."""
    t = _dev.torch()
    rows, cols = x.shape
    codes = t.empty((rows, cols), dtype=t.int8, device=x.device)
    scales = t.empty((rows, _n_groups(cols, group_size)), dtype=t.float64, device=x.device)
    flag = t.zeros(1, dtype=t.int32, device=x.device)
    L = _lib.lib()
    _lib.check(L.flexq_quantize(_lib.ptr(x), _dev.float_dtype_code(x), rows, cols, bits, group_size,
                                int(bool(fp16_scales)), _lib.ptr(codes), _lib.ptr(scales),
                                None, None, None, 0, _lib.ptr(flag), _lib.stream()))
    _check_flag(flag)
    return codes, scales


def quantize(data, bits: int, group_size: int = DEFAULT_GROUP_SIZE,
             fp16_scales: bool = False) -> QuantTensor:
    """Symmetric group quantization of a 2-D float tensor (quantize.py:118-148).

    value = clamp(round_half_away(x / s), -qmax, qmax) per (row, K-group) with
    s = max|group| / qmax (1.0 for an all-zero group); ``fp16_scales`` rounds s
    to fp16 first.  Runs on the GPU; numpy in -> numpy out.
    """
    t = _dev.torch()
    is_t = _dev.is_torch(data)
    if not is_t:
        data = np.asarray(data)
        if data.dtype.kind not in "f":
            data = data.astype(np.float64)
    if len(tuple(data.shape)) != 2:
        raise InvalidInputError(f"expected a 2-D tensor, got shape {tuple(data.shape)}")
    if not 2 <= bits <= 8:
        raise InvalidInputError(f"bits must be in 2..8, got {bits}")
    if group_size < 1:
        raise InvalidInputError(f"group_size must be >= 1, got {group_size}")
    rows, cols = data.shape
    if rows == 0 or cols == 0:  # no arithmetic to do; keep the reference's empty shapes
        vals = np.zeros((rows, cols), np.int8)
        sc = np.ones((rows, _n_groups(cols, group_size)), np.float64)
        if is_t:
            vals, sc = t.from_numpy(vals).to(data.device), t.from_numpy(sc).to(data.device)
        return QuantTensor(values=vals, scales=sc, bits=bits, group_size=group_size)
    x = _dev.to_device(data)
    if x.dtype not in (t.float16, t.bfloat16, t.float32, t.float64):
        x = x.to(t.float64)
    codes, scales = quantize_device(x, bits, group_size, fp16_scales)
    qt = QuantTensor(values=_dev.like_input(codes, data), scales=_dev.like_input(scales, data),
                     bits=bits, group_size=group_size, _device=(codes, scales))
    return qt


def dequantize(q: QuantTensor):
    """values * group scale, elementwise (quantize.py:151-154); computed on the GPU."""
    t = _dev.torch()
    codes, scales = q.device_tensors()
    cols = codes.shape[1]
    per = scales.repeat_interleave(q.group_size, dim=1)[:, :cols]
    out = codes.to(t.float64) * per
    return _dev.like_input(out, q.values)


def compute_group_scale(group, bits: int) -> float:
    """max|group| / qmax, 1.0 for an all-zero group (quantize.py:86-96), on the GPU."""
    arr = group if _dev.is_torch(group) else np.asarray(group, dtype=np.float64)
    if arr.numel() == 0 if _dev.is_torch(arr) else arr.size == 0:
        raise InvalidInputError("group must be non-empty")
    if not 2 <= bits <= 8:
        raise InvalidInputError(f"bits must be in 2..8, got {bits}")
    x = _dev.to_device(arr).reshape(1, -1)
    t = _dev.torch()
    if x.dtype not in (t.float16, t.bfloat16, t.float32, t.float64):
        x = x.to(t.float64)
    try:
        _, scales = quantize_device(x, bits, x.shape[1], False)
    except InvalidInputError as e:
        if "non-finite" in str(e):
            raise InvalidInputError("group contains non-finite values") from None
        raise
    return float(scales[0, 0].item())


# ---- per-layer bit policy (quantize.py:157-198): configuration, no arithmetic ----

@dataclass(frozen=True)
class BitPolicy:
    """Per-layer-kind activation bits; weights are uniform (quantize.py:157-169)."""

    weight_bits: int = 6
    activation_bits_by_layer: Mapping[str, int] = field(
        default_factory=lambda: MappingProxyType({}))

    def __post_init__(self):
        for kind, b in self.activation_bits_by_layer.items():
            if b not in (6, 8):
                raise InvalidInputError(f"policy maps {kind!r} to {b}, expected 6 or 8")


def uniform_policy(bits: int = 6) -> BitPolicy:
    """Same activation width for every kind, e.g. non-GLU models (quantize.py:179-184)."""
    return BitPolicy(weight_bits=6,
                     activation_bits_by_layer=MappingProxyType({k: bits for k in LAYER_KINDS}))


def _flexq_default() -> BitPolicy:
    table = dict.fromkeys(LAYER_KINDS, 6)
    table["down_proj"] = 8  # PAPER.md sec. 4.1.2: A8 for the sensitive down_proj
    return BitPolicy(weight_bits=6, activation_bits_by_layer=MappingProxyType(table))


DEFAULT_POLICY = _flexq_default()


def activation_bits(layer_kind: str, policy: BitPolicy = DEFAULT_POLICY) -> int:
    """Activation width for a layer kind (quantize.py:190-198)."""
    table = policy.activation_bits_by_layer
    if layer_kind not in table:
        raise PolicyMissError(f"no policy entry for layer kind {layer_kind!r}; "
                              f"known kinds: {sorted(table)}")
    return table[layer_kind]
