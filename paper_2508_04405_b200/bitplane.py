"""Two's-complement bit planes (drop-in for bitserial.bitplane).

On the GPU the planes are never materialised on the hot path: ``decompose``
returns a lazy BitPlaneSet holding the integer codes, and ``pack`` fuses the
decomposition into the FLXQ-P packer kernel (csrc/pack.cu, one __ballot_sync
per plane).  ``.planes`` materialises the reference's uint8 [bits, rows, cols]
array on demand (bitplane.py:55-79).
"""
from __future__ import annotations

import numpy as np

from . import _dev
from .errors import InvalidInputError
from .quantize import QuantTensor


def plane_coeff(s: int, bits: int, signed: bool = True) -> int:
    """Weight of plane s: 2^s, or -2^(b-1) for the signed MSB (bitplane.py:23-29)."""
    if not 0 <= s < bits:
        raise IndexError(f"bit index {s} out of range for {bits}-bit planes")
    return -(1 << s) if (signed and s == bits - 1) else (1 << s)


def plane_coeffs(bits: int, signed: bool = True) -> np.ndarray:
    """int64 [bits] vector of plane_coeff (bitplane.py:32-34)."""
    return np.array([plane_coeff(s, bits, signed) for s in range(bits)], dtype=np.int64)


class BitPlaneSet:
    """Bit planes of an integer tensor (bitplane.py:37-52).

    Constructed like the reference (``BitPlaneSet(planes=..., coeffs=..., bits=...,
    signed=...)``) or, by ``decompose``/``bit_planes``, lazily from the integer
    codes on the device: ``planes`` (uint8 [bits, rows, cols]) is then produced on
    the GPU only if accessed, and ``pack`` reads the codes directly.
    """

    __slots__ = ("_planes", "coeffs", "bits", "signed", "_codes", "_numpy")

    def __init__(self, planes=None, coeffs=None, bits=None, signed=True, *, _codes=None,
                 _numpy=None):
        if planes is None and _codes is None:
            raise InvalidInputError("BitPlaneSet needs planes")
        if bits is None:
            bits = int(planes.shape[0])
        object.__setattr__(self, "_planes", planes)
        object.__setattr__(self, "coeffs", np.asarray(coeffs if coeffs is not None
                                                      else plane_coeffs(bits, signed)))
        object.__setattr__(self, "bits", int(bits))
        object.__setattr__(self, "signed", bool(signed))
        object.__setattr__(self, "_codes", _codes)
        if _numpy is None:
            _numpy = not _dev.is_torch(planes)
        object.__setattr__(self, "_numpy", bool(_numpy))

    def __setattr__(self, name, value):
        raise AttributeError("BitPlaneSet is immutable")

    def __repr__(self):
        return f"BitPlaneSet(shape={self.shape}, bits={self.bits}, signed={self.signed})"

    @property
    def shape(self) -> tuple[int, int]:
        if self._codes is not None:
            return tuple(self._codes.shape)
        return tuple(self._planes.shape[1:])

    @property
    def planes(self):
        if self._planes is None:
            t = _dev.torch()
            enc = self._codes.to(t.int32) & ((1 << self.bits) - 1)
            shifts = t.arange(self.bits, device=enc.device, dtype=t.int32)[:, None, None]
            pl = ((enc[None] >> shifts) & 1).to(t.uint8)
            object.__setattr__(self, "_planes", _dev.to_host(pl) if self._numpy else pl)
        return self._planes

    def device_codes(self):
        """Integer bit patterns (int16 CUDA) whose low `bits` bits are the planes."""
        if self._codes is None:
            t = _dev.torch()
            pl = _dev.to_device(self._planes, t.int32)
            shifts = t.arange(self.bits, device=pl.device, dtype=t.int32)[:, None, None]
            enc = (pl << shifts).sum(0).to(t.int16)
            object.__setattr__(self, "_codes", enc)
        return self._codes


def bit_planes(values, bits: int, signed: bool = True) -> BitPlaneSet:
    """Decompose integers into planes (bitplane.py:55-79); range-checked on the GPU."""
    is_t = _dev.is_torch(values)
    if not is_t:
        values = np.asarray(values)
        if not np.issubdtype(values.dtype, np.integer):
            raise InvalidInputError(f"expected integer values, got dtype {values.dtype}")
    else:
        t = _dev.torch()
        if values.dtype.is_floating_point or values.dtype == t.bool:
            raise InvalidInputError(f"expected integer values, got dtype {values.dtype}")
    if values.ndim == 1:
        values = values[None, :]
    t = _dev.torch()
    lo, hi = ((-(1 << (bits - 1)), (1 << (bits - 1)) - 1) if signed else (0, (1 << bits) - 1))
    # range-check in the input's own integer type, before narrowing (65539 must not wrap to 3)
    if (values.numel() if is_t else values.size) and (int(values.min()) < lo or int(values.max()) > hi):
        raise InvalidInputError(
            f"values outside the {'signed' if signed else 'unsigned'} {bits}-bit range [{lo}, {hi}]")
    codes = _dev.to_device(values, t.int16)
    return BitPlaneSet(None, plane_coeffs(bits, signed), bits, signed, _codes=codes,
                       _numpy=not is_t)


def decompose(q: QuantTensor) -> BitPlaneSet:
    """Signed planes of a QuantTensor (bitplane.py:82-84); reuses its device codes."""
    t = _dev.torch()
    codes, _ = q.device_tensors()
    return BitPlaneSet(None, plane_coeffs(q.bits, True), q.bits, True, _codes=codes.to(t.int16),
                       _numpy=not _dev.is_torch(q.values))


def recompose(bp: BitPlaneSet):
    """sum_s coeff_s * plane_s (bitplane.py:87-89), evaluated on the GPU."""
    t = _dev.torch()
    planes = bp.planes if not bp._numpy else _dev.to_device(bp.planes)
    coeffs = t.as_tensor(bp.coeffs, device=planes.device).view(-1, 1, 1)
    out = (planes.to(t.int64) * coeffs).sum(0)
    return _dev.to_host(out) if bp._numpy else out
