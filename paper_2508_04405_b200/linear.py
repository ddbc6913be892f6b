"""FlexQLinear: the production W6A6/W6A8 linear layer on the B200.

The reference's quantized_linear (engine.py:487-513) re-quantizes and
re-packs the weights on every call.  Here the offline half (INT6 weight
quantization + T6 packing) runs once at construction, and each forward is the
online half only: fused per-token/per-group activation quantizer -> T6
tensor-core GEMV/GEMM with the fused fp32 group-dequant epilogue -> fp16 out.
Both kernels run back to back on the caller's stream through one C-ABI call
(flexq_linear_forward); buffers are preallocated per batch size so the call
never allocates and can be captured in a CUDA graph.
"""
from __future__ import annotations

from . import _dev, _lib
from .errors import InvalidInputError, ShapeError
from .packing import PackedTensor
from .quantize import DEFAULT_GROUP_SIZE, DEFAULT_POLICY, BitPolicy, QuantTensor, quantize
from .quantize import activation_bits as policy_bits


class FlexQLinear:
    """y = dequant(Q6(W)) applied to Q_q(x), fp16 in / fp16 out.

    weight: [N, K] float (numpy or torch).  ``activation_bits`` may be given
    directly or resolved from ``layer_kind`` under ``policy`` (A8 for down_proj
    in the default FlexQ policy, quantize.py:172-198).  ``fp16_scales`` stores
    the weight scales in fp16 (the kernel's 2 bytes/group; bit-exact with the
    reference's fp16-scale mode).
    """

    def __init__(self, weight, weight_bits: int = 6, activation_bits: int | None = None,
                 group_size: int = DEFAULT_GROUP_SIZE, fp16_scales: bool = True,
                 layer_kind: str | None = None, policy: BitPolicy = DEFAULT_POLICY):
        if weight_bits > 6:
            raise InvalidInputError(f"FlexQLinear packs at most 6-bit weights, got {weight_bits}")
        if activation_bits is None:
            activation_bits = policy_bits(layer_kind or "generic", policy)
        self.qweight = quantize(weight if _dev.is_torch(weight) else _dev.to_device(weight),
                                weight_bits, group_size, fp16_scales=fp16_scales)
        self._setup(self.qweight, activation_bits, fp16_scales, layer_kind)

    def _setup(self, qweight, activation_bits: int, fp16_scales: bool, layer_kind) -> None:
        """Pack the quantized weight into the T6 stream (the offline half)."""
        t = _dev.torch()
        self.qweight = qweight
        self.weight_bits = int(qweight.bits)
        self.activation_bits = int(activation_bits)
        self.group_size = int(qweight.group_size)
        self.fp16_scales = bool(fp16_scales)
        self.layer_kind = layer_kind
        codes, scales = qweight.device_tensors()
        self.n, self.k = codes.shape
        from .engine import t6_pack_weights

        self.t6, self.wscale = t6_pack_weights(codes, scales, self.k, self.group_size,
                                               scale_f16=self.fp16_scales)
        self.device = codes.device
        self._dev_index = codes.device.index if codes.device.index is not None else 0
        self._bufs: dict[int, tuple] = {}
        self._f16_ready: set[int] = set()  # batches whose act buffer holds the fp16 operand
        self.flag = t.zeros(1, dtype=t.int32, device=self.device)

    # -- construction from reference artefacts ------------------
    @classmethod
    def from_quant(cls, q, activation_bits: int | None = None, layer_kind: str | None = None,
                   policy: BitPolicy = DEFAULT_POLICY, fp16_scales: bool | None = None):
        """Serve an already-quantized weight (a QuantTensor, e.g. ``fileio.read_quant`` of a
        container written by the reference's ``bitserial quantize``) without re-quantizing.

        The codes go straight into the T6 packer.  ``fp16_scales`` defaults to True exactly
        when every scale is an fp16 value (then the 2-byte scale stream loses nothing), else
        the kernel streams fp32 scales."""
        if q.bits > 6:
            raise InvalidInputError(f"FlexQLinear packs at most 6-bit weights, got {q.bits}")
        if q.group_axis != 1:
            raise InvalidInputError("weight groups must run along K (group_axis 1)")
        _, scales = q.device_tensors()
        if fp16_scales is None:
            t = _dev.torch()
            fp16_scales = bool(t.equal(scales.to(t.float16).to(t.float64), scales))
        if activation_bits is None:
            activation_bits = policy_bits(layer_kind or "generic", policy)
        self = cls.__new__(cls)
        self._setup(q, activation_bits, fp16_scales, layer_kind)
        return self

    @classmethod
    def from_packed(cls, p, scales, group_size: int = DEFAULT_GROUP_SIZE, **kw):
        """Serve FLXQ-P packed weight planes (a PackedTensor, e.g. ``fileio.read_packed`` of
        ``bitserial pack`` output) with their per-(row, group) scales [N, n_groups].

        The planes are unpacked on the GPU (csrc/pack.cu) and re-laid into the T6 stream;
        no host pass over the weights."""
        from .packing import unpack

        if not p.signed:
            raise InvalidInputError("weight planes must be signed (two's complement)")
        if p.bits > 6:
            raise InvalidInputError(f"FlexQLinear packs at most 6-bit weights, got {p.bits}")
        t = _dev.torch()
        codes = unpack(p, p.config).device_codes().to(t.int8)
        sc = _dev.to_device(scales, t.float64)
        q = QuantTensor(values=codes, scales=sc, bits=p.bits, group_size=group_size,
                        _device=(codes, sc))
        return cls.from_quant(q, **kw)

    @classmethod
    def load(cls, path: str, scales=None, group_size: int = DEFAULT_GROUP_SIZE, **kw):
        """Build a layer from an FLXQ container: a quant tensor (kind 1) is served as is, a
        packed tensor (kind 2) needs ``scales`` (an array, or the path of a quant or float
        container holding them), a float tensor (kind 0) is quantized on the GPU."""
        from . import fileio

        obj = fileio.read(path)
        if isinstance(obj, QuantTensor):
            return cls.from_quant(obj, **kw)
        if isinstance(obj, PackedTensor):
            if scales is None:
                raise InvalidInputError(f"{path}: packed weights need their scales")
            if isinstance(scales, str):
                s = fileio.read(scales)
                scales, group_size = ((s.scales, s.group_size) if isinstance(s, QuantTensor)
                                      else (s, group_size))
            return cls.from_packed(obj, scales, group_size, **kw)
        return cls(obj, group_size=group_size, **kw)

    # -- buffers ------------------------------------------------------------------------
    def buffers(self, m: int, stream: int | None = None):
        """(act buffer, workspace) for batch m on ``stream`` (default: the current stream).

        Each stream gets its own pair: the quantizer writes the act buffer and the GEMM's
        split fixups count in the workspace, so two forwards in flight on different streams
        must not share them.  The workspace counters are zeroed once here and every launch
        leaves them zeroed (graph-safe).  A CUDA-graph capture (its own side stream) reuses the
        buffers of a stream that already ran this batch eagerly, so the graph's replays and
        eager forwards on that stream must be stream-ordered."""
        t = _dev.torch()
        key = (m, _lib.stream(self._dev_index) if stream is None else stream)
        if key not in self._bufs:
            if t.cuda.is_current_stream_capturing():
                for (mm, _), bufs in self._bufs.items():
                    if mm == m:
                        return bufs
            L = _lib.lib()
            act = t.empty(L.flexq_act_buf_bytes(m, self.k, self.group_size), dtype=t.uint8,
                          device=self.device)
            ws = t.zeros(max(L.flexq_gemm_workspace_bytes(m, self.n, self.k, self.group_size, 0), 16),
                         dtype=t.uint8, device=self.device)
            self._bufs[key] = (act, ws)
        return self._bufs[key]

    @property
    def weight_bytes(self) -> int:
        """Bytes of packed weights + scales streamed per call."""
        return self.t6.numel() * 4 + self.wscale.numel() * self.wscale.element_size()

    # -- forward --------------------------------------------------------------------------
    def _check_out(self, what: str, buf, m: int, dtype) -> None:
        if not (_dev.is_torch(buf) and buf.is_cuda and buf.device == self.device):
            raise InvalidInputError(f"{what} must be a CUDA tensor on {self.device}")
        if buf.dtype != dtype:
            raise InvalidInputError(f"{what} must be {dtype}, got {buf.dtype}")
        if tuple(buf.shape) != (m, self.n) or not buf.is_contiguous():
            raise ShapeError(f"{what} must be a contiguous [{m}, {self.n}] tensor, got "
                             f"{tuple(buf.shape)}{'' if buf.is_contiguous() else ' (strided)'}")

    def forward(self, x, out=None, residual=None, out_dtype=None):
        """x: fp16 CUDA [M, K] -> [M, N] on the layer's device (no host sync).

        ``out_dtype`` is torch.float16 (default) or torch.float32 (an unrounded fp32 y: the
        partial a row shard sums across ranks).  ``residual`` ([M, N] of the output dtype,
        may be ``out`` itself) is added in the GEMM epilogue."""
        t = _dev.torch()
        if not _dev.is_torch(x):
            raise InvalidInputError("x must be a torch tensor (use quantized_linear for arrays)")
        if x.dim() != 2 or x.shape[1] != self.k:
            raise ShapeError(f"activation shape {tuple(x.shape)} does not match K={self.k}")
        if not x.is_cuda or x.device != self.device:
            raise InvalidInputError(f"x must be a CUDA tensor on {self.device}, got {x.device}")
        if out_dtype is None:
            out_dtype = out.dtype if out is not None else t.float16
        if out_dtype not in (t.float16, t.float32):
            raise InvalidInputError(f"out_dtype must be float16 or float32, got {out_dtype}")
        if x.dtype != t.float16:
            x = x.to(t.float16)
        x = x.contiguous()
        m = x.shape[0]
        if m < 1:
            raise ShapeError("activation batch must be at least one row")
        if out is None:
            out = t.empty((m, self.n), dtype=out_dtype, device=self.device)
        else:
            self._check_out("out", out, m, out_dtype)
        if residual is not None:
            self._check_out("residual", residual, m, out_dtype)
        st = _lib.stream(self._dev_index)
        act, ws = self.buffers(m, st)
        L = _lib.lib()
        if L.flexq_linear_kernel(m, self.n, self.k, self.group_size,
                                 int(self.fp16_scales)) == _lib.KERNEL_TC16:
            self._f16_ready.add(m)
        else:  # the route can change (flexq_set_tc16_route): gemm_only follows the last forward
            self._f16_ready.discard(m)
        _lib.check(L.flexq_linear_forward_ex(
            self.t6.data_ptr(), self.wscale.data_ptr(), int(self.fp16_scales), self.activation_bits,
            x.data_ptr(), m, self.n, self.k, self.group_size, out.data_ptr(),
            _lib.OUT_F32 if out_dtype == t.float32 else _lib.OUT_F16, act.data_ptr(),
            ws.data_ptr(), self.flag.data_ptr(), _lib.ptr(residual), st))
        return out

    __call__ = forward

    def _act_views(self, m: int):
        """(act_frag, xs, corr) pointers inside the act buffer (mirrors flexq_linear_forward)."""
        L = _lib.lib()
        act, _ = self.buffers(m)
        m_pad = L.flexq_act_m_pad(m)
        ng = -(-self.k // self.group_size)
        frag = -(-L.flexq_act_frag_bytes(m_pad, self.k, self.group_size) // 256) * 256
        vec = -(-(ng * m_pad * 4) // 256) * 256
        base = act.data_ptr()
        return base, base + frag, base + frag + vec, m_pad

    def gemm_only(self, m: int, out, residual=None):
        """Re-run only the T6 GEMM on the activations quantized by the last forward(m).

        Used by bench.py to time the dominant kernel alone (roofline)."""
        t = _dev.torch()
        self._check_out("out", out, m, out.dtype if out.dtype in (t.float16, t.float32) else t.float16)
        if residual is not None:
            self._check_out("residual", residual, m, out.dtype)
        L = _lib.lib()
        act, ws = self.buffers(m)
        if m in self._f16_ready:
            # batched route: the fp16 operand the last forward(m) wrote (scales folded in);
            # operands written by other producers (the decode harness's fused quantizers) are
            # the INT8 layout and take the integer kernels below
            op = L.flexq_act_f16_operand(act.data_ptr(), m, self.k, self.group_size)
            _lib.check(L.flexq_gemm_tc16(
                _lib.ptr(self.t6), _lib.ptr(self.wscale), op, m, self.n, self.k, _lib.ptr(out),
                _lib.OUT_F32 if out.dtype == t.float32 else _lib.OUT_F16, _lib.ptr(ws),
                _lib.ptr(residual), _lib.stream(self._dev_index)))
            return out
        frag, xs, corr, m_pad = self._act_views(m)
        _lib.check(_lib.lib().flexq_gemm_t6_ex(
            _lib.ptr(self.t6), _lib.ptr(self.wscale), int(self.fp16_scales), frag, xs, corr, m,
            m_pad, self.n, self.k, self.group_size, None, _lib.ptr(out),
            _lib.OUT_F32 if out.dtype == t.float32 else _lib.OUT_F16,
            _lib.ptr(ws), 0, _lib.ptr(residual), _lib.stream(self._dev_index)))
        return out

    def check_errors(self) -> None:
        """Raise if any forward since the last check saw non-finite input (host sync)."""
        bits = int(self.flag.item())
        self.flag.zero_()
        if bits & _lib.FLAG_NONFINITE:
            raise InvalidInputError("input contains non-finite values")
        if bits & _lib.FLAG_NONPOS_SCALE:
            raise InvalidInputError("all scales must be strictly positive")
