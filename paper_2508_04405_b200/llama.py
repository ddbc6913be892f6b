"""LLaMA-2 decode on FlexQ W6A6/W6A8 linears (BASELINE.json config 5).

The reference has no model or decode code (SPEC.md:434 lists it as a non-goal); this is
the end-to-end caller the benchmark config asks for: a random-init LLaMA-2 decoder whose
every linear is a FlexQLinear, with the activation bit width per layer kind taken from a
BitPolicy (the reference's sensitivity-selected default: A8 for down_proj, A6 elsewhere,
quantize.py:172-198), so its tokens/s is the FlexQ path's tokens/s.

Per layer and token, all on the caller's stream (one CUDA graph per decode step):
  fused RMSNorm -> A6 quantize      (flexq_rmsnorm_quantize)
  qkv_proj W6A6 GEMV                 (FlexQLinear.gemm_only: q, k, v fused, N = 3 * hidden)
  RoPE + KV-cache append + attention + o_proj A6 quantize, one kernel (flexq_attn_block)
  o_proj W6A6 GEMV (residual add fused into the epilogue)
  fused RMSNorm -> A6 quantize, gate_up W6A6 GEMV (gate and up fused, N = 2 * ffn)
  fused SiLU(gate) * up -> A8 quantize, down_proj W6A8 GEMV (+ fused residual add)
then the final RMSNorm, an fp16 lm_head and a greedy argmax on the device.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import _dev, _lib
from .errors import ConfigError, InvalidInputError
from .linear import FlexQLinear
from .quantize import DEFAULT_POLICY, BitPolicy, activation_bits


@dataclass(frozen=True)
class LlamaConfig:
    hidden: int
    heads: int
    ffn: int
    layers: int
    vocab: int
    head_dim: int = 128
    eps: float = 1e-5
    rope_theta: float = 10000.0


LLAMA2_7B = LlamaConfig(hidden=4096, heads=32, ffn=11008, layers=32, vocab=32000)
LLAMA2_13B = LlamaConfig(hidden=5120, heads=40, ffn=13824, layers=40, vocab=32000)


class _Layer:
    KINDS = ("qkv_proj", "o_proj", "gate_proj", "down_proj")  # policy key of each linear

    def __init__(self, cfg: LlamaConfig, gen, dev, policy: BitPolicy, group_size: int,
                 keep_float: bool = False):
        t = _dev.torch()
        h, f = cfg.hidden, cfg.ffn
        std = h ** -0.5

        def rnd(n, k, s):
            return (t.randn((n, k), generator=gen, device=dev, dtype=t.float32) * s).half()

        self.norm1 = (1 + 0.05 * t.randn(h, generator=gen, device=dev)).half()
        self.norm2 = (1 + 0.05 * t.randn(h, generator=gen, device=dev)).half()
        ws = [rnd(3 * h, h, std), rnd(h, h, std), rnd(2 * f, h, std), rnd(h, f, f ** -0.5)]
        # gate and up share their input: one GEMV over [gate; up] (policy key gate_proj)
        self.qkv, self.o, self.gate_up, self.down = (
            FlexQLinear(w, 6, activation_bits(kind, policy), group_size, layer_kind=kind)
            for w, kind in zip(ws, self.KINDS))
        self.float_weights = ws if keep_float else None  # for sensitivity calibration

    @property
    def linears(self):
        return (self.qkv, self.o, self.gate_up, self.down)


class FlexQLlamaDecoder:
    """Greedy batched decode of a random-init LLaMA-2 on FlexQ linears."""

    def __init__(self, cfg: LlamaConfig = LLAMA2_7B, batch: int = 1, max_len: int = 512,
                 policy: BitPolicy = DEFAULT_POLICY, group_size: int = 128, seed: int = 0,
                 device="cuda", weights_from: "FlexQLlamaDecoder | None" = None,
                 keep_float_layers: int = 1):
        t = _dev.torch()
        self.cfg, self.batch, self.max_len, self.group_size = cfg, batch, max_len, group_size
        dev = t.device(device)
        self.device = dev
        gen = t.Generator(device=dev)
        gen.manual_seed(seed)
        h, f, H, D = cfg.hidden, cfg.ffn, cfg.heads, cfg.head_dim
        if H * D != h:
            raise ConfigError(f"hidden ({h}) must equal heads * head_dim ({H} * {D})")
        if group_size != D:
            # flexq_attn_block quantizes o_proj's input with head h of a token as group h
            raise ConfigError(f"the decode step fuses o_proj's quantizer into attention and needs "
                              f"group_size == head_dim ({D}), got {group_size}")
        if weights_from is not None:  # share the quantized weights (another batch size)
            src = weights_from
            self.embed, self.layers, self.norm_f, self.lm_head = (src.embed, src.layers, src.norm_f,
                                                                  src.lm_head)
        else:
            self.embed = (t.randn((cfg.vocab, h), generator=gen, device=dev) * 0.5).half()
            self.layers = [_Layer(cfg, gen, dev, policy, group_size, i < keep_float_layers)
                           for i in range(cfg.layers)]
            self.norm_f = t.ones(h, dtype=t.float16, device=dev)
            self.lm_head = (t.randn((cfg.vocab, h), generator=gen, device=dev) * h ** -0.5).half()
        B = batch
        self.k_cache = [t.zeros((B, H, max_len, D), dtype=t.float16, device=dev) for _ in self.layers]
        self.v_cache = [t.zeros((B, H, max_len, D), dtype=t.float16, device=dev) for _ in self.layers]
        self.x = t.zeros((B, h), dtype=t.float16, device=dev)
        self.qkv_out = t.empty((B, 3 * h), dtype=t.float16, device=dev)
        self.q = t.empty((B, H, D), dtype=t.float16, device=dev)
        self.attn = t.empty((B, h), dtype=t.float16, device=dev)
        self.o_out = t.empty((B, h), dtype=t.float16, device=dev)
        self.gu = t.empty((B, 2 * f), dtype=t.float16, device=dev)
        self.d_out = t.empty((B, h), dtype=t.float16, device=dev)
        self.pos = t.zeros(B, dtype=t.int32, device=dev)
        self.tokens = t.zeros(B, dtype=t.int64, device=dev)
        self.flag = t.zeros(1, dtype=t.int32, device=dev)
        for lay in self.layers:  # allocate every linear's per-batch buffers up front
            for lin in (lay.qkv, lay.o, lay.gate_up, lay.down):
                lin.buffers(B)
        self._graph = None
        self.steps_taken = 0  # host mirror of the device positions (all start at 0 on reset)

    @property
    def weight_bytes(self) -> int:
        """Bytes streamed per decode step: packed linears + fp16 lm_head (+ one embedding row)."""
        lin = sum(l.weight_bytes for lay in self.layers for l in (lay.qkv, lay.o, lay.gate_up, lay.down))
        return lin + self.lm_head.numel() * 2

    # -- one token for every sequence of the batch -------------------------------------------
    def _fused_quant(self, kind: str, src, lin: FlexQLinear, cols: int, weight=None, h_out=None):
        L = _lib.lib()
        frag, xs, corr, m_pad = lin._act_views(self.batch)
        if kind == "rmsnorm":
            rc = L.flexq_rmsnorm_quantize(_lib.ptr(src), src.stride(0), _lib.ptr(weight),
                                          self.cfg.eps, self.batch, cols, lin.activation_bits,
                                          self.group_size, frag, xs, corr, m_pad,
                                          _lib.ptr(self.flag), _lib.ptr(h_out), _lib.stream())
        else:
            rc = L.flexq_silu_mul_quantize(_lib.ptr(src), src.stride(0), self.batch, cols,
                                           lin.activation_bits, self.group_size, frag, xs, corr,
                                           m_pad, _lib.ptr(self.flag), _lib.ptr(h_out),
                                           _lib.stream())
        _lib.check(rc)

    def _step(self, record=None):
        """One decode step; ``record`` (dict) collects the fp16 inputs of every linear of
        the first len(record) layers (sensitivity calibration, eager mode only)."""
        t = _dev.torch()
        L = _lib.lib()
        cfg, B = self.cfg, self.batch
        t.index_select(self.embed, 0, self.tokens, out=self.x)
        for li, lay in enumerate(self.layers):
            rec = record.get(li) if record is not None else None
            h1 = t.empty_like(self.x) if rec is not None else None
            self._fused_quant("rmsnorm", self.x, lay.qkv, cfg.hidden, lay.norm1, h1)
            lay.qkv.gemm_only(B, self.qkv_out)
            # RoPE + KV append + attention + o_proj's activation quantizer, one kernel
            frag, xs, corr, m_pad = lay.o._act_views(B)
            _lib.check(L.flexq_attn_block(
                _lib.ptr(self.qkv_out), _lib.ptr(self.pos), _lib.ptr(self.k_cache[li]),
                _lib.ptr(self.v_cache[li]), _lib.ptr(self.attn) if rec is not None else None, B,
                cfg.heads, cfg.head_dim, self.max_len, cfg.rope_theta, lay.o.activation_bits,
                self.group_size, frag, xs, corr, m_pad, _lib.ptr(self.flag), _lib.stream()))
            lay.o.gemm_only(B, self.x, residual=self.x)  # x += o(attn), residual fused
            h2 = t.empty_like(self.x) if rec is not None else None
            self._fused_quant("rmsnorm", self.x, lay.gate_up, cfg.hidden, lay.norm2, h2)
            lay.gate_up.gemm_only(B, self.gu)
            h3 = t.empty((B, cfg.ffn), dtype=t.float16, device=self.device) if rec is not None else None
            self._fused_quant("silu", self.gu, lay.down, cfg.ffn, None, h3)
            lay.down.gemm_only(B, self.x, residual=self.x)  # x += down(h), fused
            if rec is not None:
                for kind, h in zip(_Layer.KINDS, (h1, self.attn.clone(), h2, h3)):
                    rec[kind].append(h)
        xf = self.x.float()
        hN = (xf * t.rsqrt(xf.pow(2).mean(-1, keepdim=True) + cfg.eps)).half() * self.norm_f
        logits = hN @ self.lm_head.t()
        t.argmax(logits, dim=-1, out=self.tokens)
        self.pos.add_(1)

    def record_linear_inputs(self, steps: int = 4, layers: int = 1, max_rows: int = 256):
        """LayerDumps (float weight, recorded fp16 inputs) of the first ``layers`` layers
        over ``steps`` eager decode steps from the current state."""
        from .sensitivity import LayerDump

        record = {li: {k: [] for k in _Layer.KINDS} for li in range(layers)}
        for _ in range(steps):
            self._step(record)
        dumps = []
        for li in range(layers):
            lay = self.layers[li]
            if lay.float_weights is None:
                raise ValueError(f"layer {li} kept no float weights (keep_float_layers)")
            for kind, w in zip(_Layer.KINDS, lay.float_weights):
                acts = _dev.torch().cat(record[li][kind])[:max_rows]
                dumps.append(LayerDump(layer_name=f"model.layers.{li}.{kind}", layer_kind=kind,
                                       weight=w.double().cpu().numpy(),
                                       activations=acts.double().cpu().numpy()))
        return dumps

    def apply_policy(self, policy: BitPolicy) -> None:
        """Set every linear's activation bits from ``policy`` (re-capture needed)."""
        for lay in self.layers:
            for lin, kind in zip(lay.linears, _Layer.KINDS):
                lin.activation_bits = activation_bits(kind, policy)
        self._graph = None

    def policy_table(self) -> dict:
        lay = self.layers[0]
        return {kind: lin.activation_bits for lin, kind in zip(lay.linears, _Layer.KINDS)}

    def reset(self, tokens=None):
        t = _dev.torch()
        self.pos.zero_()
        self.steps_taken = 0
        if tokens is None:
            self.tokens.copy_(t.arange(self.batch, device=self.device) % self.cfg.vocab)
        else:
            self.tokens.copy_(tokens)

    def capture(self):
        """Capture one decode step in a CUDA graph (positions and tokens live on the device)."""
        t = _dev.torch()
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        pos0, tok0 = self.pos.clone(), self.tokens.clone()
        with t.cuda.stream(s):
            self._step()  # warm-up outside capture
        t.cuda.current_stream().wait_stream(s)
        self.pos.copy_(pos0)
        self.tokens.copy_(tok0)
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g):
            self._step()
        self.pos.copy_(pos0)
        self.tokens.copy_(tok0)
        self._graph = g

    def step(self):
        """Decode one token per sequence (graph replay when captured)."""
        if self.steps_taken >= self.max_len:
            raise InvalidInputError(f"KV cache full: {self.max_len} positions decoded "
                                    f"(max_len={self.max_len}); reset() or use a longer cache")
        self.steps_taken += 1
        if self._graph is not None:
            self._graph.replay()
        else:
            self._step()
        return self.tokens

    def check_errors(self) -> None:
        bits = int(self.flag.item())
        self.flag.zero_()
        if bits & _lib.FLAG_KV_OVERFLOW:
            raise InvalidInputError("KV cache overflow: a position reached max_len")
        if bits:
            raise InvalidInputError("non-finite activations in the decode step")
