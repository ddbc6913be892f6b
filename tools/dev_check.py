"""Quick GPU self-check used during development (prints, does not assert)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2508_04405_b200 as fq
from paper_2508_04405_b200 import _lib
from oracle import c_oracle, np_oracle

g = dict(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden.npz")))
names = lambda p: [str(s) for s in g[f"{p}/names"]]
bad = 0
for n in names("q"):
    x = g[f"q/{n}/x"]; bits, gs, f16 = (int(v) for v in g[f"q/{n}/meta"])
    q = fq.quantize(x, bits, gs, bool(f16))
    ok = np.array_equal(q.values, g[f"q/{n}/values"]) and np.array_equal(q.scales, g[f"q/{n}/scales"])
    bad += not ok; print("quant", n, ok)
for n in names("p"):
    vals = g[f"p/{n}/values"]; rows, cols, bits, cm = (int(v) for v in g[f"p/{n}/meta"])
    p = fq.pack(fq.bit_planes(vals, bits), fq.PackConfig(chunk_m=cm))
    ok = p.words.tobytes() == g[f"p/{n}/words"].tobytes()
    back = fq.recompose(fq.unpack(p, fq.PackConfig(chunk_m=cm)))
    ok2 = np.array_equal(back, vals.astype(np.int64))
    bad += not (ok and ok2); print("pack", n, ok, ok2)
for n in names("g"):
    m, nn, k, p_, q_, gs, passes = (int(v) for v in g[f"g/{n}/meta"])
    wq = fq.QuantTensor(g[f"g/{n}/wv"], g[f"g/{n}/ws"], p_, gs)
    xq = fq.QuantTensor(g[f"g/{n}/xv"], g[f"g/{n}/xs"], q_, gs)
    cfg = fq.GemmConfig(m=m, n=nn, k=k, weight_bits=p_, activation_bits=q_, group_size=gs)
    wp = fq.pack(fq.decompose(wq), fq.weight_pack_config()); xp = fq.pack(fq.decompose(xq), fq.activation_pack_config(m))
    out = fq.group_matmul_fused(wp, xp, wq.scales, xq.scales, cfg, trace=True)
    ok = np.array_equal(out.data, g[f"g/{n}/y"]) and np.array_equal(out.group_partials, g[f"g/{n}/partials"]) and out.bmma_passes == passes
    ref = fq.int_matmul_reference(wq, xq, cfg, trace=True)
    ok2 = np.array_equal(ref.data, g[f"g/{n}/y"]) and np.array_equal(ref.group_partials, g[f"g/{n}/partials"])
    if not (ok and ok2):
        print("  maxdiff bs", np.abs(out.group_partials - g[f"g/{n}/partials"]).max(), "t6", np.abs(ref.group_partials - g[f"g/{n}/partials"]).max())
    bad += not (ok and ok2); print("gemm", n, (m, nn, k, p_, q_, gs), ok, ok2)
for n in names("l"):
    p_, q_, gs, passes = (int(v) for v in g[f"l/{n}/meta"])
    out = fq.quantized_linear(g[f"l/{n}/w"], g[f"l/{n}/x"], p_, q_, gs, trace=True)
    ok = np.array_equal(out.data, g[f"l/{n}/y"]) and np.array_equal(out.group_partials, g[f"l/{n}/partials"]) and out.bmma_passes == passes
    bad += not ok; print("linear", n, ok)

# fast path vs C oracle
rng = np.random.default_rng(0)
for (m, n, k, q) in [(1, 4096, 4096, 8), (4, 11008, 4096, 6), (8, 4096, 11008, 8), (16, 1024, 8192, 6), (64, 512, 4096, 6), (100, 256, 1024, 8)]:
    w = rng.standard_normal((n, k)).astype(np.float16)
    x = rng.standard_normal((m, k)).astype(np.float16)
    lin = fq.FlexQLinear(w, 6, q, 128, fp16_scales=True)
    y = lin(torch.from_numpy(x).cuda()).float().cpu().numpy()
    wc, wsc = c_oracle.quantize(w, 6, 128, True); xc, xsc = c_oracle.quantize(x, q, 128, True)
    yr, _ = c_oracle.int_matmul(wc, xc, wsc, xsc, 128)
    err = np.abs(y - yr).max() / np.abs(yr).max()
    ok = err <= 1e-3
    bad += not ok
    # trace through the fast kernel
    print("fast", (m, n, k, q), f"maxrel={err:.2e}", ok)

# fast path across group sizes / token counts, plus exact partials through the fast kernel
from paper_2508_04405_b200.engine import t6_pack_weights, t6_pack_activations
L = _lib.lib()
for (m, n, k, q, gs) in [(1, 1000, 1024, 6, 32), (3, 200, 1024, 8, 64), (5, 256, 2048, 6, 256), (2, 512, 4096, 8, 4096),
                          (16, 384, 896, 6, 128), (12, 130, 640, 8, 100), (9, 1024, 1536, 6, 512), (1, 64, 128, 6, 128)]:
    w = rng.standard_normal((n, k)).astype(np.float16)
    x = rng.standard_normal((m, k)).astype(np.float16)
    wc, wsc = c_oracle.quantize(w, 6, gs, True); xc, xsc = c_oracle.quantize(x, q, gs, True)
    yr, pr = c_oracle.int_matmul(wc, xc, wsc, xsc, gs, trace=True)
    dw = torch.from_numpy(wc).cuda(); dws = torch.from_numpy(wsc).cuda()
    t6, wsp = t6_pack_weights(dw, dws, k, gs, True)
    frag, xs, corr, m_pad = t6_pack_activations(torch.from_numpy(xc).cuda(), torch.from_numpy(xsc).cuda(), k, gs)
    ng = -(-k // gs)
    parts = torch.zeros((ng, m, n), dtype=torch.int32, device="cuda")
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    wsb = torch.zeros(L.flexq_gemm_workspace_bytes(m, n, k, gs, 0), dtype=torch.uint8, device="cuda")
    for rep in range(2):
        parts.zero_()
        _lib.check(L.flexq_gemm_t6(_lib.ptr(t6), _lib.ptr(wsp), 1, _lib.ptr(frag), _lib.ptr(xs), _lib.ptr(corr), m, m_pad, n, k, gs,
                                   _lib.ptr(parts), _lib.ptr(y), _lib.OUT_F16, _lib.ptr(wsb), 0, _lib.stream()))
    torch.cuda.synchronize()
    pe = np.array_equal(parts.cpu().numpy(), pr)
    err = np.abs(y.float().cpu().numpy() - yr).max() / np.abs(yr).max()
    ok = pe and err <= 1e-3
    bad += not ok
    print("fast+trace", (m, n, k, q, gs), "partials exact", pe, f"maxrel={err:.2e}")
print("BAD", bad)
