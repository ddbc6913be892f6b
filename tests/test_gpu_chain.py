"""GPU parity of FlexQChain (csrc/gemv_chain.cu): a stack of W6Ax linears in one persistent
launch.  Every link must give exactly what the per-linear call gives (same quantizer,
same split of the layer over the same warps, same fixed-order fixups: bit-identical fp16
y), and through it what the reference gives: codes of quantize() and int_matmul_reference
(engine.py:337-365) within the fp16 tolerance.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2508_04405_b200 as fq  # noqa: E402
from oracle import c_oracle  # noqa: E402

FP16_TOL = 1e-3


def _layers(shapes, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [fq.FlexQLinear(torch.randn((n, k), generator=g, device="cuda").half(),
                           activation_bits=q) for n, k, q in shapes]


def _inputs(layers, m, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.randn((m, lay.k), generator=g, device="cuda").half() for lay in layers]


@pytest.mark.parametrize("m", [1, 3, 8, 12, 16])
@pytest.mark.parametrize("dep", [True, False])
def test_chain_equals_per_layer(m, dep):
    # small (4-stage), mid (3-stage) and large (2-stage per-linear rings) layers mixed
    shapes = [(1024, 4096, 6), (4096, 1024, 8), (10240, 8192, 6), (2048, 3072, 8), (640, 2048, 6)]
    layers = _layers(shapes, seed=m)
    xs = _inputs(layers, m, seed=100 + m)
    ref = [lay(x) for lay, x in zip(layers, xs)]
    chain = fq.FlexQChain(layers, depends_on_prev=dep)
    ys = chain(xs)
    torch.cuda.synchronize()
    for i, (y, r) in enumerate(zip(ys, ref)):
        assert torch.equal(y, r), f"link {i}: chain differs from the per-layer call"
    ys2 = chain(xs)  # replay: workspace counters / barrier left reusable
    for y, r in zip(ys2, ref):
        assert torch.equal(y, r)
    chain.check_errors()


@pytest.mark.parametrize("m", [1, 5])
def test_chain_against_oracle(m):
    rng = np.random.default_rng(m)
    shapes = [(768, 2048, 6), (2048, 768, 8)]
    ws = [rng.standard_normal((n, k)).astype(np.float16) for n, k, _ in shapes]
    xs = [rng.standard_normal((m, k)).astype(np.float16) for _, k, _ in shapes]
    xs[1][:, 3] *= 60  # outlier channel: full-range A8 codes
    layers = [fq.FlexQLinear(w, activation_bits=q) for w, (_, _, q) in zip(ws, shapes)]
    ys = fq.FlexQChain(layers)([torch.from_numpy(x).cuda() for x in xs])
    for w, x, (_, _, q), y in zip(ws, xs, shapes, ys):
        wc, wsc = c_oracle.quantize(w, 6, 128, True)
        xc, xsc = c_oracle.quantize(x, q, 128, True)
        y_ref, _ = c_oracle.int_matmul(wc, xc, wsc, xsc, 128)
        err = np.abs(y.float().cpu().numpy() - y_ref).max() / np.abs(y_ref).max()
        assert err <= FP16_TOL


def test_chain_dependent_links_and_residual():
    """x of link i aliases y of link i-1 (a real layer stack); residual fused, aliasing out."""
    m = 4
    layers = _layers([(2048, 1024, 6), (1024, 2048, 8), (1024, 1024, 6)], seed=7)
    x0 = _inputs(layers[:1], m, seed=8)[0]
    r = torch.randn((m, 1024), device="cuda").half()
    # per-layer reference
    y0 = layers[0](x0)
    y1 = layers[1](y0)
    y2 = y1.clone()
    layers[2].forward(y1, out=y2, residual=y2)
    # chain with the same wiring: link 1 reads link 0's output, link 2 adds its residual
    o0 = torch.empty_like(y0)
    o1 = torch.empty_like(y1)
    o2 = torch.empty_like(y2)
    chain = fq.FlexQChain(layers)
    # link 2's residual is its own input y1 -> o1 (read after link 1 completes)
    chain([x0, o0, o1], outs=[o0, o1, o2], residuals=[None, None, o1])
    torch.cuda.synchronize()
    assert torch.equal(o0, y0) and torch.equal(o1, y1) and torch.equal(o2, y2)
    del r


def test_chain_graph_capture_and_validation():
    layers = _layers([(512, 1024, 6), (256, 512, 8)], seed=3)
    xs = _inputs(layers, 2, seed=4)
    chain = fq.FlexQChain(layers)
    ref = chain(xs)
    torch.cuda.synchronize()
    outs = [torch.empty_like(y) for y in ref]
    chain(xs, outs=outs)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        chain(xs, outs=outs)
    for o in outs:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert all(torch.equal(o, r) for o, r in zip(outs, ref))
    with pytest.raises(fq.ShapeError):
        chain([xs[0]])
    with pytest.raises(fq.ShapeError):
        chain([torch.zeros((17, 1024), device="cuda").half(), xs[1]])
    with pytest.raises(fq.ConfigError):
        fq.FlexQChain([layers[0], layers[0]], depends_on_prev=False)
    with pytest.raises(fq.ConfigError):
        fq.FlexQChain([fq.FlexQLinear(torch.randn((64, 256), device="cuda").half(), group_size=64)])
    bad = [xs[0].clone(), xs[1]]
    bad[0][0, 0] = float("nan")
    chain(bad)
    with pytest.raises(fq.InvalidInputError):
        chain.check_errors()
