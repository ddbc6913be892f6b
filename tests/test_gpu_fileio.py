"""Reference-written FLXQ weight containers served by the B200 kernels (sec. 8(f) f3).

The weights in tests/golden/flxq were quantized / packed by the reference itself
(make_flxq_golden.py).  Loading them into FlexQLinear must give the reference's own
quantized_linear output (within the fp16 fast-path tolerance), and the three load
routes -- quant container, packed container + scales, float container re-quantized on
the GPU -- must stream identical T6 weights."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2508_04405_b200 as fq  # noqa: E402
from paper_2508_04405_b200 import fileio  # noqa: E402

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "flxq")
FP16_TOL = 1e-3


@pytest.fixture(scope="module")
def expect():
    with np.load(os.path.join(FIX, "expect.npz")) as z:
        return {k: z[k] for k in z.files}


def fix(name):
    return os.path.join(FIX, name + ".flxq")


def max_rel(y, ref):
    return float(np.max(np.abs(y.astype(np.float64) - ref)) / np.max(np.abs(ref)))


@pytest.mark.parametrize("a_bits", [6, 8])
def test_reference_quantized_weights_serve_reference_output(expect, a_bits):
    lin = fq.FlexQLinear.load(fix("wq6_g128_f8"), activation_bits=a_bits)
    assert not lin.fp16_scales  # the reference's f8 scales are not fp16 values
    x = torch.from_numpy(expect["x"]).cuda()
    for m in (1, x.shape[0]):  # GEMV path at M=1, batched below the tcgen05 crossover
        y = lin(x[:m]).float().cpu().numpy()
        assert max_rel(y, expect[f"wq6_g128_f8_y_a{a_bits}"][:m]) <= FP16_TOL
    lin.check_errors()


def test_load_routes_stream_identical_weights(expect):
    q = fileio.read_quant(fix("wq6_g128_f8"))
    a = fq.FlexQLinear.from_quant(q)
    b = fq.FlexQLinear.load(fix("wp6_w64"), scales=fix("wq6_g128_f8"))
    c = fq.FlexQLinear.from_packed(fileio.read_packed(fix("wp6_w64")), q.scales, 128)
    assert torch.equal(a.t6, b.t6) and torch.equal(a.wscale, b.wscale)
    assert torch.equal(a.t6, c.t6)
    x = torch.from_numpy(expect["x"]).cuda()
    assert torch.equal(a(x), b(x))


def test_fp16_scale_container_matches_gpu_quantized_layer(expect):
    """wq6_g64_f2 holds fp16 scales: served in the kernel's 2-byte scale mode, and
    bit-identical to quantizing the same float weights on the GPU."""
    lin = fq.FlexQLinear.load(fix("wq6_g64_f2"))
    assert lin.fp16_scales and lin.group_size == 64
    ref = fq.FlexQLinear.load(fix("weight_f2"), group_size=64)  # kind 0 -> GPU quantizer
    assert torch.equal(lin.t6, ref.t6) and torch.equal(lin.wscale, ref.wscale)
    x = torch.from_numpy(expect["x"]).cuda()
    assert torch.equal(lin(x), ref(x))


def test_gpu_pack_writes_reference_container(tmp_path):
    """GPU quantize -> decompose -> pack, then write_packed: the same bytes the
    reference's CLI pipeline wrote."""
    w = fileio.read_float(fix("weight_f2"))
    p = fq.pack(fq.decompose(fq.quantize(w, 6, 128)), fq.weight_pack_config(64))
    out = str(tmp_path / "p.flxq")
    fileio.write_packed(out, p)
    assert open(out, "rb").read() == open(fix("wp6_w64"), "rb").read()
    q = fq.quantize(w, 6, 128)
    fileio.write_quant(str(tmp_path / "q.flxq"), q)
    assert open(tmp_path / "q.flxq", "rb").read() == open(fix("wq6_g128_f8"), "rb").read()


def test_packed_activation_container_round_trip(expect):
    xp = fileio.read_packed(fix("xp6_w32"))
    back = fq.recompose(fq.unpack(xp, xp.config))
    assert np.array_equal(back, expect["xp6_w32_values"])


def test_rejects_unservable_containers(tmp_path):
    xq = fileio.read_quant(fix("xq8_pertoken"))
    with pytest.raises(fq.InvalidInputError):
        fq.FlexQLinear.from_quant(xq)  # 8-bit codes do not fit the T6 weight stream
    with pytest.raises(fq.InvalidInputError):
        fq.FlexQLinear.load(fix("wp6_w64"))  # packed planes without scales
