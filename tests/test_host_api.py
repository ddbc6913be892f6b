"""Host-side behaviour of the drop-in API that needs no GPU: configuration
validation, error classes and messages, policy, pass accounting, shapes.
Each case restates a reference test (file:line under pkg/tests/)."""
import numpy as np
import pytest

import paper_2508_04405_b200 as fq
from paper_2508_04405_b200.engine import bmma_passes
from paper_2508_04405_b200.shapes import MODELS, gemm_bytes, layer_bytes, unfused


def test_error_taxonomy_matches_reference():  # errors.py:4-28
    for cls, base in ((fq.InvalidInputError, ValueError), (fq.ShapeError, ValueError),
                      (fq.ConfigError, ValueError), (fq.FormatError, ValueError),
                      (fq.PolicyMissError, KeyError), (fq.BoundsError, ValueError)):
        assert issubclass(cls, fq.BitserialError) and issubclass(cls, base)


def test_pack_config_validation():  # test_packing.py:24-41
    assert fq.activation_pack_config(1).chunk_m == 1
    assert fq.activation_pack_config(4).chunk_m == 4
    assert fq.activation_pack_config(100).chunk_m == 8
    assert fq.weight_pack_config().chunk_m == 8
    with pytest.raises(fq.ConfigError):
        fq.PackConfig(chunk_m=8, word_bits=48)
    with pytest.raises(fq.ConfigError):
        fq.PackConfig(chunk_m=9)


def test_gemm_config_validation():  # engine.py:52-66
    with pytest.raises(fq.ConfigError):
        fq.GemmConfig(m=0, n=8, k=128)
    with pytest.raises(fq.ConfigError):
        fq.GemmConfig(m=1, n=8, k=128, weight_bits=9)
    with pytest.raises(fq.ConfigError):
        fq.GemmConfig(m=1, n=8, k=128, group_size=0)
    with pytest.raises(fq.ConfigError):
        fq.GemmConfig(m=1, n=8, k=128, pipeline_stages=0)
    assert fq.GemmConfig(m=1, n=8, k=300).n_groups == 3


def test_policy():  # test_quantize.py:141-170
    assert fq.activation_bits("down_proj", fq.DEFAULT_POLICY) == 8
    for kind in ("qkv_proj", "o_proj", "gate_proj", "up_proj", "generic"):
        assert fq.activation_bits(kind, fq.DEFAULT_POLICY) == 6
    assert all(fq.activation_bits(k, fq.uniform_policy(6)) == 6 for k in fq.LAYER_KINDS)
    with pytest.raises(fq.PolicyMissError):
        fq.activation_bits("lm_head", fq.DEFAULT_POLICY)
    with pytest.raises(fq.InvalidInputError):
        fq.BitPolicy(weight_bits=6, activation_bits_by_layer={"generic": 5})


def test_plane_coeffs():  # test_bitplane.py:10-26, 76-80
    assert fq.plane_coeff(0, 6) == 1 and fq.plane_coeff(5, 6) == -32
    assert [fq.plane_coeff(s, 4, signed=False) for s in range(4)] == [1, 2, 4, 8]
    with pytest.raises(IndexError):
        fq.plane_coeff(6, 6)
    for bits in range(2, 9):
        for signed in (True, False):
            assert fq.plane_coeffs(bits, signed).tolist() == [fq.plane_coeff(s, bits, signed)
                                                             for s in range(bits)]


def test_quanttensor_validation_host_arrays():  # test_quantize.py:117-138
    with pytest.raises(fq.InvalidInputError):
        fq.QuantTensor(values=np.zeros((2, 256), np.int8), scales=np.ones((2, 1)), bits=6,
                       group_size=128)
    with pytest.raises(fq.InvalidInputError):
        fq.QuantTensor(values=np.zeros((1, 4), np.int8), scales=np.zeros((1, 1)), bits=6,
                       group_size=4)
    with pytest.raises(fq.InvalidInputError):
        fq.QuantTensor(values=np.full((1, 4), -32, np.int8), scales=np.ones((1, 1)), bits=6,
                       group_size=4)
    q = fq.QuantTensor(values=np.zeros((3, 300), np.int8), scales=np.ones((3, 3)), bits=6,
                       group_size=128)
    assert q.shape == (3, 300) and q.n_groups == 3
    # wide integer codes are range-checked before any narrowing (65539 & 0xffff == 3)
    with pytest.raises(fq.InvalidInputError):
        fq.QuantTensor(values=np.full((1, 4), 65539, np.int32), scales=np.ones((1, 1)), bits=6,
                       group_size=4)
    torch = pytest.importorskip("torch")
    with pytest.raises(fq.InvalidInputError):  # abs(int8 -128) wraps to -128 unless widened
        fq.QuantTensor(values=torch.full((1, 4), -128, dtype=torch.int8),
                       scales=torch.ones((1, 1), dtype=torch.float64), bits=8, group_size=4)


def test_bit_planes_range_checked_before_narrowing():  # bitplane.py:60-64 (reference raises)
    with pytest.raises(fq.InvalidInputError):
        fq.bit_planes(np.array([[65539]], np.int32), 6)
    with pytest.raises(fq.InvalidInputError):
        fq.bit_planes(np.array([[-33, 0]], np.int64), 6)
    with pytest.raises(fq.InvalidInputError):
        fq.bit_planes(np.array([[64]], np.int16), 6, signed=False)


def test_bmma_pass_accounting_matches_reference(golden):  # test_engine.py:243-271, test_bench.py:25-34
    for name in golden.names("g"):
        m, n, k, p, q, gs, passes = (int(v) for v in golden[f"g/{name}/meta"])
        cfg = fq.GemmConfig(m=m, n=n, k=k, weight_bits=p, activation_bits=q, group_size=gs)
        assert bmma_passes(cfg, min(m, 8)) == passes, name
    cfg = fq.GemmConfig(m=1, n=4096, k=4096)
    assert bmma_passes(cfg, 1) == 36 * (4096 // 128) * (4096 // 8)
    assert bmma_passes(fq.GemmConfig(m=2, n=8, k=256, activation_bits=8), 2) == 48 * 2


def test_llama_shapes_and_bytes():
    s70 = {s.name: s for s in MODELS["llama2-70b"]}
    assert (s70["qkv_proj"].n, s70["qkv_proj"].k) == (10240, 8192)
    assert (s70["down_proj"].n, s70["down_proj"].k, s70["down_proj"].act_bits) == (8192, 28672, 8)
    assert [s.name for s in unfused(MODELS["llama2-70b"])][:3] == ["q_proj", "k_proj", "v_proj"]
    # BASELINE.md sec. 2 algorithmic bytes: 4096^2 W6A8 M=1 -> 12.86 MB
    assert abs(layer_bytes(1, 4096, 4096) / 1e6 - 12.86) < 0.01
    assert abs(layer_bytes(1, 8192, 28672) / 1e6 - 179.90) < 0.01
    assert gemm_bytes(1, 4096, 4096) > 4096 * 4096 * 6 // 8
