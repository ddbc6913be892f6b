"""Sensitivity analysis on the GPU, restating the reference's
tests/test_sensitivity.py and acceptance criterion 7 (test_acceptance.py:192-209).  The
metrics come from the drop-in quantized_linear, whose float64 output is bit-identical to
the reference's, so SQNR values are compared exactly against the CPU oracle."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

from oracle import np_oracle  # noqa: E402
from paper_2508_04405_b200.errors import InvalidInputError  # noqa: E402
from paper_2508_04405_b200.quantize import LAYER_KINDS  # noqa: E402
from paper_2508_04405_b200.sensitivity import (  # noqa: E402
    LayerDump, assign_policy, calibrate_decoder, layer_error, make_glu_fixture, outlier_score,
    rank_layers)


def gaussian_dump(seed, kind="generic", name=None, tokens=16, hidden=256, out=32):
    rng = np.random.default_rng(seed)
    return LayerDump(layer_name=name or f"layer.{kind}.{seed}", layer_kind=kind,
                     weight=rng.standard_normal((out, hidden)),
                     activations=rng.standard_normal((tokens, hidden)))


def oracle_layer_error(d, w_bits, a_bits, gs=128):
    ref = d.activations @ d.weight.T
    got, _, _ = np_oracle.quantized_linear(d.weight, d.activations, w_bits, a_bits, gs)
    err = ref - got
    noise, signal = float(np.sum(err * err)), float(np.sum(ref * ref))
    if signal == 0.0 or noise == 0.0:
        return math.inf, noise / err.size
    return 10.0 * math.log10(signal / noise), noise / err.size


@pytest.mark.parametrize("seed,a_bits", [(0, 6), (1, 8), (2, 6)])
def test_layer_error_bit_identical_to_oracle(seed, a_bits):
    for d in make_glu_fixture(seed):
        assert layer_error(d, 6, a_bits) == oracle_layer_error(d, 6, a_bits)


def test_layer_error_cases():  # test_sensitivity.py:30-78
    sqnr, mse = layer_error(LayerDump("id", "generic", np.eye(8, 128), np.eye(8, 128)), 6, 6, 128)
    assert sqnr > 30 and mse < 1e-6
    sqnr, mse = layer_error(LayerDump("z", "generic", np.ones((4, 128)), np.zeros((4, 128))), 6, 6)
    assert math.isinf(sqnr) and mse == 0.0
    base = gaussian_dump(0)
    spiked = base.activations.copy()
    spiked[:, 7] *= 100
    assert layer_error(LayerDump(base.layer_name, "generic", base.weight, spiked), 6, 6)[0] < \
        layer_error(base, 6, 6)[0]
    for seed in range(5):
        d = gaussian_dump(seed)
        assert layer_error(d, 6, 8)[0] >= layer_error(d, 6, 6)[0]
    with pytest.raises(InvalidInputError):
        LayerDump("bad", "generic", np.ones((4, 128)), np.ones((4, 64)))
    with pytest.raises(InvalidInputError):
        LayerDump("bad", "mlp", np.ones((4, 64)), np.ones((4, 64)))


def test_outlier_score():  # test_sensitivity.py:81-92
    rng = np.random.default_rng(0)
    assert outlier_score(rng.standard_normal((64, 128))) < 3
    acts = np.random.default_rng(1).standard_normal((64, 128))
    acts[:, 5] *= 100
    assert outlier_score(acts) > 20


def test_glu_ranking_and_bit_monotonicity():  # acceptance criterion 7 (test_acceptance.py:193-209)
    down_first = monotone = 0
    seeds = 20
    for seed in range(seeds):
        dumps = make_glu_fixture(seed)
        down_first += rank_layers(dumps, 6, 6, 128).ranking[0].endswith("down_proj")
        down = next(d for d in dumps if d.layer_kind == "down_proj")
        monotone += layer_error(down, 6, 8, 128)[0] >= layer_error(down, 6, 6, 128)[0]
    assert down_first >= 19 and monotone == seeds


def test_ranking_and_policy():  # test_sensitivity.py:95-170
    dumps = make_glu_fixture(0)
    rep = rank_layers(dumps)
    assert sorted(rep.ranking) == sorted(d.layer_name for d in dumps)
    assert rank_layers(dumps, workers=4).ranking == rep.ranking
    base = gaussian_dump(5)
    tied = [LayerDump(n, "generic", base.weight, base.activations) for n in ("c", "a", "b")]
    assert rank_layers(tied).ranking == ("a", "b", "c")
    with pytest.raises(InvalidInputError):
        rank_layers([])
    table = assign_policy(rep, 8, budget_k=1).activation_bits_by_layer
    assert table["down_proj"] == 8 and all(table[k] == 6 for k in LAYER_KINDS if k != "down_proj")
    assert all(b == 6 for b in assign_policy(rep, 8, 0).activation_bits_by_layer.values())
    with pytest.raises(InvalidInputError):
        assign_policy(rep, 8, budget_k=len(dumps) + 1)


def test_calibrate_tiny_decoder():
    from paper_2508_04405_b200.llama import FlexQLlamaDecoder, LlamaConfig

    cfg = LlamaConfig(hidden=256, heads=2, ffn=512, layers=2, vocab=500)
    dec = FlexQLlamaDecoder(cfg, batch=4, max_len=16, seed=3)
    dec.reset()
    report, policy = calibrate_decoder(dec, steps=3, layers=1, budget_k=1)
    assert len(report.ranking) == 4
    top_kind = report.ranking[0].rsplit(".", 1)[1]
    assert dec.policy_table()[top_kind] == 8
    assert sum(v == 8 for v in dec.policy_table().values()) == 1
    dec.reset()
    dec.capture()
    toks = [dec.step().clone() for _ in range(3)]
    assert all(int(t.max()) < cfg.vocab for t in toks)
    dec.check_errors()
