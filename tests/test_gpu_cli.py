"""The CLI end to end on the GPU (restates the reference's test_cli.py), plus the
cross-implementation checks: reference-written containers as inputs, bench reports
in the reference's schema, and `verify` passing on a fresh checkout."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2508_04405_b200 import fileio  # noqa: E402
from paper_2508_04405_b200.cli import main  # noqa: E402
from paper_2508_04405_b200.quantize import dequantize  # noqa: E402
from paper_2508_04405_b200.reports import validate_json  # noqa: E402

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "flxq")


@pytest.fixture
def workdir(tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    monkeypatch.delenv("BITSERIAL_OUT_DIR", raising=False)
    rng = np.random.default_rng(42)
    fileio.write_float("w.flxq", rng.standard_normal((32, 384)))
    fileio.write_float("x.flxq", rng.standard_normal((4, 384)))
    return tmp_path


def manifest(path):
    doc = json.load(open(path))
    validate_json(doc, "manifest")
    return doc


def test_quantize_round_trip_bound_and_manifest(workdir):  # test_cli.py:28-39
    assert main(["quantize", "w.flxq", "-o", "wq.flxq", "--bits", "6", "--group", "128"]) == 0
    q, w = fileio.read_quant("wq.flxq"), fileio.read_float("w.flxq")
    bound = np.repeat(q.scales, 128, axis=1)[:, :384] / 2
    assert np.all(np.abs(w - dequantize(q)) <= bound + 1e-12)
    m = manifest("wq.flxq.manifest.json")
    assert m["command"] == "quantize" and "w.flxq" in m["inputs"]
    main(["quantize", "w.flxq", "-o", "b.flxq"])
    assert open("wq.flxq", "rb").read() == open("b.flxq", "rb").read()
    assert main(["quantize", "x.flxq", "-o", "xq.flxq", "--layer-kind", "down_proj"]) == 0
    assert fileio.read_quant("xq.flxq").bits == 8
    assert main(["quantize", "x.flxq", "-o", "xg.flxq", "--group", "4096"]) == 0
    assert fileio.read_quant("xg.flxq").scales.shape == (4, 1)


def test_pack_and_check(workdir):  # test_cli.py:66-71
    main(["quantize", "w.flxq", "-o", "wq.flxq"])
    assert main(["pack", "wq.flxq", "-o", "wp.flxq", "--operand", "weight", "--check"]) == 0
    assert fileio.read_packed("wp.flxq").words.shape == (3, 4, 6, 8, 2)


@pytest.mark.parametrize("engine", ["bitserial", "t6"])
def test_gemm_oracle_and_manifest(workdir, engine):  # test_cli.py:79-83
    assert main(["gemm", "w.flxq", "x.flxq", "-o", "y.flxq", "--oracle", "--engine", engine]) == 0
    assert manifest("y.flxq.manifest.json")["stats"]["bmma_passes"] == 36 * 3 * 4
    assert fileio.read_float("y.flxq").shape == (4, 32)


def test_gemm_deterministic_across_knobs_and_engines(workdir):  # test_cli.py:85-88
    main(["gemm", "w.flxq", "x.flxq", "-o", "a.flxq", "--stages", "1", "--workers", "1"])
    main(["gemm", "w.flxq", "x.flxq", "-o", "b.flxq", "--stages", "3", "--workers", "8"])
    main(["gemm", "w.flxq", "x.flxq", "-o", "c.flxq", "--engine", "t6"])
    assert open("a.flxq", "rb").read() == open("b.flxq", "rb").read() == open("c.flxq", "rb").read()


def test_gemm_quant_inputs(workdir):  # test_cli.py:90-93
    main(["quantize", "w.flxq", "-o", "wq.flxq"])
    main(["quantize", "x.flxq", "-o", "xq.flxq", "--bits", "8"])
    assert main(["gemm", "wq.flxq", "xq.flxq", "-o", "y.flxq", "--oracle"]) == 0


def test_gemm_on_reference_written_containers(workdir):
    """A weight container quantized by the reference CLI feeds this CLI's gemm."""
    w = os.path.join(FIX, "wq6_g128_f8.flxq")
    fileio.write_float("xr.flxq", np.random.default_rng(3).standard_normal((3, 320)))
    assert main(["gemm", w, "xr.flxq", "-o", "y.flxq", "--oracle"]) == 0
    assert fileio.read_float("y.flxq").shape == (3, 72)


def test_bench_sweep_schema_and_tie_break(workdir, capsys):  # test_cli.py:140-151
    assert main(["bench", "--suite", "sweep", "--json", "--repeat", "1", "--workers", "2"]) == 0
    doc = json.loads(capsys.readouterr().out)
    validate_json(doc, "bench_report")
    gops = [r["effective_GOPS"] for r in doc["results"]]
    assert doc["best"]["effective_GOPS"] == max(gops)
    ties = [r for r in doc["results"] if r["effective_GOPS"] == doc["best"]["effective_GOPS"]]
    assert doc["best"]["tile"] == min(t["tile"] for t in ties)


@pytest.mark.parametrize("engine", ["bitserial", "t6"])
def test_bench_llama_shapes(workdir, engine):
    assert main(["bench", "--suite", "llama-shapes", "--repeat", "2", "--engine", engine,
                 "-o", "b.json"]) == 0
    doc = json.load(open("b.json"))
    validate_json(doc, "bench_report")
    assert [r["name"] for r in doc["results"]][:3] == ["attn_4k_b1", "ffn_down_7b_b1",
                                                        "ffn_down_70b_b1"]
    assert doc["results"][0]["shape"] == [1, 4096, 4096]
    assert manifest("b.json.manifest.json")["command"] == "bench"


def test_sensitivity_report_and_policy(workdir):  # test_cli.py:175-188
    rng = np.random.default_rng(7)
    entries = []
    for kind in ("gate_proj", "down_proj", "up_proj"):
        acts = rng.standard_normal((8, 256))
        if kind == "down_proj":
            acts[:, 3] *= 100
        fileio.write_float(f"{kind}_w.flxq", rng.standard_normal((16, 256)))
        fileio.write_float(f"{kind}_x.flxq", acts)
        entries.append({"layer_name": f"blk.0.{kind}", "kind": kind,
                        "weight_file": f"{kind}_w.flxq", "act_file": f"{kind}_x.flxq"})
    json.dump(entries, open("layers.json", "w"))
    assert main(["sensitivity", "layers.json", "-o", "report.json", "--budget", "1",
                 "--policy-out", "policy.json"]) == 0
    report = json.load(open("report.json"))
    validate_json(report, "sensitivity_report")
    assert report["ranking"][0] == "blk.0.down_proj"
    policy = json.load(open("policy.json"))
    assert policy["down_proj"] == 8 and policy["gate_proj"] == 6
    assert len(manifest("report.json.manifest.json")["inputs"]) == 7


def test_verify_passes(workdir, capsys):  # test_cli.py:198-202
    assert main(["verify"]) == 0
    out = capsys.readouterr().out
    assert "FAIL" not in out and "oracle-equivalence" in out


def test_output_dir_override(workdir, monkeypatch):  # test_cli.py:204-207
    monkeypatch.setenv("BITSERIAL_OUT_DIR", str(workdir / "artifacts"))
    assert main(["quantize", "w.flxq", "-o", "wq.flxq"]) == 0
    assert os.path.exists(workdir / "artifacts" / "wq.flxq")
