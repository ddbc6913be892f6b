"""Report schemas and the CLI's host-side behaviour, no GPU.

Documents written by the real reference CLI (tests/golden/make_report_golden.py)
must validate; mutations the reference's schemas reject must be rejected with the
JSON pointer of the bad node.  The CLI cases restate the reference's test_cli.py
paths that fail before any compute (format, usage and policy errors)."""
import copy
import json
import os

import numpy as np
import pytest

from paper_2508_04405_b200 import fileio
from paper_2508_04405_b200.cli import main
from paper_2508_04405_b200.errors import FormatError
from paper_2508_04405_b200.quantize import QuantTensor
from paper_2508_04405_b200.reports import validate_json

REPORTS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reports")
DOCS = {"bench_sweep": "bench_report", "manifest_quantize": "manifest",
        "manifest_gemm": "manifest", "manifest_bench": "manifest",
        "sensitivity_manifest": "sensitivity_manifest", "sensitivity_report": "sensitivity_report"}


def load(name):
    with open(os.path.join(REPORTS, name + ".json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", sorted(DOCS))
def test_reference_documents_validate(name):
    validate_json(load(name), DOCS[name])


def mutate(doc, path, value):
    doc = copy.deepcopy(doc)
    node = doc
    for key in path[:-1]:
        node = node[key]
    if value is KeyError:
        del node[path[-1]]
    else:
        node[path[-1]] = value
    return doc


@pytest.mark.parametrize("name,path,value,pointer", [
    ("bench_sweep", ["results", 0, "shape"], [8, 256], "/results/0/shape"),
    ("bench_sweep", ["results", 3, "p"], 9, "/results/3/p"),
    ("bench_sweep", ["results", 0, "wall_ns"], 1.5, "/results/0/wall_ns"),
    ("bench_sweep", ["results", 0, "extra"], 1, "/results/0"),
    ("bench_sweep", ["best", "effective_GOPS"], -1.0, "/best/effective_GOPS"),
    ("bench_sweep", ["suite"], KeyError, "/"),
    ("manifest_gemm", ["inputs", "w.flxq"], "not-a-digest", "/inputs/w.flxq"),
    ("manifest_gemm", ["wall_ns"], True, "/wall_ns"),
    ("sensitivity_manifest", [0, "kind"], "dense", "/0/kind"),
    ("sensitivity_report", ["layers", 1, "outlier_score"], 0.5, "/layers/1/outlier_score"),
    ("sensitivity_report", ["layers", 0, "sqnr_db"], None, None),  # null = +inf: allowed
])
def test_mutations(name, path, value, pointer):
    doc = mutate(load(name), path, value)
    if pointer is None:
        validate_json(doc, DOCS[name])
        return
    with pytest.raises(FormatError) as e:
        validate_json(doc, DOCS[name])
    assert f"document at {pointer}:" in str(e.value)


@pytest.fixture
def workdir(tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    monkeypatch.delenv("BITSERIAL_OUT_DIR", raising=False)
    rng = np.random.default_rng(42)
    fileio.write_float("w.flxq", rng.standard_normal((32, 384)))
    fileio.write_float("x.flxq", rng.standard_normal((4, 384)))
    return tmp_path


def quant_file(path, rows, cols, group):
    ng = -(-cols // group)
    fileio.write_quant(path, QuantTensor(values=np.zeros((rows, cols), np.int8),
                                         scales=np.ones((rows, ng)), bits=6, group_size=group))


def test_cli_format_and_usage_errors(workdir, capsys):  # test_cli.py:44-56, 74-75, 100-116
    open("junk.flxq", "wb").write(b"JUNKJUNKJUNK")
    assert main(["quantize", "junk.flxq", "-o", "o.flxq"]) == 3
    assert "magic" in capsys.readouterr().err
    assert main(["quantize", "x.flxq", "-o", "o.flxq", "--layer-kind", "embed"]) == 2
    assert "no policy entry" in capsys.readouterr().err
    assert main(["pack", "w.flxq", "-o", "wp.flxq"]) == 3
    quant_file("wq.flxq", 32, 384, 128)
    quant_file("x2q.flxq", 4, 256, 128)
    assert main(["gemm", "wq.flxq", "x2q.flxq", "-o", "y.flxq"]) == 3
    err = capsys.readouterr().err
    assert "wq.flxq" in err and "x2q.flxq" in err
    quant_file("xg.flxq", 4, 384, 64)
    assert main(["gemm", "wq.flxq", "xg.flxq", "-o", "y.flxq"]) == 3
    assert "group" in capsys.readouterr().err
    assert main(["layout", "--golden"]) == 2
    assert not [f for f in os.listdir(workdir) if f.startswith(("y.flxq", "o.flxq", "wp.flxq"))]


def test_cli_bad_arguments(workdir):
    with pytest.raises(SystemExit) as e:
        main(["bench", "--suite", "nope"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        main(["quantize", "w.flxq", "-o", "o.flxq", "--bits", "9"])
    assert e.value.code == 2


def test_cli_malformed_sensitivity_manifest(workdir, capsys):  # test_cli.py:190-194
    json.dump([{"layer_name": "x", "kind": "dense", "weight_file": "a", "act_file": "b"}],
              open("layers.json", "w"))
    assert main(["sensitivity", "layers.json", "-o", "report.json"]) == 3
    assert "/0/kind" in capsys.readouterr().err
