"""FLXQ containers on the host, no GPU needed.

Pinned to containers written by the real reference (tests/golden/make_flxq_golden.py):
every fixture decodes to the arrays the reference wrote, and re-writing what we read
reproduces the reference's file byte for byte.  The rejection cases restate the
reference's test_fileio.py:64-116."""
import os
import shutil
import struct

import numpy as np
import pytest

from paper_2508_04405_b200 import fileio
from paper_2508_04405_b200.errors import FormatError, InvalidInputError
from paper_2508_04405_b200.packing import PackedTensor, activation_pack_config, weight_pack_config
from paper_2508_04405_b200.quantize import QuantTensor

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "flxq")
CONTAINERS = sorted(f[:-5] for f in os.listdir(FIX) if f.endswith(".flxq"))


@pytest.fixture(scope="module")
def expect():
    with np.load(os.path.join(FIX, "expect.npz")) as z:
        return {k: z[k] for k in z.files}


def fix(name):
    return os.path.join(FIX, name + ".flxq")


def raw(name):
    with open(fix(name), "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("tag", ["f8", "f4", "f2"])
def test_float_containers(tag, expect):
    got = fileio.read_float(fix(f"float_{tag}"))
    assert got.dtype == np.float64 and np.array_equal(got, expect[f"float_{tag}"])


@pytest.mark.parametrize("name", ["wq6_g128_f8", "wq6_g64_f2", "xq8_pertoken"])
def test_quant_containers(name, expect):
    q = fileio.read_quant(fix(name))
    assert q.values.dtype == np.int8 and q.scales.dtype == np.float64
    assert np.array_equal(q.values, expect[name + "_values"])
    assert np.array_equal(q.scales, expect[name + "_scales"])
    assert q.group_axis == 1


def test_packed_containers(expect):
    wp = fileio.read_packed(fix("wp6_w64"))
    assert wp.config == weight_pack_config(64) and (wp.bits, wp.signed) == (6, True)
    assert np.array_equal(wp.words, expect["wp6_w64_words"])
    xp = fileio.read_packed(fix("xp6_w32"))
    assert xp.config == activation_pack_config(3, 32)
    assert (xp.rows, xp.cols) == (3, 200) and xp.words.dtype == np.dtype("<u4")
    assert np.array_equal(xp.words, expect["xp6_w32_words"])


@pytest.mark.parametrize("name", CONTAINERS)
def test_rewrite_is_byte_identical_to_reference(name, tmp_path):
    obj = fileio.read(fix(name))
    out = str(tmp_path / "o.flxq")
    if isinstance(obj, np.ndarray):
        code = raw(name)[7]
        fileio.write_float(out, obj, dtype=("<f8", "<f4", "<f2")[code])
    elif isinstance(obj, QuantTensor):
        scode = struct.unpack_from("<BBIB", raw(name), 9 + 16)[3]
        fileio.write_quant(out, obj, scale_dtype=("<f8", "<f4", "<f2")[scode])
    else:
        fileio.write_packed(out, obj)
    assert open(out, "rb").read() == raw(name)
    assert fileio.file_digest(out) == fileio.file_digest(fix(name))


def test_writers_take_numpy_built_tensors(tmp_path, expect):
    q = QuantTensor(values=expect["wq6_g128_f8_values"], scales=expect["wq6_g128_f8_scales"],
                    bits=6, group_size=128)
    fileio.write_quant(str(tmp_path / "q.flxq"), q)
    assert open(tmp_path / "q.flxq", "rb").read() == raw("wq6_g128_f8")
    p = PackedTensor(words=expect["wp6_w64_words"], bits=6, signed=True,
                     config=weight_pack_config(64), rows=72, cols=320)
    fileio.write_packed(str(tmp_path / "p.flxq"), p)
    assert open(tmp_path / "p.flxq", "rb").read() == raw("wp6_w64")


def corrupt(tmp_path, edit):
    p = str(tmp_path / "c.flxq")
    shutil.copy(fix("wq6_g128_f8"), p)
    blob = bytearray(open(p, "rb").read())
    blob = edit(blob)
    open(p, "wb").write(bytes(blob))
    return p


@pytest.mark.parametrize("edit,match", [
    (lambda b: b"NOPE" + b[4:], "magic"),
    (lambda b: b[:4] + struct.pack("<H", 9) + b[6:], "version"),
    (lambda b: b[:7] + b"\x2a" + b[8:], "dtype code"),
    (lambda b: b[:8] + b"\x00" + b[9:], "ndim"),
    (lambda b: b[:6] + b"\x07" + b[7:], "kind"),
    (lambda b: b[:-3], "truncated"),
    (lambda b: b[:20], "truncated"),
    (lambda b: b + b"\x00\x01", "trailing"),
    (lambda b: b[:27] + bytes(4) + b[31:], "group_size"),  # u32 group_size at 27 -> 0
    (lambda b: b[:31] + b"\x09" + b[32:], "scale dtype"),
])
def test_rejects_malformed(tmp_path, edit, match):
    with pytest.raises(FormatError, match=match):
        fileio.read(corrupt(tmp_path, edit))


def test_out_of_range_codes_rejected(tmp_path):
    def edit(b):
        b[-1] = 0x7F  # 127 > qmax(6) = 31
        return b
    with pytest.raises(InvalidInputError):
        fileio.read(corrupt(tmp_path, edit))


def test_kind_mismatch(tmp_path):
    with pytest.raises(FormatError, match="kind 0"):
        fileio.read_float(fix("wq6_g128_f8"))
    with pytest.raises(FormatError, match="kind 2"):
        fileio.read_packed(fix("wq6_g128_f8"))
    with pytest.raises(FormatError, match="kind 1"):
        fileio.read_quant(fix("wp6_w64"))


def test_no_partial_file_on_failed_write(tmp_path):
    target = str(tmp_path / "out.flxq")
    with pytest.raises(FormatError):
        fileio.write_float(target, np.zeros((2, 2, 2)))
    with pytest.raises(FormatError):
        fileio.write_float(target, np.zeros((2, 2)), dtype="<c16")
    assert not os.path.exists(target)
    assert not [f for f in os.listdir(tmp_path) if f.startswith(".flxq-")]


def test_file_digest_is_sha256(tmp_path):
    p = tmp_path / "x.bin"
    p.write_bytes(b"abc")
    assert fileio.file_digest(str(p)) == \
        "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
