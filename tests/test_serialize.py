"""QTT1 container (reference serialize.py): byte-level parity with containers the reference
wrote (tests/golden/*.qtt1, make_golden.py qtt1), the reference's FormatError cases, and the
native device loader/writer (qtt_train_load_qtt1 / qtt_train_save_qtt1)."""
import os

import numpy as np
import pytest

from tests.golden_io import GOLDEN

FIXTURES = ["vec.qtt1", "op.qtt1"]


def _bad_variants(data):
    return {
        "bad magic": b"QTT2" + data[4:],
        "unknown kind tag": data[:4] + b"X" + data[5:],
        "truncated header of core": data[:9 + 8],
        "truncated values of core": data[:-8],
        "trailing bytes": data + b"\x00",
    }


@pytest.mark.parametrize("name", FIXTURES)
def test_roundtrip_bytes_identical(tmp_path, name):
    from paper_2501_12151_b200 import serialize
    path = os.path.join(GOLDEN, name)
    obj = serialize.load_tt(path)
    out = tmp_path / name
    serialize.save_tt(obj, out)
    assert open(out, "rb").read() == open(path, "rb").read()
    d = serialize.tt_to_json_dict(obj)
    assert d["format"] == "QTT1" and len(d["cores"]) == len(obj.cores)


@pytest.mark.parametrize("name", FIXTURES)
def test_format_errors(tmp_path, name):
    from paper_2501_12151_b200 import serialize
    from paper_2501_12151_b200.errors import FormatError
    data = open(os.path.join(GOLDEN, name), "rb").read()
    for what, bad in _bad_variants(data).items():
        p = tmp_path / "bad.qtt1"
        p.write_bytes(bad)
        with pytest.raises(FormatError, match=what.split()[0]):
            serialize.load_tt(p)


@pytest.mark.gpu
@pytest.mark.parametrize("name", FIXTURES)
def test_device_load_save(tmp_path, name):
    from paper_2501_12151_b200 import serialize
    from paper_2501_12151_b200.errors import FormatError
    path = os.path.join(GOLDEN, name)
    host = serialize.load_tt(path)
    dev, is_op = serialize.load_device(path)
    assert is_op == (name == "op.qtt1")
    for c, r in zip(dev.cores(), host.cores):
        assert np.array_equal(c.reshape(r.shape), r)
    out = tmp_path / name
    serialize.save_device(dev, out)
    assert open(out, "rb").read() == open(path, "rb").read()
    for what, bad in _bad_variants(open(path, "rb").read()).items():
        p = tmp_path / "bad.qtt1"
        p.write_bytes(bad)
        with pytest.raises(FormatError, match=what.split()[0]):
            serialize.load_device(p)
