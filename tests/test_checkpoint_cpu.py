"""int8flow-checkpoint-v1 (qlayers.py:598-637): byte-identical with files the reference wrote."""
import json
import os

import numpy as np
import pytest

from paper_2403_12422_b200.checkpoint import FORMAT, load_params, save_params

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _ref():
    return os.path.join(GOLD, "ckpt_ref")


def test_load_reference_checkpoint():
    params, manifest = load_params(_ref())
    assert manifest == {"step": 7, "opt_t": 7, "scheme": "per-block"}
    assert sorted(params) == ["a", "b.w", "scalar"]
    assert params["b.w"].shape == (3, 5) and params["scalar"].shape == ()
    assert all(v.dtype == np.float32 for v in params.values())


def test_save_is_byte_identical(tmp_path):
    params, manifest = load_params(_ref())
    out = tmp_path / "ck"
    save_params(out, params, manifest)
    for ext in (".bin", ".json"):
        with open(_ref() + ext, "rb") as a, open(str(out) + ext, "rb") as b:
            assert a.read() == b.read(), ext


def test_errors(tmp_path):
    out = tmp_path / "bad"
    save_params(out, {"w": np.zeros((2, 2), np.float32)})
    doc = json.loads((tmp_path / "bad.json").read_text())
    assert doc["format"] == FORMAT
    doc["format"] = "other"
    (tmp_path / "bad.json").write_text(json.dumps(doc))
    with pytest.raises(ValueError, match="unrecognized checkpoint format"):
        load_params(out)
    save_params(out, {"w": np.zeros((2, 2), np.float32)})
    (tmp_path / "bad.bin").write_bytes(b"\0" * 20)
    with pytest.raises(ValueError, match="does not match"):
        load_params(out)
