"""read_vecs / write_vecs / read_ivecs / write_ivecs (evalio.cpp:31-123) on
the host: bit-exact round trips and the reference's FormatError cases."""
import os
import struct

import numpy as np
import pytest


@pytest.mark.parametrize("kind,dt", [("f32", np.float32), ("u8", np.uint8), ("i32", np.int32)])
def test_vecs_roundtrip(knng, tmp_path, kind, dt):
    rng = np.random.default_rng(3)
    x = (rng.normal(size=(37, 13)) * 100).astype(dt) if dt != np.uint8 else \
        rng.integers(0, 256, size=(37, 13)).astype(np.uint8)
    p = str(tmp_path / f"x.{kind}vecs")
    knng.write_vecs(p, x)
    raw = open(p, "rb").read()
    esz = np.dtype(dt).itemsize
    assert len(raw) == 37 * (4 + 13 * esz)
    assert struct.unpack("<i", raw[:4])[0] == 13
    assert knng.vecs_shape(p, kind) == (37, 13)
    y = knng.read_vecs(p, kind)
    assert y.dtype == dt and np.array_equal(y.view(np.uint8), x.view(np.uint8))


def _write(path, rows):
    with open(path, "wb") as f:
        for dim, payload in rows:
            f.write(struct.pack("<i", dim) + payload)


def test_vecs_format_errors(knng, tmp_path):
    p = str(tmp_path / "bad.fvecs")
    row = np.arange(4, dtype=np.float32).tobytes()
    cases = [
        [(4, row), (4, row[:8])],            # truncated row payload
        [(4, row), (0, b"")],                # non-positive row dimension
        [(4, row), (3, row[:12])],           # inconsistent row dimension
    ]
    for rows in cases:
        _write(p, rows)
        with pytest.raises(knng.FormatError):
            knng.read_vecs(p, "f32")
    with open(p, "wb") as f:
        f.write(struct.pack("<i", 4) + row + b"\x01\x02")  # truncated dimension field
    with pytest.raises(knng.FormatError):
        knng.vecs_shape(p, "f32")
    # an empty file is an empty dataset
    open(p, "wb").close()
    assert knng.vecs_shape(p, "f32") == (0, 0)
