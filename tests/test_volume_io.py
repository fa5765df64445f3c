"""ZNNV volume files (volume_io.hpp:15-86) written and read by the C-ABI
(znn_volume_write / znn_volume_read; CPU only, no device needed): the byte
layout is the reference's ("ZNNV", u32 version 1, u32 nx, ny, nz, float32
x-major, little-endian) and malformed files fail with status 1 like the
reference's require() (structural_error)."""
import struct

import numpy as np
import pytest


def test_round_trip_and_byte_layout(tmp_path):
    from paper_1510_06706_b200 import read_volume, write_volume
    rng = np.random.default_rng(0)
    v = rng.uniform(-1, 1, size=(3, 4, 5)).astype(np.float32)
    p = str(tmp_path / "v.znnv")
    write_volume(p, v)
    raw = open(p, "rb").read()
    assert raw[:4] == b"ZNNV"
    assert struct.unpack("<4I", raw[4:20]) == (1, 3, 4, 5)
    assert len(raw) == 20 + 4 * v.size
    assert np.array_equal(np.frombuffer(raw[20:], dtype="<f4").reshape(3, 4, 5), v)
    assert np.array_equal(read_volume(p), v)


def test_reads_a_reference_layout_file(tmp_path):
    """A file assembled byte by byte from volume_io.hpp's write_volume."""
    from paper_1510_06706_b200 import read_volume
    vals = np.arange(2 * 1 * 3, dtype=np.float32) * 0.5 - 1
    p = tmp_path / "r.znnv"
    p.write_bytes(b"ZNNV" + struct.pack("<4I", 1, 2, 1, 3) + vals.astype("<f4").tobytes())
    assert np.array_equal(read_volume(str(p)), vals.reshape(2, 1, 3))


@pytest.mark.parametrize("blob,msg", [
    (b"ZNNX" + struct.pack("<4I", 1, 1, 1, 1) + b"\0" * 4, "bad magic"),
    (b"ZNNV" + struct.pack("<4I", 2, 1, 1, 1) + b"\0" * 4, "unsupported version"),
    (b"ZNNV" + struct.pack("<4I", 1, 0, 1, 1), "non-positive dims"),
    (b"ZNNV" + struct.pack("<4I", 1, 2, 2, 2) + b"\0" * 8, "truncated"),
])
def test_malformed_files_are_structural_errors(tmp_path, blob, msg):
    from paper_1510_06706_b200 import ShapeError, read_volume
    p = tmp_path / "bad.znnv"
    p.write_bytes(blob)
    with pytest.raises(ShapeError) as e:
        read_volume(str(p))
    assert msg in str(e.value)
