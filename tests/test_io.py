"""MCND file I/O (io.py): the reference's format and error behaviour
(matrix.py:122-151, tests test_matrix.py TestBinaryFormat), and the device loader."""

import struct

import numpy as np
import pytest

from paper_1811_08057_b200 import io as mio
from paper_1811_08057_b200.matrix import GENERATOR_KINDS, MatrixSpec, generate


def test_round_trip_bit_exact(tmp_path):
    for kind in GENERATOR_KINDS:
        a = generate(MatrixSpec(7, kind, seed=9))
        p = tmp_path / f"{kind}.mcnd"
        mio.write_matrix(a, p)
        assert mio.read_matrix(p).tobytes() == a.tobytes()


def test_smallest_file(tmp_path):
    p = tmp_path / "one.mcnd"
    mio.write_matrix(np.array([[2.5]]), p)
    assert p.stat().st_size == 30
    assert mio.read_matrix(p)[0, 0] == 2.5


def test_reference_reads_our_files_and_we_read_its(tmp_path):
    """Byte-identical to the reference's writer (header + LE payload)."""
    a = np.random.default_rng(3).standard_normal((5, 4))
    p = tmp_path / "x.mcnd"
    mio.write_matrix(a, p)
    raw = p.read_bytes()
    assert raw[:22] == struct.pack("<4sHQQ", b"MCND", 1, 5, 4)
    assert raw[22:] == a.astype("<f8").tobytes()


@pytest.mark.parametrize("payload,match", [
    (b"NOPE" + bytes(26), "magic"),
    (b"MC", "truncated"),
    (struct.pack("<4sHQQ", b"MCND", 99, 2, 2) + bytes(32), "version"),
    (struct.pack("<4sHQQ", b"MCND", 1, 0, 2), "zero"),
    (struct.pack("<4sHQQ", b"MCND", 1, 1 << 40, 1 << 40), "overflow"),
    (struct.pack("<4sHQQ", b"MCND", 1, 3, 3) + bytes(68), "truncated payload"),
])
def test_format_errors(tmp_path, payload, match):
    p = tmp_path / "bad.mcnd"
    p.write_bytes(payload)
    with pytest.raises(mio.FormatError, match=match):
        mio.read_matrix(p)


def test_nonfinite_payload_is_value_error(tmp_path):
    p = tmp_path / "nan.mcnd"
    p.write_bytes(struct.pack("<4sHQQ", b"MCND", 1, 1, 2) + np.array([1.0, np.nan]).tobytes())
    with pytest.raises(ValueError, match="finite"):
        mio.read_matrix(p)


@pytest.mark.gpu
def test_read_matrix_device(tmp_path):
    import torch

    a = np.random.default_rng(1).uniform(-1, 1, (1500, 1300))
    p = tmp_path / "d.mcnd"
    mio.write_matrix(a, p)
    t = mio.read_matrix_device(p, chunk_bytes=1 << 20)  # many chunks through the two pinned buffers
    assert t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
    assert t.cpu().numpy().tobytes() == a.tobytes()
    raw = bytearray(p.read_bytes())
    raw[22 + 8 * 17:22 + 8 * 18] = np.array([np.inf]).tobytes()
    p.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="finite"):
        mio.read_matrix_device(p)
    p.write_bytes(bytes(raw[:-3]))
    with pytest.raises(mio.FormatError, match="truncated payload"):
        mio.read_matrix_device(p)
