"""MCND binary matrix files, and a loader that streams them straight to the GPU.

File format (the reference's, matrix.py:15-17 and matrix.py:122-151): a
little-endian header ``<4sHQQ`` = magic ``b"MCND"``, format version 1, rows,
columns; then rows*columns little-endian float64 in row-major order.  Errors
follow the reference: ``FormatError`` (a ``ValueError``) for a bad magic or
version, a truncated header or payload, a zero or absurd dimension; the
payload then goes through the same checks as ``as_matrix`` (finite entries).

``read_matrix_device`` is SURVEY.md §8(f) rank 1: large inputs (C5 is 8.6 GB)
are read in chunks into two pinned host buffers and copied to the device
asynchronously, so the disk read of chunk i+1 overlaps the H2D copy of chunk i;
the finiteness check runs on the device.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .matrix import as_matrix

MAGIC = b"MCND"
FORMAT_VERSION = 1
HEADER = struct.Struct("<4sHQQ")
_MAX_PAYLOAD = 1 << 40  # sanity bound on rows*cols*8


class FormatError(ValueError):
    """Malformed matrix file (bad magic or version, truncation, bad dimensions)."""


def write_matrix(m, path) -> None:
    """Write ``m`` (validated like ``as_matrix``) in the MCND format; bit-exact round trip."""
    a = as_matrix(m)
    with open(path, "wb") as f:
        f.write(HEADER.pack(MAGIC, FORMAT_VERSION, a.shape[0], a.shape[1]))
        f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def _header(f):
    raw = f.read(HEADER.size)
    if len(raw) < HEADER.size:
        raise FormatError("truncated header")
    magic, version, rows, cols = HEADER.unpack(raw)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}")
    if version != FORMAT_VERSION:
        raise FormatError(f"unsupported format version {version}")
    if rows == 0 or cols == 0:
        raise FormatError("zero dimension in header")
    if rows * cols * 8 > _MAX_PAYLOAD:
        raise FormatError(f"dimensions overflow the sanity bound: {rows}x{cols}")
    return rows, cols


def read_matrix(path) -> np.ndarray:
    """Host read (numpy), same validation as the reference."""
    with open(path, "rb") as f:
        rows, cols = _header(f)
        nbytes = rows * cols * 8
        payload = f.read(nbytes)
    if len(payload) < nbytes:
        raise FormatError(f"truncated payload: expected {nbytes} bytes, got {len(payload)}")
    return as_matrix(np.frombuffer(payload, dtype="<f8").reshape(rows, cols))


def read_matrix_device(path, device=None, chunk_bytes: int = 64 << 20, check_finite: bool = True):
    """Read an MCND file into a float64 CUDA tensor (C-contiguous), streaming the
    payload through two pinned buffers; ``check_finite`` runs the reference's
    finiteness check on the device (ValueError like ``as_matrix``)."""
    import torch

    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with open(path, "rb") as f:
        rows, cols = _header(f)
        nbytes = rows * cols * 8
        have = os.fstat(f.fileno()).st_size - HEADER.size
        if have < nbytes:
            raise FormatError(f"truncated payload: expected {nbytes} bytes, got {have}")
        out = torch.empty((rows, cols), dtype=torch.float64, device=dev)
        flat = out.view(-1)
        chunk = max(8, (int(chunk_bytes) // 8) * 8)
        bufs = [torch.empty(chunk // 8, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        used = [False, False]
        stream = torch.cuda.current_stream(dev)
        off = 0
        i = 0
        while off < nbytes:
            k = i & 1
            if used[k]:
                done[k].synchronize()  # the copy out of this buffer has finished
            take = min(chunk, nbytes - off)
            view = bufs[k].numpy().view(np.uint8)[:take]
            got = f.readinto(memoryview(view))
            if got != take:
                raise FormatError(f"truncated payload: expected {nbytes} bytes, got {off + (got or 0)}")
            flat[off // 8:(off + take) // 8].copy_(bufs[k][: take // 8], non_blocking=True)
            done[k].record(stream)
            used[k] = True
            off += take
            i += 1
        stream.synchronize()
    if np.dtype("<f8") != np.dtype(np.float64):  # big-endian host: not supported by the GPU path
        raise FormatError("big-endian hosts are not supported")
    if check_finite and not bool(torch.isfinite(out).all()):
        raise ValueError("matrix entries must be finite (no NaN/Inf)")
    return out


def write_matrix_csv(m, path) -> None:
    """matrix.py:154-160: one row per line, comma-separated repr() floats, no header."""
    a = as_matrix(m)
    with open(path, "w") as f:
        for row in a:
            f.write(",".join(repr(float(v)) for v in row))
            f.write("\n")


def read_matrix_csv(path) -> np.ndarray:
    """matrix.py:163-180: blank lines skipped; a bad token or a ragged row -> FormatError
    naming the line."""
    rows = []
    with open(path) as f:
        for line_no, line in enumerate(f, 1):
            line = line.strip()
            if not line:
                continue
            try:
                rows.append([float(tok) for tok in line.split(",")])
            except ValueError as exc:
                raise FormatError(f"line {line_no}: {exc}") from exc
    if not rows:
        raise FormatError("empty CSV matrix")
    width = len(rows[0])
    for line_no, row in enumerate(rows, 1):
        if len(row) != width:
            raise FormatError(f"line {line_no}: ragged row width {len(row)} != {width}")
    return as_matrix(rows)
