"""SWS1 snapshot format (io.hpp:22-241): little-endian header, z/h/qx/qy blocks,
optional 12-byte trailing records (1 = dt_next, 2 = step_index as f64)."""
from __future__ import annotations

import struct

import numpy as np

from .stepper import FieldSet, GridSpec, IoError

HEADER = 16 + 5 * 8
TAG_DT_NEXT = 1
TAG_STEP_INDEX = 2


def snapshot_bytes(fs: FieldSet, g: float, dt_next: float | None = None, step_index: int | None = None) -> bytes:
    s = fs.spec
    out = [b"SWS1", struct.pack("<III", 1, s.nx, s.ny), struct.pack("<5d", s.dx, s.dy, fs.t, g, 0.0)]
    for a in (fs.z, fs.h, fs.qx, fs.qy):
        out.append(np.ascontiguousarray(a, dtype="<f8").tobytes())
    if dt_next is not None:
        out.append(struct.pack("<Id", TAG_DT_NEXT, dt_next))
    if step_index is not None:
        out.append(struct.pack("<Id", TAG_STEP_INDEX, float(step_index)))
    return b"".join(out)


def parse_snapshot(b: bytes):
    if len(b) < HEADER:
        raise IoError(f"snapshot: truncated header, need {HEADER} bytes, have {len(b)}")
    if b[:4] != b"SWS1":
        raise IoError("snapshot: bad magic at offset 0")
    version, nx, ny = struct.unpack_from("<III", b, 4)
    if version != 1:
        raise IoError(f"snapshot: unsupported version {version} at offset 4")
    dx, dy, t, g, _ = struct.unpack_from("<5d", b, 16)
    n = nx * ny
    end = HEADER + 32 * n
    if len(b) < end:
        raise IoError(f"snapshot: truncated payload, expected {end} bytes, have {len(b)}")
    blocks = [np.frombuffer(b, dtype="<f8", count=n, offset=HEADER + 8 * n * k).reshape(ny, nx).copy() for k in range(4)]
    fs = FieldSet(GridSpec(nx, ny, dx, dy), *blocks, t=t)
    extras = {}
    off = end
    while off < len(b):
        if len(b) - off < 12:
            raise IoError(f"snapshot: truncated trailing record at offset {off}")
        tag, val = struct.unpack_from("<Id", b, off)
        if tag == TAG_DT_NEXT:
            extras["dt_next"] = val
        elif tag == TAG_STEP_INDEX:
            extras["step_index"] = int(val)
        off += 12
    return fs, g, extras
