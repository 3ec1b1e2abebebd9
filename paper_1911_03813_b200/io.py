"""MOMV binary observation files straight into HBM.

Format (reference pkg/src/momentcp/io.py:22-23,75-99): b"MOMV", u32 version 1, u64 n, u64 p,
then n*p little-endian float64 in column-major order -- i.e. observation-major, each
observation's n values contiguous, which is exactly the device layout.  The reader memory-maps
the payload and the C ABI copies it row-pitched into HBM (finiteness checked on the device), so
no float64 n x p host copy is ever made (the reference's ObservationSet upcast costs 20.5 s at
config 3).  ``rows=(lo, hi)`` maps only a row shard -- one rank's part of a multi-GPU set.
Errors follow the reference: ParseError for a bad/truncated header or payload, ValueError for
non-finite data.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .dense import ObservationSet

MAGIC = b"MOMV"
BINARY_VERSION = 1
HEADER_BYTES = 24


class ParseError(ValueError):
    """Malformed observation file (reference io.py ParseError)."""


def _header(path: str) -> tuple[int, int]:
    with open(path, "rb") as fh:
        header = fh.read(HEADER_BYTES)
    if len(header) < HEADER_BYTES or header[:4] != MAGIC:
        raise ParseError(f"{path}: bad or truncated header (byte offset 0)")
    version, n, p = struct.unpack("<IQQ", header[4:24])
    if version != BINARY_VERSION:
        raise ParseError(f"{path}: unsupported version {version} (byte offset 4)")
    have = (os.path.getsize(path) - HEADER_BYTES) // 8
    if have < n * p:
        raise ParseError(f"{path}: expected {n * p} values, got {have} "
                         f"(byte offset {HEADER_BYTES + 8 * have})")
    return int(n), int(p)


def read_observations_binary(path: str, *, rows: tuple[int, int] | None = None,
                             device: int | None = None) -> ObservationSet:
    """Observation set backed by the file's payload (memory-mapped, uploaded on first use).

    With ``rows=(lo, hi)`` only observations lo..hi-1 are mapped and the uniform weight stays
    1/p of the whole file (a row shard of the full set).
    """
    n, p = _header(path)
    lo, hi = (0, p) if rows is None else (int(rows[0]), int(rows[1]))
    if not 0 <= lo < hi <= p:
        raise ValueError(f"row range {rows} outside [0, {p})")
    mm = np.memmap(path, dtype="<f8", mode="r", offset=HEADER_BYTES + 8 * n * lo,
                   shape=(hi - lo, n))
    # read-time finiteness, like the reference reader (io.py:89-91): chunked so a large mapped
    # payload is streamed once, never copied whole
    step = max(1, (1 << 24) // max(n, 1))
    for a in range(0, hi - lo, step):
        if not np.isfinite(mm[a:a + step]).all():
            raise ValueError(f"{path}: non-finite value in payload")
    return ObservationSet.from_obs_major_host(mm, p_total=p, device=device)


def write_observations_binary(path: str, obs: ObservationSet) -> None:
    """Write the MOMV format (reference io.py:95-99)."""
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<IQQ", BINARY_VERSION, obs.n, obs.p))
        np.ascontiguousarray(obs.V.ravel(order="F"), dtype="<f8").tofile(fh)
