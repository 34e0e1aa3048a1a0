"""On-disk formats of the reference (kronglm::io, proj/src/io.cpp:13-212).

* Array files (``.glam``, io.cpp:91-149): the 4-byte magic ``GLAM``, u16
  version (1, io.hpp:12), u16 ndim, ndim u64 extents, then the column-major
  FP64 payload; every integer and double little-endian.
* Matrix CSV (io.cpp:151-212): one row per line, comma separated, numbers in
  ``std::from_chars`` syntax, written with ``%.17g``.

Errors mirror the reference messages (``std::runtime_error`` -> RuntimeError).
"""
from __future__ import annotations

import os
import re
import struct

import numpy as np

MAGIC = b"GLAM"
ARRAY_FILE_VERSION = 1

# std::from_chars(double) general format: no leading '+' or blanks
_NUM = re.compile(r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)",
                  re.IGNORECASE)


def write_array(path, array) -> None:
    """io::write_array (io.cpp:91-110); `array` is an n-d array in column-major order."""
    a = np.asarray(array, dtype=np.float64)
    dims = a.shape if a.ndim > 0 else (1,)
    buf = bytearray(MAGIC)
    buf += struct.pack("<HH", ARRAY_FILE_VERSION, len(dims))
    for e in dims:
        buf += struct.pack("<Q", int(e))
    buf += np.asfortranarray(a).ravel(order="F").astype("<f8").tobytes()
    try:
        with open(path, "wb") as f:
            f.write(buf)
    except OSError:
        raise RuntimeError("cannot write " + str(path)) from None


def read_array(path) -> np.ndarray:
    """io::read_array (io.cpp:112-149): a Fortran-ordered float64 array."""
    name = str(path)
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise RuntimeError("cannot open " + name) from None
    pos = 0

    def need(k):
        if len(data) - pos < k:
            raise RuntimeError(name + ": truncated array file")

    need(4)
    if data[:4] != MAGIC:
        raise RuntimeError(name + ": not an array file (bad magic)")
    pos = 4
    need(2)
    (version,) = struct.unpack_from("<H", data, pos)
    pos += 2
    if version != ARRAY_FILE_VERSION:
        raise RuntimeError(f"{name}: unsupported array file version {version}")
    need(2)
    (ndim,) = struct.unpack_from("<H", data, pos)
    pos += 2
    if ndim == 0:
        raise RuntimeError(name + ": array file with zero dimensions")
    ext = []
    for _ in range(ndim):
        need(8)
        ext.append(struct.unpack_from("<Q", data, pos)[0])
        pos += 8
    size = int(np.prod(ext))
    if len(data) - pos != size * 8:
        raise RuntimeError(name + ": payload size does not match the extents")
    flat = np.frombuffer(data, dtype="<f8", count=size, offset=pos).astype(np.float64)
    return np.asfortranarray(flat.reshape(ext, order="F"))


def read_csv_matrix(path) -> np.ndarray:
    """io::read_csv_matrix (io.cpp:151-194)."""
    name = str(path)
    try:
        with open(path, "r", newline="") as f:
            lines = f.read().split("\n")
    except OSError:
        raise RuntimeError("cannot open " + name) from None
    rows = []
    for line in lines:
        if line.endswith("\r"):
            line = line[:-1]
        if not line:
            continue
        row, pos, r = [], 0, len(rows) + 1
        while pos < len(line):
            m = _NUM.match(line, pos)
            if m is None or m.end() == pos:
                raise RuntimeError(f"{name}: malformed number in row {r}")
            row.append(float(m.group(0)))
            pos = m.end()
            if pos < len(line):
                if line[pos] != ",":
                    raise RuntimeError(f"{name}: expected ',' in row {r}")
                pos += 1
        if rows and len(row) != len(rows[0]):
            raise RuntimeError(name + ": ragged rows")
        rows.append(row)
    if not rows:
        raise RuntimeError(name + ": empty matrix file")
    return np.asfortranarray(np.array(rows, dtype=np.float64))


def write_csv_matrix(path, m) -> None:
    """io::write_csv_matrix (io.cpp:196-212): %.17g, one row per line."""
    m = np.asarray(m, dtype=np.float64)
    try:
        with open(path, "w", newline="") as f:
            for row in m:
                f.write(",".join("%.17g" % v for v in row) + "\n")
    except OSError:
        raise RuntimeError("cannot write " + str(path)) from None


def exists(path) -> bool:
    return os.path.exists(path)
