"""RLFMAT01 binary container and CSV matrix files (rlftn matrix_io.cpp:1-218).

Binary: the 8-byte magic "RLFMAT01", a one-byte dtype tag (0 float64,
1 complex128), rows and cols as little-endian u64, then the entries row by row
(matrix_io.cpp:44-59).  CSV: one row per line, tokens "a", "a+bi", "a-bi" or
"bi"; any imaginary token makes the whole matrix complex; CRLF and blank lines
are tolerated (matrix_io.cpp:84-193).  Errors carry the reference's messages
(as RuntimeError, the reference's std::runtime_error).
"""
from __future__ import annotations

import re
import struct

import numpy as np

MAGIC = b"RLFMAT01"
MAX_DIM = 1 << 24
MAX_ELEMS = 1 << 28


def save_matrix_binary(path: str, a) -> None:
    a = np.asarray(a)
    cplx = np.iscomplexobj(a)
    a = a.astype(np.complex128 if cplx else np.float64)
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError("cannot open for writing: " + path)
    with f:
        f.write(MAGIC)
        f.write(bytes([1 if cplx else 0]))
        f.write(struct.pack("<QQ", a.shape[0], a.shape[1]))
        f.write(np.ascontiguousarray(a).tobytes())


def _fmt_token(v) -> str:
    if isinstance(v, complex) or np.iscomplexobj(v):
        return "%.17g%+.17gi" % (v.real, v.imag)
    return "%.17g" % v


def save_matrix_csv(path: str, a) -> None:
    a = np.asarray(a)
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError("cannot open for writing: " + path)
    with f:
        for row in a:
            f.write(",".join(_fmt_token(x) for x in row) + "\n")


def load_matrix_binary(path: str) -> np.ndarray:
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError("cannot open for reading: " + path)
    with f:
        magic = f.read(8)
        if magic != MAGIC:
            raise RuntimeError(path + ": not a matrix container (bad magic)")
        hdr = f.read(17)
        if len(hdr) < 17 or hdr[0] > 1:
            raise RuntimeError(path + ": corrupt matrix header")
        tag = hdr[0]
        rows, cols = struct.unpack("<QQ", hdr[1:])
        if rows == 0 or cols == 0 or rows > MAX_DIM or cols > MAX_DIM or rows > MAX_ELEMS // cols:
            raise RuntimeError(path + ": unreasonable matrix dimensions")
        dt = np.complex128 if tag == 1 else np.float64
        count = rows * cols
        data = f.read(count * np.dtype(dt).itemsize)
        if len(data) < count * np.dtype(dt).itemsize:
            raise RuntimeError(path + ": truncated matrix data")
        return np.frombuffer(data, dtype=dt).reshape(rows, cols).copy()


_UNUM = r"(?:\d+\.?\d*(?:[eE][+-]?\d+)?|\.\d+(?:[eE][+-]?\d+)?|inf|infinity|nan)"
_NUM = r"[+-]?" + _UNUM


def _parse_token(tok: str, path: str, line: int):
    """Returns (value, is_imaginary_form)."""
    def bad():
        raise RuntimeError("%s:%d: bad matrix entry '%s'" % (path, line, tok))

    if not tok:
        bad()
    m = re.fullmatch(_NUM, tok, re.IGNORECASE)
    if m:
        return complex(float(tok), 0.0), False
    m = re.fullmatch("(" + _NUM + ")i", tok, re.IGNORECASE)
    if m:
        return complex(0.0, float(m.group(1))), True
    m = re.fullmatch("(" + _NUM + ")([+-]" + _UNUM + ")i", tok, re.IGNORECASE)
    if m:
        return complex(float(m.group(1)), float(m.group(2))), True
    bad()


def load_matrix_csv(path: str) -> np.ndarray:
    try:
        f = open(path, "r", newline="")
    except OSError:
        raise RuntimeError("cannot open for reading: " + path)
    data = []
    saw_imag = False
    with f:
        for lineno, line in enumerate(f.read().split("\n"), start=1):
            if line.endswith("\r"):
                line = line[:-1]
            if not line.strip(" \t"):
                continue
            row = []
            for tok in line.split(","):
                t = tok.strip(" \t")
                if not t:
                    raise RuntimeError("%s:%d: bad matrix entry '%s'" % (path, lineno, tok))
                v, im = _parse_token(t, path, lineno)
                saw_imag |= im
                row.append(v)
            if data and len(row) != len(data[0]):
                raise RuntimeError("%s:%d: inconsistent column count" % (path, lineno))
            data.append(row)
    if not data:
        raise RuntimeError(path + ": empty matrix file")
    a = np.array(data, dtype=np.complex128)
    return a if saw_imag else a.real.copy()


def load_matrix(path: str) -> np.ndarray:
    """Binary when the file starts with the magic, CSV otherwise."""
    try:
        with open(path, "rb") as f:
            head = f.read(8)
    except OSError:
        raise RuntimeError("cannot open for reading: " + path)
    return load_matrix_binary(path) if head == MAGIC else load_matrix_csv(path)
