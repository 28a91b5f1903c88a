"""PACTMAT / PACTSIG files: the explicit-matrix and measurement formats of the reference
(pkg/src/pactkit/forward.py:276-330).

One ASCII header line -- ``PACTMAT <domain> <rows> <cols>`` or ``PACTSIG <domain> <sensors>
<samples>`` -- then raw little-endian float64, row-major, complex values interleaved
(re, im).  Reading maps the payload straight into a NumPy array (``np.fromfile`` at the
header offset, no intermediate copy of the whole file), which matters for dense matrices
of many GB; a matrix read this way is an explicit operator (``DenseOperator``, cuBLAS GEMV on
the device -- SURVEY.md section 8 row f3).
"""

from __future__ import annotations

import numpy as np

from .measurement import MeasurementMatrix, SensorData

__all__ = ["read_matrix", "write_matrix", "read_signal", "write_signal"]

_MAX_HEADER = 256


def _header(path, tag: str):
    with open(path, "rb") as f:
        head = f.read(_MAX_HEADER)
    end = head.find(b"\n")
    if end < 0:
        raise ValueError(f"{path}: not a {tag} file")
    fields = head[:end].decode("ascii", errors="replace").split()
    if len(fields) != 4 or fields[0] != tag:
        raise ValueError(f"{path}: not a {tag} file")
    domain = fields[1]
    if domain not in ("time", "frequency"):
        raise ValueError(f"{path}: unknown domain {domain!r}")
    return domain, int(fields[2]), int(fields[3]), end + 1


def _payload(path, offset: int, count: int, cplx: bool) -> np.ndarray:
    n = count * (2 if cplx else 1)
    flat = np.fromfile(path, dtype="<f8", count=n, offset=offset)
    if flat.size != n:
        raise ValueError(f"{path}: truncated payload ({flat.size} of {n} values)")
    flat = flat.astype(np.float64, copy=False)
    return flat.view(np.complex128) if cplx else flat


def _write(path, header: str, values: np.ndarray):
    arr = np.ascontiguousarray(values)
    flat = arr.view(np.float64) if np.iscomplexobj(arr) else arr.astype(np.float64, copy=False)
    with open(path, "wb") as f:
        f.write(header.encode("ascii"))
        flat.astype("<f8", copy=False).tofile(f)


def write_matrix(K, path):
    """forward.py:296-299: header + dense entries (materialised for geometry-backed K)."""
    _write(path, f"PACTMAT {K.domain} {K.rows} {K.cols}\n", np.asarray(K.entries))


def read_matrix(path) -> MeasurementMatrix:
    """forward.py:302-311: an explicit MeasurementMatrix (no builder provenance)."""
    domain, rows, cols, off = _header(path, "PACTMAT")
    entries = _payload(path, off, rows * cols, domain == "frequency").reshape(rows, cols)
    return MeasurementMatrix(domain, entries)


def write_signal(y: SensorData, path):
    """forward.py:314-317."""
    _write(path, f"PACTSIG {y.domain} {y.sensors} {y.samples}\n", y.values)


def read_signal(path) -> SensorData:
    """forward.py:320-330."""
    domain, p, q, off = _header(path, "PACTSIG")
    return SensorData(domain, p, q, _payload(path, off, p * q, domain == "frequency"))
