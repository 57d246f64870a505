"""Binary CSR files: graphs of up to ~1e8 vertices / 2e9 entries
are written and read at disk speed and memory-mapped, instead of going through the
reference's text edge lists (specluster/graph.py:287-361), which take minutes at that size.

Layout (little endian, every array 64-byte aligned so np.memmap views need no copy):

    0   magic      8 bytes  b"SCCSR\\x00\\x01\\x00"
    8   n          int64
    16  nnz        int64
    24  flags      uint32   bit 0: weights present, bit 1: degrees are unit row counts
    28  col_bytes  uint32   4 (int32 columns) or 8 (int64, n >= 2^31)
    32  off_rp     int64    byte offset of row_offsets  int64[n + 1]
    40  off_col    int64    byte offset of col_indices  int{32,64}[nnz]
    48  off_w      int64    byte offset of weights      float64[nnz]  (0 if absent)
    56  off_deg    int64    byte offset of degrees      float64[n]
    64  data ...

Degrees are stored verbatim (never recomputed on load: recomputing changes their rounding
for weighted graphs).
"""

from __future__ import annotations

import os

import numpy as np

from .errors import GraphFormatError
from .graph import Graph

MAGIC = b"SCCSR\x00\x01\x00"
_HDR = np.dtype([("magic", "S8"), ("n", "<i8"), ("nnz", "<i8"), ("flags", "<u4"),
                 ("col_bytes", "<u4"), ("off_rp", "<i8"), ("off_col", "<i8"),
                 ("off_w", "<i8"), ("off_deg", "<i8")])
assert _HDR.itemsize == 64
F_WEIGHTS = 1
F_UNIT_DEG = 2


def _align(x: int) -> int:
    return (x + 63) // 64 * 64


def save_csr(g: Graph, path) -> None:
    """Write ``g`` (any object with the Graph fields) to ``path``."""
    n = int(g.n)
    rp = np.ascontiguousarray(g.row_offsets, dtype="<i8")
    nnz = int(rp[-1])
    col = np.ascontiguousarray(g.col_indices)
    col_bytes = 4 if col.dtype.itemsize <= 4 and n < 2**31 else 8
    col = col.astype("<i4" if col_bytes == 4 else "<i8", copy=False)
    w = None if g.weights is None else np.ascontiguousarray(g.weights, dtype="<f8")
    deg = np.ascontiguousarray(g.degrees, dtype="<f8")
    if rp.shape != (n + 1,) or col.shape != (nnz,) or deg.shape != (n,) or (
            w is not None and w.shape != (nnz,)):
        raise GraphFormatError("inconsistent CSR array lengths")
    hdr = np.zeros(1, dtype=_HDR)
    off = 64
    hdr["magic"], hdr["n"], hdr["nnz"] = MAGIC, n, nnz
    hdr["flags"] = (F_WEIGHTS if w is not None else 0)
    hdr["col_bytes"] = col_bytes
    hdr["off_rp"] = off
    off = _align(off + rp.nbytes)
    hdr["off_col"] = off
    off = _align(off + col.nbytes)
    if w is not None:
        hdr["off_w"] = off
        off = _align(off + w.nbytes)
    hdr["off_deg"] = off
    tmp = f"{path}.tmp"
    with open(tmp, "wb") as fh:
        fh.write(hdr.tobytes())
        for arr, key in ((rp, "off_rp"), (col, "off_col"), (w, "off_w"), (deg, "off_deg")):
            if arr is None:
                continue
            fh.seek(int(hdr[key][0]))
            arr.tofile(fh)
    os.replace(tmp, path)


def load_csr(path, *, mmap: bool = True) -> Graph:
    """Read a file written by ``save_csr``; with ``mmap`` the arrays are read-only views of
    the file (pages are read on first touch, e.g. by the upload to the GPU)."""
    size = os.path.getsize(path)
    if size < 64:
        raise GraphFormatError(f"{path}: too short for a CSR header")
    hdr = np.fromfile(path, dtype=_HDR, count=1)[0]
    if bytes(hdr["magic"]) != MAGIC.rstrip(b"\x00") and bytes(hdr["magic"]) != MAGIC:
        raise GraphFormatError(f"{path}: not a binary CSR file (bad magic)")
    n, nnz, cb = int(hdr["n"]), int(hdr["nnz"]), int(hdr["col_bytes"])
    if n < 1 or nnz < 0 or cb not in (4, 8):
        raise GraphFormatError(f"{path}: bad header (n={n}, nnz={nnz}, col_bytes={cb})")
    spans = [("off_rp", 8 * (n + 1)), ("off_col", cb * nnz), ("off_deg", 8 * n)]
    if hdr["flags"] & F_WEIGHTS:
        spans.append(("off_w", 8 * nnz))
    for key, nb in spans:
        if int(hdr[key]) < 64 or int(hdr[key]) + nb > size:
            raise GraphFormatError(f"{path}: truncated ({key})")

    def arr(key, dt, count):
        o = int(hdr[key])
        if mmap:
            return np.memmap(path, dtype=dt, mode="r", offset=o, shape=(count,))
        with open(path, "rb") as fh:
            fh.seek(o)
            return np.fromfile(fh, dtype=dt, count=count)

    rp = arr("off_rp", "<i8", n + 1)
    if rp[0] != 0 or rp[-1] != nnz:
        raise GraphFormatError(f"{path}: row_offsets do not span [0, nnz]")
    col = arr("off_col", "<i4" if cb == 4 else "<i8", nnz)
    w = arr("off_w", "<f8", nnz) if hdr["flags"] & F_WEIGHTS else None
    deg = arr("off_deg", "<f8", n)
    return Graph(n=n, row_offsets=rp, col_indices=col, weights=w, degrees=deg)
