"""DMAT interchange files (reference: include/randsvd/dmat.hpp:10-19, src/dmat.cpp:17-99):
"DMAT1\\n", rows and cols as u64 little-endian, then rows*cols binary64 little-endian values
in row-major order. Host read/write mirror the reference's checks and IoError byte
offsets; ``load_dmat_device`` streams a file's row range into HBM through the library's
pinned double-buffered loader (rsvd_b200_load_dmat_device)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .rsvd import Error, Solver, default_solver

MAGIC = b"DMAT1\n"


class IoError(Error):
    """randsvd::IoError (errors.hpp): path and the failing byte offset."""

    def __init__(self, msg: str, path: str = "", offset: int = 0):
        super().__init__(msg)
        self.path = path
        self.offset = offset


def _header(path: str):
    with open(path, "rb") as f:
        magic = f.read(6)
        if magic != MAGIC:
            raise IoError(f"bad DMAT magic in {path} at byte offset 0", path, 0)
        hdr = f.read(16)
        if len(hdr) != 16:
            raise IoError(f"truncated DMAT header in {path} at byte offset {6 + len(hdr)}", path,
                          6 + len(hdr))
    rows, cols = int.from_bytes(hdr[:8], "little"), int.from_bytes(hdr[8:], "little")
    if rows == 0 or cols == 0 or rows > 2**32 or cols > 2**32:
        raise IoError(f"implausible DMAT dimensions {rows}x{cols} in {path}", path, 6)
    return rows, cols


def read_dmat(path: str) -> np.ndarray:
    """randsvd::read_dmat (dmat.cpp:34-87)."""
    if not os.path.exists(path):
        raise IoError(f"cannot open {path}", path, 0)
    rows, cols = _header(path)
    size = os.path.getsize(path)
    need = 22 + rows * cols * 8
    if size < need:
        raise IoError(f"truncated DMAT payload in {path} at byte offset {size} (expected {need} "
                      "bytes total)", path, size)
    if size > need:
        raise IoError(f"trailing bytes in {path} after byte offset {need}", path, need)
    return np.fromfile(path, dtype="<f8", count=rows * cols, offset=22).reshape(rows, cols)


def write_dmat(path: str, m) -> None:
    """randsvd::write_dmat (dmat.cpp:89-99)."""
    m = np.ascontiguousarray(m, dtype="<f8")
    if m.ndim == 1:
        m = m.reshape(-1, 1)
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(int(m.shape[0]).to_bytes(8, "little"))
        f.write(int(m.shape[1]).to_bytes(8, "little"))
        f.write(m.tobytes())


def load_dmat_device(path: str, row0: int = 0, nrows: int | None = None,
                     solver: Solver | None = None):
    """Rows [row0, row0 + nrows) of a DMAT file as a CUDA float64 tensor (a rank's shard),
    streamed through pinned staging buffers straight into HBM."""
    import torch
    s = solver or default_solver()
    lib = _lib.load()
    r, c = C.c_uint64(0), C.c_uint64(0)
    if lib.rsvd_b200_dmat_shape(path.encode(), C.byref(r), C.byref(c)) != 0:
        raise IoError(lib.rsvd_b200_dmat_last_error().decode(), path)
    rows, cols = r.value, c.value
    nrows = rows - row0 if nrows is None else nrows
    ld = cols + (cols & 1)
    out = torch.empty((nrows, ld), dtype=torch.float64, device=f"cuda:{s.device}")
    s.wait_for_torch(out.device)
    st = lib.rsvd_b200_load_dmat_device(s.h, path.encode(), row0, nrows,
                                        C.cast(out.data_ptr(), C.POINTER(C.c_double)), ld)
    if st != 0:
        raise IoError(lib.rsvd_b200_dmat_last_error().decode(), path)
    return out[:, :cols]
