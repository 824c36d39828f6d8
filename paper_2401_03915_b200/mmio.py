"""Matrix Market / vector files (src/sparsemat.py:201-372) on the native reader.

``read_matrix_market`` / ``load_matrix_market`` parse with libtls_b200's multithreaded
``tls_mm_parse`` / ``tls_mm_load`` (same dialect, validation order, error texts and line numbers
as the reference: ``MatrixMarketError(lineno, message)``) and return a ``SparseMat`` whose CSR is
the reference's canonical form; ``save_matrix_market`` writes through ``tls_mm_write`` (%.17g).
Parsing is host work (no GPU needed); the matrix reaches the device on its first SpMV / setup.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import scipy.sparse as sp

from . import _lib
from .sparsemat import SparseMat


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input; the message names the offending line (src/sparsemat.py:20-25)."""

    def __init__(self, lineno, message):
        super().__init__(f"line {lineno}: {message}")
        self.lineno = lineno


def _take(rc, h):
    lib = _lib.load()
    try:
        nr, nc, nnz, sym, eline = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32(), C.c_int64()
        msg = C.c_char_p()
        lib.tls_mm_info(h, C.byref(nr), C.byref(nc), C.byref(nnz), C.byref(sym), C.byref(eline), C.byref(msg))
        if rc == _lib.TLS_ERR_FORMAT:
            raise MatrixMarketError(int(eline.value), msg.value.decode("utf-8", "replace"))
        if rc == _lib.TLS_ERR_IO:
            raise OSError(msg.value.decode("utf-8", "replace"))
        if rc != _lib.TLS_OK:
            raise RuntimeError(f"tls_mm_parse failed ({rc})")
        n, m, z = int(nr.value), int(nc.value), int(nnz.value)
        indptr = np.zeros(n + 1, dtype=np.int64)
        indices = np.zeros(max(z, 1), dtype=np.int32)
        data = np.zeros(max(z, 1), dtype=np.float64)
        lib.tls_mm_export(h, _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(data))
        csr = sp.csr_matrix((data[:z], indices[:z], indptr), shape=(n, m))
        return SparseMat._canonical(csr, symmetric=bool(sym.value))
    finally:
        lib.tls_mm_free(h)


def read_matrix_market(text, nthreads=0):
    """Parse Matrix Market text into a SparseMat (src/sparsemat.py:227-321)."""
    raw = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    rc = _lib.load().tls_mm_parse(raw, len(raw), int(nthreads), C.byref(h))
    return _take(rc, h)


def load_matrix_market(path, nthreads=0):
    """Read a Matrix Market file natively (src/sparsemat.py:335-337)."""
    h = C.c_void_p()
    rc = _lib.load().tls_mm_load(os.fsencode(path), int(nthreads), C.byref(h))
    return _take(rc, h)


def write_matrix_market(matrix):
    """General coordinate text with 17 significant digits (src/sparsemat.py:323-332)."""
    csr = matrix.scipy()
    out = ["%%MatrixMarket matrix coordinate real general", f"{matrix.nrows} {matrix.ncols} {matrix.nnz}"]
    rows = np.repeat(np.arange(matrix.nrows), np.diff(csr.indptr))
    out.extend(f"{i + 1} {j + 1} {v:.17g}" for i, j, v in zip(rows.tolist(), csr.indices.tolist(), csr.data.tolist()))
    return "\n".join(out) + "\n"


def save_matrix_market(path, matrix, nthreads=0):
    """Write ``write_matrix_market(matrix)`` to ``path`` on all host threads."""
    csr = matrix.scipy()
    indptr = np.ascontiguousarray(csr.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(csr.indices, dtype=np.int32)
    data = np.ascontiguousarray(csr.data, dtype=np.float64)
    rc = _lib.load().tls_mm_write(os.fsencode(path), matrix.nrows, matrix.ncols, _lib.ptr(indptr),
                                  _lib.ptr(indices), _lib.ptr(data), int(nthreads))
    if rc != _lib.TLS_OK:
        raise OSError(f"cannot write {path}")


def _parse_float(tok, lineno):
    try:
        val = float(tok)
    except ValueError:
        raise MatrixMarketError(lineno, f"expected a real value, got {tok!r}") from None
    if not np.isfinite(val):
        raise MatrixMarketError(lineno, f"non-finite value {tok!r}")
    return val


def read_vector(text):
    """Matrix Market array text or one value per line (src/sparsemat.py:345-357)."""
    stripped = text.lstrip()
    if stripped.startswith("%%MatrixMarket"):
        mat = read_matrix_market(text)
        if mat.ncols != 1:
            raise ValueError(f"expected a single-column vector, got {mat.ncols} columns")
        return mat.scipy().toarray().ravel()
    vals = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("%"):
            continue
        toks = line.split()
        try:  # fast path: the whole line at once; the reference's per-token errors otherwise
            v = np.array(toks, dtype=np.float64)
            if np.isfinite(v).all():
                vals.append(v)
                continue
        except ValueError:
            pass
        vals.append(np.array([_parse_float(t, lineno) for t in toks]))
    return np.concatenate(vals) if vals else np.zeros(0)


def write_vector(vec):
    vec = np.asarray(vec, dtype=np.float64)
    return "\n".join(f"{v:.17g}" for v in vec.tolist()) + "\n"


def load_vector(path):
    with open(path, "r") as fh:
        return read_vector(fh.read())


def save_vector(path, vec):
    with open(path, "w") as fh:
        fh.write(write_vector(vec))
