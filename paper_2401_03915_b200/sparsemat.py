"""SparseMat mirror (src/sparsemat.py:28-155) whose ``matvec`` runs the sm_100a CSR SpMV.

Host storage is the same canonical scipy CSR as the reference (fp64, sorted,
duplicate-free columns, read-only buffers, verified symmetry flag); the device
copy (int32 indices) lives in a libtls_b200 handle created on first use.
Reference ``SparseMat`` objects are accepted anywhere through ``as_sparsemat``.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import device as D
from .partition import Graph, symmetrized_graph as _sym_graph

DENSE_GUARD = 5000  # src/sparsemat.py:17 (host densification only; GPU setup has no guard)


class SparseMat:
    def __init__(self, csr, symmetric=False):
        if not sp.issparse(csr):
            raise TypeError("expected a scipy sparse matrix")
        csr = csr.tocsr().astype(np.float64)
        csr.sum_duplicates()
        csr.sort_indices()
        if not np.all(np.isfinite(csr.data)):
            raise ValueError("matrix entries must be finite")
        if symmetric:
            if csr.shape[0] != csr.shape[1]:
                raise ValueError("symmetric flag requires a square matrix")
            if (csr != csr.T).nnz != 0:
                raise ValueError("symmetric flag set but values are not symmetric")
        self._csr = csr
        self.symmetric = bool(symmetric)
        for arr in (csr.data, csr.indices, csr.indptr):
            arr.flags.writeable = False
        self._handle = None

    @classmethod
    def _canonical(cls, csr, symmetric=False):
        """Wrap a CSR that is already canonical (sorted, duplicate-free, finite; symmetric by
        construction when flagged) -- the native Matrix Market reader's output."""
        self = cls.__new__(cls)
        self._csr = csr
        self.symmetric = bool(symmetric)
        for arr in (csr.data, csr.indices, csr.indptr):
            arr.flags.writeable = False
        self._handle = None
        return self

    @classmethod
    def from_coo(cls, nrows, ncols, rows, cols, vals, symmetric=False):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if rows.size and (rows.min() < 0 or rows.max() >= nrows):
            raise ValueError("row index out of range")
        if cols.size and (cols.min() < 0 or cols.max() >= ncols):
            raise ValueError("column index out of range")
        return cls(sp.coo_matrix((vals, (rows, cols)), shape=(nrows, ncols)).tocsr(), symmetric=symmetric)

    @classmethod
    def from_dense(cls, arr, symmetric=False):
        return cls(sp.csr_matrix(np.asarray(arr, dtype=np.float64)), symmetric=symmetric)

    @classmethod
    def identity(cls, n):
        return cls(sp.identity(n, format="csr"), symmetric=True)

    @property
    def nrows(self):
        return self._csr.shape[0]

    @property
    def ncols(self):
        return self._csr.shape[1]

    @property
    def shape(self):
        return self._csr.shape

    @property
    def nnz(self):
        return self._csr.nnz

    @property
    def indptr(self):
        return self._csr.indptr

    @property
    def indices(self):
        return self._csr.indices

    @property
    def data(self):
        return self._csr.data

    def scipy(self):
        return self._csr

    def value(self, i, j):
        if not (0 <= i < self.nrows and 0 <= j < self.ncols):
            raise IndexError("index out of range")
        lo, hi = self._csr.indptr[i], self._csr.indptr[i + 1]
        cols = self._csr.indices[lo:hi]
        k = np.searchsorted(cols, j)
        return float(self._csr.data[lo + k]) if k < cols.size and cols[k] == j else 0.0

    # -- device -----------------------------------------------------------------
    def device_handle(self, device=None):
        """Matrix-only handle (SpMV and unpreconditioned Krylov)."""
        if self.nrows != self.ncols:
            raise ValueError("device operators require a square matrix")
        if self._handle is None:
            h = D.Handle(device)
            h.upload_matrix(self._csr, self.symmetric)
            self._handle = h
        return self._handle

    def matvec(self, v):
        """y = A v on the GPU (K1; replaces src/sparsemat.py:125-129)."""
        h = self.device_handle()
        x, back = D.to_device(v, self.ncols, h.device)
        torch = D._torch()
        y = torch.empty_like(x)
        h.check(h.lib.tls_spmv(h.ctx, D._lib.ptr(x), D._lib.ptr(y), D.stream_ptr()))
        return back(y)

    def __matmul__(self, v):
        return self.matvec(v)

    def transpose(self):
        return SparseMat(self._csr.T.tocsr(), symmetric=self.symmetric)

    def to_dense(self):
        if self.nrows > DENSE_GUARD:
            raise ValueError(f"refusing to densify a matrix with {self.nrows} rows (guard is {DENSE_GUARD})")
        return self._csr.toarray()

    def is_numerically_symmetric(self):
        return self.nrows == self.ncols and (self._csr != self._csr.T).nnz == 0

    def as_symmetric(self):
        return SparseMat(self._csr, symmetric=True)

    def __repr__(self):
        sym = ", symmetric" if self.symmetric else ""
        return f"SparseMat({self.nrows}x{self.ncols}, nnz={self.nnz}{sym})"


def as_sparsemat(matrix):
    """Accept our SparseMat, the reference's SparseMat (duck-typed) or a scipy matrix."""
    if isinstance(matrix, SparseMat):
        return matrix
    if hasattr(matrix, "scipy") and hasattr(matrix, "symmetric"):
        cached = getattr(matrix, "_b200_mirror", None)
        if cached is None:
            cached = SparseMat(matrix.scipy(), symmetric=matrix.symmetric)
            try:
                matrix._b200_mirror = cached
            except AttributeError:
                pass
        return cached
    if sp.issparse(matrix):
        return SparseMat(matrix)
    raise TypeError("expected a SparseMat or a scipy sparse matrix")


def symmetrized_graph(matrix):
    """Adjacency of the symmetrised pattern (src/sparsemat.py:180-195)."""
    m = as_sparsemat(matrix)
    if m.nrows != m.ncols:
        raise ValueError("sparsity graph requires a square matrix")
    return _sym_graph(m.scipy(), symmetric=m.symmetric)


__all__ = ["SparseMat", "Graph", "symmetrized_graph", "as_sparsemat", "DENSE_GUARD"]
