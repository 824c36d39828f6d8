"""pcg / gmres mirror of src/krylov.py; the whole loop runs on the device.

One C-ABI call per solve (``tls_pcg`` / ``tls_gmres``): the iteration is a
replayed CUDA graph (25 PCG iterations or one GMRES cycle per replay) with a
device-side stopping flag, so the host syncs once per replay, not per kernel.
Semantics follow the reference exactly: x0 = 0, stop on ||r||/||b|| <= tol,
PCG residual replacement every 25 iterations, BreakdownError on p.Ap <= 0,
GMRES hard cap 1000, happy breakdown, x = M^{-1} V y.  ``gmres(restart=m)``
(build extension) runs GMRES(m) cycles on the true residual with the
tolerance rescaled to the original ||b||.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np
from scipy.linalg import eigvalsh_tridiagonal

from . import _lib
from . import device as D
from .errors import BreakdownError
from .sparsemat import as_sparsemat

GMRES_MAXIT_CAP = 1000  # src/krylov.py:18
REORTH_TOL = 1e-8       # src/krylov.py:19 (CGS2 always re-orthogonalises)


class _Callback:
    """ctypes trampoline for ``callback``: an exception raised by the user's callback cannot cross
    the C frame (CPython would print and drop it), so it is saved, the C loop is told to stop
    (return 1 -> TLS_ERR_CALLBACK) and ``reraise`` raises it after the call returns -- the
    reference lets it propagate out of pcg / gmres (src/krylov.py:92-93, 182-183)."""

    def __init__(self, fn, with_x, n):
        self.fn, self.with_x, self.n, self.exc = fn, with_x, n, None
        self.c = _lib.ITER_CB(self._call) if fn is not None else _lib.ITER_CB()

    def _call(self, _user, it, xp):
        try:
            x = np.ctypeslib.as_array(xp, (self.n,)).copy() if self.with_x else None
            self.fn(int(it), x)
            return 0
        except BaseException as exc:  # noqa: BLE001 -- re-raised by reraise()
            self.exc = exc
            return 1

    def reraise(self, rc):
        if self.exc is not None:
            exc, self.exc = self.exc, None
            raise exc
        if rc == _lib.TLS_ERR_CALLBACK:
            raise RuntimeError("solve stopped by the callback")


@dataclass
class SolveReport:
    iterations: int
    converged: bool
    residuals: np.ndarray
    wall_time: float
    cond_estimate: float | None = None
    gpu_launches: int = 0

    def to_text(self):
        lines = [
            f"iterations = {self.iterations}",
            f"converged = {self.converged}",
            f"final_relative_residual = {self.residuals[-1]:.6e}",
            f"wall_time_s = {self.wall_time:.6f}",
        ]
        if self.cond_estimate is not None:
            lines.append(f"condition_estimate = {self.cond_estimate:.6e}")
        return "\n".join(lines) + "\n"


def _cond_from_recurrence(alphas, betas):
    """Extreme Ritz values of the CG tridiagonal (src/krylov.py:110-124)."""
    k = len(alphas)
    if k == 1:
        return 1.0
    diag = np.empty(k)
    off = np.empty(k - 1)
    diag[0] = 1.0 / alphas[0]
    for j in range(1, k):
        diag[j] = 1.0 / alphas[j] + betas[j - 1] / alphas[j - 1]
        off[j - 1] = np.sqrt(max(betas[j - 1], 0.0)) / alphas[j - 1]
    ritz = eigvalsh_tridiagonal(diag, off)
    if ritz[0] <= 0:
        return float("inf")
    return float(ritz[-1] / ritz[0])


def _same_operator(pm, mat):
    """Whether two SparseMat objects hold the same CSR (structure and values); the outcome is
    cached on ``mat`` for ``pm`` (both are immutable: read-only buffers, src/sparsemat.py:51-52)."""
    if pm is mat:
        return True
    cache = getattr(mat, "_b200_same_as", None)
    if cache is not None and cache[0] is pm:
        return cache[1]
    a, b = pm.scipy(), mat.scipy()
    same = (a.shape == b.shape and a.nnz == b.nnz and np.array_equal(a.indptr, b.indptr)
            and np.array_equal(a.indices, b.indices) and np.array_equal(a.data, b.data))
    try:
        mat._b200_same_as = (pm, same)
    except AttributeError:
        pass
    return same


def _handle_for(matrix, precond):
    """The device handle a solve runs on.  With a preconditioner that is the preconditioner's
    handle, whose SpMV applies the matrix the preconditioner was built from; the reference applies
    ``matrix`` itself (src/krylov.py:81), so a different operator (even one with the same shape and
    sparsity, e.g. rescaled values) is refused rather than silently replaced."""
    mat = as_sparsemat(matrix)
    if precond is None:
        return mat, mat.device_handle(), 0
    if precond.n != mat.nrows:
        raise ValueError("preconditioner and matrix sizes differ")
    if not _same_operator(precond.matrix, mat):
        raise ValueError("preconditioner was built for a different matrix: this path applies the "
                         "preconditioner's own operator, so the solve matrix must be the same")
    return mat, precond.handle, 1


def pcg(matrix, precond, b, tol=1e-8, maxit=500, callback=None, track_tridiagonal=False):
    """Preconditioned CG from x0 = 0 (src/krylov.py:58-107); returns (x, SolveReport)."""
    t0 = time.perf_counter()
    mat, h, use = _handle_for(matrix, precond)
    bt, back = D.to_device(b, mat.nrows, h.device)
    x = D._torch().empty_like(bt)
    hist = np.zeros(maxit + 2)
    coeffs = np.zeros(2 * maxit + 2)
    st = _lib.TlsStatus()
    cb = _Callback(callback, True, mat.nrows)
    rc = h.lib.tls_pcg(h.ctx, _lib.ptr(bt), _lib.ptr(x), float(tol), int(maxit), use, _lib.ptr(hist),
                       _lib.ptr(coeffs), C.byref(st), cb.c, None, D.stream_ptr())
    cb.reraise(rc)
    if rc == _lib.TLS_ERR_BREAKDOWN:
        raise BreakdownError(int(st.iteration), float(st.value))
    h.check(rc)
    its = int(st.iterations)
    if its == 0 and st.converged:
        residuals = np.zeros(1) if hist[0] == 0.0 else hist[:1].copy()
    else:
        residuals = hist[: its + 1].copy()
    cond = None
    if track_tridiagonal and its > 0:
        cond = _cond_from_recurrence(coeffs[0:2 * its:2], coeffs[1:2 * its:2])
    out = back(x)
    return out, SolveReport(its, bool(st.converged), residuals, time.perf_counter() - t0, cond,
                            int(st.gpu_launches))


def gmres(matrix, precond, b, tol=1e-8, maxit=500, callback=None, restart=None):
    """Right-preconditioned GMRES (src/krylov.py:127-195); ``restart`` = GMRES(m)."""
    t0 = time.perf_counter()
    if (restart is None or restart >= maxit) and maxit > GMRES_MAXIT_CAP:
        raise ValueError(f"maxit {maxit} exceeds the hard cap {GMRES_MAXIT_CAP}")
    mat, h, use = _handle_for(matrix, precond)
    bt, back = D.to_device(b, mat.nrows, h.device)
    x = D._torch().empty_like(bt)
    hist = np.zeros(maxit + 2)
    st = _lib.TlsStatus()
    cb = _Callback(callback, False, mat.nrows)
    rc = h.lib.tls_gmres(h.ctx, _lib.ptr(bt), _lib.ptr(x), float(tol), int(maxit),
                         int(restart or 0), use, _lib.ptr(hist), C.byref(st), cb.c, None,
                         D.stream_ptr())
    cb.reraise(rc)
    h.check(rc)
    its = int(st.iterations)
    residuals = hist[: its + 1].copy()
    if its == 0 and st.converged:
        residuals = np.zeros(1)
    return back(x), SolveReport(its, bool(st.converged), residuals, time.perf_counter() - t0, None,
                                int(st.gpu_launches))
