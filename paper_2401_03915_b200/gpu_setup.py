"""Device setup: local operators, spectral coarse space, Galerkin coarse operator.

Pipeline per batch of subdomains (all on the GPU, stream-ordered with the
library calls):

1. ``tls_extract_blocks`` gathers the dense local blocks A_ii in the
   reference's local order (src/subdomain.py:53-69) — no DENSE_GUARD.
2. Factor + invert (Cholesky when symmetric, pivoted LU otherwise; the same
   failure rules as ``factor_dense``, src/subdomain.py:72-95).  The inverse
   B_i = A_ii^{-1} is what the iteration streams (``tls_store_local_inverse``:
   packed lower-triangular 64x64 tiles when symmetric).
3. Coarse columns from B_i alone — no second factorisation of A_inner:
   with ring = outermost layer, F = B[int, ring], B22 = B[ring, ring], the
   harmonic extension is ext = B[:, ring] B22^{-1} (block-inverse identity),
   so
   * "gevp" (src/spectral.py:111-132): the m x m pencil (lhs on the ring block,
     A) has the same nonzero eigenpairs as  (F^T A_II F) u = lambda B22 u
     (n_b x n_b); the lifted column is D ext y = (B[:, ring] u) restricted to
     the interior, A-normalised (u^T B22 u = 1) and sign-fixed on the full
     local vector exactly as ``_fix_signs`` (src/spectral.py:59-66);
   * "svd" (src/spectral.py:135-154): left singular vectors of
     ext[:n_int] = F B22^{-1};
   * "full" (src/coarse.py:66-67): all columns of ext[:n_int].
   Top-k (``n_modes``) or threshold (``tau``, strict with the 1e-12 tie guard)
   selection.
4. ``rank_filter`` (src/coarse.py:119-155): per-subdomain column-pivoted QR
   magnitudes against the global largest pivot (host LAPACK geqp3 on the
   n_int x k blocks — bookkeeping, not on the iteration path).
5. A0 = Z^T A Z (src/coarse.py:158-183): A Z_s = A_ii[:, :n_int] Z_s scattered
   over the subdomain's local rows, then Z_j^T (A Z_s) per touching owner j;
   symmetrised when symmetric; Cholesky/LU with the reference's failure rules;
   its inverse is stored as the coarse block of the same tile kernel.

Dense factorisations/eigensolves in steps 2-3/5 use torch.linalg (cuSOLVER) —
a library call on the SETUP path; the per-iteration path is all in-tree CUDA.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor
import warnings

import numpy as np
import scipy.sparse as sp
import scipy.linalg as sla

from . import _lib
from .device import _torch, stream_ptr
from .errors import SubdomainSetupError

VERBOSE = bool(int(os.environ.get("TLS_VERBOSE", "0")))
TIE_GUARD = 1e-12
TOPK_TAU = 1e-300
EPS = float(np.finfo(float).eps)
REFINE_COND = 1.0e8  # cond_1(A0) above which every coarse solve gets one refinement step
# SPD A0 of at least this order whose half bandwidth is < n_C / 4 is inverted by the
# block-tridiagonal recurrences (spd_inverse_block_tridiagonal) instead of dense potrf + potri
BAND_INVERSE_MIN = int(os.environ.get("TLS_A0_BANDED_MIN", "4096"))
# ... and from this order on no inverse is formed at all: the coarse solve runs as a block
# forward / backward substitution with the inverted Schur blocks (tls_coarse_chain): ~2 n_C * bs
# doubles per solve instead of n_C^2 / 2 (configuration 5: 1.5 GB instead of 9.7 GB per iteration)
def _chain_min():
    return int(os.environ.get("TLS_A0_CHAIN_MIN", "16384"))


class _LazyBasisBlocks:
    """The per-subdomain basis blocks Z_s (n_int x k_s host arrays) of one handle, fetched from the
    library's device copy (tls_coarse_basis_fetch) the first time one is read."""

    def __init__(self, handle, n_int, counts):
        self._handle, self._n_int, self._counts = handle, n_int, counts
        self._blocks = None

    def _load(self):
        if self._blocks is None:
            total = int(sum(ni * k for ni, k in zip(self._n_int, self._counts)))
            flat = np.empty(max(total, 1), dtype=np.float64)
            h = self._handle
            h.check(h.lib.tls_coarse_basis_fetch(h.ctx, _lib.ptr(flat), total))
            blocks, off = [], 0
            for ni, k in zip(self._n_int, self._counts):   # stored k x n_int (column by column)
                blocks.append(flat[off:off + ni * k].reshape(k, ni).T)
                off += ni * k
            self._blocks = blocks
        return self._blocks

    def __len__(self):
        return len(self._counts)

    def __getitem__(self, i):
        return self._load()[i]

    def __iter__(self):
        return iter(self._load())


class CoarseData:
    """Device coarse space + the host bookkeeping of CoarseSpace (src/coarse.py:23-49).

    ``restrict`` / ``solve_coarse`` / ``prolong`` run the apply's own kernels through the C ABI
    (``tls_coarse_restrict`` / ``tls_coarse_solve`` / ``tls_coarse_prolong``); ``basis`` and
    ``a00`` are materialised on the host on first access (``a00`` from the device copy kept at
    setup, or -- when A0 was too large to keep, > 4 GB -- by the reference's own sparse triple
    product, src/coarse.py:166-170)."""

    def __init__(self, n, maps, z_blocks, counts, nnz_a00):
        self._n = n
        self._maps = maps
        self._z = z_blocks            # list of host (n_int x k) arrays, kept columns
        self.ranges = tuple(self._ranges(counts))
        self.nnz_a00 = int(nnz_a00)
        self._basis = None
        self._a00 = None
        self._a00_dev = None
        self._handle = None           # set by setup() once the preconditioner is finalised
        self._csr = None
        self._symmetric = False
        self.cond1 = None
        self.refined = False
        self.solve_kind = "none"      # "dense-inverse" | "block-tridiagonal" (tls_coarse_info)
        self.solve_blocks = self.solve_block_size = 0
        self.solve_bytes = 0.0

    @staticmethod
    def _ranges(counts):
        out, c = [], 0
        for k in counts:
            out.append((c, c + k))
            c += k
        return out

    @property
    def n_coarse(self):
        return self.ranges[-1][1] if self.ranges else 0

    def column_counts(self):
        return tuple(e - s for s, e in self.ranges)

    @property
    def basis(self):
        """Global basis as a SparseMat (n x n_C), built on demand on the host."""
        if self._basis is None:
            import scipy.sparse as sp
            from .sparsemat import SparseMat
            rows, cols, vals = [], [], []
            for smap, z, (c0, _) in zip(self._maps, self._z, self.ranges):
                if z.shape[1] == 0:
                    continue
                r, c = np.nonzero(z)
                rows.append(smap.interior[r]); cols.append(c0 + c); vals.append(z[r, c])
            if rows:
                mat = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                    shape=(self._n, self.n_coarse))
            else:
                mat = sp.csr_matrix((self._n, 0))
            self._basis = SparseMat(mat)
        return self._basis

    @property
    def a00(self):
        """The Galerkin operator Z^T A Z, dense n_C x n_C, symmetrised when SPD (src/coarse.py:158-170)."""
        if self._a00 is None:
            if self._a00_dev is not None:
                self._a00 = self._a00_dev.cpu().numpy()
            else:
                b = self.basis.scipy()
                prod = (b.T @ (self._csr @ b)).toarray()
                self._a00 = 0.5 * (prod + prod.T) if self._symmetric else prod
        return self._a00

    def _call(self, name, v, n_in, n_out):
        from . import device as D
        h = self._handle
        if h is None:
            raise RuntimeError("coarse operator not factored; call galerkin_coarse first")
        x, back = D.to_device(v, n_in, h.device)
        y = _torch().empty(n_out, dtype=_torch().float64, device=x.device)
        h.check(getattr(h.lib, name)(h.ctx, _lib.ptr(x), _lib.ptr(y), stream_ptr()))
        return back(y)

    def restrict(self, r):
        """c = Z^T r (src/coarse.py:40-41)."""
        return self._call("tls_coarse_restrict", r, self._n, self.n_coarse)

    def prolong(self, y):
        """Z y (src/coarse.py:43-44)."""
        return self._call("tls_coarse_prolong", y, self.n_coarse, self._n)

    def solve_coarse(self, rhs):
        """A0^{-1} rhs (src/coarse.py:46-49)."""
        return self._call("tls_coarse_solve", rhs, self.n_coarse, self.n_coarse)


def warm_linalg(device=None):
    """Initialise torch.linalg's lazily-loaded GPU backends once, from the calling thread
    (their first use is not thread-safe; in-process rank groups call this before threading)."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    a = torch.eye(4, dtype=torch.float64, device=dev) * 2.0
    L, _ = torch.linalg.cholesky_ex(a)
    torch.cholesky_inverse(L)
    LU, piv, _ = torch.linalg.lu_factor_ex(a)
    torch.linalg.lu_solve(LU, piv, a)
    torch.linalg.eigh(a)
    torch.linalg.svd(a, full_matrices=False)
    torch.linalg.solve(a, a, left=False)
    torch.linalg.solve_triangular(L, a, upper=False)
    torch.linalg.cholesky(a)
    torch.cuda.synchronize(dev)


_STAGE = {}


def _stage(name, t_prev):
    """Accumulate synchronized stage times (verbose mode only); returns the new timestamp."""
    if not VERBOSE:
        return t_prev
    _torch().cuda.synchronize()
    t = time.perf_counter()
    _STAGE[name] = _STAGE.get(name, 0.0) + (t - t_prev)
    return t


class _nvtx:
    """NVTX range around a setup stage (torch.cuda.nvtx; a no-op without an attached tool)."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        try:
            _torch().cuda.nvtx.range_push(self.name)
            self.on = True
        except Exception:
            self.on = False

    def __exit__(self, *exc):
        if self.on:
            _torch().cuda.nvtx.range_pop()
        return False


def _log(t0, msg):
    if VERBOSE:
        print(f"[tls setup {time.perf_counter() - t0:7.1f}s] {msg}", flush=True)


def _symmetrize_lower_inplace(torch, A, bs=4096):
    """A[lower incl. diagonal blocks] <- 0.5 (A + A^T) without a dense temporary copy."""
    n = A.shape[0]
    for i0 in range(0, n, bs):
        i1 = min(i0 + bs, n)
        A[i0:i1, :i1] = 0.5 * (A[i0:i1, :i1] + A[:i1, i0:i1].mT)


def _select(values, tau, n_modes):
    thr = TOPK_TAU if n_modes is not None else tau
    keep = np.nonzero(values > thr * (1.0 + TIE_GUARD))[0]
    if n_modes is not None:
        keep = keep[:n_modes]
    return keep


def _fix_signs(torch, v):
    """Flip columns so the largest-|.| component (first occurrence) is positive."""
    if v.shape[1] == 0:
        return v
    idx = torch.argmax(v.abs(), dim=0)
    sgn = torch.where(v.gather(0, idx[None, :])[0] < 0, -1.0, 1.0).to(v.dtype)
    return v * sgn[None, :]


def _cut_gap(values, keep):
    """Relative gap between the last selected and the first rejected value (inf if none)."""
    if keep.size == 0 or keep[-1] + 1 >= values.size or values[keep[-1]] <= 0:
        return float("inf")
    return float((values[keep[-1]] - values[keep[-1] + 1]) / values[keep[-1]])


def _pou_columns(torch, A, n, ni, nu):
    """Partition-of-unity modes (src/spectral.py:93-108, added by src/coarse.py:81-82) on the
    device: the m x m pencil (D A D) u = lam A u with D = diag(pou_mask) reduces, for lam != 0,
    to the n_int pencil A_II y = lam S_I y with S_I = A_II - A_IG A_GG^{-1} A_GI (the interior
    Schur complement) and u = [y; -A_GG^{-1} A_GI y]; y^T S_I y = u^T A u = 1 is the reference's
    normalisation.  Values descending, kept when lam > nu (1 + TIE_GUARD), signs fixed on the full
    u, columns = D u = y (interior rows)."""
    dev = A.device
    if ni == n:  # no overlap rows: S_I = A_II, every lam = 1 <= nu
        return torch.zeros((ni, 0), dtype=torch.float64, device=dev)
    AII = A[:ni, :ni]
    AIG = A[:ni, ni:n]
    AGG = A[ni:n, ni:n]
    LG = torch.linalg.cholesky(0.5 * (AGG + AGG.mT))
    X = torch.cholesky_solve(AIG.mT.contiguous(), LG)        # A_GG^{-1} A_GI
    S = AII - AIG @ X
    LS = torch.linalg.cholesky(0.5 * (S + S.mT))
    Y = torch.linalg.solve_triangular(LS, AII, upper=False)
    C = torch.linalg.solve_triangular(LS, Y.mT, upper=False)
    w, Q = torch.linalg.eigh(0.5 * (C + C.mT))
    w = torch.flip(w, dims=[0]).cpu().numpy()
    keep = np.nonzero(w > nu * (1.0 + TIE_GUARD))[0]
    if keep.size == 0:
        return torch.zeros((ni, 0), dtype=torch.float64, device=dev)
    Q = torch.flip(Q, dims=[1])[:, torch.as_tensor(keep, device=dev)]
    Yv = torch.linalg.solve_triangular(LS.mT, Q, upper=True)
    U = _fix_signs(torch, torch.cat([Yv, -(X @ Yv)], dim=0))
    return U[:ni].contiguous()


def _with_pou(torch, Z, A, n, ni, nu):
    """[harmonic columns, PoU columns] (src/coarse.py:72-84), all-zero columns dropped
    (src/coarse.py:99-103)."""
    if nu is None:
        return Z
    P = _pou_columns(torch, A, n, ni, nu)
    if P.shape[1] == 0:
        return Z
    Z = torch.cat([Z, P], dim=1) if Z.shape[1] else P
    nz = torch.any(Z != 0, dim=0)
    return Z if bool(nz.all()) else Z[:, nz].contiguous()


def _subdomain_columns(torch, kind, A, Bring, n, ni, nin, tau, n_modes):
    """Coarse columns (n_int x k, device) of one subdomain, and the selection's cut gap.

    ``A`` = dense A_ii (local order), ``Bring`` = A_ii^{-1}[:, ring] (n x n_b, local order).
    The cut gap (sigma_k - sigma_{k+1}) / sigma_k measures how well-posed the selected span
    is: a gap near rounding level means the top-k cut splits a multiplet.
    """
    nb = n - nin
    dev = A.device
    if nb == 0 or kind == "none":
        return torch.zeros((ni, 0), dtype=torch.float64, device=dev), float("inf")
    F = Bring[:ni]
    B22 = Bring[nin:n]
    if kind == "gevp":
        H = F.mT @ (A[:ni, :ni] @ F)
        H = 0.5 * (H + H.mT)
        B22s = 0.5 * (B22 + B22.mT)
        C = torch.linalg.cholesky(B22s)
        X = torch.linalg.solve_triangular(C, H, upper=False)
        M = torch.linalg.solve_triangular(C, X.mT, upper=False)
        M = 0.5 * (M + M.mT)
        w, Q = torch.linalg.eigh(M)
        w = torch.flip(w, dims=[0])
        Q = torch.flip(Q, dims=[1])
        sig = torch.sqrt(torch.clamp(w, min=0.0)).cpu().numpy()
        keep = _select(sig, tau, n_modes)
        if keep.size == 0:
            return torch.zeros((ni, 0), dtype=torch.float64, device=dev), float("inf")
        U = torch.linalg.solve_triangular(C.mT, Q[:, torch.as_tensor(keep, device=dev)], upper=True)
        V = Bring @ U
        V = _fix_signs(torch, V)
        return V[:ni].contiguous(), _cut_gap(sig, keep)
    E = torch.linalg.solve(B22, F, left=False)  # E B22 = F  ->  ext[:n_int]
    if kind == "full":
        return E.contiguous(), float("inf")
    U, S, _ = torch.linalg.svd(E, full_matrices=False)
    sv = S.cpu().numpy()
    keep = _select(sv, tau, n_modes)
    if keep.size == 0:
        return torch.zeros((ni, 0), dtype=torch.float64, device=dev), float("inf")
    V = _fix_signs(torch, U[:, torch.as_tensor(keep, device=dev)])
    return V.contiguous(), _cut_gap(sv, keep)


def _svd_columns_lu_batch(torch, A, LU, piv, P, n_loc, n_int, n_bnd, first, cnt, ld, tau, n_modes):
    """Top-k SVD coarse columns (src/spectral.py:135-154, fixed k) of a batch of LU-factored
    subdomains, batched by shape: B[:, ring] by one batched lu_solve, E = F B22^{-1} (= ext[:n_int],
    block-inverse identity) by one batched solve, then a batched Householder QR E = Q R and the SVD
    of the small R (n_b x n_b) -- instead of one thin SVD of the tall E per subdomain.  Returns
    {b: (Z (n_int x k), cut gap)}."""
    dev = A.device
    out = {}
    groups = {}
    for b in range(cnt):
        s = first + b
        groups.setdefault((int(n_loc[s]), int(n_int[s]), int(n_loc[s] - n_bnd[s])), []).append(b)
    for (n, ni, nin), bs in groups.items():
        nb = n - nin
        if nb == 0:
            for b in bs:
                out[b] = (torch.zeros((ni, 0), dtype=torch.float64, device=dev), float("inf"))
            continue
        g = len(bs)
        bi = torch.as_tensor(bs, device=dev)
        Pg = P.index_select(0, bi)
        pinv = torch.empty_like(Pg)
        pinv.scatter_(1, Pg, torch.arange(ld, device=dev).expand_as(Pg))
        E = torch.zeros((g, ld, nb), dtype=torch.float64, device=dev)
        E.view(g, -1)[torch.arange(g, device=dev)[:, None],
                      pinv[:, nin:n] * nb + torch.arange(nb, device=dev)[None, :]] = 1.0
        X = torch.linalg.lu_solve(LU.index_select(0, bi), piv.index_select(0, bi), E)
        del E
        Bring = torch.gather(X, 1, pinv[:, :n, None].expand(g, n, nb))
        del X
        Eint = torch.linalg.solve(Bring[:, nin:n], Bring[:, :ni], left=False)   # (g, ni, nb)
        del Bring
        kk = min(n_modes + 1, nb)
        # backward-stable thin SVD: E = Q R (batched Householder QR), then the small n_b x n_b SVD
        # of R; U = Q U_R.  (A Gram-matrix eigensolve loses ~cond(A0) x eps in the coarse
        # correction on the saddle point: 1e-6 vs the reference, measured.)
        Q, R = torch.linalg.qr(Eint)
        del Eint
        UR, sig = _svd_left_topk(torch, R, kk)
        U = Q @ UR
        del Q, R, UR
        sig_h = sig.cpu().numpy()
        for j, b in enumerate(bs):
            keep = _select(sig_h[j], tau, n_modes)
            if keep.size == 0:
                out[b] = (torch.zeros((ni, 0), dtype=torch.float64, device=dev), float("inf"))
                continue
            Z = _fix_signs(torch, U[j][:, torch.as_tensor(keep, device=dev)])
            out[b] = (Z.contiguous(), _cut_gap(sig_h[j], keep))
    return out


def _svd_left_topk(torch, R, kk):
    """Leading kk left singular vectors (b, r, kk) and singular values (b, kk), descending, of a
    batch of small matrices R (b, r, n).  Preconditioned one-sided Jacobi (Drmac-Veselic): a second
    QR, R^T = Q2 R2, leaves R = L2 Q2^T with L2 = R2^T lower triangular and close to column-graded
    form, so the left singular vectors of R are those of L2 (R's rows are sorted by norm before that
    QR and the vectors permuted back); the in-tree batched kernel
    (tls_svdj_batched) rotates the columns of L2 until they are mutually orthogonal -- column j
    ends as sigma_j u_j.  LAPACK-grade accuracy (also for graded spectra) without a cuSOLVER call
    per matrix.  TLS_SVDJ=0 keeps torch.linalg.svd."""
    b, r, n = R.shape
    if not R.is_cuda or os.environ.get("TLS_SVDJ", "1") == "0":
        UR, sig, _ = torch.linalg.svd(R, full_matrices=False)
        return UR[:, :, :kk], sig[:, :kk]
    # rows of R by descending norm first (a cheap stand-in for column pivoting in the second QR:
    # 13 instead of 18 Jacobi sweeps on a harmonic extension)
    order = torch.argsort(R.norm(dim=2), dim=1, descending=True)
    Rs = torch.gather(R, 1, order[:, :, None].expand(b, r, n))
    X = torch.linalg.qr(Rs.mT, mode="r").R.contiguous()  # R2 row-major = L2 column-major (r x k)
    del Rs
    k = X.shape[1]
    sig = torch.empty((b, k), dtype=R.dtype, device=R.device)
    info = torch.empty((b,), dtype=torch.int32, device=R.device)
    rc = _lib.load().tls_svdj_batched(_lib.ptr(X), b, X.shape[2], k, _lib.ptr(sig), _lib.ptr(info), stream_ptr())
    if rc != 0:
        raise RuntimeError(f"tls_svdj_batched failed ({rc})")
    kk = min(kk, k)
    sv, idx = torch.topk(sig, kk, dim=1)                 # descending
    W = torch.gather(X, 1, idx[:, :, None].expand(b, kk, X.shape[2]))
    UR = torch.empty((b, r, kk), dtype=R.dtype, device=R.device)
    UR.scatter_(1, order[:, :, None].expand(b, r, kk), (W / sv.clamp(min=1e-300)[:, :, None]).mT)
    if int(info.min()) < 0:                              # sweep limit reached: LAPACK for those
        for j in torch.nonzero(info < 0).flatten().tolist():
            Uj, sj, _ = torch.linalg.svd(R[j], full_matrices=False)
            UR[j] = Uj[:, :kk]
            sv[j] = sj[:kk]
    return UR, sv


def _orth(torch, X, check=True):
    """Batched orthonormalisation: CholeskyQR2 (two GEMM + p x p Cholesky passes).

    check=False skips the per-call host test of the Cholesky info (a device sync); the caller
    then tests the result for non-finite values at its next sync point and falls back."""
    X0 = X
    bad = None
    for _ in range(2):
        G = X.mT @ X
        R, info = torch.linalg.cholesky_ex(G, upper=True)
        if check and bool((info != 0).any()):  # numerically rank-deficient block: Householder
            return torch.linalg.qr(X0).Q
        bad = info != 0 if bad is None else bad | (info != 0)
        X = torch.linalg.solve_triangular(R, X, upper=True, left=False)
    return X if check else (X, bad)


def _orth_shifted(torch, X):
    """Shifted CholeskyQR3 (Fukaya et al.): one Cholesky pass of X^T X + s I with
    s = 11 (m p + p (p + 1)) u ||X||_F^2 -- positive definite for any X, so it cannot break down on
    the ill-conditioned blocks a Chebyshev filter produces (cond up to ~1e8) -- then CholeskyQR2 on
    the now well-conditioned result.  No host synchronisation; returns (Q, bad) with ``bad``
    flagging a non-positive pivot (non-finite input), tested at the caller's next check."""
    b, m, p = X.shape
    G = X.mT @ X
    tr = G.diagonal(dim1=1, dim2=2).sum(dim=1)
    sh = 11.0 * (m * p + p * (p + 1)) * EPS * tr
    G = G + sh[:, None, None] * torch.eye(p, dtype=X.dtype, device=X.device)
    R, info = torch.linalg.cholesky_ex(G, upper=True)
    X = torch.linalg.solve_triangular(R, X, upper=True, left=False)
    Q, bad = _orth(torch, X, check=False)
    return Q, bad | (info != 0)


def _rayleigh_ritz(torch, M, X, k, bad=None):
    MX = M @ X
    T = X.mT @ MX
    # the p x p projected problem is tiny: solve it on the host (batched GPU eigh loops one
    # cuSOLVER call per matrix once p > 32)
    Th = (0.5 * (T + T.mT)).cpu()
    if bad is not None and bool(bad.cpu().any()):  # (no extra stall: the copy above synced)
        return None  # CholeskyQR2 broke down on X's block (caller falls back)
    th_all, S = torch.linalg.eigh(Th)
    th_all = torch.flip(th_all, dims=[-1]).to(M.device)
    S = torch.flip(S, dims=[-1]).to(M.device)
    Xr = X @ S
    MXr = MX @ S
    return th_all, Xr, MXr


def topk_subspace(torch, M, k, tol=1e-14, maxit=2000, seed=20240103, p=None):
    """Top-k eigenpairs (descending) of a batch of symmetric PSD matrices M (b, m, m).

    Block subspace iteration with the squared operator (two batched GEMMs per sweep) on
    p = max(3k, k + 16) vectors, CholeskyQR2 re-orthonormalisation and Rayleigh-Ritz every 4
    sweeps; stops when every wanted Ritz pair has ||M x - theta x|| <= tol * theta_1 and raises
    if that does not happen (never returns an unconverged span).  Batched replacement of the
    dense generalized eigensolve of src/spectral.py:69-85 for a fixed number of modes; small
    matrices go to a dense batched eigh.  Converges like (theta_{p+1} / theta_k)^2 per sweep:
    slow on flat spectra, where ``topk_chebyshev`` (the setup's default) needs ~4x fewer products.
    """
    b, m, _ = M.shape
    p = min(m, p or max(3 * k, k + 16))
    if m <= max(96, 2 * p):
        w, Q = torch.linalg.eigh(M)
        return torch.flip(w, dims=[-1])[:, :k], torch.flip(Q, dims=[-1])[:, :, :k], 0
    gen = torch.Generator(device=M.device)
    gen.manual_seed(seed)
    X = _orth(torch, torch.randn((b, m, p), generator=gen, dtype=M.dtype, device=M.device))
    scale = None
    res = float("inf")
    for it in range(1, maxit + 1):
        X = _orth(torch, M @ (M @ X))
        if it % 4 == 0:
            th_all, Xr, MXr = _rayleigh_ritz(torch, M, X, k)
            if scale is None:
                scale = th_all[:, :1].abs().clamp(min=1e-300)
            R = MXr[:, :, :k] - Xr[:, :, :k] * th_all[:, None, :k]
            res = float((R.norm(dim=1) / scale).max())
            if res <= tol:
                return th_all[:, :k], Xr[:, :, :k], it
            X = Xr  # continue from the Ritz basis (sorted, orthonormal)
    raise RuntimeError(f"subspace iteration did not converge: residual {res:.2e} after {maxit} sweeps")


def _topk_chebyshev_host(torch, M, k, tol=1e-14, p=None, maxit=400, seed=20240103, rmax=1e8, dmax=16,
                   trace=None, X0=None):
    """Top-k eigenpairs (descending) of a batch of symmetric PSD matrices M (b, m, m).

    Chebyshev-filtered subspace iteration: each outer step applies T_d((M - c) / e) to the Ritz
    block (columns = current Ritz vectors), with [0, a] (a = the block's smallest Ritz value, per
    matrix) mapped onto [-1, 1]; the filtered columns are normalised, re-orthonormalised
    (CholeskyQR2) and Rayleigh-Ritz'ed (p x p).  Every matrix gets its own degree d_b (the batch
    runs the largest d_b among unconverged matrices; a matrix whose degree is reached stops
    updating), capped so the filter's spread over its wanted Ritz values,
    R = T_d(x_1) / T_d(x_k), stays below ``rmax``.  Because each column starts as a Ritz vector,
    column i's pull toward the top modes is (its residual) x R, not R: the columns stay far from
    collinear and the k-th keeps ~eps * (1 + residual * R) relative precision.  (From a random
    block an uncapped degree amplifies the top modes ~1e19 x more than the k-th and collapses the
    block.)  Same stopping rule as ``topk_subspace``; raises when it does not converge.  Returns
    (theta, X, block products).
    """
    b, m, _ = M.shape
    p = min(m, p or max(3 * k, k + 16))
    if m <= max(96, 2 * p):
        w, Q = torch.linalg.eigh(M)
        return torch.flip(w, dims=[-1])[:, :k], torch.flip(Q, dims=[-1])[:, :, :k], 0
    if X0 is None:
        gen = torch.Generator(device=M.device)
        gen.manual_seed(seed)
        X = _orth(torch, torch.randn((b, m, p), generator=gen, dtype=M.dtype, device=M.device))
        X = _orth(torch, M @ (M @ X))
    else:  # continue from an orthonormal block (the device iteration's last checkpoint)
        X = X0
    th, X, MX = _rayleigh_ritz(torch, M, X, p)  # checked _orth: always orthonormal here
    scale = th[:, :1].abs().clamp(min=1e-300)
    res = float("inf")
    products = 3
    for it in range(1, maxit + 1):
        R = MX[:, :, :k] - X[:, :, :k] * th[:, None, :k]
        res_b = (R.norm(dim=1) / scale).amax(dim=1)                     # (b,)
        a = th[:, p - 1].clamp(min=0.0)
        e = (0.5 * a).clamp(min=1e-300)
        x1 = ((th[:, 0] - e) / e).clamp(min=1.0 + 1e-12)
        xk = ((th[:, k - 1] - e) / e).clamp(min=1.0 + 1e-12)
        per = (torch.acosh(x1) - torch.acosh(xk)).clamp(min=1e-12)
        d_b = torch.floor(np.log(rmax) / per).clamp(min=1, max=dmax)
        d_b = torch.where(res_b > tol, d_b, torch.zeros_like(d_b))       # converged: leave as is
        host = torch.stack([res_b.max(), d_b.max()]).cpu()               # ONE sync per step
        res, d = float(host[0]), int(host[1])
        if res <= tol:
            return th[:, :k], X[:, :, :k], products
        if trace is not None:
            trace.append((d, res, int((res_b > tol).sum()), float(per.max())))
        c = e[:, None, None]
        inv_e = (1.0 / e)[:, None, None]
        Y0 = X
        Y1 = torch.where((d_b >= 1)[:, None, None], (MX - c * X) * inv_e, X)
        for j in range(2, d + 1):
            Y2 = 2.0 * (M @ Y1 - c * Y1) * inv_e - Y0
            live = (d_b >= j)[:, None, None]
            Y0 = torch.where(live, Y1, Y0)
            Y1 = torch.where(live, Y2, Y1)
        products += d
        Y1 = Y1 / Y1.norm(dim=1, keepdim=True).clamp(min=1e-300)
        Xo, bad = _orth(torch, Y1, check=False)  # no sync in _orth: tested with the RR copy
        rr = _rayleigh_ritz(torch, M, Xo, p, bad=bad)
        if rr is None:  # CholeskyQR2 broke down: Householder QR of the same block
            rr = _rayleigh_ritz(torch, M, torch.linalg.qr(Y1).Q, p)
        th, X, MX = rr
        products += 1
    raise RuntimeError(f"Chebyshev subspace iteration did not converge: residual {res:.2e} after {maxit} steps")


def _eigh_desc(torch, T):
    """Eigenpairs of a batch of small symmetric matrices, descending: the in-tree batched Jacobi
    kernel (tls_syevj_batched, stream-ordered, no host round trip) for p <= 64."""
    b, p, _ = T.shape
    if p > 64 or not T.is_cuda:
        w, S = torch.linalg.eigh(0.5 * (T + T.mT))
        return torch.flip(w, dims=[-1]), torch.flip(S, dims=[-1])
    Tc = T.contiguous()
    w = torch.empty((b, p), dtype=T.dtype, device=T.device)
    S = torch.empty((b, p, p), dtype=T.dtype, device=T.device)
    rc = _lib.load().tls_syevj_batched(_lib.ptr(Tc), b, p, _lib.ptr(w), _lib.ptr(S), stream_ptr())
    if rc != 0:
        raise RuntimeError(f"tls_syevj_batched failed ({rc})")
    return w, S


def _block_width(k):
    """Columns of the subspace-iteration block for k wanted pairs (TLS_CHEB_P overrides)."""
    e = int(os.environ.get("TLS_CHEB_P", "0"))
    return e if e > 0 else max(3 * k, k + 16)


def topk_chebyshev(torch, M, k, tol=1e-14, p=None, maxit=400, seed=20240103, rmax=1e8, dmax=16,
                   trace=None, check_every=2):
    """Top-k eigenpairs (descending) of a batch of symmetric PSD matrices M (b, m, m).

    Chebyshev-filtered subspace iteration: each outer step applies T_d((M - c) / e) to the Ritz
    block (columns = current Ritz vectors), with [0, a] (a = the block's smallest Ritz value, per
    matrix) mapped onto [-1, 1]; the filtered columns are normalised, re-orthonormalised
    (CholeskyQR2) and Rayleigh-Ritz'ed (p x p, on the device: tls_syevj_batched).  Every matrix
    gets its own degree d_b (a matrix whose degree is reached stops updating), capped so the
    filter's spread over its wanted Ritz values, R = T_d(x_1) / T_d(x_k), stays below ``rmax``.
    Because each column starts as a Ritz vector, column i's pull toward the top modes is (its
    residual) x R, not R: the columns stay far from collinear and the k-th keeps
    ~eps * (1 + residual * R) relative precision.  Stops when every wanted Ritz pair has
    ||M x - theta x|| <= tol * theta_1.  The whole iteration is stream-ordered: the host looks at
    the residuals (one small copy) only every ``check_every`` steps, and the Chebyshev loop runs
    the degree of that check (per-matrix degrees are masks), so batches pipeline on the device.
    The filtered block (cond up to ~rmax) is re-orthonormalised by shifted CholeskyQR3; when that
    breaks down (non-finite block: ~30% of the configuration-5 batches at some step) the iteration
    resumes from the last checked Ritz block on ``_topk_chebyshev_host`` (host checks every step,
    Householder QR where CholeskyQR2 fails).  ``TLS_CHEB_ORTH=qr``: batched Householder QR on every
    step instead (no breakdowns, but measured 13.0 vs 9.2 s on configuration 5).  Returns
    (theta, X, block products).
    """
    b, m, _ = M.shape
    p = min(m, p or _block_width(k))
    if m <= max(96, 2 * p) or p > 64:
        return _topk_chebyshev_host(torch, M, k, tol=tol, p=p, maxit=maxit, seed=seed, rmax=rmax,
                                    dmax=dmax, trace=trace)
    gen = torch.Generator(device=M.device)
    gen.manual_seed(seed)
    X = _orth(torch, torch.randn((b, m, p), generator=gen, dtype=M.dtype, device=M.device))
    X = _orth(torch, M @ (M @ X))
    MX = M @ X
    th, S = _eigh_desc(torch, X.mT @ MX)
    X, MX = X @ S, MX @ S
    scale = th[:, :1].abs().clamp(min=1e-300)
    products = 3
    d = dmax
    bad = torch.zeros(b, dtype=torch.bool, device=M.device)
    res = float("inf")
    ckpt = X
    for it in range(1, maxit + 1):
        R = MX[:, :, :k] - X[:, :, :k] * th[:, None, :k]
        res_b = (R.norm(dim=1) / scale).amax(dim=1)                     # (b,)
        a = th[:, p - 1].clamp(min=0.0)
        e = (0.5 * a).clamp(min=1e-300)
        x1 = ((th[:, 0] - e) / e).clamp(min=1.0 + 1e-12)
        xk = ((th[:, k - 1] - e) / e).clamp(min=1.0 + 1e-12)
        per = (torch.acosh(x1) - torch.acosh(xk)).clamp(min=1e-12)
        d_b = torch.floor(np.log(rmax) / per).clamp(min=1, max=dmax)
        d_b = torch.where(res_b > tol, d_b, torch.zeros_like(d_b))       # converged: leave as is
        if (it - 1) % check_every == 0:
            host = torch.stack([torch.nan_to_num(res_b, nan=np.inf).max(), d_b.max(),
                                bad.any().to(res_b.dtype)]).cpu()       # one small copy
            res, d = float(host[0]), int(host[1])
            if float(host[2]) != 0.0 or not np.isfinite(res):
                # a re-orthonormalisation broke down since the last check: resume from that
                # check's Ritz block on the host-checked path (Householder QR where needed)
                th_h, X_h, pr = _topk_chebyshev_host(torch, M, k, tol=tol, p=p, maxit=maxit, seed=seed,
                                                     rmax=rmax, dmax=dmax, trace=trace, X0=ckpt)
                return th_h, X_h, products + pr
            ckpt = X
            if res <= tol:
                return th[:, :k], X[:, :, :k], products
            if trace is not None:
                trace.append((d, res, int((res_b > tol).sum()), float(per.max())))
        c = e[:, None, None]
        inv_e = (1.0 / e)[:, None, None]
        Y0 = X
        Y1 = torch.where((d_b >= 1)[:, None, None], (MX - c * X) * inv_e, X)
        for j in range(2, d + 1):
            Y2 = 2.0 * (M @ Y1 - c * Y1) * inv_e - Y0
            live = (d_b >= j)[:, None, None]
            Y0 = torch.where(live, Y1, Y0)
            Y1 = torch.where(live, Y2, Y1)
        products += d
        Y1 = Y1 / Y1.norm(dim=1, keepdim=True).clamp(min=1e-300)
        if os.environ.get("TLS_CHEB_ORTH", "scqr3") == "qr":
            Xo = torch.linalg.qr(Y1).Q                # Householder: no breakdown, no host sync
        else:
            Xo, bad_o = _orth_shifted(torch, Y1)     # non-finite -> host path at the next check
            bad = bad | bad_o
        MX = M @ Xo
        th, S = _eigh_desc(torch, Xo.mT @ MX)
        X, MX = Xo @ S, MX @ S
        products += 1
    raise RuntimeError(f"Chebyshev subspace iteration did not converge: residual {res:.2e} after {maxit} steps")


def band_solve_multi(torch, L, Dinv, kc, E, lead=None):
    """X = (L L^T)^{-1} E for a batch of banded Cholesky factors and many right-hand sides.

    ``lead`` (host, ascending, one entry per right-hand side): no right-hand side j has a nonzero
    above row ``lead[j]`` in any matrix of the batch, so the forward sweep skips the columns that
    are still identically zero at each block row (unit right-hand sides: half the forward work).

    Default: the blocked restatement ``_band_solve_multi_torch`` (per 64-row block one batched
    cuBLAS DGEMM over all right-hand sides).  ``TLS_K10=1``: the in-tree K10 kernel
    (``tls_band_solve_multi``: one CTA per (subdomain, 64 right-hand sides), both sweeps on the
    FP64 tensor cores) -- correct (tests/test_gpu_setup_kernels.py) but measured 3x slower than the
    batched DGEMMs on configuration 5 (16.0 vs 5.1 s; profiles/prof_setup_cfg5_r02b.txt): each
    64 x 64 panel tile is staged for one 64-column chunk only, where cuBLAS reuses it over all of
    them.
    """
    if E.is_cuda and os.environ.get("TLS_K10", "0") == "1":
        b, ld, nrhs = E.shape
        X = E.contiguous().clone()
        kci = np.ascontiguousarray(np.asarray(kc, dtype=np.int32).reshape(b, ld // 64))
        rc = _lib.load().tls_band_solve_multi(_lib.ptr(L.contiguous()), ld, b, _lib.ptr(Dinv.contiguous()),
                                              _lib.ptr(kci), ld // 64, _lib.ptr(X), nrhs, stream_ptr())
        if rc != 0:
            raise RuntimeError(f"tls_band_solve_multi failed ({rc})")
        return X
    return _band_solve_multi_torch(torch, L, Dinv, kc, E, lead)


def _band_solve_multi_torch(torch, L, Dinv, kc, E, lead=None):
    """X = (L L^T)^{-1} E for a batch of banded Cholesky factors and many right-hand sides.

    Blocked banded forward/backward substitution over 64-row blocks with batched GEMMs: block
    row I touches only the panel L[I, I-K .. I-1] (K = the batch's largest panel count there),
    so the work is ~ n * bandwidth * nrhs instead of the dense n^2 * nrhs of cholesky_solve.
    ``Dinv`` holds the inverted diagonal tiles; ``kc`` (host, (b, nb)) the panel counts.
    """
    b, ld, nrhs = E.shape
    nb = ld // 64
    kmax = kc.max(axis=0) if kc.size else np.zeros(nb, dtype=np.int64)
    X = E.clone()
    # columns [0, live[I]) can be nonzero in block rows <= I (the others start further down)
    live = (np.searchsorted(np.asarray(lead), np.arange(1, nb + 1) * 64, side="left")
            if lead is not None else np.full(nb, nrhs))
    for I in range(nb):  # forward: X_I = D_I^{-1} (E_I - L[I, J0:I] X[J0:I])
        r0, r1 = I * 64, (I + 1) * 64
        K = int(kmax[I])
        nc = int(live[I])
        if nc == 0:
            continue
        if nc == nrhs:
            if K:
                c0 = r0 - K * 64
                X[:, r0:r1] -= L[:, r0:r1, c0:r0] @ X[:, c0:r0]
            X[:, r0:r1] = Dinv[:, I] @ X[:, r0:r1]
            continue
        if K:
            c0 = r0 - K * 64
            X[:, r0:r1, :nc] -= L[:, r0:r1, c0:r0] @ X[:, c0:r0, :nc]
        X[:, r0:r1, :nc] = Dinv[:, I] @ X[:, r0:r1, :nc]
    for I in range(nb - 1, -1, -1):  # backward: X_I = D_I^{-T} X_I; X[J0:I] -= L[I, J0:I]^T X_I
        r0, r1 = I * 64, (I + 1) * 64
        X[:, r0:r1] = Dinv[:, I].mT @ X[:, r0:r1]
        K = int(kmax[I])
        if K:
            c0 = r0 - K * 64
            X[:, c0:r0] -= L[:, r0:r1, c0:r0].mT @ X[:, r0:r1]
    return X


def _harmonic_h(torch, Ag, Bring, n, ni):
    """H = F^T A_II F for F = Bring[:ni] without the dense (ni x ni) A_II product.

    Interior rows of A Bring vanish (Bring = A^{-1} restricted to the ring columns, and the ring
    lies outside the interior), so A_II F = -A[:ni, ni:n] Bring[ni:n].  Only the interior rows
    adjacent to the overlap have a nonzero there; their sparse rows (at most D nonzeros, taken
    with topk from the dense block) times Bring give those rows of A_II F, and
    H = -F[R]^T (A[R, ni:n] Bring[ni:n]) costs |R| * nbr^2 instead of ni^2 * nbr + ni * nbr^2.
    """
    g = Ag.shape[0]
    Gb = Ag[:, :ni, ni:n]
    nnz = (Gb != 0).sum(dim=2)                                       # (g, ni)
    D = int(nnz.max()) if nnz.numel() else 0
    if D == 0:
        return torch.zeros((g, Bring.shape[2], Bring.shape[2]), dtype=Bring.dtype, device=Bring.device)
    cntR = (nnz > 0).sum(dim=1)
    Rm = int(cntR.max())
    R = torch.argsort((nnz == 0).to(torch.int8), dim=1, stable=True)[:, :Rm]   # rows with a nonzero
    Gr = torch.gather(Gb, 1, R[:, :, None].expand(g, Rm, n - ni))
    _, cols = torch.topk(Gr.abs(), D, dim=2)
    vals = torch.gather(Gr, 2, cols)                                 # signed entries (0 pads)
    del Gr
    nbr = Bring.shape[2]
    Blay = Bring[:, ni:n]
    Y = torch.zeros((g, Rm, nbr), dtype=Bring.dtype, device=Bring.device)
    for d in range(D):
        Y.addcmul_(vals[:, :, d:d + 1], torch.gather(Blay, 1, cols[:, :, d:d + 1].expand(g, Rm, nbr)))
    Fr = torch.gather(Bring[:, :ni], 1, R[:, :, None].expand(g, Rm, nbr))
    return -(Fr.mT @ Y)


def _ctac(torch, C, S):
    """C^T S C (symmetric, both triangles filled) for batched lower-triangular C and symmetric S,
    skipping the zero blocks of C in a 2 x 2 splitting and computing the off-diagonal block once:
    1.25 m^3 multiply-adds instead of the 2 m^3 of two full GEMMs.

      C = [C11 0; C21 C22]   W = S C = [S[:, :h] C11 + S[:, h:] C21,  S[:, h:] C22]
      M11 = C[:, :h]^T W[:, :h],  M21 = C22^T W[h:, :h],  M22 = C22^T W[h:, h:]
    """
    m = C.shape[1]
    h = (m // 2 + 63) // 64 * 64
    if m < 256 or h >= m or os.environ.get("TLS_PENCIL_CTAC", "1") == "0":
        M = C.mT @ (S @ C)
        return 0.5 * (M + M.mT)
    S = S.contiguous()                         # one copy of the strided ring-ring slice
    W1 = S @ C[:, :, :h]                       # (g, m, h)   columns of C11 / C21
    W2 = S[:, :, h:] @ C[:, h:, h:]            # (g, m, m-h) columns of C22 (rows below h only)
    C22t = C[:, h:, h:].mT
    M = torch.empty_like(C)
    M11 = C[:, :, :h].mT @ W1
    M[:, :h, :h] = 0.5 * (M11 + M11.mT)
    del M11
    M21 = C22t @ W1[:, h:]                     # (g, m-h, h)
    M[:, h:, :h] = M21
    M[:, :h, h:] = M21.mT
    del M21, W1
    M22 = C22t @ W2[:, h:]
    M[:, h:, h:] = 0.5 * (M22 + M22.mT)
    return M


def _coarse_band_batch(torch, kind, A, L, P, ns, nis, nins, tau, n_modes, Dinv=None, kc=None):
    """Coarse columns of a batch of band-factored subdomains, batched by shape.

    Returns per subdomain (Z, cut_gap); gevp with a fixed mode count runs the batched subspace
    iteration, everything else the per-subdomain dense path.
    """
    cnt = A.shape[0]
    ld = A.shape[1]
    dev = A.device
    out = [None] * cnt
    groups = {}
    for b in range(cnt):
        groups.setdefault((ns[b], nis[b], nins[b]), []).append(b)
    for (n, ni, nin), bs in groups.items():
        nbr = n - nin
        bi = torch.as_tensor(bs, device=dev)
        if nbr == 0 or kind == "none":
            for b in bs:
                out[b] = (torch.zeros((ni, 0), dtype=torch.float64, device=dev), float("inf"), None)
            continue
        # a group that is the whole batch (the common case) reads the batch tensors in place
        sel = (lambda t: t) if len(bs) == cnt else (lambda t: t.index_select(0, bi))
        Pg = sel(P)
        pinv = torch.empty_like(Pg)
        pinv.scatter_(1, Pg, torch.arange(ld, device=dev).expand_as(Pg))
        E = torch.zeros((len(bs), ld, nbr), dtype=torch.float64, device=dev)
        rows = pinv[:, nin:n]                                       # (g, nbr) factor positions of the ring
        direct = (kind == "gevp" and n_modes is not None and ni == nin
                  and os.environ.get("TLS_PENCIL_DIRECT", "1") != "0")
        # unit right-hand sides sorted by the factor position of their 1: the forward sweep skips
        # the columns that are still zero (column j of E is zero above row rows[b, j]).  Bring then
        # has its columns in that order; only the direct pencil below reads it that way (B22's
        # columns and the rows of U are permuted instead of the n x n_b block)
        order = lead = inv = None
        if Dinv is not None and direct and os.environ.get("TLS_RING_SKIP", "1") != "0":
            rows, order = rows.sort(dim=1)
            lead = rows.amin(dim=0).cpu().numpy()
            inv = torch.empty_like(order)
            inv.scatter_(1, order, torch.arange(nbr, device=dev).expand_as(order))
        E.view(len(bs), -1)[torch.arange(len(bs), device=dev)[:, None],
                            rows * nbr + torch.arange(nbr, device=dev)[None, :]] = 1.0
        ts = _stage("coarse: ring rhs", time.perf_counter() if VERBOSE else 0.0)
        if Dinv is not None:   # banded blocked solve (batched GEMMs on the band only)
            X = band_solve_multi(torch, sel(L), sel(Dinv), kc[bs], E, lead)
        else:
            X = torch.cholesky_solve(E, sel(L))                     # A_P^{-1} E  (factor order)
        del E
        Bring = torch.gather(X, 1, pinv[:, :n, None].expand(len(bs), n, nbr))  # local order
        del X
        ts = _stage("coarse: ring solve", ts)
        if kind == "gevp" and n_modes is not None:
            F = Bring[:, :ni]
            B22 = Bring[:, nin:n]
            if inv is not None:  # columns back to the ring order (n_b x n_b only)
                B22 = torch.gather(B22, 2, inv[:, None, :].expand(len(bs), nbr, nbr))
            Ag = sel(A)
            if direct:
                # overlap 1 (F = all non-ring rows of Bring): the rows of A Bring = E_ring give
                # A_II F = -A_IG B22 and A_GI F = I - A_GG B22 (G = ring), hence
                #   H = F^T A_II F = B22 A_GG B22 - B22   and, with B22 = C C^T,
                #   M = C^{-1} H C^{-T} = C^T A_GG C - I
                # -- two GEMMs with the Cholesky factor instead of the sparse-row gathers + GEMM
                # for H and two triangular solves.  The top eigenvalues wanted are O(1) or larger
                # relative to the subtracted identity's rounding (eps * ||C^T A_GG C||).
                ts = _stage("coarse: H = F^T A_II F", ts)
                C, info = torch.linalg.cholesky_ex(0.5 * (B22 + B22.mT))
                M = _ctac(torch, C, Ag[:, nin:n, nin:n])
                M.diagonal(dim1=1, dim2=2).sub_(1.0)
                H = Xs = None
            else:
                H = _harmonic_h(torch, Ag, Bring, n, ni)
                H = 0.5 * (H + H.mT)
                ts = _stage("coarse: H = F^T A_II F", ts)
                C, info = torch.linalg.cholesky_ex(0.5 * (B22 + B22.mT))
                Xs = torch.linalg.solve_triangular(C, H, upper=False)
                M = torch.linalg.solve_triangular(C, Xs.mT, upper=False)
                M = 0.5 * (M + M.mT)
            kk = min(n_modes + 1, nbr)
            ts = _stage("coarse: pencil reduction", ts)
            th, Q, _ = topk_chebyshev(torch, M, kk)
            ts = _stage("coarse: subspace iteration", ts)
            sig = torch.sqrt(torch.clamp(th, min=0.0)).cpu().numpy()
            U = torch.linalg.solve_triangular(C.mT, Q, upper=True)
            if order is not None:  # Bring's columns are in sorted order: permute U's rows to match
                U = torch.gather(U, 1, order[:, :, None].expand(len(bs), nbr, U.shape[2]))
            V = Bring @ U
            idx = torch.argmax(V.abs(), dim=1)
            sgn = torch.where(torch.gather(V, 1, idx[:, None, :])[:, 0, :] < 0, -1.0, 1.0)
            V = V * sgn[:, None, :]
            keeps = [_select(sig[j], tau, n_modes) for j in range(len(bs))]
            kk0 = keeps[0].size
            if all(kp.size == kk0 and np.array_equal(kp, np.arange(kk0)) for kp in keeps):
                # common case (fixed mode count): one batched epilogue for the whole group
                Zg = V[:, :ni, :kk0].contiguous()
                Wg = Ag[:, :n, :ni] @ Zg
                if kk0 and not bool((Zg != 0).any(dim=1).all()):
                    Wg = None  # a zero column: let the caller drop it subdomain by subdomain
                for j, b in enumerate(bs):
                    out[b] = (Zg[j], _cut_gap(sig[j], keeps[j]), None if Wg is None else Wg[j])
            else:
                for j, b in enumerate(bs):
                    out[b] = (V[j][:ni, torch.as_tensor(keeps[j], device=dev)].contiguous(),
                              _cut_gap(sig[j], keeps[j]), None)
            del Ag, H, C, Xs, M, U, V
            ts = _stage("coarse: epilogue", ts)
        else:
            for j, b in enumerate(bs):
                out[b] = _subdomain_columns(torch, kind, A[b], Bring[j], n, ni, nin, tau, n_modes) + (None,)
        del Bring
    return out


def _rank_pivots(torch, z_dev, own, dev):
    """(|R_jj|, subdomain, original column) of the column-pivoted QR of every block z_dev[s]
    (n_int x k), the pivots of src/coarse.py:133-141, computed on the device (K12a)."""
    blocks = [s for s in own if z_dev[s].shape[1] > 0]
    if not blocks:
        return []
    if any(z_dev[s].shape[1] > 64 for s in blocks):  # wide blocks (coarse="full"): host geqp3
        out = []
        for s in blocks:
            r, perm = sla.qr(z_dev[s].cpu().numpy(), mode="r", pivoting=True)
            rd = np.abs(np.diag(r))
            out += [(rd[j] if j < rd.size else 0.0, s, int(perm[j])) for j in range(z_dev[s].shape[1])]
        return out
    W = torch.cat([z_dev[s].mT.contiguous().reshape(-1) for s in blocks])   # column-major blocks
    nr = np.array([z_dev[s].shape[0] for s in blocks], dtype=np.int32)
    nc = np.array([z_dev[s].shape[1] for s in blocks], dtype=np.int32)
    woff = np.concatenate([[0], np.cumsum(nr.astype(np.int64) * nc)[:-1]]).astype(np.int64)
    rd = np.empty(int(nc.sum()), dtype=np.float64)
    pm = np.empty(int(nc.sum()), dtype=np.int32)
    rc = _lib.load().tls_rank_filter_pivots(_lib.ptr(W), _lib.ptr(woff), _lib.ptr(nr), _lib.ptr(nc), len(blocks),
                                            _lib.ptr(rd), _lib.ptr(pm), stream_ptr())
    if rc != 0:
        raise RuntimeError(f"tls_rank_filter_pivots failed ({rc})")
    out, o = [], 0
    for s, k in zip(blocks, nc):
        out += [(float(rd[o + j]), s, int(pm[o + j])) for j in range(int(k))]
        o += int(k)
    return out


def _profile_bytes(adj, perm):
    """Bytes of the 64-blocked band panels of a factor with row order ``perm``."""
    n = perm.size
    pos = np.empty(n, dtype=np.int64)
    pos[perm] = np.arange(n)
    coo = adj.tocoo()
    f = pos.copy()
    np.minimum.at(f, coo.row, pos[coo.col])
    f_by_pos = np.empty(n, dtype=np.int64)
    f_by_pos[pos] = f
    nb = -(-n // 64)
    pad = np.concatenate([f_by_pos, np.arange(n, nb * 64)])
    bmin = pad.reshape(nb, 64).min(axis=1)
    K = np.arange(nb) - bmin // 64
    return float(K.sum() * 64 * 64 * 8 + nb * 2304 * 8)


class _LocalGraphs:
    """Local sparsity graphs of subdomains from the global adjacency: one global->local position
    map (reset after each use) instead of scipy's column fancy-indexing, and an RCM cache keyed
    on the local pattern -- subdomains of a tiled grid share a handful of local patterns."""

    def __init__(self, adj_csr):
        self.adj = adj_csr
        self.pos = np.full(adj_csr.shape[0], -1, dtype=np.int64)
        self.cache = {}

    def local(self, idx):
        """(local row pointer, local columns): per row the diagonal first, then the neighbours
        in DESCENDING global index -- the entry order scipy produces for the pattern of
        ``adj[idx][:, idx] + I`` that RCM walks, so the orders equal the dense-path ones."""
        a = self.adj
        n = idx.size
        self.pos[idx] = np.arange(n)
        starts, ends = a.indptr[idx], a.indptr[idx + 1]
        lens = ends - starts
        tot = int(lens.sum())
        # each row's global columns are ascending in the CSR: read them back to front
        rev = np.repeat(ends - 1 + np.cumsum(np.concatenate([[0], lens[:-1]])), lens) - np.arange(tot)
        lc = self.pos[a.indices[rev]]
        self.pos[idx] = -1
        rows = np.repeat(np.arange(n), lens)
        keep = lc >= 0
        rows, lc = rows[keep], lc[keep]
        cnt = np.bincount(rows, minlength=n) + 1
        ptr = np.concatenate([[0], np.cumsum(cnt)])
        cols = np.empty(int(ptr[-1]), dtype=np.int64)
        cols[ptr[:-1]] = np.arange(n)
        off = np.arange(rows.size) - np.concatenate([[0], np.cumsum(cnt - 1)])[rows]
        cols[ptr[rows] + 1 + off] = lc
        return ptr, cols

    def rcm(self, idx):
        from scipy.sparse.csgraph import reverse_cuthill_mckee
        ptr, cols = self.local(idx)
        key = (idx.size, hash(ptr.tobytes()), hash(cols.tobytes()))
        hit = self.cache.get(key)
        if hit is not None and np.array_equal(hit[0], ptr) and np.array_equal(hit[1], cols):
            return hit[2]
        n = idx.size
        sub = sp.csr_matrix((np.ones(cols.size, dtype=np.int8), cols.astype(np.int32), ptr.astype(np.int32)),
                            shape=(n, n))
        out = np.asarray(reverse_cuthill_mckee(sub, symmetric_mode=True), dtype=np.int64)
        self.cache[key] = (ptr, cols, out)
        return out


_LG = {}


def local_orders(adj_csr, maps, kind):
    """Factor row order of every subdomain: "lex" = ascending global index (a plane sweep for
    grid operators), "rcm" = reverse Cuthill-McKee of the local graph (with the diagonal, as
    scipy's RCM on A_ii's pattern)."""
    out = []
    if kind == "lex":
        return [np.argsort(m.indices, kind="stable").astype(np.int64) for m in maps]
    lg = _LG.get(id(adj_csr))
    if lg is None or lg.adj is not adj_csr:
        _LG.clear()
        lg = _LG[id(adj_csr)] = _LocalGraphs(adj_csr)
    for m in maps:
        out.append(lg.rcm(np.asarray(m.indices, dtype=np.int64)))
    return out


def choose_local_order(adj_csr, maps, symmetric, forced=False):
    """Pick lex or RCM by the band bytes on sample subdomains; None (unless ``forced``) when the
    dense inverse is cheaper to stream (then the inverse-tile path is used)."""
    sample = sorted({0, len(maps) // 2, len(maps) - 1})
    best = None
    for kind in ("lex", "rcm"):
        tot = inv = 0.0
        for s in sample:
            m = maps[s]
            adj = adj_csr[m.indices][:, m.indices]
            perm = local_orders(adj_csr, [m], kind)[0]
            band = _profile_bytes(adj, perm)
            # Cholesky: L read twice; LU: L and U (about twice the lower profile) once each
            tot += 2.0 * band
            n = m.n_local
            inv += (8.0 * n * (n + 1) / 2) if symmetric else 8.0 * n * n
        if best is None or tot < best[1]:
            best = (kind, tot, inv)
    kind, tot, inv = best
    return (kind if forced or tot < 0.8 * inv else None), tot / inv


def lu_growth(torch, csr, maps, perm_kind, adj_csr, device, sample=None):
    """Largest pivot growth max|U| / max|A| of the banded LU on sample subdomains.

    Partial pivoting in a bandwidth-reducing order can grow the factors of saddle-point blocks
    (the tiny pressure block is eliminated early); the reference factors in its own local order.
    A large growth makes the band-LU solve less accurate, so "auto" keeps the inverse tiles then.
    """
    sample = sample or sorted({0, len(maps) // 2, len(maps) - 1})
    worst = 1.0
    for s in sample:
        m = maps[s]
        perm = local_orders(adj_csr, [m], perm_kind)[0]
        blk = csr[m.indices[perm]][:, m.indices[perm]].toarray()
        A = torch.as_tensor(blk, device=device)
        LU, piv, info = torch.linalg.lu_factor_ex(A)
        worst = max(worst, float(torch.triu(LU).abs().max() / A.abs().max()))
    return worst


def _lex_perm(torch, A, perms, n_list, ld):
    cnt = A.shape[0]
    dev = A.device
    Ph = np.tile(np.arange(ld, dtype=np.int64), (cnt, 1))  # built on the host, one upload
    for b in range(cnt):
        Ph[b, : n_list[b]] = perms[b]
    P = torch.from_numpy(Ph).to(dev)
    AP = torch.gather(A, 1, P[:, :, None].expand(cnt, ld, ld))
    AP = torch.gather(AP, 2, P[:, None, :].expand(cnt, ld, ld)).contiguous()
    return AP, P, perms


def _bandwidths(torch, AP):
    """(lower, upper) bandwidth of a batch of dense blocks (max over the batch)."""
    cnt, ld, _ = AP.shape
    ar = torch.arange(ld, device=AP.device)
    lo, up = 0, 0
    for b0 in range(0, cnt, 16):  # bounded temporaries
        nz = AP[b0:b0 + 16] != 0
        has = nz.any(dim=2)
        first = torch.argmax(nz.to(torch.int8), dim=2)
        last = ld - 1 - torch.argmax(torch.flip(nz, dims=[2]).to(torch.int8), dim=2)
        lo = max(lo, int(torch.where(has, ar[None, :] - first, 0).max()))
        up = max(up, int(torch.where(has, last - ar[None, :], 0).max()))
    return lo, up


def band_lu_kernel(torch, AP):
    """K9b (libtls_b200 ``tls_band_lu``): in-place banded LU with partial pivoting of the batch AP
    (cnt, ld, ld); returns (LU, piv, info) in torch.linalg.lu_factor_ex's (LAPACK getrf) format."""
    cnt, ld, _ = AP.shape
    nbk = ld // 64
    kl, ku = _bandwidths(torch, AP)
    J = np.arange(nbk, dtype=np.int64)
    up64 = lambda x: -(-x // 64) * 64  # noqa: E731
    lreach = np.minimum(ld, up64(64 * (J + 1) + kl)).astype(np.int32)
    ureach = np.minimum(ld, up64(64 * (J + 1) + kl + ku)).astype(np.int32)
    piv = torch.empty((cnt, ld), dtype=torch.int32, device=AP.device)
    info = torch.empty(cnt, dtype=torch.int32, device=AP.device)
    AP = AP.contiguous()
    rc = _lib.load().tls_band_lu(_lib.ptr(AP), ld, cnt, _lib.ptr(lreach), _lib.ptr(ureach), nbk, _lib.ptr(piv),
                                 _lib.ptr(info), stream_ptr())
    if rc != 0:
        raise RuntimeError(f"tls_band_lu failed ({rc})")
    return AP, piv, info


def _band_lu_factor(torch, A, perm_list, n_list, ld):
    """Banded LU (partial pivoting) of a batch in lexicographic factor order.

    Returns (LU, piv, Ldinv, Udinv, perm_in, perm_out, lcodes, ucodes, info, P): getrf of
    A_P = P_piv L U; the row interchanges stay inside the band, so L (row profile) and U (last
    nonzero per row) keep narrow profiles; perm_in composes the factor order with the pivots.
    """
    cnt = A.shape[0]
    dev = A.device
    nbk = ld // 64
    AP, P, perms = _lex_perm(torch, A, perm_list, n_list, ld)
    if AP.is_cuda and os.environ.get("TLS_BAND_LU_KERNEL", "1") != "0":
        LU, piv, info = band_lu_kernel(torch, AP)
    else:
        LU, piv, info = torch.linalg.lu_factor_ex(AP)
    del AP
    LU = LU.contiguous()
    nzm = LU != 0
    ar = torch.arange(ld, device=dev)
    lower = nzm & (ar[None, :] < ar[:, None])[None]
    has = lower.any(dim=2)
    firstL = torch.where(has, torch.argmax(lower.to(torch.int8), dim=2), ar[None, :].expand(cnt, ld))
    upper = nzm & (ar[None, :] >= ar[:, None])[None]
    lastU = ld - 1 - torch.argmax(torch.flip(upper, dims=[2]).to(torch.int8), dim=2)
    lastU = torch.maximum(lastU, ar[None, :].expand(cnt, ld))
    del nzm, lower, upper
    fmin = firstL.view(cnt, nbk, 64).min(dim=2).values
    gmax = lastU.view(cnt, nbk, 64).max(dim=2).values
    Ib = torch.arange(nbk, device=dev)[None, :]
    K = (Ib - fmin // 64).clamp(min=0)
    fz = torch.where(K > 0, (fmin % 64) // 8, torch.zeros_like(K))
    R = (gmax // 64 - Ib).clamp(min=0)
    nzs = (gmax - (Ib + 1) * 64) // 8 + 1                 # nonzero strips of the right panel
    tz = torch.where(R > 0, 8 * R - nzs, torch.zeros_like(R))
    lc = (K | (fz << 16)).cpu().numpy().astype(np.int32)
    uc = (R | (tz << 16)).cpu().numpy().astype(np.int32)
    Ld = LU.view(cnt, nbk, 64, nbk, 64).diagonal(dim1=1, dim2=3).permute(0, 3, 1, 2)
    eye = torch.eye(64, dtype=torch.float64, device=dev).expand(cnt, nbk, 64, 64)
    Ldinv = torch.linalg.solve_triangular(Ld, eye, upper=False, unitriangular=True).contiguous()
    Udinv = torch.linalg.solve_triangular(Ld, eye, upper=True).contiguous()
    piv_h = piv.cpu().numpy()
    perm_in, perm_out, lcodes, ucodes = [], [], [], []
    for b in range(cnt):
        n = n_list[b]
        nb = -(-n // 64)
        q = np.arange(ld)
        for i, j in enumerate(piv_h[b] - 1):          # LAPACK interchanges, in order
            if j != i:
                q[i], q[j] = q[j], q[i]
        if q[:n].max() >= n:
            raise RuntimeError("pivoting left the subdomain block")
        perm_out.append(perms[b].astype(np.int32))
        perm_in.append(perms[b][q[:n]].astype(np.int32))
        lcodes.append(lc[b, :nb])
        ucodes.append(uc[b, :nb])
    return LU, piv, Ldinv, Udinv, perm_in, perm_out, lcodes, ucodes, info, P


def _band_cholesky_inplace(torch, AP, kmax):
    """Blocked right-looking Cholesky of a batch of banded SPD matrices, in place (lower).

    ``kmax[I]`` = the batch's largest panel count left of the diagonal in block row I (64-row
    blocks); the factor keeps the row profile of AP (no fill outside the envelope), so step J
    only touches block rows J+1 .. rmax[J] = max{I : I - kmax[I] <= J}: a 64 x 64 batched
    Cholesky, one batched TRSM on the panel below it and one batched GEMM update of the trailing
    band square -- ~n * bandwidth^2 flops instead of the dense n^3 / 3.  Entries above the
    diagonal are zeroed at the end.  Returns (L, info) with info[b] = 1-based row of the first
    non-positive pivot (0 = success), like ``torch.linalg.cholesky_ex``.
    """
    cnt, ld, _ = AP.shape
    nbk = ld // 64
    kmax = np.asarray(kmax, dtype=np.int64)
    rows = np.arange(nbk)
    info = torch.zeros(cnt, dtype=torch.int32, device=AP.device)
    for J in range(nbk):
        j0, j1 = J * 64, (J + 1) * 64
        reach = rows[(rows > J) & (rows - kmax <= J)]
        r1 = (int(reach.max()) + 1) * 64 if reach.size else j1
        D = AP[:, j0:j1, j0:j1]
        Ljj, inf = torch.linalg.cholesky_ex(D)
        info = torch.where((info == 0) & (inf > 0), inf + j0, info)
        D.copy_(Ljj)
        if r1 > j1:
            P = AP[:, j1:r1, j0:j1]
            P.copy_(torch.linalg.solve_triangular(Ljj.mT, P, upper=True, left=False))
            AP[:, j1:r1, j1:r1].baddbmm_(P, P.mT, alpha=-1.0)
    AP.masked_fill_(torch.ones(ld, ld, dtype=torch.bool, device=AP.device).triu_(1), 0.0)
    return AP, info


BAND_CHOL = os.environ.get("TLS_BAND_CHOL", "kernel")


def _band_reach(kmax, nbk):
    """End row of the band below each panel J: rows I > J with I - kmax[I] <= J."""
    rows = np.arange(nbk)
    out = np.empty(nbk, dtype=np.int32)
    for J in range(nbk):
        r = rows[(rows > J) & (rows - kmax <= J)]
        out[J] = (int(r.max()) + 1) * 64 if r.size else (J + 1) * 64
    return out


def band_cholesky_kernel(torch, AP, kmax, clear_upper=True):
    """K9 (libtls_b200 ``tls_band_cholesky``): in-place banded Cholesky of the batch AP
    (cnt, ld, ld) in factor order; returns (L, Dinv, info) like the library path."""
    cnt, ld, _ = AP.shape
    nbk = ld // 64
    reach = _band_reach(np.asarray(kmax, dtype=np.int64), nbk)
    Dinv = torch.empty((cnt, nbk, 64, 64), dtype=torch.float64, device=AP.device)
    info = torch.empty(cnt, dtype=torch.int32, device=AP.device)
    rc = _lib.load().tls_band_cholesky(_lib.ptr(AP), ld, cnt, _lib.ptr(reach), nbk, _lib.ptr(Dinv),
                                       _lib.ptr(info), stream_ptr())
    if rc != 0:
        raise RuntimeError(f"tls_band_cholesky failed ({rc})")
    if clear_upper:  # (tls_perm_lower's output is zero above the diagonal and the kernel keeps it so)
        AP.masked_fill_(torch.ones(ld, ld, dtype=torch.bool, device=AP.device).triu_(1), 0.0)
    return AP, Dinv, info


def _band_factor(torch, A, perm_list, n_list, ld, out=None):
    """Lexicographic factor order, band profile, Cholesky and diagonal-tile inverses of a batch.

    Returns (L_P, Dinv, perms, kcnts, info, P, codes): L_P[b] is the Cholesky factor of A[b] with
    rows and columns in factor order (``perm_list[b]``: ascending global index or RCM), so L is
    banded; kcnts[b][I] = panel tiles left of the diagonal in block-row I; codes add the leading
    all-zero 8-column strips.
    """
    cnt = A.shape[0]
    dev = A.device
    nbk = ld // 64
    use_kernel = A.is_cuda and BAND_CHOL != "torch"
    if use_kernel and os.environ.get("TLS_PERM_KERNEL", "1") != "0":
        # one pass (tls_perm_lower): factor-order lower triangle + row profile
        Ph = np.tile(np.arange(ld, dtype=np.int64), (cnt, 1))
        for b in range(cnt):
            Ph[b, : n_list[b]] = perm_list[b]
        P = torch.from_numpy(Ph).to(dev)
        perms = perm_list
        AP = out[:cnt] if out is not None else torch.empty_like(A)  # (the caller's reused buffer)
        first = torch.empty((cnt, ld), dtype=torch.int32, device=dev)
        rc = _lib.load().tls_perm_lower(_lib.ptr(A), _lib.ptr(P), _lib.ptr(AP), _lib.ptr(first), cnt, ld,
                                        stream_ptr())
        if rc != 0:
            raise RuntimeError(f"tls_perm_lower failed ({rc})")
        first = first.to(torch.int64)
        lower_only = True
    else:
        AP, P, perms = _lex_perm(torch, A, perm_list, n_list, ld)
        first = torch.argmax((AP != 0).to(torch.int8), dim=2)       # row profile f(i)
        lower_only = False
    perms = [p.astype(np.int32) for p in perms]
    fmin = first.view(cnt, nbk, 64).min(dim=2).values
    bmin = fmin // 64
    kc = (torch.arange(nbk, device=dev)[None, :] - bmin).clamp(min=0).cpu().numpy().astype(np.int32)
    # leading all-zero 8-column strips of each panel (the factor keeps the profile of A_P)
    fz = ((fmin % 64) // 8).cpu().numpy().astype(np.int32)
    fz = np.where(kc > 0, fz, 0)
    if BAND_CHOL == "torch" or not AP.is_cuda:  # library path (batched potrf / trsm + bmm per
        # panel); also the CPU-tensor path the host tests of the setup algebra use
        L, info = _band_cholesky_inplace(torch, AP, kc.max(axis=0))
        Ld = L.view(cnt, nbk, 64, nbk, 64).diagonal(dim1=1, dim2=3).permute(0, 3, 1, 2)
        eye = torch.eye(64, dtype=torch.float64, device=dev).expand(cnt, nbk, 64, 64)
        Dinv = torch.linalg.solve_triangular(Ld, eye, upper=False).contiguous()
    else:  # in-tree K9: one launch for the batch, DMMA tile products
        L, Dinv, info = band_cholesky_kernel(torch, AP, kc.max(axis=0), clear_upper=not lower_only)
    kcnts = [kc[b, : -(-n_list[b] // 64)] for b in range(cnt)]
    codes = [(kc[b] | (fz[b] << 16))[: -(-n_list[b] // 64)].astype(np.int32) for b in range(cnt)]
    return L, Dinv, perms, kcnts, info, P, codes


def assemble_a0_columns(maps, owner, z_blocks, w_blocks, counts, own, device):
    """Column blocks of A0 = Z^T (A Z) for the owned subdomains (src/coarse.py:158-168).

    ``w_blocks[s]`` = A_ii[:, :n_int] Z_s on the local rows of s (A Z_s is supported there,
    because every graph neighbour of an interior row lies in layer 1); rows are split by their
    owner j and contracted with Z_j.  Returns the dense n_C x n_C matrix holding only the
    column blocks of ``own`` (sum over ranks = A0).
    """
    torch = _torch()
    cstart = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    nC = int(cstart[-1])
    posint = np.empty(int(max(m.indices.max() for m in maps)) + 1, dtype=np.int64)
    for m in maps:
        posint[m.interior] = np.arange(m.interior.size)
    A0 = torch.zeros((nC, nC), dtype=torch.float64, device=device)
    # host planning: every (s, owner j) group of rows, as slices of two index arrays that are
    # uploaded once (no per-group host->device transfers)
    plan, rows_cat, grp_cat, off = [], [], [], 0
    for s in own:
        if counts[s] == 0:
            continue
        m = maps[s]
        own_rows = owner[m.indices]
        order = np.argsort(own_rows, kind="stable")
        cuts = np.nonzero(np.diff(own_rows[order]))[0] + 1
        for grp in np.split(order, cuts):
            j = int(own_rows[grp[0]])
            if counts[j] == 0:
                continue
            rows_cat.append(posint[m.indices[grp]])
            grp_cat.append(grp)
            plan.append((s, j, off, off + grp.size))
            off += grp.size
    if not plan:
        return A0
    if device.type == "cuda" and max(counts) <= 64:
        # K12b: one CTA per (s, j) block (tls_galerkin_assemble) instead of one small GEMM per pair
        zs = {j: z_blocks[j].contiguous() for j in {p[1] for p in plan}}
        ws = {s: w_blocks[s].contiguous() for s in {p[0] for p in plan}}
        N = len(maps)
        zptr = np.zeros(N, dtype=np.int64)
        wptr = np.zeros(N, dtype=np.int64)
        for j, t in zs.items():
            zptr[j] = t.data_ptr()
        for s, t in ws.items():
            wptr[s] = t.data_ptr()
        sj = np.array([(p[0], p[1]) for p in plan], dtype=np.int32).reshape(-1)
        poff = np.array([p[2] for p in plan] + [plan[-1][3]], dtype=np.int64)
        rows = np.concatenate(rows_cat).astype(np.int64)
        grp = np.concatenate(grp_cat).astype(np.int64)
        kc32 = np.asarray(counts, dtype=np.int32)
        cs64 = cstart.astype(np.int64)
        rc = _lib.load().tls_galerkin_assemble(_lib.ptr(sj), _lib.ptr(poff), len(plan), _lib.ptr(zptr),
                                               _lib.ptr(wptr), _lib.ptr(kc32), _lib.ptr(cs64), N, _lib.ptr(rows),
                                               _lib.ptr(grp), rows.size, _lib.ptr(A0), nC, stream_ptr())
        if rc != 0:
            raise RuntimeError(f"tls_galerkin_assemble failed ({rc})")
        return A0
    rows_d = torch.as_tensor(np.concatenate(rows_cat), device=device)
    grp_d = torch.as_tensor(np.concatenate(grp_cat), device=device)
    for s, j, o0, o1 in plan:
        Zj = z_blocks[j].index_select(0, rows_d[o0:o1])
        Wg = w_blocks[s].index_select(0, grp_d[o0:o1])
        A0[cstart[j]:cstart[j + 1], cstart[s]:cstart[s + 1]] += Zj.mT @ Wg
    return A0


def coarse_bandwidth(maps, owner, counts, own):
    """Half bandwidth (in coarse columns) of A0 = Z^T A Z from its block structure: the block
    (j, s) is structurally nonzero only when subdomain j owns a row of subdomain s's index set
    (the (s, j) groups of ``assemble_a0_columns``); the largest column distance inside such a
    block pair bounds |row - col| over all nonzeros."""
    cstart = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    bw = 0
    for s in own:
        if counts[s] == 0:
            continue
        js = np.unique(owner[maps[s].indices])
        js = js[np.asarray(counts)[js] > 0]
        if js.size == 0:
            continue
        lo_, hi_ = int(min(js.min(), s)), int(max(js.max(), s))
        # farthest column of a coupled block from a column of block s, either side
        bw = max(bw, int(cstart[hi_ + 1] - cstart[s]) - 1, int(cstart[s + 1] - cstart[lo_]) - 1)
    return bw


def spd_inverse_block_tridiagonal(torch, A, bs):
    """In place: the lower triangle (and the full diagonal blocks) of A^{-1} for an SPD matrix
    whose nonzeros lie within the block-tridiagonal pattern of block size ``bs`` (half bandwidth
    < bs); only the lower triangle of ``A`` is read.  Returns 0, or the 1-based index of the
    leading minor that is not positive definite (LAPACK potrf's info).

    A0 = Z^T A Z couples neighbouring subdomains only, so in subdomain order it is banded
    (configuration 5: n_C = 49,152, half bandwidth 3,287).  A dense potrf + potri costs n^3
    flops (119 TFLOP, 7.1 s through cuSOLVER); here
      * block Cholesky of the tridiagonal blocks: L_ii, L_{i+1,i}, and G_i = L_{i+1,i} L_ii^{-1};
      * X = A^{-1} from X L = L^{-T} column block by column block, last to first:
        X_{j,i} = -X_{j,i+1} G_i (j > i),  X_ii = L_ii^{-T} L_ii^{-1} - G_i^T X_{i+1,i}
      -- a right-hand triangular substitution with the Cholesky factor (as backward stable as
      potri's), ~ bs * n^2 flops (11 TFLOP there), all cuBLAS GEMMs on (n - r) x bs panels, and
      one n_C^2 buffer instead of three (src/coarse.py:178-182 factorises A0 and solves).
    """
    n = A.shape[0]
    cuts = list(range(0, n, bs)) + [n]
    nb = len(cuts) - 1
    G = [None] * nb
    Dinv = [None] * nb
    Lprev = None
    for i in range(nb):
        r0, r1 = cuts[i], cuts[i + 1]
        Aii = A[r0:r1, r0:r1]
        if i > 0:
            p0 = cuts[i - 1]
            # L_{i,i-1} = A_{i,i-1} L_{i-1,i-1}^{-T};  G_{i-1} = L_{i,i-1} L_{i-1,i-1}^{-1}
            Lij = torch.linalg.solve_triangular(Lprev, A[r0:r1, p0:r0].mT, upper=False).mT
            Aii = Aii - Lij @ Lij.mT
            G[i - 1] = torch.linalg.solve_triangular(Lprev.mT, Lij.mT, upper=True).mT.contiguous()
            del Lij
        Lii, info = torch.linalg.cholesky_ex(Aii)
        del Aii
        if int(info) != 0:
            return r0 + int(info)
        Dinv[i] = torch.cholesky_inverse(Lii)
        Lprev = Lii
    del Lprev, Lii
    r0 = cuts[nb - 1]
    A[r0:, r0:] = Dinv[nb - 1]
    Dinv[nb - 1] = None
    for i in range(nb - 2, -1, -1):
        r0, r1, r2 = cuts[i], cuts[i + 1], cuts[i + 2]
        A[r1:, r0:r1] = -(A[r1:, r1:r2] @ G[i])
        D = Dinv[i] - G[i].mT @ A[r1:r2, r0:r1]
        A[r0:r1, r0:r1] = 0.5 * (D + D.mT)
        G[i] = Dinv[i] = None
        del D
    return 0


def spd_block_tridiagonal_chain(torch, A, bs):
    """Block-tridiagonal factorisation of an SPD matrix whose nonzeros lie within the
    block-tridiagonal pattern of block size ``bs`` (only the lower triangle of ``A`` is read), for
    the coarse solve by block substitution (``tls_coarse_chain``):

      S_0 = A_00,  S_i = A_ii - A_{i,i-1} S_{i-1}^{-1} A_{i-1,i}   (formed as A_ii - L_{i,i-1} L_{i,i-1}^T
      from the block Cholesky factor, as in ``spd_inverse_block_tridiagonal``).

    Returns ``(info, sinv, lo, up)``: ``info`` = 0 or the 1-based index of the leading minor that
    is not positive definite (LAPACK potrf's info); ``sinv[i]`` = S_i^{-1} (dense, symmetric);
    ``lo`` / ``up`` = (indptr, indices, values) CSR triples (int32 / fp64, device) of the strictly
    block-lower part of A and of its transpose, over all rows, global column indices.
    src/coarse.py:178-182 factorises A0 once and solves with the factor; this is the same
    Cholesky factorisation organised by blocks, n * bs^2 flops instead of n^3 / 3.
    """
    n = A.shape[0]
    dev = A.device
    cuts = list(range(0, n, bs)) + [n]
    nb = len(cuts) - 1
    sinv = []
    lo_r, lo_c, lo_v, up_r, up_c, up_v = [], [], [], [], [], []
    Lprev = None
    for i in range(nb):
        r0, r1 = cuts[i], cuts[i + 1]
        Aii = A[r0:r1, r0:r1]
        if i > 0:
            p0 = cuts[i - 1]
            B = A[r0:r1, p0:r0]
            Lij = torch.linalg.solve_triangular(Lprev, B.mT, upper=False).mT
            Aii = Aii - Lij @ Lij.mT
            del Lij
            nz = B.nonzero()
            lo_r.append(nz[:, 0] + r0)
            lo_c.append(nz[:, 1] + p0)
            lo_v.append(B[nz[:, 0], nz[:, 1]])
            Bt = B.mT.contiguous()
            nz = Bt.nonzero()
            up_r.append(nz[:, 0] + p0)
            up_c.append(nz[:, 1] + r0)
            up_v.append(Bt[nz[:, 0], nz[:, 1]])
            del B, Bt, nz
        Lii, info = torch.linalg.cholesky_ex(Aii)
        del Aii
        if int(info) != 0:
            return r0 + int(info), None, None, None
        D = torch.cholesky_inverse(Lii)
        sinv.append((0.5 * (D + D.mT)).contiguous())
        del D
        Lprev = Lii
    del Lprev, Lii

    def csr(rows, cols, vals):
        if rows:
            r, c, v = torch.cat(rows), torch.cat(cols), torch.cat(vals)
        else:
            r = c = torch.zeros(0, dtype=torch.int64, device=dev)
            v = torch.zeros(0, dtype=torch.float64, device=dev)
        ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        ptr[1:] = torch.cumsum(torch.bincount(r, minlength=n), 0)
        return ptr.to(torch.int32).contiguous(), c.to(torch.int32).contiguous(), v.contiguous()

    return 0, sinv, csr(lo_r, lo_c, lo_v), csr(up_r, up_c, up_v)


def _band_bytes(codes):
    """Device bytes the library allocates for band panels with these codes (band_layout)."""
    k = (np.asarray(codes, dtype=np.int64) & 0xFFFF)
    return 8 * int((k * 4096 + 2304).sum()) + 12 * k.size


def _release_cache(torch, dev, frac=0.25):
    """End of setup: hand torch's cached setup workspace back to the driver only when it is a
    large share of the device (every cudaFree synchronises and costs ms; SURVEY.md §8d TTS)."""
    free, total = torch.cuda.mem_get_info(dev)
    cached = torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
    # ... and only when the device is nearly full: the flush itself cost 5.6 s at the end of a
    # configuration-5 setup (thousands of cudaFree calls), the cached blocks are reused by the
    # solves' work vectors, and torch flushes on its own when an allocation does not fit
    if cached > frac * total and free < 0.1 * total:
        torch.cuda.empty_cache()


def _make_room(torch, dev, nbytes, slack=1 << 29):
    """Return torch's cached blocks to the driver only when the library's next cudaMalloc of
    ``nbytes`` would not fit (emptying the cache every batch costs a re-map of the batch
    buffers)."""
    free, _ = torch.cuda.mem_get_info(dev)
    if free < nbytes + slack:
        torch.cuda.empty_cache()


def build_device_operators(handle, csr, symmetric, maps, owner, coarse, tau, n_modes, drop_tol,
                           batch=None, mem_fraction=0.35, shard=None, local="auto", graph=None, nu=None):
    """Run steps 1-5 into ``handle`` (this rank's slab when ``shard``); returns CoarseData or None.

    ``local``: "inverse" (packed A_ii^{-1} tiles), "band" (banded Cholesky factors; SPD only) or
    "auto" (band for symmetric matrices, inverse otherwise).
    """
    torch = _torch()
    lib = handle.lib
    dev = torch.device("cuda", handle.device)
    N = len(maps)
    n_loc = np.array([m.n_local for m in maps], dtype=np.int64)
    n_int = np.array([m.interior.size for m in maps], dtype=np.int64)
    n_bnd = np.array([m.n_boundary for m in maps], dtype=np.int64)
    sharded = shard is not None and shard.active
    if sharded:
        from .distributed import slab_ranges
        lo, hi = slab_ranges(n_loc.astype(np.float64) ** 2, shard.nranks)[shard.rank]
        shard.lo, shard.hi = lo, hi
        handle.check(lib.tls_set_owned_range(handle.ctx, lo, hi))
        shard.attach(handle)
    else:
        lo, hi = 0, N
    if local not in ("auto", "band", "inverse"):
        raise ValueError(f"unknown local operator kind {local!r}")
    forced = local == "band"
    band = local in ("auto", "band")
    order_kind = None
    if band:
        # k_band_solve keeps a whole local vector in shared memory (csrc/tls_b200.cu
        # band_max_rows): larger subdomains keep the inverse tiles
        optin = int(getattr(torch.cuda.get_device_properties(dev), "shared_memory_per_block_optin",
                            227 * 1024))
        max_rows = (optin // 8 - 8 * 64 - 64) // 64 * 64
        if int(n_loc.max()) > max_rows:
            if forced:
                raise ValueError(f"local='band': a subdomain of {int(n_loc.max())} rows exceeds the "
                                 f"{max_rows}-row shared-memory limit of the band solve")
            band = False
    if band:
        import scipy.sparse as sp
        if graph is None:
            from .partition import symmetrized_graph as _sg
            graph = _sg(csr, symmetric=symmetric)
        adj = sp.csr_matrix((np.ones(graph.adjacency.size, dtype=np.int8), graph.adjacency, graph.indptr),
                            shape=csr.shape)
        order_kind, ratio = choose_local_order(adj, maps, symmetric, forced)
        _log(time.perf_counter(), f"band order {order_kind} (band/inverse bytes {ratio:.2f})")
        if order_kind is None:
            band = False  # "auto": no ordering beats streaming the dense inverse
        elif not symmetric and not forced:
            growth = lu_growth(torch, csr, maps, order_kind, adj, dev)
            _log(time.perf_counter(), f"band LU pivot growth {growth:.2e}")
            if growth > 1.0e3:
                band = False  # keep the inverse tiles (factored in the reference's local order)
    band_lu = band and not symmetric
    handle.local_kind = ("band-lu" if band_lu else "band") if band else "inverse"
    handle.local_order = order_kind
    if band:
        handle.check(lib.tls_set_local_kind(handle.ctx, 2 if band_lu else 1))
    offsets = np.concatenate([[0], np.cumsum(n_loc)]).astype(np.int64)
    indices = np.concatenate([m.indices for m in maps]).astype(np.int64)
    n_int32 = n_int.astype(np.int32)  # keep alive across the call (raw pointer below)
    handle.check(lib.tls_subdomains_upload(handle.ctx, N, _lib.ptr(offsets), _lib.ptr(indices),
                                           _lib.ptr(n_int32)))
    ld = int(n_loc[lo:hi].max())
    if band:
        ld = -(-ld // 64) * 64  # factor tiles are 64 x 64
    if batch is None:
        free, _ = torch.cuda.mem_get_info(dev)
        per = 8.0 * ld * ld * 4.0 + 4.0 * csr.shape[0]
        batch = max(1, min(hi - lo, int(mem_fraction * free / per)))
    s_ptr = stream_ptr()
    want_coarse = coarse != "none"
    z_dev = {}
    w_dev = {}
    gaps = {}
    t0 = time.perf_counter()
    _log(t0, f"subdomains [{lo},{hi}) of {N}, local={local}, ld={ld}, batch={batch}")
    a_buf = torch.empty((min(batch, hi - lo), ld, ld), dtype=torch.float64, device=dev)
    # factor-order copy of the batch (band Cholesky path), allocated once like a_buf
    ap_buf = torch.empty_like(a_buf) if band and not band_lu else None
    # the host factor orders of batch b+1 are computed on one worker thread while batch b's device
    # work runs (the main thread mostly waits in stream syncs); a single worker, so the shared
    # _LocalGraphs scratch is never used by two threads at once
    order_pool = ThreadPoolExecutor(max_workers=1) if band else None

    def _orders_of(f):
        return local_orders(adj, [maps[f + b] for b in range(min(batch, hi - f))], order_kind)

    next_orders = order_pool.submit(_orders_of, lo) if band else None
    try:
        for first in range(lo, hi, batch):
            cnt = min(batch, hi - first)
            if band:
                perm_list = next_orders.result()
                next_orders = order_pool.submit(_orders_of, first + batch) if first + batch < hi else None
            if first > lo:
                _log(t0, f"batch at {first}")
            tb0 = time.perf_counter() if VERBOSE else 0.0
            A = a_buf[:cnt]
            with _nvtx("tls.setup.extract_blocks"):
                handle.check(lib.tls_extract_blocks(handle.ctx, first, cnt, _lib.ptr(A), ld, s_ptr))
            if band_lu:
                n_list = [int(n_loc[first + b]) for b in range(cnt)]
                with _nvtx("tls.setup.band_lu_factor"):
                    LU, piv, Ldinv, Udinv, pin, pout, lcodes, ucodes, info, P = _band_lu_factor(
                        torch, A, perm_list, n_list, ld)
                for b in range(cnt):  # the reference's singularity rule (src/subdomain.py:86-88)
                    nb_ = n_list[b]
                    blk = LU[b, :nb_, :nb_]
                    if int(info[b]) != 0 or float(blk.diagonal().abs().min()) <= nb_ * EPS * float(blk.abs().max()):
                        raise SubdomainSetupError(first + b, "local block is numerically singular")
                pin_c = np.concatenate(pin).astype(np.int32)
                pout_c = np.concatenate(pout).astype(np.int32)
                lc_c = np.concatenate(lcodes).astype(np.int32)
                uc_c = np.concatenate(ucodes).astype(np.int32)
                _make_room(torch, dev, _band_bytes(lc_c) + _band_bytes(uc_c))
                handle.check(lib.tls_store_local_band_lu(handle.ctx, first, cnt, _lib.ptr(LU), ld, _lib.ptr(Ldinv),
                                                         _lib.ptr(Udinv), ld // 64, _lib.ptr(pin_c),
                                                         _lib.ptr(pout_c), _lib.ptr(lc_c), _lib.ptr(uc_c), s_ptr))
                torch.cuda.current_stream().synchronize()
                del Ldinv, Udinv
                if want_coarse and coarse == "svd" and n_modes is not None and nu is None and \
                        os.environ.get("TLS_SVD_GRAM", "1") != "0":
                    for b, (Z, gap) in _svd_columns_lu_batch(torch, A, LU, piv, P, n_loc, n_int, n_bnd, first, cnt,
                                                             ld, tau, n_modes).items():
                        s = first + b
                        n, ni = int(n_loc[s]), int(n_int[s])
                        gaps[s] = gap
                        if Z.shape[1]:
                            nz = torch.any(Z != 0, dim=0)
                            if not bool(nz.all()):
                                Z = Z[:, nz].contiguous()
                        z_dev[s] = Z
                        w_dev[s] = A[b, :n, :ni] @ Z if Z.shape[1] else None
                elif want_coarse:
                    for b in range(cnt):
                        s = first + b
                        n, ni = int(n_loc[s]), int(n_int[s])
                        nin = n - int(n_bnd[s])
                        if n == nin:
                            Bring = torch.zeros((n, 0), dtype=torch.float64, device=dev)
                        else:
                            pinv = torch.empty(ld, dtype=torch.long, device=dev)
                            pinv[P[b]] = torch.arange(ld, device=dev)
                            E = torch.zeros((ld, n - nin), dtype=torch.float64, device=dev)
                            E[pinv[nin:n], torch.arange(n - nin, device=dev)] = 1.0
                            Bring = torch.linalg.lu_solve(LU[b], piv[b], E)[pinv[:n]]
                        Z, gaps[s] = _subdomain_columns(torch, coarse, A[b], Bring, n, ni, nin, tau, n_modes)
                        if Z.shape[1]:
                            nz = torch.any(Z != 0, dim=0)
                            if not bool(nz.all()):
                                Z = Z[:, nz].contiguous()
                        Z = _with_pou(torch, Z, A[b], n, ni, nu)
                        z_dev[s] = Z
                        w_dev[s] = A[b, :n, :ni] @ Z if Z.shape[1] else None
                del A, LU, piv
                continue
            if band:
                tb = _stage("extract", tb0)
                tb = _stage("orders (host, wait)", tb)
                n_list = [int(n_loc[first + b]) for b in range(cnt)]
                with _nvtx("tls.setup.band_factor"):
                    L, Dinv, perms, kcnts, info, P, codes = _band_factor(torch, A, perm_list, n_list, ld,
                                                                         out=ap_buf)
                tb = _stage("band factor", tb)
                bad = torch.nonzero(info).flatten().cpu().numpy()
                if bad.size:
                    s = first + int(bad[0])
                    raise SubdomainSetupError(s, "factorization failed: the local block is not positive definite")
                perm_cat = np.concatenate(perms).astype(np.int32)
                k_cat = np.concatenate(codes).astype(np.int32)
                _make_room(torch, dev, _band_bytes(k_cat))
                handle.check(lib.tls_store_local_band(handle.ctx, first, cnt, _lib.ptr(L), ld, _lib.ptr(Dinv),
                                                      ld // 64, _lib.ptr(perm_cat), _lib.ptr(k_cat), s_ptr))
                torch.cuda.current_stream().synchronize()  # the host arrays above stay alive until here
                tb = _stage("band pack", tb)
                if want_coarse:
                    kc_full = np.zeros((cnt, ld // 64), dtype=np.int64)
                    for b in range(cnt):
                        kc_full[b, : kcnts[b].size] = kcnts[b]
                    with _nvtx("tls.setup.coarse_modes"):
                        cols = _coarse_band_batch(torch, coarse, A, L, P,
                                                  [int(n_loc[first + b]) for b in range(cnt)],
                                                  [int(n_int[first + b]) for b in range(cnt)],
                                                  [int(n_loc[first + b] - n_bnd[first + b]) for b in range(cnt)],
                                                  tau, n_modes, Dinv=Dinv, kc=kc_full)
                    for b in range(cnt):
                        s = first + b
                        n, ni = int(n_loc[s]), int(n_int[s])
                        Z, gaps[s], W = cols[b]
                        if W is None and Z.shape[1]:
                            nz = torch.any(Z != 0, dim=0)
                            if not bool(nz.all()):
                                Z = Z[:, nz].contiguous()
                            W = A[b, :n, :ni] @ Z
                        if nu is not None:
                            Z = _with_pou(torch, Z, A[b], n, ni, nu)
                            W = A[b, :n, :ni] @ Z if Z.shape[1] else None
                        z_dev[s] = Z
                        w_dev[s] = W if Z.shape[1] else None
                del A, L, Dinv
                continue
            if symmetric:
                L, info = torch.linalg.cholesky_ex(A)
                bad = torch.nonzero(info).flatten().cpu().numpy()
                if bad.size:
                    s = first + int(bad[0])
                    raise SubdomainSetupError(s, f"factorization failed: {int(info[bad[0]])}-th leading minor not positive")
                Binv = torch.cholesky_inverse(L)
                del L
                Binv = (0.5 * (Binv + Binv.mT)).contiguous()
            else:
                LU, piv, info = torch.linalg.lu_factor_ex(A)
                for b in range(cnt):
                    s = first + b
                    nb_ = int(n_loc[s])
                    blk = LU[b, :nb_, :nb_]
                    if int(info[b]) != 0 or float(blk.diagonal().abs().min()) <= nb_ * EPS * float(blk.abs().max()):
                        raise SubdomainSetupError(s, "local block is numerically singular")
                eye = torch.eye(ld, dtype=torch.float64, device=dev).expand(cnt, ld, ld)
                Binv = torch.linalg.lu_solve(LU, piv, eye).contiguous()  # lu_solve returns column-major
                del LU, piv
            handle.check(lib.tls_store_local_inverse(handle.ctx, first, cnt, _lib.ptr(Binv), ld, s_ptr))
            if want_coarse:
                for b in range(cnt):
                    s = first + b
                    n, ni = int(n_loc[s]), int(n_int[s])
                    nin = n - int(n_bnd[s])
                    Z, gaps[s] = _subdomain_columns(torch, coarse, A[b], Binv[b, :n, nin:n], n, ni, nin, tau,
                                                    n_modes)
                    # assemble_coarse_basis drops identically zero columns (src/coarse.py:99-103)
                    if Z.shape[1]:
                        nz = torch.any(Z != 0, dim=0)
                        if not bool(nz.all()):
                            Z = Z[:, nz].contiguous()
                    Z = _with_pou(torch, Z, A[b], n, ni, nu)
                    z_dev[s] = Z
                    w_dev[s] = A[b, :n, :ni] @ Z if Z.shape[1] else None
            del A, Binv
    finally:
        # an error in a batch must not leave the next batch's order computation running
        if order_pool is not None:
            order_pool.shutdown(cancel_futures=True)
    del a_buf, ap_buf
    if not want_coarse:
        _release_cache(torch, dev)
        return None
    # rank filter (src/coarse.py:119-155): pivoted-QR magnitudes vs the GLOBAL largest pivot
    own = range(lo, hi)
    # one device->host copy of every owned block (the host keeps the basis for CoarseData), and
    # the column-pivoted QR of every block on the device (K12a, tls_rank_filter_pivots; the
    # reference runs LAPACK geqp3 per block)
    # Defragment before the coarse stage: the per-group Z / W blocks were allocated between the
    # multi-GB batch workspaces, so they pin partly-used allocator segments that empty_cache()
    # cannot return.  Copy them into two flat tensors (views replace the blocks) and release the
    # rest: the three n_C^2 coarse buffers (58 GB on configuration 5, next to 95 GB of factors)
    # then get whole segments.  (PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True also avoids the
    # fragmentation but measured +3 s on the cold setups of configurations 2-4: every fresh block
    # is mapped page by page.)
    zflat = torch.cat([z_dev[s].reshape(-1) for s in own]) if len(own) else torch.zeros(0, dtype=torch.float64,
                                                                                         device=dev)
    off = 0
    for s in own:
        sh = tuple(z_dev[s].shape)
        z_dev[s] = zflat[off:off + sh[0] * sh[1]].view(sh)
        off += sh[0] * sh[1]
    wl = [s for s in own if w_dev.get(s) is not None]
    if wl:
        wflat = torch.cat([w_dev[s].reshape(-1) for s in wl])
        off = 0
        for s in wl:
            sh = tuple(w_dev[s].shape)
            w_dev[s] = wflat[off:off + sh[0] * sh[1]].view(sh)
            off += sh[0] * sh[1]
        del wflat
    _release_cache(torch, dev)
    # one GPU: the host copy of the basis (CoarseData._z, behind the ``basis`` attribute of
    # src/coarse.py:23-38) is fetched from the library on first use, not during setup
    # (configuration 5: 1.6 GB through pageable memory, 1.2 s); sharded: copied now (the blocks of
    # the other ranks are gathered below)
    z_host = {}
    if sharded:
        flat = zflat.cpu().numpy() if len(own) else np.zeros(0)
        off = 0
        for s in own:
            sh = tuple(z_dev[s].shape)
            z_host[s] = flat[off:off + sh[0] * sh[1]].reshape(sh)
            off += sh[0] * sh[1]
    del zflat
    _log(t0, "basis defragmented; rank filter")
    pivots = _rank_pivots(torch, z_dev, own, dev) if len(own) else []
    _log(t0, "rank filter done")
    largest = max((p[0] for p in pivots), default=0.0)
    any_cols = float(len(pivots))
    if sharded:
        t = torch.tensor([largest, any_cols], dtype=torch.float64, device=dev)
        shard.coll.allreduce(t, op="max")
        largest, any_cols = float(t[0]), float(t[1])
    keep_cols = {s: [] for s in own}
    for mag, s, j in pivots:
        if mag >= drop_tol * largest:
            keep_cols[s].append(j)
    for s in own:
        kc = sorted(keep_cols[s])
        if len(kc) != z_dev[s].shape[1]:
            idx = torch.as_tensor(kc, dtype=torch.long, device=dev)
            z_dev[s] = z_dev[s][:, idx].contiguous()
            w_dev[s] = w_dev[s][:, idx].contiguous() if len(kc) else None
            if s in z_host:
                z_host[s] = z_host[s][:, kc]
    counts_own = np.array([z_dev[s].shape[1] for s in own], dtype=np.int64)
    if sharded:
        parts = shard.coll.allgather_list(torch.as_tensor(counts_own, device=dev))
        counts = np.concatenate([p.cpu().numpy() for p in parts]).astype(np.int64)
        flat = torch.cat([z_dev[s].reshape(-1) for s in own]) if len(own) else torch.zeros(0, device=dev)
        zparts = shard.coll.allgather_list(flat.to(torch.float64))
        z_all = {}
        # unpack every rank's concatenated blocks in global subdomain order
        from .distributed import slab_ranges
        ranges = slab_ranges(n_loc.astype(np.float64) ** 2, shard.nranks)
        for (rlo, rhi), zp in zip(ranges, zparts):
            off = 0
            for s in range(rlo, rhi):
                sz = int(n_int[s]) * int(counts[s])
                z_all[s] = zp[off:off + sz].reshape(int(n_int[s]), int(counts[s]))
                off += sz
    else:
        counts = counts_own
        z_all = z_dev
    if counts.sum() == 0:
        if any_cols > 0:
            warnings.warn("rank filter removed every coarse column; coarse level disabled")
        _release_cache(torch, dev)
        return CoarseData(csr.shape[0], maps, [np.zeros((int(n_int[s]), 0)) for s in range(N)],
                          [0] * N, 0) if any_cols > 0 else None
    nC = int(counts.sum())
    owner = np.asarray(owner, dtype=np.int64)
    # half bandwidth of A0 from its block structure (max over the ranks)
    a0_band = coarse_bandwidth(maps, owner, counts, own) if symmetric else nC
    if sharded:
        t = torch.tensor([float(a0_band)], dtype=torch.float64, device=dev)
        shard.coll.allreduce(t, op="max")
        a0_band = int(t[0])
    banded = (symmetric and nC >= BAND_INVERSE_MIN and 4 * (-(-(a0_band + 1) // 64) * 64) <= nC
              and os.environ.get("TLS_A0_BANDED", "1") != "0")
    # dense path: A0, its factor and inverse (torch allocations); banded: one buffer + panels
    _make_room(torch, dev, 8 * nC * nC * (3 if not banded else 1) + (8 * nC * 4 * a0_band if banded else 0))
    if VERBOSE:
        _log(t0, "stage times: " + ", ".join(f"{k} {v:.2f}s" for k, v in _STAGE.items()))
    _log(t0, f"local operators done; assembling A0 ({nC} x {nC})")
    with _nvtx("tls.setup.galerkin_a0"):
        A0 = assemble_a0_columns(maps, owner, z_all, w_dev, counts, own, dev)
    del w_dev
    if sharded:
        shard.coll.allreduce(A0, op="sum")
    # count_nonzero (src/coarse.py:168) in row blocks: no n_C^2 temporary next to A0
    nnz = sum(int(torch.count_nonzero(A0[i:i + 4096])) for i in range(0, nC, 4096))
    _log(t0, "A0 assembled; factorising")
    # A0 itself is kept on the device when it is small (<= 4 GB): the ``a00`` attribute
    # (src/coarse.py:26) and the coarse refinement step read it; larger A0 (configuration 5:
    # 19.3 GB) is rebuilt on demand from the basis
    keep_a0 = 8 * nC * nC <= (4 << 30)
    norm_a0 = None
    if not keep_a0 and not banded:  # the factor and the inverse are two more n_C^2 buffers: defragment first
        torch.cuda.empty_cache()
    if symmetric:
        # symmetrise (src/coarse.py:169-170) the lower triangle Cholesky reads, in place
        _symmetrize_lower_inplace(torch, A0)
        if keep_a0:
            A0 = torch.tril(A0) + torch.tril(A0, -1).mT
            norm_a0 = float(A0.abs().sum(0).max())
        # A0 couples neighbouring subdomains only: when its band is narrow (configuration 5:
        # 3.3k of 49k) the inverse comes from the block-tridiagonal recurrences, in place
        bs = -(-(a0_band + 1) // 64) * 64
        chain = banded and nC >= _chain_min()
        if chain:
            # TLS_A0_CHAIN_MUL: blocks of mul * (smallest admissible size) -- fewer, larger steps
            mul = max(1, int(os.environ.get("TLS_A0_CHAIN_MUL", "1")))
            while mul > 1 and -(-nC // (bs * mul)) < 2:
                mul -= 1
            bs *= mul
            info, sinv, lo_csr, up_csr = spd_block_tridiagonal_chain(torch, A0, bs)
            if info != 0:
                raise RuntimeError(f"coarse operator is not positive definite: {info}-th leading minor")
            if not keep_a0:
                A0 = None
            A0inv = None
            _log(t0, f"A0 factorised by blocks for the block-tridiagonal coarse solve (half bandwidth "
                     f"{a0_band}, block {bs}, {len(sinv)} blocks, {int(lo_csr[2].numel())} off-diagonal entries)")
        elif banded:
            A0inv = A0.clone() if keep_a0 else A0
            if not keep_a0:
                A0 = None
            info = spd_inverse_block_tridiagonal(torch, A0inv, bs)
            if info != 0:
                raise RuntimeError(f"coarse operator is not positive definite: {info}-th leading minor")
            if keep_a0:  # cond_1 below sums whole columns
                A0inv = torch.tril(A0inv) + torch.tril(A0inv, -1).mT
            _log(t0, f"A0^-1 by block-tridiagonal recurrences (half bandwidth {a0_band}, block {bs})")
        else:
            L, info = torch.linalg.cholesky_ex(A0)
            if not keep_a0:
                del A0
                A0 = None
            if int(info) != 0:
                raise RuntimeError(f"coarse operator is not positive definite: {int(info)}-th leading minor")
            # the packed-tile store reads the lower triangle (and full diagonal tiles) only
            A0inv = torch.cholesky_inverse(L).contiguous()
            del L
    else:
        norm_a0 = float(A0.abs().sum(0).max())
        LU, piv, info = torch.linalg.lu_factor_ex(A0)
        if not keep_a0:
            del A0
            A0 = None
        if int(info) != 0 or float(LU.diagonal().abs().min()) <= nC * EPS * float(LU.abs().max()):
            raise RuntimeError("coarse operator is numerically singular")
        A0inv = torch.linalg.lu_solve(LU, piv, torch.eye(nC, dtype=torch.float64, device=dev)).contiguous()
        del LU, piv
    # 1-norm condition number ||A0||_1 ||A0^{-1}||_1 (both explicit here): above 1e8 the explicit
    # inverse alone leaves a coarse residual ~cond * eps, so every coarse solve gets one
    # refinement step (tls_coarse_refine) -- the reference's LU/Cholesky solve is backward stable
    cond1 = norm_a0 * float(A0inv.abs().sum(0).max()) if norm_a0 is not None and A0inv is not None else None
    refine = (A0 is not None and cond1 is not None and cond1 > REFINE_COND and not sharded
              and os.environ.get("TLS_COARSE_REFINE", "1") != "0")
    _log(t0, "coarse operator inverted; uploading")
    # column-major blocks (k x n_int): coalesced restriction and prolongation loads
    zcat = (torch.cat([z_dev[s].mT.contiguous().reshape(-1) for s in own]) if len(own) else
            torch.zeros(1, dtype=torch.float64, device=dev)).contiguous()
    k32 = np.asarray(counts, dtype=np.int32)
    # the library cudaMalloc's the packed coarse operator (~4 nC^2 bytes, 8 nC^2 if general):
    # torch's cached blocks go back to the driver only when that would not fit
    if A0inv is None:  # block-tridiagonal coarse solve: the inverted Schur blocks + sparse off-diagonals
        _make_room(torch, dev, sum(4 * t.numel() + 8 * 64 * t.shape[0] for t in sinv) + 24 * int(lo_csr[2].numel()))
        handle.check(lib.tls_coarse_upload(handle.ctx, nC, _lib.ptr(k32), _lib.ptr(zcat), None, s_ptr))
        ptrs = np.array([t.data_ptr() for t in sinv], dtype=np.uint64)
        handle.check(lib.tls_coarse_chain(handle.ctx, len(sinv), bs, _lib.ptr(ptrs),
                                          _lib.ptr(lo_csr[0]), _lib.ptr(lo_csr[1]), _lib.ptr(lo_csr[2]),
                                          _lib.ptr(up_csr[0]), _lib.ptr(up_csr[1]), _lib.ptr(up_csr[2]),
                                          int(lo_csr[2].numel()), s_ptr))
        torch.cuda.current_stream().synchronize()
        del sinv, lo_csr, up_csr
    else:
        _make_room(torch, dev, 8 * nC * nC if not symmetric else 4 * nC * nC + 8 * nC * 64)
        handle.check(lib.tls_coarse_upload(handle.ctx, nC, _lib.ptr(k32), _lib.ptr(zcat),
                                           _lib.ptr(A0inv), s_ptr))
    if sharded:  # the restriction's all-gather layout: rank q's columns are contiguous
        from .distributed import slab_ranges
        csum = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        starts = np.array([csum[rlo] for rlo, _ in slab_ranges(n_loc.astype(np.float64) ** 2, shard.nranks)]
                          + [nC], dtype=np.int64)
        handle.check(lib.tls_set_coarse_layout(handle.ctx, shard.nranks, _lib.ptr(starts)))
    if refine:
        _make_room(torch, dev, 8 * nC * nC)
        handle.check(lib.tls_coarse_refine(handle.ctx, _lib.ptr(A0.contiguous()), s_ptr))
    torch.cuda.current_stream().synchronize()
    _log(t0, "coarse operator uploaded")
    if sharded:
        z_list = [z_host[s] if s in z_host else z_all[s].cpu().numpy() for s in range(N)]
    else:
        z_list = _LazyBasisBlocks(handle, [int(n_int[s]) for s in range(N)], [int(c) for c in counts])
    del A0inv, zcat, z_dev, z_all
    _release_cache(torch, dev)
    cd = CoarseData(csr.shape[0], maps, z_list, [int(c) for c in counts], nnz)
    cd.cut_gaps = gaps  # owned subdomains only
    cd.cond1 = cond1
    cd.refined = refine
    cd._a00_dev = A0
    cd._csr = csr
    cd._symmetric = symmetric
    _log(t0, "build_device_operators done")
    return cd
