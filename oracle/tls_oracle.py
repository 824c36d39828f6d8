"""CPU oracle for the two-level Schwarz Krylov hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference algorithm
(``tlschwarz``, /root/reference/pkg/src/tlschwarz) for the path named in
BASELINE.json's north star.  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it.  The product package
(``paper_2401_03915_b200``) never imports it and has no CPU fallback.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by running the *reference itself* in this
container (``oracle/make_golden.py`` → ``tests/golden/*.npz``).

The reference's arithmetic lives in numpy >= 1.24 / scipy >= 1.10 (unpinned,
``pkg/pyproject.toml:9-12``; this container: numpy 2.3.5, scipy 1.18.1 with
OpenBLAS 0.3.30), so the oracle calls the same LAPACK drivers.

Two oracle-side adapters that the reference lacks:
* ``n_modes`` — fixed top-k coarse vectors per subdomain: the reference's
  selection with tau = 1e-300, first k columns kept.
* ``gmres_restarted`` — GMRES(m) as repeated reference GMRES cycles on the
  current true residual with the tolerance rescaled to the original ||b||.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.linalg import cho_factor, cho_solve, eigh, lu_factor, lu_solve, qr, solve_triangular

TIE_GUARD = 1e-12          # src/spectral.py:31
DROP_TOL = 1e-10           # src/coarse.py:20
REORTH_TOL = 1e-8          # src/krylov.py:19
GMRES_MAXIT_CAP = 1000     # src/krylov.py:18
TOPK_TAU = 1e-300          # top-k adapter threshold


class OracleBreakdown(RuntimeError):
    def __init__(self, iteration, curvature):
        super().__init__(f"non-positive curvature {curvature:.3e} at iteration {iteration}")
        self.iteration = iteration
        self.curvature = curvature


# -- graph, overlap, colouring ---------------------------------------------------

def symmetrized_graph(a):
    """Edges where |a_ij| > 0 or |a_ji| > 0, i != j (src/sparsemat.py:180-195)."""
    a = sp.csr_matrix(a)
    pat = sp.csr_matrix((np.abs(a.data), a.indices.copy(), a.indptr.copy()), shape=a.shape)
    pat.eliminate_zeros()
    pat = (pat + pat.T).tocsr()
    pat.setdiag(0.0)
    pat.eliminate_zeros()
    pat.sort_indices()
    return pat.indptr.astype(np.int64), pat.indices.astype(np.int64)


def extend_overlap(gptr, gadj, owner, n_sub, overlap):
    """Interior + BFS rings sorted ascending (src/partition.py:278-301).

    Returns a list of (interior, [layer_1, ..., layer_delta]).
    """
    n = gptr.size - 1
    maps = []
    for s in range(n_sub):
        interior = np.nonzero(owner == s)[0].astype(np.int64)
        seen = np.zeros(n, dtype=bool)
        seen[interior] = True
        layers = []
        front = interior
        for _ in range(overlap):
            nb = np.concatenate([gadj[gptr[u]:gptr[u + 1]] for u in front]) if front.size else np.empty(0, np.int64)
            ring = np.unique(nb)
            ring = ring[~seen[ring]]
            seen[ring] = True
            layers.append(ring.astype(np.int64))
            front = ring
        maps.append((interior, layers))
    return maps


def indices_of(mp):
    interior, layers = mp
    return np.concatenate([interior] + list(layers)) if layers else interior.copy()


def color_subdomains(maps, n):
    """Greedy largest-degree-first colouring (src/partition.py:304-334)."""
    n_sub = len(maps)
    incident = [[] for _ in range(n)]
    for s, mp in enumerate(maps):
        for g in indices_of(mp):
            incident[g].append(s)
    adj = [set() for _ in range(n_sub)]
    for subs in incident:
        for a in subs:
            for b in subs:
                if a != b:
                    adj[a].add(b)
    order = sorted(range(n_sub), key=lambda i: (-len(adj[i]), i))
    colors = np.full(n_sub, -1, dtype=np.int64)
    for i in order:
        used = {colors[j] for j in adj[i] if colors[j] >= 0}
        c = 0
        while c in used:
            c += 1
        colors[i] = c
    return int(colors.max()) + 1, colors


# -- local algebra ---------------------------------------------------------------

def _factor(a, symmetric):
    """Cholesky (upper) or pivoted LU + singular check (src/subdomain.py:72-95)."""
    if a.shape[0] == 0:
        return lambda rhs: np.zeros_like(rhs, dtype=np.float64)
    if symmetric:
        fac = cho_factor(a)
        return lambda rhs: cho_solve(fac, rhs)
    lu, piv = lu_factor(a)
    if np.abs(np.diag(lu)).min() <= a.shape[0] * np.finfo(float).eps * np.abs(lu).max():
        raise np.linalg.LinAlgError("local block is numerically singular")
    return lambda rhs: lu_solve((lu, piv), rhs)


def _fix_signs(v):
    """Largest-magnitude component positive (src/spectral.py:59-66)."""
    for j in range(v.shape[1]):
        k = int(np.argmax(np.abs(v[:, j])))
        if v[k, j] < 0:
            v[:, j] = -v[:, j]
    return v


class OracleSubdomain:
    """Dense block, factor, harmonic extension of one subdomain."""

    def __init__(self, a_csr, mp, symmetric):
        self.interior, self.layers = mp
        self.indices = indices_of(mp)
        self.n_local = self.indices.size
        self.n_int = self.interior.size
        self.n_bnd = self.layers[-1].size if self.layers else 0
        self.n_inner = self.n_local - self.n_bnd
        self.mask = np.zeros(self.n_local)
        self.mask[: self.n_int] = 1.0
        self.a = a_csr[self.indices][:, self.indices].toarray()   # src/subdomain.py:59-60
        self.symmetric = symmetric
        self.solve = _factor(self.a, symmetric)

    def extension(self):
        """[-A_inner^{-1} A_inner,ring ; I] (src/subdomain.py:108-120)."""
        ni, nb = self.n_inner, self.n_bnd
        ext = np.zeros((self.n_local, nb))
        if nb:
            if ni:
                ext[:ni] = -_factor(self.a[:ni, :ni], self.symmetric)(self.a[:ni, ni:])
            ext[ni:] = np.eye(nb)
        return ext


def harmonic_modes(sd, ext, tau, n_modes=None):
    """Harmonic-pencil modes (src/spectral.py:111-132) [+ top-k adapter]."""
    m, ni = sd.n_local, sd.n_inner
    masked = ext * sd.mask[:, None]
    gram = masked.T @ sd.a @ masked
    lhs = np.zeros((m, m))
    lhs[ni:, ni:] = 0.5 * (gram + gram.T)
    vals, vecs = eigh(lhs, sd.a)
    vals = vals[::-1].copy()
    vecs = _fix_signs(vecs[:, ::-1].copy())
    sig = np.sqrt(np.clip(vals, 0.0, None))
    thr = TOPK_TAU if n_modes is not None else tau
    keep = sig > thr * (1.0 + TIE_GUARD)
    vecs, sig_sel = vecs[:, keep], sig[keep]
    if n_modes is not None:
        vecs, sig_sel = vecs[:, :n_modes], sig_sel[:n_modes]
    return vecs, sig_sel, sig


def svd_modes(sd, ext, tau, n_modes=None):
    """Left singular vectors of ext[:n_interior] (src/spectral.py:135-154)."""
    m, ni = sd.n_local, sd.n_int
    block = ext[:ni, :]
    if block.size == 0:
        return np.zeros((m, 0)), np.zeros(0), np.zeros(0)
    u, s, _ = np.linalg.svd(block, full_matrices=False)
    thr = TOPK_TAU if n_modes is not None else tau
    keep = s > thr * (1.0 + TIE_GUARD)
    if n_modes is not None:
        idx = np.nonzero(keep)[0][:n_modes]
        keep = np.zeros_like(keep)
        keep[idx] = True
    vec = np.zeros((m, int(keep.sum())))
    vec[:ni] = u[:, keep]
    return _fix_signs(vec), s[keep], s.copy()


# -- the oracle preconditioner -----------------------------------------------------

class OraclePreconditioner:
    """setup + apply restated (src/precond.py:142-257, 114-136)."""

    def __init__(self, a_csr, symmetric, owner, n_sub, overlap=2, tau=0.1, coarse="auto",
                 one_level=None, combine=None, drop_tol=DROP_TOL, n_modes=None):
        self.a = sp.csr_matrix(a_csr)
        self.symmetric = bool(symmetric)
        if coarse == "auto":
            coarse = "gevp" if symmetric else "svd"
        one_level = one_level or ("asm" if symmetric else "ras")
        combine = combine or ("additive" if symmetric else "deflated")
        if coarse == "none":
            combine = "none"
        self.coarse_kind, self.one_level, self.combine = coarse, one_level, combine
        self.n = self.a.shape[0]
        gptr, gadj = symmetrized_graph(self.a)
        self.owner = np.asarray(owner, dtype=np.int64)
        self.maps = extend_overlap(gptr, gadj, self.owner, n_sub, overlap)
        self.k_c, self.colors = color_subdomains(self.maps, self.n)
        self.subs = [OracleSubdomain(self.a, mp, symmetric) for mp in self.maps]
        self.basis = None
        self.mode_counts = tuple(0 for _ in self.subs)
        self.n_coarse = 0
        self.nnz_a00 = 0
        if coarse != "none":
            self._build_coarse(coarse, tau, drop_tol, n_modes)

    def _build_coarse(self, kind, tau, drop_tol, n_modes):
        blocks = []
        for sd in self.subs:
            ext = sd.extension()
            if kind == "full":
                cols = ext * sd.mask[:, None]                      # src/coarse.py:66-67
            elif kind == "gevp":
                vecs, _, _ = harmonic_modes(sd, ext, tau, n_modes)
                cols = (ext @ vecs[sd.n_inner:, :]) * sd.mask[:, None]   # src/coarse.py:68-73
            else:
                cols, _, _ = svd_modes(sd, ext, tau, n_modes)      # src/coarse.py:74-78
            blocks.append(cols)
        # assemble: drop identically-zero columns (src/coarse.py:88-116)
        rows, cidx, vals, ranges, k = [], [], [], [], 0
        kept_blocks = []
        for sd, blk in zip(self.subs, blocks):
            start = k
            keep = [j for j in range(blk.shape[1]) if np.any(blk[:, j] != 0)]
            kept_blocks.append(blk[:, keep])
            k += len(keep)
            ranges.append((start, k))
        # rank filter: per-subdomain pivoted QR vs global largest pivot (src/coarse.py:119-155)
        piv = []
        for (s0, s1), blk in zip(ranges, kept_blocks):
            if s1 == s0:
                continue
            r, perm = qr(blk, mode="r", pivoting=True)
            rd = np.abs(np.diag(r))
            for j in range(blk.shape[1]):
                piv.append((rd[j] if j < rd.size else 0.0, s0 + perm[j]))
        if not piv:
            self._disable_coarse(ranges)
            return
        largest = max(mg for mg, _ in piv)
        keep = set(c for mg, c in piv if mg >= drop_tol * largest)
        if not keep:
            self._disable_coarse(ranges)
            return
        cols_all, counts, k = [], [], 0
        for sd, (s0, s1), blk in zip(self.subs, ranges, kept_blocks):
            sel = [j for j in range(s1 - s0) if (s0 + j) in keep]
            counts.append(len(sel))
            for j in sel:
                col = blk[:, j]
                nz = np.nonzero(col)[0]
                rows.append(sd.indices[nz]); cidx.append(np.full(nz.size, k)); vals.append(col[nz])
                k += 1
        self.mode_counts = tuple(counts)
        self.n_coarse = k
        self.basis = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cidx))),
                                   shape=(self.n, k))
        # Galerkin operator (src/coarse.py:158-183)
        prod = (self.basis.T @ (self.a @ self.basis)).toarray()
        if self.symmetric:
            prod = 0.5 * (prod + prod.T)
        self.nnz_a00 = int(np.count_nonzero(prod))
        self.a00 = prod
        if self.symmetric:
            fac = cho_factor(prod)
            self._csolve = lambda rhs: cho_solve(fac, rhs)
        else:
            lu, pv = lu_factor(prod)
            if np.abs(np.diag(lu)).min() <= prod.shape[0] * np.finfo(float).eps * np.abs(lu).max():
                raise RuntimeError("coarse operator is numerically singular")
            self._csolve = lambda rhs: lu_solve((lu, pv), rhs)

    def _disable_coarse(self, ranges):
        self.basis = None
        self.combine = "none"
        self.mode_counts = tuple(0 for _ in ranges)

    # -- apply (src/precond.py:114-136)
    def apply_one_level(self, r):
        out = np.zeros(self.n)
        for sd in self.subs:
            y = sd.solve(r[sd.indices])
            if self.one_level == "ras":
                y = y * sd.mask
            np.add.at(out, sd.indices, y)
        return out

    def coarse_apply(self, r):
        return self.basis @ self._csolve(self.basis.T @ r)

    def apply(self, r):
        r = np.asarray(r, dtype=np.float64)
        if self.basis is None or self.combine == "none":
            return self.apply_one_level(r)
        if self.combine == "additive":
            return self.apply_one_level(r) + self.coarse_apply(r)
        q = self.coarse_apply(r)
        w = self.apply_one_level(r - self.a @ q)
        return q + w - self.coarse_apply(self.a @ w)


# -- Krylov (src/krylov.py:58-107, 127-195) ------------------------------------------

def pcg(a, precond, b, tol=1e-8, maxit=500):
    """Returns (x, iterations, converged, history)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return x, 0, True, np.zeros(1)
    app = (lambda v: v.copy()) if precond is None else precond.apply
    r = b.copy()
    z = app(r)
    p = z.copy()
    rz = float(r @ z)
    hist = [1.0]
    conv = False
    it = 0
    for it in range(1, maxit + 1):
        ap = a @ p
        curv = float(p @ ap)
        if curv <= 0.0:
            raise OracleBreakdown(it, curv)
        alpha = rz / curv
        x += alpha * p
        r -= alpha * ap
        if it % 25 == 0:
            r = b - a @ x
        hist.append(float(np.linalg.norm(r)) / bn)
        if hist[-1] <= tol:
            conv = True
            break
        z = app(r)
        rzn = float(r @ z)
        beta = rzn / rz
        p = z + beta * p
        rz = rzn
    return x, it, conv, np.asarray(hist)


def gmres(a, precond, b, tol=1e-8, maxit=500):
    """Unrestarted right-preconditioned GMRES; returns (x, k, converged, history)."""
    if maxit > GMRES_MAXIT_CAP:
        raise ValueError(f"maxit {maxit} exceeds the hard cap {GMRES_MAXIT_CAP}")
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return np.zeros(n), 0, True, np.zeros(1)
    app = (lambda v: v.copy()) if precond is None else precond.apply
    m = min(maxit, n)
    V = np.zeros((n, m + 1))
    H = np.zeros((m + 1, m))
    cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
    g[0] = bn
    V[:, 0] = b / bn
    hist = [1.0]
    conv = False
    k = 0
    for j in range(m):
        w = a @ app(V[:, j])
        nb0 = float(np.linalg.norm(w))
        for i in range(j + 1):
            h = float(V[:, i] @ w)
            H[i, j] = h
            w -= h * V[:, i]
        corr = V[:, : j + 1].T @ w
        if float(np.linalg.norm(corr)) > REORTH_TOL * max(nb0, 1e-300):
            w -= V[:, : j + 1] @ corr
            H[: j + 1, j] += corr
        hn = float(np.linalg.norm(w))
        H[j + 1, j] = hn
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        den = np.hypot(H[j, j], H[j + 1, j])
        cs[j] = H[j, j] / den if den else 1.0
        sn[j] = H[j + 1, j] / den if den else 0.0
        H[j, j] = den
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        k = j + 1
        hist.append(abs(g[j + 1]) / bn)
        if hist[-1] <= tol:
            conv = True
            break
        if hn <= 1e-14 * bn:
            conv = True
            break
        V[:, j + 1] = w / hn
    y = solve_triangular(H[:k, :k], g[:k])
    x = app(V[:, :k] @ y)
    return x, k, conv, np.asarray(hist)


def gmres_restarted(a, precond, b, tol=1e-8, maxit=500, restart=None):
    """GMRES(restart) adapter over reference cycles.

    Cycle c solves A d = r_c = b - A x_c with tolerance tol*||b||/||r_c|| and
    at most min(restart, remaining) steps; x_{c+1} = x_c + d.  The history
    is relative to the original ||b||; iterations are summed over cycles.
    """
    if restart is None or restart >= maxit:
        return gmres(a, precond, b, tol, maxit)
    b = np.asarray(b, dtype=np.float64)
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return np.zeros_like(b), 0, True, np.zeros(1)
    x = np.zeros_like(b)
    hist = [1.0]
    total = 0
    conv = False
    while total < maxit:
        r = b - a @ x if total else b.copy()
        rn = float(np.linalg.norm(r))
        if rn == 0.0:
            conv = True
            break
        d, k, c, h = gmres(a, precond, r, tol * bn / rn, min(restart, maxit - total))
        x = x + d
        hist.extend((h[1:] * (rn / bn)).tolist())
        total += k
        if c:
            conv = True
            break
        if k == 0:
            break
    return x, total, conv, np.asarray(hist)
