"""In-tree setup kernels against numpy/LAPACK on the same inputs: the batched Jacobi eigensolver
of the Rayleigh-Ritz step (tls_syevj_batched; the dense eigh of src/spectral.py:69-85 on the
projected problem) and the sync-light Chebyshev subspace iteration built on it."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_03915_b200 import build
    build.build()
    from paper_2401_03915_b200 import gpu_setup
    return gpu_setup


@pytest.mark.parametrize("p", [1, 2, 7, 8, 33, 39, 64])
def test_syevj_batched_matches_lapack(G, p):
    rng = np.random.default_rng(p)
    b = 5
    T = rng.standard_normal((b, p, p))
    T = T + T.transpose(0, 2, 1)
    T[1] = np.diag(np.arange(p, dtype=float))          # already diagonal
    T[2] = np.eye(p) * 3.0                              # fully degenerate
    q, _ = np.linalg.qr(rng.standard_normal((p, p)))
    T[3] = q @ np.diag(np.repeat([5.0, 1.0, -2.0], -(-p // 3))[:p]) @ q.T   # clustered
    Td = torch.as_tensor(T, device="cuda")
    w, V = G._eigh_desc(torch, Td)
    w, V = w.cpu().numpy(), V.cpu().numpy()
    for j in range(b):
        ref = np.sort(np.linalg.eigvalsh(T[j]))[::-1]
        nrm = max(np.abs(T[j]).max(), 1.0)
        assert np.abs(w[j] - ref).max() <= 1e-13 * nrm * p, j
        assert np.abs(T[j] @ V[j] - V[j] * w[j][None, :]).max() <= 1e-12 * nrm, j
        assert np.abs(V[j].T @ V[j] - np.eye(p)).max() <= 1e-12, j
        assert np.all(np.diff(w[j]) <= 0)


@pytest.mark.parametrize("decay", [0.5, 0.97])
def test_chebyshev_on_device_matches_dense_eigh(G, decay):
    rng = np.random.default_rng(3)
    b, m, k = 6, 300, 12
    Ms = []
    for j in range(b):
        q, _ = np.linalg.qr(rng.standard_normal((m, m)))
        ev = decay ** np.arange(m) * (1 + 0.1 * j)
        Ms.append((q * ev) @ q.T)
    M = torch.as_tensor(np.array(Ms), device="cuda")
    th, X, _ = G.topk_chebyshev(torch, M, k)
    for j in range(b):
        w, Q = np.linalg.eigh(Ms[j])
        w, Q = w[::-1][:k], Q[:, ::-1][:, :k]
        assert np.abs(th[j].cpu().numpy() - w).max() <= 1e-12 * w[0]
        Xj = X[j].cpu().numpy()
        # same span: projector difference
        assert np.abs(Xj @ Xj.T - Q @ Q.T).max() <= 1e-9


def test_band_solve_multi_kernel_matches_torch_and_dense(G):
    """K10 (tls_band_solve_multi, DMMA) = the blocked torch restatement = a dense Cholesky solve,
    on banded SPD blocks with varying per-block panel counts and a ragged RHS count."""
    rng = np.random.default_rng(11)
    b, nb, nrhs = 3, 5, 70
    ld = 64 * nb
    A = np.zeros((b, ld, ld))
    kc = np.zeros((b, nb), dtype=np.int64)
    for j in range(b):
        bw = [40, 100, 150][j]
        M = np.zeros((ld, ld))
        for d in range(bw + 1):
            v = rng.standard_normal(ld - d) * 0.1
            M += np.diag(v, -d)
        M = M @ M.T + ld * np.eye(ld)
        band = np.abs(np.subtract.outer(np.arange(ld), np.arange(ld))) <= bw
        A[j] = np.where(band, M, 0.0) + 2 * bw * np.eye(ld)
        for I in range(nb):
            kc[j, I] = min(I, -(-bw // 64))
    At = torch.as_tensor(A, device="cuda")
    L = torch.linalg.cholesky(At)
    Ld = L.view(b, nb, 64, nb, 64).diagonal(dim1=1, dim2=3).permute(0, 3, 1, 2)
    eye = torch.eye(64, dtype=torch.float64, device="cuda").expand(b, nb, 64, 64)
    Dinv = torch.linalg.solve_triangular(Ld, eye, upper=False).contiguous()
    E = torch.as_tensor(rng.standard_normal((b, ld, nrhs)), device="cuda")
    import os
    os.environ["TLS_K10"] = "1"
    try:
        Xk = G.band_solve_multi(torch, L.contiguous(), Dinv, kc, E)
    finally:
        os.environ.pop("TLS_K10")
    Xt = G._band_solve_multi_torch(torch, L, Dinv, kc, E)
    Xd = torch.cholesky_solve(E, L)
    scale = Xd.abs().max().item()
    assert (Xk - Xd).abs().max().item() <= 1e-12 * scale
    assert (Xk - Xt).abs().max().item() <= 1e-12 * scale


def test_rank_filter_pivots_match_lapack_geqp3(G):
    """K12a (device column-pivoted Householder QR) = LAPACK geqp3 (src/coarse.py:136): pivot order
    and |R_jj| on well-separated blocks, incl. an exactly dependent column and a zero column."""
    import scipy.linalg as sla
    rng = np.random.default_rng(2)
    blocks = {}
    for s, (n, k) in enumerate([(300, 12), (64, 20), (1000, 3), (50, 1)]):
        z = rng.standard_normal((n, k)) * np.logspace(0, -6, k)[None, :]
        if k >= 3:
            z[:, 2] = z[:, 0] - 2.0 * z[:, 1]      # dependent
        if k >= 5:
            z[:, 4] = 0.0                          # zero column
        blocks[s] = torch.as_tensor(z, device="cuda")
    piv = G._rank_pivots(torch, blocks, range(len(blocks)), torch.device("cuda"))
    o = 0
    for s in range(len(blocks)):
        z = blocks[s].cpu().numpy()
        r, perm = sla.qr(z, mode="r", pivoting=True)
        rd = np.abs(np.diag(r))
        mine = [p for p in piv if p[1] == s]
        got = np.array([p[0] for p in mine])
        want = np.array([rd[j] if j < rd.size else 0.0 for j in range(z.shape[1])])
        big = want > 1e-10 * want.max()            # the filter's decision range (drop_tol 1e-10)
        assert [p[2] for p, b in zip(mine, big) if b] == [int(q) for q, b in zip(perm, big) if b], s
        assert np.abs(got[big] - want[big]).max() <= 1e-12 * want.max(), s
        assert np.all(got[~big] <= 1e-10 * want.max()), s


def test_band_lu_kernel_matches_lapack(G):
    """K9b (in-tree banded LU with partial pivoting, DMMA trailing updates) reproduces LAPACK
    getrf (torch.linalg.lu_factor_ex): same pivots on a nonsymmetric banded batch, LU to 1e-12,
    and P L U = A."""
    rng = np.random.default_rng(8)
    b, nb = 3, 6
    ld = 64 * nb
    A = np.zeros((b, ld, ld))
    for j in range(b):
        kl, ku = [30, 70, 130][j], [50, 20, 90][j]
        for d in range(-kl, ku + 1):
            A[j] += np.diag(rng.standard_normal(ld - abs(d)), d)
        A[j] += np.diag(np.full(ld, 0.5))
    At = torch.as_tensor(A, device="cuda")
    LUr, pivr, infor = torch.linalg.lu_factor_ex(At.clone())
    LUk, pivk, infok = G.band_lu_kernel(torch, At.clone())
    assert torch.equal(pivk.cpu(), pivr.cpu().to(torch.int32))
    assert int(infok.abs().sum()) == 0
    assert (LUk - LUr).abs().max().item() <= 1e-11 * LUr.abs().max().item()
    P, L, U = torch.lu_unpack(LUk, pivk)
    assert (P @ L @ U - At).abs().max().item() <= 1e-12 * At.abs().max().item()


@pytest.mark.parametrize("shape", [(1, 1), (5, 3), (3, 5), (40, 40), (131, 131), (268, 268), (100, 37)])
def test_svdj_batched_matches_lapack(G, shape):
    """K13 one-sided Jacobi SVD (tls_svdj_batched) against LAPACK on the same matrices: the thin
    SVD of src/spectral.py:143.  Upper-triangular inputs (the R of E = QR), graded singular values
    over 12 decades, a rank-deficient and a zero matrix."""
    r, n = shape
    rng = np.random.default_rng(r * 1000 + n)
    b = 5
    R = rng.standard_normal((b, r, n))
    R[0] = np.triu(R[0])
    k = min(r, n)
    u, _ = np.linalg.qr(rng.standard_normal((r, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    R[1] = (u[:, :k] * np.logspace(0, -12, k)) @ v[:, :k].T           # graded
    R[2] = (u[:, :max(k // 2, 1)] * 2.0) @ v[:, :max(k // 2, 1)].T     # rank-deficient, multiple sigma
    R[3] = 0.0
    kk = min(k, 21)
    UR, sv = G._svd_left_topk(torch, torch.as_tensor(R, device="cuda"), kk)
    UR, sv = UR.cpu().numpy(), sv.cpu().numpy()
    for j in range(b):
        U, S, Vt = np.linalg.svd(R[j], full_matrices=False)
        s0 = max(S[0], 1e-300)
        assert np.abs(sv[j] - S[:kk]).max() <= 2e-13 * s0, j
        assert np.all(np.diff(sv[j]) <= 0)
        live = np.nonzero(sv[j] > 1e-13 * s0)[0]
        if live.size == 0:
            continue
        Uj = UR[j][:, live]
        assert np.abs(Uj.T @ Uj - np.eye(live.size)).max() <= 1e-9, j
        # singular-vector residual: |R^T u| = sigma, and R R^T u = sigma^2 u
        res = R[j] @ (R[j].T @ Uj) - Uj * sv[j][live] ** 2
        assert np.abs(res).max() <= 1e-12 * s0 * s0, j


def test_perm_lower_matches_torch_gathers(G):
    """tls_perm_lower (factor-order lower triangle + row profile in one pass) against the torch
    gathers / argmax it replaces in the banded setup."""
    from paper_2401_03915_b200 import _lib
    from paper_2401_03915_b200.device import stream_ptr
    rng = np.random.default_rng(5)
    cnt, ld = 3, 192
    A = np.zeros((cnt, ld, ld))
    for b in range(cnt):
        M = rng.standard_normal((ld, ld)) * (rng.random((ld, ld)) < 0.05)
        A[b] = M + M.T + np.diag(1.0 + rng.random(ld))
    P = np.stack([rng.permutation(ld) for _ in range(cnt)]).astype(np.int64)
    Ad = torch.as_tensor(A, device="cuda")
    Pd = torch.as_tensor(P, device="cuda")
    AP = torch.empty_like(Ad)
    first = torch.empty((cnt, ld), dtype=torch.int32, device="cuda")
    rc = _lib.load().tls_perm_lower(_lib.ptr(Ad), _lib.ptr(Pd), _lib.ptr(AP), _lib.ptr(first), cnt, ld, stream_ptr())
    assert rc == 0
    ref = np.stack([A[b][np.ix_(P[b], P[b])] for b in range(cnt)])
    assert np.array_equal(AP.cpu().numpy(), np.tril(ref))
    assert np.array_equal(first.cpu().numpy(), np.argmax(ref != 0, axis=2))


@pytest.mark.parametrize("cl", [1, 2, 4])
def test_band_cholesky_kernel_matches_lapack(G, cl, monkeypatch):
    """K9 k_band_chol<CL> (banded Cholesky, a CL-CTA cluster per block) against LAPACK potrf on the
    same banded SPD blocks: factor, inverted diagonal tiles, info of a non-SPD block."""
    monkeypatch.setenv("TLS_K9_CLUSTER", str(cl))
    rng = np.random.default_rng(cl)
    cnt, ld, bw = 3, 320, 150
    A = np.zeros((cnt, ld, ld))
    for b in range(cnt):
        M = rng.standard_normal((ld, ld))
        M = np.tril(np.triu(M, -bw), bw)
        A[b] = M @ M.T * 0.05 + np.diag(2.0 + rng.random(ld))
        A[b] = np.tril(np.triu(A[b], -bw), bw)
        A[b] += np.eye(ld) * (np.abs(A[b]).sum(axis=1).max())      # diagonally dominant -> SPD
    A[2, 200, 200] = -1.0                                           # not positive definite
    nbk = ld // 64
    rows = np.arange(ld)
    first = np.maximum(rows - bw, 0)
    kmax = (np.arange(nbk) - first.reshape(nbk, 64).min(axis=1) // 64).clip(min=0)
    AP = torch.as_tensor(np.tril(A), device="cuda").contiguous()
    L, Dinv, info = G.band_cholesky_kernel(torch, AP, kmax, clear_upper=False)
    L, Dinv, info = L.cpu().numpy(), Dinv.cpu().numpy(), info.cpu().numpy()
    assert info[0] == 0 and info[1] == 0 and info[2] == 201
    for b in range(2):
        ref = np.linalg.cholesky(A[b])
        assert np.abs(L[b] - ref).max() <= 1e-12 * np.abs(ref).max()
        assert np.abs(np.triu(L[b], 1)).max() == 0.0
        for J in range(nbk):
            d = ref[64 * J:64 * J + 64, 64 * J:64 * J + 64]
            assert np.abs(Dinv[b, J] @ d - np.eye(64)).max() <= 1e-11


def test_tma_ring_kernel_is_bit_identical(G, monkeypatch):
    """K3e k_band_solve_tma (rings fed by bulk TMA copies + mbarriers) against the default cp.async
    ring kernel on the same band factors: identical sweeps, so identical bits (Cholesky and LU)."""
    import paper_2401_03915_b200 as B
    for cid, m, part in ((1, 48, 16), (3, 48, 16)):
        cfg = B.problems.CONFIGS[cid].scaled(m, part)
        a, sym, owner, nsub = cfg.build()
        mat = B.SparseMat(a, symmetric=sym)
        r = np.random.default_rng(7).standard_normal(a.shape[0])
        outs = []
        for tma in ("0", "4", "5"):
            monkeypatch.setenv("TLS_BAND_TMA", tma)
            pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=4, local="band")
            assert pre.local_kind.startswith("band")
            outs.append(pre.apply_one_level(r))
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
