"""Setup algebra on CPU tensors (no GPU): the batched band-path coarse columns (batched ring
solves, pencil reduction, block subspace iteration + Rayleigh-Ritz) span the same spaces as the
per-subdomain dense eigensolve, and the band factor layout matches the dense Cholesky."""

import numpy as np
import pytest
import torch

from conftest import golden, golden_csr
from paper_2401_03915_b200 import partition as Pt
from paper_2401_03915_b200 import gpu_setup as G


def _batch(name, sel):
    d = golden(name)
    a = golden_csr(d)
    maps = Pt.extend_overlap(Pt.symmetrized_graph(a), Pt.Partition(int(d["n_sub"]), d["owner"]),
                             int(d["overlap"]))
    ms = [maps[s] for s in sel]
    ld = -(-max(m.n_local for m in ms) // 64) * 64
    A = torch.zeros(len(ms), ld, ld, dtype=torch.float64)
    for b, m in enumerate(ms):
        A[b, : m.n_local, : m.n_local] = torch.as_tensor(a[m.indices][:, m.indices].toarray())
        A[b, m.n_local:, m.n_local:] = torch.eye(ld - m.n_local, dtype=torch.float64)
    return d, ms, A, ld


def test_topk_subspace_matches_dense_eigh():
    torch.manual_seed(0)
    m, k = 300, 12
    Q, _ = torch.linalg.qr(torch.randn(3, m, m, dtype=torch.float64))
    lam = torch.logspace(0, -12, m, dtype=torch.float64)
    M = Q @ torch.diag_embed(lam.expand(3, m)) @ Q.mT
    th, X, its = G.topk_subspace(torch, M, k)
    assert its > 0
    np.testing.assert_allclose(th.numpy(), lam[:k].expand(3, k).numpy(), rtol=1e-12)
    for b in range(3):
        sv = torch.linalg.svdvals(X[b].mT @ Q[b][:, :k])
        assert float(sv.min()) > 1 - 1e-12


@pytest.mark.parametrize("decay", ["flat", "fast"])
def test_topk_chebyshev_matches_dense_eigh(decay):
    torch.manual_seed(1)
    m, k = 400, 13
    Q, _ = torch.linalg.qr(torch.randn(2, m, m, dtype=torch.float64))
    i = torch.arange(m, dtype=torch.float64)
    lam = torch.exp(-0.003 * i) if decay == "flat" else torch.logspace(0, -12, m, dtype=torch.float64)
    M = Q @ torch.diag_embed(lam.expand(2, m)) @ Q.mT
    th, X, mv = G.topk_chebyshev(torch, M, k)
    assert mv > 0
    np.testing.assert_allclose(th.numpy(), lam[:k].expand(2, k).numpy(), rtol=1e-12)
    for b in range(2):
        sv = torch.linalg.svdvals(X[b].mT @ Q[b][:, :k])
        assert float(sv.min()) > 1 - 1e-12


@pytest.mark.parametrize("direct", ["1", "0"])
@pytest.mark.parametrize("name,sel", [("cfg2_m24", [0, 4, 13, 26]), ("cfg5_m16", [0, 3, 7])])
def test_batched_band_coarse_columns_match_dense_path(name, sel, direct, monkeypatch):
    # direct = "1": the reduced pencil formed as M = C^T A_GG C - I (overlap 1), "0": from
    # H = F^T A_II F by two triangular solves; both against the dense eigensolve of the pencil
    monkeypatch.setenv("TLS_PENCIL_DIRECT", direct)
    d, ms, A, ld = _batch(name, sel)
    k = int(d["n_modes"])
    L, Dinv, perms, kcnts, info, P, codes = G._band_factor(torch, A, [np.argsort(m.indices, kind="stable") for m in ms],
                                                    [m.n_local for m in ms], ld)
    assert int(info.abs().sum()) == 0
    ns = [m.n_local for m in ms]
    nis = [m.interior.size for m in ms]
    nins = [m.n_local - m.n_boundary for m in ms]
    kc = np.zeros((len(ms), ld // 64), dtype=np.int64)
    for b in range(len(ms)):
        kc[b, : kcnts[b].size] = kcnts[b]
    cols = G._coarse_band_batch(torch, "gevp", A, L, P, ns, nis, nins, 0.1, k, Dinv=Dinv, kc=kc)
    for b, m in enumerate(ms):
        n, ni, nin = ns[b], nis[b], nins[b]
        Binv = torch.linalg.inv(A[b, :n, :n])
        Zd, gap_d = G._subdomain_columns(torch, "gevp", A[b], Binv[:, nin:n], n, ni, nin, 0.1, k)
        Zb, gap_b, Wb = cols[b]
        if Wb is not None:
            np.testing.assert_allclose(Wb.numpy(), (A[b, :n, :ni] @ Zb).numpy(), atol=1e-12 * float(Wb.abs().max()))
        assert Zb.shape == Zd.shape == (ni, k)
        qb, _ = torch.linalg.qr(Zb)
        qd, _ = torch.linalg.qr(Zd)
        sine = torch.linalg.matrix_norm(qb - qd @ (qd.mT @ qb), ord=2)  # largest principal-angle sine
        assert float(sine) < 1e-9
        assert abs(gap_b - gap_d) <= 1e-6 * max(gap_d, 1e-12)
        # the lifted columns agree up to sign conventions
        np.testing.assert_allclose(np.abs(Zb.numpy()), np.abs(Zd.numpy()), atol=1e-9 * float(Zd.abs().max()))


def test_band_solve_multi_matches_dense():
    d, ms, A, ld = _batch("cfg2_m24", [0, 13])
    L, Dinv, perms, kcnts, info, P, codes = G._band_factor(torch, A, [np.argsort(m.indices, kind="stable") for m in ms],
                                                    [m.n_local for m in ms], ld)
    kc = np.zeros((len(ms), ld // 64), dtype=np.int64)
    for b in range(len(ms)):
        kc[b, : kcnts[b].size] = kcnts[b]
    E = torch.randn(len(ms), ld, 37, dtype=torch.float64, generator=torch.Generator().manual_seed(3))
    X = G.band_solve_multi(torch, L, Dinv, kc, E)
    ref = torch.cholesky_solve(E, L)
    assert float((X - ref).abs().max() / ref.abs().max()) < 1e-12


def test_band_solve_multi_skips_leading_zero_columns():
    """Unit right-hand sides sorted by the row of their 1 (the ring solve of the harmonic
    extension): the forward sweep restricted to the live columns gives the same X bit for bit."""
    d, ms, A, ld = _batch("cfg2_m24", [0, 13])
    L, Dinv, perms, kcnts, info, P, codes = G._band_factor(torch, A, [np.argsort(m.indices, kind="stable") for m in ms],
                                                    [m.n_local for m in ms], ld)
    kc = np.zeros((len(ms), ld // 64), dtype=np.int64)
    for b in range(len(ms)):
        kc[b, : kcnts[b].size] = kcnts[b]
    rng = np.random.default_rng(5)
    nrhs = 41
    rows = np.sort(np.stack([rng.choice(min(m.n_local for m in ms), nrhs, replace=False) for _ in ms]), axis=1)
    E = torch.zeros(len(ms), ld, nrhs, dtype=torch.float64)
    for b in range(len(ms)):
        E[b, rows[b], np.arange(nrhs)] = 1.0
    lead = rows.min(axis=0)
    X = G.band_solve_multi(torch, L, Dinv, kc, E, lead)
    X0 = G.band_solve_multi(torch, L, Dinv, kc, E)
    assert torch.equal(X, X0)
    ref = torch.cholesky_solve(E, L)
    assert float((X - ref).abs().max() / ref.abs().max()) < 1e-12


def test_band_cholesky_matches_dense_and_flags_indefinite():
    d, ms, A, ld = _batch("cfg5_m16", [0, 3, 7])
    perm_list = [np.argsort(m.indices, kind="stable") for m in ms]
    n_list = [m.n_local for m in ms]
    AP, P, _ = G._lex_perm(torch, A, perm_list, n_list, ld)
    L, Dinv, perms, kcnts, info, P2, codes = G._band_factor(torch, A, perm_list, n_list, ld)
    assert int(info.abs().sum()) == 0
    assert float(torch.triu(L, 1).abs().max()) == 0.0
    ref = torch.linalg.cholesky(AP)
    assert float((L - ref).abs().max() / ref.abs().max()) < 1e-12
    # an indefinite block is reported with the 1-based failing row, like cholesky_ex
    B = A.clone()
    B[1, 70, 70] = -10.0
    _, _, _, _, info, _, _ = G._band_factor(torch, B, perm_list, n_list, ld)
    assert int(info[0]) == 0 and int(info[1]) > 0 and int(info[2]) == 0


def test_pou_columns_equal_full_pencil():
    """_pou_columns (reduced n_int pencil with the interior Schur complement) = the reference's
    m x m pencil (D A D) u = lam A u (src/spectral.py:93-108): same selected values, same
    columns D u (A-normalised, sign-fixed on the full vector)."""
    import scipy.linalg as sla
    from paper_2401_03915_b200.gpu_setup import _pou_columns
    from paper_2401_03915_b200 import problems as PR
    from paper_2401_03915_b200.partition import Partition, extend_overlap, symmetrized_graph
    a = PR.poisson2d(12)
    owner = PR.tile_owner_2d(12, 6)
    maps = extend_overlap(symmetrized_graph(a, symmetric=True), Partition(4, owner), 2)
    for smap in maps:
        idx = smap.indices
        A = a[idx][:, idx].toarray()
        n, ni = A.shape[0], smap.interior.size
        d = np.zeros(n)
        d[:ni] = 1.0
        vals, vecs = sla.eigh(A * np.outer(d, d), A)
        vals, vecs = vals[::-1], vecs[:, ::-1]
        nu = 1.3
        keep = vals > nu * (1 + 1e-12)
        ref = vecs[:, keep]
        for j in range(ref.shape[1]):
            k = int(np.argmax(np.abs(ref[:, j])))
            if ref[k, j] < 0:
                ref[:, j] = -ref[:, j]
        got = _pou_columns(torch, torch.as_tensor(A), n, ni, nu).numpy()
        assert got.shape[1] == ref.shape[1] and got.shape[1] > 0
        np.testing.assert_allclose(got, ref[:ni], rtol=0, atol=1e-10 * np.abs(ref).max())


@pytest.mark.parametrize("n,bw,bs,scale", [(1000, 90, 128, 1.5), (777, 63, 64, 1.5), (512, 300, 512, 1.5),
                                           (640, 63, 64, 1.0 + 1e-7)])
def test_spd_inverse_block_tridiagonal_matches_dense(n, bw, bs, scale):
    """The block-tridiagonal recurrences give the lower triangle and the full diagonal blocks of
    A^{-1} (only A's lower triangle read), to the accuracy of the dense Cholesky inverse -- also
    on an ill-conditioned matrix (last case: diagonally semi-dominant, cond ~ 1e7)."""
    rng = np.random.default_rng(n)
    mask = np.abs(np.subtract.outer(np.arange(n), np.arange(n))) <= bw
    B = np.abs(rng.standard_normal((n, n))) * mask
    A = -(B + B.T) / 2
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, -A.sum(axis=1) * scale)   # weakly diagonally dominant M-matrix: SPD
    ref = np.linalg.inv(A)
    X = torch.tril(torch.tensor(A)) + torch.triu(torch.full((n, n), 7.0, dtype=torch.float64), 1)
    assert G.spd_inverse_block_tridiagonal(torch, X, bs) == 0
    X = X.numpy()
    dense = torch.cholesky_inverse(torch.linalg.cholesky(torch.tensor(A))).numpy()
    tol = max(1e-13, 20 * np.abs(dense - ref).max() / np.abs(ref).max())
    assert np.abs(np.tril(X) - np.tril(ref)).max() <= tol * np.abs(ref).max()
    for r in range(0, n, bs):   # diagonal blocks are stored in full (the packed-tile store reads them)
        assert np.abs(X[r:r + bs, r:r + bs] - ref[r:r + bs, r:r + bs]).max() <= tol * np.abs(ref).max()
    # residual of the symmetric completion: A X = I
    Xs = np.tril(X) + np.tril(X, -1).T
    assert np.abs(A @ Xs - np.eye(n)).max() <= 1e-9 * max(1.0, np.linalg.cond(A) * 1e-7)


def _chain_solve(sinv, lo, up, bs, c):
    """Host restatement of the library's block substitution (enq_coarse_chain in csrc/tls_b200.cu)."""
    import scipy.sparse as sp
    n = c.size
    Lo = sp.csr_matrix((lo[2].numpy(), lo[1].numpy(), lo[0].numpy()), shape=(n, n))
    Up = sp.csr_matrix((up[2].numpy(), up[1].numpy(), up[0].numpy()), shape=(n, n))
    z, y = c.copy(), np.zeros(n)
    nb = len(sinv)
    for i in range(nb):
        r = slice(i * bs, min(n, (i + 1) * bs))
        if i > 0:
            z[r] -= (Lo @ y)[r]
        y[r] = sinv[i].numpy() @ z[r]
    for i in range(nb - 2, -1, -1):
        r = slice(i * bs, min(n, (i + 1) * bs))
        z[r] -= (Up @ y)[r]
        y[r] = sinv[i].numpy() @ z[r]
    return y


@pytest.mark.parametrize("n,bw,bs,scale", [(1000, 90, 128, 1.5), (777, 63, 64, 1.5), (640, 63, 64, 1.0 + 1e-7)])
def test_spd_block_tridiagonal_chain_solves(n, bw, bs, scale):
    """The block factorisation behind tls_coarse_chain: the substitution with the inverted Schur
    blocks and the sparse off-diagonal blocks solves A x = c like a dense Cholesky solve
    (src/coarse.py:178-182); the two CSR parts are each other's transposes and only hold entries
    of the neighbouring block; only A's lower triangle is read."""
    import scipy.sparse as sp
    rng = np.random.default_rng(n)
    mask = np.abs(np.subtract.outer(np.arange(n), np.arange(n))) <= bw
    Bm = np.abs(rng.standard_normal((n, n))) * mask
    A = -(Bm + Bm.T) / 2
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, -A.sum(axis=1) * scale)
    X = torch.tril(torch.tensor(A)) + torch.triu(torch.full((n, n), 7.0, dtype=torch.float64), 1)
    info, sinv, lo, up = G.spd_block_tridiagonal_chain(torch, X, bs)
    assert info == 0 and len(sinv) == -(-n // bs)
    Lo = sp.csr_matrix((lo[2].numpy(), lo[1].numpy(), lo[0].numpy()), shape=(n, n))
    Up = sp.csr_matrix((up[2].numpy(), up[1].numpy(), up[0].numpy()), shape=(n, n))
    assert abs(Lo - Up.T).max() == 0.0
    r, cidx = Lo.nonzero()
    assert np.all(cidx // bs == r // bs - 1)
    full = np.zeros((n, n))
    for i in range(len(sinv)):
        full[i * bs:(i + 1) * bs, i * bs:(i + 1) * bs] = A[i * bs:(i + 1) * bs, i * bs:(i + 1) * bs]
    assert np.abs(full + Lo.toarray() + Up.toarray() - A).max() == 0.0
    c = rng.standard_normal(n)
    y = _chain_solve(sinv, lo, up, bs, c)
    ref = np.linalg.solve(A, c)
    dense = torch.cholesky_solve(torch.tensor(c)[:, None], torch.linalg.cholesky(torch.tensor(A)))[:, 0].numpy()
    tol = max(1e-13, 20 * np.abs(dense - ref).max() / np.abs(ref).max())
    assert np.abs(y - ref).max() <= tol * np.abs(ref).max()


def test_spd_block_tridiagonal_chain_flags_indefinite():
    A = np.eye(300) * 2.0
    A[200, 200] = -1.0
    assert G.spd_block_tridiagonal_chain(torch, torch.tensor(A), 64)[0] == 201


def test_spd_inverse_block_tridiagonal_flags_indefinite():
    n, bs = 300, 64
    A = np.eye(n) * 2.0
    A[200, 200] = -1.0
    X = torch.tensor(A)
    assert G.spd_inverse_block_tridiagonal(torch, X, bs) == 201


def test_coarse_bandwidth_bounds_a0_nonzeros():
    """Every structurally nonzero entry of A0 = Z^T A Z lies within the half bandwidth computed from
    the subdomain adjacency (the block-tridiagonal inverse relies on it)."""
    d = golden("cfg2_m24")
    a = golden_csr(d)
    nsub = int(d["n_sub"])
    owner = np.asarray(d["owner"], dtype=np.int64)
    from paper_2401_03915_b200.sparsemat import SparseMat, symmetrized_graph
    maps = Pt.extend_overlap(symmetrized_graph(SparseMat(a, symmetric=True)), Pt.Partition(nsub, owner),
                             int(d["overlap"]))
    rng = np.random.default_rng(1)
    for counts in (rng.integers(0, 5, nsub), np.full(nsub, 3)):
        cstart = np.concatenate([[0], np.cumsum(counts)])
        nC = int(cstart[-1])
        Z = np.zeros((a.shape[0], nC))
        for s, m in enumerate(maps):
            Z[np.ix_(m.interior, np.arange(cstart[s], cstart[s + 1]))] = rng.standard_normal((m.interior.size, counts[s]))
        A0 = Z.T @ (a @ Z)
        bw = G.coarse_bandwidth(maps, owner, counts, range(nsub))
        i, j = np.nonzero(A0)
        assert np.abs(i - j).max() <= bw < nC
    assert np.abs(i - j).max() == bw   # dense blocks: the bound is attained
