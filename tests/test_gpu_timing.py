"""In-graph timing of the band local-solve kernel (bench roofline inside real solves): the event
nodes see one launch per PCG iteration that did work, and do not change the solve."""

import ctypes as C

import numpy as np
import pytest

from conftest import golden, golden_csr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_03915_b200 import build
    build.build()
    import paper_2401_03915_b200 as mod
    return mod


@pytest.mark.parametrize("name,solver", [("cfg2_m24", "pcg"), ("cfg3_m64", "gmres")])
def test_in_graph_band_timing(B, name, solver):
    d = golden(name)
    a = golden_csr(d)
    mat = B.SparseMat(a, symmetric=bool(d["symmetric"]))
    pre = B.setup(mat, int(d["n_sub"]), overlap=int(d["overlap"]), owner=d["owner"], coarse=str(d["coarse"]),
                  n_modes=int(d["n_modes"]), local="band")
    run = (lambda: B.pcg(mat, pre, d["b"], tol=float(d["tol"]))) if solver == "pcg" else \
        (lambda: B.gmres(mat, pre, d["b"], tol=float(d["tol"]), restart=int(d["restart"])))
    x0, r0 = run()
    h = pre.handle
    h.check(h.lib.tls_set_kernel_timing(h.ctx, 1))
    x1, r1 = run()
    ms, n = C.c_double(), C.c_int64()
    h.check(h.lib.tls_kernel_timing(h.ctx, C.byref(ms), C.byref(n)))
    h.check(h.lib.tls_set_kernel_timing(h.ctx, 0))
    assert np.array_equal(x0, x1) and r0.iterations == r1.iterations
    assert ms.value > 0.0
    if solver == "pcg":  # one band solve per iteration inside the graph (the first apply is outside)
        assert r1.iterations - 2 <= n.value <= r1.iterations
    else:
        assert n.value >= r1.iterations


@pytest.mark.parametrize("name,sel", [("cfg2_m24", [0, 4, 13, 26]), ("cfg5_m16", [0, 3, 7])])
def test_band_cholesky_kernel_matches_library_path(B, name, sel):
    """K9 (in-tree DMMA banded Cholesky) = the batched cuSOLVER path: same factor and inverted
    diagonal blocks to rounding, identical (zero) info; a non-SPD block reports its pivot row."""
    from paper_2401_03915_b200 import gpu_setup as G
    from paper_2401_03915_b200 import partition as Pt
    d = golden(name)
    a = golden_csr(d)
    maps = Pt.extend_overlap(Pt.symmetrized_graph(a), Pt.Partition(int(d["n_sub"]), d["owner"]), int(d["overlap"]))
    ms = [maps[s] for s in sel]
    ld = -(-max(m.n_local for m in ms) // 64) * 64
    A = torch.zeros(len(ms), ld, ld, dtype=torch.float64, device="cuda")
    for b, m in enumerate(ms):
        A[b, : m.n_local, : m.n_local] = torch.as_tensor(a[m.indices][:, m.indices].toarray())
        A[b, m.n_local:, m.n_local:] = torch.eye(ld - m.n_local, dtype=torch.float64)
    import scipy.sparse as sp
    g = Pt.symmetrized_graph(a)
    adj = sp.csr_matrix((np.ones(g.adjacency.size, dtype=np.int8), g.adjacency, g.indptr), shape=a.shape)
    perms = G.local_orders(adj, ms, "rcm")
    n_list = [m.n_local for m in ms]
    old = G.BAND_CHOL
    try:
        G.BAND_CHOL = "torch"
        L1, D1, _, k1, i1, _, _ = G._band_factor(torch, A.clone(), perms, n_list, ld)
        G.BAND_CHOL = "kernel"
        L2, D2, _, k2, i2, _, _ = G._band_factor(torch, A.clone(), perms, n_list, ld)
    finally:
        G.BAND_CHOL = old
    assert int(i1.abs().sum()) == 0 and int(i2.abs().sum()) == 0
    assert all(np.array_equal(x, y) for x, y in zip(k1, k2))
    assert float((L1 - L2).abs().max()) <= 1e-11 * float(L1.abs().max())
    assert float((D1 - D2).abs().max()) <= 1e-11 * float(D1.abs().max())
    # a block made indefinite reports a pivot
    Abad = A.clone()
    Abad[0, 5, 5] = -1.0
    _, _, _, _, ib, _, _ = G._band_factor(torch, Abad, perms, n_list, ld)
    assert int(ib[0]) > 0 and int(ib[1:].abs().sum()) == 0
