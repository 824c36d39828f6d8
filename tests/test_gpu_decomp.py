"""Decomposition on the device (tls_graph_build / tls_overlap_build) against
the host restatements that are pinned bit-exact to the reference (tests/test_host_logic.py,
tests/golden/*): symmetrised graph (src/sparsemat.py:180-195: |a_ij| > 0 or |a_ji| > 0, stored
zeros and the diagonal dropped), overlap rings (src/partition.py:278-301) for 1-3 layers and the
greedy colouring (src/partition.py:304-334) -- every index bit for bit."""

import numpy as np
import pytest
import scipy.sparse as sp

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


def _cases(B):
    P = B.problems
    out = []
    a = P.poisson2d(24).tolil()
    a[3, 4] = 0.0  # stored zeros on both sides: no edge
    a[4, 3] = 0.0
    a[10, 40] = 0.0  # one-sided stored zero + its nonzero mirror: an edge
    a[40, 10] = 0.5
    out.append(("poisson2d+zeros", a.tocsr(), False, P.tile_owner_2d(24, 6), 16))
    out.append(("poisson2d", P.poisson2d(24), True, P.tile_owner_2d(24, 8), 9))
    out.append(("advection2d", P.advection2d(20), False, P.tile_owner_2d(20, 5), 16))
    c5 = P.CONFIGS[5].scaled(16, 8, angle_block=8)
    a5, _, o5, n5 = c5.build()
    out.append(("aniso27_q1", a5, True, o5, n5))
    c3 = P.CONFIGS[3].scaled(48, 12)
    a3, _, o3, n3 = c3.build()
    out.append(("recirc2d", a3, False, o3, n3))
    rng = np.random.default_rng(4)
    r = sp.random(300, 300, density=0.02, random_state=5, format="csr") + sp.identity(300)
    out.append(("random-nonsym", r.tocsr(), False, rng.integers(0, 7, 300), 7))
    return out


def test_device_graph_overlap_colouring_bit_exact(B):
    from paper_2401_03915_b200 import device as D
    from paper_2401_03915_b200 import partition as H
    for name, a, sym, owner, nsub in _cases(B):
        a = sp.csr_matrix(a)
        a.sort_indices()
        if sym:
            assert (a != a.T).nnz == 0
        h = D.Handle()
        h.upload_matrix(a, sym)
        g = D.device_graph(h)
        gh = H.symmetrized_graph(a, symmetric=sym)
        assert np.array_equal(g.indptr, gh.indptr), name
        assert np.array_equal(g.adjacency.astype(np.int64), gh.adjacency), name
        part = H.Partition(nsub, owner)
        for delta in (1, 2, 3):
            if delta > 1:
                D.device_graph(h)  # device_overlap releases the graph
            maps, k_c, colors = D.device_overlap(h, part, delta)
            ref = H.extend_overlap(gh, part, delta)
            kr, cr = H.color_subdomains(ref)
            assert len(maps) == nsub
            for m, r in zip(maps, ref):
                assert np.array_equal(m.interior, r.interior), (name, delta)
                assert len(m.layers) == len(r.layers) == delta
                for la, lb in zip(m.layers, r.layers):
                    assert np.array_equal(la, lb), (name, delta)
            assert k_c == kr and np.array_equal(colors, cr), (name, delta)


def test_setup_uses_device_decomposition(B, monkeypatch):
    """setup() decomposes on the device (same maps / colours as the host path)."""
    P = B.problems
    a = P.poisson2d(32)
    mat = B.SparseMat(a, symmetric=True)
    owner = P.tile_owner_2d(32, 8)
    pd = B.setup(mat, 16, overlap=2, owner=owner, n_modes=4)
    monkeypatch.setenv("TLS_GPU_DECOMP", "0")
    ph = B.setup(mat, 16, overlap=2, owner=owner, n_modes=4)
    for m1, m2 in zip(pd.maps, ph.maps):
        assert np.array_equal(m1.indices, m2.indices)
    assert pd.k_c == ph.k_c and np.array_equal(pd.colors, ph.colors)
    r = np.random.default_rng(0).standard_normal(a.shape[0])
    assert np.array_equal(pd.apply(r), ph.apply(r))
