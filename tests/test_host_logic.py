"""CPU tests of the product's host logic: generators, decomposition (bit-exact index sets),
ABI symbol table.  No GPU needed."""

import re

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import CONFIG_CASES, REPO, golden, golden_csr
from paper_2401_03915_b200 import partition as Pt
from paper_2401_03915_b200 import problems as P


def test_config1_generator_is_reference_matrix():
    d = golden("cfg1")
    a, sym, owner, nsub = P.CONFIGS[1].build()
    ref = golden_csr(d)
    assert sym and nsub == 16
    assert np.array_equal(a.indptr, ref.indptr) and np.array_equal(a.indices, ref.indices)
    assert np.array_equal(a.data, ref.data)
    assert np.array_equal(owner, d["owner"])


@pytest.mark.parametrize("name", CONFIG_CASES + ["cfg2_m48"])
def test_overlap_and_coloring_bit_exact(name):
    d = golden(name)
    a = golden_csr(d)
    g = Pt.symmetrized_graph(a)
    maps = Pt.extend_overlap(g, Pt.Partition(int(d["n_sub"]), d["owner"]), int(d["overlap"]))
    assert np.array_equal(np.concatenate([m.indices for m in maps]), d["indices"])
    assert np.array_equal([m.interior.size for m in maps], d["n_interior"])
    assert np.array_equal([m.n_boundary for m in maps], d["n_boundary"])
    k_c, colors = Pt.color_subdomains(maps)
    assert k_c == int(d["k_c"]) and np.array_equal(colors, d["colors"])


@pytest.mark.parametrize("key", ["p2d8_4", "p2d30_16", "spd40_4", "spd80_7"])
def test_partition_graph_matches_reference(key):
    d = golden("partitions")
    a = sp.csr_matrix((d[key + "_data"], d[key + "_indices"], d[key + "_indptr"]))
    part = Pt.partition_graph(Pt.symmetrized_graph(a), int(d[key + "_nsub"]))
    assert np.array_equal(part.owner, d[key + "_owner"])


def test_banded7_index_sets():
    """tests/test_partition.py:101-119 of the reference."""
    rows = [0, 0, 1, 1, 1, 2, 2, 2, 3, 3, 3, 4, 4, 4, 5, 5, 5, 6, 6]
    cols = [0, 1, 0, 1, 2, 1, 2, 3, 2, 3, 4, 3, 4, 5, 4, 5, 6, 5, 6]
    vals = [1, 2, 3, 4, 5, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20]
    a = sp.csr_matrix((vals, (rows, cols)), shape=(7, 7)).astype(float)
    g = Pt.symmetrized_graph(a)
    part = Pt.Partition(2, np.array([0, 0, 0, 1, 1, 1, 1]))
    m1 = Pt.extend_overlap(g, part, 1)
    assert m1[0].indices.tolist() == [0, 1, 2, 3] and m1[1].indices.tolist() == [3, 4, 5, 6, 2]
    m2 = Pt.extend_overlap(g, part, 2)
    assert m2[0].indices.tolist() == [0, 1, 2, 3, 4] and m2[1].indices.tolist() == [3, 4, 5, 6, 2, 1]
    assert Pt.boolean_pou(m2[1]).tolist() == [1, 1, 1, 1, 0, 0]


def test_stored_zeros_are_not_edges():
    """symmetrized_graph drops explicit zeros (src/sparsemat.py:189-190)."""
    a = sp.csr_matrix((np.array([2.0, 0.0, 0.0, 2.0, 1.0, 1.0, 2.0]),
                       np.array([0, 1, 0, 1, 2, 1, 2]), np.array([0, 2, 5, 7])), shape=(3, 3))
    g = Pt.symmetrized_graph(a)
    assert g.neighbors(0).tolist() == [] and g.neighbors(1).tolist() == [2]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_symmetric_fast_path_matches_general_graph(seed):
    rng = np.random.default_rng(seed)
    n = 300
    a = sp.random(n, n, density=0.03, random_state=seed, format="csr")
    a = (a + a.T).tocsr()
    a.setdiag(rng.standard_normal(n))
    a = a.tocsr()
    a.data[rng.random(a.data.size) < 0.1] = 0.0       # explicit stored zeros (symmetric ones too)
    a = (0.5 * (a + a.T)).tocsr()
    a.sort_indices()
    assert (a != a.T).nnz == 0
    g0 = Pt.symmetrized_graph(a)
    g1 = Pt.symmetrized_graph(a, symmetric=True)
    assert np.array_equal(g0.indptr, g1.indptr) and np.array_equal(g0.adjacency, g1.adjacency)
    for name in ["cfg1", "cfg2_m16", "cfg5_m16"]:
        d = golden(name)
        b = golden_csr(d)
        h0, h1 = Pt.symmetrized_graph(b), Pt.symmetrized_graph(b, symmetric=True)
        assert np.array_equal(h0.indptr, h1.indptr) and np.array_equal(h0.adjacency, h1.adjacency)


def test_partition_validation():
    with pytest.raises(ValueError):
        Pt.Partition(2, np.array([0, 0]))
    with pytest.raises(ValueError):
        Pt.Partition(2, np.array([0, 2]))


@pytest.mark.parametrize("cid,m,part,n_expected", [(2, 16, 8, 16 ** 3), (3, 32, 16, 32 ** 2),
                                                   (4, 16, 8, 2 * 15 * 16 + 256), (5, 12, 4, 12 ** 3)])
def test_config_generators_scaled(cid, m, part, n_expected):
    a, sym, owner, nsub = P.CONFIGS[cid].scaled(m, part).build()
    assert a.shape == (n_expected, n_expected)
    assert owner.size == n_expected and np.bincount(owner).min() > 0 and owner.max() + 1 == nsub
    assert np.all(np.diff(a.indptr) > 0)
    sym_vals = (a != a.T).nnz == 0
    assert sym_vals == (cid != 3)  # configs 2, 4, 5 exactly symmetric; 3 is nonsymmetric
    assert sym == (cid in (2, 5))


def test_config2_full_size_table_s():
    """SURVEY.md §8 Table S: n = 2,097,152, nnz = 14,581,760, 512 subdomains."""
    a, sym, owner, nsub = P.CONFIGS[2].build()
    assert a.shape[0] == 2097152 and a.nnz == 14581760 and nsub == 512
    assert np.bincount(owner).tolist() == [4096] * 512


def test_config3_and_4_sizes():
    a, _, _, nsub = P.CONFIGS[3].scaled(128, 64).build()
    assert a.nnz == 5 * 128 * 128 - 4 * 128 and nsub == 4
    # config 4 at full size: n = 785,408 (SURVEY.md Table S)
    m = 512
    assert 2 * (m - 1) * m + m * m == 785408


def test_aniso27_positive_definite_and_27_point():
    a, sym, owner, nsub = P.CONFIGS[5].scaled(8, 4, angle_block=4).build()
    assert a.nnz == 22 ** 3 - 0 or a.nnz == (3 * 8 - 2) ** 3
    assert np.linalg.eigvalsh(a.toarray()).min() > 0


def test_abi_exports_every_header_symbol(built_lib):
    """The C ABI library loads and exports every function declared in include/tls_b200.h."""
    import ctypes
    src = open(f"{REPO}/include/tls_b200.h").read()
    names = set(re.findall(r"^(?:int32_t|int64_t|void|const char\*)\s+(tls_[a-z_0-9]+)\s*\(", src, re.M))
    assert len(names) >= 18
    lib = ctypes.CDLL(f"{REPO}/paper_2401_03915_b200/libtls_b200.so")
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    from paper_2401_03915_b200 import _lib
    assert set(_lib.SIGNATURES) == names
    assert built_lib.tls_abi_version() == 2


def test_product_does_not_import_oracle():
    """The product path never routes through the oracle (no CPU fallback)."""
    import glob
    for path in glob.glob(f"{REPO}/paper_2401_03915_b200/**/*.py", recursive=True):
        text = open(path).read()
        assert "oracle" not in text.replace("no CPU fallback", ""), path


def test_gpu_entry_points_refuse_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import paper_2401_03915_b200 as B
    a, sym, owner, nsub = P.CONFIGS[1].scaled(16, 8).build()
    with pytest.raises(RuntimeError, match="CUDA"):
        B.SparseMat(a, symmetric=True).matvec(np.ones(a.shape[0]))
    with pytest.raises(RuntimeError, match="CUDA"):
        B.setup(B.SparseMat(a, symmetric=True), nsub, overlap=1, owner=owner, n_modes=2)
