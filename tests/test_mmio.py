"""Matrix Market boundary (src/sparsemat.py:201-372) on the native reader, CPU only.

Every case in tests/golden/mm_cases.json was produced by the REFERENCE's own reader
(oracle/make_golden_io.py): the native parser must return the identical canonical CSR (bit for
bit) or raise MatrixMarketError with the identical line number and message."""

import json
import os

import numpy as np
import pytest

import paper_2401_03915_b200 as P

GOLD = os.path.join(os.path.dirname(__file__), "golden", "mm_cases.json")


def _cases():
    with open(GOLD) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def lib():
    from paper_2401_03915_b200 import build
    build.build()


def _check(m, exp):
    csr = m.scipy()
    assert list(csr.shape) == exp["shape"] and m.symmetric == exp["symmetric"]
    assert csr.indptr.tolist() == exp["indptr"] and csr.indices.tolist() == exp["indices"]
    assert [float(v).hex() for v in csr.data] == exp["data"]


@pytest.mark.parametrize("nthreads", [1, 3])
def test_reader_matches_reference(lib, nthreads):
    for case in _cases()["matrices"]:
        if "ok" in case:
            _check(P.read_matrix_market(case["text"], nthreads=nthreads), case["ok"])
        else:
            with pytest.raises(P.MatrixMarketError) as ei:
                P.read_matrix_market(case["text"], nthreads=nthreads)
            assert [ei.value.lineno, str(ei.value)] == case["error"], case["text"][:80]


def test_writer_matches_reference_bytes(lib, tmp_path):
    for case in _cases()["matrices"]:
        if not case.get("roundtrip"):
            continue
        m = P.read_matrix_market(case["text"])
        assert P.write_matrix_market(m) == case["text"]
        path = tmp_path / "m.mtx"
        P.save_matrix_market(str(path), m, nthreads=3)
        assert path.read_text() == case["text"]
        _check(P.load_matrix_market(str(path)), case["ok"])


def test_vectors_match_reference(lib):
    for case in _cases()["vectors"]:
        if "ok" in case:
            assert [float(v).hex() for v in P.read_vector(case["text"])] == case["ok"]
        elif "error" in case:
            with pytest.raises(P.MatrixMarketError) as ei:
                P.read_vector(case["text"])
            assert [ei.value.lineno, str(ei.value)] == case["error"]
        else:
            with pytest.raises(ValueError, match=case["value_error"]):
                P.read_vector(case["text"])


def test_large_parallel_parse_equals_serial(lib, tmp_path):
    """A multi-chunk file (> 1 MiB, 8 threads) parses to the same CSR as one thread, including
    the line number of an error placed deep inside a later chunk."""
    import scipy.sparse as sp
    rng = np.random.default_rng(3)
    nnz = 600_000
    a = sp.csr_matrix((rng.standard_normal(nnz), (rng.integers(0, 20000, nnz), rng.integers(0, 20000, nnz))),
                      shape=(20000, 20000))
    m = P.SparseMat(a)
    text = P.write_matrix_market(m)
    assert len(text) > (1 << 20)
    m1 = P.read_matrix_market(text, nthreads=1)
    m8 = P.read_matrix_market(text, nthreads=8)
    for x in (m1, m8):
        assert (x.scipy() != a).nnz == 0 and np.array_equal(x.scipy().data, a.data)
    lines = text.splitlines()
    bad = len(lines) - 17
    lines[bad] = lines[bad].rsplit(" ", 1)[0] + " 1.2.3"
    with pytest.raises(P.MatrixMarketError) as ei:
        P.read_matrix_market("\n".join(lines) + "\n", nthreads=8)
    assert ei.value.lineno == bad + 1 and "expected a real value, got '1.2.3'" in str(ei.value)


def test_missing_file_raises_oserror(lib, tmp_path):
    with pytest.raises(OSError):
        P.load_matrix_market(str(tmp_path / "nope.mtx"))


def test_cli_usage_error_without_gpu(capsys):
    from paper_2401_03915_b200 import cli
    assert cli.main([]) == 2
    assert "need --matrix or --kind" in capsys.readouterr().err
    args = cli.build_parser().parse_args(["--kind", "hetero2d", "--N", "9", "--delta", "1", "--one-level", "ras"])
    cfg = cli.config_from_args(args)
    assert (cfg.kind, cfg.n_subdomains, cfg.overlap, cfg.one_level, cfg.solver) == ("hetero2d", 9, 1, "ras", "cg")


def test_generate_matches_reference_fixture_kinds():
    """generate(): the reference's four model problems, rhs = A * ones on the host."""
    from paper_2401_03915_b200 import harness as H
    with pytest.raises(ValueError):
        H.ProblemSpec("poisson4d", 8)
    with pytest.raises(ValueError):
        H.ProblemSpec("poisson2d", 2)
    m, b = H.generate(H.ProblemSpec("advection2d", 6))
    assert not m.symmetric and np.array_equal(b, m.scipy() @ np.ones(36))
