"""Golden fixtures for the file boundary (Matrix Market) by running the REFERENCE itself.

    python oracle/make_golden_io.py                 # writes tests/golden/mm_cases.json
    python oracle/make_golden_io.py --experiments   # writes tests/golden/experiments.json
    python oracle/make_golden_io.py --pou           # writes tests/golden/pou.npz

Test infrastructure only (this container: /root/reference is imported read-only).  Every case is
a Matrix Market / vector text and what the reference's ``read_matrix_market`` / ``read_vector``
(src/sparsemat.py:227-357) returns for it: the canonical CSR (shape, symmetric flag, indptr,
indices, values as hex floats) or the MatrixMarketError line and message.  Round-trip cases pin
``write_matrix_market`` (src/sparsemat.py:323-332) byte for byte.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import scipy.sparse as sp  # noqa: E402
import tlschwarz as T  # noqa: E402
from tlschwarz import sparsemat as SM  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden", "mm_cases.json")

H_GEN = "%%MatrixMarket matrix coordinate real general"
H_SYM = "%%MatrixMarket matrix coordinate real symmetric"
H_ARR = "%%MatrixMarket matrix array real general"
H_ARS = "%%MatrixMarket matrix array real symmetric"

HAND = [
    H_GEN + "\n3 3 4\n1 1 2\n2 2 3\n3 3 4\n1 3 -1.5\n",
    H_SYM + "\n3 3 4\n1 1 2\n2 1 -1\n3 3 5\n3 2 0\n",                   # explicit zero kept
    H_GEN + "\n2 2 3\n1 1 1\n1 1 2.5\n2 1 1e-3\n",                       # duplicates summed
    "\n\n  " + H_GEN + "  \n% comment\n\n2 3 2\n% c\n1 3 7\n\n2 1 -0.0\n",  # blanks, comments
    H_GEN + "\r\n2 2 2\r\n1 1 1\r\n2 2 2\r\n",                          # CRLF
    H_GEN + "\r2 2 1\r2 2 5\r",                                         # bare CR
    H_GEN + "\n3 3 0\n",
    H_GEN + "\n0 0 0\n",
    H_ARR + "\n2 3\n1\n0\n3\n4\n0\n6\n",
    H_ARS + "\n3 3\n1\n2\n3\n4\n5\n6\n",
    H_ARR + "\n2 2\n1 2\n3 4\n",                                        # several values per line
    "%%matrixmarket MATRIX Coordinate REAL General\n1 1 1\n1 1 +1.5E+02\n",
    H_GEN + "\n2 2 1\n0002 1_0 1\n".replace("1_0", "1"),
    H_GEN + "\n2 2 1\n2 1 1_000.5\n",
    H_GEN + "\n2 2 1\n2 1 .5\n",
    H_GEN + "\n2 2 1\n2 1 5.\n",
    H_GEN + "\n2 2 1\n2 1 1e-400\n",
    # errors
    "",
    "\n\n",
    "% not a header\n",
    "%%MatrixMarket matrix coordinate real\n1 1 0\n",
    "%%MatrixMarket vector coordinate real general\n1 1 0\n",
    "%%MatrixMarket matrix sparse real general\n1 1 0\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 0\n",
    "%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n",
    H_GEN + "\n",
    H_GEN + "\n% only comments\n\n",
    H_GEN + "\n2 2\n",
    H_GEN + "\n2 x 1\n1 1 1\n",
    H_GEN + "\n2 2 1.0\n1 1 1\n",
    H_GEN + "\n-2 2 1\n1 1 1\n",
    H_GEN + "\n2 2 3\n1 1 1\n2 2 1\n",
    H_GEN + "\n2 2 1\n1 1 1\n2 2 1\n\n% trailing\n",
    H_GEN + "\n2 2 0\n\n",
    H_GEN + "\n2 2 2\n1 1\n2 2 1\n",
    H_GEN + "\n2 2 2\n1 1 1\n2 2 1 9\n",
    H_GEN + "\n2 2 1\n1.0 1 1\n",
    H_GEN + "\n2 2 1\n1 b 1\n",
    H_GEN + "\n2 2 1\n3 1 1\n",
    H_GEN + "\n2 2 1\n0 1 1\n",
    H_GEN + "\n2 2 1\n1 1 abc\n",
    H_GEN + "\n2 2 1\n1 1 inf\n",
    H_GEN + "\n2 2 1\n1 1 NaN\n",
    H_GEN + "\n2 2 1\n1 1 1e400\n",
    H_GEN + "\n2 2 1\n1 1 0x10\n",
    H_GEN + "\n2 2 1\n1 1 'q'\n",
    H_SYM + "\n2 2 1\n1 2 1\n",
    H_GEN + "\n2 2 2\n1 1 x\n9 9 1\n",                                  # first error wins
    H_ARR + "\n2 2\n1\n2\n3\n",
    H_ARS + "\n2 3\n1\n2\n3\n",
    H_ARR + "\n2 2\n1\n2\nz\n4\n",
    H_ARR + "\n2\n1\n",
]


def canonical(m):
    csr = m.scipy()
    return {"shape": list(csr.shape), "symmetric": bool(m.symmetric), "indptr": csr.indptr.tolist(),
            "indices": csr.indices.tolist(), "data": [float(v).hex() for v in csr.data]}


def run(text):
    try:
        return {"ok": canonical(SM.read_matrix_market(text))}
    except SM.MatrixMarketError as e:
        return {"error": [int(e.lineno), str(e)]}


def main():
    rng = np.random.default_rng(11)
    cases = [{"text": t, **run(t)} for t in HAND]
    # random round trips through the reference writer (+ comment / blank-line noise)
    for k in range(12):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(1, 40)) if k % 3 else n
        dens = float(rng.uniform(0.02, 0.4))
        a = sp.random(n, m, density=dens, random_state=int(rng.integers(1 << 30)), format="csr")
        a.data = rng.standard_normal(a.nnz) * 10.0 ** rng.integers(-8, 9, a.nnz)
        if k % 3 == 0:
            a = (a + a.T).tocsr()
        mat = T.SparseMat(a, symmetric=(k % 3 == 0))
        text = SM.write_matrix_market(mat)
        lines = text.splitlines()
        noisy = [lines[0]]
        for ln in lines[1:]:
            if rng.random() < 0.1:
                noisy.append("% noise " + str(rng.integers(100)))
            if rng.random() < 0.05:
                noisy.append("   ")
            noisy.append(ln)
        cases.append({"text": text, "roundtrip": True, **run(text)})
        cases.append({"text": "\n".join(noisy) + "\n", **run("\n".join(noisy) + "\n")})
        # symmetric lower-triangle storage of the same symmetric matrix
        if k % 3 == 0:
            low = sp.tril(a).tocoo()
            body = [f"{i + 1} {j + 1} {v:.17g}" for i, j, v in zip(low.row, low.col, low.data)]
            t2 = H_SYM + f"\n{n} {n} {len(body)}\n" + "\n".join(body) + "\n"
            cases.append({"text": t2, **run(t2)})
    vec_cases = []
    for t in ["1\n2.5\n-3e-2\n", "% c\n1 2\n3\n\n", "%%MatrixMarket matrix array real general\n3 1\n1\n0\n2\n",
              "1\nfoo\n", "1\ninf\n", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n"]:
        try:
            vec_cases.append({"text": t, "ok": [float(v).hex() for v in SM.read_vector(t)]})
        except SM.MatrixMarketError as e:
            vec_cases.append({"text": t, "error": [int(e.lineno), str(e)]})
        except ValueError as e:
            vec_cases.append({"text": t, "value_error": str(e)})
    with open(OUT, "w") as fh:
        json.dump({"matrices": cases, "vectors": vec_cases}, fh, indent=0)
    print(f"{len(cases)} matrix cases, {len(vec_cases)} vector cases -> {OUT}")


if __name__ == "__main__" and not {"--experiments", "--pou"} & set(sys.argv):
    main()


# -- run_experiment / CLI (src/harness.py:326-371) ---------------------------------------------
EXP_OUT = os.path.join(REPO, "tests", "golden", "experiments.json")

EXPERIMENTS = [
    dict(kind="poisson2d", m=24, n_subdomains=4, overlap=2, tau=0.1, solver="cg"),
    dict(kind="hetero2d", m=24, n_subdomains=9, overlap=1, tau=0.1, solver="cg", seed=3),
    dict(kind="advection2d", m=24, n_subdomains=4, overlap=2, tau=0.1, solver="gmres"),
    dict(kind="poisson3d", m=9, n_subdomains=8, overlap=1, tau=0.2, solver="cg", coarse="gevp",
         one_level="ras", combine="deflated"),
    dict(kind="poisson2d", m=24, n_subdomains=4, overlap=1, tau=0.1, solver="gmres", coarse="svd"),
    dict(kind="poisson2d", m=24, n_subdomains=4, overlap=1, solver="cg", coarse="none", maxit=60),
    dict(matrix="mm", rhs="vec", n_subdomains=4, overlap=1, tau=0.1, solver="cg"),
]


def experiments():
    import tempfile
    from tlschwarz import harness as Hh
    out = []
    tmp = tempfile.mkdtemp()
    mat, _ = T.generate(T.ProblemSpec("hetero-diffusion2d", 22, channel_seed=5))
    mm_text = SM.write_matrix_market(mat)
    rhs = np.random.default_rng(9).uniform(-1, 1, mat.nrows)
    vec_text = SM.write_vector(rhs)
    for e in EXPERIMENTS:
        kw = dict(e)
        if kw.pop("matrix", None):
            kw.pop("rhs")
            mp, vp = os.path.join(tmp, "a.mtx"), os.path.join(tmp, "b.txt")
            with open(mp, "w") as fh:
                fh.write(mm_text)
            with open(vp, "w") as fh:
                fh.write(vec_text)
            kw.update(matrix_path=mp, rhs_path=vp)
        res = Hh.run_experiment(Hh.ExperimentConfig(report_path=os.path.join(tmp, "r.txt"), **kw))
        with open(os.path.join(tmp, "r.txt.history")) as fh:
            hist = fh.read()
        out.append({"config": e, "report": res.precond.report.to_text(),
                    "iterations": res.solve_report.iterations, "converged": bool(res.solve_report.converged),
                    "residuals": [float(v) for v in res.solve_report.residuals],
                    "cond_estimate": res.solve_report.cond_estimate, "x": [float(v) for v in res.x],
                    "history_lines": len(hist.splitlines()), "bound_check": res.bound_check is not None})
    with open(EXP_OUT, "w") as fh:
        json.dump({"mm_text": mm_text, "vec_text": vec_text, "cases": out}, fh)
    print(f"{len(out)} experiments -> {EXP_OUT}")


if __name__ == "__main__" and "--experiments" in sys.argv:
    experiments()


# -- partition-of-unity modes (src/spectral.py:93-108) -------------------
POU_OUT = os.path.join(REPO, "tests", "golden", "pou.npz")

POU_CASES = [
    ("poisson2d", 16, 4, 2, 0.1, 1.5, "gevp"),
    ("hetero-diffusion2d", 16, 4, 1, 0.1, 1.3, "gevp"),
    ("poisson2d", 20, 9, 1, 0.1, 1.2, "full"),
    ("poisson3d", 8, 8, 1, 0.2, 1.25, "gevp"),
    ("poisson2d", 16, 4, 2, 0.1, 1.5, "svd"),
    ("poisson2d", 16, 4, 1, 0.1, 50.0, "gevp"),   # threshold above every PoU value: none added
]


def pou():
    arrs = {}
    rng = np.random.default_rng(21)
    for c, (kind, m, N, d, tau, nu, coarse) in enumerate(POU_CASES):
        mat, b = T.generate(T.ProblemSpec(kind, m))
        pre = T.setup(mat, N, overlap=d, tau=tau, nu=nu, coarse=coarse)
        csr = mat.scipy()
        r = rng.standard_normal(mat.nrows)
        x, rep = T.pcg(mat, pre, b, tol=1e-10)
        pou_counts = [pb.n_selected for pb in pre.pou_bases]
        gaps = []
        for pb in pre.pou_bases:  # distance of the threshold to the nearest PoU value
            v = pb.all_values
            gaps.append(float(np.min(np.abs(v - nu)) / nu))
        Z = pre.coarse.basis.scipy().toarray()
        cond_a0 = float(np.linalg.cond(Z.T @ (csr @ Z)))
        p = f"c{c}_"
        arrs.update({p + "cond_a0": cond_a0, p + "indptr": csr.indptr, p + "indices": csr.indices, p + "data": csr.data,
                     p + "params": np.array([m, N, d, tau, nu]), p + "kind": np.array(kind),
                     p + "coarse": np.array(coarse), p + "mode_counts": np.array(pre.report.mode_counts),
                     p + "pou_counts": np.array(pou_counts), p + "n_coarse": pre.report.n_coarse,
                     p + "r": r, p + "z": pre.apply(r), p + "b": b, p + "x": x,
                     p + "iterations": rep.iterations, p + "residuals": rep.residuals,
                     p + "min_gap": min(gaps)})
        print(kind, coarse, nu, pre.report.mode_counts, pou_counts, rep.iterations, f"gap {min(gaps):.2e}",
              f"cond(A0) {cond_a0:.2e}")
    arrs["n_cases"] = len(POU_CASES)
    np.savez_compressed(POU_OUT, **arrs)


if __name__ == "__main__" and "--pou" in sys.argv:
    pou()
