"""Configuration-4 family numerics on the default band-LU path, with and without the coarse
refinement step (TLS_COARSE_REFINE): cond_1(A0), apply / coarse-apply error vs the reference
fixtures, GMRES(50) history error, iterations, true residual.  Run on the GPU box."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import golden, golden_csr  # noqa: E402

import paper_2401_03915_b200 as B  # noqa: E402
from paper_2401_03915_b200 import gpu_setup as G  # noqa: E402

for name in ("cfg4_m32", "cfg4_m64_stall"):
    d = golden(name)
    a = golden_csr(d)
    for ref_on in ("1", "0"):
        os.environ["TLS_COARSE_REFINE"] = ref_on
        old = G.REFINE_COND
        G.REFINE_COND = 0.0 if ref_on == "1" else old  # force the step on every case
        mat = B.SparseMat(a)
        pre = B.setup(mat, int(d["n_sub"]), overlap=int(d["overlap"]), owner=d["owner"], coarse="svd",
                      n_modes=20)
        G.REFINE_COND = old
        r, z, zc = d["r"][0], d["z"][0], d["z_coarse"][0]
        ez = float(np.abs(pre.apply(r) - z).max() / np.abs(z).max())
        ec = float(np.abs(pre.coarse_apply(r) - zc).max() / np.abs(zc).max())
        maxit = int(d["maxit"])
        x, rep = B.gmres(mat, pre, d["b"], tol=float(d["tol"]), maxit=maxit, restart=50)
        k = min(rep.residuals.size, d["history"].size)
        eh = float(np.abs(rep.residuals[:k] - d["history"][:k]).max())
        tr = float(np.linalg.norm(d["b"] - a @ x) / np.linalg.norm(d["b"]))
        print(json.dumps({"case": name, "refine": pre.coarse.refined, "cond1": pre.coarse.cond1,
                          "local": pre.local_kind, "apply_err": ez, "coarse_err": ec, "hist_err": eh,
                          "its": rep.iterations, "ref_its": int(d["iterations"]), "true_res": tr,
                          "ref_true": float(d["true_residual"])}), flush=True)
