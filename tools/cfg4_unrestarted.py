"""Configuration 4 at full size with the reference's DEFAULT solver settings: unrestarted GMRES
(src/krylov.py:127-195, maxit <= GMRES_MAXIT_CAP = 1000), tol 1e-7 -- does it converge where
GMRES(50) stagnates?  Prints iterations, converged, final reported and true
residual and the solve time (one B200)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_03915_b200 as B  # noqa: E402

cfg = B.problems.CONFIGS[4]
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
t0 = time.perf_counter()
pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
torch.cuda.synchronize()
t_setup = time.perf_counter() - t0
b = cfg.rhs(a.shape[0])
for maxit in (1000,):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = B.gmres(mat, pre, b, tol=cfg.tol, maxit=maxit)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    true = float(np.linalg.norm(b - a @ x) / np.linalg.norm(b))
    h = rep.residuals
    print(json.dumps({"config": cfg.name, "solver": "gmres unrestarted", "maxit": maxit, "iterations": rep.iterations,
                      "converged": bool(rep.converged), "final_reported": float(h[-1]), "true_residual": true,
                      "history_at": {str(k): float(h[k]) for k in (50, 100, 200, 400, 600, 800) if k < h.size},
                      "solve_s": t, "setup_s": t_setup, "time_to_solution_s": t_setup + t}), flush=True)
