"""Short profiling driver: set up one configuration, one warm solve, then a few solves.

    python tools/prof_apply.py --config 2 [--solves 1]

Used under ncu (launch list / --set full on k_symv_tiles); prints timing of the plain run.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2401_03915_b200 as B
from paper_2401_03915_b200 import problems as PR

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--scale", type=int, default=0)
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--maxit", type=int, default=0)
ap.add_argument("--applies", type=int, default=0)
args = ap.parse_args()
cfg = PR.CONFIGS[args.config]
if args.scale:
    cfg = cfg.scaled(args.scale)
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
t0 = time.perf_counter()
pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
torch.cuda.synchronize()
print(f"setup {time.perf_counter() - t0:.2f}s n_coarse={pre.report.n_coarse} bytes={pre.device_bytes()}", flush=True)
b = torch.as_tensor(cfg.rhs(a.shape[0]), device="cuda")
for i in range(args.applies):
    t0 = time.perf_counter()
    z = pre.apply(b)
    torch.cuda.synchronize()
    print(f"apply {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
maxit = args.maxit or 500
for i in range(args.solves + 1):
    t0 = time.perf_counter()
    if cfg.solver == "pcg":
        x, rep = B.pcg(mat, pre, b, tol=cfg.tol, maxit=maxit)
    else:
        x, rep = B.gmres(mat, pre, b, tol=cfg.tol, maxit=maxit, restart=cfg.restart)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"solve {i}: {rep.iterations} its, {dt*1e3:.1f} ms, {rep.iterations/dt:.1f} it/s, "
          f"final {rep.residuals[-1]:.3e}, launches {rep.gpu_launches}", flush=True)
