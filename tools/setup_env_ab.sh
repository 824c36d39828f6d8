#!/bin/bash
# setup wall time under an env toggle (GPU box): VAR, VALUES, CID, REPS
for rep in $(seq 1 ${REPS:-2}); do
  for v in $VALUES; do
    env $VAR=$v timeout 900 python - <<'PY'
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2401_03915_b200 as B
from paper_2401_03915_b200 import problems as PR
from paper_2401_03915_b200.gpu_setup import warm_linalg
cid = int(os.environ.get("CID", "2"))
cfg = PR.CONFIGS[cid]
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
warm_linalg()
torch.cuda.synchronize()
t = time.perf_counter()
pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
torch.cuda.synchronize()
ts = time.perf_counter() - t
x, rep = (B.pcg(mat, pre, cfg.rhs(a.shape[0]), tol=cfg.tol, maxit=cfg.maxit) if cfg.solver == "pcg" else
          B.gmres(mat, pre, cfg.rhs(a.shape[0]), tol=cfg.tol, maxit=cfg.maxit, restart=cfg.restart))
print(os.environ.get("VAR"), "=", os.environ.get(os.environ.get("VAR", ""), ""), "cfg", cid, "setup", round(ts, 2),
      "its", rep.iterations, flush=True)
PY
  done
done
