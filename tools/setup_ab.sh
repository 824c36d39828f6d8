#!/bin/bash
# setup wall time A/B: current tree vs _old worktree, alternating (GPU box)
for rep in 1 2; do
  for tree in . _old; do
    (cd $tree && timeout 600 python - <<'PY'
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2401_03915_b200 as B
from paper_2401_03915_b200 import problems as PR
cid = int(os.environ.get("CID", "3"))
cfg = PR.CONFIGS[cid]
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
from paper_2401_03915_b200.gpu_setup import warm_linalg
warm_linalg()
torch.cuda.synchronize()
t = time.perf_counter()
B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
torch.cuda.synchronize()
print(os.getcwd().split("/")[-1], "cfg", cid, "setup", round(time.perf_counter() - t, 2), flush=True)
PY
    )
  done
done
