"""TLS_VERBOSE timeline of one warm setup() (GPU box): python tools/setup_timeline.py [cfg]"""
import os
import sys
import time
os.environ["TLS_VERBOSE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2401_03915_b200 as B  # noqa: E402
from paper_2401_03915_b200.gpu_setup import warm_linalg  # noqa: E402
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = B.problems.CONFIGS[cid]
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
warm_linalg()
torch.cuda.synchronize()
t0 = time.perf_counter()
pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
torch.cuda.synchronize()
print(f"setup total {time.perf_counter() - t0:.2f} s", flush=True)
