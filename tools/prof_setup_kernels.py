"""Setup under ncu: warm setup once, then profile ONE setup between cudaProfilerStart/Stop.

    ncu --profile-from-start off ... python tools/prof_setup_kernels.py [cfg] [m] [part]

Also prints the setup's wall time without the profiler when run plainly.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_03915_b200 as B  # noqa: E402
from paper_2401_03915_b200 import problems as PR  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = PR.CONFIGS[cid]
if len(sys.argv) > 3:
    cfg = cfg.scaled(int(sys.argv[2]), int(sys.argv[3]))
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
torch.cuda.synchronize()
torch.cuda.profiler.start()
t0 = time.perf_counter()
pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"setup {time.perf_counter() - t0:.3f} s, n={a.shape[0]}, subdomains={nsub}", file=sys.stderr)
