"""torch.profiler (CPU + CUDA activity) of one setup() on a configuration (GPU box): where the
host time goes, how busy the GPU is.  python tools/torchprof_setup.py [cfg] [m part]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

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
t0 = time.perf_counter()
B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
torch.cuda.synchronize()
print(f"setup wall (no profiler) {time.perf_counter() - t0:.3f} s")
torch.cuda.empty_cache()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=False) as prof:
    t0 = time.perf_counter()
    B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ka = prof.key_averages()
cuda_total = sum(e.self_device_time_total for e in ka) / 1e6
print(f"setup wall (profiled) {wall:.3f} s, GPU kernel time {cuda_total:.3f} s")
print(ka.table(sort_by="self_cpu_time_total", row_limit=25, max_name_column_width=60))
print(ka.table(sort_by="self_device_time_total", row_limit=25, max_name_column_width=60))
