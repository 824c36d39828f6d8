"""Device memory across repeated setups (leak / cycle check): python tools/mem_check.py [cfg]"""
import gc
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_03915_b200 as B  # noqa: E402
from paper_2401_03915_b200 import problems as PR  # noqa: E402

cfg = PR.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)


def report(tag):
    free, total = torch.cuda.mem_get_info()
    print(f"{tag:28s} used {(total - free) / 2**30:7.2f} GiB  torch alloc {torch.cuda.memory_allocated() / 2**30:6.2f}"
          f"  reserved {torch.cuda.memory_reserved() / 2**30:6.2f}", flush=True)


report("start")
for i in range(3):
    pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
    report(f"after setup {i}")
    del pre
    report(f"after del {i}")
    print("gc collected", gc.collect())
    report(f"after gc {i}")
