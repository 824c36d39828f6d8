"""cProfile + stage timing of setup() on one configuration (run on the GPU box)."""
import cProfile, pstats, sys, os, time, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_03915_b200 as B
from paper_2401_03915_b200 import problems as PR
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = PR.CONFIGS[cid]
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
if "--no-warm" not in sys.argv:
    B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)  # warm (cuSOLVER init)
else:
    from paper_2401_03915_b200.gpu_setup import warm_linalg
    warm_linalg()
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
torch.cuda.synchronize()
pr.disable()
print("setup", time.perf_counter() - t0)
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(60)
s2 = io.StringIO()
pstats.Stats(pr, stream=s2).sort_stats("tottime").print_stats(25)
print(s2.getvalue())
print(s.getvalue())
