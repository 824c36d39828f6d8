"""GPU utilisation (NVML, 20 ms samples) during one setup() of a configuration: how much of the
setup wall time the device is busy (the rest is host orchestration / synchronisation)."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import pynvml as N  # noqa: E402
import torch  # noqa: E402

import paper_2401_03915_b200 as B  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = B.problems.CONFIGS[cid]
a, sym, owner, nsub = cfg.build()
mat = B.SparseMat(a, symmetric=sym)
from paper_2401_03915_b200.gpu_setup import warm_linalg  # noqa: E402
warm_linalg()
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], threading.Event()


def run():
    while not stop.wait(0.02):
        samples.append((time.perf_counter(), N.nvmlDeviceGetUtilizationRates(h).gpu))


t = threading.Thread(target=run, daemon=True)
t.start()
t0 = time.perf_counter()
pre = B.setup(mat, nsub, overlap=cfg.overlap, owner=owner, n_modes=cfg.n_modes)
torch.cuda.synchronize()
t1 = time.perf_counter()
stop.set()
t.join()
u = np.array([s[1] for s in samples if t0 <= s[0] <= t1])
print(f"cfg{cid} setup {t1 - t0:.1f} s, GPU utilisation mean {u.mean():.0f}%, "
      f"share of samples >= 90%: {(u >= 90).mean():.2f}, == 0%: {(u == 0).mean():.2f}", flush=True)
