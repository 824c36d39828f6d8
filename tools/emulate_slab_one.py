"""One rank's slab of a configuration, band local operators only (as tools/emulate_slabs.py), for
profiling its k_band_solve* launch under ncu:  python tools/emulate_slab_one.py <cfg> <N> <q>."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n, q = int(sys.argv[2]), int(sys.argv[3])
sys.argv = sys.argv[:2]
import tools.emulate_slabs as E  # noqa: E402  (sets up the maps of configuration argv[1])

ms, algo, cnt = E.band_time(n, q)
print(f"rank {q} of {n}: {cnt} subdomains, band launch {ms:.4f} ms, {algo / ms / 1e6:.1f} GB/s", flush=True)
