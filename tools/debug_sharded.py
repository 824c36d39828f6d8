import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import golden, golden_csr
import paper_2401_03915_b200 as B
from paper_2401_03915_b200.distributed import LocalGroup
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_m16"
for nr in (2, 1, 2):
    d = dict(golden(name)); a = golden_csr(d)
    grp = LocalGroup(nr)
    def body(shard):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            mat = B.SparseMat(a, symmetric=bool(d["symmetric"]))
            pre = B.setup(mat, int(d["n_sub"]), overlap=int(d["overlap"]), owner=d["owner"],
                          coarse=str(d["coarse"]), n_modes=int(d["n_modes"]), shard=shard)
            r = d["r"][0]
            z0 = pre.apply(r)
            out = (pre.apply_one_level(r), pre.coarse_apply(r), z0, (shard.lo, shard.hi))
            st.synchronize()
            return out
    res = grp.run(body)
    for rk, (z1, zc, z, slab) in enumerate(res):
        e1 = np.abs(z1 - d["z_one"][0]).max() / np.abs(d["z_one"][0]).max()
        ec = np.abs(zc - d["z_coarse"][0]).max() / np.abs(d["z_coarse"][0]).max()
        ez = np.abs(z - d["z"][0]).max() / np.abs(d["z"][0]).max()
        bad = np.nonzero(np.abs(zc - d["z_coarse"][0]) > 1e-8 * np.abs(d["z_coarse"][0]).max())[0]
        print(f"nr={nr} rank={rk} slab={slab} one={e1:.2e} coarse={ec:.2e} apply={ez:.2e} badc={bad[:5]} nbad={bad.size}", flush=True)
