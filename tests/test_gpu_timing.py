"""In-graph timing of the band local-solve kernel (bench roofline inside real solves): the event
nodes see one launch per PCG iteration that did work, and do not change the solve."""

import ctypes as C

import numpy as np
import pytest

from conftest import golden, golden_csr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_03915_b200 import build
    build.build()
    import paper_2401_03915_b200 as mod
    return mod


@pytest.mark.parametrize("name,solver", [("cfg2_m24", "pcg"), ("cfg3_m64", "gmres")])
def test_in_graph_band_timing(B, name, solver):
    d = golden(name)
    a = golden_csr(d)
    mat = B.SparseMat(a, symmetric=bool(d["symmetric"]))
    pre = B.setup(mat, int(d["n_sub"]), overlap=int(d["overlap"]), owner=d["owner"], coarse=str(d["coarse"]),
                  n_modes=int(d["n_modes"]), local="band")
    run = (lambda: B.pcg(mat, pre, d["b"], tol=float(d["tol"]))) if solver == "pcg" else \
        (lambda: B.gmres(mat, pre, d["b"], tol=float(d["tol"]), restart=int(d["restart"])))
    x0, r0 = run()
    h = pre.handle
    h.check(h.lib.tls_set_kernel_timing(h.ctx, 1))
    x1, r1 = run()
    ms, n = C.c_double(), C.c_int64()
    h.check(h.lib.tls_kernel_timing(h.ctx, C.byref(ms), C.byref(n)))
    h.check(h.lib.tls_set_kernel_timing(h.ctx, 0))
    assert np.array_equal(x0, x1) and r0.iterations == r1.iterations
    assert ms.value > 0.0
    if solver == "pcg":  # one band solve per iteration inside the graph (the first apply is outside)
        assert r1.iterations - 2 <= n.value <= r1.iterations
    else:
        assert n.value >= r1.iterations
