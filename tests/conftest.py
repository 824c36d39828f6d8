import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def golden_csr(d, prefix="a_"):
    if prefix + "data" not in d and "gen" in d and str(d["gen"]):
        # large fixtures store the generator spec, not the matrix (generators are pinned by
        # tests/test_host_logic.py and the stored small cases)
        from paper_2401_03915_b200 import problems
        cid, m, part = (int(v) for v in str(d["gen"]).split(":"))
        return problems.CONFIGS[cid].scaled(m, part).build()[0]
    return sp.csr_matrix((d[prefix + "data"], d[prefix + "indices"], d[prefix + "indptr"]))


CONFIG_CASES = ["cfg1", "cfg2_m16", "cfg2_m24", "cfg3_m64", "cfg4_m32", "cfg5_m16"]


@pytest.fixture(scope="session")
def built_lib():
    from paper_2401_03915_b200 import build
    build.build()
    from paper_2401_03915_b200 import _lib
    return _lib.load()
