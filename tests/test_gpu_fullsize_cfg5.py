"""Configuration 5 at FULL size (n = 16.8 M, nnz = 449 M, 4,096 subdomains; 96 GB on the device)
against the reference (tests/golden/full_cfg5.npz, oracle/make_golden_fullsize.py): every index
set and the colouring bit for bit (SHA-256 of the reference's own extend_overlap /
color_subdomains), 8 sampled subdomains' dense local solves to 1e-10 and top-k harmonic-pencil
spans to 1e-8, the Galerkin projection property, and the 534-iteration PCG solve's true residual.
Its own module so that it starts from an empty device (the smaller configurations' handles of
test_gpu_fullsize.py are released at that module's end)."""

import gc

import pytest

from test_gpu_fullsize import B, _check_sampled, _sampled_setup  # noqa: F401  (B: fixture)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_full_cfg5_against_reference(B):  # noqa: F811
    gc.collect()
    torch.cuda.empty_cache()
    data = _sampled_setup(B, 5)
    _check_sampled(B, data, 534)
