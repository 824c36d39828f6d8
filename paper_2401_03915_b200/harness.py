"""Experiment driver on the GPU backend (src/harness.py:26-53, 276-371).

``run_experiment(config)`` loads a Matrix Market problem (native reader) or generates one of the
reference's model problems (``generate``: bit-identical CSR, rhs = A * ones computed on the host
like the reference), builds the preconditioner with ``setup`` and solves with ``pcg`` (with the
tridiagonal condition estimate) or ``gmres`` -- all on the device -- and writes the same report
and ``.history`` files.  The theory bound check of the reference (``_bound_verdict``: dense
lambda*, partition-of-unity spectra and the exact condition number for n <= 400) is out of scope
(theory diagnostics); ``bound_check`` is None and the report omits those lines.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import krylov
from . import problems as PR
from .mmio import load_matrix_market, load_vector
from .precond import Preconditioner, setup
from .sparsemat import SparseMat

PROBLEM_KINDS = ("poisson2d", "poisson3d", "hetero-diffusion2d", "advection2d")


@dataclass(frozen=True)
class ProblemSpec:
    """Parameters of a generated test problem (src/harness.py:26-41)."""

    kind: str
    m: int
    contrast: float = 1.0e4
    channel_seed: int = 0
    velocity: tuple = (1.0, 0.0)
    eps: float = 1.0e-2

    def __post_init__(self):
        if self.kind not in PROBLEM_KINDS:
            raise ValueError(f"unknown problem kind {self.kind!r}")
        if self.m < 3:
            raise ValueError("grid size m must be at least 3")


def generate(spec):
    """(matrix, rhs) with rhs = A * ones (src/harness.py:44-53)."""
    if spec.kind == "poisson2d":
        csr, sym = PR.poisson2d(spec.m), True
    elif spec.kind == "poisson3d":
        csr, sym = PR.poisson3d(spec.m), True
    elif spec.kind == "hetero-diffusion2d":
        csr, sym = PR.hetero2d(spec.m, contrast=spec.contrast, channel_seed=spec.channel_seed), True
    else:
        csr, sym = PR.advection2d(spec.m, velocity=spec.velocity, eps=spec.eps), False
    matrix = SparseMat(csr, symmetric=sym)
    return matrix, matrix.scipy() @ np.ones(matrix.nrows)


@dataclass
class ExperimentConfig:
    """src/harness.py:276-293."""

    matrix_path: str | None = None
    rhs_path: str | None = None
    kind: str | None = None
    m: int = 20
    n_subdomains: int = 4
    overlap: int = 2
    tau: float = 0.1
    nu: float | None = None
    coarse: str = "auto"
    one_level: str | None = None
    combine: str | None = None
    solver: str = "cg"
    tol: float = 1e-8
    maxit: int = 500
    report_path: str | None = None
    seed: int = 0


@dataclass
class ExperimentResult:
    matrix: SparseMat
    rhs: np.ndarray
    x: np.ndarray
    precond: Preconditioner
    solve_report: krylov.SolveReport
    bound_check: dict | None
    report_text: str


def _load_problem(config):
    """src/harness.py:307-323."""
    if config.matrix_path:
        matrix = load_matrix_market(config.matrix_path)
        if not matrix.symmetric and matrix.is_numerically_symmetric():
            matrix = matrix.as_symmetric()
        if config.rhs_path:
            rhs = load_vector(config.rhs_path)
            if rhs.size != matrix.nrows:
                raise ValueError("right-hand side length does not match the matrix")
        else:
            rhs = matrix.scipy() @ np.ones(matrix.nrows)
        return matrix, rhs
    if not config.kind:
        raise ValueError("either a matrix file or a problem kind is required")
    kind = {"hetero2d": "hetero-diffusion2d"}.get(config.kind, config.kind)
    return generate(ProblemSpec(kind=kind, m=config.m, channel_seed=config.seed))


def run_experiment(config):
    """Set up, solve on the GPU, write the report (src/harness.py:326-371)."""
    matrix, rhs = _load_problem(config)
    precond = setup(matrix, config.n_subdomains, overlap=config.overlap, tau=config.tau, nu=config.nu,
                    coarse=config.coarse, one_level=config.one_level, combine=config.combine)
    if config.solver == "cg":
        x, solve_report = krylov.pcg(matrix, precond, rhs, tol=config.tol, maxit=config.maxit,
                                     track_tridiagonal=True)
    elif config.solver == "gmres":
        x, solve_report = krylov.gmres(matrix, precond, rhs, tol=config.tol, maxit=config.maxit)
    else:
        raise ValueError(f"unknown solver {config.solver!r}")
    report_text = precond.report.to_text() + solve_report.to_text()
    if config.report_path:
        with open(config.report_path, "w") as fh:
            fh.write(report_text)
        with open(config.report_path + ".history", "w") as fh:
            for k, res in enumerate(solve_report.residuals):
                fh.write(f"{k} {res:.17g}\n")
    return ExperimentResult(matrix, rhs, x, precond, solve_report, None, report_text)
