"""B200-native two-level Schwarz preconditioned Krylov hot path (arXiv:2401.03915).

Drop-in mirror of the reference ``tlschwarz`` API for the solve path:
``SparseMat``, ``setup``, ``Preconditioner.apply``, ``pcg``, ``gmres`` (plus the
decomposition helpers whose index sets are bit-exact with the reference).  The
numerics run in libtls_b200.so (hand-written sm_100a CUDA, C ABI in
include/tls_b200.h).
"""

from .errors import BreakdownError, SubdomainSetupError
from .partition import (
    Graph,
    Partition,
    SubdomainMap,
    boolean_pou,
    color_subdomains,
    extend_overlap,
    partition_graph,
)
from .sparsemat import DENSE_GUARD, SparseMat, as_sparsemat, symmetrized_graph
from .mmio import (
    MatrixMarketError,
    load_matrix_market,
    load_vector,
    read_matrix_market,
    read_vector,
    save_matrix_market,
    save_vector,
    write_matrix_market,
    write_vector,
)
from .precond import Preconditioner, SetupReport, setup
from .krylov import SolveReport, gmres, pcg
from . import problems

__all__ = [name for name in dir() if not name.startswith("_")]
__version__ = "0.1.0"
