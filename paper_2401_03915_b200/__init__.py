"""B200-native two-level Schwarz preconditioned Krylov hot path (arXiv:2401.03915).

Drop-in mirror of the reference ``tlschwarz`` API for the solve path:
``SparseMat``, ``setup``, ``Preconditioner.apply``, ``pcg``, ``gmres`` (plus the
decomposition helpers whose index sets are bit-exact with the reference).  The
numerics run in libtls_b200.so (hand-written sm_100a CUDA, C ABI in
include/tls_b200.h).
"""

import os as _os

# The setup interleaves multi-GB batch workspaces with small long-lived blocks (coarse columns);
# PyTorch's default caching allocator then pins partly-used segments and fragments the device:
# configuration 5 (95 GB of factors + three 19 GB coarse buffers on a 178 GB device) needs its
# expandable (virtual-memory) segments.  Read when the allocator is first used; a user setting wins.
_os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

from .errors import BreakdownError, SubdomainSetupError  # noqa: E402
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
