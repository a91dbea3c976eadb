"""B200-native additive FAC / adaFACx multigrid (hot path of arXiv 1903.10367).

Public surface mirrors the reference package ``treemg``:
``spacetree`` (mesh model), ``solvers`` (``SolverConfig``, ``CycleStats``,
``GpuEngine`` -- the ReferenceEngine protocol on the GPU), ``workloads``
(seeded BASELINE inputs).  Compute lives in ``libtmg.so`` (csrc/, C ABI in
include/tmg.h); there is no CPU fallback.
"""

from .spacetree import (CellId, EpsilonField, Spacetree, VertexKind, build_regular,  # noqa: F401
                        constant_field, half_domain_jump, needle_inclusion, skew_checkerboard)
from .spacetree3d import Spacetree3, build_regular3  # noqa: F401
from .solvers import CycleStats, GpuEngine, SolverConfig, count_updates  # noqa: F401

__version__ = "0.1.0"
