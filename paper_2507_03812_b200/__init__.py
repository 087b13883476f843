"""B200-native GMGPolar multigrid solve path (sm_100a FP64 kernels behind a C ABI).

The product is ``lib/libpolarmg_b200.so`` (csrc/, C ABI in include/polarmg_b200.h);
this package is its host-side mirror of the reference ``polarmg::MultigridSolver``
API.  There is no CPU fallback.
"""
from .solver import (  # noqa: F401
    LAYOUT_CANONICAL, LAYOUT_NODE, ConvergenceReport, GeometryMap, MultigridSettings,
    MultigridSolver, PmgError, PolarGrid, ProblemCase, grid_hierarchy, load_library,
)
from .configs import baseline_config, section_scales, SEED  # noqa: F401
