"""B200-native (sm_100a) hot path of arXiv 1910.01260 behind the reference's API.

Mirrors the public names of the reference package ``strom`` for the north-star
path: streaming incremental SVD, per-mode temporal bases, the spatial and the
block-structured space-time reduced operators and the space-time solve.  Every
numerical step runs in ``_lib/libstrom_b200.so`` (C ABI: include/strom_b200.h).
"""

from .errors import BasisError, CapExceededError, ConvergenceError, SingularMatrixError
from .basis import (BasisSet, SvdState, build_basis_set, ingest_simulation, isvd_init, isvd_update,
                    temporal_snapshots)
from .system import FomResult, LinearDynamicalSystem, TimeGrid, fom_march
from .spatial import SpatialRom, build_spatial_rom
from .spacetime import (SpaceTimeRom, build_st_init, build_st_input, build_st_matrix, build_st_rom,
                        reconstruct_states, solve_st_rom)

__version__ = "0.1.0"

__all__ = [
    "BasisError", "BasisSet", "CapExceededError", "ConvergenceError", "FomResult", "LinearDynamicalSystem",
    "SingularMatrixError", "SpaceTimeRom", "SpatialRom", "SvdState", "TimeGrid", "build_basis_set",
    "build_spatial_rom", "build_st_init", "build_st_input", "build_st_matrix", "build_st_rom", "fom_march",
    "ingest_simulation", "isvd_init", "isvd_update", "reconstruct_states", "solve_st_rom",
    "temporal_snapshots",
]
