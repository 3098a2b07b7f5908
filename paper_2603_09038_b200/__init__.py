"""B200-native partial-assembly operator apply (CEED BP1 / BP3) for high-order
H1 hexahedra, with the Jacobi-PCG solve that calls it and a z-slab
multi-GPU exchange.  Drop-in sibling of the reference package ``feklab``'s
operator API; the compute path is libfk_b200.so (sm_100a CUDA, C-ABI in
include/fk.h).  See DESIGN.md.
"""

from .fem import (
    Basis1D,
    Counters,
    GeometryError,
    Mesh,
    Restriction,
    ShapeError,
    boundary_dofs,
    build_mesh,
    gauss_points,
    gll_points,
    h1_gather_ids,
    h1_node_coords,
    h1_restriction,
)
from . import mapping
from .mixed import MixedOperator, rk4_step
from .mixed import State as MixedState
from .operator import (
    Comm,
    PAData,
    PAOperator,
    bytes_per_apply,
    cg_solve,
    flops_per_element,
    setup_pa_data,
)

__version__ = "0.1.0"

__all__ = [
    "Basis1D", "Comm", "Counters", "GeometryError", "Mesh", "MixedOperator", "MixedState",
    "PAData", "PAOperator", "rk4_step",
    "Restriction", "ShapeError", "boundary_dofs", "build_mesh", "bytes_per_apply",
    "cg_solve", "flops_per_element", "gauss_points", "gll_points", "h1_gather_ids",
    "h1_node_coords", "h1_restriction", "mapping", "setup_pa_data", "__version__",
]
