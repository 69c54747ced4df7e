"""spechp_b200: B200-native (sm_100a) Collections operators for spechp.

Drop-in GPU path for the reference's Collections hot path
(/root/reference/pkg/src/spechp/collections.py): BwdTrans, IProductWRTBase,
PhysDeriv, IProductWRTDerivBase and the fused matrix-free Helmholtz
operator over batches of quad and hex elements, FP64, with the C0
scatter/assemble of assembly.py.  Python is a thin host layer over the C ABI
in include/spechp_b200.h (libspechp_b200.so, built in-tree).
"""
from . import _lib  # noqa: F401  (fails loudly if the CUDA library is missing)
from .assembly import (AssemblyError, AssemblyMap, GlobalHelmholtz, assemble,
                       hex_variable_codes, hex_variable_maps, scatter)
from .basis import BasisError, BasisKey, BasisType
from .collections import (CONCRETE_STRATEGIES, Collection, CollectionError, CollectionKey,
                          OperatorKind, Strategy, autotune, create_collection, pack, unpack)
from .geometry import (GEOM_AFFINE, GEOM_METRIC, GEOM_NONE, GEOM_POINT, MAP_AFFINE,
                       MAP_HEX_SINE, MAP_QUAD_SINE, ElementBatch, GeometryError, GeomFactors,
                       from_factors, structured_geometry)
from .quadrature import PointsKey, PointsType, QuadratureError, diff_matrix, make_rule
from .solvers import (ConvergenceError, HelmholtzSolver, assembled_diagonal,
                      quad_structured_maps, solve_pcg)
from .stdregions import (ExpansionError, Shape, StdExpansion, make_expansion, make_hex, make_tri,
                         make_quad, make_seg)

__version__ = "0.1.0"
LIBRARY = str(_lib.LIB_PATH)
