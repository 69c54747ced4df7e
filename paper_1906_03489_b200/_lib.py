"""ctypes binding of libspechp_b200.so (the C ABI in include/spechp_b200.h).

The shared library is built in-tree (``make -C paper_1906_03489_b200/csrc``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing the package raises — the product path is the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libspechp_b200.so"
# tuning experiments may point at an alternative in-tree build
if os.environ.get("SPHP_LIBRARY_VARIANT", ""):
    LIB_PATH = _HERE.parent / "build" / "variants" / os.environ["SPHP_LIBRARY_VARIANT"] / "libspechp_b200.so"

# error codes (include/spechp_b200.h)
OK = 0
ERR_BAD_SHAPE = -1
ERR_BAD_ARG = -2
ERR_UNSUPPORTED = -3
ERR_CUDA = -4
ERR_ALLOC = -5

SHAPE_SEG, SHAPE_QUAD, SHAPE_TRI, SHAPE_HEX = 0, 1, 2, 3
POINTS = {"gauss_legendre": 0, "gauss_lobatto_legendre": 1, "gauss_radau_m_legendre": 2}
BASIS = {"modified_a": 0, "modified_b": 1, "lagrange_gll": 2}
OP_BWD_TRANS, OP_IPRODUCT_WRT_BASE, OP_PHYS_DERIV, OP_IPRODUCT_WRT_DERIV_BASE, OP_HELMHOLTZ = range(5)
STRATEGY_CUDA_SUMFAC, STRATEGY_CUDA_STDMAT = 0, 1
GEOM_NONE, GEOM_AFFINE, GEOM_POINT, GEOM_METRIC = 0, 1, 2, 3
MAP_AFFINE, MAP_QUAD_SINE, MAP_HEX_SINE = 0, 1, 2
ASSEMBLY_OWNER, ASSEMBLY_COLOUR, ASSEMBLY_SPLIT, ASSEMBLY_CLASS = 0, 1, 2, 3
RESERVE_DEVICE, RESERVE_HOST = 1, 2
RIEMANN = {"upwind": 0, "laxfriedrichs": 1}
BC_INTERIOR, BC_RIGID_WALL, BC_FARFIELD, BC_DIRICHLET = 0, 1, 2, 3


class LibraryError(RuntimeError):
    """A C-ABI call failed; `code` is the SPHP_ERR_* value."""

    def __init__(self, code, message):
        super().__init__(message)
        self.code = code


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (the spechp_b200 product path has no CPU fallback)")
    return C.CDLL(str(LIB_PATH))


lib = _load()

_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_d = C.c_double
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)
_pp = C.POINTER(C.c_void_p)

_SIGS = {
    "sphp_abi_version": (_i, []),
    "sphp_last_error": (C.c_char_p, []),
    "sphp_device_sm_count": (_i, []),
    "sphp_hex_helmholtz_plan": (_i, [_i, _i]),
    "sphp_tables_create": (_i, [_i, _ip, _ip, _ip, _ip, _pp]),
    "sphp_tables_destroy": (_i, [_p]),
    "sphp_tables_query": (_i, [_p, _i, _p, _p, _p, _p, _p]),
    "sphp_tables_sizes": (_i, [_p, _i64p, _i64p, _ip]),
    "sphp_geom_stride": (_i64, [_p, _i]),
    "sphp_geom_analytic": (_i, [_p, _i, _i, _i, _dp, _d, _i64, _i64, _p, _p, _p]),
    "sphp_geom_from_factors": (_i, [_p, _i, _i64, _p, _p, _p, _p]),
    "sphp_collection_create": (_i, [_p, _i, _i, _i64, _i, _p, _d, _pp]),
    "sphp_collection_destroy": (_i, [_p]),
    "sphp_collection_set_lambda": (_i, [_p, _d]),
    "sphp_collection_info": (_i, [_p, _i64p, _i64p, _i64p, _i64p]),
    "sphp_apply": (_i, [_p, _i64, _i64, _p, _p, _p]),
    "sphp_apply_host": (_i, [_p, _i64, _i64, _p, _p, _p]),
    "sphp_amap_create_explicit": (_i, [_i64, _i, _p, _i64, _pp]),
    "sphp_amap_create_hex_periodic": (_i, [_i, _i, _pp]),
    "sphp_hexmap_variable": (_i, [_i, _p, _i64p, _p, _p]),
    "sphp_amap_destroy": (_i, [_p]),
    "sphp_amap_set_algorithm": (_i, [_p, _i]),
    "sphp_amap_algorithm": (_i, [_p, _p]),
    "sphp_amap_info": (_i, [_p, _i64p, _ip, _i64p, _ip]),
    "sphp_amap_codes": (_i, [_p, _p]),
    "sphp_hexmap_periodic_codes": (_i, [_i, _i, _i64, _i64, _p]),
    "sphp_index_gather": (_i, [_i64, _p, _p, _p, _p]),
    "sphp_index_sum2": (_i, [_i64, _p, _p, _p, _p, _p]),
    "sphp_scatter": (_i, [_p, _p, _p, _p]),
    "sphp_assemble": (_i, [_p, _p, _p, _p]),
    "sphp_helmholtz_assembled": (_i, [_p, _p, _p, _p, _i, _p]),
    "sphp_helmholtz_assembled_host": (_i, [_p, _p, _p, _p, _p]),
    "sphp_helmholtz_assembled_phases": (_i, [_p, _p, _p, _p, _p, _i, _p, _p]),
    "sphp_collection_reserve": (_i, [_p, _p, _i, _p]),
    "sphp_gsys_reserve": (_i, [_p, _p]),
    "sphp_gsys_create": (_i, [_pp, _pp, _i, _i64, _pp]),
    "sphp_gsys_apply": (_i, [_p, _p, _p, _p]),
    "sphp_gsys_destroy": (_i, [_p]),
    "sphp_helmholtz_diagonal": (_i, [_p, _p, _p]),
    "sphp_reduction_workspace": (_i64, []),
    "sphp_vec_dot2": (_i, [_i64, _p, _p, _p, _p, _p, _p]),
    "sphp_cg_init": (_i, [_i64, _p, _p, _p, _p, _p, _p, _p, _p]),
    "sphp_cg_update": (_i, [_i64, _d, _p, _p, _p, _p, _p, _p, _p, _p]),
    "sphp_cg_direction": (_i, [_i64, _d, _p, _p, _p]),
    "sphp_cg_state_size": (_i64, [_i]),
    "sphp_cg_init_dev": (_i, [_i64, _p, _p, _p, _p, _p, _p, _p, _i, _d, _p]),
    "sphp_cg_step_dev": (_i, [_i64, _p, _p, _p, _p, _p, _p, _p, _i, _p]),
    "sphp_quadmap_structured": (_i, [_i, _i, _p, _i, _i64p, _i64p, _p, _p]),
    "sphp_geom_from_jacobian": (_i, [_p, _i, _i64, _p, _p, _p, _i64p, _p]),
    "sphp_batched_matvec": (_i, [_i64, _i, _i, _p, _p, _p, _d, _i, _p, _p]),
    "sphp_trace_extract": (_i, [_i64, _i, _i, _p, _p, _p, _p, _p]),
    "sphp_trace_lift": (_i, [_i, _i64, _i, _i, _i64, _p, _p, _p, _p, _p, _p, _p, _p]),
    "sphp_ape_trace_flux": (_i, [_i64, _i, _i, _p, _p, _p, _p, _p, _p, _p, _i64, _p]),
    "sphp_ape_volume": (_i, [_i64, _i, _p, _p, _p, _p, _p, _p]),
    "sphp_advect_volume": (_i, [_i64, _i, _p, _p, _p, _p, _p]),
    "sphp_advect_trace_flux": (_i, [_i64, _i, _p, _p, _p, _p, _p, _p]),
    "sphp_scale_points": (_i, [_i64, _p, _p, _p, _p, _p]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


def last_error() -> str:
    msg = lib.sphp_last_error()
    return msg.decode() if msg else ""


def check(rc, exc=None):
    """Raise on a negative return code; `exc` overrides the exception type
    (e.g. CollectionError for shape errors, mirroring collections.py)."""
    if rc == OK:
        return
    msg = last_error()
    if exc is not None:
        raise exc(msg)
    raise LibraryError(rc, msg)


def ptr(t):
    """Raw address of a torch tensor / numpy array / None."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t.ctypes.data)


def stream_ptr(stream=None):
    """cudaStream_t of a torch stream (current stream when None)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def raw_stream(stream, device_index):
    """cudaStream_t as an int: the given torch stream's, or the current
    stream of `device_index` (the per-call fast path: no Stream object)."""
    if stream is not None:
        return stream.cuda_stream
    import torch

    return torch._C._cuda_getCurrentRawStream(device_index)


def abi_version():
    return lib.sphp_abi_version()


os.environ.setdefault("SPHP_LIB", str(LIB_PATH))
