"""GPU Collections: batched elemental operators over homogeneous element
groups (drop-in for spechp.collections, collections.py:1-323).

Same surface as the reference — `OperatorKind`, `Strategy`,
`CollectionError`, `CollectionKey`, `Collection(elements, operator,
strategy)`, `.apply(block, out=None)`, `.input_size`, `.output_shape`,
`.mac_count()`, `create_collection`, `autotune`, `pack`, `unpack` — with:

* GPU strategies `CUDA_SUMFAC` (fused sum-factorisation kernels, K1-K4) and
  `CUDA_STDMAT` (dense elemental operators, FP64 GEMM, K6).  The reference's
  CPU strategy names stay in the enum so configs parse; a Collection only
  accepts the GPU ones (the CPU path is the reference itself).
* `Shape.HEX` expansions and two more operator kinds: `IPRODUCT_WRT_DERIV_BASE`
  (geometry.py:163-168 batched, solvers.py:361-365) and `HELMHOLTZ` (the
  fused mass + lambda-Laplacian operator, geometry.py:171-184).
* elements may be the reference's own objects (StdExpansion, or anything with
  `.exp`/`.gf`, collections.py:54-73) or a device-resident `ElementBatch`.

Blocks: a torch CUDA float64 tensor is used in place (zero-copy, result on
the device); anything else is converted with `np.asarray(block, float)`
(collections.py:196) and the result comes back as a numpy array.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from .geometry import (GEOM_AFFINE, GEOM_METRIC, GEOM_NONE, GEOM_POINT, ElementBatch,
                       from_factors)
from .stdregions import native_key, native_tables


class OperatorKind(Enum):
    BWD_TRANS = "bwdtrans"
    IPRODUCT_WRT_BASE = "iproductwrtbase"
    PHYS_DERIV = "physderiv"
    IPRODUCT_WRT_DERIV_BASE = "iproductwrtderivbase"
    HELMHOLTZ = "helmholtz"


class Strategy(Enum):
    STD_MAT = "stdmat"
    ITER_PER_EXP = "iterperexp"
    SUM_FAC = "sumfac"
    AUTO = "auto"
    CUDA_SUMFAC = "cuda_sumfac"
    CUDA_STDMAT = "cuda_stdmat"


CONCRETE_STRATEGIES = (Strategy.CUDA_SUMFAC, Strategy.CUDA_STDMAT)
_CPU_STRATEGIES = (Strategy.STD_MAT, Strategy.ITER_PER_EXP, Strategy.SUM_FAC)

_OP_CODE = {
    OperatorKind.BWD_TRANS: _lib.OP_BWD_TRANS,
    OperatorKind.IPRODUCT_WRT_BASE: _lib.OP_IPRODUCT_WRT_BASE,
    OperatorKind.PHYS_DERIV: _lib.OP_PHYS_DERIV,
    OperatorKind.IPRODUCT_WRT_DERIV_BASE: _lib.OP_IPRODUCT_WRT_DERIV_BASE,
    OperatorKind.HELMHOLTZ: _lib.OP_HELMHOLTZ,
}
_STRAT_CODE = {Strategy.CUDA_SUMFAC: _lib.STRATEGY_CUDA_SUMFAC,
               Strategy.CUDA_STDMAT: _lib.STRATEGY_CUDA_STDMAT}


class CollectionError(ValueError):
    pass


@dataclass(frozen=True)
class CollectionKey:
    shape: object
    basis_keys: tuple
    operator: OperatorKind
    num_elements: int


def _normalise(elements):
    """collections.py:54-73 plus ElementBatch: returns (exp, geoms | batch)."""
    if isinstance(elements, ElementBatch):
        return elements.exp, elements
    exps, geoms = [], []
    for e in elements:
        if hasattr(e, "exp") and hasattr(e, "gf"):
            exps.append(e.exp)
            geoms.append(e.gf)
        else:
            exps.append(e)
            geoms.append(None)
    if not exps:
        raise CollectionError("empty element group")
    ref = exps[0]
    ref_key = native_key(ref)
    for e in exps[1:]:
        if e is not ref and native_key(e) != ref_key:
            raise CollectionError(
                "heterogeneous group: all elements must share shape and basis")
    if any(g is None for g in geoms) and any(g is not None for g in geoms):
        raise CollectionError("mix of standard and physical elements")
    return ref, (None if geoms[0] is None else geoms)


_APPLY = _lib.lib.sphp_apply


def _is_cuda_tensor(x):
    return torch.is_tensor(x) and x.is_cuda


class Collection:
    """One operator over one homogeneous element group under one GPU strategy."""

    def __init__(self, elements, operator: OperatorKind, strategy: Strategy, lam: float = 1.0):
        if strategy in _CPU_STRATEGIES:
            raise CollectionError(
                f"strategy {strategy.value!r} is the reference CPU path; "
                "spechp_b200 collections take cuda_sumfac or cuda_stdmat")
        if strategy not in CONCRETE_STRATEGIES:
            raise CollectionError(f"strategy must be concrete, got {strategy}")
        exp, geoms = _normalise(elements)
        self.exp = exp
        self.operator = operator
        self.strategy = strategy
        self.lam = float(lam)
        self._tables = native_tables(exp)
        self.dim = self._tables.dim
        if isinstance(geoms, ElementBatch):
            self.num_elements = geoms.num_elements
            self._geom = geoms.geometry
            kind = geoms.geom_kind
            if operator is OperatorKind.HELMHOLTZ and kind == GEOM_POINT:
                raise CollectionError("Helmholtz batches need METRIC or AFFINE geometry")
            if operator is not OperatorKind.HELMHOLTZ and kind == GEOM_METRIC:
                raise CollectionError("METRIC geometry only feeds the Helmholtz operator")
        else:
            self.num_elements = len(elements)
            if geoms is None:
                self._geom, kind = None, GEOM_NONE
                if operator is OperatorKind.HELMHOLTZ:
                    # standard elements: identity map -> wJ = w, G = w I
                    E, npts, d = self.num_elements, int(np.prod(exp_points(exp))), self.dim
                    inv = np.broadcast_to(np.eye(d), (E, npts, d, d))
                    wts = np.broadcast_to(std_weights(exp), (E, npts))
                    self._geom = from_factors(exp, wts, inv, GEOM_METRIC)
                    kind = GEOM_METRIC
            else:
                wts = np.stack([g.weights_world for g in geoms])
                inv = np.stack([g.inv for g in geoms])
                kind = GEOM_METRIC if operator is OperatorKind.HELMHOLTZ else GEOM_POINT
                self._geom = None if operator is OperatorKind.BWD_TRANS else \
                    from_factors(exp, wts, inv, kind)
                if operator is OperatorKind.BWD_TRANS:
                    kind = GEOM_NONE
        self.geom_kind = kind
        self.geoms = None if kind == GEOM_NONE else self._geom
        self.key = CollectionKey(exp.shape, tuple(exp.basis_keys), operator, self.num_elements)
        self._handle = C.c_void_p()
        rc = _lib.lib.sphp_collection_create(
            self._tables.handle, _OP_CODE[operator], _STRAT_CODE[strategy], self.num_elements,
            kind, _lib.ptr(self._geom), self.lam, C.byref(self._handle))
        if rc == _lib.ERR_UNSUPPORTED:
            raise CollectionError(_lib.last_error())
        _lib.check(rc, CollectionError)
        ins, outs, macs, hbm = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(_lib.lib.sphp_collection_info(self._handle, C.byref(ins), C.byref(outs),
                                                 C.byref(macs), C.byref(hbm)))
        self._in, self._out, self._macs, self._hbm = ins.value, outs.value, macs.value, hbm.value
        self._h = self._handle.value
        self._in_shape = torch.Size((self.num_elements, self._in))
        self._out_numel = self.num_elements * self._out

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h and _lib is not None and _lib.lib is not None:
            _lib.lib.sphp_collection_destroy(h)
            self._handle = None

    # -- shapes (collections.py:94-108) ----------------------------------------
    @property
    def input_size(self):
        return self._in

    @property
    def output_shape(self):
        if self.operator is OperatorKind.PHYS_DERIV:
            return (self.num_elements, self.dim, self._out // self.dim)
        return (self.num_elements, self._out)

    def set_lambda(self, lam):
        self.lam = float(lam)
        _lib.check(_lib.lib.sphp_collection_set_lambda(self._handle, self.lam))

    # -- apply (collections.py:189-246) ------------------------------------------
    def _shape_error(self, shape):
        return CollectionError(
            f"block shape {tuple(shape)} does not match ({self.num_elements}, {self.input_size})")

    def _as_2d(self, block):
        shape = tuple(block.shape)
        if self.operator is OperatorKind.IPRODUCT_WRT_DERIV_BASE and len(shape) == 3:
            if shape[0] * shape[1] * shape[2] == self.num_elements * self.input_size and \
                    shape[0] == self.num_elements:
                return block.reshape(self.num_elements, self.input_size)
        if shape != (self.num_elements, self.input_size):
            raise self._shape_error(shape)
        return block

    def apply(self, block, out=None, stream=None):
        """Evaluate the operator over the packed block."""
        # fast path (device float64 contiguous blocks of the exact shape, the
        # repeated-apply case): one ctypes call, raw ints, no Stream object
        if type(block) is torch.Tensor and block.is_cuda and block.dtype is torch.float64 \
                and block.shape == self._in_shape and block.is_contiguous():
            if out is None:
                out = torch.empty(self.output_shape, dtype=torch.float64, device=block.device)
            elif not (type(out) is torch.Tensor and out.is_cuda and out.dtype is torch.float64
                      and out.is_contiguous() and out.numel() == self._out_numel):
                raise CollectionError("out must be a contiguous float64 CUDA tensor of output_shape")
            rc = _APPLY(self._h, self.num_elements, self._in, block.data_ptr(), out.data_ptr(),
                        _lib.raw_stream(stream, block.device.index))
            if rc:
                _lib.check(rc, CollectionError)
            return out
        if _is_cuda_tensor(block):
            if block.dtype != torch.float64:
                block = block.to(torch.float64)
            block = self._as_2d(block).contiguous()
            if out is None:
                out = torch.empty(self.output_shape, dtype=torch.float64, device=block.device)
            elif not (_is_cuda_tensor(out) and out.dtype == torch.float64 and out.is_contiguous()
                      and out.numel() == self.num_elements * self._out):
                raise CollectionError("out must be a contiguous float64 CUDA tensor of output_shape")
            rc = _lib.lib.sphp_apply(self._handle, block.shape[0], block.shape[1],
                                     _lib.ptr(block), _lib.ptr(out), _lib.stream_ptr(stream))
            _lib.check(rc, CollectionError)
            return out
        arr = np.asarray(block, dtype=float)
        arr = np.ascontiguousarray(self._as_2d(arr))
        res = np.empty(self.output_shape)
        rc = _lib.lib.sphp_apply_host(self._handle, arr.shape[0], arr.shape[1], _lib.ptr(arr),
                                      _lib.ptr(res), _lib.stream_ptr(stream))
        _lib.check(rc, CollectionError)
        if out is not None:
            out[...] = res
            return out
        return res

    __call__ = apply

    def reserve(self, stream=None, host=False):
        """Size the per-stream workspace of applies on `stream` (StdMat
        scratch; host staging with host=True) ahead of the first apply, e.g.
        before capturing applies into a CUDA graph."""
        flags = _lib.RESERVE_DEVICE | (_lib.RESERVE_HOST if host else 0)
        _lib.check(_lib.lib.sphp_collection_reserve(self._handle, None, flags, _lib.stream_ptr(stream)),
                   CollectionError)
        return self

    # -- cost model (collections.py:250-273 generalised) ------------------------
    def mac_count(self):
        return self._macs

    def hbm_bytes(self):
        """Algorithmic HBM bytes of one apply (inputs, outputs, geometry)."""
        return self._hbm


def exp_points(exp):
    return tuple(k.points_key.num_points for k in exp.basis_keys)


def std_weights(exp):
    if hasattr(exp, "weights"):
        return np.asarray(exp.weights, float)
    raise CollectionError("expansion exposes no quadrature weights")


def create_collection(elements, operator, strategy=Strategy.AUTO, trials=5, warmups=2, lam=1.0):
    """Build a collection; AUTO autotunes at creation time (collections.py:276-282)."""
    if strategy is Strategy.AUTO:
        strategy, _ = autotune(elements, operator, trials=trials, warmups=warmups, lam=lam)
    return Collection(elements, operator, strategy, lam=lam)


def hbm_peak_gbs():
    """(GB/s, kind) of the HBM roofline the reports are quoted against:
    SPHP_HBM_PEAK_GBS, else the driver-measured copy bandwidth in
    MEASURED_PEAKS.json at the repository root, else the B200 nominal 8 TB/s."""
    import json
    import os
    from pathlib import Path
    env = os.environ.get("SPHP_HBM_PEAK_GBS")
    if env:
        return float(env), "env"
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    except (OSError, ValueError, KeyError):
        return 8000.0, "nominal"


def autotune(elements, operator, trials=5, warmups=2, candidates=None, lam=1.0):
    """Time each GPU strategy on this group and pick the fastest median
    (collections.py:285-313).  Times are CUDA-event device times of one
    apply on a resident `standard_normal` block from `default_rng(0)`.
    The report keeps the reference's shape (`median_s`, `times_s`,
    `mac_count` per strategy, collections.py:308-311) extended with
    `hbm_bytes`, `dof_per_s` (elements x modes per second), `hbm_gbs_achieved`
    (algorithmic bytes / median) and `roofline_frac` (of `hbm_peak_gbs()`).
    Candidates that cannot run this key are reported with an "error" entry.
    Synchronises the device; must not run concurrently with other timed work.
    """
    if trials < 1:
        raise CollectionError("trials must be >= 1")
    candidates = tuple(candidates or CONCRETE_STRATEGIES)
    report = {}
    rng = np.random.default_rng(0)
    best, best_time = None, np.inf
    peak = hbm_peak_gbs()[0]
    for strat in candidates:
        try:
            coll = Collection(elements, operator, strat, lam=lam)
        except CollectionError as exc:
            report[strat.value] = {"error": str(exc)}
            continue
        block = torch.as_tensor(rng.standard_normal((coll.num_elements, coll.input_size)),
                                device="cuda")
        outb = torch.empty(coll.output_shape, dtype=torch.float64, device="cuda")
        try:
            for _ in range(warmups):
                coll.apply(block, outb)
            torch.cuda.synchronize()
            times = []
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * trials)]
            for t in range(trials):
                ev[2 * t].record()
                coll.apply(block, outb)
                ev[2 * t + 1].record()
            torch.cuda.synchronize()
        except (CollectionError, _lib.LibraryError) as exc:
            report[strat.value] = {"error": str(exc)}
            continue
        times = [ev[2 * t].elapsed_time(ev[2 * t + 1]) * 1e-3 for t in range(trials)]
        med = float(np.median(times))
        gbs = coll.hbm_bytes() / med / 1e9
        report[strat.value] = {"median_s": med, "times_s": times, "mac_count": coll.mac_count(),
                               "hbm_bytes": coll.hbm_bytes(),
                               "dof_per_s": coll.num_elements * coll._tables.num_modes / med,
                               "hbm_gbs_achieved": gbs, "roofline_frac": gbs / peak}
        if med < best_time:
            best, best_time = strat, med
    if best is None:
        raise CollectionError("no GPU strategy can run this collection: "
                              + "; ".join(f"{k}: {v.get('error')}" for k, v in report.items()))
    return best, report


def pack(vectors):
    """Stack per-element vectors into the packed block layout (collections.py:316-319)."""
    return np.ascontiguousarray(np.stack([np.asarray(v, float) for v in vectors]))


def unpack(block):
    if torch.is_tensor(block):
        block = block.detach().cpu().numpy()
    return [np.array(row) for row in np.asarray(block)]
