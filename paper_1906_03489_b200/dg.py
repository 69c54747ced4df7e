"""DG right-hand sides on the device.

The reference's main production caller of Collections is its DG solver:
`DGSystem` (solvers.py:189-392) stacks per-element operator data and
exposes batched primitives — bwd, iproduct, iproduct_deriv, mass_solve,
trace_minus/plus, lift_interior/boundary — from which
`AdvectionOperator.rhs` (solvers.py:425-457) and `ape_rhs`
(solvers.py:546-642) are composed.  This module mirrors those three on the
device:

* `DGOperators(system)` takes any object with a reference DGSystem's
  precomputed arrays (`exp`, `ww`, `inv`, `minv`, `xy`, `int_li`, `int_ri`,
  `int_exm`, `int_lm`, `int_exp`, `int_lp`, `int_warc`, `int_nrm`,
  `int_xy`, `bnd`, `bcs`) — the reference's own DGSystem, or the committed
  fixtures — uploads them once, and runs every primitive as CUDA kernels:
  the Collections operators through the fused tile kernels, the rest
  through `csrc/dg.cu` (batched mat-vec, trace extraction, a deterministic
  CSR trace lift in np.add.at order, the APE Riemann fluxes with their
  ghost states, the advection upwind flux).
* `ApeOperator` / `AdvectionOperator` compose the right-hand sides with
  the reference's call sequence and sign conventions.

Mesh handling, trace construction and periodic matching stay with the
reference's DGSystem (host setup, out of scope here); expressions (base
flow, boundary values, sources) are host callables evaluated at the stored
world points and uploaded, exactly as the reference samples them.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .collections import Collection, OperatorKind, Strategy
from .geometry import ElementBatch, from_factors
from .stdregions import native_key

__all__ = ["SolverError", "DGOperators", "ApeOperator", "AdvectionOperator"]


class SolverError(ValueError):
    """Mirror of spechp.solvers.SolverError."""


def _dev(a, device, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=device).contiguous()


def _eval(fn, xy, t):
    """Sample an expression at world points the way solvers.sample does."""
    try:
        vals = fn(x=xy[..., 0], y=xy[..., 1], t=t)
    except TypeError:
        vals = fn(xy[..., 0], xy[..., 1])
    return np.asarray(vals, float) * np.ones(xy.shape[:-1])


def _csr(E, groups):
    """CSR of lift codes per element; groups = [(element ids (T,), trace
    offset, plus, neg)] in accumulation order.  Within an element the codes
    keep group order, then trace order: the order np.add.at applies them."""
    ee, cc = [], []
    for ids, off, plus, neg in groups:
        ids = np.asarray(ids, dtype=np.int64)
        t = np.arange(ids.size, dtype=np.int64) + off
        ee.append(ids)
        cc.append((t << 2) | (plus << 1) | neg)
    if not ee:
        return np.zeros(E + 1, np.int64), np.zeros(0, np.int64)
    ee, cc = np.concatenate(ee), np.concatenate(cc)
    order = np.argsort(ee, kind="stable")
    rowp = np.zeros(E + 1, np.int64)
    np.cumsum(np.bincount(ee, minlength=E), out=rowp[1:])
    return rowp, cc[order]


class DGOperators:
    """Device mirror of DGSystem's batched primitives (solvers.py:350-392)."""

    def __init__(self, system, device=None, strategy=Strategy.CUDA_SUMFAC):
        self.device = torch.device(device or "cuda")
        dev = self.device
        self.exp = system.exp
        if native_key(self.exp)[0] != _lib.SHAPE_QUAD:
            raise SolverError("the reference's DG system is 2D: quad expansions only")
        self.ww = _dev(system.ww, dev)
        E, npts = self.ww.shape
        self.num_elements, self.num_points = E, npts
        self.minv = _dev(system.minv, dev)
        self.num_modes = self.minv.shape[1]
        self.xy = np.asarray(system.xy, float)
        self.bcs = dict(getattr(system, "bcs", {}) or {})
        geom = from_factors(self.exp, system.ww, system.inv, kind=_lib.GEOM_POINT, device=dev)
        batch = ElementBatch(self.exp, E, geom, _lib.GEOM_POINT)
        self._geom = geom
        self._bwd = Collection(ElementBatch.standard(self.exp, E), OperatorKind.BWD_TRANS, strategy)
        self._ip = Collection(batch, OperatorKind.IPRODUCT_WRT_BASE, strategy)
        self._ipd = Collection(batch, OperatorKind.IPRODUCT_WRT_DERIV_BASE, strategy)
        li = np.asarray(system.int_li, dtype=np.int64)
        self._nint = li.size
        self.int_li_host = li
        self.int_ri_host = np.asarray(system.int_ri, dtype=np.int64)
        if self._nint:
            self.int_li = _dev(li, dev, torch.int64)
            self.int_ri = _dev(self.int_ri_host, dev, torch.int64)
            for k in ("exm", "lm", "exp", "lp", "warc", "nrm"):
                setattr(self, f"int_{k}", _dev(getattr(system, f"int_{k}"), dev))
            self.int_xy = np.asarray(system.int_xy, float)
            self.num_trace_points = self.int_warc.shape[1]
        self.bnd = {}
        for name, grp in system.bnd.items():
            g = {"li_host": np.asarray(grp["li"], dtype=np.int64),
                 "xy": np.asarray(grp["xy"], float)}
            g["li"] = _dev(g["li_host"], dev, torch.int64)
            for k in ("exm", "lm", "nrm", "warc"):
                g[k] = _dev(grp[k], dev)
            self.bnd[name] = g
            self.num_trace_points = g["warc"].shape[1]
        self._csrs = {}

    # -- Collections primitives -------------------------------------------------
    def bwd(self, coeffs, out=None):
        return self._bwd.apply(coeffs, out)

    def iproduct(self, phys, out=None):
        return self._ip.apply(phys, out)

    def iproduct_deriv(self, fx, fy=None, out=None):
        """b_n = int grad(phi_n) . (fx, fy); or pass one (E, 2, np) block."""
        f = fx if fy is None else torch.stack([fx, fy], dim=1)
        return self._ipd.apply(f.contiguous(), out)

    # -- batched mass solve / traces / lift ------------------------------------
    def mass_solve(self, b, out=None, alpha=1.0, scale=None, accumulate=False):
        """out = alpha * minv (scale * b) (+ out)."""
        b = b.contiguous()
        if out is None:
            out = torch.empty_like(b)
        _lib.check(_lib.lib.sphp_batched_matvec(
            self.num_elements, self.num_modes, self.num_modes, _lib.ptr(self.minv), _lib.ptr(b),
            _lib.ptr(scale), float(alpha), int(accumulate), _lib.ptr(out), _lib.stream_ptr()))
        return out

    def _extract(self, ex, idx, phys, out=None):
        T, nq, npts = ex.shape
        if out is None:
            out = torch.empty((T, nq), dtype=torch.float64, device=self.device)
        _lib.check(_lib.lib.sphp_trace_extract(T, nq, npts, _lib.ptr(ex), _lib.ptr(idx),
                                               _lib.ptr(phys.contiguous()), _lib.ptr(out),
                                               _lib.stream_ptr()))
        return out

    def trace_minus(self, phys, out=None):
        return self._extract(self.int_exm, self.int_li, phys, out)

    def trace_plus(self, phys, out=None):
        return self._extract(self.int_exp, self.int_ri, phys, out)

    def _lift(self, key, groups, Lm, Lp, w, s, b, nrhs=1):
        if key not in self._csrs:
            rowp, codes = _csr(self.num_elements, groups)
            self._csrs[key] = (_dev(rowp, self.device, torch.int64), _dev(codes, self.device, torch.int64))
        rowp, codes = self._csrs[key]
        T, nq = s.shape[-2], s.shape[-1]
        _lib.check(_lib.lib.sphp_trace_lift(nrhs, self.num_elements, self.num_modes, nq, T,
                                            _lib.ptr(rowp), _lib.ptr(codes), _lib.ptr(Lm),
                                            _lib.ptr(Lp), _lib.ptr(w), _lib.ptr(s.contiguous()),
                                            _lib.ptr(b), _lib.stream_ptr()))
        return b

    def lift_interior(self, b, s):
        """b[li] -= lm (warc s); b[ri] += lp (warc s)  (solvers.py:374-381)."""
        groups = [(self.int_li_host, 0, 0, 1), (self.int_ri_host, 0, 1, 0)]
        return self._lift("interior", groups, self.int_lm, self.int_lp, self.int_warc, s, b)

    def lift_boundary(self, b, name, s):
        """b[li] -= lm (warc s) for one boundary region (solvers.py:383-387)."""
        g = self.bnd[name]
        return self._lift(("bnd", name), [(g["li_host"], 0, 0, 1)], g["lm"], g["lm"], g["warc"], s, b)

    def trace_extract_boundary(self, name, phys, out=None):
        g = self.bnd[name]
        return self._extract(g["exm"], g["li"], phys, out)

    @property
    def num_interior(self):
        return self._nint


class ApeOperator:
    """ape_rhs (solvers.py:546-642) on the device.  `base`, `base_trace`,
    `base_bnd` are the sampled base-flow dicts of make_ape_state
    (solvers.py:461-495); `bcs` the system's boundary specs; `sources` maps
    'p'/'ux'/'uy' to expressions."""

    def __init__(self, dg: DGOperators, base, base_trace=None, base_bnd=None, bcs=None,
                 riemann="upwind", sources=None, c2_per_element=None):
        if riemann not in _lib.RIEMANN:
            raise SolverError(f"unknown Riemann flux kind {riemann!r}")
        self.dg = dg
        dev = dg.device
        E, npts = dg.num_elements, dg.num_points
        self.riemann = riemann
        self.bcs = dict(bcs if bcs is not None else dg.bcs)
        self.sources = dict(sources or {})
        keys = ("ux", "uy", "rho", "c2")
        self.base = _dev(np.stack([np.asarray(base[k], float).reshape(E, npts) for k in keys]), dev)
        self.neg_c2 = (-self.base[3]).contiguous()
        self.c2e = None if c2_per_element is None else _dev(-np.asarray(c2_per_element, float), dev)
        nq = dg.num_trace_points if (dg.num_interior or dg.bnd) else 0
        self.groups = []          # (name, bc code, offset, T)
        off = dg.num_interior
        Lm, Lp = [], []
        if dg.num_interior:
            self.base_tr = _dev(np.stack([np.asarray(base_trace[k], float).reshape(-1) for k in keys]), dev)
            Lm.append(dg.int_lm)
            Lp.append(dg.int_lp)
        for name, g in dg.bnd.items():
            spec = self.bcs.get(name)
            if spec is None:
                raise SolverError(f"no boundary condition for region {name!r}")
            kind = spec.get("type")
            code = {"rigid_wall": _lib.BC_RIGID_WALL, "farfield": _lib.BC_FARFIELD,
                    "dirichlet": _lib.BC_DIRICHLET}.get(kind)
            if code is None:
                raise SolverError(f"bc type {kind!r} unsupported for the acoustic system")
            T = g["warc"].shape[0]
            bb = _dev(np.stack([np.asarray(base_bnd[name][k], float).reshape(-1) for k in keys]), dev)
            self.groups.append((name, code, off, T, bb))
            Lm.append(g["lm"])
            Lp.append(g["lm"])
            off += T
        self.T_all, self.nq = off, nq
        if off:
            self.Lm = torch.cat(Lm).contiguous()
            self.Lp = torch.cat(Lp).contiguous()
            self.S = torch.empty((3, off, nq), dtype=torch.float64, device=dev)
            # accumulation order of ape_rhs: interior li (+lm), interior ri
            # (-lp), then each boundary region's li (+lm) in dict order
            csr_groups = []
            if dg.num_interior:
                csr_groups += [(dg.int_li_host, 0, 0, 0), (dg.int_ri_host, 0, 1, 1)]
            for name, code, o, T, bb in self.groups:
                csr_groups.append((dg.bnd[name]["li_host"], o, 0, 0))
            rowp, codes = _csr(E, csr_groups)
            self.rowp, self.codes = _dev(rowp, dev, torch.int64), _dev(codes, dev, torch.int64)

    @classmethod
    def from_state(cls, state, dg=None, device=None):
        """From a reference ApeState (solvers.py:461-478)."""
        dg = dg or DGOperators(state.system, device=device)
        return cls(dg, state.base, state.base_trace, state.base_bnd, state.system.bcs,
                   state.riemann, state.sources,
                   state.c2_per_element if state.c2_elementwise_constant else None)

    def rhs(self, coeffs, t=0.0):
        """Time derivative of the (3, E, nm) coefficients at time t."""
        dg = self.dg
        dev = dg.device
        E, npts, nm = dg.num_elements, dg.num_points, dg.num_modes
        coeffs = torch.as_tensor(coeffs, dtype=torch.float64, device=dev).contiguous()
        q = torch.empty((3, E, npts), dtype=torch.float64, device=dev)
        for i in range(3):
            dg.bwd(coeffs[i], out=q[i])
        G = torch.empty((E, 2, npts), dtype=torch.float64, device=dev)
        HX, HY = torch.empty_like(G), torch.empty_like(G)
        _lib.check(_lib.lib.sphp_ape_volume(E, npts, _lib.ptr(q), _lib.ptr(self.base), _lib.ptr(G),
                                            _lib.ptr(HX), _lib.ptr(HY), _lib.stream_ptr()))
        b = torch.empty((3, E, nm), dtype=torch.float64, device=dev)
        dg.iproduct_deriv(G, out=b[0])
        dg.iproduct_deriv(HX, out=b[1])
        dg.iproduct_deriv(HY, out=b[2])
        riem = _lib.RIEMANN[self.riemann]
        if self.T_all:
            nq, ostride = self.nq, self.T_all * self.nq
            if dg.num_interior:
                Ti = dg.num_interior
                qm = torch.empty((3, Ti, nq), dtype=torch.float64, device=dev)
                qp = torch.empty_like(qm)
                for i in range(3):
                    dg.trace_minus(q[i], out=qm[i])
                    dg.trace_plus(q[i], out=qp[i])
                _lib.check(_lib.lib.sphp_ape_trace_flux(
                    Ti * nq, riem, _lib.BC_INTERIOR, _lib.ptr(qm), _lib.ptr(qp), None,
                    _lib.ptr(dg.int_nrm), _lib.ptr(self.base_tr), _lib.ptr(dg.int_warc),
                    _lib.ptr(self.S), ostride, _lib.stream_ptr()))
            for name, code, off, T, bb in self.groups:
                g = dg.bnd[name]
                qm = torch.empty((3, T, nq), dtype=torch.float64, device=dev)
                for i in range(3):
                    dg._extract(g["exm"], g["li"], q[i], out=qm[i])
                gv = None
                if code == _lib.BC_DIRICHLET:
                    gv = _dev(_eval(self.bcs[name]["value"], g["xy"], t), dev)
                _lib.check(_lib.lib.sphp_ape_trace_flux(
                    T * nq, riem, code, _lib.ptr(qm), None, _lib.ptr(gv), _lib.ptr(g["nrm"]),
                    _lib.ptr(bb), _lib.ptr(g["warc"]), _lib.ptr(self.S[0, off]), ostride,
                    _lib.stream_ptr()))
            _lib.check(_lib.lib.sphp_trace_lift(3, E, nm, nq, self.T_all, _lib.ptr(self.rowp),
                                                _lib.ptr(self.codes), _lib.ptr(self.Lm),
                                                _lib.ptr(self.Lp), None, _lib.ptr(self.S),
                                                _lib.ptr(b), _lib.stream_ptr()))
        rhs = torch.empty((3, E, nm), dtype=torch.float64, device=dev)

        def src(var):
            fn = self.sources.get(var)
            return None if fn is None else _dev(_eval(fn, dg.xy, t), dev)

        sp = src("p")
        if self.c2e is not None:
            # element-constant c2 pulled through the mass solve (solvers.py:612-618)
            dg.mass_solve(b[0], out=rhs[0], scale=self.c2e)
            if sp is not None:
                dg.mass_solve(dg.iproduct(sp), out=rhs[0], accumulate=True)
        else:
            div_g = dg.bwd(dg.mass_solve(b[0]))
            rp = torch.empty_like(div_g)
            _lib.check(_lib.lib.sphp_scale_points(E * npts, _lib.ptr(self.neg_c2), _lib.ptr(div_g),
                                                  _lib.ptr(sp), _lib.ptr(rp), _lib.stream_ptr()))
            dg.mass_solve(dg.iproduct(rp), out=rhs[0])
        for i, var in ((1, "ux"), (2, "uy")):
            dg.mass_solve(b[i], out=rhs[i], alpha=-1.0)
            sv = src(var)
            if sv is not None:
                dg.mass_solve(dg.iproduct(sv), out=rhs[i], accumulate=True)
        return rhs


class AdvectionOperator:
    """AdvectionOperator.rhs (solvers.py:400-457) on the device:
    du/dt = -div(a u) with upwind trace fluxes."""

    def __init__(self, dg: DGOperators, velocity, bcs=None):
        self.dg = dg
        dev = dg.device
        self.bcs = dict(bcs if bcs is not None else dg.bcs)
        ax, ay = velocity
        self.ax = _dev(_eval(ax, dg.xy, 0.0), dev)
        self.ay = _dev(_eval(ay, dg.xy, 0.0), dev)
        if dg.num_interior:
            txy = dg.int_xy
            nrm = dg.int_nrm.cpu().numpy()
            an = _eval(ax, txy, 0.0) * nrm[..., 0] + _eval(ay, txy, 0.0) * nrm[..., 1]
            self.an_int = _dev(an, dev)
        self.an_bnd = {}
        for name, g in dg.bnd.items():
            nrm = g["nrm"].cpu().numpy()
            an = _eval(ax, g["xy"], 0.0) * nrm[..., 0] + _eval(ay, g["xy"], 0.0) * nrm[..., 1]
            self.an_bnd[name] = _dev(an, dev)

    def rhs(self, coeffs, t=0.0):
        dg = self.dg
        dev = dg.device
        E, npts = dg.num_elements, dg.num_points
        coeffs = torch.as_tensor(coeffs, dtype=torch.float64, device=dev).contiguous()
        u = dg.bwd(coeffs)
        F = torch.empty((E, 2, npts), dtype=torch.float64, device=dev)
        _lib.check(_lib.lib.sphp_advect_volume(E, npts, _lib.ptr(self.ax), _lib.ptr(self.ay),
                                               _lib.ptr(u), _lib.ptr(F), _lib.stream_ptr()))
        b = dg.iproduct_deriv(F)
        if dg.num_interior:
            um, up = dg.trace_minus(u), dg.trace_plus(u)
            flux = torch.empty_like(um)
            _lib.check(_lib.lib.sphp_advect_trace_flux(um.numel(), _lib.BC_INTERIOR,
                                                       _lib.ptr(self.an_int), _lib.ptr(um),
                                                       _lib.ptr(up), None, _lib.ptr(flux),
                                                       _lib.stream_ptr()))
            dg.lift_interior(b, flux)
        for name, g in dg.bnd.items():
            spec = self.bcs.get(name)
            if spec is None:
                raise SolverError(f"no boundary condition for region {name!r}")
            kind = spec["type"]
            if kind not in ("dirichlet", "farfield"):
                raise SolverError(f"bc type {kind!r} unsupported for advection")
            um = dg.trace_extract_boundary(name, u)
            gv = _dev(_eval(spec["value"], g["xy"], t), dev) if kind == "dirichlet" else None
            flux = torch.empty_like(um)
            code = _lib.BC_DIRICHLET if kind == "dirichlet" else _lib.BC_FARFIELD
            _lib.check(_lib.lib.sphp_advect_trace_flux(um.numel(), code, _lib.ptr(self.an_bnd[name]),
                                                       _lib.ptr(um), None, _lib.ptr(gv),
                                                       _lib.ptr(flux), _lib.stream_ptr()))
            dg.lift_boundary(b, name, flux)
        return dg.mass_solve(b)
