"""C0 assembly on the device (drop-in for assembly.py:44-215).

`AssemblyMap` wraps an `sphp_amap` handle:
  * `AssemblyMap.explicit(codes, num_global)` / `.from_reference(amap)` take
    the reference's local_to_global + signs (assembly.py:44-56) — bit-exact
    by construction, encoded as gid / -1 (pinned) / -(gid+2) (sign -1);
  * `AssemblyMap.hex_periodic(n, P)` is the periodic structured hex map of
    cfg4 with indices computed on the fly on the device (no map traffic);
  * `hex_variable_maps(n, orders)` builds the variable-order map of cfg5
    (edge order = min over the 4 sharing elements, face order = min over 2,
    excess modes pinned) and splits it into per-order batches.

`scatter` / `assemble` mirror assembly.py:141-160; `GlobalHelmholtz.apply`
is `GlobalSystem.apply` (assembly.py:177-182).  Deterministic, atomic-free
assembly algorithms (`AssemblyMap.set_algorithm`):
  "owner"  (default on explicit maps) one kernel gathers x, applies the
           fused elemental operator and writes the local block; a second
           sums every global dof from its contributions in a fixed order;
  "class"  (default on periodic hex maps, every order) the fused operator
           gathers x by entity-class ranges (16-byte cp.async chunks) and
           writes a tile-major class block (interiors straight into y); one
           streaming owner-computes sum reduces it — two launches, no local
           block; falls back to split where its tiles do not fit;
  "split"  scatter kernel -> fused operator on the local block ->
           owner-computes sum (the fallback of "class");
  "colour" one fused gather -> operator -> scatter-add kernel per colour
           class, colours in a fixed order.
Several per-order batches on explicit "owner" maps (the variable-order
configuration) run as one C-ABI global system (`sphp_gsys_*`): a scatter and
the fused operator per batch into one concatenated local block, then a
single owner-computes pass over the global dofs.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib


class AssemblyError(ValueError):
    pass


def encode(local_to_global, signs):
    """Reference (l2g, signs) lists -> (E, nm) int64 codes."""
    rows = []
    for l2g, sgn in zip(local_to_global, signs):
        l2g = np.asarray(l2g, dtype=np.int64)
        sgn = np.asarray(sgn)
        c = l2g.copy()
        neg = sgn < 0
        c[neg] = -(l2g[neg] + 2)
        c[l2g < 0] = -1
        rows.append(c)
    return np.ascontiguousarray(np.stack(rows))


def decode(codes):
    codes = np.asarray(codes, dtype=np.int64)
    gid = np.where(codes >= 0, codes, np.where(codes == -1, -1, -codes - 2))
    sgn = np.where(codes >= 0, 1.0, np.where(codes == -1, 0.0, -1.0))
    return gid, sgn


class AssemblyMap:
    def __init__(self, handle):
        self._h = handle
        ne, nm, ng, nc = C.c_int64(), C.c_int(), C.c_int64(), C.c_int()
        _lib.check(_lib.lib.sphp_amap_info(self._h, C.byref(ne), C.byref(nm), C.byref(ng),
                                           C.byref(nc)))
        self.num_elements, self.nmodes = ne.value, nm.value
        self.num_global, self.num_colours = ng.value, nc.value
        self.periodic = False

    @property
    def algorithm(self):
        """'owner', 'colour', 'split' or 'class' (the library default: class
        on periodic maps, split there at P = 7, owner on explicit maps)."""
        a = C.c_int()
        _lib.check(_lib.lib.sphp_amap_algorithm(self._h, C.byref(a)), AssemblyError)
        return {_lib.ASSEMBLY_OWNER: "owner", _lib.ASSEMBLY_COLOUR: "colour",
                _lib.ASSEMBLY_SPLIT: "split", _lib.ASSEMBLY_CLASS: "class"}[a.value]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and _lib.lib is not None:
            _lib.lib.sphp_amap_destroy(h)
            self._h = None

    @classmethod
    def explicit(cls, codes, num_global):
        codes = np.ascontiguousarray(codes, dtype=np.int64)
        E, nm = codes.shape
        h = C.c_void_p()
        _lib.check(_lib.lib.sphp_amap_create_explicit(E, nm, _lib.ptr(codes), int(num_global),
                                                      C.byref(h)), AssemblyError)
        return cls(h)

    @classmethod
    def from_reference(cls, amap):
        """Any object with local_to_global, signs, num_global (assembly.py:44-56)."""
        return cls.explicit(encode(amap.local_to_global, amap.signs), amap.num_global)

    @classmethod
    def hex_periodic(cls, n, P):
        h = C.c_void_p()
        _lib.check(_lib.lib.sphp_amap_create_hex_periodic(int(n), int(P), C.byref(h)),
                   AssemblyError)
        m = cls(h)
        m.periodic = True
        return m

    def set_algorithm(self, alg):
        """'owner' (gather -> local -> owner-computes sum), 'split' (scatter
        kernel -> local operator -> owner sum), 'colour' (fused
        colour-ordered scatter-add) or, periodic maps only, 'class'
        (class-range gather in the operator -> class block -> owner sum)."""
        code = {"owner": _lib.ASSEMBLY_OWNER, "colour": _lib.ASSEMBLY_COLOUR,
                "split": _lib.ASSEMBLY_SPLIT, "class": _lib.ASSEMBLY_CLASS}[alg]
        _lib.check(_lib.lib.sphp_amap_set_algorithm(self._h, code), AssemblyError)
        return self

    def codes(self):
        out = np.empty((self.num_elements, self.nmodes), dtype=np.int64)
        _lib.check(_lib.lib.sphp_amap_codes(self._h, _lib.ptr(out)))
        return out

    @property
    def local_to_global(self):
        return list(decode(self.codes())[0])

    @property
    def signs(self):
        return list(decode(self.codes())[1])


def hex_variable_codes(n, orders):
    """Full variable-order periodic hex map: (num_global, offsets, codes)."""
    orders = np.ascontiguousarray(orders, dtype=np.int32)
    if orders.size != n ** 3:
        raise AssemblyError(f"need {n ** 3} orders, got {orders.size}")
    ng = C.c_int64()
    _lib.check(_lib.lib.sphp_hexmap_variable(int(n), _lib.ptr(orders), C.byref(ng), None, None),
               AssemblyError)
    offsets = np.empty(n ** 3 + 1, dtype=np.int64)
    total = int(np.sum((orders.astype(np.int64) + 1) ** 3))
    codes = np.empty(total, dtype=np.int64)
    _lib.check(_lib.lib.sphp_hexmap_variable(int(n), _lib.ptr(orders), C.byref(ng),
                                             _lib.ptr(offsets), _lib.ptr(codes)), AssemblyError)
    return ng.value, offsets, codes


def hex_variable_maps(n, orders):
    """Per-order batches of the variable-order map: {P: (elem_ids, AssemblyMap)}."""
    orders = np.asarray(orders).ravel()
    ng, offsets, codes = hex_variable_codes(n, orders)
    out = {}
    for P in sorted(set(int(p) for p in orders)):
        ids = np.nonzero(orders == P)[0]
        nm = (P + 1) ** 3
        rows = np.stack([codes[offsets[e]:offsets[e] + nm] for e in ids])
        out[P] = (ids, AssemblyMap.explicit(rows, ng))
    return ng, out


def _device_input(x, numel, name):
    """(tensor, was_host): x as a contiguous float64 CUDA tensor of `numel`
    values.  Host inputs (numpy arrays / CPU tensors, what the reference's
    assembly.py takes) are copied to the current device; the returned tensor
    must stay referenced until the launch that reads it has been issued."""
    was_host = not (torch.is_tensor(x) and x.is_cuda)
    if was_host:
        t = torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)) if not torch.is_tensor(x)
                            else x.to(torch.float64).contiguous())
        t = t.to(device=torch.device("cuda", torch.cuda.current_device()))
    else:
        t = x if x.dtype == torch.float64 else x.to(torch.float64)
        t = t.contiguous()
    if t.numel() != numel:
        raise AssemblyError(f"{name} has {t.numel()} values, expected {numel}")
    return t, was_host


def _device_output(out, numel, device, shape):
    if out is None:
        return torch.empty(shape, dtype=torch.float64, device=device)
    if not (torch.is_tensor(out) and out.is_cuda and out.dtype == torch.float64 and out.is_contiguous()
            and out.numel() == numel and out.device == device):
        raise AssemblyError(f"out must be a contiguous float64 CUDA tensor of {numel} values on {device}")
    return out


def _overlaps(a, b):
    a0, b0 = a.data_ptr(), b.data_ptr()
    return a0 < b0 + 8 * b.numel() and b0 < a0 + 8 * a.numel()


def scatter(amap: AssemblyMap, x, out=None, stream=None):
    """Global -> local (E, nm), pinned modes -> 0 (assembly.py:150-160).
    Host x -> host result; device x -> device result."""
    xd, host = _device_input(x, amap.num_global, "x")
    out_d = _device_output(None if host else out, amap.num_elements * amap.nmodes, xd.device,
                           (amap.num_elements, amap.nmodes))
    if _overlaps(xd, out_d):
        raise AssemblyError("x and out must not alias")
    _lib.check(_lib.lib.sphp_scatter(amap._h, _lib.ptr(xd), _lib.ptr(out_d), _lib.stream_ptr(stream)),
               AssemblyError)
    return _to_caller(out_d, out, host)


def assemble(amap: AssemblyMap, local, out=None, stream=None):
    """Local (E, nm) -> global, signed, deterministic (assembly.py:141-147).
    Host local -> host result; device local -> device result."""
    ld, host = _device_input(local, amap.num_elements * amap.nmodes, "local")
    out_d = _device_output(None if host else out, amap.num_global, ld.device, (amap.num_global,))
    if _overlaps(ld, out_d):
        raise AssemblyError("local and out must not alias")
    _lib.check(_lib.lib.sphp_assemble(amap._h, _lib.ptr(ld), _lib.ptr(out_d), _lib.stream_ptr(stream)),
               AssemblyError)
    return _to_caller(out_d, out, host)


def _to_caller(out_d, out, host):
    """Device result -> what the caller passed: the device tensor, or (host
    input) a numpy array / the caller's host `out` filled in."""
    if not host:
        return out_d
    res = out_d.cpu().numpy()
    if out is not None:
        out[...] = res if not torch.is_tensor(out) else torch.as_tensor(res)
        return out
    return res


class GlobalHelmholtz:
    """Matrix-free assembled Helmholtz y = A^T H A x over one or more
    per-order batches [(Collection(HELMHOLTZ), AssemblyMap)] that share the
    global numbering (GlobalSystem.apply, assembly.py:177-182)."""

    def __init__(self, batches, num_global):
        self.batches = list(batches)
        self.num_global = int(num_global)
        for coll, amap in self.batches:
            if amap.num_global != self.num_global:
                raise AssemblyError("batches disagree on num_global")
        self._gsys = None
        if len(self.batches) > 1 and all(not a.periodic and a.algorithm == "owner"
                                         for _, a in self.batches):
            # several per-order batches on explicit maps: one C-ABI global
            # system (concatenated local block, one owner-computes pass)
            n = len(self.batches)
            colls = (C.c_void_p * n)(*[c._handle for c, _ in self.batches])
            maps = (C.c_void_p * n)(*[a._h for _, a in self.batches])
            h = C.c_void_p()
            _lib.check(_lib.lib.sphp_gsys_create(colls, maps, n, self.num_global, C.byref(h)),
                       AssemblyError)
            self._gsys = h

    def reserve(self, stream=None, host=False):
        """Size the per-stream workspaces this operator's applies on `stream`
        use (they are otherwise sized at the first apply on a stream); needed
        before capturing applies into a CUDA graph."""
        if self._gsys is not None:
            _lib.check(_lib.lib.sphp_gsys_reserve(self._gsys, _lib.stream_ptr(stream)), AssemblyError)
            return self
        flags = _lib.RESERVE_DEVICE | (_lib.RESERVE_HOST if host else 0)
        for coll, amap in self.batches:
            _lib.check(_lib.lib.sphp_collection_reserve(coll._handle, amap._h, flags, _lib.stream_ptr(stream)),
                       AssemblyError)
        return self

    def __del__(self):
        h = getattr(self, "_gsys", None)
        if h and _lib is not None and _lib.lib is not None:
            _lib.lib.sphp_gsys_destroy(h)
            self._gsys = None

    def apply(self, x, out=None, stream=None):
        """y = A^T H A x.  Device x (contiguous float64 CUDA tensor) -> device
        y; host x (numpy / CPU tensor, the reference's GlobalSystem.apply
        argument) -> host y.  x and out must not alias (every algorithm
        reads x while writing y)."""
        xd, host = _device_input(x, self.num_global, "x")
        out_d = _device_output(None if host else out, self.num_global, xd.device, (self.num_global,))
        if _overlaps(xd, out_d):
            raise AssemblyError("x and out must not alias")
        if self._gsys is not None:
            _lib.check(_lib.lib.sphp_gsys_apply(self._gsys, _lib.ptr(xd), _lib.ptr(out_d),
                                                _lib.stream_ptr(stream)), AssemblyError)
            return _to_caller(out_d, out, host)
        for k, (coll, amap) in enumerate(self.batches):
            rc = _lib.lib.sphp_helmholtz_assembled(coll._handle, amap._h, _lib.ptr(xd), _lib.ptr(out_d),
                                                   1 if k else 0, _lib.stream_ptr(stream))
            _lib.check(rc, AssemblyError)
        return _to_caller(out_d, out, host)

    def apply_phases(self, x, out, stream=None):
        """One apply (single batch) with CUDA events between its launches on
        `stream`: returns the launches' durations in ms (class: operator,
        owner sum; split: scatter, operator, owner sum).  Synchronises."""
        if len(self.batches) != 1:
            raise AssemblyError("apply_phases takes one (collection, map) batch")
        coll, amap = self.batches[0]
        if not (torch.is_tensor(x) and x.is_cuda):
            raise AssemblyError("apply_phases takes device vectors")
        x, _ = _device_input(x, self.num_global, "x")
        out = _device_output(out, self.num_global, x.device, (self.num_global,))
        if _overlaps(x, out):
            raise AssemblyError("x and out must not alias")
        ms = (C.c_float * 8)()
        nph = C.c_int()
        _lib.check(_lib.lib.sphp_helmholtz_assembled_phases(coll._handle, amap._h, _lib.ptr(x), _lib.ptr(out),
                                                            _lib.stream_ptr(stream), 8, ms, C.byref(nph)),
                   AssemblyError)
        return [float(ms[i]) for i in range(nph.value)]

    def apply_host(self, x, out=None, stream=None):
        """y = A^T H A x with HOST vectors (numpy or CPU tensor; pinned for
        full overlap): the C-ABI call sphp_helmholtz_assembled_host, which on
        periodic split maps pipelines the copies over z-slabs.  Single batch."""
        if len(self.batches) != 1:
            raise AssemblyError("apply_host takes one (collection, map) batch")
        coll, amap = self.batches[0]
        if torch.is_tensor(x):
            if x.is_cuda or x.dtype != torch.float64 or not x.is_contiguous():
                raise AssemblyError("x must be a contiguous float64 host tensor")
        else:
            x = np.ascontiguousarray(x, dtype=np.float64)
        if out is None:
            out = np.empty(self.num_global) if not torch.is_tensor(x) else torch.empty_like(x)
        rc = _lib.lib.sphp_helmholtz_assembled_host(coll._handle, amap._h, _lib.ptr(x), _lib.ptr(out),
                                                    _lib.stream_ptr(stream))
        _lib.check(rc, AssemblyError)
        return out

    __call__ = apply
