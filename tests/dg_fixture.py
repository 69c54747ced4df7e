"""Rebuild DGSystem-like objects and reference states from
tests/golden/reference_dg.npz (written by tests/golden/make_golden_dg.py)."""
from pathlib import Path
from types import SimpleNamespace

import numpy as np

from dg_cases import CASES

G = np.load(Path(__file__).resolve().parent / "golden" / "reference_dg.npz")


def system(tag, make_quad):
    P, Q = int(G[f"{tag}/P"]), int(G[f"{tag}/Q"])
    ns = SimpleNamespace(exp=make_quad(P, Q), bcs=CASES[tag]["bcs"])
    for k in ("ww", "inv", "minv", "xy", "int_li", "int_ri"):
        setattr(ns, k, G[f"{tag}/{k}"])
    if ns.int_li.size:
        for k in ("exm", "lm", "exp", "lp", "warc", "nrm", "xy"):
            setattr(ns, f"int_{k}", G[f"{tag}/int_{k}"])
    ns.bnd = {}
    for name in G[f"{tag}/bnd_names"]:
        name = str(name)
        if name:
            ns.bnd[name] = {k: G[f"{tag}/bnd/{name}/{k}"] for k in ("li", "exm", "lm", "nrm", "warc", "xy")}
    return ns


def sample(fn, xy, t=0.0):
    vals = fn(x=xy[..., 0], y=xy[..., 1], t=t)
    return np.asarray(vals, float) * np.ones(xy.shape[:-1])


def ape_state(tag, k, sys_ns):
    """Base-flow samples the way make_ape_state takes them (solvers.py:461-495)."""
    case = CASES[tag]["ape"][k]
    keys = ("ux", "uy", "rho", "c2")
    base = {v: sample(case["base"][v], sys_ns.xy) for v in keys}
    base_trace = ({v: sample(case["base"][v], sys_ns.int_xy) for v in keys}
                  if sys_ns.int_li.size else {})
    base_bnd = {name: {v: sample(case["base"][v], g["xy"]) for v in keys}
                for name, g in sys_ns.bnd.items()}
    const = bool(G[f"{tag}/ape{k}/c2_constant"])
    return dict(base=base, base_trace=base_trace, base_bnd=base_bnd, riemann=case["riemann"],
                sources=case.get("sources"), c2_per_element=base["c2"][:, 0].copy() if const else None,
                t=case.get("t", 0.0))
