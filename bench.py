#!/usr/bin/env python
"""Benchmark of the matrix-free hex Helmholtz operator (BASELINE.json cfg4).

One step = one assembled matrix-free Helmholtz apply y = A^T H A x on the
64^3 periodic deformed hex mesh (x' = x + 0.03 sin 2πy sin 2πz), P=4, Q=6
GLL, lambda = 1, per-point geometric factors stored (6 metric terms + |J|):
the map's default (class-range) algorithm — one fused launch gathers x by
entity-class ranges, runs BwdTrans -> PhysDeriv -> metric ->
IProductWRTDerivBase + lambda IProductWRTBase and writes the tile-major class
block (interiors straight into y), then the deterministic streaming
owner-computes C0 sum.  `value` is local DoF/s (E (P+1)^3 /
step time); global DoF/s is reported too.

Arms:
  default            the CUDA path (libspechp_b200.so) through the public API
  --impl reference   the reference algorithm's CPU port (oracle/, numpy,
                     all host threads) on a bounded sample of the same
                     workload (the reference itself is Python with no hex
                     path)

Multi-GPU (torchrun): every rank runs an independent 64^3 mesh (weak
scaling: elemental operators shard by element with no data-path exchange);
time = max over ranks of the CUDA-event time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SEED = int(os.environ.get("SPECHP_SEED", "20240801"))
AMP = 0.03


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--P", type=int, default=4)
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--no-sweep", dest="sweep", action="store_false",
                    help="skip the P=2..8 sweep (extra JSON key, on by default)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extras", action="store_true", help="skip the other BASELINE configs")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sharded", action="store_true",
                    help="one n^3 mesh cut into z-slabs across the ranks (strong scaling, one "
                         "interface exchange per apply) instead of one mesh per rank")
    return ap.parse_args()


def metric_name(P, n):
    return (f"matrix-free Helmholtz DoF/s (assembled, hex P={P}, {n}^3 deformed periodic, "
            "FP64, 1 B200 per rank)")


def workload_bytes(P, n):
    """Algorithmic HBM bytes of one assembled apply:
    geometry 7 Q^3 doubles per element + x read + y written (global)."""
    E = n ** 3
    Q = P + 2
    ng = (n * P) ** 3
    return 8 * (7 * Q ** 3 * E + 2 * ng)


def local_bytes(P, E):
    m, Q = P + 1, P + 2
    return 8 * (2 * m ** 3 + 7 * Q ** 3) * E


def helm_flops(P, E):
    m, Q = P + 1, P + 2
    staged = m ** 3 * Q + m * m * Q * Q + m * Q ** 3
    return 2 * E * (2 * staged + 6 * Q ** 4 + 11 * Q ** 3)


TRAFFIC_FILE = ROOT / "profiles" / "r02_ncu_traffic.json"
FP64_PEAK_TFS = 34.2   # DFMA microbenchmark on this pool (tools/fp64_peak.cu, profiles/r02_fp64_peak.log)
NOMINAL_HBM_GBS = 8000.0


def ncu_traffic(kernel, P, n):
    """(DRAM bytes per launch, kernel name) of `kernel` at (P, n) from the
    committed ncu capture (profiles/r02_ncu_traffic.json), or (None, None)."""
    if not TRAFFIC_FILE.exists():
        return None, None
    d = json.loads(TRAFFIC_FILE.read_text()).get(kernel)
    if d and d.get("P") == P and d.get("n") == n:
        return d["bytes_per_launch"], d.get("kernel")
    return None, None


def class_op_bytes(P, n):
    """Algorithmic bytes of the class-range operator launch: geometry
    (7 Q^3 per element) + x read once + every local result written once
    (tile-major class block + interiors into y)."""
    E, Q, m = n ** 3, P + 2, P + 1
    return 8 * (7 * Q ** 3 * E + (n * P) ** 3 + E * m ** 3)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi, during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
                for k, nm in enumerate(names):
                    if r[5 + k].lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU legs (oracle port; test infrastructure, timed here as the baseline)
# ---------------------------------------------------------------------------
def cpu_port_assembled(P, n_sample, seconds, seed=SEED):
    """The reference algorithm (GlobalSystem.apply = scatter -> elemental
    Helmholtz -> assemble, assembly.py:177-182, with the sum-factorised
    elemental operator of collections.py restated for hex) on an
    n_sample^3 periodic sub-mesh with the same mapping; numpy, BLAS threads
    = all host cores.  Returns (local DoF/s, runs, seconds, cores)."""
    from oracle import assembly as oa
    from oracle import geometry as og
    from oracle import ops as oo

    oe = oo.Expansion("hex", P, P + 2)
    E = n_sample ** 3
    _, _, inv, wj = og.factors(oe, n_sample, np.arange(E), og.MAP_HEX_SINE, AMP)
    G = oo.metric_from_inv(wj, inv)
    om = oa.hex_periodic_map(n_sample, P)
    codes = oa.pack_map(om)
    x = np.random.default_rng(seed).uniform(-1, 1, om.num_global)

    def step():
        loc = x[codes]                                  # signed gather (all +1)
        yl = oo.helmholtz(oe, loc, 1.0, G, wj)
        y = np.zeros(om.num_global)
        np.add.at(y, codes.ravel(), yl.ravel())        # assemble (np.add.at)
        return y

    step()
    runs, t0 = 0, time.perf_counter()
    while True:
        step()
        runs += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return runs * E * (P + 1) ** 3 / el, runs, el, os.cpu_count() or 1, E


def parity_sample(P, n, x, y, c, yl, seed=SEED):
    """Parity of the measured applies against the oracle (the checker; run
    outside every timed region): the assembled y on the global dofs of 24
    sampled elements (exact given their 27-element neighbourhoods, map =
    the oracle's numbering of assembly.py:72-138) and the local K4 output
    on 512 sampled elements including the first and last ones."""
    from oracle import assembly as oa
    from oracle import geometry as og
    from oracle import ops as oo

    E = n ** 3
    oe = oo.Expansion("hex", P, P + 2)
    rng = np.random.default_rng(seed)

    def helm(ids, coeffs):
        _, _, inv, wj = og.factors(oe, n, ids, og.MAP_HEX_SINE, AMP)
        return oo.helmholtz(oe, coeffs, 1.0, oo.metric_from_inv(wj, inv), wj)

    def errs(got, ref):
        return {"rel_l2": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
                "max_abs": float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))}

    _, _, codes = oa.hex_periodic_codes(n, P)
    codes = codes.reshape(E, -1)
    sample = np.unique(np.concatenate([[0, E - 1], rng.choice(E, 22, replace=False)]))
    ex, ey, ez = sample % n, (sample // n) % n, sample // (n * n)
    nb = np.unique(np.concatenate([((ex + a) % n) + n * (((ey + b) % n) + n * ((ez + cc) % n))
                                   for a in (-1, 0, 1) for b in (-1, 0, 1) for cc in (-1, 0, 1)]))
    ylo = helm(nb, x[codes[nb]])
    yref = np.bincount(codes[nb].ravel(), weights=ylo.ravel(), minlength=x.size)
    dofs = np.unique(codes[sample])
    out = {"assembled": dict(errs(y[dofs], yref[dofs]), dofs=int(dofs.size)),
           "tolerance": {"rel_l2": 1e-12, "max_abs": 1e-11}}
    ids = np.unique(np.concatenate([np.arange(128), np.arange(E - 128, E),
                                    rng.choice(E, 256, replace=False)]))
    out["local"] = dict(errs(yl[ids], helm(ids, c[ids])), elements=int(ids.size))
    out["ok"] = all(out[k]["rel_l2"] < 1e-12 and out[k]["max_abs"] < 1e-11 for k in ("assembled", "local"))
    return out


# ---------------------------------------------------------------------------
class FullMeshPort:
    """The reference algorithm (GlobalSystem.apply: scatter -> elemental
    Helmholtz -> assemble, assembly.py:177-182, with collections.py's
    sum-factorised elemental operator restated for hex by oracle/) on the
    FULL n^3 mesh, chunked over elements (geometry of all chunks prepared
    once: 3.2 GB at P = 4, n = 64).  One apply = every chunk's gather,
    operator and np.add.at assembly."""

    def __init__(self, P, n, chunk=8192, seed=SEED):
        from oracle import assembly as oa
        from oracle import geometry as og
        from oracle import ops as oo

        self.oo = oo
        self.oe = oo.Expansion("hex", P, P + 2)
        E = n ** 3
        _, _, codes = oa.hex_periodic_codes(n, P)
        self.codes = codes.reshape(E, -1)
        self.ng = (n * P) ** 3
        self.x = np.random.default_rng(seed).uniform(-1, 1, self.ng)
        self.chunks = []
        for c0 in range(0, E, chunk):
            ids = np.arange(c0, min(E, c0 + chunk))
            _, _, inv, wj = og.factors(self.oe, n, ids, og.MAP_HEX_SINE, AMP)
            self.chunks.append((ids, oo.metric_from_inv(wj, inv), wj))
        self.local_dofs = E * (P + 1) ** 3

    def apply(self):
        y = np.zeros(self.ng)
        for ids, G, wj in self.chunks:
            cod = self.codes[ids]
            yl = self.oo.helmholtz(self.oe, self.x[cod], 1.0, G, wj)
            np.add.at(y, cod.ravel(), yl.ravel())
        return y


def reference_2d(seconds_budget=150.0):
    """The reference ITSELF (baseline/_ref, installed from /root/reference;
    pure Python/numpy) on the 2D BASELINE configs, in its own protocol:
    autotune (collections.py:285-313: median of trials over every strategy)
    per operator on cfg1 (32x32 affine quads, P=4, Q=6 GLL) and the
    assembled matrix-free GlobalSystem.apply (assembly.py:177-182) of the
    Helmholtz operator on 256x256 quads, P=6, Q=8 (cfg2's size; the
    reference's geometry cannot express cfg2's curved map, so the mesh is
    affine).  None when baseline/_ref is absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "spechp").is_dir():
        return None
    sys.path.insert(0, str(ref))
    from spechp.assembly import build_assembly_map, build_global_system
    from spechp.collections import OperatorKind, autotune
    from spechp.meshio import structured_quad_mesh
    from spechp.region import build_elements

    out = {"source": "baseline/_ref (pip install --no-index --no-deps of /root/reference/pkg)"}
    t_start = time.perf_counter()
    mesh = structured_quad_mesh(32, 32)
    els = build_elements(mesh, orders=4, num_points=6)
    cfg1 = {}
    for op in (OperatorKind.BWD_TRANS, OperatorKind.IPRODUCT_WRT_BASE, OperatorKind.PHYS_DERIV):
        pick, rep = autotune(els, op, trials=5, warmups=2)
        cfg1[op.value] = {"pick": pick.value,
                          "median_s": {k: v.get("median_s") for k, v in rep.items() if isinstance(v, dict)}}
    out["cfg1_autotune"] = cfg1
    if time.perf_counter() - t_start < seconds_budget:
        t0 = time.perf_counter()
        mesh = structured_quad_mesh(256, 256)
        els = build_elements(mesh, orders=6, num_points=8)
        amap = build_assembly_map(mesh, els, ())
        system = build_global_system(els, amap, "helmholtz", 1.0)
        setup = time.perf_counter() - t0
        x = np.random.default_rng(SEED).uniform(-1, 1, amap.num_global)
        system.apply(x)
        times = []
        for _ in range(3):
            t1 = time.perf_counter()
            system.apply(x)
            times.append(time.perf_counter() - t1)
        t = statistics.median(times)
        out["cfg2_global_apply"] = {"s": t, "global_dofs": int(amap.num_global),
                                    "local_dofs": int(len(els) * 49),
                                    "global_dof_s": amap.num_global / t, "local_dof_s": len(els) * 49 / t,
                                    "matrix_free": system.matrix is None, "setup_s": setup,
                                    "mesh": "256x256 affine quads P=6 Q=8 (cfg2 size, affine map)"}
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on the host cores (tier
    rules: the CPU restatement in oracle/, BLAS threads = all cores), on the
    FULL 64^3 cfg4 mesh (chunked), one assembled apply per step; plus the
    reference itself (baseline/_ref) on the 2D configs."""
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits

    cores = os.cpu_count() or 1
    with threadpool_limits(limits=cores):
        port = FullMeshPort(args.P, args.n)
        t0 = time.perf_counter()
        port.apply()  # first (untimed) apply also sizes the step budget
        first = time.perf_counter() - t0
        warm = max(0, args.warmup - 1)
        # each step is one full apply; keep the whole run within ~3 minutes
        steps = max(3, min(args.steps, int(150.0 / max(first, 1e-3)) - warm))
        for _ in range(warm):
            port.apply()
        times = []
        for _ in range(steps):
            t1 = time.perf_counter()
            port.apply()
            times.append(time.perf_counter() - t1)
        t = statistics.median(times)
        value = port.local_dofs / t
        r2d = None
        try:
            r2d = reference_2d()
        except Exception as exc:  # the 2D extra must not sink the line
            r2d = {"error": repr(exc)}
    sample = (f"full {args.n}^3 mesh, one assembled apply per step (median of {steps}), "
              f"chunks of 8192 elements, numpy + BLAS threads = {cores}")
    line = {
        "metric": metric_name(args.P, args.n), "value": value, "unit": "DoF/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, SPECHP_SEED)",
        "config": {"workload": f"cfg4 hex Helmholtz P={args.P} n={args.n} (full mesh)",
                   "P": args.P, "Q": args.P + 2, "n": args.n, "lambda": 1.0},
        "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_2d": r2d,
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1906_03489_b200 as sp
    from paper_1906_03489_b200 import _lib, parallel

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    P, n = args.P, args.n
    E = n ** 3
    m = P + 1

    def build(P):
        exp = sp.make_hex(P, P + 2)
        batch = sp.ElementBatch.structured(exp, n, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE,
                                           amp=AMP, device=dev)
        coll = sp.Collection(batch, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC, lam=1.0)
        amap = sp.AssemblyMap.hex_periodic(n, P)
        return exp, batch, coll, amap

    exp, batch, coll, amap = build(P)
    op = sp.GlobalHelmholtz([(coll, amap)], amap.num_global)
    ng = amap.num_global
    rng = np.random.default_rng(SEED + rank)
    x_host = torch.from_numpy(rng.uniform(-1, 1, ng)).pin_memory()
    y_host = torch.empty(ng, dtype=torch.float64).pin_memory()
    x = x_host.to(dev)
    y = torch.empty(ng, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ms = parallel.max_over_ranks(e0.elapsed_time(e1), device=dev)
        return ms / steps

    # ---- headline: assembled apply, inputs resident ------------------------
    clocks = Clocks(local_rank)
    for _ in range(args.warmup):
        op.apply(x, y)
    torch.cuda.synchronize(dev)
    clocks.start()
    ms = timed(lambda: op.apply(x, y), args.steps, 0)
    clk = clocks.stop()
    value = world * E * m ** 3 / (ms * 1e-3)
    # replicas were fed rank-seeded inputs; the same input on every rank must
    # give bitwise-identical outputs (deterministic kernels)
    if world > 1:
        x_same = torch.as_tensor(np.random.default_rng(SEED).uniform(-1, 1, ng), device=dev)
        lo, hi = parallel.replica_checksum(op.apply(x_same, y))
        replicas_identical = lo == hi
    else:
        replicas_identical = None

    # ---- e2e: the C-ABI host-buffer call (H2D x, apply, D2H y, sync) -------
    def e2e_step():
        rc = _lib.lib.sphp_helmholtz_assembled_host(coll._handle, amap._h, _lib.ptr(x_host),
                                                    _lib.ptr(y_host), _lib.stream_ptr(stream))
        _lib.check(rc)

    e2e_ms = timed(e2e_step, max(3, args.steps // 2), 2)
    e2e_value = world * E * m ** 3 / (e2e_ms * 1e-3)

    # ---- dominant kernel of the step: its launches timed by CUDA events on
    # the launch stream (sphp_helmholtz_assembled_phases), averaged over
    # `steps` applies; the fused local Helmholtz (block in/out) timed alone
    phase_runs = [op.apply_phases(x, y, stream) for _ in range(args.steps)]
    nph = len(phase_runs[0])
    phase_ms = [statistics.mean(r[i] for r in phase_runs) for i in range(nph)]
    c = torch.as_tensor(np.random.default_rng(SEED).uniform(-1, 1, (E, m ** 3)), device=dev)
    yl = torch.empty_like(c)
    k_ms = timed(lambda: coll.apply(c, yl), args.steps, args.warmup)
    peak, peak_kind = measured_peaks()
    kb = local_bytes(P, E)
    if amap.algorithm == "class" and nph == 2:
        dom_ms, dom_bytes = phase_ms[0], class_op_bytes(P, n)
        dom_name = "pipe_kernel<HexHelm, MODE 5> (class-range fused Helmholtz, launch 1 of 2)"
        traffic, traffic_kernel = ncu_traffic("helmholtz_class", P, n)
    else:
        dom_ms, dom_bytes = k_ms, kb
        dom_name = "pipe_kernel<HexHelm, MODE 0> (fused local Helmholtz)"
        traffic, traffic_kernel = ncu_traffic("helmholtz_local", P, n)
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    # assembled apply as a whole against the same roofline
    ab = workload_bytes(P, n)
    a_achieved = ab / (ms * 1e-3) / 1e9
    parity = None
    if rank == 0:
        # checked outside every timed region: the last timed outputs y, yl
        op.apply(x, y)
        coll.apply(c, yl)
        parity = parity_sample(P, n, x_host.numpy(), y.cpu().numpy(), c.cpu().numpy(), yl.cpu().numpy())
    del c, yl

    plan_names = {0: "k-row", 1: "j-pencil", 3: "i-column"}

    def plan_of(Ps):
        return plan_names.get(sp._lib.lib.sphp_hex_helmholtz_plan(Ps + 1, Ps + 2), "none")

    sweep = None
    if args.sweep:
        sweep = {}
        for Ps in range(2, 9):
            if Ps == P:
                sweep[str(Ps)] = {"assembled_ms": ms, "local_ms": k_ms, "plan": plan_of(Ps),
                                  "assembled_roofline_frac": workload_bytes(Ps, n) / (ms * 1e-3) / 1e9 / peak}
                continue
            _, b2, c2, a2 = build(Ps)
            op2 = sp.GlobalHelmholtz([(c2, a2)], a2.num_global)
            x2 = torch.as_tensor(np.random.default_rng(Ps).uniform(-1, 1, a2.num_global), device=dev)
            y2 = torch.empty_like(x2)
            t_as = timed(lambda: op2.apply(x2, y2), max(5, args.steps // 2), 3)
            cc = torch.as_tensor(np.random.default_rng(Ps).uniform(-1, 1, (E, (Ps + 1) ** 3)), device=dev)
            yy = torch.empty_like(cc)
            t_lo = timed(lambda: c2.apply(cc, yy), max(5, args.steps // 2), 3)
            lb = local_bytes(Ps, E)
            sweep[str(Ps)] = {
                "assembled_ms": t_as, "local_ms": t_lo,
                "assembled_local_dof_s": E * (Ps + 1) ** 3 / (t_as * 1e-3),
                "local_dof_s": E * (Ps + 1) ** 3 / (t_lo * 1e-3),
                "local_hbm_gbs": lb / (t_lo * 1e-3) / 1e9,
                "local_roofline_frac": lb / (t_lo * 1e-3) / 1e9 / peak,
                "local_fp64_tflops": helm_flops(Ps, E) / (t_lo * 1e-3) / 1e12,
                "assembled_roofline_frac": workload_bytes(Ps, n) / (t_as * 1e-3) / 1e9 / peak,
                "plan": plan_of(Ps),
            }
            del b2, c2, a2, op2, x2, y2, cc, yy
            torch.cuda.empty_cache()

    extras = None
    if not args.no_extras:
        try:
            extras = config_extras(sp, dev, timed, peak)
        except Exception as exc:  # extras must never sink the headline line
            extras = {"error": repr(exc)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from threadpoolctl import threadpool_limits

        n_s = 12 if P <= 4 else 8
        with threadpool_limits(limits=os.cpu_count() or 1):
            v, runs, el, cores, Es = cpu_port_assembled(P, n_s, args.cpu_seconds)
        cpu = {"value": v, "unit": "DoF/s", "cores": cores, "kind": "port",
               "sample": f"{runs} assembled applies on a {n_s}^3 periodic sub-mesh ({Es} elements, "
                         f"same map, P={P}) in {el:.1f} s, numpy + BLAS threads = {cores} (threadpoolctl); "
                         f"the rate is quoted per local DoF, i.e. extrapolated to the {n}^3 mesh — "
                         "bench.py --impl reference times the full mesh (chunked)"}

    if rank != 0:
        return
    line = {
        "metric": metric_name(P, n), "value": value, "unit": "DoF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SPECHP_SEED; analytic deformed mesh)",
        "config": {"workload": f"cfg4: assembled matrix-free hex Helmholtz P={P} Q={P + 2} n={n} "
                               "periodic deformed, lambda=1", "P": P, "Q": P + 2, "n": n,
                   "elements_per_rank": E, "global_dofs_per_rank": ng,
                   "local_dofs_per_rank": E * m ** 3, "parallelism": f"replicas x{world} (weak)",
                   "assembly": amap.algorithm,
                   "l2": "inputs larger than L2 (geometry 3.2 GB/apply at P=4)"},
        "global_dof_s": world * ng / (ms * 1e-3),
        "e2e": {"value": e2e_value, "unit": "DoF/s", "h2d_bytes_per_step": 8 * ng,
                "d2h_bytes_per_step": 8 * ng, "ms_per_step": e2e_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "traffic_source": (f"{TRAFFIC_FILE.relative_to(ROOT)} (ncu dram__bytes_read+write, "
                                        f"{traffic_kernel})") if traffic else None,
                     "kernel": dom_name, "bytes_per_launch": dom_bytes, "launch_ms": dom_ms,
                     "share_of_step": dom_ms / ms, "phase_ms": phase_ms,
                     "frac_nominal_8tbs": achieved / NOMINAL_HBM_GBS,
                     "fp64_tflops": helm_flops(P, E) / (dom_ms * 1e-3) / 1e12,
                     "fp64_frac": helm_flops(P, E) / (dom_ms * 1e-3) / 1e12 / FP64_PEAK_TFS,
                     "local": {"kernel": "pipe_kernel<HexHelm, MODE 0> (block in/out, timed alone)",
                               "launch_ms": k_ms, "bytes_per_launch": kb,
                               "achieved": kb / (k_ms * 1e-3) / 1e9,
                               "frac": kb / (k_ms * 1e-3) / 1e9 / peak},
                     "assembled_achieved": a_achieved, "assembled_frac": a_achieved / peak,
                     "assembled_bytes_per_step": ab},
        "cpu_baseline": cpu,
        "clocks": clk,
        # class: class-range operator + owner sum; split: scatter, operator,
        # owner sum; owner: gather-fused operator + owner sum
        "gpu_launches": args.steps * (3 if amap.algorithm == "split" else 2),
        "replicas_identical": replicas_identical,
        "parity": parity,
    }
    if sweep is not None:
        line["sweep"] = sweep
    if extras is not None:
        line["configs"] = extras
    print(json.dumps(line), flush=True)


def config_extras(sp, dev, timed, peak):
    """The other BASELINE.json configs, timed on the device (parity cases,
    reported for the roofline picture, not bench lines)."""
    import torch

    out = {}
    rng = np.random.default_rng(SEED)

    def graph_ms(coll, x, y, reps=20):
        """Device time per apply without the Python call overhead: `reps`
        applies captured in one CUDA graph, replayed (small configs are
        host-bound when launched one call at a time)."""
        try:
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                coll.apply(x, y)
            torch.cuda.current_stream(dev).wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(reps):
                    coll.apply(x, y)
            return timed(lambda: g.replay(), 5, 2) / reps
        except Exception:  # capture unsupported here: report the plain timing only
            return None

    def op_entry(name, coll, x):
        y = torch.empty(coll.output_shape, dtype=torch.float64, device=dev)
        ms = timed(lambda: coll.apply(x, y), 20, 3)
        b = coll.hbm_bytes()
        gms = graph_ms(coll, x, y)
        out[name] = {"ms": ms, "elements": coll.num_elements, "hbm_bytes": b,
                     "hbm_gbs": b / (ms * 1e-3) / 1e9, "frac": b / (ms * 1e-3) / 1e9 / peak,
                     "dof_s": coll.num_elements * (x.shape[1] if coll.operator.value == "bwdtrans"
                                                   else coll.output_shape[-1]) / (ms * 1e-3),
                     "graph_ms": gms,
                     "graph_frac": (b / (gms * 1e-3) / 1e9 / peak) if gms else None}

    # cfg1: 32x32 affine quads, P=4, Q=6: BwdTrans + IProductWRTBase
    q = sp.make_quad(4, 6)
    b1 = sp.ElementBatch.structured(q, 32, kind=sp.GEOM_AFFINE, device=dev)
    for op, size in (("bwdtrans", 25), ("iproductwrtbase", 36)):
        c = sp.Collection(b1, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC)
        op_entry(f"cfg1_quad_{op}", c, torch.as_tensor(rng.uniform(-1, 1, (1024, size)), device=dev))
    # cfg2: 256x256 curved quads, P=6, Q=8: PhysDeriv + Helmholtz
    q6 = sp.make_quad(6, 8)
    bp = sp.ElementBatch.structured(q6, 256, kind=sp.GEOM_POINT, mapping=sp.MAP_QUAD_SINE, amp=0.05,
                                    device=dev)
    c = sp.Collection(bp, sp.OperatorKind.PHYS_DERIV, sp.Strategy.CUDA_SUMFAC)
    op_entry("cfg2_quad_physderiv", c, torch.as_tensor(rng.uniform(-1, 1, (65536, 64)), device=dev))
    bm = sp.ElementBatch.structured(q6, 256, kind=sp.GEOM_METRIC, mapping=sp.MAP_QUAD_SINE, amp=0.05,
                                    device=dev)
    c = sp.Collection(bm, sp.OperatorKind.HELMHOLTZ, sp.Strategy.CUDA_SUMFAC, lam=1.0)
    op_entry("cfg2_quad_helmholtz", c, torch.as_tensor(rng.uniform(-1, 1, (65536, 49)), device=dev))
    del bp, bm
    # cfg3: 64^3 affine hexes, P=4, Q=6: BwdTrans, IProductWRTBase, PhysDeriv
    h = sp.make_hex(4, 6)
    ba = sp.ElementBatch.structured(h, 64, kind=sp.GEOM_AFFINE, device=dev)
    for op, size in (("bwdtrans", 125), ("iproductwrtbase", 216), ("physderiv", 216)):
        c = sp.Collection(ba, sp.OperatorKind(op), sp.Strategy.CUDA_SUMFAC)
        op_entry(f"cfg3_hex_{op}", c, torch.as_tensor(rng.standard_normal((262144, size)), device=dev))
        torch.cuda.empty_cache()
    # cfg5: 48^3 deformed hexes, variable P in {3..7}, assembled Helmholtz
    n5 = 48
    orders = np.random.default_rng(SEED + 5).integers(3, 8, n5 ** 3)
    ng, maps = sp.hex_variable_maps(n5, orders)
    batches = []
    choice = {}
    for P, (ids, amap) in maps.items():
        e = sp.make_hex(P, P + 2)
        bb = sp.ElementBatch.structured(e, n5, kind=sp.GEOM_METRIC, mapping=sp.MAP_HEX_SINE, amp=AMP,
                                        elem_ids=ids, device=dev)
        strat, rep = sp.autotune(bb, sp.OperatorKind.HELMHOLTZ, trials=3, warmups=1)
        choice[str(P)] = {k: (v.get("median_s") if "median_s" in v else v.get("error", "")[:60])
                          for k, v in rep.items()}
        choice[str(P)]["pick"] = strat.value
        batches.append((sp.Collection(bb, sp.OperatorKind.HELMHOLTZ, strat), amap))
    g = sp.GlobalHelmholtz(batches, ng)
    x = torch.as_tensor(rng.uniform(-1, 1, ng), device=dev)
    y = torch.empty_like(x)
    ms = timed(lambda: g.apply(x, y), 10, 3)
    ldofs = int(np.sum((orders + 1) ** 3))
    out["cfg5_hex_variable_assembled"] = {"ms": ms, "elements": n5 ** 3, "global_dofs": ng,
                                          "local_dof_s": ldofs / (ms * 1e-3),
                                          "global_dof_s": ng / (ms * 1e-3), "selector": choice}
    return out


def run_sharded(args, rank, world, local_rank):
    """--sharded: ONE n^3 mesh cut into z-slabs across the ranks (SURVEY
    §8(e)): each rank applies its slab's elements and the operator's one
    exchange step swaps the interface partial sums with the ring neighbours
    (pack / combine kernels + NCCL point-to-point).  Strong scaling: value =
    the whole mesh's local DoFs / max-over-ranks step time."""
    import torch
    import torch.distributed as dist

    from paper_1906_03489_b200 import parallel
    from paper_1906_03489_b200.distributed import DistributedHelmholtz, SlabPartition

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    P, n = args.P, args.n
    part = SlabPartition(n, P, rank, world)
    op = DistributedHelmholtz.from_gpu(part, device=dev)
    x_global = np.random.default_rng(SEED).uniform(-1, 1, part.num_global_total)
    x = torch.as_tensor(x_global[part.gids], device=dev)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        op.apply(x, y)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        op.apply(x, y)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = parallel.max_over_ranks(e0.elapsed_time(e1), device=dev) / args.steps
    value = n ** 3 * (P + 1) ** 3 / (ms * 1e-3)
    if rank != 0:
        return
    line = {
        "metric": metric_name(P, n), "value": value, "unit": "DoF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SPECHP_SEED; analytic deformed mesh)",
        "config": {"workload": f"cfg4 assembled hex Helmholtz P={P} n={n}, one mesh in z-slabs",
                   "P": P, "n": n, "parallelism": f"z-slabs x{world}",
                   "interface_dofs_per_neighbour": int(n * n * P * P),
                   "slab_algorithm": "explicit slab map, split (scatter, fused operator, CSR owner sum)"},
        "gpu_launches": args.steps * (3 + 2 * (world > 1)),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if world > 1 and rank != 0:
            return
        run_reference(args, rank, world)
        return
    if world > 1:
        from paper_1906_03489_b200 import parallel

        parallel.init("nccl")
    if args.sharded:
        run_sharded(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
