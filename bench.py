#!/usr/bin/env python
"""bench.py — fp64 cell-RHS evaluations per second of the narrow-stencil
operator (a U_x)_x + (a U_y)_y + (a U_z)_z, BASELINE.json configs[1]
(256^3 per GPU, periodic; weak scaling over z-slabs with a 4-plane NCCL halo
exchange overlapped with the interior for N > 1, configs[3]-style).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one evaluation of the operator over the whole job's box.
value   = cells of all ranks / max-over-ranks device time of K steps.
e2e     = the same metric through the public API with host (pinned) buffers:
          H2D of U, the operator, D2H of the result, inside the timed region.
roofline: dominant kernel (narrow_kernel), FP64-bound: 341 flop/cell
           against a DFMA-loop FP64 peak measured here.
cpu_baseline: the reference's own kernels (oracle/_ref, built from
          /root/reference) composed in 3-D, all host threads, rank 0, N=1.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOP_PER_CELL = 341          # 3 x 112 + 3 + 2
BYTES_PER_CELL = 24          # read U, a; write out (compulsory)
N_CELLS_SIDE = 256


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=4000)
    p.add_argument("--warmup", type=int, default=50)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--n", type=int, default=N_CELLS_SIDE)
    p.add_argument("--kc", type=int, default=0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=20)
    p.add_argument("--no-ns", action="store_true")
    p.add_argument("--no-advance", action="store_true",
                   help="skip the configs[2] SDC / configs[4] MRSDC time-advance blocks")
    p.add_argument("--ns-steps", type=int, default=5)
    p.add_argument("--overlap", action="store_true",
                   help="N>1: interior planes run while the halo is in flight (split launch)")
    p.add_argument("--slab", action="store_true",
                   help="use the multi-GPU z-slab path also at N=1 (ghosts by self-copy)")
    p.add_argument("--halo", choices=["peer", "nccl"], default="nccl",
                   help="slab halo: nccl (default) = send/recv into ghost planes before the "
                        "kernel; peer = the kernel reads the neighbours' planes over CUDA IPC / "
                        "NVLink (falls back to nccl if the mapping fails).  At N=1 the step is "
                        "0.302 ms (nccl) vs 0.311 ms (peer): the peer instantiation's per-plane "
                        "base selection costs more than the 4-plane exchange")
    return p.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU baselines
def cpu_reference_rate(n: int, budget_s: float = 12.0, max_reps: int = 5):
    """The reference's own line kernels composed in 3-D (oracle/_ref), all
    host threads; returns (cells/s, cores, kind, sample)."""
    import numpy as np
    from oracle import oracle as O
    from paper_1309_7327_b200 import workloads as W
    a, u = W.narrow3d_inputs(n)
    m, s = O.build_narrow(8, (3557.0 / 44100.0, -2083.0 / 117600.0))
    if O.have_ref(fast=True):
        r = O.ref(fast=True)
        r.ref_set_workers(0)
        cores = int(r.ref_worker_limit())
        fn = lambda: O.ref_narrow3d(m, s, a, u, 1 / n, 1 / n, 1 / n, fast=True)  # noqa: E731
        kind = "reference"
        sample = f"full {n}^3 box per rep, reference kernels narrow_interfaces<4>/_rows<4> " \
                 f"composed as narrow_rhs_rows (oracle/ref_capi.cpp), parallel_for over z planes"
    else:
        n = min(n, 96)
        a, u = W.narrow3d_inputs(n)
        cores = 1
        fn = lambda: O.narrow3d(m, s, a, u, 1 / n, 1 / n, 1 / n)  # noqa: E731
        kind = "port"
        sample = f"full {n}^3 box per rep, C restatement oracle/oracle.c, 1 thread"
    fn()  # warm-up
    best, spent, reps = math.inf, 0.0, 0
    while reps < max_reps and (spent < budget_s or reps < 1):
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        best = min(best, dt)
        spent += dt
        reps += 1
    return n ** 3 / best, cores, kind, sample + f", best of {reps}", best


def run_reference(args):
    """--impl reference: the reference CPU path on the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.n
    import numpy as np
    from oracle import oracle as O
    from paper_1309_7327_b200 import workloads as W
    if not O.have_ref(fast=True):
        O.build_ref()
    a, u = W.narrow3d_inputs(n)
    m, s = O.build_narrow(8, (3557.0 / 44100.0, -2083.0 / 117600.0))
    have = O.have_ref(fast=True)
    if have:
        r = O.ref(fast=True)
        r.ref_set_workers(0)
        cores = int(r.ref_worker_limit())
        step = lambda: O.ref_narrow3d(m, s, a, u, 1 / n, 1 / n, 1 / n, fast=True)  # noqa: E731
        kind = "reference"
    else:
        cores = 1
        step = lambda: O.narrow3d(m, s, a, u, 1 / n, 1 / n, 1 / n)  # noqa: E731
        kind = "port"
    for _ in range(min(args.warmup, 1)):
        step()
    t_one = None
    times = []
    budget = 120.0
    k = 0
    t_start = time.perf_counter()
    while k < args.steps:
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
        k += 1
        if time.perf_counter() - t_start > budget:
            break
    total = sum(times)
    value = n ** 3 * k / total
    out = {
        "metric": "fp64 cell-RHS evals/sec (narrow operator, configs[1])",
        "value": value, "unit": "cell-RHS/s", "n_gpus": args.gpus, "steps": k,
        "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / k, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"configs[1] narrow operator {n}^3 periodic (CPU reference path)",
                   "cells": n ** 3},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "cell-RHS/s", "cores": cores, "kind": kind,
                         "sample": f"full {n}^3 box per step; {k} steps (time-capped at "
                                   f"{budget:.0f} s)"},
        "e2e": {"value": value, "unit": "cell-RHS/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------- NS secondary
NS_FLOP_PER_CELL = 8850   # frozen algorithmic count, DESIGN.md "NS RHS flop count"
NS_BYTES_PER_CELL = 224   # 14 conserved fp64 in + 14 out (fully fused minimum)
# DRAM bytes per cell-RHS the direction-split design moves (sum over its
# kernels of ncu dram__bytes_read + write at 128^3, profiles/ncu_ns_r01.json:
# prim 452, phase A 3 x 632, mixed 138, phase B 3 x 29, assemble2 738)
NS_DESIGN_BYTES_PER_CELL = 3311


def heat2d_measurement(dev, stream, fp64_peak, n=4096, reps=100):
    """The reference's own RHS (HeatOperator::rhs, pde.cpp:266-274; the 2-D
    T2 problem, narrow SMC stencil) on the GPU at n^2 next to the reference
    CPU path on all host threads (oracle/_ref, operator built once, best of 3
    calls).  Roofline: 2 x 112 + 3 + 2 flop per cell (two directions, the
    1/d^2 scalings and combine), 32 B per cell (u, a, b in; out)."""
    import ctypes as C
    import numpy as np
    import torch
    import paper_1309_7327_b200 as P
    xs = np.arange(n) * (2 * math.pi / n)
    X, Y = np.meshgrid(xs, xs)
    a = 1.0 + 0.9 * np.cos(2 * X) * np.sin(2 * Y + math.pi / 3)
    b = 1.0 + 0.9 * np.cos(2 * X + math.pi / 3) * np.sin(2 * Y)
    u = torch.from_numpy(np.sin(X) * np.sin(Y)).to(dev)
    out = torch.empty_like(u)
    op = P.HeatOperator(n, n, P.StencilChoice.narrow8(P.SMC_M47, P.SMC_M48), a, b)
    op.set_stream(stream)
    for _ in range(5):
        op(0.0, u, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        op(0.0, u, out)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flop = 2 * 112 + 3 + 2
    res = {"workload": f"HeatOperator::rhs, T2 coefficients, narrow SMC, {n}^2 periodic",
           "value": n * n / (ms * 1e-3), "unit": "cell-RHS/s", "ms_per_rhs": ms,
           "roofline": {"bound": "fp64", "achieved": flop * n * n / (ms * 1e-3) / 1e12,
                        "peak": fp64_peak, "unit": "TFLOP/s",
                        "frac": flop * n * n / (ms * 1e-3) / 1e12 / fp64_peak,
                        "flop_per_cell": flop, "bytes_per_cell": 32}}
    try:
        from oracle import oracle as O
        if O.have_ref(fast=True):
            r = O.ref(fast=True)
            r.ref_set_workers(0)
            best = C.c_double()
            pp = np.array([P.SMC_M47, P.SMC_M48])
            rc = r.ref_heat2d_time(2, n, n, 0, O.dp(pp), 3, C.byref(best))
            if rc == 0:
                res["cpu_baseline"] = {"value": n * n / best.value, "unit": "cell-RHS/s",
                                       "cores": int(r.ref_worker_limit()), "kind": "reference",
                                       "sample": f"HeatOperator::rhs at {n}^2, operator built "
                                                 "once, best of 3 calls"}
    except Exception as exc:  # noqa: BLE001
        res["cpu_baseline"] = {"value": None, "sample": f"failed: {exc}"}
    return res


def ns_rhs_measurement(n, dev, stream, fp64_peak, hbm_peak, steps):
    """Full NS RHS (ctoprim, hypterm, narrow diffterm + transport, wdot) on
    the configs[3] state generator (hot spot), n^3 periodic, dx = 1e-4 m."""
    import torch
    import paper_1309_7327_b200 as P
    from paper_1309_7327_b200 import workloads as W
    T, p, uvw, Y = W.ns_primitives(n, hot_spot=True)
    U = P.ns_conserved(*(torch.from_numpy(a).to(dev) for a in (T, p, uvw, Y)))
    del T, p, uvw, Y
    op = P.NsOperator(n, n, n, 1e-4)
    op.set_stream(stream)
    out = torch.empty_like(U)
    op.full(0.0, U, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        op.full(0.0, U, out)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    cells = n ** 3
    tf = NS_FLOP_PER_CELL * cells / (ms * 1e-3) / 1e12
    gbs = NS_BYTES_PER_CELL * cells / (ms * 1e-3) / 1e9
    res = {"workload": f"configs[3] full reacting-NS RHS, {n}^3, hot spot, 9-species synthetic "
                       "mechanism, periodic", "value": cells / (ms * 1e-3),
           "unit": "cell-RHS/s", "ms_per_rhs": ms, "steps": steps,
           "roofline": {"bound": "fp64", "achieved": tf, "peak": fp64_peak, "unit": "TFLOP/s",
                        "frac": tf / fp64_peak, "flop_per_cell": NS_FLOP_PER_CELL,
                        "hbm": {"achieved": gbs, "peak": hbm_peak, "frac": gbs / hbm_peak,
                                "bytes_per_cell": NS_BYTES_PER_CELL},
                        # the traffic this design moves at the HBM peak: how close the
                        # split kernels are to their own memory floor
                        "hbm_design": {"bytes_per_cell": NS_DESIGN_BYTES_PER_CELL,
                                       "floor_ms": NS_DESIGN_BYTES_PER_CELL * cells / hbm_peak / 1e6,
                                       "frac": NS_DESIGN_BYTES_PER_CELL * cells / hbm_peak / 1e6 / ms}}}
    # the oracle (C restatement, 1 thread) on a 24^3 sample of the same generator
    try:
        import time as _t
        from oracle import oracle as O
        Tn, pn, un, Yn = W.ns_primitives(24, hot_spot=True)
        Uh = O.ns_conserved(Tn, pn, un, Yn)
        O.ns_rhs(Uh, 1e-4, 0)
        t0 = _t.perf_counter()
        O.ns_rhs(Uh, 1e-4, 0)
        res["cpu_baseline"] = {"value": 24 ** 3 / (_t.perf_counter() - t0), "unit": "cell-RHS/s",
                               "cores": 1, "kind": "port",
                               "sample": "24^3 box, oracle/ns_oracle.c (no reference NS exists)"}
    except Exception as exc:  # noqa: BLE001
        res["cpu_baseline"] = {"value": None, "kind": "unavailable", "sample": str(exc)}
    del U, out
    torch.cuda.empty_cache()
    return res


def acoustic_dt(T, p, uvw, Y, dx, cfl=0.5):
    """CFL 0.5 on max(|u_i| + c) (the synthetic thermodynamics of
    include/smc_mechanism.h), host side."""
    import numpy as np
    W_ = np.array([2.01588e-3, 31.9988e-3, 18.01528e-3, 1.00794e-3, 15.9994e-3, 17.00734e-3,
                   33.00674e-3, 34.01468e-3, 28.0134e-3])
    a = np.array([[3.40, 1.0e-4, 1.0e-8], [3.30, 6.0e-4, -1.0e-7], [3.60, 9.0e-4, -1.0e-7],
                  [2.50, 0.0, 0.0], [2.60, -1.0e-4, 2.0e-8], [3.50, 1.0e-4, 1.0e-8],
                  [4.00, 1.2e-3, -2.0e-7], [4.50, 2.0e-3, -3.0e-7], [3.25, 5.0e-4, -8.0e-8]])
    Ru = 8.314462618
    cp = sum(Y[k] * Ru / W_[k] * (a[k, 0] + a[k, 1] * T + a[k, 2] * T * T) for k in range(9))
    Rm = sum(Y[k] * Ru / W_[k] for k in range(9))
    c = np.sqrt(cp / (cp - Rm) * Rm * T)
    return cfl * dx / float((np.abs(uvw).max(axis=0) + c).max())


def advance_measurement(dev, stream):
    """configs[2]: 10 SDC steps (3 Gauss-Lobatto nodes, 4 sweeps) at CFL 0.5
    of the configs[0] generator on 128^3; configs[4] (one GPU point): one
    MRSDC mode-1 step (GL(3) coarse advection-diffusion, GL(5) fine
    chemistry per coarse interval) on the ignition state at 128^3; MRSDC
    mode 2 (chemistry implicit on the GL(3) coarse
    nodes through the per-cell block Newton, advection-diffusion explicit on
    the GL(5) fine nodes) on the same state, one step of twice the acoustic
    dt."""
    import torch
    import paper_1309_7327_b200 as P
    from paper_1309_7327_b200 import workloads as W
    n, dx, res = 128, 1e-4, {}
    for name, kw in (("sdc_configs2", {}), ("mrsdc_configs4", {"ignition": True}),
                     ("mrsdc_mode2_implicit_chem", {"ignition": True})):
        T, p, uvw, Y = W.ns_primitives(n, **kw)
        dt = acoustic_dt(T, p, uvw, Y, dx) * (2.0 if "mode2" in name else 1.0)
        U = P.ns_conserved(*(torch.from_numpy(x).to(dev) for x in (T, p, uvw, Y)))
        op = P.NsOperator(n, n, n, dx)
        op.set_stream(stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if name.startswith("sdc"):
            st = P.SdcStepper(3, P.StepControls(4, 0.0))
            st.integrate(op.full, U, 0.0, dt, 1)  # warm-up (buffers)
            torch.cuda.synchronize()
            e0.record(stream)
            out, d = st.integrate(op.full, U, 0.0, 10 * dt, 10)
            e1.record(stream)
            torch.cuda.synchronize()
            steps, evals = 10, d.fresh_evals
        elif "mode2" in name:
            st = P.MrsdcStepper(3, 5, P.StepControls(4, 0.0),
                                stiff=P.StiffOptions(block=14, interleaved=True))
            st.integrate_mode2(op.chem, op.advdiff, U, 0.0, dt, 1)
            torch.cuda.synchronize()
            e0.record(stream)
            out, d = st.integrate_mode2(op.chem, op.advdiff, U, 0.0, dt, 1)
            e1.record(stream)
            torch.cuda.synchronize()
            steps, evals = 1, d.f1_evals + d.f2_evals + d.newton_f1_evals
        else:
            st = P.MrsdcStepper(3, 5, P.StepControls(4, 0.0))
            st.integrate_mode1(op.advdiff, op.chem, U, 0.0, dt, 1)
            torch.cuda.synchronize()
            e0.record(stream)
            out, d = st.integrate_mode1(op.advdiff, op.chem, U, 0.0, dt, 1)
            e1.record(stream)
            torch.cuda.synchronize()
            steps, evals = 1, d.f1_evals + d.f2_evals
        ms = e0.elapsed_time(e1)
        res[name] = {"cells": n ** 3, "steps": steps, "dt_s": dt, "ms_per_step": ms / steps,
                     "rhs_evals": evals, "sweeps": d.sweeps,
                     "final_residual": d.residual_history[-1] if d.residual_history else None,
                     "finite": bool(torch.isfinite(out).all().item())}
        if "mode2" in name:
            res[name].update(implicit_solves=d.implicit_solves, newton_f1_evals=d.newton_f1_evals)
        del U, out, op, st
        torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------- ours
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import paper_1309_7327_b200 as P
    from paper_1309_7327_b200 import _capi, workloads as W
    from paper_1309_7327_b200.distributed import DistributedNarrow3D, Slab
    import ctypes as C

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = args.n
    cells_rank = n ** 3
    cells_total = cells_rank * world
    stream = torch.cuda.current_stream()

    # ---- inputs resident in HBM
    slab_mode = world > 1 or args.slab
    halo = None
    if not slab_mode:
        a, u = W.narrow3d_inputs(n, xp=torch, device=dev)
        op = P.Narrow3DOperator(a, 1 / n, 1 / n, 1 / n)
        op.set_stream(stream)
        if args.kc:
            op.set_kc(args.kc)
        out = torch.empty_like(u)

        def step():
            op(0.0, u, out)
    else:
        slab = Slab(rank, world, n)
        zg = torch.tensor(slab.global_planes(), dtype=torch.float64, device=dev) / n
        x = torch.arange(n, dtype=torch.float64, device=dev) / n
        tw = 2 * math.pi
        a = (1.0 + 0.5 * torch.sin(tw * x).view(1, 1, n) * torch.cos(tw * x).view(1, n, 1)
             * torch.sin(tw * zg).view(-1, 1, 1)).contiguous()
        ks, amps, ph = W.modes()
        u = torch.zeros_like(a)
        for k, A, p in zip(ks, amps, ph):
            u += A * torch.sin(tw * (k[0] * x.view(1, 1, n) + k[1] * x.view(1, n, 1)
                                     + k[2] * zg.view(-1, 1, 1)) + p)
        out = torch.empty((n, n, n), dtype=torch.float64, device=dev)
        halo = args.halo
        if halo == "peer":
            try:
                from paper_1309_7327_b200.distributed import PeerNarrow3D
                pdop = PeerNarrow3D(a, slab, 1 / n, 1 / n, 1 / n, dist if world > 1 else None,
                                    exchange_a=False, sync="nccl")
                for b in pdop.bufs:
                    b.copy_(u[4:4 + n])
            except Exception as exc:  # noqa: BLE001  (a GPU path either way)
                print(f"peer halo unavailable ({exc}); using the NCCL exchange", file=sys.stderr)
                halo = "nccl"
        if halo == "peer":
            if args.kc:
                pdop.op.set_kc(args.kc)
            op = pdop.op
            counter = [0]

            def step():
                pdop.apply(counter[0], out)
                counter[0] += 1
        else:
            dop = DistributedNarrow3D(a, slab, 1 / n, 1 / n, 1 / n, dist, exchange_a=False)
            if args.kc:
                dop.op.set_kc(args.kc)
            op = dop.op

            def step():
                dop.apply(u, out, overlap=args.overlap)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- FP64 peak of this device (roofline denominator)
    peak = C.c_double()
    _capi.check(_capi.lib().smc_measure_fp64_peak(20000, C.byref(peak)))
    fp64_peak = max_over_ranks(peak.value)

    # ---- warm-up + timed region (inputs 403 MB/step per rank > 126 MB L2)
    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    barrier()
    launches0 = P.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    launches = P.launch_count() - launches0
    clocks = sampler.stop()
    ms = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms / args.steps
    value = cells_total * args.steps / (ms * 1e-3)

    # ---- dominant kernel alone (for N > 1 the step also holds the exchange)
    if not slab_mode:
        k_ms = ms_step
    else:
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        k0.record(stream)
        kk = max(10, args.steps // 10)
        for _ in range(kk):
            op.apply_planes(u, out, 0, n)
        k1.record(stream)
        barrier()
        k_ms = max_over_ranks(k0.elapsed_time(k1)) / kk
    achieved_tf = FLOP_PER_CELL * cells_rank / (k_ms * 1e-3) / 1e12
    achieved_gbs = BYTES_PER_CELL * cells_rank / (k_ms * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_narrow3d.json")))
        traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass

    # ---- e2e through the public API with host buffers
    e2e_steps = max(3, min(args.e2e_steps, args.steps))
    if not slab_mode:
        uh = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
        oh = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
        uh.copy_(u.cpu())

        def e2e_step():
            op(0.0, uh, oh)          # H2D, kernel, D2H, synchronize (smc_rhs_eval, SMC_HOST)
    else:
        uh = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
        oh = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
        uh.copy_(u[4:4 + n].cpu())

        if halo == "peer":
            def e2e_step():
                i = counter[0]
                pdop.buffer(i).copy_(uh, non_blocking=True)
                pdop.apply(i, out)
                counter[0] += 1
                oh.copy_(out, non_blocking=True)
                torch.cuda.current_stream().synchronize()
        else:
            def e2e_step():
                u[4:4 + n].copy_(uh, non_blocking=True)
                dop.apply(u, out, overlap=args.overlap)
                oh.copy_(out, non_blocking=True)
                torch.cuda.current_stream().synchronize()
    e2e_step()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    f1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1)) / e2e_steps
    e2e_value = cells_total / (e2e_ms * 1e-3)

    # ---- secondary: the full reacting-NS RHS (configs[3] state, this GPU's block)
    ns = None
    if not args.no_ns and world == 1:
        try:
            ns = ns_rhs_measurement(n, dev, stream, fp64_peak, hbm_peak, args.ns_steps)
        except Exception as exc:  # noqa: BLE001
            ns = {"error": str(exc)}

    heat = None
    if not args.no_ns and world == 1:
        try:
            heat = heat2d_measurement(dev, stream, fp64_peak)
        except Exception as exc:  # noqa: BLE001
            heat = {"error": str(exc)}

    adv = None
    if not args.no_advance and world == 1:
        try:
            adv = advance_measurement(dev, stream)
        except Exception as exc:  # noqa: BLE001
            adv = {"error": str(exc)}

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            v, cores, kind, sample, best = cpu_reference_rate(n)
            cpu = {"value": v, "unit": "cell-RHS/s", "cores": cores, "kind": kind,
                   "sample": sample}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "cell-RHS/s", "cores": 0, "kind": "unavailable",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": "fp64 cell-RHS evals/sec (narrow operator, configs[1])",
            "value": value, "unit": "cell-RHS/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": f"configs[1] narrow 8th-order (a U_x)_x+(a U_y)_y+(a U_z)_z, "
                            f"{n}^3 per GPU, periodic" +
                            ("" if not slab_mode else f", z-slabs of a {n}x{n}x{n * world} box, "
                                                      + ("4-plane halo read by the kernel over peer memory (CUDA IPC / NVLink)"
                                                         if halo == "peer" else
                                                         "4-plane NCCL halo" + (", overlapped" if args.overlap else ""))),
                "cells_per_gpu": cells_rank, "stencil": "SMC (m47=3557/44100, m48=-2083/117600)",
                "l2": f"inputs larger than L2 ({(2 * 8 * cells_rank) / 1e6:.0f} MB read + "
                      f"{8 * cells_rank / 1e6:.0f} MB written per step per GPU)",
                "kc": args.kc or "heuristic",
            },
            "roofline": {
                "bound": "fp64", "achieved": achieved_tf, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": achieved_tf / fp64_peak, "traffic": traffic,
                "peak_source": "DFMA-loop peak measured in this run (smc_measure_fp64_peak); "
                               "MEASURED_PEAKS.json has no FP64 figure",
                "flop_per_cell": FLOP_PER_CELL, "kernel_ms": k_ms,
                "hbm": {"achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                        "frac": achieved_gbs / hbm_peak, "bytes_per_cell": BYTES_PER_CELL},
            },
            "e2e": {"value": e2e_value, "unit": "cell-RHS/s",
                    "h2d_bytes_per_step": 8 * cells_rank, "d2h_bytes_per_step": 8 * cells_rank,
                    "ms_per_step": e2e_ms},
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "ns_rhs": ns,
            "heat2d_rhs": heat,
            "time_advance": adv,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
