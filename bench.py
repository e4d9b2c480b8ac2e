#!/usr/bin/env python
"""bench.py -- fp64 cell-RHS evaluations per second of the full reacting
Navier-Stokes right-hand side (ctoprim, hypterm, narrow-stencil diffterm with
transport, wdot): BASELINE.json's metric on its configs[3] workload, 256^3
cells per GPU, weak scaling over z-slabs of one periodic box with the 4-plane
halo exchanged by NCCL inside the library, overlapped with the interior work.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one full RHS evaluation over the whole job's box (every rank
its 256^3 slab).
value    = cells of all ranks / max-over-ranks device time of K steps.
e2e      = the same metric through the public API with host (pinned) buffers:
           the state H2D, the RHS, the result D2H inside the timed region.
roofline = the whole RHS (the frozen 8,850 flop per cell-RHS, DESIGN.md
           §4.3) against the best FP64 probe measured in this run (DFMA
           variants and DMMA, all reported); `kernels` = one evaluation
           timed per kernel with CUDA events; `traffic` = the ncu DRAM bytes
           of one RHS (profiles/ncu_ns_r02.json).
cpu_baseline = the CPU restatement of the same RHS (oracle/ns_oracle.c,
           OpenMP over every host thread) on the full 256^3 box, rank 0, N=1.
--impl reference times that CPU path alone on the same config (no reference
NS implementation exists: SURVEY.md §0).  Secondary blocks at N=1: configs[1]
(the narrow operator, with the reference's own kernels as its CPU path),
the 2-D heat RHS (the reference's HeatOperator), and the configs[2]/[4]
time advances with their CPU baselines.
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

NS_FLOP_PER_CELL = 8850   # frozen algorithmic count
NS_BYTES_PER_CELL = 224   # compulsory: 14 conserved fp64 in + 14 out
NS_DX = 1e-4
NARROW_FLOP_PER_CELL = 341   # 3 x 112 + 3 + 2
NARROW_BYTES_PER_CELL = 24   # read U, a; write out
METRIC = "fp64 cell-RHS evals/sec (full reacting-NS RHS, configs[3])"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--n", type=int, default=256, help="cells per side per GPU")
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the configs[1] / heat / time-advance blocks")
    p.add_argument("--no-advance", action="store_true")
    p.add_argument("--narrow-steps", type=int, default=2000)
    p.add_argument("--slab", action="store_true",
                   help="N=1: run the library's NCCL slab path (self halo) instead of the "
                        "periodic operator")
    p.add_argument("--workload", choices=["rhs", "mrsdc"], default="rhs",
                   help="rhs: configs[3] (default, weak scaling); mrsdc: configs[4], MRSDC "
                        "mode 1 on a fixed n_global^3 box over the ranks (strong scaling)")
    p.add_argument("--n-global", type=int, default=512, help="mrsdc: global box side")
    p.add_argument("--mrsdc-steps", type=int, default=20)
    return p.parse_args()


def ns_config(n: int, world: int) -> dict:
    """The workload, identical in both arms."""
    return {
        "workload": f"configs[3] full reacting-NS RHS (ctoprim, hypterm, narrow diffterm + "
                    f"transport, wdot), {n}^3 cells per GPU",
        "box": f"{n}x{n}x{n * world} periodic" + (f", z-slabs of {n} planes per GPU, 4-plane "
                                                  "NCCL halo overlapped" if world > 1 else ""),
        "cells_per_gpu": n ** 3,
        "state": "seeded configs[0] generator + Gaussian hot spot (T peak 1800 K, radius 20 "
                 "cells), 9-species synthetic mechanism, dx = 1e-4 m",
        "stencil": "narrow SMC (m47=3557/44100, m48=-2083/117600)",
        "l2": f"inputs larger than L2 ({14 * 8 * n ** 3 / 1e9:.2f} GB state per GPU), no flush",
    }


class stdout_to_stderr:
    """NCCL may print its version banner on stdout at communicator creation;
    rank 0's stdout carries exactly one JSON line, so route fd 1 to fd 2
    meanwhile."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def cpu_info() -> dict:
    model, threads = None, os.cpu_count()
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"model": model, "threads": threads}


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


# ------------------------------------------------------------- FP64 peaks
def fp64_peaks(max_over_ranks) -> dict:
    """The FP64 roofline denominator: the best of the DFMA probe variants
    (chains per thread, operand placement, warps per SM) and the DMMA probe
    (mma.sync f64 shares the FP64 pipe on B200), clocks sampled meanwhile."""
    import ctypes as C
    from paper_1309_7327_b200 import _capi
    L = _capi.lib()
    sampler = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    sampler.start()
    time.sleep(0.2)
    v = (C.c_double * 5)()
    _capi.check(L.smc_measure_fp64_variants(4000, v, 5))
    dm = C.c_double()
    _capi.check(L.smc_measure_dmma_peak(4000, 0, C.byref(dm)))
    clocks = sampler.stop()
    names = ["dfma_8chains", "dfma_16chains", "dfma_8chains_own_multiplier",
             "dfma_8chains_const_operands", "dfma_const_operands_half_warps"]
    probes = {nm: max_over_ranks(x) for nm, x in zip(names, list(v))}
    probes["dmma_m8n8k4"] = max_over_ranks(dm.value)
    best = max(probes, key=probes.get)
    return {"peak": probes[best], "best": best, "probes": probes, "clocks": clocks}


# ------------------------------------------------------------ CPU baselines
def cpu_ns_rate(n: int):
    """The NS RHS restated on the CPU (oracle/ns_oracle.c), every host thread,
    on the full n^3 box (one evaluation after a warm-up on a small box), plus
    one thread on a 64^3 sample."""
    from oracle import oracle as O
    from paper_1309_7327_b200 import workloads as W
    threads = O.set_threads(0)
    U = O.ns_conserved(*W.ns_primitives(n, hot_spot=True))
    Us = O.ns_conserved(*W.ns_primitives(32, hot_spot=True))
    O.ns_rhs(Us, NS_DX, 0)
    t0 = time.perf_counter()
    O.ns_rhs(U, NS_DX, 0)
    dt = time.perf_counter() - t0
    O.set_threads(1)
    U64 = O.ns_conserved(*W.ns_primitives(64, hot_spot=True))
    t1 = time.perf_counter()
    O.ns_rhs(U64, NS_DX, 0)
    one = 64 ** 3 / (time.perf_counter() - t1)
    O.set_threads(0)
    return {"value": n ** 3 / dt, "unit": "cell-RHS/s", "cores": threads, "kind": "port",
            "sample": f"one full {n}^3 RHS (configs[3] state), oracle/ns_oracle.c with OpenMP "
                      f"over {threads} host threads; no reference NS implementation exists "
                      "(SURVEY.md §0)",
            "one_thread": {"value": one, "unit": "cell-RHS/s", "sample": "64^3 box, 1 thread"},
            "cpu": cpu_info()}


def run_reference(args):
    """--impl reference: the CPU path of the same RHS on the same config
    (rank 0 only), every host thread, each step one full per-GPU block."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_1309_7327_b200 import workloads as W
    n = args.n
    threads = O.set_threads(0)
    U = O.ns_conserved(*W.ns_primitives(n, hot_spot=True))
    Us = O.ns_conserved(*W.ns_primitives(32, hot_spot=True))
    for _ in range(max(1, min(args.warmup, 1))):
        O.ns_rhs(Us, NS_DX, 0)
    times, budget = [], 150.0
    t_start = time.perf_counter()
    while len(times) < args.steps:
        t0 = time.perf_counter()
        O.ns_rhs(U, NS_DX, 0)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget:
            break
    k = len(times)
    total = sum(times)
    value = n ** 3 * k / total
    sample = (f"{k} full {n}^3 RHS evaluations (one per-GPU block per step; time-capped at "
              f"{budget:.0f} s), oracle/ns_oracle.c with OpenMP over {threads} host threads")
    out = {
        "metric": METRIC, "value": value, "unit": "cell-RHS/s", "n_gpus": world, "steps": k,
        "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / k,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": ns_config(n, world), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "cell-RHS/s", "cores": threads, "kind": "port",
                         "sample": sample, "cpu": cpu_info()},
        "e2e": {"value": value, "unit": "cell-RHS/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------- secondary: configs[1]
def narrow_block(dev, stream, peak, steps):
    """configs[1]: the narrow operator alone, 256^3 periodic, with its own
    roofline (341 flop / 24 B per cell), e2e and the reference's own kernels
    composed in 3-D as its CPU path (oracle/_ref, every host thread)."""
    import torch
    import paper_1309_7327_b200 as P
    from paper_1309_7327_b200 import workloads as W
    n = 256
    a, u = W.narrow3d_inputs(n, xp=torch, device=dev)
    op = P.Narrow3DOperator(a, 1 / n, 1 / n, 1 / n)
    op.set_stream(stream)
    out = torch.empty_like(u)
    for _ in range(20):
        op(0.0, u, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        op(0.0, u, out)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    tf = NARROW_FLOP_PER_CELL * n ** 3 / (ms * 1e-3) / 1e12
    gbs = NARROW_BYTES_PER_CELL * n ** 3 / (ms * 1e-3) / 1e9
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_narrow3d.json"))).get(
            "dram_bytes_per_launch")
    except Exception:
        pass
    uh = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
    oh = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
    uh.copy_(u.cpu())
    op(0.0, uh, oh)
    t0 = time.perf_counter()
    for _ in range(5):
        op(0.0, uh, oh)  # H2D, kernel, D2H, synchronize (smc_rhs_eval, SMC_HOST)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / 5
    res = {"workload": "configs[1] narrow 8th-order (a U_x)_x+(a U_y)_y+(a U_z)_z, 256^3 "
                       "periodic, SMC stencil", "value": n ** 3 / (ms * 1e-3),
           "unit": "cell-RHS/s", "ms_per_step": ms, "steps": steps,
           "roofline": {"bound": "fp64", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                        "frac": tf / peak, "traffic": traffic,
                        "flop_per_cell": NARROW_FLOP_PER_CELL,
                        "hbm": {"achieved": gbs, "bytes_per_cell": NARROW_BYTES_PER_CELL}},
           "e2e": {"value": n ** 3 / (e2e_ms * 1e-3), "unit": "cell-RHS/s",
                   "h2d_bytes_per_step": 8 * n ** 3, "d2h_bytes_per_step": 8 * n ** 3,
                   "ms_per_step": e2e_ms}}
    try:
        from oracle import oracle as O
        if not O.have_ref(fast=True):
            O.build_ref()
        if O.have_ref(fast=True):
            ah, uhn = W.narrow3d_inputs(n)
            m, s = O.build_narrow(8, (3557.0 / 44100.0, -2083.0 / 117600.0))
            r = O.ref(fast=True)
            r.ref_set_workers(0)
            O.ref_narrow3d(m, s, ah, uhn, 1 / n, 1 / n, 1 / n, fast=True)
            best = math.inf
            for _ in range(3):
                t0 = time.perf_counter()
                O.ref_narrow3d(m, s, ah, uhn, 1 / n, 1 / n, 1 / n, fast=True)
                best = min(best, time.perf_counter() - t0)
            res["cpu_baseline"] = {"value": n ** 3 / best, "unit": "cell-RHS/s",
                                   "cores": int(r.ref_worker_limit()), "kind": "reference",
                                   "sample": "full 256^3 box, the reference's narrow_interfaces"
                                             "<4>/_rows<4> composed as narrow_rhs_rows "
                                             "(oracle/ref_capi.cpp), best of 3"}
    except Exception as exc:  # noqa: BLE001
        res["cpu_baseline"] = {"value": None, "sample": f"failed: {exc}"}
    del a, u, out
    torch.cuda.empty_cache()
    return res


def hbm_peak_gbs() -> float:
    """MEASURED_PEAKS.json's HBM copy bandwidth (driver-written), else the
    profiling recipe's fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def heat2d_block(dev, stream, peak, n=4096, reps=100):
    """The reference's own RHS (HeatOperator::rhs, pde.cpp:266-274; T2, narrow
    SMC) at n^2, next to the reference CPU path on every host thread."""
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
                        "peak": peak, "unit": "TFLOP/s",
                        "frac": flop * n * n / (ms * 1e-3) / 1e12 / peak,
                        "flop_per_cell": flop, "bytes_per_cell": 32}}
    # the same RHS through the wide stencil (the paper's alternative route,
    # HBM-bound: u, a, b read and the result written once, 32 B per cell)
    wop = P.HeatOperator(n, n, P.StencilChoice.wide8(), a, b)
    wop.set_stream(stream)
    for _ in range(5):
        wop(0.0, u, out)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        wop(0.0, u, out)
    e1.record(stream)
    torch.cuda.synchronize()
    wms = e0.elapsed_time(e1) / reps
    hbm = hbm_peak_gbs()
    res["wide_route"] = {"ms_per_rhs": wms, "value": n * n / (wms * 1e-3), "unit": "cell-RHS/s",
                         "roofline": {"bound": "hbm", "achieved": 32 * n * n / (wms * 1e-3) / 1e9,
                                      "peak": hbm, "unit": "GB/s",
                                      "frac": 32 * n * n / (wms * 1e-3) / 1e9 / hbm,
                                      "bytes_per_cell": 32}}
    try:
        from oracle import oracle as O
        if O.have_ref(fast=True):
            r = O.ref(fast=True)
            r.ref_set_workers(0)
            best = C.c_double()
            pp = np.array([P.SMC_M47, P.SMC_M48])
            if r.ref_heat2d_time(2, n, n, 0, O.dp(pp), 3, C.byref(best)) == 0:
                res["cpu_baseline"] = {"value": n * n / best.value, "unit": "cell-RHS/s",
                                       "cores": int(r.ref_worker_limit()), "kind": "reference",
                                       "sample": f"HeatOperator::rhs at {n}^2, best of 3"}
    except Exception as exc:  # noqa: BLE001
        res["cpu_baseline"] = {"value": None, "sample": f"failed: {exc}"}
    return res


def acoustic_dt(T, p, uvw, Y, dx, cfl=0.5):
    """CFL 0.5 on max(|u_i| + c) (include/smc_mechanism.h thermodynamics)."""
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


def advance_block(dev, stream, cpu: bool):
    """configs[2]: SDC (3 Gauss-Lobatto nodes, 4 sweeps) at CFL 0.5 of the
    configs[0] state, 10 steps at 128^3; configs[4] (one-GPU point): MRSDC
    mode 1 (GL(3) advection-diffusion, GL(5) chemistry per coarse interval)
    on the ignition state at 128^3, one step; MRSDC mode 2 (chemistry
    implicit through the per-cell block Newton) on the same state.  CPU
    baselines: one step of the oracle's SDC and MRSDC restatements driving
    the threaded NS oracle on the same 128^3 states."""
    import numpy as np
    import torch
    import paper_1309_7327_b200 as P
    from paper_1309_7327_b200 import workloads as W
    n, res = 128, {}
    for name, kw in (("sdc_configs2", {}), ("mrsdc_configs4", {"ignition": True}),
                     ("mrsdc_mode2_implicit_chem", {"ignition": True})):
        T, p, uvw, Y = W.ns_primitives(n, **kw)
        dt = acoustic_dt(T, p, uvw, Y, NS_DX) * (2.0 if "mode2" in name else 1.0)
        U = P.ns_conserved(*(torch.from_numpy(x).to(dev) for x in (T, p, uvw, Y)))
        op = P.NsOperator(n, n, n, NS_DX)
        op.set_stream(stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if name.startswith("sdc"):
            st = P.SdcStepper(3, P.StepControls(4, 0.0))
            st.integrate(op.full, U, 0.0, dt, 1)
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
        if cpu and "mode2" not in name:
            try:
                from oracle import oracle as O
                threads = O.set_threads(0)
                Uh = U.cpu().numpy()
                shape = Uh.shape
                t0 = time.perf_counter()
                if name.startswith("sdc"):
                    q, s = P.integration_matrices(0, 3)
                    O.integrate_sdc(O.ns_callback(shape, NS_DX, 0), Uh, 0.0, dt, 1, P.nodes(0, 3),
                                    q, s)
                else:
                    h = P.build_hierarchy(3, 5)
                    h["coarse"] = P.nodes(0, 3)
                    O.integrate_mrsdc1(O.ns_callback(shape, NS_DX, 1),
                                       O.ns_callback(shape, NS_DX, 2), Uh, 0.0, dt, 1, h)
                cpu_ms = (time.perf_counter() - t0) * 1e3
                res[name]["cpu_baseline"] = {
                    "ms_per_step": cpu_ms, "cores": threads, "kind": "port",
                    "sample": f"one step at {n}^3: the oracle's integrator restatement "
                              "(oracle.c) driving the threaded NS oracle",
                    "speedup": cpu_ms / (ms / steps)}
            except Exception as exc:  # noqa: BLE001
                res[name]["cpu_baseline"] = {"ms_per_step": None, "sample": f"failed: {exc}"}
        del U, out, op, st
        torch.cuda.empty_cache()
    return res


# ------------------------------------------------- configs[4]: MRSDC strong
def run_mrsdc(args):
    """configs[4]: MRSDC mode 1 (GL(3) coarse nodes for advection-diffusion,
    GL(5) fine nodes for the chemistry per coarse interval, 4 sweeps) on the
    stiff ignition state (1500 K kernel in 600 K H2/air, phi = 1) of an
    n_global^3 periodic box split into z-slabs over the ranks, 20 steps at
    CFL 0.5.  Strong scaling: the box is fixed.  The device stepper advances
    each rank's slab with the library's slab RHS (NCCL halo) and reduces the
    residual over the ranks in the library.  Device memory per cell: the
    MRSDC mode-1 stepper holds 43 states of 14 fields (9 fine-node values,
    F1 and F2 double-buffered, 8 node integrals, carries) plus the state and
    the result, the NS workspace 78 fields: ~5.7 KB per cell, ~760 GB for
    512^3, so the 512^3 series starts at 8 GPUs."""
    import torch
    import torch.distributed as dist
    import paper_1309_7327_b200 as P
    from paper_1309_7327_b200 import workloads as W
    from paper_1309_7327_b200.distributed import Comm, NsSlab
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ng = args.n_global
    nz = ng // world
    cells_local = ng * ng * nz
    need = 8.0 * (14 * (43 + 2) + 78) * cells_local
    free, _ = torch.cuda.mem_get_info(dev)
    base = {"metric": f"configs[4] MRSDC mode-1 cell-steps/sec ({ng}^3, strong scaling)",
            "unit": "cell-steps/s", "n_gpus": world, "higher_is_better": True,
            "scaling": "strong", "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"configs[4] MRSDC GL(3)/GL(5) mode 1, K=4, ignition state, "
                                   f"{ng}^3 periodic, z-slabs of {nz} planes", "cells": ng ** 3}}
    if ng % world or nz < 8 or need > 0.97 * free:
        if rank == 0:
            base["unavailable"] = (f"{ng}^3 over {world} GPU(s): {nz} planes per rank need "
                                   f"~{need / 1e9:.0f} GB of device memory, {free / 1e9:.0f} GB "
                                   "free" if need > 0.97 * free else "box does not split")
            print(json.dumps(base), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    T, p, uvw, Y = W.ns_primitives(ng, nz=nz, z0=rank * nz, nz_global=ng, ignition=True)
    dt = acoustic_dt(T, p, uvw, Y, NS_DX)
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        dt = float(t.item())
    U = P.ns_conserved(*(torch.from_numpy(a).to(dev) for a in (T, p, uvw, Y)))
    del T, p, uvw, Y
    with stdout_to_stderr():
        comm = Comm.nccl(dist if world > 1 else None, device=dev)
    slab = NsSlab(comm, ng, ng, nz, NS_DX)
    stream = torch.cuda.current_stream()
    slab.set_stream(stream)
    st = P.MrsdcStepper(3, 5, P.StepControls(4, 0.0))
    st.set_comm(comm)
    out = torch.empty_like(U)
    st.integrate_mode1(slab.advdiff, slab.chem, U, 0.0, dt, 1, out=out)  # buffers, warm-up
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = args.mrsdc_steps
    e0.record(stream)
    out, d = st.integrate_mode1(slab.advdiff, slab.chem, U, 0.0, steps * dt, steps, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    finite = bool(torch.isfinite(out).all().item())
    if rank == 0:
        base.update({"value": ng ** 3 * steps / (ms * 1e-3), "steps": steps,
                     "ms_per_step": ms / steps, "dt_s": dt, "sweeps": d.sweeps,
                     "f1_evals": d.f1_evals, "f2_evals": d.f2_evals,
                     "final_residual": d.residual_history[-1] if d.residual_history else None,
                     "finite": finite, "vs_baseline": None})
        print(json.dumps(base), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------- ours
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.workload == "mrsdc":
        run_mrsdc(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1309_7327_b200 as P
    from paper_1309_7327_b200 import workloads as W
    from paper_1309_7327_b200.distributed import Comm, NsSlab

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

    # ---- this rank's state, resident in HBM (slab z0 = rank * n of the box)
    T, p, uvw, Y = W.ns_primitives(n, nz=n, z0=rank * n, nz_global=n * world, hot_spot=True)
    U = P.ns_conserved(*(torch.from_numpy(a).to(dev) for a in (T, p, uvw, Y)))
    del T, p, uvw, Y
    out = torch.empty_like(U)
    slab_mode = world > 1 or args.slab
    if slab_mode:
        with stdout_to_stderr():
            comm = Comm.nccl(dist if world > 1 else None, device=dev)
        op = NsSlab(comm, n, n, n, NS_DX)
    else:
        op = P.NsOperator(n, n, n, NS_DX)
    op.set_stream(stream)

    def step():
        op.full(0.0, U, out)

    peaks = fp64_peaks(max_over_ranks)
    peak = peaks["peak"]

    # ---- warm-up + timed region (1.9 GB state per rank > 126 MB L2)
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

    # ---- per-kernel times of one evaluation (periodic operator view)
    kernels = None
    if not slab_mode:
        prof = op.profile(U, out)
        tot = sum(t for _, t in prof)
        kernels = {"ms": {f"{i:02d}_{k}": t for i, (k, t) in enumerate(prof)},
                   "sum_ms": tot,
                   "phase_a_share": sum(t for k, t in prof if k.startswith("phase_a")) / tot}

    tf = NS_FLOP_PER_CELL * cells_rank / (ms_step * 1e-3) / 1e12
    gbs = NS_BYTES_PER_CELL * cells_rank / (ms_step * 1e-3) / 1e9
    traffic = None
    try:
        nprof = json.load(open(os.path.join(ROOT, "profiles", "ncu_ns_r02.json")))
        traffic = nprof["dram_bytes_per_cell_rhs"] * cells_rank
    except Exception:
        pass
    meas = {}
    try:
        meas = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = meas.get("hbm_gbs", hbm_peak_gbs())

    # ---- e2e through the public API with host (pinned) buffers
    Uh = torch.empty(U.shape, dtype=torch.float64).pin_memory()
    Oh = torch.empty(U.shape, dtype=torch.float64).pin_memory()
    Uh.copy_(U.cpu())
    e2e_steps = max(1, args.e2e_steps)

    def e2e_step():  # smc_rhs_eval with SMC_HOST buffers: the library's host pipeline
        op.full(0.0, Uh, Oh)
    e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    barrier()
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / e2e_steps)
    e2e_value = cells_total / (e2e_ms * 1e-3)
    del Uh, Oh

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_ns_rate(n)
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "cell-RHS/s", "cores": 0, "kind": "unavailable",
                   "sample": f"failed: {exc}"}

    secondary = {}
    if world == 1 and not args.no_secondary:
        del U, out
        torch.cuda.empty_cache()
        for key, fn in (("narrow_configs1", lambda: narrow_block(dev, stream, peak,
                                                                 args.narrow_steps)),
                        ("heat2d_rhs", lambda: heat2d_block(dev, stream, peak)),
                        ("time_advance", lambda: None if args.no_advance else
                         advance_block(dev, stream, not args.no_cpu_baseline))):
            try:
                secondary[key] = fn()
            except Exception as exc:  # noqa: BLE001
                secondary[key] = {"error": str(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cell-RHS/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": ns_config(n, world),
            "roofline": {
                "bound": "fp64", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                "frac": tf / peak, "traffic": traffic,
                "scope": "the whole RHS (its kernels in sequence), 8,850 flop per cell-RHS",
                "peak_source": f"best FP64 probe measured in this run ({peaks['best']}); "
                               "MEASURED_PEAKS.json has no FP64 figure",
                "probes_tflops": peaks["probes"], "probe_clocks": peaks["clocks"],
                "flop_per_cell": NS_FLOP_PER_CELL,
                "hbm": {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                        "frac": gbs / hbm_peak, "bytes_per_cell": NS_BYTES_PER_CELL},
            },
            "kernels": kernels,
            "e2e": {"value": e2e_value, "unit": "cell-RHS/s",
                    "h2d_bytes_per_step": 14 * 8 * cells_rank,
                    "d2h_bytes_per_step": 14 * 8 * cells_rank, "ms_per_step": e2e_ms},
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        line.update(secondary)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
