"""the narrow vs wide route on B200 against the paper's
cost model (costmodel.hpp:9-43).

Times one heat-operator RHS (T2 coefficients, no source) with the narrow8 and
the wide8 stencils at n x n on cuda:0 with CUDA events, and the 3-D narrow
operator for reference, then evaluates the model with this box's measured
FP64 peak and HBM bandwidth: narrow pays 112N+111 - (23N+8) extra flops per
point, wide streams 64 extra bytes per point (N = 1 for the heat equation).
"model_fused_wide" is the same comparison for a single-pass wide kernel (no
temporaries: both routes move 32 B per point).  Prints one JSON object;
profiles/cost_model_r0*.json keep runs."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_7327_b200 as P  # noqa: E402


def timed(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    xs = np.arange(n) * (2 * math.pi / n)
    X, Y = np.meshgrid(xs, xs)
    a = 1.0 + 0.9 * np.cos(2 * X) * np.sin(2 * Y + math.pi / 3)
    b = 1.0 + 0.9 * np.cos(2 * X + math.pi / 3) * np.sin(2 * Y)
    u = torch.from_numpy(np.sin(X) * np.sin(Y)).cuda()
    out = torch.empty_like(u)
    res = {"grid": f"{n}^2", "points": n * n}
    for name, choice in (("narrow8", P.StencilChoice.narrow8(P.SMC_M47, P.SMC_M48)),
                         ("wide8", P.StencilChoice.wide8())):
        op = P.HeatOperator(n, n, choice, a, b)
        t = timed(lambda: op(0.0, u, out))
        res[name] = {"s_per_rhs": t, "ns_per_point": t / (n * n) * 1e9}
    import ctypes as C
    from paper_1309_7327_b200 import _capi
    v = (C.c_double * 5)()
    _capi.check(_capi.lib().smc_measure_fp64_variants(4000, v, 5))
    dm = C.c_double()
    _capi.check(_capi.lib().smc_measure_dmma_peak(4000, 0, C.byref(dm)))
    peak = max(list(v) + [dm.value])
    bw = 6531.9e9
    try:
        bw = json.load(open(os.path.join(os.path.dirname(__file__), "..",
                                         "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
    except Exception:
        pass
    flops = peak * 1e12 if peak else 34.2e12
    N = 1
    narrow_f, wide_f = 112 * N + 111, 23 * N + 8
    model_delta = (narrow_f - wide_f) / flops - 64.0 / bw
    res["model"] = {"N": N, "narrow_flops": narrow_f, "wide_flops": wide_f,
                    "machine_flops": flops, "machine_bandwidth": bw,
                    "time_delta_ns_per_point": model_delta * 1e9,
                    "crossover_bandwidth_GBs": 64.0 * flops / (narrow_f - wide_f) / 1e9}
    res["measured_delta_ns_per_point"] = (res["narrow8"]["ns_per_point"] -
                                          res["wide8"]["ns_per_point"])
    # the same machine with a single-pass (fused) wide route: no temporaries,
    # both routes move 32 B per point, each bound by its own roofline
    t_n = max(32.0 / bw, narrow_f / flops)
    t_w = max(32.0 / bw, wide_f / flops)
    res["model_fused_wide"] = {"narrow_ns_per_point": t_n * 1e9, "wide_ns_per_point": t_w * 1e9,
                               "time_delta_ns_per_point": (t_n - t_w) * 1e9}
    # the single-pass wide kernel's HBM floor: u, a, b in, out written
    res["wide8"]["hbm_floor_s"] = 32.0 * n * n / bw
    res["wide8"]["hbm_frac"] = res["wide8"]["hbm_floor_s"] / res["wide8"]["s_per_rhs"]
    res["narrow8"]["fp64_frac"] = (2 * 112 + 3 + 2) * n * n / flops / res["narrow8"]["s_per_rhs"]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
