"""Generates tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libnsdc_ref.so, built from /root/reference/proj/core sources with
-ffp-contract=off by oracle/Makefile).  Run here (the reference does not exist
on the GPU box):  python tests/golden/gen_golden.py

Contents (all fp64):
  m8_smc, m8_zero, m8_optimal, m6_default   build_narrow (stencil.cpp:117-132)
  n3d_a, n3d_u, n3d_out                      oracle3d composition of the reference
                                             kernels (ref_capi.cpp) on a seeded 16^3 box
  heat_<pid>_<kind>_u / _out                 HeatOperator::rhs at t=0.3 on 24x20
                                             (pid 1=T1, 2=T2, 3=x-only; kind 0/1/2)
  sdc_t2_u0 / _u / _res / _meta              integrate_sdc, T2, SMC, 32^2, GL(3), K=4,
                                             cutoff 0, 10 steps at appendix_dt
  mr_u0 / mr_u / mr_res / mr_meta            integrate_mrsdc mode 1, dim 3 linear split
                                             problem, GL(3) / TypeB GL(5), K=4, 4 steps
  m2_<case>_u0 / _u / _res / _meta           integrate_mrsdc mode 2 (f1 implicit, dense
                                             FD-Jacobian Newton): osc = Prothero-Robinson
                                             sigma 1e4, GL(3)/TypeB GL(5), K=6, 5 steps of
                                             0.02, rtol 1e-12 atol 1e-13; rob = 4 Robertson
                                             cells (tests/mode2_problems.py), K=4, 5 steps
                                             of 0.01; oscc = sigma 1e3, GL(5)/TypeC{GL(3),2},
                                             K=4, 2 steps of 0.01.  meta = sweeps, f1, f2,
                                             implicit solves, Newton f1 evals
  st_<case>_u0 / _u                          integrate_stiff: rob1 = one Robertson cell
                                             to t = 1, rob4 = four interleaved cells to
                                             t = 0.5 (rtol 1e-6), osc = sigma 1e4 forced
                                             oscillator (f1 + f2) to t = 1
  q_gl3, s_gl3, q_gl5, s_gl5, nodes_gl9,     quadrature tables
  q_cc5, s_cc5, h_*                          build_hierarchy(GL3, TypeB GL5)
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1309_7327_b200 import workloads  # noqa: E402

SMC = (3557.0 / 44100.0, -2083.0 / 117600.0)
OPT = (1059283.0 / 13608000.0, -856481.0 / 40824000.0)
M36 = (281.0 / 3600.0,)


def ref_m(order, params):
    p = np.array(params, dtype=np.float64)
    m = np.zeros(64)
    s = C.c_int()
    assert O.ref().ref_build_narrow(order, O.dp(p), len(p), O.dp(m), C.byref(s)) == 0
    return m, s.value


def main():
    assert O.build_ref(), "reference library unavailable"
    g = {}
    g["m8_smc"], _ = ref_m(8, SMC)
    g["m8_zero"], _ = ref_m(8, (0.0, 0.0))
    g["m8_optimal"], _ = ref_m(8, OPT)
    g["m6_default"], _ = ref_m(6, M36)

    n = 16
    a, u = workloads.narrow3d_inputs(n, seed=7)
    g["n3d_a"], g["n3d_u"] = a, u
    g["n3d_out"] = O.ref_narrow3d(g["m8_smc"], 4, a, u, 1.0 / n, 1.0 / n, 1.0 / n)

    nx, ny = 24, 20
    for pid in (1, 2, 3):
        A, B, G, U0 = O.ref_heat2d_fields(pid, nx, ny)
        for kind, params in ((0, SMC), (1, M36), (2, ())):
            g[f"heat_{pid}_{kind}_u"] = U0
            g[f"heat_{pid}_{kind}_out"] = O.ref_heat2d_rhs(pid, kind, params, 0.3, U0)
        g[f"heat_{pid}_a"], g[f"heat_{pid}_b"], g[f"heat_{pid}_g0"] = A, B, G

    # integrate_sdc on T2
    nn = 32
    A, B, G, U0 = O.ref_heat2d_fields(2, nn, nn)
    dt = O.ref().ref_appendix_dt(2, nn, nn)
    steps = 10
    uo = np.zeros_like(U0)
    res = np.zeros(64)
    sw, fe = C.c_int(), C.c_int()
    p = np.array(SMC)
    rc = O.ref().ref_heat2d_integrate_sdc(2, nn, nn, 0, O.dp(p), O.dp(U0), C.c_double(0.0),
                                          C.c_double(steps * dt), steps, 0, 3, 4, C.c_double(0.0),
                                          O.dp(uo), O.dp(res), 64, C.byref(sw), C.byref(fe))
    assert rc == 0
    g["sdc_t2_u0"], g["sdc_t2_u"], g["sdc_t2_res"] = U0, uo, res[: sw.value]
    g["sdc_t2_meta"] = np.array([nn, steps, steps * dt, sw.value, fe.value], dtype=np.float64)

    # integrate_mrsdc mode 1 on a 3-component split linear problem
    l1 = np.array([-1.0, -0.5, -2.0])
    l2 = np.array([-10.0, -4.0, -7.0])

    def f1(t, uu, out, nd, ctx):
        for i in range(nd):
            out[i] = l1[i] * uu[i]

    def f2(t, uu, out, nd, ctx):
        for i in range(nd):
            out[i] = l2[i] * uu[i] + 0.1 * np.sin(t)

    c1, c2 = O.RHS_CB(f1), O.RHS_CB(f2)
    u0 = np.array([1.0, 0.5, -0.25])
    uo = np.zeros(3)
    res = np.zeros(64)
    sw, n1, n2 = C.c_int(), C.c_int(), C.c_int()
    rc = O.ref().ref_integrate_mrsdc1(c1, None, c2, None, 3, O.dp(u0), C.c_double(0.0),
                                      C.c_double(0.4), 4, 0, 3, 1, 0, 5, 1, 4, C.c_double(0.0),
                                      O.dp(uo), O.dp(res), 64, C.byref(sw), C.byref(n1),
                                      C.byref(n2))
    assert rc == 0, O.ref().ref_last_error()
    g["mr_u0"], g["mr_u"], g["mr_res"] = u0, uo, res[: sw.value]
    g["mr_meta"] = np.array([sw.value, n1.value, n2.value], dtype=np.float64)

    # integrate_mrsdc mode 2 (mrsdc.cpp:137-206) on the reference's own stiff
    # problem and on block-local Robertson kinetics
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import mode2_problems as MP
    cases = {
        "osc": (("oscillator", dict(sigma=1.0e4)), np.array([1.0]), 0.1, 5,
                dict(coarse_n=3, fine_type=1, fine_n=5, iterations=6, rtol=1e-12, atol=1e-13)),
        "rob": (("robertson", dict(ncell=4, inter=False)), MP.robertson_u0(4, False), 0.05, 5,
                dict(coarse_n=3, fine_type=1, fine_n=5, iterations=4)),
        "oscc": (("oscillator", dict(sigma=1.0e3)), np.array([1.0]), 0.02, 2,
                 dict(coarse_n=5, fine_type=2, fine_n=3, repeats=2, iterations=4)),
    }
    for name, ((pname, pkw), u0m, t1m, nst, kw) in cases.items():
        f1, f2 = MP.np_callbacks(pname, **pkw)
        rc, um, dg, msg = O.ref_integrate_mrsdc2(O.RHS_CB(f1), O.RHS_CB(f2), u0m, 0.0, t1m, nst,
                                                 **kw)
        assert rc == 0, msg
        g[f"m2_{name}_u0"], g[f"m2_{name}_u"], g[f"m2_{name}_res"] = u0m, um, dg["residuals"]
        g[f"m2_{name}_meta"] = np.array([dg[k] for k in ("sweeps", "f1_evals", "f2_evals",
                                                         "implicit_solves", "newton_f1_evals")],
                                        dtype=np.float64)

    # integrate_stiff (stiff.cpp:115-188): one Robertson cell to t = 1, four
    # interleaved cells to t = 0.5 (rtol 1e-6), the forced oscillator to t = 1
    import math
    def osc_full(t, up, op, nd, ctx):
        for i in range(nd):
            op[i] = -1.0e4 * (up[i] - math.cos(t)) - math.sin(t)
    rob1, _ = MP.np_callbacks("robertson", ncell=1, inter=False)
    rob4, _ = MP.np_callbacks("robertson", ncell=4, inter=True)
    stiff_cases = {
        "rob1": (rob1, MP.robertson_u0(1, False), 1.0, {}),
        "rob4": (rob4, MP.robertson_u0(4, True), 0.5, dict(rtol=1e-6, atol=1e-10)),
        "osc": (osc_full, np.array([1.0]), 1.0, {}),
    }
    for name, (fn, u0s, t1s, kw) in stiff_cases.items():
        rc, us, msg = O.ref_integrate_stiff(O.RHS_CB(fn), u0s, 0.0, t1s, **kw)
        assert rc == 0, msg
        g[f"st_{name}_u0"], g[f"st_{name}_u"] = u0s, us

    for fam, nm, sz in ((0, "gl", 3), (0, "gl", 5), (1, "cc", 5)):
        nodes, q, s = O.ref_integration_matrices(fam, sz)
        g[f"q_{nm}{sz}"], g[f"s_{nm}{sz}"], g[f"nodes_{nm}{sz}"] = q, s, nodes
    g["nodes_gl9"] = O.ref_integration_matrices(0, 9)[0]
    h = O.ref_hierarchy(0, 3, 1, 0, 5)
    for k, v in h.items():
        g[f"h_{k}"] = v.astype(np.float64)

    out = os.path.join(os.path.dirname(__file__), "golden.npz")
    np.savez_compressed(out, **g)
    print(out, sum(v.nbytes for v in g.values()), "bytes")


if __name__ == "__main__":
    main()
