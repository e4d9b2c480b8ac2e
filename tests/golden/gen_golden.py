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
