"""GPU parity of the reacting-NS path at BASELINE.json's own sizes, against
the threaded CPU oracle (oracle/ns_oracle.c, OpenMP over every host thread):

* configs[3]: one full RHS of the 256^3 hot-spot state (T peak 1800 K,
  radius 20 cells) -- per-component max error <= 1e-10 of the field max;
* configs[2]: 10 SDC steps (GL(3), K = 4, cutoff 0) at CFL 0.5 of the
  configs[0] state on a 128^3 box -- <= 1e-9 of the field max;
* configs[4]: MRSDC mode 1 (GL(3) coarse / GL(5) fine, K = 4) on the
  ignition state at 128^3, 2 steps -- <= 1e-9 of the field max.

The errors, and the chemistry's gross/net ratio on the hot spot (how much
cancellation the wdot sum does there), are printed and, when
SMC_PARITY_REPORT names a file, appended to it as JSON lines.  Together they
take a few minutes of host time (the oracle)."""
import ctypes as C
import json
import os
import time

import numpy as np
import pytest

import paper_1309_7327_b200 as P
from paper_1309_7327_b200 import workloads as W
from oracle import oracle as O

from test_gpu_ns_steppers import acoustic_dt

pytestmark = pytest.mark.gpu
DX = 1e-4


def _percomp(a, b):
    return [float(np.abs(a[v] - b[v]).max() / max(np.abs(b[v]).max(), 1e-300))
            for v in range(a.shape[0])]


def _report(**kw):
    print(json.dumps(kw))
    path = os.environ.get("SMC_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(kw) + "\n")


def _cb(n, part, counter):
    shape = (14, n, n, n)

    def f(t, u, out, dim, ctx):
        uu = np.ctypeslib.as_array(u, shape=(dim,)).reshape(shape)
        np.ctypeslib.as_array(out, shape=(dim,))[:] = O.ns_rhs(uu, DX, part).ravel()
        counter[0] += 1

    return O.RHS_CB(f)


def test_configs3_full_rhs_256(cuda):
    n = 256
    threads = O.set_threads(0)
    T, p, uvw, Y = W.ns_primitives(n, hot_spot=True)
    U = O.ns_conserved(T, p, uvw, Y)
    del T, p, uvw, Y
    t0 = time.time()
    ref = O.ns_rhs(U, DX, P.NS_FULL)
    t_oracle = time.time() - t0
    op = P.NsOperator(n, n, n, DX)
    got = op.full(0.0, U)
    errs = _percomp(got, ref)
    del got
    chem = O.ns_rhs(U, DX, P.NS_CHEM)[5:]
    gross = O.ns_chem_gross(U)
    ratio = [float(np.abs(gross[k]).max() / max(np.abs(chem[k]).max(), 1e-300))
             for k in range(9)]
    _report(test="configs3_full_rhs_256", cells=n ** 3, max_rel_err=max(errs), per_component=errs,
            chem_gross_over_net=ratio, oracle_threads=threads, oracle_s=t_oracle)
    assert max(errs) <= 1e-10, errs


def test_configs2_sdc_ten_steps_128(cuda, golden):
    n, steps = 128, 10
    threads = O.set_threads(0)
    T, p, uvw, Y = W.ns_primitives(n)
    U0 = O.ns_conserved(T, p, uvw, Y)
    dt = acoustic_dt((T, p, uvw, Y), DX)
    del T, p, uvw, Y
    t1 = steps * dt
    calls = [0]
    cb = _cb(n, 0, calls)
    u0 = U0.ravel().copy()
    uo = np.empty_like(u0)
    res = np.zeros(64)
    sw, fe, es = C.c_int(), C.c_int(), C.c_int()
    t0 = time.time()
    rc = O.lib().or_integrate_sdc(cb, None, u0.size, O.dp(u0), C.c_double(0.0), C.c_double(t1),
                                  steps, 2, O.dp(golden["nodes_gl3"]), O.dp(golden["q_gl3"]),
                                  O.dp(golden["s_gl3"]), 4, C.c_double(0.0), 1, O.dp(uo),
                                  O.dp(res), 64, C.byref(sw), C.byref(fe), C.byref(es))
    t_oracle = time.time() - t0
    assert rc == 0
    del u0
    ref = uo.reshape(U0.shape)
    op = P.NsOperator(n, n, n, DX)
    st = P.SdcStepper(3, P.StepControls(4, 0.0))
    got, d = st.integrate(op.full, U0, 0.0, t1, steps)
    errs = _percomp(got, ref)
    _report(test="configs2_sdc_10_steps_128", cells=n ** 3, steps=steps, dt=dt,
            rhs_evals=d.fresh_evals, max_rel_err=max(errs), per_component=errs,
            final_residual_gpu=d.residual_history[-1], final_residual_oracle=float(res[sw.value - 1]),
            oracle_threads=threads, oracle_s=t_oracle)
    assert d.sweeps == sw.value and d.fresh_evals == fe.value == 81
    assert max(errs) <= 1e-9, errs
    # the residual is a max-norm of a difference of nearly equal states (~1e-11
    # of the field): its low digits are rounding, so only 1e-3 relative
    np.testing.assert_allclose(d.residual_history, res[: sw.value], rtol=1e-3, atol=1e-300)


def test_configs4_mrsdc_mode1_128(cuda, golden):
    n, steps = 128, 2
    threads = O.set_threads(0)
    T, p, uvw, Y = W.ns_primitives(n, ignition=True)
    U0 = O.ns_conserved(T, p, uvw, Y)
    dt = acoustic_dt((T, p, uvw, Y), DX)
    del T, p, uvw, Y
    t1 = steps * dt
    calls = [0]
    c1, c2 = _cb(n, 1, calls), _cb(n, 2, calls)
    h = {k[2:]: golden[k] for k in golden if k.startswith("h_")}
    I = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
    D = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    m2 = len(h["fine"]) - 1
    u0 = U0.ravel().copy()
    uo = np.empty_like(u0)
    res = np.zeros(64)
    sw, n1, n2 = C.c_int(), C.c_int(), C.c_int()
    foc, pm = I(h["fine_of_coarse"]), I(h["p_map"])
    arrs = [D(h[k]) for k in ("coarse", "fine", "s21", "q21", "s22", "q22")]
    t0 = time.time()
    rc = O.lib().or_integrate_mrsdc1(
        c1, None, c2, None, u0.size, O.dp(u0), C.c_double(0.0), C.c_double(t1), steps, 2,
        O.dp(arrs[0]), m2, O.dp(arrs[1]), O.dp(arrs[2]), O.dp(arrs[3]), O.dp(arrs[4]),
        O.dp(arrs[5]), O.ip(foc), O.ip(pm), 4, C.c_double(0.0), O.dp(uo), O.dp(res), 64,
        C.byref(sw), C.byref(n1), C.byref(n2))
    t_oracle = time.time() - t0
    assert rc == 0
    del u0
    ref = uo.reshape(U0.shape)
    op = P.NsOperator(n, n, n, DX)
    st = P.MrsdcStepper(3, 5, P.StepControls(4, 0.0))
    got, d = st.integrate_mode1(op.advdiff, op.chem, U0, 0.0, t1, steps)
    errs = _percomp(got, ref)
    _report(test="configs4_mrsdc_mode1_128", cells=n ** 3, steps=steps, dt=dt,
            f1_evals=d.f1_evals, f2_evals=d.f2_evals, max_rel_err=max(errs), per_component=errs,
            oracle_threads=threads, oracle_s=t_oracle)
    assert (d.sweeps, d.f1_evals, d.f2_evals) == (sw.value, n1.value, n2.value)
    assert max(errs) <= 1e-9, errs
