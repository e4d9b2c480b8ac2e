"""GPU parity of the time advance of the reacting-NS state (configs[2]: SDC
with 3 Gauss-Lobatto nodes; configs[4]: MRSDC mode 1, advection-diffusion on
GL(3) coarse nodes, chemistry on GL(5) fine nodes per coarse interval).
Device-resident steppers + NS kernels vs the oracle's integrators
(oracle.c, restating sdc.cpp / mrsdc.cpp) driving the NS oracle.  Tolerance:
1e-9 of each component's max magnitude after the steps (north_star)."""
import ctypes as C
import math

import numpy as np
import pytest

import paper_1309_7327_b200 as P
from paper_1309_7327_b200 import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu
DX = 1e-4


def _state(n, **kw):
    T, p, uvw, Y = W.ns_primitives(n, **kw)
    return O.ns_conserved(T, p, uvw, Y), (T, p, uvw, Y)


def acoustic_dt(prims, dx, cfl=0.5):
    """CFL 0.5 on max(|u_i| + c): c^2 = gamma R T / W_mix (host, from the
    primitive state; smc_mechanism.h thermodynamics)."""
    T, p, uvw, Y = prims
    W_ = np.array([2.01588e-3, 31.9988e-3, 18.01528e-3, 1.00794e-3, 15.9994e-3, 17.00734e-3,
                   33.00674e-3, 34.01468e-3, 28.0134e-3])
    a = np.array([[3.40, 1.0e-4, 1.0e-8], [3.30, 6.0e-4, -1.0e-7], [3.60, 9.0e-4, -1.0e-7],
                  [2.50, 0.0, 0.0], [2.60, -1.0e-4, 2.0e-8], [3.50, 1.0e-4, 1.0e-8],
                  [4.00, 1.2e-3, -2.0e-7], [4.50, 2.0e-3, -3.0e-7], [3.25, 5.0e-4, -8.0e-8]])
    Ru = 8.314462618
    cp = sum(Y[k] * Ru / W_[k] * (a[k, 0] + a[k, 1] * T + a[k, 2] * T * T) for k in range(9))
    Rm = sum(Y[k] * Ru / W_[k] for k in range(9))
    c = np.sqrt(cp / (cp - Rm) * Rm * T)
    return cfl * dx / (np.abs(uvw).max(axis=0) + c).max()


def _percomp(a, b):
    return max(float(np.abs(a[v] - b[v]).max() / max(np.abs(b[v]).max(), 1e-300))
               for v in range(a.shape[0]))


def _cb(n, part):
    shape = (14, n, n, n)

    def f(t, u, out, dim, ctx):
        uu = np.ctypeslib.as_array(u, shape=(dim,)).reshape(shape).copy()
        np.ctypeslib.as_array(out, shape=(dim,))[:] = O.ns_rhs(uu, DX, part).ravel()

    return O.RHS_CB(f)


@pytest.mark.parametrize("n", [12, 32])
def test_sdc_ten_steps_vs_oracle(cuda, golden, n):
    """configs[2] (10 SDC steps at CFL 0.5 of the configs[0] state) at 12^3 and
    32^3 (81 oracle RHS evaluations of the 32^3 box: ~20 s on the host)."""
    steps = 10
    U0, prims = _state(n)  # configs[2]: the configs[0] generator (T = 1200 +- 300 K)
    dt = acoustic_dt(prims, DX)
    t1 = steps * dt
    # oracle: integrate_sdc restated (sdc.cpp:38-127) over the NS oracle
    cb = _cb(n, 0)
    u0 = U0.ravel().copy()
    uo = np.empty_like(u0)
    res = np.zeros(64)
    sw, fe, es = C.c_int(), C.c_int(), C.c_int()
    rc = O.lib().or_integrate_sdc(cb, None, u0.size, O.dp(u0), C.c_double(0.0), C.c_double(t1),
                                  steps, 2, O.dp(golden["nodes_gl3"]), O.dp(golden["q_gl3"]),
                                  O.dp(golden["s_gl3"]), 4, C.c_double(0.0), 1, O.dp(uo),
                                  O.dp(res), 64, C.byref(sw), C.byref(fe), C.byref(es))
    assert rc == 0
    ref = uo.reshape(U0.shape)
    # device: NS kernels + device-resident SDC
    op = P.NsOperator(n, n, n, DX)
    st = P.SdcStepper(3, P.StepControls(4, 0.0))
    got, d = st.integrate(op.full, U0, 0.0, t1, steps)
    assert d.sweeps == sw.value and d.fresh_evals == fe.value
    assert _percomp(got, ref) <= 1e-9
    np.testing.assert_allclose(d.residual_history, res[: sw.value], rtol=1e-5, atol=1e-300)
    assert not d.nonfinite


def test_mrsdc_mode1_vs_oracle(cuda, golden):
    n, steps = 12, 3
    U0, prims = _state(n, ignition=True)  # configs[4]: 1500 K kernel in 600 K H2/air
    dt = acoustic_dt(prims, DX)
    t1 = steps * dt
    c1, c2 = _cb(n, 1), _cb(n, 2)
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
    rc = O.lib().or_integrate_mrsdc1(
        c1, None, c2, None, u0.size, O.dp(u0), C.c_double(0.0), C.c_double(t1), steps, 2,
        O.dp(arrs[0]), m2, O.dp(arrs[1]), O.dp(arrs[2]), O.dp(arrs[3]), O.dp(arrs[4]),
        O.dp(arrs[5]), O.ip(foc), O.ip(pm), 4, C.c_double(0.0), O.dp(uo), O.dp(res), 64,
        C.byref(sw), C.byref(n1), C.byref(n2))
    assert rc == 0
    ref = uo.reshape(U0.shape)
    op = P.NsOperator(n, n, n, DX)
    st = P.MrsdcStepper(3, 5, P.StepControls(4, 0.0))
    got, d = st.integrate_mode1(op.advdiff, op.chem, U0, 0.0, t1, steps)
    assert (d.sweeps, d.f1_evals, d.f2_evals) == (sw.value, n1.value, n2.value)
    assert _percomp(got, ref) <= 1e-9


def test_sdc_device_buffers_and_stream(cuda):
    """The whole advance on device buffers, on a non-default stream."""
    import torch
    n = 16
    U0, prims = _state(n)
    dt = acoustic_dt(prims, DX)
    op = P.NsOperator(n, n, n, DX)
    s = torch.cuda.Stream()
    op.set_stream(s)
    st = P.SdcStepper(3, P.StepControls(4, 0.0))
    Ud = torch.from_numpy(U0).to(cuda)
    with torch.cuda.stream(s):
        out, d = st.integrate(op.full, Ud, 0.0, 2 * dt, 2)
    s.synchronize()
    host, _ = st.integrate(op.full, U0, 0.0, 2 * dt, 2)
    assert np.array_equal(out.cpu().numpy(), host)
    assert math.isfinite(d.residual_history[-1])


def test_distributed_ns_single_rank_through_device_callback(cuda):
    """The multi-GPU NS path at world size 1 (slab with self-copied ghosts,
    RHS as a device callback into the device-resident stepper) reproduces
    the periodic operator's time advance bitwise."""
    import torch
    from paper_1309_7327_b200.distributed import DistributedNs, Slab, allreduce_max
    n = 12
    U0, prims = _state(n)
    dt = acoustic_dt(prims, DX)
    dns = DistributedNs(Slab(0, 1, n), n, n, DX)
    rhs = dns.rhs(P.NS_FULL)
    rhs.set_stream(torch.cuda.current_stream())
    st = P.SdcStepper(3, P.StepControls(4, 0.0))
    st.set_reducer(allreduce_max(None))
    Ud = torch.from_numpy(U0).to(cuda)
    got, d = st.integrate(rhs, Ud, 0.0, 3 * dt, 3)
    torch.cuda.synchronize()
    op = P.NsOperator(n, n, n, DX)
    ref, _ = P.SdcStepper(3, P.StepControls(4, 0.0)).integrate(op.full, U0, 0.0, 3 * dt, 3)
    assert np.array_equal(got.cpu().numpy(), ref)
    assert d.fresh_evals == 3 * 8 + 1
