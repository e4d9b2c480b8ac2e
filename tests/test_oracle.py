"""CPU: pin the oracle (oracle/oracle.c) against the reference's golden vectors
(tests/golden/golden.npz, generated from the unmodified reference by
tests/golden/gen_golden.py) and against the reference's own known-answer tests
(proj/tests/stencil_test.cpp, pde_test.cpp, sdc_test.cpp, mrsdc_test.cpp),
and — where oracle/_ref exists — against the live reference library."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import oracle as O

SMC = (3557.0 / 44100.0, -2083.0 / 117600.0)
OPT = (1059283.0 / 13608000.0, -856481.0 / 40824000.0)
M36 = (281.0 / 3600.0,)


def test_coupling_matrix_golden(golden):
    for key, order, p in (("m8_smc", 8, SMC), ("m8_zero", 8, (0.0, 0.0)),
                          ("m8_optimal", 8, OPT), ("m6_default", 6, M36)):
        m, s = O.build_narrow(order, p)
        assert np.array_equal(m, golden[key]), key


def test_coupling_matrix_kats():
    # stencil_test.cpp:55-67
    m, s = O.build_narrow(8, (0.0, 0.0))
    at = lambda mm, nn: m[(mm + s - 1) * 8 + nn + s - 1]  # noqa: E731
    assert at(-3, 1) == pytest.approx(1.0 / 1120, rel=1e-15)
    assert at(0, 0) == pytest.approx(-445.0 / 2016, rel=1e-15)
    assert at(-1, -1) == pytest.approx(-1349.0 / 10080, rel=1e-15)
    assert at(-1, -3) == pytest.approx(-1.0 / 280, rel=1e-15)
    assert at(0, 3) == 0.0 and at(0, 4) == 0.0
    m6, s6 = O.build_narrow(6, (0.0,))
    at6 = lambda mm, nn: m6[(mm + s6 - 1) * 8 + nn + s6 - 1]  # noqa: E731
    assert at6(-2, 1) == pytest.approx(1.0 / 180, rel=1e-15)
    assert at6(0, 0) == pytest.approx(-101.0 / 360, rel=1e-15)
    # structure: antisymmetry + zero pattern (stencil_test.cpp:33-53), 52 nonzeros, zero row sums
    rng = np.random.default_rng(7)
    for order in (8, 6):
        s = 4 if order == 8 else 3
        p = rng.uniform(-0.5, 0.5, size=2 if order == 8 else 1)
        mm, _ = O.build_narrow(order, p)
        M = mm.reshape(8, 8)[: 2 * s, : 2 * s]
        assert np.allclose(M, -M[::-1, ::-1], rtol=1e-15, atol=0)
        assert np.all(M[0, s + 1:] == 0) and np.all(M[1, s + 2:] == 0)
    M8 = O.build_narrow(8, SMC)[0].reshape(8, 8)
    assert np.count_nonzero(M8) == 52
    assert np.abs(M8.sum(axis=1)).max() < 1e-15


def test_bad_orders_rejected():
    with pytest.raises(ValueError):
        O.build_narrow(8, (0.0,))
    with pytest.raises(ValueError):
        O.build_narrow(6, (0.0, 0.0))
    with pytest.raises(ValueError):
        O.build_narrow(4, (0.0,))


def _apply(m, s, a, u, dx):
    out = np.empty_like(u)
    assert O.lib().or_apply_narrow(O.dp(m), s, O.dp(a), O.dp(u), len(u), C.c_double(dx),
                                   O.dp(out)) == 0
    return out


def test_nyquist_kats():
    # stencil_test.cpp:121-138
    n = 32
    a = np.ones(n)
    u = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    for p in (SMC, (0.0, 0.0), OPT):
        m, s = O.build_narrow(8, p)
        np.testing.assert_allclose(_apply(m, s, a, u, 1.0), -2048.0 / 315.0 * u, rtol=1e-13)
    m, s = O.build_narrow(6, M36)
    np.testing.assert_allclose(_apply(m, s, a, u, 1.0), -272.0 / 45.0 * u, rtol=1e-13)
    w = np.empty(n)
    assert O.lib().or_apply_wide(O.dp(a), O.dp(u), n, C.c_double(1.0), O.dp(w)) == 0
    assert np.all(w == 0.0)


def test_polynomial_exactness_and_conservation():
    # stencil_test.cpp:75-119
    for order, degree in ((8, 9), (6, 7)):
        n, dx = 64, 1.0 / 64
        s = 4 if order == 8 else 3
        m, _ = O.build_narrow(order, SMC if order == 8 else M36)
        x = np.arange(n) * dx
        u = sum((x - 0.37) ** d / (d + 1.0) for d in range(degree + 1))
        exact = 2.5 * sum(d * (d - 1) * (x - 0.37) ** (d - 2) / (d + 1.0)
                          for d in range(2, degree + 1))
        out = _apply(m, s, np.full(n, 2.5), u, dx)
        sl = slice(s, n - s)
        assert np.abs(out[sl] - exact[sl]).max() <= 1e-11 * np.abs(exact[sl]).max()
    rng = np.random.default_rng(11)
    a = rng.uniform(0.5, 2.0, 128)
    u = rng.uniform(0.5, 2.0, 128) - 1.2
    for order in (8, 6):
        m, s = O.build_narrow(order, SMC if order == 8 else M36)
        out = _apply(m, s, a, u, 1.0)
        assert abs(out.sum()) <= 100 * 128 * np.finfo(float).eps * np.abs(out).max()


def test_narrow3d_golden(golden):
    m, s = O.build_narrow(8, SMC)
    n = golden["n3d_u"].shape[0]
    out = O.narrow3d(m, s, golden["n3d_a"], golden["n3d_u"], 1.0 / n, 1.0 / n, 1.0 / n)
    assert np.array_equal(out, golden["n3d_out"])


@pytest.mark.parametrize("pid", [1, 2, 3])
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_heat2d_golden(golden, pid, kind):
    u = golden[f"heat_{pid}_{kind}_u"]
    ny, nx = u.shape
    if kind == 0:
        m, s = O.build_narrow(8, SMC)
    elif kind == 1:
        m, s = O.build_narrow(6, M36)
    else:
        m, s = np.zeros(64), 0
    g0 = golden[f"heat_{pid}_g0"] if pid == 1 else None
    out = O.heat2d_rhs(kind, m, s, golden[f"heat_{pid}_a"], golden[f"heat_{pid}_b"], g0,
                       math.exp(-0.3), u, 2 * math.pi / nx, 2 * math.pi / ny)
    assert np.array_equal(out, golden[f"heat_{pid}_{kind}_out"])


def _heat_cb(pid, nx, ny, golden_fields):
    m, s = O.build_narrow(8, SMC)
    A, B, G = golden_fields

    def f(t, u, out, n, ctx):
        uu = np.ctypeslib.as_array(u, shape=(n,)).reshape(ny, nx).copy()
        r = O.heat2d_rhs(0, m, s, A, B, G, math.exp(-t) if G is not None else 0.0, uu,
                         2 * math.pi / nx, 2 * math.pi / ny)
        np.ctypeslib.as_array(out, shape=(n,))[:] = r.ravel()

    return O.RHS_CB(f)


def test_sdc_golden(golden):
    nn, steps, t1, sweeps, fresh = golden["sdc_t2_meta"]
    nn, steps = int(nn), int(steps)
    A, B, _, _ = (None,) * 4
    # T2 fields on the 32^2 grid (no source)
    from oracle.oracle import ref_heat2d_fields, have_ref  # noqa: F401
    # rebuild coefficient samples independently of the reference: T2 closed form (pde.cpp:36-50)
    x = np.arange(nn) * 2 * math.pi / nn
    X, Y = np.meshgrid(x, x)
    A = 1.0 + 0.9 * np.cos(2 * X) * np.sin(2 * Y + math.pi / 3)
    B = 1.0 + 0.9 * np.cos(2 * X + math.pi / 3) * np.sin(2 * Y)
    cb = _heat_cb(2, nn, nn, (A, B, None))
    q, s = golden["q_gl3"], golden["s_gl3"]
    tau = golden["nodes_gl3"]
    u0 = golden["sdc_t2_u0"].ravel().copy()
    uo = np.empty_like(u0)
    res = np.zeros(64)
    sw, fe, es = C.c_int(), C.c_int(), C.c_int()
    rc = O.lib().or_integrate_sdc(cb, None, len(u0), O.dp(u0), C.c_double(0.0), C.c_double(t1),
                                  steps, 2, O.dp(tau), O.dp(q), O.dp(s), 4, C.c_double(0.0), 1,
                                  O.dp(uo), O.dp(res), 64, C.byref(sw), C.byref(fe), C.byref(es))
    assert rc == 0
    assert sw.value == int(sweeps) and fe.value == int(fresh)
    # coefficients recomputed with numpy's sin/cos may differ from glibc's by an ulp
    ref = golden["sdc_t2_u"].ravel()
    assert np.abs(uo - ref).max() <= 1e-13 * np.abs(ref).max()
    np.testing.assert_allclose(res[: sw.value], golden["sdc_t2_res"], rtol=1e-6, atol=1e-15)


def test_mrsdc_golden(golden):
    l1 = np.array([-1.0, -0.5, -2.0])
    l2 = np.array([-10.0, -4.0, -7.0])

    def f1(t, u, out, n, ctx):
        for i in range(n):
            out[i] = l1[i] * u[i]

    def f2(t, u, out, n, ctx):
        for i in range(n):
            out[i] = l2[i] * u[i] + 0.1 * math.sin(t)

    c1, c2 = O.RHS_CB(f1), O.RHS_CB(f2)
    h = {k[2:]: golden[k] for k in golden if k.startswith("h_")}
    m2 = len(h["fine"]) - 1
    u0 = golden["mr_u0"].copy()
    uo = np.empty(3)
    res = np.zeros(64)
    sw, n1, n2 = C.c_int(), C.c_int(), C.c_int()
    I = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
    foc, pm = I(h["fine_of_coarse"]), I(h["p_map"])
    rc = O.lib().or_integrate_mrsdc1(
        c1, None, c2, None, 3, O.dp(u0), C.c_double(0.0), C.c_double(0.4), 4, 2,
        O.dp(np.ascontiguousarray(h["coarse"])), m2, O.dp(np.ascontiguousarray(h["fine"])),
        O.dp(np.ascontiguousarray(h["s21"])), O.dp(np.ascontiguousarray(h["q21"])),
        O.dp(np.ascontiguousarray(h["s22"])), O.dp(np.ascontiguousarray(h["q22"])), O.ip(foc),
        O.ip(pm), 4, C.c_double(0.0), O.dp(uo), O.dp(res), 64, C.byref(sw), C.byref(n1),
        C.byref(n2))
    assert rc == 0
    assert [sw.value, n1.value, n2.value] == [int(v) for v in golden["mr_meta"]]
    assert np.array_equal(uo, golden["mr_u"])
    assert np.array_equal(res[: sw.value], golden["mr_res"])


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_matches_live_reference():
    rng = np.random.default_rng(3)
    for (nx, ny, nz) in ((12, 10, 9), (16, 8, 11)):
        a = rng.uniform(0.5, 2.0, (nz, ny, nx))
        u = rng.standard_normal((nz, ny, nx))
        for order, p in ((8, SMC), (6, M36)):
            m, s = O.build_narrow(order, p)
            o1 = O.narrow3d(m, s, a, u, 0.1, 0.2, 0.3)
            o2 = O.ref_narrow3d(m, s, a, u, 0.1, 0.2, 0.3)
            assert np.array_equal(o1, o2)
    # 1-D operators
    for n in (9, 16, 33):
        a = rng.uniform(0.5, 2.0, n)
        u = rng.standard_normal(n)
        m, s = O.build_narrow(8, SMC)
        r = np.empty(n)
        pp = np.array(SMC)
        assert O.ref().ref_apply_narrow(8, O.dp(pp), 2, O.dp(a), O.dp(u), n, C.c_double(0.3),
                                        O.dp(r)) == 0
        assert np.array_equal(_apply(m, s, a, u, 0.3), r)
        w1, w2 = np.empty(n), np.empty(n)
        O.ref().ref_apply_wide(O.dp(a), O.dp(u), n, C.c_double(0.3), O.dp(w1))
        O.lib().or_apply_wide(O.dp(a), O.dp(u), n, C.c_double(0.3), O.dp(w2))
        assert np.array_equal(w1, w2)
