"""The oracle's MRSDC mode 2 / backward-Euler Newton (oracle.c
or_integrate_mrsdc2, or_solve_backward_euler) pinned to the reference
(mrsdc.cpp:137-206, stiff.cpp:16-76, matrix.cpp:9-51): bitwise against the
golden vectors the reference produced (tests/golden/gen_golden.py) and, when
oracle/_ref is built here, against the live reference — including the block
(colored finite-difference, per-block LU) form the device solver uses."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
import mode2_problems as MP

META = ("sweeps", "f1_evals", "f2_evals", "implicit_solves", "newton_f1_evals")
CASES = {
    "osc": (("oscillator", dict(sigma=1.0e4)), 0.1, 5, (3, 1, 5, 1), 6,
            dict(rtol=1e-12, atol=1e-13)),
    "rob": (("robertson", dict(ncell=4, inter=False)), 0.05, 5, (3, 1, 5, 1), 4, {}),
    "oscc": (("oscillator", dict(sigma=1.0e3)), 0.02, 2, (5, 2, 3, 2), 4, {}),
}


def _hier(coarse_n, fine_type, fine_n, repeats):
    """build_hierarchy tables: the reference's when built here, else the
    library's host builder (equal bit for bit, test_capi.py)."""
    if O.have_ref():
        return O.ref_hierarchy(0, coarse_n, fine_type, 0, fine_n, repeats)
    import paper_1309_7327_b200 as P
    h = P.build_hierarchy(coarse_n, fine_n, repeats if fine_type == 2 else 1)
    h["coarse"] = P.nodes(P.GAUSS_LOBATTO, coarse_n)
    return h


def _run_oracle(name, golden, block=0, inter=False, u0=None):
    (pname, pkw), t1, nst, hk, K, skw = CASES[name]
    f1, f2 = MP.np_callbacks(pname, **pkw)
    c1, c2 = O.RHS_CB(f1), O.RHS_CB(f2)
    h = _hier(*hk)
    u0 = golden[f"m2_{name}_u0"] if u0 is None else u0
    return O.integrate_mrsdc2(c1, c2, u0, 0.0, t1, nst, h, iterations=K, block=block,
                              interleaved=inter, **skw)


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_mode2_equals_reference_golden(golden, name):
    rc, u, d = _run_oracle(name, golden)
    assert rc == 0
    assert np.array_equal(u, golden[f"m2_{name}_u"])
    assert np.array_equal(d["residuals"], golden[f"m2_{name}_res"])
    assert [d[k] for k in META] == [int(v) for v in golden[f"m2_{name}_meta"]]


def test_block_newton_equals_dense_reference(golden):
    """4 Robertson cells: the block form (block 3, one colored FD column per
    block column, per-block LU) reproduces the reference's dense Newton bit for
    bit — contiguous and interleaved (structure-of-arrays) layouts."""
    ref_u = golden["m2_rob_u"]
    rc, u, d = _run_oracle("rob", golden, block=3)
    assert rc == 0 and np.array_equal(u, ref_u)
    # the same problem in interleaved order: component j of cell c at j*4 + c
    f1, f2 = MP.np_callbacks("robertson", ncell=4, inter=True)
    h = _hier(3, 1, 5, 1)
    u0 = MP.robertson_u0(4, True)
    rc, ui, di = O.integrate_mrsdc2(O.RHS_CB(f1), O.RHS_CB(f2), u0, 0.0, 0.05, 5, h,
                                    iterations=4, block=3, interleaved=True)
    assert rc == 0
    perm = MP._idx(4, True).ravel()  # interleaved index of (c, j) in contiguous order
    assert np.array_equal(ui[perm], ref_u)
    assert np.array_equal(di["residuals"], golden["m2_rob_res"])
    # the colored Jacobian spends block (3) f1 evaluations per Newton step, not dim (12)
    assert di["newton_f1_evals"] == d["newton_f1_evals"] < golden["m2_rob_meta"][4]


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (no /root/reference)")
def test_block_newton_interleaved_matches_live_reference():
    f1, f2 = MP.np_callbacks("robertson", ncell=5, inter=True)
    c1, c2 = O.RHS_CB(f1), O.RHS_CB(f2)
    u0 = MP.robertson_u0(5, True)
    rc, ur, dr, msg = O.ref_integrate_mrsdc2(c1, c2, u0, 0.0, 0.03, 3, iterations=3)
    assert rc == 0, msg
    h = O.ref_hierarchy(0, 3, 1, 0, 5)
    rc, uo, do = O.integrate_mrsdc2(c1, c2, u0, 0.0, 0.03, 3, h, iterations=3, block=3,
                                    interleaved=True)
    assert rc == 0
    assert np.array_equal(uo, ur)
    assert np.array_equal(do["residuals"], dr["residuals"])
    for k in ("sweeps", "f1_evals", "f2_evals", "implicit_solves"):
        assert do[k] == dr[k]


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (no /root/reference)")
def test_solve_backward_euler_matches_reference():
    f1, _ = MP.np_callbacks("robertson", ncell=3, inter=False)
    cb = O.RHS_CB(f1)
    c = MP.robertson_u0(3, False)
    for beta in (1e-3, 0.05, 0.5):
        wr, rr = O.ref_solve_backward_euler(cb, 9, 0.0, beta, c, c)
        wo, ro = O.solve_backward_euler(cb, 9, 0.0, beta, c, c)
        assert np.array_equal(wo, wr)
        assert (ro.iterations, bool(ro.converged), ro.f_evals) == \
            (rr["iterations"], rr["converged"], rr["f_evals"])
        assert ro.final_residual == rr["final_residual"]


def test_newton_failure_reports_coarse_node():
    """mrsdc_test.cpp:215-228: w = c + beta w^2 has no real root for c = 5."""
    f1, f2 = MP.np_callbacks("quadratic")
    c1, c2 = O.RHS_CB(f1), O.RHS_CB(f2)
    h = _hier(3, 1, 2, 1)
    rc, _, d = O.integrate_mrsdc2(c1, c2, np.array([5.0]), 0.0, 1.0, 1, h, iterations=4)
    assert rc == 2 and d["fail_node"] == 1 and d["fail_sweep"] == 1
    if O.have_ref():
        rc, _, _, msg = O.ref_integrate_mrsdc2(c1, c2, np.array([5.0]), 0.0, 1.0, 1, fine_n=2)
        assert rc == 2 and "coarse node 1" in msg and "sweep 1" in msg


def test_mode2_with_vanishing_implicit_term_equals_mode1():
    """mrsdc_test.cpp:163-173."""
    h = _hier(3, 1, 5, 1)
    zero = O.RHS_CB(lambda t, up, op, n, ctx: [op.__setitem__(i, 0.0) for i in range(n)])

    def lin(t, up, op, n, ctx):
        for i in range(n):
            op[i] = -3.0 * up[i]
    f2 = O.RHS_CB(lin)
    rc, u2, _ = O.integrate_mrsdc2(zero, f2, np.array([1.0]), 0.0, 0.2, 1, h, iterations=4)
    assert rc == 0
    D = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    uo, res = np.empty(1), np.zeros(16)
    sw, n1, n2 = C.c_int(), C.c_int(), C.c_int()
    u0 = np.array([1.0])
    arrs = [D(h[k]) for k in ("coarse", "fine", "s21", "q21", "s22", "q22")]
    foc = np.ascontiguousarray(h["fine_of_coarse"], dtype=np.int32)
    pm = np.ascontiguousarray(h["p_map"], dtype=np.int32)
    assert O.lib().or_integrate_mrsdc1(
        zero, None, f2, None, 1, O.dp(u0), C.c_double(0.0), C.c_double(0.2), 1, 2,
        O.dp(arrs[0]), len(h["fine"]) - 1, O.dp(arrs[1]), O.dp(arrs[2]), O.dp(arrs[3]),
        O.dp(arrs[4]),
        O.dp(arrs[5]), O.ip(foc), O.ip(pm), 4, C.c_double(0.0), O.dp(uo), O.dp(res), 16,
        C.byref(sw), C.byref(n1), C.byref(n2)) == 0
    assert abs(u2[0] - uo[0]) <= 1e-15


STIFF = {"rob1": ({}, 1.0, 1, False), "rob4": (dict(rtol=1e-6, atol=1e-10), 0.5, 4, True),
         "osc": ({}, 1.0, 0, False)}


def _stiff_cb(name):
    import math
    if name == "osc":
        def f(t, up, op, n, ctx):
            for i in range(n):
                op[i] = -1.0e4 * (up[i] - math.cos(t)) - math.sin(t)
        return O.RHS_CB(f)
    ncell, inter = STIFF[name][2], STIFF[name][3]
    return O.RHS_CB(MP.np_callbacks("robertson", ncell=ncell, inter=inter)[0])


@pytest.mark.parametrize("name", list(STIFF))
def test_integrate_stiff_oracle_equals_reference_golden(golden, name):
    """or_integrate_stiff (oracle.c) restates stiff.cpp:80-188 bit for bit;
    rob4 also through the block (3, interleaved) Newton."""
    kw, t1, ncell, inter = STIFF[name]
    cb = _stiff_cb(name)
    rc, u, acc, rej = O.integrate_stiff(cb, golden[f"st_{name}_u0"], 0.0, t1, **kw)
    assert rc == 0 and acc > 0
    assert np.array_equal(u, golden[f"st_{name}_u"])
    if inter:
        rc, ub, _, _ = O.integrate_stiff(cb, golden[f"st_{name}_u0"], 0.0, t1, block=3,
                                         interleaved=True, **kw)
        assert rc == 0 and np.array_equal(ub, golden[f"st_{name}_u"])


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (no /root/reference)")
def test_integrate_stiff_errors_match_reference():
    cb = _stiff_cb("rob1")
    u0 = MP.robertson_u0(1, False)
    rc, _, msg = O.ref_integrate_stiff(cb, u0, 1.0, 0.0)
    assert rc == 1 and "t1 must be >= t0" in msg
    assert O.integrate_stiff(cb, u0, 1.0, 0.0)[0] == 1
    rc, _, msg = O.ref_integrate_stiff(cb, u0, 0.0, 1.0, rtol=0.0)
    assert rc == 1 and "bad tolerances" in msg
    assert O.integrate_stiff(cb, u0, 0.0, 1.0, rtol=0.0)[0] == 1
