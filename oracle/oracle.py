"""TEST INFRASTRUCTURE ONLY — ctypes access to the checkers.

* ``lib()``  -> oracle/liboracle.so, the C restatement (oracle.c, ns_oracle.c)
* ``ref()``  -> oracle/_ref/libnsdc_ref.so, the unmodified reference library
  (built from /root/reference sources by oracle/Makefile) plus ref_capi.cpp
* ``ref_fast()`` -> the same with the reference's Release flags (CPU baseline)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)

RHS_CB = C.CFUNCTYPE(None, C.c_double, _D, _D, C.c_longlong, C.c_void_p)

_lib = None
_ref = {}


def dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def ip(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_I)


def build_oracle() -> None:
    """Compile the C restatement (gcc; present on the GPU box too)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def build_ref() -> bool:
    """Compile oracle/_ref from /root/reference (only where it exists)."""
    if not os.path.isdir("/root/reference/proj/core/src"):
        return os.path.exists(os.path.join(REF_DIR, "libnsdc_ref.so"))
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    return True


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build_oracle()
        _lib = C.CDLL(path)
        _lib.or_narrow_dir.restype = None
        _lib.or_deriv8_dir.restype = None
        _lib.or_narrow_interfaces.restype = None
    return _lib


def have_ref(fast: bool = False) -> bool:
    name = "libnsdc_ref_fast.so" if fast else "libnsdc_ref.so"
    return os.path.exists(os.path.join(REF_DIR, name))


def ref(fast: bool = False):
    name = "libnsdc_ref_fast.so" if fast else "libnsdc_ref.so"
    if name not in _ref:
        r = C.CDLL(os.path.join(REF_DIR, name))
        r.ref_last_error.restype = C.c_char_p
        r.ref_truncation_bound.restype = C.c_double
        r.ref_appendix_dt.restype = C.c_double
        r.ref_set_workers.restype = None
        _ref[name] = r
    return _ref[name]


# ----------------------------------------------------------------- helpers
def build_narrow(order: int, params) -> tuple[np.ndarray, int]:
    p = np.ascontiguousarray(params, dtype=np.float64)
    m = np.zeros(64)
    s = C.c_int()
    rc = lib().or_build_narrow(order, dp(p), len(p), dp(m), C.byref(s))
    if rc:
        raise ValueError("or_build_narrow: bad order/params")
    return m, s.value


def apply_narrow_bounded(params8, a, u, dx, m36=281.0 / 3600.0) -> np.ndarray:
    """or_apply_narrow_bounded on one non-periodic line."""
    m8, _ = build_narrow(8, params8)
    m6, _ = build_narrow(6, (m36,))
    a = np.ascontiguousarray(a, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    rc = lib().or_apply_narrow_bounded(dp(m8), dp(m6), dp(a), dp(u), len(u), C.c_double(dx),
                                       dp(out))
    if rc:
        raise ValueError("or_apply_narrow_bounded: bad args")
    return out


def first_derivative_bounded(u, dx) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    rc = lib().or_first_derivative_bounded(dp(u), len(u), C.c_double(dx), dp(out))
    if rc:
        raise ValueError("or_first_derivative_bounded: bad args")
    return out


def first_derivative8(u, dx) -> np.ndarray:
    """or_first_derivative8 (periodic)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    assert lib().or_first_derivative8(dp(u), len(u), C.c_double(dx), dp(out)) == 0
    return out


def narrow3d(m64, s, a, u, dx, dy, dz) -> np.ndarray:
    nz, ny, nx = u.shape
    out = np.empty_like(u)
    rc = lib().or_narrow3d(dp(m64), s, dp(a), dp(u), nx, ny, nz, C.c_double(dx), C.c_double(dy),
                           C.c_double(dz), dp(out))
    assert rc == 0
    return out


def ref_narrow3d(m64, s, a, u, dx, dy, dz, fast: bool = False) -> np.ndarray:
    nz, ny, nx = u.shape
    out = np.empty_like(u)
    r = ref(fast)
    rc = r.ref_narrow3d(dp(m64), s, dp(a), dp(u), nx, ny, nz, C.c_double(dx), C.c_double(dy),
                        C.c_double(dz), dp(out))
    if rc:
        raise ValueError(r.ref_last_error().decode())
    return out


def heat2d_rhs(kind, m64, s, a, b, g0, gt, u, dx, dy) -> np.ndarray:
    ny, nx = u.shape
    out = np.empty_like(u)
    g0p = dp(g0) if g0 is not None else None
    rc = lib().or_heat2d_rhs(kind, dp(m64), s, dp(a), dp(b), g0p, C.c_double(gt), dp(u), nx, ny,
                             C.c_double(dx), C.c_double(dy), dp(out))
    if rc:
        raise ValueError("or_heat2d_rhs: bad args")
    return out


def ref_heat2d_fields(pid: int, nx: int, ny: int):
    a, b, g0, u0 = (np.zeros((ny, nx)) for _ in range(4))
    rc = ref().ref_heat2d_fields(pid, nx, ny, dp(a), dp(b), dp(g0), dp(u0))
    assert rc == 0
    return a, b, g0, u0


def ref_heat2d_rhs(pid, kind, params, t, u, a=None, b=None, g0=None, fast=False) -> np.ndarray:
    ny, nx = u.shape
    p = np.ascontiguousarray(list(params) + [0.0] * (2 - len(params)), dtype=np.float64)
    out = np.empty_like(u)
    r = ref(fast)
    rc = r.ref_heat2d_rhs(pid, nx, ny, kind, dp(p), dp(a) if a is not None else None,
                          dp(b) if b is not None else None, dp(g0) if g0 is not None else None,
                          C.c_double(t), dp(u), dp(out))
    if rc:
        raise ValueError(r.ref_last_error().decode())
    return out


def ref_integration_matrices(family: int, n: int):
    q = np.zeros((n - 1, n))
    s = np.zeros((n - 1, n))
    nodes = np.zeros(n)
    assert ref().ref_nodes(family, n, dp(nodes)) == 0
    assert ref().ref_integration_matrices(family, n, dp(q), dp(s)) == 0
    return nodes, q, s


def ref_hierarchy(coarse_family, coarse_n, fine_type, fine_family, fine_n, repeats=1):
    m2p1 = C.c_int()
    big = 1 + (coarse_n - 1) * repeats * (fine_n - 1)
    fine = np.zeros(big)
    m1 = coarse_n - 1
    q21 = np.zeros((big - 1, m1 + 1))
    s21 = np.zeros((big - 1, m1 + 1))
    q22 = np.zeros((big - 1, big))
    s22 = np.zeros((big - 1, big))
    foc = np.zeros(coarse_n, dtype=np.int32)
    pm = np.zeros(big, dtype=np.int32)
    r = ref()
    rc = r.ref_build_hierarchy(coarse_family, coarse_n, fine_type, fine_family, fine_n, repeats,
                               C.byref(m2p1), dp(fine), dp(q21), dp(s21), dp(q22), dp(s22), ip(foc),
                               ip(pm))
    assert rc == 0, r.ref_last_error()
    n2 = m2p1.value
    assert n2 == big
    coarse = np.zeros(coarse_n)
    r.ref_nodes(coarse_family, coarse_n, dp(coarse))
    return dict(coarse=coarse, fine=fine, q21=q21, s21=s21, q22=q22, s22=s22,
                fine_of_coarse=foc, p_map=pm)


# ------------------------------------------------------------------ NS
def ns_conserved(T, p, uvw, Y) -> np.ndarray:
    n = T.size
    U = np.empty((14,) + T.shape)
    lib().or_ns_conserved(dp(T), dp(p), dp(uvw), dp(Y), C.c_longlong(n), dp(U))
    return U


def ns_rhs(U, dx, part=0, m64=None, s=4, dy=None, dz=None) -> np.ndarray:
    _, nz, ny, nx = U.shape
    if m64 is None:
        m64, s = build_narrow(8, (3557.0 / 44100.0, -2083.0 / 117600.0))
    out = np.empty_like(U)
    dy = dx if dy is None else dy
    dz = dx if dz is None else dz
    rc = lib().or_ns_rhs(dp(U), nx, ny, nz, C.c_double(dx), C.c_double(dy), C.c_double(dz),
                         dp(m64), s, part, dp(out))
    assert rc == 0
    return out


def set_threads(n: int = 0) -> int:
    """OpenMP threads of the oracle's loops (0 = every host thread); results
    are bitwise independent of it.  Returns the count in effect."""
    lib().or_set_threads(int(n))
    lib().or_get_threads.restype = C.c_int
    return int(lib().or_get_threads())


def ns_chem_gross(U) -> np.ndarray:
    """Per-species gross chemistry magnitude (see ns_oracle.h)."""
    n = U[0].size
    g = np.empty((9,) + U.shape[1:])
    lib().or_ns_chem_gross(dp(U), C.c_longlong(n), dp(g))
    return g


def ns_rhs_terms(U, dx, terms, part=0, m64=None, s=4) -> np.ndarray:
    """or_ns_rhs_terms: the RHS restricted to the OR_T_* terms in `terms`."""
    _, nz, ny, nx = U.shape
    if m64 is None:
        m64, s = build_narrow(8, (3557.0 / 44100.0, -2083.0 / 117600.0))
    out = np.empty_like(U)
    rc = lib().or_ns_rhs_terms(dp(U), nx, ny, nz, C.c_double(dx), C.c_double(dx), C.c_double(dx),
                               dp(m64), s, part, int(terms), dp(out))
    assert rc == 0
    return out


def ns_callback(shape, dx, part, counter=None):
    """RHS_CB evaluating the NS oracle on a state of `shape` (14, nz, ny, nx)."""
    def f(t, u, out, dim, ctx):
        uu = np.ctypeslib.as_array(u, shape=(dim,)).reshape(shape)
        np.ctypeslib.as_array(out, shape=(dim,))[:] = ns_rhs(uu, dx, part).ravel()
        if counter is not None:
            counter[0] += 1
    return RHS_CB(f)


def integrate_sdc(fcb, u0, t0, t1, nsteps, nodes, q, s, iterations=4, cutoff=0.0):
    """or_integrate_sdc (sdc.cpp:38-127 restated): (u, sweeps, fresh_evals)."""
    u0 = np.ascontiguousarray(u0, dtype=np.float64).ravel()
    uo = np.empty_like(u0)
    res = np.zeros(256)
    sw, fe, es = C.c_int(), C.c_int(), C.c_int()
    D = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    nodes, q, s = D(nodes), D(q), D(s)
    rc = lib().or_integrate_sdc(fcb, None, u0.size, dp(u0), C.c_double(t0), C.c_double(t1),
                                nsteps, len(nodes) - 1, dp(nodes), dp(q), dp(s), iterations,
                                C.c_double(cutoff), 1, dp(uo), dp(res), res.size, C.byref(sw),
                                C.byref(fe), C.byref(es))
    assert rc == 0
    return uo, sw.value, fe.value


def integrate_mrsdc1(f1cb, f2cb, u0, t0, t1, nsteps, h, iterations=4, cutoff=0.0):
    """or_integrate_mrsdc1 (mrsdc.cpp:43-135, :227-259 restated) with the
    hierarchy dict h (coarse, fine, s21, q21, s22, q22, fine_of_coarse,
    p_map): (u, sweeps, f1_evals, f2_evals)."""
    u0 = np.ascontiguousarray(u0, dtype=np.float64).ravel()
    uo = np.empty_like(u0)
    res = np.zeros(256)
    sw, n1, n2 = C.c_int(), C.c_int(), C.c_int()
    D = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    I = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
    arrs = [D(h[k]) for k in ("coarse", "fine", "s21", "q21", "s22", "q22")]
    foc, pm = I(h["fine_of_coarse"]), I(h["p_map"])
    rc = lib().or_integrate_mrsdc1(
        f1cb, None, f2cb, None, u0.size, dp(u0), C.c_double(t0), C.c_double(t1), nsteps,
        len(arrs[0]) - 1, dp(arrs[0]), len(arrs[1]) - 1, dp(arrs[1]), dp(arrs[2]), dp(arrs[3]),
        dp(arrs[4]), dp(arrs[5]), ip(foc), ip(pm), iterations, C.c_double(cutoff), dp(uo),
        dp(res), res.size, C.byref(sw), C.byref(n1), C.byref(n2))
    assert rc == 0
    return uo, sw.value, n1.value, n2.value


def ns_temperature_pressure(U):
    n = U[0].size
    T, p = np.empty(U.shape[1:]), np.empty(U.shape[1:])
    lib().or_ns_temperature_pressure(dp(U), C.c_longlong(n), dp(T), dp(p))
    return T, p


# ------------------------------------------------ implicit (MRSDC mode 2)
class Stiff(C.Structure):
    """or_stiff (oracle.h): StiffOptions + the block structure of f1."""
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("max_newton_iters", C.c_int),
                ("block", C.c_longlong), ("interleaved", C.c_int)]


class NewtonReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("final_residual", C.c_double), ("converged", C.c_int),
                ("f_evals", C.c_int)]


def _stiff(rtol=1e-8, atol=1e-10, max_newton_iters=16, block=0, interleaved=False) -> Stiff:
    return Stiff(rtol, atol, max_newton_iters, block, int(interleaved))


def solve_backward_euler(fcb, dim, t, beta, c, guess, **stiff):
    """or_solve_backward_euler; fcb is an RHS_CB.  Returns (w, report)."""
    w = np.empty(dim)
    rep = NewtonReport()
    st = _stiff(**stiff)
    rc = lib().or_solve_backward_euler(fcb, None, C.c_longlong(dim), C.c_double(t),
                                       C.c_double(beta), dp(c), dp(guess), C.byref(st), dp(w),
                                       C.byref(rep))
    assert rc == 0
    return w, rep


def ref_solve_backward_euler(fcb, dim, t, beta, c, guess, rtol=1e-8, atol=1e-10,
                             max_newton_iters=16):
    w = np.empty(dim)
    ints = np.zeros(3, dtype=np.int32)
    fr = C.c_double()
    rc = ref().ref_solve_backward_euler(fcb, None, C.c_longlong(dim), C.c_double(t),
                                        C.c_double(beta), dp(c), dp(guess), C.c_double(rtol),
                                        C.c_double(atol), max_newton_iters, dp(w), ip(ints),
                                        C.byref(fr))
    if rc:
        raise RuntimeError(ref().ref_last_error().decode())
    return w, dict(iterations=int(ints[0]), converged=bool(ints[1]), f_evals=int(ints[2]),
                   final_residual=fr.value)


def integrate_mrsdc2(f1cb, f2cb, u0, t0, t1, nsteps, h, iterations=4, cutoff=0.0, **stiff):
    """or_integrate_mrsdc2 with hierarchy h (ref_hierarchy dict).  Returns
    (rc, u, diag dict)."""
    D = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    u0 = D(u0)
    dim = u0.size
    m1, m2 = len(h["coarse"]) - 1, len(h["fine"]) - 1
    uo = np.empty(dim)
    res = np.zeros(4096)
    ints = [C.c_int() for _ in range(7)]
    st = _stiff(**stiff)
    foc = np.ascontiguousarray(h["fine_of_coarse"], dtype=np.int32)
    arrs = [D(h[k]) for k in ("coarse", "fine", "s21", "q21", "s22", "q22")]
    rc = lib().or_integrate_mrsdc2(
        f1cb, None, f2cb, None, C.c_longlong(dim), dp(u0), C.c_double(t0), C.c_double(t1), nsteps,
        m1, dp(arrs[0]), m2, dp(arrs[1]), dp(arrs[2]), dp(arrs[3]), dp(arrs[4]), dp(arrs[5]),
        ip(foc), iterations, C.c_double(cutoff), C.byref(st), dp(uo), dp(res), res.size,
        *[C.byref(i) for i in ints])
    sw, n1, n2, imp, nf1, fnode, fsweep = (i.value for i in ints)
    return rc, uo, dict(sweeps=sw, f1_evals=n1, f2_evals=n2, implicit_solves=imp,
                        newton_f1_evals=nf1, residuals=res[:sw].copy(), fail_node=fnode,
                        fail_sweep=fsweep)


def ref_integrate_mrsdc2(f1cb, f2cb, u0, t0, t1, nsteps, coarse_n=3, fine_type=1, fine_n=5,
                         repeats=1, iterations=4, cutoff=0.0, rtol=1e-8, atol=1e-10,
                         max_newton_iters=16, coarse_family=0, fine_family=0):
    """The reference's integrate_mrsdc with f1 implicit.  Returns (rc, u, diag
    dict, error message)."""
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    dim = u0.size
    uo = np.empty(dim)
    res = np.zeros(4096)
    ints = [C.c_int() for _ in range(5)]
    r = ref()
    rc = r.ref_integrate_mrsdc2(
        f1cb, None, f2cb, None, C.c_longlong(dim), dp(u0), C.c_double(t0), C.c_double(t1), nsteps,
        coarse_family, coarse_n, fine_type, fine_family, fine_n, repeats, iterations,
        C.c_double(cutoff), C.c_double(rtol), C.c_double(atol), max_newton_iters, dp(uo), dp(res),
        res.size, *[C.byref(i) for i in ints])
    sw, n1, n2, imp, nf1 = (i.value for i in ints)
    msg = r.ref_last_error().decode() if rc else ""
    return rc, uo, dict(sweeps=sw, f1_evals=n1, f2_evals=n2, implicit_solves=imp,
                        newton_f1_evals=nf1, residuals=res[:sw].copy()), msg


def integrate_stiff(fcb, u0, t0, t1, initial_step_fraction=1e-3, **stiff):
    """or_integrate_stiff: (rc, u, accepted, rejected)."""
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    uo = np.empty_like(u0)
    acc, rej, tf = C.c_int(), C.c_int(), C.c_double()
    st = _stiff(**stiff)
    rc = lib().or_integrate_stiff(fcb, None, C.c_longlong(u0.size), dp(u0), C.c_double(t0),
                                  C.c_double(t1), C.byref(st), C.c_double(initial_step_fraction),
                                  dp(uo), C.byref(acc), C.byref(rej), C.byref(tf))
    return rc, uo, acc.value, rej.value


def ref_integrate_stiff(fcb, u0, t0, t1, rtol=1e-8, atol=1e-10, max_newton_iters=16,
                        initial_step_fraction=1e-3):
    """The reference's integrate_stiff: (rc, u, error message)."""
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    uo = np.empty_like(u0)
    r = ref()
    rc = r.ref_integrate_stiff(fcb, None, C.c_longlong(u0.size), dp(u0), C.c_double(t0),
                               C.c_double(t1), C.c_double(rtol), C.c_double(atol),
                               max_newton_iters, C.c_double(initial_step_fraction), dp(uo))
    return rc, uo, (r.ref_last_error().decode() if rc else "")
