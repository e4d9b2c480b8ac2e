"""B200-native RHS hot path of the SMC method (arXiv 1309.7327).

Python view of the C ABI (include/smc_b200.h) for tests and bench.py.  The
names mirror the reference `nsdc` C++ API (/root/reference/proj/core/include/nsdc):
build_narrow / apply_narrow / apply_wide / first_derivative8 (stencil.hpp),
HeatOperator (pde.hpp), SdcStepper / integrate_sdc (sdc.hpp), MrsdcStepper /
integrate_mrsdc (mrsdc.hpp), gauss_lobatto / integration_matrices /
build_hierarchy (quadrature.hpp).  The C++ drop-in with the reference's exact
signatures is include/nsdc_b200/.

Arrays: numpy float64 (host, synchronous) or torch.float64 CUDA tensors
(device, stream-ordered on the operator's stream).  There is no CPU fallback:
without libsmc_b200.so (built by __graft_entry__.build()) every call raises.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import (CLENSHAW_CURTIS, DEVICE, GAUSS_LOBATTO, HOST, NARROW6, NARROW8, WIDE8,
                    SmcError, SmcIntegrationError, SmcInvalidArgument, check, check_arrays, defer,
                    dptr, where_of)

__all__ = [
    "SmcError", "SmcInvalidArgument", "SmcIntegrationError", "StencilChoice", "stencil_preset",
    "build_narrow", "apply_narrow", "apply_wide", "first_derivative8",
    "apply_narrow_bounded", "first_derivative_bounded", "HeatOperator",
    "Narrow3DOperator", "Narrow3DSlab", "CallbackRhs", "DeviceCallbackRhs", "SdcStepper",
    "MrsdcStepper", "StepControls", "StiffOptions", "NewtonReport", "solve_backward_euler", "integrate_stiff", "nodes",
    "integration_matrices", "build_hierarchy", "SMC_M47", "SMC_M48", "OPTIMAL_M47", "NsOperator",
    "ns_conserved", "NS_FULL", "NS_ADVDIFF", "NS_CHEM",
    "OPTIMAL_M48", "DEFAULT_M36", "launch_count",
]

# stencil.hpp:29-35
SMC_M47 = 3557.0 / 44100.0
SMC_M48 = -2083.0 / 117600.0
OPTIMAL_M47 = 1059283.0 / 13608000.0
OPTIMAL_M48 = -856481.0 / 40824000.0
DEFAULT_M36 = 281.0 / 3600.0


def launch_count() -> int:
    return int(_capi.lib().smc_launch_count())


@dataclass
class StencilChoice:
    """StencilChoice (stencil.hpp:65-75)."""
    kind: int = NARROW8
    params: tuple = (SMC_M47, SMC_M48)

    @staticmethod
    def narrow8(m47, m48):
        return StencilChoice(NARROW8, (m47, m48))

    @staticmethod
    def narrow6(m36):
        return StencilChoice(NARROW6, (m36,))

    @staticmethod
    def wide8():
        return StencilChoice(WIDE8, ())

    @property
    def order(self) -> int:
        return 8 if self.kind == NARROW8 else 6


def stencil_preset(name: str) -> StencilChoice:
    """stencil_preset (stencil.cpp:235-242)."""
    table = {"SMC": StencilChoice.narrow8(SMC_M47, SMC_M48),
             "ZERO": StencilChoice.narrow8(0.0, 0.0),
             "OPTIMAL": StencilChoice.narrow8(OPTIMAL_M47, OPTIMAL_M48),
             "NARROW6": StencilChoice.narrow6(DEFAULT_M36),
             "WIDE": StencilChoice.wide8()}
    if name not in table:
        raise SmcInvalidArgument(f"unknown stencil preset: {name}")
    return table[name]


def _params(params):
    p = (C.c_double * 2)(*(list(params) + [0.0, 0.0])[:2])
    return C.cast(p, C.POINTER(C.c_double)), p


def build_narrow(order: int, params) -> tuple[np.ndarray, int]:
    m = np.zeros(64)
    s = C.c_int()
    pp, keep = _params(params)
    check(_capi.lib().smc_build_narrow(order, pp, len(params), m.ctypes.data_as(
        C.POINTER(C.c_double)), C.byref(s)))
    return m.reshape(8, 8), s.value


def _out_like(u):
    if hasattr(u, "is_cuda"):
        import torch
        return torch.empty_like(u)
    return np.empty_like(u)


def apply_narrow(order: int, params, a, u, dx: float):
    w = check_arrays(_capi.numel(u), a, u, names=("a", "u"))
    out = _out_like(u)
    pp, keep = _params(params)
    check(_capi.lib().smc_apply_narrow(order, pp, len(params), dptr(a), dptr(u), len(u), dx,
                                       dptr(out), w))
    return out


def first_derivative8(u, dx: float):
    w = check_arrays(_capi.numel(u), u, names=("u",))
    out = _out_like(u)
    check(_capi.lib().smc_first_derivative8(dptr(u), len(u), dx, dptr(out), w))
    return out


def apply_wide(a, u, dx: float):
    w = check_arrays(_capi.numel(u), a, u, names=("a", "u"))
    out = _out_like(u)
    check(_capi.lib().smc_apply_wide(dptr(a), dptr(u), len(u), dx, dptr(out), w))
    return out


def _lines(u):
    """(n, nlines) of a 1-D line or a (nlines, n) batch of lines."""
    shape = tuple(u.shape)
    if len(shape) == 1:
        return shape[0], 1
    if len(shape) == 2:
        return shape[1], shape[0]
    raise SmcInvalidArgument("expected one line (n,) or a batch of lines (nlines, n)")


def apply_narrow_bounded(a, u, dx: float, params=()):
    """(a u_x)_x on non-periodic lines with the paper's boundary closure
    (include/smc_b200.h smc_apply_narrow_bounded).  u, a:
    (n,) or (nlines, n); params = () / (m47, m48) / (m47, m48, m36)."""
    n, nl = _lines(u)
    w = check_arrays(n * nl, a, u, names=("a", "u"))
    if len(params) not in (0, 2, 3):
        raise SmcInvalidArgument("params: (), (m47, m48) or (m47, m48, m36)")
    keep = (C.c_double * 3)(*(list(params) + [0.0] * 3)[:3])
    out = _out_like(u)
    check(_capi.lib().smc_apply_narrow_bounded(C.cast(keep, C.POINTER(C.c_double)), len(params),
                                               dptr(a), dptr(u), n, nl, dx, dptr(out), w))
    return out


def first_derivative_bounded(u, dx: float):
    """du/dx on non-periodic lines with the paper's boundary closure."""
    n, nl = _lines(u)
    w = check_arrays(n * nl, u, names=("u",))
    out = _out_like(u)
    check(_capi.lib().smc_first_derivative_bounded(dptr(u), n, nl, dx, dptr(out), w))
    return out


class _Rhs:
    """Owner of an smc_rhs handle."""

    def __init__(self, handle):
        self._h = handle
        self._keep = []

    @property
    def handle(self):
        return self._h

    @property
    def dim(self) -> int:
        return int(_capi.lib().smc_rhs_dim(self._h))

    def set_stream(self, stream) -> None:
        """stream: torch.cuda.Stream, raw cudaStream_t int, or None."""
        raw = getattr(stream, "cuda_stream", stream)
        check(_capi.lib().smc_rhs_set_stream(self._h, C.c_void_p(raw or 0)))

    def __call__(self, t: float, u, out=None):
        """Rhs contract (field.hpp:14-16): out = f(t, u)."""
        if out is None:
            out = _out_like(u)
        w = check_arrays(self.dim, u, out, names=("u", "out"))
        check(_capi.lib().smc_rhs_eval(self._h, t, dptr(u), dptr(out), w))
        return out

    def close(self):
        if self._h:
            _capi.lib().smc_rhs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HeatOperator(_Rhs):
    """HeatOperator (pde.hpp:69-84) on the periodic [0, 2pi)^2 node grid.

    a, b, g_space: arrays (ny, nx) sampled on the nodes, or callables f(x, y);
    g_time: callable of t (separable source, pde.cpp:107-108) or None."""

    def __init__(self, nx: int, ny: int, choice: StencilChoice, a, b, g_space=None,
                 g_time=None):
        self.nx, self.ny = nx, ny
        xs = np.arange(nx) * (2 * math.pi / nx)
        ys = np.arange(ny) * (2 * math.pi / ny)

        def grid(f):
            if f is None:
                return None
            if callable(f):
                return np.ascontiguousarray(
                    np.array([[f(x, y) for x in xs] for y in ys], dtype=np.float64))
            return np.ascontiguousarray(f, dtype=np.float64)

        A, B, G = grid(a), grid(b), grid(g_space)
        h = C.c_void_p()
        pp, keep = _params(choice.params)
        D = C.POINTER(C.c_double)
        check(_capi.lib().smc_heat_create(nx, ny, choice.kind, pp, A.ctypes.data_as(D),
                                          B.ctypes.data_as(D),
                                          G.ctypes.data_as(D) if G is not None else None,
                                          C.byref(h)))
        super().__init__(h)
        if G is not None and g_time is not None:
            def gt(t, ctx):
                try:
                    return float(g_time(t))
                except BaseException as e:  # re-raised by check() after the C call
                    defer(e)
                    return math.nan

            cb = _capi.TIME_FN(gt)
            self._keep.append(cb)
            check(_capi.lib().smc_heat_set_time_source(self._h, cb, None))


class Narrow3DOperator(_Rhs):
    """(a U_x)_x + (a U_y)_y + (a U_z)_z on a periodic nz x ny x nx box."""

    def __init__(self, a, dx: float, dy: float, dz: float, choice: StencilChoice = None):
        choice = choice or StencilChoice()
        nz, ny, nx = a.shape
        self.shape = (nz, ny, nx)
        h = C.c_void_p()
        pp, keep = _params(choice.params)
        check(_capi.lib().smc_narrow3d_create(nx, ny, nz, dx, dy, dz, choice.order, pp,
                                              len(choice.params), dptr(a), where_of(a),
                                              C.byref(h)))
        super().__init__(h)

    def set_kc(self, kc: int) -> None:
        check(_capi.lib().smc_narrow3d_set_kc(self._h, kc))


class Narrow3DSlab(_Rhs):
    """The narrow operator on one z-slab of a block-decomposed periodic box:
    a (device tensor) has nz + 2*zghost planes; u passed to apply_planes too."""

    def __init__(self, a, nz: int, zghost: int, dx: float, dy: float, dz: float,
                 choice: StencilChoice = None):
        choice = choice or StencilChoice()
        nzg, ny, nx = a.shape
        assert nzg == nz + 2 * zghost
        self.nz, self.zghost = nz, zghost
        h = C.c_void_p()
        pp, keep = _params(choice.params)
        check(_capi.lib().smc_narrow3d_create_slab(nx, ny, nz, zghost, dx, dy, dz, choice.order,
                                                   pp, len(choice.params), dptr(a), where_of(a),
                                                   C.byref(h)))
        super().__init__(h)

    def apply_planes(self, u, out, kbeg: int, kend: int) -> None:
        check(_capi.lib().smc_narrow3d_apply_planes(self._h, dptr(u), dptr(out), kbeg, kend))

    def apply_peer(self, u, u_lo, nz_lo: int, u_hi, out, kbeg: int = 0, kend: int = None) -> None:
        """Peer halo: u holds only the nz interior planes; the ghost planes are
        read in the kernel from the neighbours' interior arrays u_lo / u_hi
        (tensors on this device or raw device pointers, e.g. IPC-mapped)."""
        kend = self.nz if kend is None else kend
        check(_capi.lib().smc_narrow3d_apply_peer(self._h, dptr(u), _ptr(u_lo), nz_lo, _ptr(u_hi),
                                                  dptr(out), kbeg, kend))

    def set_kc(self, kc: int) -> None:
        check(_capi.lib().smc_narrow3d_set_kc(self._h, kc))


def _ptr(x):
    """device pointer of a tensor, or a raw integer pointer as given"""
    return x if isinstance(x, int) else dptr(x)


class _CudaPtr:
    """Minimal __cuda_array_interface__ view of a raw device pointer."""

    def __init__(self, ptr: int, n: int, stream: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None,
                                         "stream": stream if stream else None}


def device_tensor(ptr: int, n: int, stream: int = 0):
    """torch.float64 CUDA tensor aliasing n doubles at device pointer ptr."""
    import torch
    return torch.as_tensor(_CudaPtr(ptr, n, stream), device="cuda")


class DeviceCallbackRhs(_Rhs):
    """fn(t, u, out) on torch CUDA tensors (views of the stepper's buffers),
    called with the operator's stream current; for RHS whose work includes
    host-issued collectives (multi-GPU halo exchange)."""

    def __init__(self, dim: int, fn):
        import torch

        def tramp(t, u, out, n, stream, ctx):
            try:
                s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
                with torch.cuda.stream(s):
                    fn(t, device_tensor(u, n, stream), device_tensor(out, n, stream))
            except BaseException as e:  # re-raised by check() after the C call
                defer(e)
                with torch.cuda.stream(s):
                    device_tensor(out, n, stream).fill_(math.nan)

        cb = _capi.DEV_RHS_FN(tramp)
        h = C.c_void_p()
        check(_capi.lib().smc_rhs_from_device_callback(dim, cb, None, C.byref(h)))
        super().__init__(h)
        self._keep.append(cb)


class CallbackRhs(_Rhs):
    """A Python callable f(t, u: np.ndarray) -> np.ndarray as an operator."""

    def __init__(self, dim: int, fn):
        def tramp(t, u, out, n, ctx):
            uu = np.ctypeslib.as_array(u, shape=(n,))
            oo = np.ctypeslib.as_array(out, shape=(n,))
            try:
                oo[:] = fn(t, uu)
            except BaseException as e:  # re-raised by check() after the C call
                defer(e)
                oo[:] = math.nan

        cb = _capi.RHS_FN(tramp)
        h = C.c_void_p()
        check(_capi.lib().smc_rhs_from_callback(dim, cb, None, C.byref(h)))
        super().__init__(h)
        self._keep.append(cb)


@dataclass
class StepControls:
    """StepControls (sdc.hpp:12-20)."""
    num_iterations: int = 4
    residual_ratio_cutoff: float = 0.05
    reuse_first_eval: bool = True


@dataclass
class SweepDiagnostics:
    residual_history: list = field(default_factory=list)
    sweeps: int = 0
    fresh_evals: int = 0
    f1_evals: int = 0
    f2_evals: int = 0
    early_stop: bool = False
    nonfinite: bool = False
    implicit_solves: int = 0     # MRSDC mode 2 (mrsdc.hpp:30-38)
    newton_f1_evals: int = 0


def _diag(cap=4096):
    buf = (C.c_double * cap)()
    d = _capi.Diag()
    d.residual_capacity = cap
    d.residuals = C.cast(buf, C.POINTER(C.c_double))
    return d, buf


def _from_diag(d, buf) -> SweepDiagnostics:
    n = min(d.n_residuals, d.residual_capacity)
    return SweepDiagnostics(list(buf[:n]), d.sweeps, d.fresh_evals, d.f1_evals, d.f2_evals,
                            bool(d.early_stop), bool(d.nonfinite), d.implicit_solves,
                            d.newton_f1_evals)


@dataclass
class StiffOptions:
    """StiffOptions (stiff.hpp:10-20) plus the block structure of the implicit
    term: f couples only the `block` components of one block (0 = dense).
    `interleaved`: component j of block b at j*(n/block) + b (structure of
    arrays — NsOperator state: block=14, interleaved=True), else b*block + j."""
    rtol: float = 1e-8
    atol: float = 1e-10
    max_newton_iters: int = 16
    block: int = 0
    interleaved: bool = False
    initial_step_fraction: float = 1e-3

    def c(self):
        return _capi.Stiff(self.rtol, self.atol, self.max_newton_iters, self.block,
                           int(self.interleaved), self.initial_step_fraction)


@dataclass
class NewtonReport:
    """NewtonReport (stiff.hpp:22-27)."""
    iterations: int = 0
    final_residual: float = 0.0
    converged: bool = False
    f_evals: int = 0


def integrate_stiff(f: "_Rhs", u0, t0: float, t1: float, stiff: "StiffOptions" = None):
    """integrate_stiff (stiff.cpp:115-188) on the device: adaptive backward Euler
    / variable-step BDF2 with step doubling.  Returns (u, (accepted, rejected))."""
    u = _out_like(u0)
    so = (stiff or StiffOptions()).c()
    acc, rej = C.c_int(), C.c_int()
    w = check_arrays(f.dim, u0, u, names=("u0", "u"))
    check(_capi.lib().smc_integrate_stiff(f.handle, dptr(u0), t0, t1, dptr(u), w,
                                          C.byref(so), C.byref(acc), C.byref(rej)))
    return u, (acc.value, rej.value)


def solve_backward_euler(f: "_Rhs", t: float, beta: float, c, guess, stiff: "StiffOptions" = None,
                         report: bool = True):
    """solve_backward_euler (stiff.cpp:34-76): w = c + beta f(t, w) by Newton
    from guess, on the device.  Returns (w, NewtonReport) with report=True;
    with report=False a failed solve raises SmcIntegrationError."""
    w = _out_like(c)
    rep = _capi.NewtonReport()
    so = (stiff or StiffOptions()).c()
    wh = check_arrays(f.dim, c, guess, w, names=("c", "guess", "w"))
    check(_capi.lib().smc_solve_backward_euler(f.handle, t, beta, dptr(c), dptr(guess), dptr(w),
                                               wh, C.byref(so),
                                               C.byref(rep) if report else None))
    return w, NewtonReport(rep.iterations, rep.final_residual, bool(rep.converged), rep.f_evals)


def _reducer(fn):
    def red(v, ctx):
        try:
            return float(fn(v))
        except BaseException as e:  # re-raised by check() after the C call
            defer(e)
            return math.nan

    return _capi.REDUCE_FN(red)


class SdcStepper:
    """Device-resident SdcStepper (sdc.hpp:45-69)."""

    def __init__(self, num_nodes: int = 3, controls: StepControls = None,
                 family: int = GAUSS_LOBATTO):
        c = controls or StepControls()
        h = C.c_void_p()
        check(_capi.lib().smc_sdc_create(family, num_nodes, c.num_iterations,
                                         c.residual_ratio_cutoff, int(c.reuse_first_eval),
                                         C.byref(h)))
        self._h = h
        self._keep = []

    def set_reducer(self, fn) -> None:
        """fn(local_max) -> global max over ranks (multi-GPU)."""
        cb = _reducer(fn)
        self._keep.append(cb)
        check(_capi.lib().smc_sdc_set_reducer(self._h, cb, None))

    def set_comm(self, comm) -> None:
        """Reduce the residual over a distributed.Comm's ranks (in the library)."""
        self._keep.append(comm)
        check(_capi.lib().smc_sdc_set_comm(self._h, comm.handle))

    def step(self, f: _Rhs, u0, t_n: float, dt: float, f0=None):
        u = _out_like(u0)
        fe = _out_like(u0)
        d, buf = _diag()
        w = check_arrays(f.dim, u0, f0, u, fe, names=("u0", "f0", "u", "f_end"))
        check(_capi.lib().smc_sdc_step(self._h, f.handle, dptr(u0), t_n, dt, dptr(f0), dptr(u),
                                       dptr(fe), w, C.byref(d)))
        return u, fe, _from_diag(d, buf)

    def integrate(self, f: _Rhs, u0, t0: float, t1: float, nsteps: int, out=None):
        u = out if out is not None else _out_like(u0)
        d, buf = _diag()
        w = check_arrays(f.dim, u0, u, names=("u0", "out"))
        check(_capi.lib().smc_sdc_integrate(self._h, f.handle, dptr(u0), t0, t1, nsteps, dptr(u),
                                            w, C.byref(d)))
        return u, _from_diag(d, buf)

    def __del__(self):
        try:
            _capi.lib().smc_sdc_destroy(self._h)
        except Exception:
            pass


class MrsdcStepper:
    """Device-resident MrsdcStepper (mrsdc.hpp:51-82), modes 1 and 2, hierarchy
    build_hierarchy(coarse, TypeB{inner}) (repeats=1) or TypeC{inner, repeats}.
    Mode 2 solves f1 implicitly with StiffOptions `stiff` (block structure:
    see StiffOptions)."""

    def __init__(self, coarse_nodes=3, inner_nodes=5, controls: StepControls = None, repeats=1,
                 coarse_family=GAUSS_LOBATTO, inner_family=GAUSS_LOBATTO,
                 stiff: StiffOptions = None):
        c = controls or StepControls()
        h = C.c_void_p()
        check(_capi.lib().smc_mrsdc_create(coarse_family, coarse_nodes, inner_family, inner_nodes,
                                           repeats, c.num_iterations, c.residual_ratio_cutoff,
                                           int(c.reuse_first_eval), C.byref(h)))
        self._h = h
        self._keep = []
        if stiff is not None:
            self.set_stiff(stiff)

    def set_stiff(self, stiff: StiffOptions) -> None:
        so = stiff.c()
        check(_capi.lib().smc_mrsdc_set_stiff(self._h, C.byref(so)))

    def set_reducer(self, fn) -> None:
        cb = _reducer(fn)
        self._keep.append(cb)
        check(_capi.lib().smc_mrsdc_set_reducer(self._h, cb, None))

    def set_comm(self, comm) -> None:
        """Reduce the residual and the implicit solver's norms over a
        distributed.Comm's ranks (in the library)."""
        self._keep.append(comm)
        check(_capi.lib().smc_mrsdc_set_comm(self._h, comm.handle))

    def step_mode1(self, f1: _Rhs, f2: _Rhs, u0, t_n, dt, f0_1=None, f0_2=None):
        u, e1, e2 = _out_like(u0), _out_like(u0), _out_like(u0)
        d, buf = _diag()
        w = self._arrays(f1, f2, u0, f0_1, f0_2, u, e1, e2)
        check(_capi.lib().smc_mrsdc_step_mode1(self._h, f1.handle, f2.handle, dptr(u0), t_n, dt,
                                               dptr(f0_1), dptr(f0_2), dptr(u), dptr(e1),
                                               dptr(e2), w, C.byref(d)))
        return u, e1, e2, _from_diag(d, buf)

    def integrate_mode1(self, f1: _Rhs, f2: _Rhs, u0, t0, t1, nsteps, out=None):
        return self._integrate(1, f1, f2, u0, t0, t1, nsteps, out)

    def step_mode2(self, f1: _Rhs, f2: _Rhs, u0, t_n, dt, f0_1=None, f0_2=None):
        u, e1, e2 = _out_like(u0), _out_like(u0), _out_like(u0)
        d, buf = _diag()
        w = self._arrays(f1, f2, u0, f0_1, f0_2, u, e1, e2)
        check(_capi.lib().smc_mrsdc_step_mode2(self._h, f1.handle, f2.handle, dptr(u0), t_n, dt,
                                               dptr(f0_1), dptr(f0_2), dptr(u), dptr(e1),
                                               dptr(e2), w, C.byref(d)))
        return u, e1, e2, _from_diag(d, buf)

    def integrate_mode2(self, f1: _Rhs, f2: _Rhs, u0, t0, t1, nsteps, out=None):
        return self._integrate(2, f1, f2, u0, t0, t1, nsteps, out)

    @staticmethod
    def _arrays(f1, f2, *arrays):
        if f1.dim != f2.dim:
            raise SmcInvalidArgument("mrsdc: f1 and f2 have different dimensions")
        return check_arrays(f1.dim, *arrays)

    def _integrate(self, mode, f1, f2, u0, t0, t1, nsteps, out):
        u = out if out is not None else _out_like(u0)
        d, buf = _diag()
        fn = _capi.lib().smc_mrsdc_integrate_mode2 if mode == 2 else \
            _capi.lib().smc_mrsdc_integrate_mode1
        w = self._arrays(f1, f2, u0, u)
        check(fn(self._h, f1.handle, f2.handle, dptr(u0), t0, t1, nsteps, dptr(u), w,
                 C.byref(d)))
        return u, _from_diag(d, buf)

    def __del__(self):
        try:
            _capi.lib().smc_mrsdc_destroy(self._h)
        except Exception:
            pass


# ---------------------------------------------------------------- quadrature
def nodes(family: int, n: int) -> np.ndarray:
    t = np.zeros(n)
    check(_capi.lib().smc_nodes(family, n, t.ctypes.data_as(C.POINTER(C.c_double))))
    return t


def integration_matrices(family: int, n: int):
    q = np.zeros((n - 1, n))
    s = np.zeros((n - 1, n))
    D = C.POINTER(C.c_double)
    check(_capi.lib().smc_integration_matrices(family, n, q.ctypes.data_as(D),
                                               s.ctypes.data_as(D)))
    return q, s


def build_hierarchy(coarse_n, inner_n, repeats=1, coarse_family=GAUSS_LOBATTO,
                    inner_family=GAUSS_LOBATTO) -> dict:
    D, I = C.POINTER(C.c_double), C.POINTER(C.c_int)
    L = _capi.lib()
    m2p1 = C.c_int()
    check(L.smc_build_hierarchy(coarse_family, coarse_n, inner_family, inner_n, repeats,
                                C.byref(m2p1), None, None, None, None, None, None, None))
    n2, m1 = m2p1.value, coarse_n - 1
    fine = np.zeros(n2)
    q21, s21 = np.zeros((n2 - 1, m1 + 1)), np.zeros((n2 - 1, m1 + 1))
    q22, s22 = np.zeros((n2 - 1, n2)), np.zeros((n2 - 1, n2))
    foc, pm = np.zeros(coarse_n, dtype=np.int32), np.zeros(n2, dtype=np.int32)
    check(L.smc_build_hierarchy(coarse_family, coarse_n, inner_family, inner_n, repeats,
                                C.byref(m2p1), fine.ctypes.data_as(D), q21.ctypes.data_as(D),
                                s21.ctypes.data_as(D), q22.ctypes.data_as(D),
                                s22.ctypes.data_as(D), foc.ctypes.data_as(I),
                                pm.ctypes.data_as(I)))
    return dict(fine=fine, q21=q21, s21=s21, q22=q22, s22=s22, fine_of_coarse=foc, p_map=pm)


# ------------------------------------------------------------------ NS RHS
NVAR = 14
NS_FULL, NS_ADVDIFF, NS_CHEM = 0, 1, 2


class NsOperator:
    """The reacting-NS RHS on a periodic nz x ny x nx box (zghost = 0) or on
    one z-slab with zghost ghost planes: .full, .advdiff (MRSDC f1) and
    .chem (MRSDC f2) are Rhs views sharing one device workspace."""

    def __init__(self, nx, ny, nz, dx, dy=None, dz=None, choice: StencilChoice = None,
                 zghost: int = 0):
        choice = choice or StencilChoice()
        dy = dy or dx
        dz = dz or dx
        self.shape = (nz, ny, nx)
        self.zghost = zghost
        hs = [C.c_void_p() for _ in range(3)]
        pp, keep = _params(choice.params)
        check(_capi.lib().smc_ns_create(nx, ny, nz, zghost, dx, dy, dz, choice.order, pp,
                                        len(choice.params), C.byref(hs[0]), C.byref(hs[1]),
                                        C.byref(hs[2])))
        self.full, self.advdiff, self.chem = (_Rhs(h) for h in hs)

    def set_stream(self, stream) -> None:
        for r in (self.full, self.advdiff, self.chem):
            r.set_stream(stream)

    def rhs_ghosted(self, U, out, part: int = NS_FULL) -> None:
        h = (self.full, self.advdiff, self.chem)[part].handle
        check(_capi.lib().smc_ns_rhs_ghosted(h, dptr(U), dptr(out)))

    def profile(self, U, out, part: int = NS_FULL):
        """One evaluation on device tensors with an event after every kernel:
        [(kernel, ms)] in launch order."""
        h = (self.full, self.advdiff, self.chem)[part].handle
        cap = 64
        ms = (C.c_double * cap)()
        names = (C.c_char_p * cap)()
        cnt = C.c_int()
        check(_capi.lib().smc_ns_profile(h, dptr(U), dptr(out), ms, names, cap, C.byref(cnt)))
        return [(names[i].decode(), ms[i]) for i in range(min(cnt.value, cap))]

    def temperature_pressure(self, U):
        nz, ny, nx = self.shape
        if hasattr(U, "is_cuda"):
            import torch
            T = torch.empty((nz, ny, nx), dtype=torch.float64, device=U.device)
            p = torch.empty_like(T)
        else:
            T, p = np.empty((nz, ny, nx)), np.empty((nz, ny, nx))
        check(_capi.lib().smc_ns_temperature_pressure(self.full.handle, dptr(U), dptr(T),
                                                      dptr(p), where_of(U)))
        return T, p


def ns_conserved(T, p, uvw, Y):
    """Conserved state (14 fields) from T, p, velocity (3 fields), Y (9 fields)."""
    n = T.size if not hasattr(T, "numel") else T.numel()
    shape = (NVAR,) + tuple(T.shape)
    if hasattr(T, "is_cuda"):
        import torch
        U = torch.empty(shape, dtype=torch.float64, device=T.device)
    else:
        U = np.empty(shape)
    check(_capi.lib().smc_ns_conserved(dptr(T), dptr(p), dptr(uvw), dptr(Y), n, dptr(U),
                                       where_of(T)))
    return U
