"""ctypes bindings of the C ABI (include/smc_b200.h) for Python callers
(tests, bench.py).  No fallback: if libsmc_b200.so is missing or cannot be
loaded, every entry point raises."""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# SMC_LIB_PATH points at another build of the same library (A/B timing of two
# builds on one box); the default is the in-tree build.
LIB_PATH = os.environ.get("SMC_LIB_PATH") or os.path.join(HERE, "libsmc_b200.so")
HEADER = os.path.join(HERE, "..", "include", "smc_b200.h")

OK, EINVAL, EINTEGRATION, ECUDA = 0, 1, 2, 3
HOST, DEVICE = 0, 1
NARROW8, NARROW6, WIDE8 = 0, 1, 2
GAUSS_LOBATTO, CLENSHAW_CURTIS = 0, 1

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_VP = C.c_void_p

RHS_FN = C.CFUNCTYPE(None, C.c_double, _D, _D, C.c_longlong, C.c_void_p)
TIME_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)
FIELD_FN = C.CFUNCTYPE(None, C.c_double, _D, C.c_void_p)
REDUCE_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)
DEV_RHS_FN = C.CFUNCTYPE(None, C.c_double, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p,
                         C.c_void_p)


class SmcError(RuntimeError):
    pass


class SmcInvalidArgument(SmcError, ValueError):
    pass


class SmcIntegrationError(SmcError):
    pass


class Diag(C.Structure):
    _fields_ = [("sweeps", C.c_int), ("fresh_evals", C.c_int), ("f1_evals", C.c_int),
                ("f2_evals", C.c_int), ("early_stop", C.c_int), ("nonfinite", C.c_int),
                ("n_residuals", C.c_int), ("residual_capacity", C.c_int), ("residuals", _D),
                ("implicit_solves", C.c_int), ("newton_f1_evals", C.c_int)]


class Stiff(C.Structure):
    """smc_stiff: StiffOptions (stiff.hpp:10-20) + block structure of f."""
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("max_newton_iters", C.c_int),
                ("block", C.c_longlong), ("interleaved", C.c_int),
                ("initial_step_fraction", C.c_double)]


class NewtonReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("final_residual", C.c_double), ("converged", C.c_int),
                ("f_evals", C.c_int)]


_lib = None

# name -> (restype, argtypes)
_SIG = {
    "smc_version": (C.c_int, []),
    "smc_last_error": (C.c_char_p, []),
    "smc_launch_count": (C.c_longlong, []),
    "smc_synchronize": (C.c_int, []),
    "smc_measure_fp64_peak": (C.c_int, [C.c_int, _D]),
    "smc_measure_dmma_peak": (C.c_int, [C.c_int, C.c_int, _D]),
    "smc_measure_fp64_variants": (C.c_int, [C.c_int, _D, C.c_int]),
    "smc_build_narrow": (C.c_int, [C.c_int, _D, C.c_int, _D, _I]),
    "smc_apply_narrow": (C.c_int, [C.c_int, _D, C.c_int, _VP, _VP, C.c_int, C.c_double, _VP,
                                   C.c_int]),
    "smc_first_derivative8": (C.c_int, [_VP, C.c_int, C.c_double, _VP, C.c_int]),
    "smc_apply_narrow_bounded": (C.c_int, [_D, C.c_int, _VP, _VP, C.c_int, C.c_int, C.c_double,
                                           _VP, C.c_int]),
    "smc_first_derivative_bounded": (C.c_int, [_VP, C.c_int, C.c_int, C.c_double, _VP,
                                               C.c_int]),
    "smc_apply_wide": (C.c_int, [_VP, _VP, C.c_int, C.c_double, _VP, C.c_int]),
    "smc_heat_create": (C.c_int, [C.c_int, C.c_int, C.c_int, _D, _D, _D, _D, C.POINTER(_VP)]),
    "smc_heat_set_time_source": (C.c_int, [_VP, TIME_FN, _VP]),
    "smc_heat_set_full_source": (C.c_int, [_VP, FIELD_FN, _VP]),
    "smc_narrow3d_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                      C.c_double, C.c_int, _D, C.c_int, _VP, C.c_int,
                                      C.POINTER(_VP)]),
    "smc_narrow3d_set_kc": (C.c_int, [_VP, C.c_int]),
    "smc_narrow3d_create_slab": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                           C.c_double, C.c_double, C.c_int, _D, C.c_int, _VP,
                                           C.c_int, C.POINTER(_VP)]),
    "smc_narrow3d_apply_planes": (C.c_int, [_VP, _VP, _VP, C.c_int, C.c_int]),
    "smc_narrow3d_apply_peer": (C.c_int, [_VP, _VP, _VP, C.c_int, _VP, _VP, C.c_int, C.c_int]),
    "smc_ipc_export": (C.c_int, [_VP, C.c_char_p]),
    "smc_ipc_import": (C.c_int, [C.c_char_p, C.POINTER(_VP)]),
    "smc_ipc_close": (C.c_int, [_VP]),
    "smc_device_alloc": (C.c_int, [C.c_longlong, C.POINTER(_VP)]),
    "smc_device_free": (C.c_int, [_VP]),
    "smc_ns_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                C.c_double, C.c_int, _D, C.c_int, C.POINTER(_VP), C.POINTER(_VP),
                                C.POINTER(_VP)]),
    "smc_ns_rhs_ghosted": (C.c_int, [_VP, _VP, _VP]),
    "smc_ns_temperature_pressure": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int]),
    "smc_ns_profile": (C.c_int, [_VP, _VP, _VP, _D, C.POINTER(C.c_char_p), C.c_int, _I]),
    "smc_ns_conserved": (C.c_int, [_VP, _VP, _VP, _VP, C.c_longlong, _VP, C.c_int]),
    "smc_rhs_from_callback": (C.c_int, [C.c_longlong, RHS_FN, _VP, C.POINTER(_VP)]),
    "smc_rhs_from_device_callback": (C.c_int, [C.c_longlong, DEV_RHS_FN, _VP, C.POINTER(_VP)]),
    "smc_rhs_eval": (C.c_int, [_VP, C.c_double, _VP, _VP, C.c_int]),
    "smc_rhs_dim": (C.c_longlong, [_VP]),
    "smc_rhs_set_stream": (C.c_int, [_VP, _VP]),
    "smc_rhs_destroy": (C.c_int, [_VP]),
    "smc_nodes": (C.c_int, [C.c_int, C.c_int, _D]),
    "smc_integration_matrices": (C.c_int, [C.c_int, C.c_int, _D, _D]),
    "smc_build_hierarchy": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _I, _D, _D,
                                      _D, _D, _D, _I, _I]),
    "smc_sdc_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                 C.POINTER(_VP)]),
    "smc_sdc_step": (C.c_int, [_VP, _VP, _VP, C.c_double, C.c_double, _VP, _VP, _VP, C.c_int,
                               C.POINTER(Diag)]),
    "smc_sdc_integrate": (C.c_int, [_VP, _VP, _VP, C.c_double, C.c_double, C.c_int, _VP,
                                    C.c_int, C.POINTER(Diag)]),
    "smc_sdc_set_reducer": (C.c_int, [_VP, REDUCE_FN, _VP]),
    "smc_sdc_destroy": (C.c_int, [_VP]),
    "smc_mrsdc_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_double, C.c_int, C.POINTER(_VP)]),
    "smc_mrsdc_step_mode1": (C.c_int, [_VP, _VP, _VP, _VP, C.c_double, C.c_double, _VP, _VP,
                                       _VP, _VP, _VP, C.c_int, C.POINTER(Diag)]),
    "smc_mrsdc_integrate_mode1": (C.c_int, [_VP, _VP, _VP, _VP, C.c_double, C.c_double, C.c_int,
                                            _VP, C.c_int, C.POINTER(Diag)]),
    "smc_mrsdc_set_stiff": (C.c_int, [_VP, C.POINTER(Stiff)]),
    "smc_mrsdc_step_mode2": (C.c_int, [_VP, _VP, _VP, _VP, C.c_double, C.c_double, _VP, _VP,
                                       _VP, _VP, _VP, C.c_int, C.POINTER(Diag)]),
    "smc_mrsdc_integrate_mode2": (C.c_int, [_VP, _VP, _VP, _VP, C.c_double, C.c_double, C.c_int,
                                            _VP, C.c_int, C.POINTER(Diag)]),
    "smc_solve_backward_euler": (C.c_int, [_VP, C.c_double, C.c_double, _VP, _VP, _VP, C.c_int,
                                           C.POINTER(Stiff), C.POINTER(NewtonReport)]),
    "smc_integrate_stiff": (C.c_int, [_VP, _VP, C.c_double, C.c_double, _VP, C.c_int,
                                      C.POINTER(Stiff), _I, _I]),
    "smc_mrsdc_set_reducer": (C.c_int, [_VP, REDUCE_FN, _VP]),
    "smc_comm_unique_id": (C.c_int, [C.c_char_p]),
    "smc_comm_init": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(_VP)]),
    "smc_comm_init_local": (C.c_int, [C.c_int, C.POINTER(_VP)]),
    "smc_comm_rank": (C.c_int, [_VP, _I, _I]),
    "smc_comm_allreduce_max": (C.c_int, [_VP, _D]),
    "smc_comm_destroy": (C.c_int, [_VP]),
    "smc_ns_slab_create": (C.c_int, [_VP, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                     C.c_double, C.c_int, _D, C.c_int, C.POINTER(_VP),
                                     C.POINTER(_VP), C.POINTER(_VP)]),
    "smc_ns_slab_publish": (C.c_int, [_VP, _VP]),
    "smc_sdc_set_comm": (C.c_int, [_VP, _VP]),
    "smc_mrsdc_set_comm": (C.c_int, [_VP, _VP]),
    "smc_mrsdc_destroy": (C.c_int, [_VP]),
}


def header_symbols() -> list[str]:
    """Every function declared in include/smc_b200.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(smc_\w+)\s*\(", text,
                                 flags=re.M)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SmcError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                           "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIG.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


# Exceptions raised inside Python callbacks (RHS trampolines, reducers) cannot
# cross the C frames that called them: ctypes would print and swallow them and
# hand the C side an undefined value.  The trampolines store them here and
# return a poisoned value (NaN); check() re-raises after the C call returns.
_pending: list = []


def defer(exc: BaseException) -> None:
    _pending.append(exc)


def check(rc: int) -> None:
    if _pending:
        exc = _pending[0]
        _pending.clear()
        raise exc
    if rc == OK:
        return
    msg = lib().smc_last_error().decode()
    if rc == EINVAL:
        raise SmcInvalidArgument(msg)
    if rc == EINTEGRATION:
        raise SmcIntegrationError(msg)
    raise SmcError(msg)


def dptr(a) -> C.c_void_p:
    """Raw pointer of a C-contiguous float64 numpy array or torch tensor."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not (a.is_contiguous() and str(a.dtype) == "torch.float64"):
            raise SmcInvalidArgument("expected a contiguous torch.float64 tensor")
        return C.c_void_p(a.data_ptr())
    if not (getattr(a, "dtype", None) is not None and a.dtype.name == "float64"
            and a.flags.c_contiguous):
        raise SmcInvalidArgument("expected a C-contiguous float64 numpy array")
    return C.c_void_p(a.ctypes.data)


def numel(a) -> int:
    return int(a.numel()) if hasattr(a, "numel") else int(a.size)


def check_arrays(dim: int, *arrays, names=None) -> int:
    """The C side copies / reads dim doubles through every array argument:
    each given array (None = absent) must hold exactly dim float64 values and
    all of them must live on the same side (host numpy or CUDA tensor);
    device arrays must be 16-byte aligned (the kernels' vector accesses).
    Returns the common where_of."""
    where = None
    for i, a in enumerate(arrays):
        if a is None:
            continue
        name = names[i] if names else f"argument {i}"
        dptr(a)  # dtype / contiguity
        if numel(a) != dim:
            raise SmcInvalidArgument(f"{name}: holds {numel(a)} values, the operator's "
                                     f"dimension is {dim}")
        w = where_of(a)
        if where is None:
            where = w
        elif w != where:
            raise SmcInvalidArgument(f"{name}: host and device arrays mixed in one call")
        if w == DEVICE and a.data_ptr() % 16:
            raise SmcInvalidArgument(f"{name}: device array is not 16-byte aligned")
    return HOST if where is None else where


def where_of(a) -> int:
    return DEVICE if hasattr(a, "is_cuda") and a.is_cuda else HOST


def cdouble_array(vals):
    arr = (C.c_double * max(1, len(vals)))(*vals)
    return C.cast(arr, _D), arr
