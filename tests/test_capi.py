"""CPU: the C-ABI library loads, exports every symbol include/smc_b200.h
declares, and its host-side logic (coupling matrix, quadrature tables,
argument validation) matches the reference — no GPU compute here."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_1309_7327_b200 as P
from paper_1309_7327_b200 import _capi


def test_library_exports_header():
    lib = C.CDLL(_capi.LIB_PATH)
    declared = _capi.header_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_capi._SIG), "bindings out of sync with the header"


def test_library_is_sm100a():
    # the fatbin must carry sm_100a SASS
    import subprocess
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in r.stdout


def test_build_narrow_matches_reference(golden):
    for key, order, p in (("m8_smc", 8, (P.SMC_M47, P.SMC_M48)), ("m8_zero", 8, (0.0, 0.0)),
                          ("m8_optimal", 8, (P.OPTIMAL_M47, P.OPTIMAL_M48)),
                          ("m6_default", 6, (P.DEFAULT_M36,))):
        m, s = P.build_narrow(order, p)
        assert np.array_equal(m.ravel(), golden[key]), key


def test_quadrature_matches_reference(golden):
    for fam, nm, n in ((0, "gl", 3), (0, "gl", 5), (1, "cc", 5)):
        q, s = P.integration_matrices(fam, n)
        np.testing.assert_allclose(q, golden[f"q_{nm}{n}"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(s, golden[f"s_{nm}{n}"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(P.nodes(fam, n), golden[f"nodes_{nm}{n}"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(P.nodes(0, 9), golden["nodes_gl9"], rtol=0, atol=1e-15)
    h = P.build_hierarchy(3, 5)
    for k in ("fine", "q21", "s21", "q22", "s22", "fine_of_coarse", "p_map"):
        np.testing.assert_allclose(h[k], golden[f"h_{k}"], rtol=0, atol=1e-15)
    # closed forms, quadrature_test.cpp:58-67
    q, s = P.integration_matrices(0, 3)
    np.testing.assert_allclose(s, [[5 / 24, 1 / 3, -1 / 24], [-1 / 24, 1 / 3, 5 / 24]], atol=1e-14)
    np.testing.assert_allclose(q, [[5 / 24, 1 / 3, -1 / 24], [1 / 6, 2 / 3, 1 / 6]], atol=1e-14)
    gl5 = P.nodes(0, 5)
    assert gl5[1] == pytest.approx(0.5 - np.sqrt(21) / 14, rel=1e-15)


def test_invalid_arguments_raise():
    with pytest.raises(P.SmcInvalidArgument):
        P.build_narrow(4, (0.0,))
    with pytest.raises(P.SmcInvalidArgument):
        P.build_narrow(8, (0.0,))
    # pde_test.cpp:243-263: grid too small / non-positive coefficient
    with pytest.raises(P.SmcInvalidArgument, match="too small"):
        P.HeatOperator(8, 20, P.stencil_preset("SMC"), lambda x, y: 1.0, lambda x, y: 1.0)
    with pytest.raises(P.SmcInvalidArgument, match="too small"):
        P.HeatOperator(20, 6, P.stencil_preset("NARROW6"), lambda x, y: 1.0, lambda x, y: 1.0)
    with pytest.raises(P.SmcInvalidArgument, match="too small"):
        P.HeatOperator(8, 8, P.stencil_preset("WIDE"), lambda x, y: 1.0, lambda x, y: 1.0)
    with pytest.raises(P.SmcInvalidArgument, match="not positive"):
        P.HeatOperator(20, 20, P.stencil_preset("SMC"), lambda x, y: np.cos(x), lambda x, y: 1.0)
    with pytest.raises(P.SmcInvalidArgument):
        P.stencil_preset("smc")
    with pytest.raises(P.SmcInvalidArgument):
        P.nodes(0, 1)


def test_presets():
    smc = P.stencil_preset("SMC")
    assert smc.kind == P.NARROW8 and smc.params == (P.SMC_M47, P.SMC_M48)
    assert P.stencil_preset("ZERO").params[0] == 0.0
    assert P.stencil_preset("WIDE").kind == P.WIDE8


def test_no_cpu_fallback(monkeypatch, tmp_path):
    """The product path fails loudly when the CUDA library is absent."""
    monkeypatch.setattr(_capi, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_capi, "_lib", None)
    with pytest.raises(_capi.SmcError, match="no CPU fallback"):
        _capi.lib()


def test_product_never_imports_oracle():
    root = os.path.dirname(P.__file__)
    for dirpath, _, files in os.walk(root):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text and "libnsdc_ref" not in text, f


def test_wrappers_validate_array_sizes():
    """The C side copies dim() doubles through every array argument, so the
    Python wrappers check sizes, dtype and host/device placement before any
    call (an undersized host array would overflow the staging copy)."""
    f = P.CallbackRhs(8, lambda t, u: u)
    with pytest.raises(P.SmcInvalidArgument, match="dimension is 8"):
        f(0.0, np.zeros(7))
    with pytest.raises(P.SmcInvalidArgument, match="dimension is 8"):
        f(0.0, np.zeros(8), np.zeros(9))
    with pytest.raises(P.SmcInvalidArgument, match="float64"):
        f(0.0, np.zeros(8, dtype=np.float32))
    st = P.SdcStepper(3, P.StepControls(2, 0.0))
    with pytest.raises(P.SmcInvalidArgument):
        st.step(f, np.zeros(8), 0.0, 0.1, f0=np.zeros(4))
    with pytest.raises(P.SmcInvalidArgument, match="different dimensions"):
        P.MrsdcStepper._arrays(f, P.CallbackRhs(9, lambda t, u: u), np.zeros(8))


def test_callback_exceptions_are_deferred():
    """An exception inside a callback is stored and re-raised by check() after
    the C call returns (ctypes cannot propagate it through C frames)."""
    _capi.defer(KeyError("from a callback"))
    with pytest.raises(KeyError, match="from a callback"):
        _capi.check(_capi.OK)
    _capi.check(_capi.OK)  # cleared


def test_allreduce_max_device_default():
    """Under NCCL the reducer's tensor lives on the current CUDA device; under
    gloo (and with one rank) it stays on the host."""
    from paper_1309_7327_b200.distributed import allreduce_max

    class Fake:
        def __init__(self, backend):
            self.backend, self.seen = backend, None

        def is_initialized(self):
            return True

        def get_world_size(self):
            return 2

        def get_backend(self):
            return self.backend

        class ReduceOp:
            MAX = "max"

        def all_reduce(self, t, op=None):
            self.seen = t.device.type

    d = Fake("gloo")
    assert allreduce_max(d)(3.5) == 3.5 and d.seen == "cpu"
