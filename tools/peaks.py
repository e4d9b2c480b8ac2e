import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1309_7327_b200 import _capi
L = _capi.lib()
v = C.c_double()
L.smc_measure_fp64_peak(20000, C.byref(v)); print("dfma", v.value)
L.smc_measure_dmma_peak(20000, 0, C.byref(v)); print("dmma", v.value)
L.smc_measure_dmma_peak(20000, 1, C.byref(v)); print("mixed", v.value)
