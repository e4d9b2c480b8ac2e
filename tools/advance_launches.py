"""One SDC GL(3) K=4 step (configs[2] shape) and one MRSDC mode-1 step
(configs[4] shape) of the NS RHS at n^3 on cuda:0, for an ncu launch list
(`ncu --metrics gpu__time_duration.sum --clock-control none --csv`): the
kernel shares of a time step (RHS vs sweep kernels)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1309_7327_b200 as P
from paper_1309_7327_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
which = sys.argv[2] if len(sys.argv) > 2 else "sdc"
dev = torch.device('cuda:0')
T, p, uvw, Y = W.ns_primitives(n, ignition=(which != "sdc"))
U = P.ns_conserved(*(torch.from_numpy(a).to(dev) for a in (T, p, uvw, Y)))
op = P.NsOperator(n, n, n, 1e-4)
dt = 5e-8
if which == "sdc":
    st = P.SdcStepper(3, P.StepControls(4, 0.0))
    for _ in range(2):
        st.integrate(op.full, U, 0.0, dt, 1)
else:
    st = P.MrsdcStepper(3, 5, P.StepControls(4, 0.0))
    for _ in range(2):
        st.integrate_mode1(op.advdiff, op.chem, U, 0.0, dt, 1)
torch.cuda.synchronize()
print("done")
