"""One MRSDC mode-2 step (chemistry implicit on GL(3) coarse nodes via the
per-cell block Newton, advection-diffusion explicit on GL(5) fine nodes) on
the configs[4] ignition state at n^3; prints ms/step and the counts."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_7327_b200 as P  # noqa: E402
from paper_1309_7327_b200 import workloads as W  # noqa: E402
from bench import acoustic_dt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dev = torch.device("cuda:0")
T, p, uvw, Y = W.ns_primitives(n, ignition=True)
dt = 2.0 * acoustic_dt(T, p, uvw, Y, 1e-4)
U = P.ns_conserved(*(torch.from_numpy(x).to(dev) for x in (T, p, uvw, Y)))
op = P.NsOperator(n, n, n, 1e-4)
st = P.MrsdcStepper(3, 5, P.StepControls(4, 0.0), stiff=P.StiffOptions(block=14, interleaved=True))
st.integrate_mode2(op.chem, op.advdiff, U, 0.0, dt, 1)
torch.cuda.synchronize()
t = time.perf_counter()
out, d = st.integrate_mode2(op.chem, op.advdiff, U, 0.0, dt, 1)
torch.cuda.synchronize()
print(f"mode2 {n}^3: {1e3 * (time.perf_counter() - t):.1f} ms/step, solves {d.implicit_solves}, "
      f"newton f1 evals {d.newton_f1_evals}, f1 {d.f1_evals}, f2 {d.f2_evals}")
