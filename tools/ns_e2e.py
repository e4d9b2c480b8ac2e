"""Time the NS RHS through the public API with pinned host buffers (the
library's z-chunk pipeline) at n^3: prints ms per call over `reps` calls.
SMC_NS_E2E_CHUNK selects the middle chunk size (planes)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1309_7327_b200 as P  # noqa: E402
from paper_1309_7327_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda:0")
U = P.ns_conserved(*(torch.from_numpy(a).to(dev) for a in W.ns_primitives(n, hot_spot=True)))
Uh = U.cpu().pin_memory()
Oh = torch.empty_like(Uh).pin_memory()
op = P.NsOperator(n, n, n, 1e-4)
op.full(0.0, Uh, Oh)
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    op.full(0.0, Uh, Oh)
    ts.append((time.perf_counter() - t0) * 1e3)
gb = 14 * 8 * n ** 3 / 1e9
t0 = time.perf_counter()
U.copy_(Uh)
torch.cuda.synchronize()
h2d = (time.perf_counter() - t0) * 1e3
t0 = time.perf_counter()
Oh.copy_(U)
torch.cuda.synchronize()
d2h = (time.perf_counter() - t0) * 1e3
print(f"chunk={os.environ.get('SMC_NS_E2E_CHUNK', 32)} e2e ms {min(ts):.1f} (median "
      f"{sorted(ts)[len(ts) // 2]:.1f}); H2D {h2d:.1f} ms ({gb / h2d * 1e3:.0f} GB/s), "
      f"D2H {d2h:.1f} ms ({gb / d2h * 1e3:.0f} GB/s)")
