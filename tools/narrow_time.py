"""Time the configs[1] narrow operator at n^3 on cuda:0 (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1309_7327_b200 as P  # noqa: E402
from paper_1309_7327_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
dev = torch.device("cuda:0")
a, u = W.narrow3d_inputs(n, xp=torch, device=dev)
op = P.Narrow3DOperator(a, 1 / n, 1 / n, 1 / n)
out = torch.empty_like(u)
for _ in range(20):
    op(0.0, u, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    op(0.0, u, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"narrow {n}^3: {ms:.4f} ms, {341 * n ** 3 / ms / 1e9:.2f} TF/s "
      f"(ZRING={os.environ.get('SMC_NARROW_ZRING', '0')})")
