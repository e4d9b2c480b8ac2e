"""Time HeatOperator::rhs (T2 coefficients, narrow SMC) at n^2 on cuda:0."""
import math, sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1309_7327_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
dev = torch.device('cuda:0')
xs = np.arange(n) * (2 * math.pi / n)
X, Y = np.meshgrid(xs, xs)
a = 1.0 + 0.9 * np.cos(2 * X) * np.sin(2 * Y + math.pi / 3)
b = 1.0 + 0.9 * np.cos(2 * X + math.pi / 3) * np.sin(2 * Y)
u = torch.from_numpy(np.sin(X) * np.sin(Y)).to(dev)
out = torch.empty_like(u)
op = P.HeatOperator(n, n, P.StencilChoice.narrow8(P.SMC_M47, P.SMC_M48), a, b)
s = torch.cuda.current_stream()
op.set_stream(s)
for _ in range(5):
    op(0.0, u, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(reps):
    op(0.0, u, out)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(json.dumps({"n": n, "ms": ms, "tflops": 229 * n * n / ms / 1e9}))
