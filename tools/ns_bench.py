"""Time the NS RHS parts at n^3 on cuda:0 (state generated on the GPU box's
host then uploaded)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1309_7327_b200 as P
from paper_1309_7327_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device('cuda:0')
t0 = time.time()
T, p, uvw, Y = W.ns_primitives(n, hot_spot=True)
U = P.ns_conserved(*(torch.from_numpy(a).to(dev) for a in (T, p, uvw, Y)))
print('state', time.time() - t0, 's', flush=True)
op = P.NsOperator(n, n, n, 1e-4)
s = torch.cuda.current_stream()
op.set_stream(s)
out = torch.empty_like(U)
res = {}
for name, r in (('full', op.full), ('advdiff', op.advdiff), ('chem', op.chem)):
    r(0.0, U, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        r(0.0, U, out)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[name] = ms
    print(name, round(ms, 3), 'ms', round(n ** 3 / ms / 1e6, 3), 'G cell-RHS/s', flush=True)
print(json.dumps(res))
# per-kernel CUDA-event times of one full evaluation (minimum over 3)
prof = {}
for _ in range(3):
    for k, ms in op.profile(U, out):
        prof[k] = min(prof.get(k, 1e9), ms)
print('kernels', json.dumps({k: round(v, 3) for k, v in prof.items()}))
