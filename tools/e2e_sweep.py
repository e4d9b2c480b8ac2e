"""configs[1] through the public API with pinned host buffers: ms per call for
several mid-chunk sizes (SMC_E2E_CHUNK_PLANES, one subprocess each), beside
the bare PCIe copies of the same bytes (H2D alone, D2H alone, both at once)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json, torch
sys.path.insert(0, sys.argv[1])
import paper_1309_7327_b200 as P
from paper_1309_7327_b200 import workloads as W
n = 256
a, u = W.narrow3d_inputs(n, seed=1)
dev = torch.device("cuda:0")
op = P.Narrow3DOperator(torch.from_numpy(a).to(dev), 1 / n, 1 / n, 1 / n)
uh = torch.from_numpy(u).pin_memory()
oh = torch.empty_like(uh).pin_memory()
s = torch.cuda.current_stream()
for _ in range(3):
    op(0.0, uh, oh)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for rep in range(5):
    e0.record(s)
    for _ in range(5):
        op(0.0, uh, oh)
    e1.record(s)
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 5)
res = {"e2e_ms": best}
if len(sys.argv) > 2:
    d = torch.empty_like(uh, device=dev)
    d2 = torch.empty_like(uh, device=dev)
    s2 = torch.cuda.Stream()
    def t(fn):
        fn(); torch.cuda.synchronize()
        e0.record(s)
        for _ in range(5): fn()
        torch.cuda.synchronize(); e1.record(s); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 5
    res["h2d_ms"] = t(lambda: d.copy_(uh, non_blocking=True))
    res["d2h_ms"] = t(lambda: oh.copy_(d, non_blocking=True))
    def both():
        with torch.cuda.stream(s2):
            oh.copy_(d2, non_blocking=True)
        d.copy_(uh, non_blocking=True)
        s.wait_stream(s2)
    res["both_ms"] = t(both)
print(json.dumps(res))
"""

out = {}
for i, planes in enumerate([8, 16, 24, 32, 48, 64]):
    env = dict(os.environ, SMC_E2E_CHUNK_PLANES=str(planes))
    args = [sys.executable, "-c", CHILD, ROOT] + (["copies"] if i == 0 else [])
    r = subprocess.run(args, env=env, capture_output=True, text=True, timeout=600)
    out[planes] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
    print(planes, out[planes], flush=True)
