"""Host<->device copy bandwidth on the box (pinned, 134 MB = one 256^3 f64
field): H2D alone, D2H alone, both at once on two streams, and the
narrow operator's host-buffer call at several chunk counts."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

n = 256
h = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
h2 = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
d = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
d2 = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nb = h.numel() * 8


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    d.copy_(h, non_blocking=True)


def d2h():
    h2.copy_(d2, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    t = timeit(fn)
    print(f"{name}: {t * 1e3:.3f} ms  {nb / t / 1e9:.1f} GB/s per direction")

import numpy as np  # noqa: E402

import paper_1309_7327_b200 as P  # noqa: E402

a = torch.rand((n, n, n), dtype=torch.float64, device="cuda") + 1
op = P.Narrow3DOperator(a, 1 / n, 1 / n, 1 / n)
for _ in range(2):
    t = timeit(lambda: op(0.0, h, h2))
    print(f"narrow host call (chunks={os.environ.get('SMC_E2E_CHUNKS', 'default')}): "
          f"{t * 1e3:.3f} ms")
