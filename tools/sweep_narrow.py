"""Tuning sweep of the narrow3d_fast knobs (environment variables) on the
configs[1] bench: python tools/sweep_narrow.py VAR=a,b VAR2=c,d ..."""
import itertools
import json
import os
import subprocess
import sys

axes = [(kv.split("=")[0], kv.split("=")[1].split(",")) for kv in sys.argv[1:]]
for combo in itertools.product(*[v for _, v in axes]):
    env = dict(os.environ)
    tag = []
    for (k, _), v in zip(axes, combo):
        env[k] = v
        tag.append(f"{k}={v}")
    r = subprocess.run([sys.executable, "bench.py", "--steps", "1000", "--warmup", "20",
                        "--no-cpu-baseline", "--no-ns", "--no-advance"], env=env,
                       capture_output=True, text=True, timeout=600)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(" ".join(tag), round(d["ms_per_step"], 4), round(d["value"] / 1e9, 2),
              round(d["roofline"]["frac"], 3), d["clocks"]["sm_mhz"], flush=True)
    except Exception:
        print(" ".join(tag), "FAILED", r.stderr[-500:], flush=True)
