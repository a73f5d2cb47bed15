"""Runs one staged search over a pair range of a workload (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import native, workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
b = int(sys.argv[2]) if len(sys.argv) > 2 else 0
e = int(sys.argv[3]) if len(sys.argv) > 3 else -1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
wl = workloads.CONFIGS[cfg]()
with native.Context(0) as ctx:
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    for _ in range(reps):
        res = ctx.search_staged(wl.seed, b, e)
        print(f"kernel_ms={res.kernel_ms:.3f} pairs={res.n_pairs} best={res.best_candidate}", flush=True)
