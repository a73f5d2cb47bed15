"""Splits the end-to-end C-ABI call (pdsim_gpu_plan_search) of a workload
into host staging (validate + pack + precheck + H2D) and the staged search."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import native, workloads  # noqa: E402

wl = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]()
with native.Context(0) as ctx:
    for _ in range(2):
        ctx.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed)
    for _ in range(3):
        t0 = time.perf_counter()
        ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
        t1 = time.perf_counter()
        r = ctx.search_staged(wl.seed)
        t2 = time.perf_counter()
        r2 = ctx.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed)
        t3 = time.perf_counter()
        print(f"stage {1e3*(t1-t0):.1f} ms  search_staged {1e3*(t2-t1):.1f} ms (kernel {r.kernel_ms:.1f}, device {r.device_ms:.1f})"
              f"  plan_search {1e3*(t3-t2):.1f} ms", flush=True)
