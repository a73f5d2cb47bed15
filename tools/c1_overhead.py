"""Where a single replay's (C1) search call spends its time: wall vs device
(ev0..ev3) vs replay kernel, for stage, search_staged and plan_search."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import native, workloads  # noqa: E402

wl = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]()
with native.Context(0) as ctx:
    for k in range(4):
        t0 = time.perf_counter()
        ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
        t1 = time.perf_counter()
        r = ctx.search_staged(wl.seed)
        t2 = time.perf_counter()
        r2 = ctx.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed)
        t3 = time.perf_counter()
        print(f"stage {1e3*(t1-t0):.2f} ms | search wall {1e3*(t2-t1):.2f} device {r.device_ms:.2f} kernel {r.kernel_ms:.2f}"
              f" | plan_search wall {1e3*(t3-t2):.2f} device {r2.device_ms:.2f} kernel {r2.kernel_ms:.2f}", flush=True)
