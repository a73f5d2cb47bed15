"""Host staging time (validate + pack + precheck + H2D) of a workload: python tools/stage_time.py CONFIG"""
import sys, time
sys.path.insert(0, '.')
from paper_2602_14516_b200 import native, workloads
wl = workloads.CONFIGS[sys.argv[1]]()
with native.Context(0) as ctx:
    ts = []
    for _ in range(4):
        t0 = time.perf_counter(); ctx.stage(wl.traces, wl.plans, wl.profile, wl.params); ts.append(time.perf_counter() - t0)
print(sys.argv[1], "stage ms", [round(1e3 * t, 1) for t in ts])
