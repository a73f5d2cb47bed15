"""Per-pair SM cycles / events of one staged search (tail analysis).

usage: python tools/pair_times.py CONFIG [top]   -> gpurun_out/pair_times_<CONFIG>.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = workloads.CONFIGS[cfg]()
with native.Context(0) as ctx:
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    r = ctx.search_staged(wl.seed)
    nt = len(wl.traces)
    cyc = [r.pair_cycles[p] for p in range(r.n_pairs)]
    ev = [r.pair_events[p] for p in range(r.n_pairs)]
    order = sorted(range(r.n_pairs), key=lambda p: -cyc[p])
    out = {"config": cfg, "kernel_ms": r.kernel_ms, "pairs": r.n_pairs,
           "mean_ms": sum(cyc) / len(cyc) / 1.965e6, "max_ms": cyc[order[0]] / 1.965e6,
           "top": [{"pair": p, "plan": abi.format_plan(wl.plans[p // nt]), "replica": p % nt,
                    "ms": cyc[p] / 1.965e6, "events": ev[p], "slo_ok": r.pair_attainment[p].slo_ok}
                   for p in order[:top]]}
json.dump(out, open(f"gpurun_out/pair_times_{cfg}.json", "w"), indent=1)
print(json.dumps({k: out[k] for k in ("config", "kernel_ms", "pairs", "mean_ms", "max_ms")}))
