"""Per-SM-list load of the candidate-affine queues: pair cycles by list (the
host's n*s/L chunks of the candidate-grouped launch order), max vs mean.

usage: python tools/affinity_spread.py [CONFIG]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import native, workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3s"
wl = workloads.CONFIGS[cfg]()
L = 148
with native.Context(0) as ctx:
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    for aff in ("0", "1"):
        os.environ["PDSIM_SM_AFFINITY"] = aff
        ctx.search_staged(wl.seed)
        res = ctx.search_staged(wl.seed)
        n = res.n_pairs
        cyc = [res.pair_cycles[p] for p in range(n)]
        ev = [res.pair_events[p] for p in range(n)]
        lists = [list(range(n * s // L, n * (s + 1) // L)) for s in range(L)]
        lmax = [max(cyc[p] for p in li) for li in lists]
        lsum_ev = [sum(ev[p] for p in li) for li in lists]
        ghz = 1.965e6
        print(json.dumps({"affinity": aff, "kernel_ms": res.kernel_ms, "pair_ms_max": max(cyc) / ghz,
                          "pair_ms_mean": statistics.mean(cyc) / ghz,
                          "list_max_ms_q": [sorted(lmax)[int(f * (L - 1))] / ghz for f in (0, .1, .5, .9, 1)],
                          "list_events_q": [sorted(lsum_ev)[int(f * (L - 1))] for f in (0, .1, .5, .9, 1)],
                          "cycles_per_event": sum(cyc) / sum(ev)}), flush=True)
