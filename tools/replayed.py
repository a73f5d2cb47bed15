"""Exact-replay count and events of one staged search (lazy-attempt aborts).

usage: python tools/replayed.py CONFIG PAIR_BEGIN PAIR_END
"""
import os
sys_path_root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import sys
sys.path.insert(0, sys_path_root)
from paper_2602_14516_b200 import native, workloads
cfg, b, e = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
wl = workloads.CONFIGS[cfg]()
with native.Context(0) as ctx:
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    r = ctx.search_staged(wl.seed, b, e)
    cy, n, rep = ctx.profile_counters()
    ev = sum(r.pair_events[p] for p in range(r.n_pairs))
    print(cfg, "kernel", round(r.kernel_ms,1), "replayed", rep, "of", r.n_pairs, "events", ev)
