"""Per-candidate slo_ok counts and SM cycles of the C2 search (pruning study)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import native, workloads
wl = workloads.c2()
with native.Context(0) as ctx:
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    r = ctx.search_staged(wl.seed)
    out = {"best": r.best_candidate, "best_ok": r.best_slo_ok,
           "ok": [r.candidate_slo_ok[c] for c in range(len(wl.plans))],
           "cyc": [r.pair_cycles[c] for c in range(len(wl.plans))]}
json.dump(out, open("gpurun_out/c2_cands.json","w"))
print("ok")
