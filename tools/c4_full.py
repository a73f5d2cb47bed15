"""The full C4 grid (BASELINE.json configs[3]): llama3-70b, 8 arrival rates x
64 seeds of mixed toolbench+hotpotqa 100k-session traces, all 169 N=8 plans
= 86 528 pairs, one full search on one B200 (plus the argmax-mode search).
Prints one JSON line; the CPU reference is projected from the bench's
sampled per-pair rate (profiles/round1/bench_c4_slice_v12.json).

usage: python tools/c4_full.py [seeds]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 64
t0 = time.perf_counter()
wl = workloads.c4(seeds=seeds)
gen_s = time.perf_counter() - t0
out = {"workload": wl.desc, "pairs": wl.n_pairs, "host_gen_merge_s": gen_s,
       "request_rounds": wl.request_rounds}
with native.Context(0) as ctx:
    t0 = time.perf_counter()
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    out["stage_s"] = time.perf_counter() - t0
    r = ctx.search_staged(wl.seed)
    out.update({"kernel_s": r.kernel_ms / 1e3, "best_candidate": r.best_candidate, "best_slo_ok": r.best_slo_ok,
                "request_rounds_per_s": wl.request_rounds / (r.kernel_ms / 1e3),
                "replays_per_s": wl.n_pairs / (r.kernel_ms / 1e3)})
    ctx.set_search_mode(abi.SEARCH_ARGMAX)
    a = ctx.search_staged(wl.seed)
    out["argmax_mode"] = {"kernel_s": a.kernel_ms / 1e3, "best_candidate": a.best_candidate,
                          "best_slo_ok": a.best_slo_ok,
                          "pruned": sum(1 for c in range(len(wl.plans)) if a.candidate_slo_ok[c] == -2)}
print(json.dumps(out), flush=True)
