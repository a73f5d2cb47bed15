"""The full C5 grid (BASELINE.json configs[4]): 3 cost models x 32 arrival
rates x 128 seeds of 1000-session toolbench traces x all 169 N=8 plans
= 2 076 672 pairs, one search per cost model on one B200 (full mode, then
argmax mode). Prints one JSON line.

usage: python tools/c5_full.py [seeds]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 128
out = {"models": {}, "pairs": 0, "request_rounds": 0, "kernel_s": 0.0, "argmax_kernel_s": 0.0}
with native.Context(0) as ctx:
    for model in ("llama3-8b", "qwen-32b", "llama3-70b"):
        t0 = time.perf_counter()
        wl = workloads.c5(model=model, seeds=seeds)
        gen_s = time.perf_counter() - t0
        ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
        ctx.set_search_mode(abi.SEARCH_FULL)
        r = ctx.search_staged(wl.seed)
        ctx.set_search_mode(abi.SEARCH_ARGMAX)
        a = ctx.search_staged(wl.seed)
        ctx.set_search_mode(abi.SEARCH_FULL)
        out["models"][model] = {"pairs": wl.n_pairs, "host_gen_s": gen_s, "kernel_s": r.kernel_ms / 1e3,
                                "best_candidate": r.best_candidate, "best_slo_ok": r.best_slo_ok,
                                "argmax_kernel_s": a.kernel_ms / 1e3,
                                "argmax_same_plan": (a.best_candidate, a.best_slo_ok) == (r.best_candidate, r.best_slo_ok)}
        out["pairs"] += wl.n_pairs
        out["request_rounds"] += wl.request_rounds
        out["kernel_s"] += r.kernel_ms / 1e3
        out["argmax_kernel_s"] += a.kernel_ms / 1e3
        print(model, out["models"][model], flush=True, file=sys.stderr)
out["request_rounds_per_s"] = out["request_rounds"] / out["kernel_s"]
out["replays_per_s"] = out["pairs"] / out["kernel_s"]
print(json.dumps(out), flush=True)
