"""Per-pair GPU diagnostics for a workload: events and SM cycles per pair."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402


NAMES = ["select", "arrival", "interaction", "writeback", "decode_step", "local_prefill_done", "prefill_done",
         "history_read", "~route", "~enqueue", "~catch_up", "~finisher", "~advance_decode", "~complete_task",
         "~heap", "~dequeue", "~seg_append", "~fh", "~ttft_add", "~itl_slack", "~ttft_slack", "~bulk", "~seg_sum",
         "~try_stage", "#catch_up_idle", "~stable_run", "#catch_up_iter", "~bind_catch_up"]


def phases(prof):
    return {name: {"cycles": prof[0][k], "count": prof[1][k], "cycles_per": prof[0][k] / max(prof[1][k], 1)}
            for k, name in enumerate(NAMES)}


def main(cfg="C2"):
    wl = workloads.CONFIGS[cfg]()
    with native.Context(0) as ctx:
        ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
        ctx.search_staged(wl.seed)
        ctx.set_profiling(True)
        ctx.search_staged(wl.seed)
        prof = ctx.profile_counters()
        ctx.set_profiling(False)
        t0 = time.time()
        res = ctx.search_staged(wl.seed)
        wall = time.time() - t0
        slowest = max(range(res.n_pairs), key=lambda p: res.pair_cycles[p])
        ctx.set_profiling(True)
        ctx.search_staged(wl.seed, slowest, slowest + 1)
        prof1 = ctx.profile_counters()
        ctx.set_profiling(False)
    rows = []
    for p in range(res.n_pairs):
        rows.append((res.pair_cycles[p], res.pair_events[p], p, abi.format_plan(wl.plans[p // len(wl.traces)])))
    rows.sort(reverse=True)
    out = {"config": cfg, "kernel_ms": res.kernel_ms, "wall_s": wall, "pairs": res.n_pairs,
           "top": [{"cycles": c, "events": e, "ns_per_event_at_1.965GHz": c / 1.965 / max(e, 1), "pair": p,
                    "plan": s} for c, e, p, s in rows[:10]],
           "total_events": sum(r[1] for r in rows), "total_cycles": sum(r[0] for r in rows),
           "phases": phases(prof), "slowest_pair": slowest, "slowest_phases": phases(prof1),
           "replayed_pairs": prof[2]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
