"""Per-pair duration spread of a search under full load, and the same pairs
replayed alone (contention factor): where does a throughput config's
makespan go?

usage: python tools/pair_spread.py [CONFIG] [SOLO_PAIRS]
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402


def q(xs, f):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(f * len(xs)))]


def main(cfg="C3", n_solo="4"):
    wl = workloads.CONFIGS[cfg]()
    nt = len(wl.traces)
    with native.Context(0) as ctx:
        ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
        ctx.search_staged(wl.seed)
        t0 = time.time()
        res = ctx.search_staged(wl.seed)
        wall = time.time() - t0
        cyc = [res.pair_cycles[p] for p in range(res.n_pairs)]
        ev = [res.pair_events[p] for p in range(res.n_pairs)]
        order = sorted(range(res.n_pairs), key=lambda p: -cyc[p])
        picks = [order[0], order[len(order) // 2], order[-1]][: int(n_solo)]
        solo = []
        for p in picks:
            r1 = ctx.search_staged(wl.seed, p, p + 1)
            solo.append({"pair": p, "plan": abi.format_plan(wl.plans[p // nt]), "events": ev[p],
                         "loaded_cycles": cyc[p], "solo_cycles": r1.pair_cycles[0],
                         "contention": cyc[p] / max(r1.pair_cycles[0], 1),
                         "solo_cycles_per_event": r1.pair_cycles[0] / max(ev[p], 1)})
    by_cand = {}
    for p in range(res.n_pairs):
        by_cand.setdefault(p // nt, []).append(cyc[p])
    cand_mean = sorted(((statistics.mean(v), c) for c, v in by_cand.items()), reverse=True)
    ghz = 1.965e9
    out = {"config": cfg, "kernel_ms": res.kernel_ms, "wall_s": wall, "pairs": res.n_pairs,
           "cycles_q": {k: q(cyc, f) for k, f in (("p0", 0.0), ("p10", .1), ("p50", .5), ("p90", .9), ("p99", .99),
                                                   ("max", 1.0))},
           "max_pair_s": max(cyc) / ghz, "mean_pair_s": statistics.mean(cyc) / ghz,
           "sum_pair_s_over_148sm": sum(cyc) / ghz / 148,
           "events_q": {k: q(ev, f) for k, f in (("p0", 0.0), ("p50", .5), ("max", 1.0))},
           "total_events": sum(ev),
           "cycles_per_event_loaded": sum(cyc) / max(sum(ev), 1),
           "slowest_candidates": [{"cand": c, "plan": abi.format_plan(wl.plans[c]), "mean_s": m / ghz}
                                  for m, c in cand_mean[:8]],
           "fastest_candidates": [{"cand": c, "plan": abi.format_plan(wl.plans[c]), "mean_s": m / ghz}
                                  for m, c in cand_mean[-4:]],
           "solo": solo}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
