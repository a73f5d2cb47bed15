"""Does co-residency of similar pairs relieve the instruction-fetch bound?

Replays C3s (2704 pairs, every SM holding ~18 warps) as the normal mixed
search and as homogeneous searches in which every pair runs the SAME plan
(the plan list is one candidate repeated), and reports SM cycles per event
under load and alone (contention = loaded / solo) for each.

usage: python tools/homog.py [CONFIG] [N_PLANS]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402


def measure(ctx, wl, plans, label):
    ctx.stage(wl.traces, plans, wl.profile, wl.params)
    ctx.search_staged(wl.seed)
    res = ctx.search_staged(wl.seed)
    cyc = sum(res.pair_cycles[p] for p in range(res.n_pairs))
    ev = sum(res.pair_events[p] for p in range(res.n_pairs))
    solo = ctx.search_staged(wl.seed, 0, 1)
    solo_cpe = solo.pair_cycles[0] / max(solo.pair_events[0], 1)
    out = {"label": label, "kernel_ms": res.kernel_ms, "pairs": res.n_pairs, "events": ev,
           "events_per_ms": ev / res.kernel_ms, "loaded_cycles_per_event": cyc / max(ev, 1),
           "solo_cycles_per_event_pair0": solo_cpe, "contention": (cyc / max(ev, 1)) / max(solo_cpe, 1e-9)}
    print(json.dumps(out), flush=True)
    return out


def main(cfg="C3s", n_plans="6"):
    wl = workloads.CONFIGS[cfg]()
    nc = len(wl.plans)
    with native.Context(0) as ctx:
        measure(ctx, wl, wl.plans, "mixed")
        step = max(1, nc // int(n_plans))
        for c in range(0, nc, step):
            measure(ctx, wl, [wl.plans[c]] * nc, f"homog c{c} {abi.format_plan(wl.plans[c])}")


if __name__ == "__main__":
    main(*sys.argv[1:])
