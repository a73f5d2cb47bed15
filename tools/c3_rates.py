"""GPU timing of the C3 search at several arrival rates (rate pick for the
headline, VERDICT r1 'next' 1a): kernel ms, per-pair cycles spread and the
attainment spread over candidates.

usage: python tools/c3_rates.py RATE [RATE ...]   -> gpurun_out/c3_rates.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import native, workloads  # noqa: E402

rows = []
for rate in [float(x) for x in sys.argv[1:]]:
    t0 = time.time()
    wl = workloads.c3(rate=rate)
    gen_s = time.time() - t0
    with native.Context(0) as ctx:
        ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
        r = ctx.search_staged(wl.seed)
        nt, S = len(wl.traces), wl.traces[0].n_sessions
        cyc = sorted(r.pair_cycles[p] / 1.965e6 for p in range(r.n_pairs))
        cand = [r.candidate_slo_ok[c] / (nt * S) for c in range(len(wl.plans))]
        row = {"rate": rate, "gen_s": gen_s, "kernel_ms": r.kernel_ms, "pairs": r.n_pairs,
               "pair_ms_p50": cyc[len(cyc) // 2], "pair_ms_p90": cyc[int(len(cyc) * 0.9)], "pair_ms_max": cyc[-1],
               "best": r.best_candidate, "best_frac": r.best_slo_ok / (nt * S),
               "cands_ge90": sum(f >= 0.9 for f in cand), "cands_lt10": sum(f < 0.1 for f in cand),
               "rounds": wl.request_rounds}
    rows.append(row)
    print(json.dumps(row), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/c3_rates.json", "w"), indent=1)
