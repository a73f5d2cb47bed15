"""Surrogate planner on the GPU: coefficient-sweep
throughput against the reference's CPU estimate_coefficients, and the plan
it selects against the replay argmax (the paper's Table 2 question: does the
P95-coefficient planner pick a plan whose replayed SLO attainment matches the
best candidate's?).

usage: python tools/planner_bench.py [rates] [seeds]   (prints one JSON line)
"""
import concurrent.futures as cf
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import refbind  # noqa: E402  (CPU baseline + checker only)
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402

DEGREES = [1, 2, 4, 8]


def main(n_rates=32, n_seeds=128):
    n_rates, n_seeds = int(n_rates), int(n_seeds)
    prof = workloads.model_profile("llama3-8b")
    st = native.preset_stats("toolbench")
    rates = [1.0 + 0.5 * k for k in range(n_rates)]
    sets = [(r, 1000 + s) for r in rates for s in range(n_seeds)]
    out = {"workload": f"estimate_coefficients over {n_rates} rates x {n_seeds} seeds x degrees {DEGREES}, "
                       f"toolbench, llama3-8b cost model, N=8", "sets": len(sets), "jobs": len(sets) * len(DEGREES)}
    with native.Context(0) as ctx:
        ctx.estimate_coefficients(st, [r for r, _ in sets[:8]], [s for _, s in sets[:8]], prof, DEGREES, 8)  # warm
        t0 = time.perf_counter()
        got = ctx.estimate_coefficients(st, [r for r, _ in sets], [s for _, s in sets], prof, DEGREES, 8)
        gpu_s = time.perf_counter() - t0
        out["gpu_wall_s"] = gpu_s
        out["gpu_sets_per_s"] = len(sets) / gpu_s

        # split: host trace generation vs device phase sims for the same jobs
        t0 = time.perf_counter()
        trs = [native.gen_trace(st, r * d / 8.0, 256, (s + 0x9E3779B97F4A7C15 * d) % (1 << 64))
               for r, s in sets[:1024] for d in DEGREES]
        out["host_gen_s_1024_sets_1_thread"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        ctx.phase_sims([t.view for t in trs], DEGREES * 1024, prof)
        out["gpu_phase_sims_s_1024_sets"] = time.perf_counter() - t0

        # reference CPU (unmodified planner.cpp) on all host threads, bounded sample
        threads = os.cpu_count() or 1
        sample = sets[:: max(1, len(sets) // (threads * 8))][: threads * 8]
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(threads) as ex:
            ref = list(ex.map(lambda rs: refbind.estimate_coefficients(st, rs[0], prof, DEGREES, 8, rs[1],
                                                                      "toolbench"), sample))
        cpu_s = time.perf_counter() - t0
        out["cpu_baseline"] = {"sets_per_s": len(sample) / cpu_s, "cores": threads, "kind": "reference",
                               "sample": f"{len(sample)} of {len(sets)} settings"}
        out["speedup_vs_cpu"] = out["gpu_sets_per_s"] / out["cpu_baseline"]["sets_per_s"]
        index = {rs: k for k, rs in enumerate(sets)}
        mism = 0
        for rs, (c, rc) in zip(sample, ref):
            gc, gs = got[index[rs]]
            if gs != rc or (rc == 0 and gc.as_dict() != c.as_dict()):
                mism += 1
        out["parity_mismatches_on_sample"] = mism

        # surrogate plan vs replay argmax on C2
        wl = workloads.c2()
        coeff, status = ctx.estimate_coefficients(st, [16.0], [5], prof, DEGREES, 8)[0]
        sol = native.solve(coeff, 8) if status == 0 else None
        res = ctx.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed)
        cand = [res.candidate_slo_ok[c] for c in range(len(wl.plans))]
        out["c2"] = {"replay_best": abi.format_plan(wl.plans[res.best_candidate]), "replay_best_slo_ok": res.best_slo_ok,
                     "sessions": wl.traces[0].n_sessions}
        if sol:
            key = abi.plan_dict(sol[0])
            idx = [k for k, p in enumerate(wl.plans) if abi.plan_dict(p) == key]
            out["c2"].update({"surrogate_plan": abi.format_plan(sol[0]), "surrogate_z": sol[1],
                              "surrogate_plan_replay_slo_ok": cand[idx[0]] if idx else None,
                              "candidates_at_best": sum(1 for v in cand if v == res.best_slo_ok)})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
