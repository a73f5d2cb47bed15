"""`pdsim sweep` on the GPU vs the reference's serial sweep loop (SURVEY.md
§8(f)2): a C1-like plan (P:2x1, D:2x1) over rates x alpha x beta x window,
toolbench traces of 1000 sessions. The GPU side is one pdsim_gpu_sweep call
(trace generation on the host, reports + sweep.csv back); the reference side
is refbind.report (unmodified run() + build_report) per combination on all
host threads, over a bounded sample. Parity of every sampled report is
checked. Prints one JSON line.

usage: python tools/sweep_bench.py [n_rates]
"""
import concurrent.futures as cf
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import refbind  # noqa: E402  (CPU baseline + checker only)
from paper_2602_14516_b200 import abi, native, sweep, workloads  # noqa: E402


def main(n_rates=16):
    n_rates = int(n_rates)
    rates = [1.0 + k for k in range(n_rates)]
    alphas, betas, windows = [0.5, 0.7, 0.9, 1.0], [0.5, 0.85, 1.0], [1, 3, 5]
    prof = workloads.model_profile("llama3-8b")
    plan = abi.make_plan({1: 2}, {1: 2})
    base, seed = abi.default_params(), 1
    with native.Context(0) as ctx:
        sweep.run_sweep(ctx, "toolbench", 1000, rates[:2], plan, prof, base, seed, alphas, betas, windows)  # warm
        t0 = time.perf_counter()
        csv, settings, res = sweep.run_sweep(ctx, "toolbench", 1000, rates, plan, prof, base, seed,
                                             alphas, betas, windows)
        wall = time.perf_counter() - t0
    n = len(rates) * len(settings)
    out = {"workload": f"sweep: P:2x1,D:2x1, toolbench 1000 sessions, {len(rates)} rates x {len(alphas)} alphas x "
                       f"{len(betas)} betas x {len(windows)} windows", "combinations": n,
           "gpu_wall_s": wall, "gpu_kernel_ms": res.kernel_ms, "gpu_combinations_per_s": n / wall,
           "csv_bytes": len(csv)}
    stats = native.preset_stats("toolbench")
    trs = {r: native.gen_trace(stats, r, 1000, seed) for r in rates}
    threads = os.cpu_count() or 1
    jobs = [(k, r) for k in range(len(settings)) for r in range(len(rates))]
    sample = jobs[:: max(1, len(jobs) // (threads * 6))][: threads * 6]
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        ref = list(ex.map(lambda kr: refbind.report(trs[rates[kr[1]]].view, plan, prof, settings[kr[0]], seed),
                          sample))
    cpu = time.perf_counter() - t0
    out["cpu_baseline"] = {"combinations_per_s": len(sample) / cpu, "cores": threads, "kind": "reference",
                           "sample": f"{len(sample)} of {n} combinations"}
    out["speedup_vs_cpu"] = out["gpu_combinations_per_s"] / out["cpu_baseline"]["combinations_per_s"]
    out["parity_mismatches_on_sample"] = sum(
        1 for (k, r), want in zip(sample, ref) if res.reports[k * len(rates) + r].as_tuple() != want.as_tuple())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
