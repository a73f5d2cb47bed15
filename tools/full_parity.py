"""Whole-search parity and an un-extrapolated CPU baseline for one config:
the GPU search (every pair) against the unmodified reference (oracle/_ref,
std::thread pool on all host threads, heaviest pairs first) over EVERY pair.
Test/measurement infrastructure (tools/), not part of the product.

usage: python tools/full_parity.py [CONFIG ...]   -> one JSON line per config
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402

FIELDS = ("sessions_total", "sessions_completed", "slo_ok", "ttft_ok", "itl_ok")


def main(cfgs):
    from oracle import refbind
    import bench
    for cfg in cfgs:
        wl = workloads.CONFIGS[cfg]()
        nt, C = len(wl.traces), len(wl.plans)
        with native.Context(0) as ctx:
            ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
            ctx.search_staged(wl.seed)
            t0 = time.perf_counter()
            g = ctx.search_staged(wl.seed)
            gpu_wall = time.perf_counter() - t0
            build = ctx.last_kernel_build()
        pairs = bench.heavy_first(list(range(wl.n_pairs)), wl.traces, wl.plans)
        n_threads = os.cpu_count() or 1
        att, st, cpu_wall = refbind.plan_search_list(wl.traces, wl.plans, wl.profile, wl.params, wl.seed, pairs,
                                                     n_threads)
        mism, status_mism = 0, 0
        sums, bad = [0] * C, [False] * C
        for k, p in enumerate(pairs):
            if g.pair_status[p] != st[k]:
                status_mism += 1
            if st[k] == 0:
                if any(getattr(g.pair_attainment[p], f) != getattr(att[k], f) for f in FIELDS):
                    mism += 1
                sums[p // nt] += att[k].slo_ok
            else:
                bad[p // nt] = True
        ref_best = max(range(C), key=lambda c: (-1 if bad[c] else sums[c], -c))
        rounds = sum(int(t.n_rounds) for t in wl.traces) * C
        out = {"config": cfg, "workload": wl.spec.desc, "pairs": wl.n_pairs, "pairs_checked": wl.n_pairs,
               "status_mismatches": status_mism, "attainment_mismatches": mism,
               "gpu_best": [g.best_candidate, g.best_slo_ok], "reference_best": [ref_best, sums[ref_best]],
               "argmax_identical": g.best_candidate == ref_best and g.best_slo_ok == sums[ref_best],
               "gpu_search_s": gpu_wall, "gpu_kernel_ms": g.kernel_ms,
               "gpu_kernel_build": {abi.BUILD_LATENCY: "latency", abi.BUILD_THROUGHPUT: "throughput"}.get(build),
               "cpu_search_s": cpu_wall, "cpu_threads": n_threads, "cpu_sample": "every pair (not extrapolated)",
               "request_rounds": rounds, "gpu_request_rounds_per_s": rounds / gpu_wall,
               "cpu_request_rounds_per_s": rounds / cpu_wall, "speedup_resident": cpu_wall / gpu_wall}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C3"])
