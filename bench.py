#!/usr/bin/env python3
"""bench.py — candidate-plan replay search throughput on B200.

One "step" = one full plan search over the workload: every (candidate,
replica) pair replayed by the GPU engine, SLO counts reduced per candidate
(in-library NCCL all-reduce across GPUs when N > 1), argmax taken.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

Default workload: C3 (BASELINE.json configs[2], the largest configuration
that fits one B200 and runs in seconds per search): qwen-32b cost model, all
169 N=8 plans x 16 hotpotqa 8-round replicas of 50 000 sessions @2/s = 2704
replays, 6.4 M request-rounds per replica-candidate sweep. At N > 1 the SAME
search is sharded over the GPUs (strong scaling; pdsim_shard_pairs).

Prints ONE JSON line (rank 0). `value` is whole-job request-rounds/s with
inputs resident in HBM; `e2e` is the same metric through the host-buffer
C-ABI call (H2D + kernels + D2H every step). `cpu_baseline` is the unmodified
reference (oracle/_ref) on all host threads over a fixed-seed stratified
random sample of the pairs (one random replica per candidate), extrapolated
to the whole search; the same sampled pairs are the line's parity check.
`secondary` repeats the measurement on C2 (configs[1]), on a C5 slice
(configs[4]: llama3-8b, 169 plans x 128 toolbench traces = 21 632 pairs) and
on C1 (configs[0]: one replay, the reference's own CPU-runnable case).
"""
import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2602_14516_b200 import abi, specs  # noqa: E402  (plain data, no library load)

METRIC = "candidate-plan trace replays/sec (request-rounds/sec); planner wall-time"
UNIT = "request-rounds/s"
SAMPLE_SEED = 20260217


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--secondary", default="C2,C5,C1",
                    help="comma-separated configs measured in the same line ('none' to skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-argmax-mode", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.out = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


# ---- sampling shared by both arms (plain Python, no library) -----------------

def plan_workers(p):
    x, y = abi.plan_dict(p)
    return sum(x.values()) + sum(y.values())


def heavy_first(pairs, traces, plans):
    """Pool order for the reference's thread pool: the same cost heuristic as
    the product's shard planner (rounds x (workers + 2)), heaviest first, so
    the reference's wall time is not inflated by a long pair starting last."""
    nt = len(traces)
    return sorted(pairs, key=lambda p: (-int(traces[p % nt].n_rounds) * (plan_workers(plans[p // nt]) + 2), p))


def stratified_sample(n_traces, n_cand, seed=SAMPLE_SEED):
    """One uniformly random replica per candidate (every pair has inclusion
    probability 1/n_traces; every candidate shape is covered). Single-replica
    searches are sampled whole."""
    if n_traces == 1:
        return list(range(n_cand))
    rng = random.Random(seed)
    return [c * n_traces + rng.randrange(n_traces) for c in range(n_cand)]


def rounds_of(wl, pairs):
    nt = len(wl.traces)
    return sum(int(wl.traces[p % nt].n_rounds) for p in pairs)


def all_rounds(wl):
    return sum(int(t.n_rounds) for t in wl.traces) * len(wl.plans)


def cpu_baseline(wl, gpu_pairs=None):
    """The reference's own CPU path (oracle/_ref: the unmodified reference
    run() in a std::thread pool on all host threads) over the stratified
    sample; extrapolated linearly to the whole search by request-rounds.
    gpu_pairs (pair -> (status, attainment)) makes the sample the GPU run's
    parity check: per-pair status and attainment must be identical."""
    from oracle import refbind
    if not refbind.available():
        return None, None
    n_threads = os.cpu_count() or 1
    sample = heavy_first(stratified_sample(len(wl.traces), len(wl.plans)), wl.traces, wl.plans)
    att, st, wall = refbind.plan_search_list(wl.traces, wl.plans, wl.profile, wl.params, wl.seed, sample, n_threads)
    r_sample, r_all = rounds_of(wl, sample), all_rounds(wl)
    value = r_sample / wall
    full = len(sample) == wl.n_pairs
    base = {"value": value, "unit": UNIT, "cores": n_threads, "kind": "reference",
            "sample": (f"{len(sample)}/{wl.n_pairs} pairs ({100.0 * len(sample) / wl.n_pairs:.2f} %), "
                       + ("every pair" if full else f"stratified random: one uniformly random replica per candidate "
                          f"(seed {SAMPLE_SEED}), all {len(wl.plans)} candidates")
                       + f"; {wall:.1f} s wall on {n_threads} threads, std::thread pool over pdsim::run"),
            "extrapolated": not full, "sample_wall_s": wall, "sample_pairs": len(sample),
            "projected_full_search_s": wall * r_all / r_sample, "replays_per_s": len(sample) / wall}
    parity = None
    if gpu_pairs is not None:
        mism, cands = 0, set()
        sums = [0] * len(wl.plans)
        bad = [False] * len(wl.plans)
        for k, p in enumerate(sample):
            g_st, g = gpu_pairs(p)
            same = g_st == st[k] and all(getattr(g, f) == getattr(att[k], f) for f in
                                         ("sessions_total", "sessions_completed", "slo_ok", "ttft_ok", "itl_ok"))
            mism += 0 if same else 1
            c = p // len(wl.traces)
            cands.add(c)
            if st[k] != 0:
                bad[c] = True
            else:
                sums[c] += att[k].slo_ok
        parity = {"pairs_checked": len(sample), "pairs_total": wl.n_pairs, "candidates_covered": len(cands),
                  "attainment_mismatches": mism, "sample": "the cpu_baseline sample",
                  "checker": "oracle/_ref (unmodified reference run())"}
        if full:
            key = [(-1 if bad[c] else sums[c], -c) for c in range(len(wl.plans))]
            parity["reference_best_candidate"] = max(range(len(wl.plans)), key=lambda c: key[c])
    return base, parity


def attainment_spread(res, wl):
    """How the candidates split between the regimes (SLO-attaining sessions over
    all sessions of the candidate's replicas): the search is informative only
    when both appear."""
    total = sum(int(t.n_sessions) for t in wl.traces)
    fr = sorted(res.candidate_slo_ok[c] / total for c in range(len(wl.plans)) if res.candidate_slo_ok[c] >= 0)
    if not fr:
        return None
    return {"best": fr[-1], "median": fr[len(fr) // 2], "worst": fr[0], "candidates_ge_90pct": sum(f >= 0.9 for f in fr),
            "candidates_lt_10pct": sum(f < 0.1 for f in fr), "valid_candidates": len(fr)}


# ---- reference arm ------------------------------------------------------------

def run_reference(args, rank, world):
    """The unmodified reference's CPU plan search (oracle/_ref), inputs built
    through the reference itself (oracle/ref_workloads.py: its gen_trace,
    synth_profile and top_k) — no product code is loaded. Each step replays a
    bounded random sample of the pairs (the next n_threads of a fixed-seed
    permutation) on all host threads; value = request-rounds / wall."""
    if rank != 0:
        return
    from oracle import ref_workloads, refbind
    spec = specs.SPECS[args.config]()
    wl = ref_workloads.build(spec)
    n_threads = os.cpu_count() or 1
    perm = list(range(wl.n_pairs))
    random.Random(SAMPLE_SEED).shuffle(perm)
    # three pairs per thread per step, heaviest first, so the pool's wall time
    # is not one long pair with idle threads (a bias against the reference)
    step_pairs = min(wl.n_pairs, 3 * n_threads) if wl.n_pairs > 4 * n_threads else wl.n_pairs
    cursor = 0

    def take(n):
        nonlocal cursor
        out = [perm[(cursor + k) % wl.n_pairs] for k in range(n)]
        cursor += n
        return heavy_first(out, wl.traces, wl.plans)

    for _ in range(args.warmup):
        refbind.plan_search_list(wl.traces, wl.plans, wl.profile, wl.params, wl.seed, take(min(step_pairs, n_threads)),
                                 n_threads)
    total_t, total_rounds, total_pairs = 0.0, 0, 0
    for _ in range(args.steps):
        pairs = take(step_pairs)
        _, _, wall = refbind.plan_search_list(wl.traces, wl.plans, wl.profile, wl.params, wl.seed, pairs, n_threads)
        total_t += wall
        total_rounds += sum(wl.rounds_of_pair(p) for p in pairs)
        total_pairs += len(pairs)
    v = total_rounds / total_t
    full = step_pairs == wl.n_pairs
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference gen_trace presets on the reference's own RNG; synth_profile seed 7)",
            "config": specs.config_dict(spec),
            "planner_wall_s_projected": total_t / total_rounds * (sum(int(t.n_rounds) for t in wl.traces) * len(wl.plans)),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": n_threads, "kind": "reference",
                             "sample": (f"{step_pairs} pairs per step" + (" (every pair)" if full else
                                        f" of {wl.n_pairs}: consecutive slices of a fixed-seed random permutation "
                                        f"({total_pairs} distinct-or-wrapped pairs timed, extrapolated)"))},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- our arm ------------------------------------------------------------------

def measure(ctx, wl, pairs, args, stream, flush, world, steps, warmup, clock_index=None):
    """Warm-up, then `steps` timed searches of `pairs` with inputs resident;
    L2 flushed before each. Returns (per-step ms list, kernel ms list,
    launches, last result, clock summary)."""
    import torch
    for _ in range(warmup):
        ctx.search_staged_list(wl.seed, pairs)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    times, kernel_ms, launches, res = [], [], 0, None
    sampler = ClockSampler(clock_index) if clock_index is not None else None
    if sampler:
        sampler.__enter__()
    try:
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            res = ctx.search_staged_list(wl.seed, pairs)
            ev1.record(stream)
            torch.cuda.synchronize()
            times.append(ev0.elapsed_time(ev1))
            kernel_ms.append(res.kernel_ms)
            launches += res.kernel_launches
    finally:
        if sampler:
            sampler.__exit__()
    return times, kernel_ms, launches, res, (sampler.summary() if sampler else None)


def max_over_ranks(x, world):
    import torch
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args, rank, world, local):
    import torch
    from paper_2602_14516_b200 import native, workloads

    # PDSIM_BENCH_SHARED_GPU=1 (functional check of the N > 1 path on a
    # one-GPU box only): ranks share the visible GPU; never a reported number.
    shared = os.environ.get("PDSIM_BENCH_SHARED_GPU") == "1"
    if shared:
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if shared else "nccl", device_id=None if shared else torch.device("cuda", local))
    spec = specs.SPECS[args.config]()
    wl = workloads.build(spec)
    stream = torch.cuda.current_stream()
    ctx = native.Context(local)
    ctx.set_stream(stream.cuda_stream)
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    if world > 1 and not shared:
        # the one collective: per-candidate counts all-reduced over NCCL by
        # the library itself, at the end of every search (pdsim_gpu_comm_init)
        obj = [native.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.comm_init(world, rank, obj[0])
        ctx.set_global_sessions(sum(int(t.n_sessions) for t in wl.traces))
    # this GPU's shard of the SAME search, heaviest pairs first
    pairs = native.shard_pairs(wl.traces, wl.plans, world, rank)
    C = len(wl.plans)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    times, kernel_ms, launches, res, clocks = measure(ctx, wl, pairs, args, stream, flush, world, args.steps,
                                                      args.warmup, clock_index=local)
    if shared and world > 1:
        # NCCL refuses two ranks on one device: the functional mode reduces the
        # shards' counts with the same rule over gloo (distributed.py)
        from paper_2602_14516_b200 import distributed
        totals = distributed.reduce_counts([res.candidate_slo_ok[c] for c in range(len(wl.plans))])
        res.best_candidate, res.best_slo_ok = distributed.argmax(totals)
    build = {abi.BUILD_LATENCY: "latency (hot subroutines inlined)",
             abi.BUILD_THROUGHPUT: "throughput (shared hot subroutines out of line)"}.get(ctx.last_kernel_build())
    total_ms = max_over_ranks(sum(times), world)
    rounds_all = all_rounds(wl)
    value = rounds_all * args.steps / (total_ms / 1e3)
    best, best_cnt = res.best_candidate, res.best_slo_ok

    # e2e: host buffers through the public C-ABI call every step — stage
    # (pack + H2D) + replay + reduction + D2H.
    e2e_ms, h2d, d2h = [], 0, 0
    reps = 1 if total_ms / args.steps > 5000 else 2  # bounded bench time on the long searches
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world == 1:
            r_e = ctx.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed)
            h2d = r_e.h2d_bytes
        else:
            ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
            r_e = ctx.search_staged_list(wl.seed, pairs)
            # packed trace arrays staged per rank (pack.hpp: f64 arrival, i32
            # round offsets, i32 incr / decode, f64 delay, i64 id, i32 ranks)
            # + the pair list
            h2d = sum(28 * int(t.n_sessions) + 4 + 16 * int(t.n_rounds) for t in wl.traces) + r_e.h2d_bytes
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        d2h = r_e.d2h_bytes
        assert shared or (r_e.best_candidate == best and r_e.best_slo_ok == best_cnt)
    te = max_over_ranks(statistics.median(e2e_ms), world)
    e2e_value = rounds_all / (te / 1e3)

    # Search mode ARGMAX (exact pruning): same plan and count, fewer replays;
    # reported beside the full-replay headline, which alone defines `value`.
    arg = None
    if world == 1 and not args.no_argmax_mode and C > 1:
        ctx.set_search_mode(abi.SEARCH_ARGMAX)
        am = []
        for _ in range(reps):
            flush.zero_()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            res_a = ctx.search_staged_list(wl.seed, pairs)
            ev1.record(stream)
            torch.cuda.synchronize()
            am.append(ev0.elapsed_time(ev1))
        ctx.set_search_mode(abi.SEARCH_FULL)
        arg = {"planner_wall_ms": statistics.median(am), "best_candidate": res_a.best_candidate,
               "best_slo_ok": res_a.best_slo_ok,
               "same_plan_as_full": res_a.best_candidate == best and res_a.best_slo_ok == best_cnt,
               "pruned_candidates": sum(1 for c in range(C) if res_a.candidate_slo_ok[c] == -2)}

    # Roofline of the dominant kernel (replay_kernel): algorithmic input bytes
    # per launch (24 B/round + 16 B/session for every pair of this shard,
    # SURVEY.md §8(d)) / its average CUDA-event duration.
    peak, peak_src = peaks()
    nt = len(wl.traces)
    bytes_launch = sum(24 * int(wl.traces[p % nt].n_rounds) + 16 * int(wl.traces[p % nt].n_sessions) for p in pairs)
    avg_k = statistics.mean(kernel_ms)
    achieved = bytes_launch / (avg_k / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{wl.name}.json")
    if os.path.exists(tp) and world == 1:
        try:
            t = json.load(open(tp))
            if t.get("config_desc") == spec.desc:
                traffic = t.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    pos = {p: k for k, p in enumerate(pairs)}
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, parity = cpu_baseline(wl, lambda p: (res.pair_status[pos[p]], res.pair_attainment[pos[p]]))
        if parity is not None and "reference_best_candidate" in parity:
            parity["argmax_identical"] = parity["reference_best_candidate"] == best

    secondary = {}
    sec_names = [] if not args.secondary or args.secondary.lower() == "none" else \
        [x for x in args.secondary.split(",") if x and x != args.config]
    for sec in (sec_names if world == 1 else []):
        s_spec = specs.SPECS[sec]()
        swl = workloads.build(s_spec)
        ctx.stage(swl.traces, swl.plans, swl.profile, swl.params)
        spairs = native.shard_pairs(swl.traces, swl.plans, 1, 0)
        s_times, s_kms, s_launches, s_res, _ = measure(ctx, swl, spairs, args, stream, flush, 1, 3, 1)
        s_rounds = all_rounds(swl)
        se = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r_se = ctx.plan_search(swl.traces, swl.plans, swl.profile, swl.params, swl.seed)
            torch.cuda.synchronize()
            se.append((time.perf_counter() - t0) * 1e3)
        entry = {"config": specs.config_dict(s_spec), "value": s_rounds * len(s_times) / (sum(s_times) / 1e3),
                 "unit": UNIT, "ms_per_step": statistics.mean(s_times), "kernel_ms": statistics.mean(s_kms),
                 "e2e": {"value": s_rounds / (statistics.median(se) / 1e3), "unit": UNIT,
                         "h2d_bytes_per_step": r_se.h2d_bytes, "d2h_bytes_per_step": r_se.d2h_bytes},
                 "best_candidate": s_res.best_candidate, "best_slo_ok": s_res.best_slo_ok, "steps": len(s_times),
                 "candidate_attainment": attainment_spread(s_res, swl)}
        if not args.no_cpu_baseline:
            spos = {p: k for k, p in enumerate(spairs)}
            scpu, spar = cpu_baseline(swl, lambda p: (s_res.pair_status[spos[p]], s_res.pair_attainment[spos[p]]))
            if scpu:
                entry["cpu_baseline"] = scpu
            if spar:
                if "reference_best_candidate" in spar:
                    spar["argmax_identical"] = spar["reference_best_candidate"] == s_res.best_candidate
                entry["parity"] = spar
        entry["kernel_build"] = {abi.BUILD_LATENCY: "latency", abi.BUILD_THROUGHPUT: "throughput"}.get(
            ctx.last_kernel_build())
        secondary[sec] = entry

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference gen_trace presets on the host RNG; synth_profile seed 7)",
            "config": specs.config_dict(spec),
            "parallelism": (f"the same search sharded over {world} GPUs (cost-aware LPT split, pdsim_shard_pairs); "
                            "per-candidate counts all-reduced in-library over NCCL" if world > 1 else
                            "1 GPU, pairs in cost order (persistent kernel; above 8 pairs per SM, "
                            "per-SM queues grouping each candidate's pairs)"),
            "replays_per_s": wl.n_pairs * args.steps / (total_ms / 1e3),
            "planner_wall_ms": total_ms / args.steps,
            "kernel_ms": avg_k,
            "best_candidate": best, "best_slo_ok": best_cnt,
            "candidate_attainment": attainment_spread(res, wl),
            "best_plan": abi.format_plan(wl.plans[best]) if best >= 0 else None,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_launch": bytes_launch, "kernel": "replay_kernel", "kernel_build": build,
                         "note": "latency-bound serial DES per pair; see DESIGN.md §5 for issue/stall figures"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": te},
            "clocks": clocks,
        }
        if shared:
            line["functional_only"] = "PDSIM_BENCH_SHARED_GPU=1: ranks share one GPU; not a scaling number"
        if arg:
            line["argmax_mode"] = arg
        if cpu:
            line["cpu_baseline"] = cpu
        if parity:
            line["parity"] = parity
        if secondary:
            line["secondary"] = secondary
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
