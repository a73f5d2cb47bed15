#!/usr/bin/env python3
"""bench.py — candidate-plan replay search throughput on B200.

One "step" = one full plan search over the workload: every (candidate,
replica) pair replayed through the GPU engine, SLO counts reduced per
candidate (NCCL all-reduce across ranks when N > 1), argmax taken.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

Prints ONE JSON line (rank 0). `value` is whole-job request-rounds/s with
inputs resident in HBM; `e2e` is the same metric through the host-buffer
C-ABI call (H2D + kernels + D2H every step).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate-plan trace replays/sec (request-rounds/sec); planner wall-time"
UNIT = "request-rounds/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
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
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def shard(n_pairs, rank, world):
    b = n_pairs * rank // world
    e = n_pairs * (rank + 1) // world
    return b, e


def cpu_baseline(wl, seconds, gpu_res=None):
    """The reference's own CPU path (oracle/_ref, unmodified reference sources)
    on all host threads over a bounded sample of the workload's pairs. When
    the GPU result of the same search is given, the sampled pairs double as a
    parity check of the timed run: per-pair attainment must be identical, and
    when every pair was sampled, so must the argmax."""
    from oracle import refbind
    if not refbind.available():
        return None, None
    n_threads = os.cpu_count() or 1
    pairs = wl.n_pairs
    t_total, rounds, done = 0.0, 0, 0
    chunk = max(n_threads, 1)
    mism = 0
    sums = [0] * len(wl.plans)
    bad = [False] * len(wl.plans)
    while done < pairs and t_total < seconds:
        e = min(pairs, done + chunk)
        att, st, wall = refbind.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed,
                                            n_threads=n_threads, pair_begin=done, pair_end=e)
        if gpu_res is not None:
            for k in range(e - done):
                p = done + k
                c = p // len(wl.traces)
                g = gpu_res.pair_attainment[p]
                same = gpu_res.pair_status[p] == st[k] and all(
                    getattr(g, f) == getattr(att[k], f) for f in ("sessions_total", "sessions_completed", "slo_ok",
                                                                  "ttft_ok", "itl_ok"))
                mism += 0 if same else 1
                if st[k] != 0:
                    bad[c] = True
                else:
                    sums[c] += att[k].slo_ok
        t_total += wall
        rounds += wl.rounds_in(done, e)
        done = e
    base = {"value": rounds / t_total, "unit": UNIT, "cores": n_threads, "kind": "reference",
            "sample": f"{done}/{pairs} pairs of {wl.name} (first {done} in enumeration order), "
                      f"{t_total:.1f} s on {n_threads} threads, std::thread pool over pdsim::run",
            "replays_per_s": done / t_total}
    parity = None
    if gpu_res is not None:
        parity = {"pairs_checked": done, "pairs_total": pairs, "attainment_mismatches": mism,
                  "checker": "oracle/_ref (unmodified reference run())"}
        if done == pairs:
            key = [(-1 if bad[c] else sums[c], -c) for c in range(len(wl.plans))]
            ref_best = max(range(len(wl.plans)), key=lambda c: key[c])
            parity["reference_best_candidate"] = ref_best
            parity["argmax_identical"] = ref_best == gpu_res.best_candidate
    return base, parity


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_2602_14516_b200 import workloads
    from oracle import refbind
    # same workload as our arm: at N > 1 the C2 search grows to N replicas
    wl = workloads.c2(replicas=world) if (args.config == "C2" and world > 1) else workloads.CONFIGS[args.config]()
    n_threads = os.cpu_count() or 1
    # each step = a bounded sample of the pairs (~10 s of CPU work at most)
    probe_end = min(wl.n_pairs, n_threads)
    _, _, w0 = refbind.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed, n_threads, 0, probe_end)
    per_pair = w0 / probe_end * n_threads
    step_pairs = int(max(n_threads, min(wl.n_pairs, 8.0 * n_threads / max(per_pair, 1e-6))))
    for _ in range(args.warmup):
        refbind.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed, n_threads, 0,
                            min(step_pairs, n_threads))
    total_t, total_rounds, cursor = 0.0, 0, 0
    for _ in range(args.steps):
        b = cursor % wl.n_pairs
        e = min(wl.n_pairs, b + step_pairs)
        _, _, wall = refbind.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed, n_threads, b, e)
        total_t += wall
        total_rounds += wl.rounds_in(b, e)
        cursor = e
    v = total_rounds / total_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference gen_trace presets, host RNG)",
            "config": {"workload": wl.desc, "config": wl.name, "pairs": wl.n_pairs,
                       "step_sample_pairs": step_pairs},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": n_threads, "kind": "reference",
                             "sample": f"{step_pairs} pairs per step of {wl.n_pairs}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_2602_14516_b200 import abi, native, workloads

    # PDSIM_BENCH_SHARED_GPU=1 (functional check of the N > 1 path on a
    # one-GPU box only): ranks share the visible GPUs and reduce over gloo.
    # Never used for a reported number: NCCL over one GPU per rank is the path.
    shared = os.environ.get("PDSIM_BENCH_SHARED_GPU") == "1"
    if shared:
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # N > 1: weak scaling over trace replicas. The workload grows to N
    # replicas of the trace; rank r replays every candidate on replica r
    # (no data-path communication), and the per-candidate SLO counts are
    # summed over replicas by the one collective before the argmax.
    if args.config == "C2" and world > 1:
        wl = workloads.c2(replicas=world)
    else:
        wl = workloads.CONFIGS[args.config]()
    n_pairs = wl.n_pairs
    if len(wl.traces) == world and world > 1:
        my_traces = [wl.traces[rank]]
        b, e = 0, len(wl.plans)
        my_bytes = (24 * wl.traces[rank].n_rounds + 16 * wl.traces[rank].n_sessions) * len(wl.plans)
    else:
        my_traces = wl.traces
        b, e = shard(n_pairs, rank, world)
        my_bytes = wl.input_bytes(b, e)
    stream = torch.cuda.current_stream()
    ctx = native.Context(local)
    ctx.set_stream(stream.cuda_stream)
    ctx.stage(my_traces, wl.plans, wl.profile, wl.params)
    C = len(wl.plans)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def step(staged=True):
        res = ctx.search_staged(wl.seed, b, e) if staged else ctx.plan_search(
            my_traces, wl.plans, wl.profile, wl.params, wl.seed, b, e)
        if world == 1:  # the library's own device argmax (argmax_kernel)
            return res, res.best_candidate, res.best_slo_ok
        cand = torch.tensor([res.candidate_slo_ok[c] for c in range(C)], dtype=torch.int64, device="cuda")
        bad = (cand < 0).to(torch.int64)
        cnt = torch.clamp(cand, min=0)
        if world > 1:  # the one collective: per-candidate counts over NVLink
            dist.all_reduce(cnt)
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        key = torch.where(bad > 0, torch.full_like(cnt, -1), cnt)
        best = int(torch.argmax(key).item())  # first max = smallest index
        return res, best, int(key[best].item())

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times, kernel_ms, launches = [], [], 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            res, best, best_cnt = step()
            ev1.record(stream)
            torch.cuda.synchronize()
            times.append(ev0.elapsed_time(ev1))
            kernel_ms.append(res.kernel_ms)
            launches += res.kernel_launches
    my_ms = sum(times)
    t = torch.tensor([my_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    rounds_all = wl.rounds_in(0, n_pairs)
    value = rounds_all * args.steps / (total_ms / 1e3)

    # e2e: host buffers through the public C-ABI call (H2D + kernels + D2H)
    e2e_ms, h2d, d2h = [], 0, 0
    for _ in range(max(2, min(args.steps, 3))):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res_e, _, _ = step(staged=False)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d, d2h = res_e.h2d_bytes, res_e.d2h_bytes
    te = torch.tensor([statistics.median(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = rounds_all / (float(te.item()) / 1e3)

    # Search mode ARGMAX (exact pruning, include/pdsim_gpu.h): same plan and
    # count, fewer replays; reported beside the full-replay headline, which
    # alone defines `value`.
    arg = None
    if world == 1:
        ctx.set_search_mode(abi.SEARCH_ARGMAX)
        am = []
        for _ in range(max(2, min(args.steps, 3))):
            flush.zero_()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            res_a = ctx.search_staged(wl.seed, b, e)
            ev1.record(stream)
            torch.cuda.synchronize()
            am.append(ev0.elapsed_time(ev1))
        ctx.set_search_mode(abi.SEARCH_FULL)
        arg = {"planner_wall_ms": statistics.median(am), "best_candidate": res_a.best_candidate,
               "best_slo_ok": res_a.best_slo_ok, "same_plan_as_full": res_a.best_candidate == best and
               res_a.best_slo_ok == best_cnt,
               "pruned_candidates": sum(1 for c in range(C) if res_a.candidate_slo_ok[c] == -2)}

    # roofline of the dominant kernel (replay_kernel): algorithmic input bytes
    # per launch (24 B/round + 16 B/session per pair of this shard) / its
    # average CUDA-event duration.
    peak, peak_src = peaks()
    bytes_launch = my_bytes
    avg_k = statistics.mean(kernel_ms)
    achieved = bytes_launch / (avg_k / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{wl.name}.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, parity = cpu_baseline(wl, args.cpu_sample_seconds, gpu_res=res)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": ("weak" if len(wl.traces) == world else "strong") if world > 1 else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference gen_trace presets on the host RNG; synth_profile seed 7)",
            "config": {"workload": wl.desc, "config": wl.name, "model_cost": wl.model, "pairs": n_pairs,
                       "candidates": C, "replicas": len(wl.traces),
                       "sessions": [int(x.n_sessions) for x in wl.traces][:4],
                       "parallelism": (f"one trace replica per GPU ({world} GPUs), counts all-reduced"
                                       if len(wl.traces) == world and world > 1
                                       else f"pairs sharded over {world} GPU(s)"),
                       "l2": "flushed between timed steps (256 MiB write)"},
            "replays_per_s": n_pairs * args.steps / (total_ms / 1e3),
            "planner_wall_ms": total_ms / args.steps,
            "kernel_ms": avg_k,
            "best_candidate": best, "best_slo_ok": best_cnt,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_launch": bytes_launch, "kernel": "replay_kernel"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": float(te.item())},
            "clocks": clk.summary(),
        }
        if arg:
            line["argmax_mode"] = arg
        if cpu:
            line["cpu_baseline"] = cpu
        if parity:
            line["parity"] = parity
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
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
