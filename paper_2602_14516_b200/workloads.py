"""Pinned synthetic workloads for BASELINE.json configs C1-C5.

The reference has no named model cost models, no PP dimension and no
ReAct / mixed presets; this module is the repo's pinned mapping:

* cost-model presets as SynthProfileSpec overrides (perf_model.hpp:110-139),
  profile seed 7: ``llama3-8b`` = defaults with 131072 KV B/token,
  ``qwen-32b`` = prefill/decode alpha/beta ranges x4 with 262144 B/token,
  ``llama3-70b`` = ranges x8.75 with 327680 B/token;
* degrees {1,2,4,8}: TP{1,2,4} x PP{1,2} folded into degree = TP*PP;
* traces from the reference presets (workload.cpp:136-168) via gen_trace.

All generation runs on the host through the product library's generators
(bit-identical to the reference's, see tests/test_generators.py).
"""
import ctypes as C

import numpy as np

from . import abi, native

PROFILE_SEED = 7
ENGINE_SEED = 1
DEGREES = (1, 2, 4, 8)

MODEL_PRESETS = {
    "llama3-8b": dict(scale=1.0, kv_bytes_per_token=131072),
    "qwen-32b": dict(scale=4.0, kv_bytes_per_token=262144),
    "llama3-70b": dict(scale=8.75, kv_bytes_per_token=327680),
}


def model_spec(name):
    p = MODEL_PRESETS[name]
    s = native.default_synth_spec()
    k = p["scale"]
    for f in ("prefill_alpha_min", "prefill_alpha_max", "prefill_beta_min", "prefill_beta_max",
              "decode_alpha_min", "decode_alpha_max", "decode_beta_min", "decode_beta_max"):
        setattr(s, f, getattr(s, f) * k)
    s.kv_bytes_per_token = p["kv_bytes_per_token"]
    return s


def model_profile(name):
    return native.synth_profile(model_spec(name), PROFILE_SEED)


def trace_stats(kind):
    """toolbench / gaia / hotpotqa / dureader presets, plus the two
    fixed-round variants the configs name."""
    if kind == "toolbench-4fixed":  # C1: ReAct-style 4 fixed rounds
        st = native.preset_stats("toolbench")
        st.mean_rounds = 4.0
        st.fixed_rounds = 1
        return st
    if kind == "hotpotqa-8fixed":  # C3: iterative RAG, 8 fixed rounds
        st = native.preset_stats("hotpotqa")
        st.mean_rounds = 8.0
        st.fixed_rounds = 1
        return st
    return native.preset_stats(kind)


class Workload:
    def __init__(self, name, model, traces, plans, params, seed, total_gpus, desc):
        self.name = name
        self.model = model
        self.profile = model_profile(model)
        self.trace_bufs = traces
        self.traces = [t.view for t in traces]
        self.plans = plans
        self.params = params
        self.seed = seed
        self.total_gpus = total_gpus
        self.desc = desc

    @property
    def n_pairs(self):
        return len(self.traces) * len(self.plans)

    @property
    def request_rounds(self):
        """Σ over pairs of the trace's round count (the metric's unit)."""
        return sum(t.n_rounds for t in self.traces) * len(self.plans)

    def input_bytes(self, pair_begin=0, pair_end=-1):
        """Algorithmic bytes: 24 B per round + 16 B per session, per pair
        (Round = int64+int64+f64, workload.hpp:28-34; SessionSpec
        arrival_time f64 + session_id int64, workload.hpp:36-39)."""
        nt = len(self.traces)
        end = self.n_pairs if pair_end < 0 else pair_end
        per_trace = [24 * t.n_rounds + 16 * t.n_sessions for t in self.traces]
        return sum(per_trace[p % nt] for p in range(pair_begin, end))

    def rounds_in(self, pair_begin=0, pair_end=-1):
        nt = len(self.traces)
        end = self.n_pairs if pair_end < 0 else pair_end
        return sum(self.traces[p % nt].n_rounds for p in range(pair_begin, end))


def c1():
    st = trace_stats("toolbench-4fixed")
    tr = native.gen_trace(st, 8.0, 1000, 1)
    plan = abi.make_plan({1: 2}, {1: 2})
    return Workload("C1", "llama3-8b", [tr], [plan], abi.default_params(), ENGINE_SEED, 4,
                    "llama3-8b, fixed P:2x1 D:2x1, toolbench 1k sessions x 4 fixed rounds @8/s, 1 replay")


def c2(sessions=10000, rate=16.0, seed=5, total_gpus=8, replicas=1):
    """C2; with replicas > 1 (the multi-GPU weak-scaling form) trace replica
    k uses gen seed seed + k."""
    st = trace_stats("toolbench")
    trs = [native.gen_trace(st, rate, sessions, seed + k) for k in range(replicas)]
    plans = native.enumerate_plans(DEGREES, total_gpus)
    rep = "" if replicas == 1 else f" x {replicas} replicas (seeds {seed}..{seed + replicas - 1})"
    return Workload("C2", "llama3-8b", trs, plans, abi.default_params(), ENGINE_SEED, total_gpus,
                    f"llama3-8b, all {len(plans)} N={total_gpus} P/D plans over degrees {{1,2,4,8}}, "
                    f"toolbench {sessions} sessions @{rate}/s{rep}")


def c3(sessions=50000, rate=20.0, replicas=16, total_gpus=8):
    st = trace_stats("hotpotqa-8fixed")
    trs = native.gen_traces(st, [rate] * replicas, sessions, list(range(1, replicas + 1)))
    plans = native.enumerate_plans(DEGREES, total_gpus)
    return Workload("C3", "qwen-32b", trs, plans, abi.default_params(), ENGINE_SEED, total_gpus,
                    f"qwen-32b, {len(plans)} plans x {replicas} hotpotqa-8-round replicas of {sessions} sessions")


def c5(model="llama3-8b", rates=None, seeds=4, sessions=1000, total_gpus=8):
    """One model slice of C5: toolbench 1k-session traces over rates x seeds."""
    rates = rates or [1.0 + 0.5 * k for k in range(32)]
    st = trace_stats("toolbench")
    rs = [r for r in rates for _ in range(seeds)]
    trs = native.gen_traces(st, rs, sessions, [1000 + s for _ in rates for s in range(seeds)])
    plans = native.enumerate_plans(DEGREES, total_gpus)
    return Workload("C5", model, trs, plans, abi.default_params(), ENGINE_SEED, total_gpus,
                    f"{model}, {len(plans)} plans x {len(trs)} toolbench traces ({len(rates)} rates x {seeds} seeds)")


class OwnedTrace:
    """A host-built trace: numpy arrays kept alive, ``.view`` their pdsim_trace."""

    def __init__(self, sid, arrival, round_offset, incr, dec, delay, ttft_thres, itl_thres):
        self._arrays = [np.ascontiguousarray(sid, np.int64), np.ascontiguousarray(arrival, np.float64),
                        np.ascontiguousarray(round_offset, np.int64), np.ascontiguousarray(incr, np.int64),
                        np.ascontiguousarray(dec, np.int64), np.ascontiguousarray(delay, np.float64)]
        a = self._arrays
        ptr = lambda x, t: x.ctypes.data_as(C.POINTER(t))  # noqa: E731
        self.view = abi.Trace(len(a[0]), len(a[3]), ptr(a[0], C.c_int64), ptr(a[1], C.c_double),
                              ptr(a[2], C.c_int64), ptr(a[3], C.c_int64), ptr(a[4], C.c_int64),
                              ptr(a[5], C.c_double), ttft_thres, itl_thres)


def _arrays(v):
    S, R = int(v.n_sessions), int(v.n_rounds)
    get = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0)  # noqa: E731
    return (get(v.session_id, S).astype(np.int64), get(v.arrival_time, S), get(v.round_offset, S + 1).astype(np.int64),
            get(v.incr_input_len, R).astype(np.int64), get(v.decode_len, R).astype(np.int64),
            get(v.interaction_delay, R))


def merge_traces(a, b):
    """C4's mixed agent + RAG trace: the sessions of two
    traces merged by arrival time (stable: ties keep a's sessions first), ids
    renumbered 0..S-1 in merged order, each session keeping its rounds. The
    two presets share their SLO (workload.cpp:144, 156)."""
    if (a.ttft_thres, a.itl_thres) != (b.ttft_thres, b.itl_thres):
        raise ValueError("merge_traces: the traces' SLOs differ")
    sa, aa, oa, ia, da, ya = _arrays(a)
    sb, ab, ob, ib, db, yb = _arrays(b)
    arr = np.concatenate([aa, ab])
    order = np.argsort(arr, kind="stable")
    starts = np.concatenate([oa[:-1], ob[:-1] + len(ia)])
    lens = np.concatenate([np.diff(oa), np.diff(ob)])
    inc, dec, dly = np.concatenate([ia, ib]), np.concatenate([da, db]), np.concatenate([ya, yb])
    l_sorted = lens[order]
    off = np.zeros(len(order) + 1, np.int64)
    np.cumsum(l_sorted, out=off[1:])
    # gather each session's round slice in merged order
    idx = np.repeat(starts[order] - off[:-1], l_sorted) + np.arange(off[-1])
    return OwnedTrace(np.arange(len(order)), arr[order], off, inc[idx], dec[idx], dly[idx], a.ttft_thres, a.itl_thres)


C4_RATES = (0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0, 8.0)


def c4(rates=None, seeds=1, sessions=100000, total_gpus=8):
    """C4: llama3-70b, mixed toolbench + hotpotqa traces (sessions/2 each at
    rate/2 each, merged by arrival), an arrival-rate sweep x seeds. The full
    grid is 8 rates x 64 seeds (512 traces x 169 plans = 86 528 pairs, ~5 GB
    of host trace arrays); the default is its first seed."""
    rates = list(rates or C4_RATES)
    half = sessions // 2
    jobs = [(r, s) for s in range(seeds) for r in rates]
    tool = native.gen_traces(trace_stats("toolbench"), [r / 2 for r, _ in jobs], half,
                             [1 + 2 * k for k in range(len(jobs))])
    hot = native.gen_traces(trace_stats("hotpotqa"), [r / 2 for r, _ in jobs], sessions - half,
                            [2 + 2 * k for k in range(len(jobs))])
    trs = [merge_traces(t.view, h.view) for t, h in zip(tool, hot)]
    plans = native.enumerate_plans(DEGREES, total_gpus)
    return Workload("C4", "llama3-70b", trs, plans, abi.default_params(), ENGINE_SEED, total_gpus,
                    f"llama3-70b, {len(plans)} plans x {len(trs)} mixed toolbench+hotpotqa traces of {sessions} "
                    f"sessions ({len(rates)} rates x {seeds} seed(s))")


def c2_small():
    """C2 with a 2000-session trace (profiling / quick checks only)."""
    wl = c2(sessions=2000)
    wl.name = "C2s"
    return wl


CONFIGS = {"C1": c1, "C2": c2, "C2s": c2_small, "C3": c3, "C4": c4, "C5": c5}
