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

from . import abi, native, specs
from .specs import DEGREES, ENGINE_SEED, MODEL_PRESETS, PROFILE_SEED  # noqa: F401


def model_spec(name):
    return specs.apply_model(native.default_synth_spec(), name)


def model_profile(name):
    return native.synth_profile(model_spec(name), PROFILE_SEED)


def trace_stats(kind):
    """toolbench / gaia / hotpotqa / dureader presets, plus the two
    fixed-round variants the configs name."""
    return specs.apply_stats(native.preset_stats(specs.STATS[kind][0]), kind)


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


def build_trace(job):
    """A spec TraceJob through the product generators (merged jobs: C4)."""
    tr = native.gen_trace(trace_stats(job.kind), job.rate, job.sessions, job.seed)
    if job.merge_with is None:
        return tr
    other = build_trace(job.merge_with)
    return merge_traces(tr.view, other.view)


def build(spec):
    """Workload of a specs.Spec: traces (all host threads for plain jobs),
    cost model, candidates (the reference's enumeration order)."""
    plain = all(j.merge_with is None for j in spec.jobs)
    if plain and len(spec.jobs) > 1 and len({j.kind for j in spec.jobs}) == 1 and len({j.sessions for j in spec.jobs}) == 1:
        trs = native.gen_traces(trace_stats(spec.jobs[0].kind), [j.rate for j in spec.jobs], spec.jobs[0].sessions,
                                [j.seed for j in spec.jobs])
    else:
        trs = [build_trace(j) for j in spec.jobs]
    if spec.fixed_plan:
        plans = [abi.make_plan(*spec.fixed_plan)]
    else:
        plans = native.enumerate_plans(spec.degrees, spec.total_gpus)
    wl = Workload(spec.name, spec.model, trs, plans, abi.default_params(), spec.engine_seed, spec.total_gpus, spec.desc)
    wl.spec = spec
    return wl


def c1():
    return build(specs.c1())


def c2(sessions=10000, rate=16.0, seed=5, total_gpus=8, replicas=1):
    """C2; with replicas > 1 trace replica k uses gen seed seed + k."""
    s = specs.c2(sessions, rate, seed, replicas)
    s.total_gpus = total_gpus
    return build(s)


def c3(sessions=50000, rate=specs.C3_RATE, replicas=16, total_gpus=8):
    s = specs.c3(sessions, rate, replicas)
    s.total_gpus = total_gpus
    return build(s)


def c5(model="llama3-8b", rates=None, seeds=4, sessions=1000, total_gpus=8):
    """One model slice of C5: toolbench 1k-session traces over rates x seeds."""
    s = specs.c5(model, rates, seeds, sessions)
    s.total_gpus = total_gpus
    return build(s)


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


C4_RATES = specs.C4_RATES


def c4(rates=None, seeds=1, sessions=100000, total_gpus=8):
    """C4: llama3-70b, mixed toolbench + hotpotqa traces (sessions/2 each at
    rate/2 each, merged by arrival), an arrival-rate sweep x seeds. The full
    grid is 8 rates x 64 seeds (512 traces x 169 plans = 86 528 pairs, ~5 GB
    of host trace arrays); the default is its first seed."""
    s = specs.c4(rates, seeds, sessions)
    s.total_gpus = total_gpus
    return build(s)


def c2_small():
    """C2 with a 2000-session trace (profiling / quick checks only)."""
    return build(specs.c2_small())


def c3_small():
    """C3 with 10 000-session replicas: the same 2704 pairs and per-SM
    concurrency, a fifth of the events (profiling only)."""
    return c3(sessions=10000)


CONFIGS = {"C1": c1, "C2": c2, "C2s": c2_small, "C3": c3, "C3s": c3_small, "C4": c4, "C5": c5}
