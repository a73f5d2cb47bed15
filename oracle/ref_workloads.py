"""Benchmark workloads built through the UNMODIFIED reference (TEST / BASELINE
INFRASTRUCTURE ONLY).

bench.py's reference arm replays the reference's own CPU path on the same
inputs as the product arm, and must not load product code to build them.
This module turns a plain-data spec (paper_2602_14516_b200/specs.py, no
library behind it) into reference inputs with oracle/_ref only:

* traces: the reference's gen_trace (workload.cpp:170-229) per TraceJob;
  C4's mixed jobs are merged by arrival time here with numpy (stable, ids
  renumbered), the same rule as the product's workloads.merge_traces;
* cost model: the reference's synth_profile (perf_model.cpp:207-273) on the
  reference's default SynthProfileSpec scaled by the preset;
* candidates: the reference's top_k over every plan (planner.cpp:604-657),
  put in enumerate_counts order (specs.enumeration_order) so candidate
  indices — and so the argmax tie-break — mean the same in both arms.

tests/test_oracle.py checks that these inputs are byte-identical to the
product arm's (trace and profile hashes, plan order).
"""
import ctypes as C

import numpy as np

from paper_2602_14516_b200 import abi, specs

from . import refbind


class RefWorkload:
    def __init__(self, spec, traces, keep, profile, plans):
        self.spec = spec
        self.name = spec.name
        self.traces = traces
        self._keep = keep
        self.profile = profile
        self.plans = plans
        self.params = abi.default_params()
        self.seed = spec.engine_seed

    @property
    def n_pairs(self):
        return len(self.traces) * len(self.plans)

    def rounds_of_pair(self, p):
        return self.traces[p % len(self.traces)].n_rounds


def synth_spec_default():
    out = abi.SynthSpec()
    L = refbind.lib()
    L.ref_synth_spec_default.argtypes = [C.POINTER(abi.SynthSpec)]
    refbind._check(L.ref_synth_spec_default(C.byref(out)))
    return out


def model_profile(model):
    return refbind.synth_profile(specs.apply_model(synth_spec_default(), model), specs.PROFILE_SEED)


def trace_stats(kind):
    return specs.apply_stats(refbind.preset_stats(specs.STATS[kind][0]), kind)


class _Owned:
    def __init__(self, arrays, slo):
        self.arrays = arrays
        a = arrays
        ptr = lambda x, t: x.ctypes.data_as(C.POINTER(t))  # noqa: E731
        self.view = abi.Trace(len(a[0]), len(a[3]), ptr(a[0], C.c_int64), ptr(a[1], C.c_double),
                              ptr(a[2], C.c_int64), ptr(a[3], C.c_int64), ptr(a[4], C.c_int64),
                              ptr(a[5], C.c_double), slo[0], slo[1])


def _arrays(v):
    S, R = int(v.n_sessions), int(v.n_rounds)
    get = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0)  # noqa: E731
    return (get(v.session_id, S).astype(np.int64), get(v.arrival_time, S), get(v.round_offset, S + 1).astype(np.int64),
            get(v.incr_input_len, R).astype(np.int64), get(v.decode_len, R).astype(np.int64),
            get(v.interaction_delay, R))


def _merge(a, b):
    sa, aa, oa, ia, da, ya = _arrays(a)
    sb, ab, ob, ib, db, yb = _arrays(b)
    arr = np.concatenate([aa, ab])
    order = np.argsort(arr, kind="stable")
    starts = np.concatenate([oa[:-1], ob[:-1] + len(ia)])
    lens = np.concatenate([np.diff(oa), np.diff(ob)])
    l_sorted = lens[order]
    off = np.zeros(len(order) + 1, np.int64)
    np.cumsum(l_sorted, out=off[1:])
    idx = np.repeat(starts[order] - off[:-1], l_sorted) + np.arange(off[-1])
    inc, dec, dly = np.concatenate([ia, ib]), np.concatenate([da, db]), np.concatenate([ya, yb])
    arrays = (np.arange(len(order), dtype=np.int64), arr[order], off, inc[idx], dec[idx], dly[idx])
    return _Owned([np.ascontiguousarray(x) for x in arrays], (a.ttft_thres, a.itl_thres))


def _trace(job):
    t = refbind.gen_trace(trace_stats(job.kind), specs.STATS[job.kind][0], job.rate, job.sessions, job.seed)
    if job.merge_with is None:
        return t
    other = _trace(job.merge_with)  # keeps the reference-owned arrays alive while merging
    return _merge(t.view, other.view)


def plans_in_enumeration_order(degrees, total_gpus):
    ref = refbind.top_k_plans(list(degrees), total_gpus)
    order = {(tuple(sorted(x.items())), tuple(sorted(y.items()))): k
             for k, (x, y) in enumerate(specs.enumeration_order(degrees, total_gpus))}

    def key(p):
        x, y = abi.plan_dict(p)
        return order[(tuple(sorted(x.items())), tuple(sorted(y.items())))]

    out = sorted(ref, key=key)
    if [key(p) for p in out] != list(range(len(order))):
        raise RuntimeError("reference top_k and enumerate_counts disagree on the candidate set")
    return out


def build(spec):
    owned = [_trace(j) for j in spec.jobs]
    plans = [abi.make_plan(*spec.fixed_plan)] if spec.fixed_plan else plans_in_enumeration_order(spec.degrees,
                                                                                              spec.total_gpus)
    return RefWorkload(spec, [t.view for t in owned], owned, model_profile(spec.model), plans)
