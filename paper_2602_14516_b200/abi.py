"""ctypes mirror of include/pdsim_gpu.h (the C-ABI of the replay engine).

Plain data layouts only; the loaders live in :mod:`paper_2602_14516_b200.native`.
Field order and sizes must match the header exactly (checked by
tests/test_abi.py against the compiled library's struct sizes).
"""
import ctypes as C

MAX_DEGREES = 8
MAX_BREAKPOINTS = 7
MAX_SEGMENTS = MAX_BREAKPOINTS + 1
MAX_GROUPS = 8
MAX_WORKERS = 64

OK, ERR_CONFIG, ERR_DOMAIN, ERR_CUDA, ERR_INTERNAL, ERR_PARSE = 0, 1, 2, 3, 4, 5
ROUTING_ADAPTIVE, ROUTING_ALWAYS_REMOTE, ROUTING_ALWAYS_LOCAL = 0, 1, 2
RATIONALES = ("slack_remote", "slack_local", "argmin", "forced_remote", "forced_local")
PAIR_OK, PAIR_INVALID, PAIR_ERROR, PAIR_PRUNED = 0, 1, 2, 3
SEARCH_FULL, SEARCH_ARGMAX = 0, 1
BUILD_AUTO, BUILD_LATENCY, BUILD_THROUGHPUT = 0, 1, 2  # pdsim_gpu_set_kernel_build


class Curve(C.Structure):
    _fields_ = [
        ("n_breakpoints", C.c_int32),
        ("reserved", C.c_int32),
        ("breakpoints", C.c_double * MAX_BREAKPOINTS),
        ("alpha", C.c_double * MAX_SEGMENTS),
        ("beta", C.c_double * MAX_SEGMENTS),
    ]


class Profile(C.Structure):
    _fields_ = [
        ("n_degrees", C.c_int32),
        ("degrees", C.c_int32 * MAX_DEGREES),
        ("reserved", C.c_int32),
        ("prefill", Curve * MAX_DEGREES),
        ("decode", Curve * MAX_DEGREES),
        ("kv", (Curve * MAX_DEGREES) * MAX_DEGREES),
        ("kv_bytes_per_token", C.c_int64),
        ("gpu_memory_capacity", C.c_int64),
        ("history_weight", C.c_double),
    ]


class Trace(C.Structure):
    _fields_ = [
        ("n_sessions", C.c_int64),
        ("n_rounds", C.c_int64),
        ("session_id", C.POINTER(C.c_int64)),
        ("arrival_time", C.POINTER(C.c_double)),
        ("round_offset", C.POINTER(C.c_int64)),
        ("incr_input_len", C.POINTER(C.c_int64)),
        ("decode_len", C.POINTER(C.c_int64)),
        ("interaction_delay", C.POINTER(C.c_double)),
        ("ttft_thres", C.c_double),
        ("itl_thres", C.c_double),
    ]


class Plan(C.Structure):
    _fields_ = [
        ("n_prefill_groups", C.c_int32),
        ("n_decode_groups", C.c_int32),
        ("prefill_degree", C.c_int32 * MAX_GROUPS),
        ("prefill_count", C.c_int32 * MAX_GROUPS),
        ("decode_degree", C.c_int32 * MAX_GROUPS),
        ("decode_count", C.c_int32 * MAX_GROUPS),
    ]


class SchedParams(C.Structure):
    _fields_ = [
        ("routing", C.c_int32),
        ("reorder", C.c_int32),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("window", C.c_int32),
        ("reserved", C.c_int32),
        ("stat_window", C.c_double),
    ]


class Decision(C.Structure):
    _fields_ = [
        ("time", C.c_double),
        ("session_id", C.c_int64),
        ("round", C.c_int32),
        ("worker", C.c_int32),
        ("local", C.c_int8),
        ("rationale", C.c_int8),
        ("has_estimate", C.c_int8),
        ("reserved", C.c_int8 * 5),
        ("estimated_cost", C.c_double),
    ]


class TtftSample(C.Structure):
    _fields_ = [
        ("session_id", C.c_int64),
        ("round", C.c_int32),
        ("kind", C.c_int8),
        ("local", C.c_int8),
        ("reserved", C.c_int8 * 2),
        ("created_time", C.c_double),
        ("completion_time", C.c_double),
        ("value", C.c_double),
    ]


class SessionOutcome(C.Structure):
    _fields_ = [
        ("session_id", C.c_int64),
        ("arrival_time", C.c_double),
        ("completion_time", C.c_double),
        ("admission_wait", C.c_double),
        ("mean_itl", C.c_double),
        ("rounds", C.c_int32),
        ("ttft_ok", C.c_int8),
        ("itl_ok", C.c_int8),
        ("slo_ok", C.c_int8),
        ("reserved", C.c_int8),
    ]


class Counters(C.Structure):
    _fields_ = [
        ("tasks_created", C.c_int64),
        ("tasks_completed", C.c_int64),
        ("tokens_decoded", C.c_int64),
        ("kv_bytes_residual", C.c_int64),
        ("max_postpone_observed", C.c_int32),
        ("events_in_order", C.c_int32),
    ]


class Attainment(C.Structure):
    _fields_ = [
        ("sessions_total", C.c_int64),
        ("sessions_completed", C.c_int64),
        ("slo_ok", C.c_int64),
        ("ttft_ok", C.c_int64),
        ("itl_ok", C.c_int64),
    ]


class ItlSample(C.Structure):
    """ItlSample (sim_engine.hpp:66-72)."""
    _fields_ = [
        ("session_id", C.c_int64),
        ("round", C.c_int32),
        ("token_index", C.c_int32),
        ("completion_time", C.c_double),
        ("value", C.c_double),
    ]


class MetricStat(C.Structure):
    _fields_ = [("mean", C.c_double), ("p95", C.c_double), ("count", C.c_int64)]


class Report(C.Structure):
    """Report (metrics.hpp:38-51)."""
    _fields_ = [
        ("sessions_total", C.c_int64),
        ("sessions_completed", C.c_int64),
        ("slo_attainment", C.c_double),
        ("ttft_attainment", C.c_double),
        ("itl_attainment", C.c_double),
        ("ttft_initial", MetricStat),
        ("ttft_incremental", MetricStat),
        ("itl", MetricStat),
        ("e2e_mean", C.c_double),
        ("local_fraction", C.c_double),
        ("empty", C.c_int32),
        ("reserved", C.c_int32),
    ]

    def as_tuple(self):
        m = lambda x: (x.mean, x.p95, x.count)  # noqa: E731
        return (self.sessions_total, self.sessions_completed, self.slo_attainment, self.ttft_attainment,
                self.itl_attainment, m(self.ttft_initial), m(self.ttft_incremental), m(self.itl), self.e2e_mean,
                self.local_fraction, self.empty)


class RunOutput(C.Structure):
    _fields_ = [
        ("decisions", C.POINTER(Decision)),
        ("ttft_samples", C.POINTER(TtftSample)),
        ("sessions", C.POINTER(SessionOutcome)),
        ("n_decisions", C.c_int64),
        ("n_ttft", C.c_int64),
        ("n_sessions", C.c_int64),
        ("counters", Counters),
        ("attainment", Attainment),
        ("itl_samples", C.POINTER(ItlSample)),
        ("itl_capacity", C.c_int64),
        ("n_itl", C.c_int64),
    ]


class SearchInput(C.Structure):
    _fields_ = [
        ("n_traces", C.c_int32),
        ("n_candidates", C.c_int32),
        ("traces", C.POINTER(Trace)),
        ("candidates", C.POINTER(Plan)),
        ("pair_begin", C.c_int64),
        ("pair_end", C.c_int64),
    ]


class SearchOutput(C.Structure):
    _fields_ = [
        ("pair_attainment", C.POINTER(Attainment)),
        ("pair_counters", C.POINTER(Counters)),
        ("pair_status", C.POINTER(C.c_int8)),
        ("candidate_slo_ok", C.POINTER(C.c_int64)),
        ("pair_events", C.POINTER(C.c_int64)),
        ("pair_cycles", C.POINTER(C.c_int64)),
        ("best_candidate", C.c_int32),
        ("reserved", C.c_int32),
        ("best_slo_ok", C.c_int64),
        ("kernel_ms", C.c_double),
        ("device_ms", C.c_double),
        ("kernel_launches", C.c_int64),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("pair_report", C.POINTER(Report)),
    ]


class SynthSpec(C.Structure):
    _fields_ = [
        ("n_degrees", C.c_int32),
        ("degrees", C.c_int32 * MAX_DEGREES),
        ("n_prefill_breakpoints", C.c_int32),
        ("n_decode_breakpoints", C.c_int32),
        ("prefill_alpha_min", C.c_double),
        ("prefill_alpha_max", C.c_double),
        ("prefill_beta_min", C.c_double),
        ("prefill_beta_max", C.c_double),
        ("prefill_breakpoints", C.c_double * MAX_BREAKPOINTS),
        ("decode_alpha_min", C.c_double),
        ("decode_alpha_max", C.c_double),
        ("decode_beta_min", C.c_double),
        ("decode_beta_max", C.c_double),
        ("decode_breakpoints", C.c_double * MAX_BREAKPOINTS),
        ("segment_growth_min", C.c_double),
        ("segment_growth_max", C.c_double),
        ("scaling_exponent", C.c_double),
        ("kv_bandwidth_bytes_per_sec", C.c_double),
        ("kv_latency_seconds", C.c_double),
        ("kv_reshard_penalty", C.c_double),
        ("kv_bytes_per_token", C.c_int64),
        ("gpu_memory_capacity", C.c_int64),
        ("history_weight", C.c_double),
    ]


class TraceStats(C.Structure):
    _fields_ = [
        ("mean_rounds", C.c_double),
        ("fixed_rounds", C.c_int32),
        ("reserved", C.c_int32),
        ("mean_prefill_len", C.c_double),
        ("mean_decode_len", C.c_double),
        ("length_cv", C.c_double),
        ("first_round_fraction", C.c_double),
        ("mean_interaction_delay", C.c_double),
        ("ttft_thres", C.c_double),
        ("itl_thres", C.c_double),
    ]


class PhaseResult(C.Structure):
    """PhaseSimResult (planner.hpp:62-66) + the status the reference would throw."""
    _fields_ = [
        ("p95", C.c_double),
        ("sample_count", C.c_int64),
        ("infeasible", C.c_int32),
        ("status", C.c_int32),
    ]


class Coefficients(C.Structure):
    """LatencyCoefficients (planner.hpp:55-60) over the sorted degree list."""
    _fields_ = [
        ("n_degrees", C.c_int32),
        ("degrees", C.c_int32 * MAX_DEGREES),
        ("reserved", C.c_int32),
        ("tau_pre", C.c_double * MAX_DEGREES),
        ("tau_dec", C.c_double * MAX_DEGREES),
        ("infeasible_pre", C.c_int8 * MAX_DEGREES),
        ("infeasible_dec", C.c_int8 * MAX_DEGREES),
    ]

    def as_dict(self):
        n = self.n_degrees
        return {
            "tau_pre": {self.degrees[i]: self.tau_pre[i] for i in range(n) if not self.infeasible_pre[i]},
            "tau_dec": {self.degrees[i]: self.tau_dec[i] for i in range(n) if not self.infeasible_dec[i]},
            "infeasible_pre": sorted(self.degrees[i] for i in range(n) if self.infeasible_pre[i]),
            "infeasible_dec": sorted(self.degrees[i] for i in range(n) if self.infeasible_dec[i]),
        }


def make_coefficients(tau_pre, tau_dec, infeasible_pre=(), infeasible_dec=()):
    """Coefficients from {degree: tau} dicts (+ infeasible degree sets)."""
    c = Coefficients()
    degs = sorted(set(tau_pre) | set(tau_dec) | set(infeasible_pre) | set(infeasible_dec))
    c.n_degrees = len(degs)
    for i, d in enumerate(degs):
        c.degrees[i] = d
        c.infeasible_pre[i] = 1 if d in infeasible_pre else 0
        c.infeasible_dec[i] = 1 if d in infeasible_dec else 0
        c.tau_pre[i] = tau_pre.get(d, 0.0)
        c.tau_dec[i] = tau_dec.get(d, 0.0)
    return c


STRUCTS = {
    "pdsim_curve": Curve,
    "pdsim_profile": Profile,
    "pdsim_trace": Trace,
    "pdsim_plan": Plan,
    "pdsim_sched_params": SchedParams,
    "pdsim_decision": Decision,
    "pdsim_ttft_sample": TtftSample,
    "pdsim_session_outcome": SessionOutcome,
    "pdsim_counters": Counters,
    "pdsim_attainment": Attainment,
    "pdsim_run_output": RunOutput,
    "pdsim_itl_sample": ItlSample,
    "pdsim_metric_stat": MetricStat,
    "pdsim_report": Report,
    "pdsim_search_input": SearchInput,
    "pdsim_search_output": SearchOutput,
    "pdsim_synth_spec": SynthSpec,
    "pdsim_trace_stats": TraceStats,
    "pdsim_phase_result": PhaseResult,
    "pdsim_coefficients": Coefficients,
}


def default_synth_spec():
    """SynthProfileSpec{} defaults (reference perf_model.hpp:110-139)."""
    s = SynthSpec()
    s.n_degrees = 4
    for i, d in enumerate((1, 2, 4, 8)):
        s.degrees[i] = d
    s.prefill_alpha_min, s.prefill_alpha_max = 0.008, 0.015
    s.prefill_beta_min, s.prefill_beta_max = 1.5e-5, 3.0e-5
    s.n_prefill_breakpoints = 2
    s.prefill_breakpoints[0], s.prefill_breakpoints[1] = 2048.0, 8192.0
    s.decode_alpha_min, s.decode_alpha_max = 0.004, 0.008
    s.decode_beta_min, s.decode_beta_max = 3.0e-4, 6.0e-4
    s.n_decode_breakpoints = 1
    s.decode_breakpoints[0] = 64.0
    s.segment_growth_min, s.segment_growth_max = 1.05, 1.30
    s.scaling_exponent = 0.7
    s.kv_bandwidth_bytes_per_sec = 2.0e10
    s.kv_latency_seconds = 0.002
    s.kv_reshard_penalty = 1.25
    s.kv_bytes_per_token = 163840
    s.gpu_memory_capacity = 96 * 1000 * 1000 * 1000
    s.history_weight = 0.1
    return s


def make_plan(x, y):
    """Plan from {degree: count} dicts (ascending degree order, like std::map)."""
    p = Plan()
    for i, d in enumerate(sorted(x)):
        p.prefill_degree[i], p.prefill_count[i] = d, x[d]
    p.n_prefill_groups = len(x)
    for i, d in enumerate(sorted(y)):
        p.decode_degree[i], p.decode_count[i] = d, y[d]
    p.n_decode_groups = len(y)
    return p


def plan_dict(p):
    x = {p.prefill_degree[i]: p.prefill_count[i] for i in range(p.n_prefill_groups)}
    y = {p.decode_degree[i]: p.decode_count[i] for i in range(p.n_decode_groups)}
    return x, y


def format_plan(p):
    """format_plan (reference planner.cpp:659-678)."""
    x, y = plan_dict(p)

    def phase(c):
        if not c:
            return "<none>"
        return " + ".join(f"<TP={d}, DP={n}>" for d, n in sorted(c.items()))

    return f"P:{phase(x)}, D:{phase(y)}"


def default_params(**kw):
    """SchedulerParams{} defaults (reference sim_engine.hpp:46-54)."""
    p = SchedParams(ROUTING_ADAPTIVE, 1, 0.9, 0.85, 3, 0, 10.0)
    for k, v in kw.items():
        setattr(p, k, v)
    return p
