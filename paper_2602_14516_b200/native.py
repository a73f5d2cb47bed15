"""Loader and thin Python mirror of the C-ABI (include/pdsim_gpu.h).

The product is ``libpdsim_gpu.so`` (CUDA sm_100a kernels + host C++). This
module only marshals arguments; every replay runs on the GPU. There is no CPU
fallback: if the library or a B200 is missing, calls raise :class:`PdsimError`.

Python names follow the reference's C++ API (proj/include/pdsim/*.hpp):
``run`` (sim_engine.hpp:125-127), ``gen_trace`` / ``preset_stats``
(workload.hpp:78-86), ``synth_profile`` (perf_model.hpp:141-142), and the
batched ``plan_search`` added on top of them.
"""
import ctypes as C
import os

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
# PDSIM_LIB points at another in-tree build of the same library (A/B timing
# in tools/ab.py); the default is the package's own libpdsim_gpu.so.
LIB_PATH = os.environ.get("PDSIM_LIB") or os.path.join(HERE, "libpdsim_gpu.so")

_lib = None
ABI_VERSION = 3  # include/pdsim_gpu.h PDSIM_ABI_VERSION


class PdsimError(RuntimeError):
    """Raised for a non-zero status. ``code`` is the PDSIM_ERR_* value."""

    def __init__(self, code, msg):
        super().__init__(f"pdsim error {code}: {msg}")
        self.code = code


class ConfigError(PdsimError):
    pass


class DomainError(PdsimError):
    pass


def lib():
    """Loads libpdsim_gpu.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PdsimError(abi.ERR_CUDA, f"{LIB_PATH} not built (run __graft_entry__.build() or `make`)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.pdsim_abi_version.restype = C.c_int
        L.pdsim_last_error.restype = C.c_char_p
        L.pdsim_gpu_create.argtypes = [C.c_int, P(C.c_void_p)]
        L.pdsim_gpu_destroy.argtypes = [C.c_void_p]
        L.pdsim_gpu_last_error.argtypes = [C.c_void_p]
        L.pdsim_gpu_last_error.restype = C.c_char_p
        L.pdsim_gpu_set_stream.argtypes = [C.c_void_p, C.c_void_p]
        L.pdsim_gpu_run.argtypes = [C.c_void_p, P(abi.Trace), P(abi.Plan), P(abi.Profile), P(abi.SchedParams),
                                    C.c_uint64, P(abi.RunOutput)]
        L.pdsim_gpu_plan_search.argtypes = [C.c_void_p, P(abi.SearchInput), P(abi.Profile), P(abi.SchedParams),
                                            C.c_uint64, P(abi.SearchOutput)]
        L.pdsim_gpu_stage.argtypes = [C.c_void_p, P(abi.SearchInput), P(abi.Profile), P(abi.SchedParams)]
        L.pdsim_gpu_sweep.argtypes = [C.c_void_p, C.c_int32, P(abi.Trace), P(abi.Plan), C.c_int32,
                                      P(abi.SchedParams), P(abi.Profile), C.c_uint64, P(abi.SearchOutput)]
        L.pdsim_format_double.argtypes = [C.c_double, C.c_char_p, C.c_int32]
        L.pdsim_format_double.restype = C.c_int32
        L.pdsim_gpu_set_profiling.argtypes = [C.c_void_p, C.c_int]
        L.pdsim_gpu_set_search_mode.argtypes = [C.c_void_p, C.c_int]
        L.pdsim_gpu_set_kernel_build.argtypes = [C.c_void_p, C.c_int]
        L.pdsim_gpu_last_kernel_build.argtypes = [C.c_void_p]
        L.pdsim_gpu_profile_counters.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_int64), P(C.c_int64)]
        L.pdsim_gpu_search_staged.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_uint64, P(abi.SearchOutput)]
        L.pdsim_synth_spec_default.argtypes = [P(abi.SynthSpec)]
        L.pdsim_synth_profile.argtypes = [P(abi.SynthSpec), C.c_uint64, P(abi.Profile)]
        L.pdsim_profile_validate.argtypes = [P(abi.Profile)]
        L.pdsim_preset_stats.argtypes = [C.c_char_p, P(abi.TraceStats)]
        L.pdsim_gen_trace.argtypes = [P(abi.TraceStats), C.c_double, C.c_int32, C.c_uint64, P(C.c_void_p)]
        L.pdsim_trace_buf_view.argtypes = [C.c_void_p, P(abi.Trace)]
        L.pdsim_gen_trace_batch.argtypes = [P(abi.TraceStats), C.c_int32, P(C.c_double), C.c_int32,
                                            P(C.c_uint64), P(C.c_void_p)]
        L.pdsim_trace_buf_free.argtypes = [C.c_void_p]
        L.pdsim_trace_validate.argtypes = [P(abi.Trace)]
        L.pdsim_enumerate_plans.argtypes = [P(C.c_int32), C.c_int32, C.c_int32, P(abi.Plan), C.c_int64]
        L.pdsim_enumerate_plans.restype = C.c_int64
        L.pdsim_argmax_candidates.argtypes = [P(C.c_int64), C.c_int32]
        L.pdsim_argmax_candidates.restype = C.c_int32
        L.pdsim_gpu_phase_sims.argtypes = [C.c_void_p, C.c_int32, P(abi.Trace), P(C.c_int32), P(abi.Profile),
                                           P(abi.PhaseResult), P(abi.PhaseResult)]
        L.pdsim_gpu_estimate_coefficients.argtypes = [C.c_void_p, P(abi.TraceStats), C.c_int32, P(C.c_double),
                                                      P(C.c_uint64), P(abi.Profile), P(C.c_int32), C.c_int32,
                                                      C.c_int32, P(abi.Coefficients), P(C.c_int32)]
        L.pdsim_solve.argtypes = [P(abi.Coefficients), C.c_int32, P(abi.Plan), P(C.c_double), P(C.c_int32),
                                  P(C.c_int32)]
        L.pdsim_top_k.argtypes = [P(abi.Coefficients), C.c_int32, C.c_int32, P(abi.Plan), P(C.c_double),
                                  P(C.c_int32)]
        L.pdsim_top_k.restype = C.c_int64
        L.pdsim_gpu_set_global_sessions.argtypes = [C.c_void_p, C.c_int64]
        L.pdsim_shard_pairs.argtypes = [C.c_int32, P(C.c_int64), C.c_int32, P(abi.Plan), C.c_int32, C.c_int32,
                                        P(C.c_int64), C.c_int64]
        L.pdsim_shard_pairs.restype = C.c_int64
        L.pdsim_gpu_search_staged_list.argtypes = [C.c_void_p, P(C.c_int64), C.c_int64, C.c_uint64,
                                                   P(abi.SearchOutput)]
        L.pdsim_nccl_unique_id.argtypes = [P(C.c_uint8)]
        L.pdsim_gpu_comm_init.argtypes = [C.c_void_p, C.c_int32, C.c_int32, P(C.c_uint8)]
        L.pdsim_multi_plan_search.argtypes = [C.c_int32, P(C.c_int32), P(abi.SearchInput), P(abi.Profile),
                                              P(abi.SchedParams), C.c_uint64, C.c_int32, P(abi.SearchOutput)]
        if L.pdsim_abi_version() != ABI_VERSION:
            raise PdsimError(abi.ERR_INTERNAL, "ABI version mismatch")
        _lib = L
    return _lib


def _raise(rc, msg):
    msg = msg.decode() if isinstance(msg, bytes) else msg
    if rc == abi.ERR_CONFIG:
        raise ConfigError(rc, msg)
    if rc == abi.ERR_DOMAIN:
        raise DomainError(rc, msg)
    raise PdsimError(rc, msg)


def _check(rc, ctx=None):
    if rc != 0:
        L = lib()
        _raise(rc, L.pdsim_gpu_last_error(ctx) if ctx else L.pdsim_last_error())


# ---- host generators (reference RNG, host libm) -----------------------------

def default_synth_spec():
    s = abi.SynthSpec()
    lib().pdsim_synth_spec_default(C.byref(s))
    return s


def synth_profile(spec=None, seed=7):
    spec = spec or default_synth_spec()
    out = abi.Profile()
    _check(lib().pdsim_synth_profile(C.byref(spec), seed, C.byref(out)))
    return out


def preset_stats(name):
    out = abi.TraceStats()
    _check(lib().pdsim_preset_stats(name.encode(), C.byref(out)))
    return out


class TraceBuf:
    """An owned generated trace; ``.view`` is the pdsim_trace over its arrays."""

    def __init__(self, handle):
        self._h = handle
        self.view = abi.Trace()
        _check(lib().pdsim_trace_buf_view(handle, C.byref(self.view)))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.pdsim_trace_buf_free(self._h)
            self._h = None


def gen_trace(stats, arrival_rate, num_sessions, seed):
    h = C.c_void_p()
    _check(lib().pdsim_gen_trace(C.byref(stats), arrival_rate, num_sessions, seed, C.byref(h)))
    return TraceBuf(h)


def gen_traces(stats, rates, num_sessions, seeds):
    """Batched gen_trace on all host threads (bit-identical to gen_trace)."""
    n = len(rates)
    hs = (C.c_void_p * max(n, 1))()
    _check(lib().pdsim_gen_trace_batch(C.byref(stats), n, (C.c_double * max(n, 1))(*rates), num_sessions,
                                       (C.c_uint64 * max(n, 1))(*seeds), hs))
    return [TraceBuf(C.c_void_p(hs[k])) for k in range(n)]


def enumerate_plans(degrees, total_gpus):
    ds = (C.c_int32 * len(degrees))(*degrees)
    n = lib().pdsim_enumerate_plans(ds, len(degrees), total_gpus, None, 0)
    if n < 0:
        raise ConfigError(abi.ERR_CONFIG, "bad degree set")
    out = (abi.Plan * max(n, 1))()
    lib().pdsim_enumerate_plans(ds, len(degrees), total_gpus, out, n)
    return list(out)[:n]


# ---- device context -----------------------------------------------------------

class RunResult:
    """Mirror of SimResult (sim_engine.hpp:105-114); itl_samples is filled
    when run(..., itl=True)."""

    def __init__(self, out, dec, ttft, sess):
        self.counters = out.counters
        self.attainment = out.attainment
        self.decisions = list(dec)[: out.n_decisions] if dec is not None else None
        self.ttft_samples = list(ttft)[: out.n_ttft] if ttft is not None else None
        self.sessions = list(sess)[: out.n_sessions] if sess is not None else None
        self.n_decisions = out.n_decisions
        self.n_ttft = out.n_ttft
        self.n_sessions = out.n_sessions
        self.n_itl = out.n_itl
        self.itl_samples = []


class SearchResult:
    def __init__(self, out, att, ctr, st, cand, n_pairs):
        self.best_candidate = out.best_candidate
        self.best_slo_ok = out.best_slo_ok
        self.kernel_ms = out.kernel_ms
        self.device_ms = out.device_ms
        self.kernel_launches = out.kernel_launches
        self.h2d_bytes = out.h2d_bytes
        self.d2h_bytes = out.d2h_bytes
        self.pair_attainment = att
        self.pair_counters = ctr
        self.pair_status = st
        self.candidate_slo_ok = cand
        self.n_pairs = n_pairs
        self.pair_events, self.pair_cycles = out._diag
        self.reports = list(out._reports)[:n_pairs] if out._reports is not None else None


def search_input(traces, plans, pair_begin=0, pair_end=-1):
    tarr = (abi.Trace * len(traces))(*traces)
    parr = (abi.Plan * len(plans))(*plans)
    inp = abi.SearchInput(len(traces), len(plans), tarr, parr, pair_begin, pair_end)
    inp._keep = (tarr, parr)
    return inp


# ---- surrogate planner: exact assignment over coefficients (host C++) ------

def solve(coeffs, total_gpus):
    """solve (reference planner.cpp:482-578). Returns (plan, objective_z,
    gpus_used) or None when infeasible."""
    plan, z, g, f = abi.Plan(), C.c_double(), C.c_int32(), C.c_int32()
    _check(lib().pdsim_solve(C.byref(coeffs), total_gpus, C.byref(plan), C.byref(z), C.byref(g), C.byref(f)))
    return (plan, z.value, g.value) if f.value else None


def top_k(coeffs, total_gpus, k):
    """top_k (reference planner.cpp:605-657): [(plan, objective_z, gpus_used)]."""
    plans = (abi.Plan * k)()
    zs = (C.c_double * k)()
    gs = (C.c_int32 * k)()
    n = lib().pdsim_top_k(C.byref(coeffs), total_gpus, k, plans, zs, gs)
    if n < 0:
        _raise(abi.ERR_CONFIG, lib().pdsim_last_error())
    return [(plans[i], zs[i], gs[i]) for i in range(n)]


class Context:
    """A device context (pdsim_gpu_create). One per GPU / process."""

    def __init__(self, device=0):
        h = C.c_void_p()
        _check(lib().pdsim_gpu_create(device, C.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            lib().pdsim_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc):
        _check(rc, self._h)

    def phase_sims(self, traces, degrees, profile):
        """simulate_prefill_replica / simulate_decode_replica (reference
        planner.cpp:75-226) for jobs (traces[k], degrees[k]) in one launch.
        Returns [(prefill PhaseResult, decode PhaseResult)]."""
        n = len(traces)
        tv = (abi.Trace * max(n, 1))(*traces)
        dg = (C.c_int32 * max(n, 1))(*degrees)
        pre = (abi.PhaseResult * max(n, 1))()
        dec = (abi.PhaseResult * max(n, 1))()
        self._check(lib().pdsim_gpu_phase_sims(self._h, n, tv, dg, C.byref(profile), pre, dec))
        return [(pre[k], dec[k]) for k in range(n)]

    def estimate_coefficients(self, stats, rates, seeds, profile, degrees, total_gpus):
        """estimate_coefficients (reference planner.cpp:228-283) for every
        (rates[s], seeds[s]) setting in one device launch. Returns
        [(Coefficients, status)]."""
        n = len(rates)
        rs = (C.c_double * max(n, 1))(*rates)
        ss = (C.c_uint64 * max(n, 1))(*seeds)
        dg = (C.c_int32 * len(degrees))(*degrees)
        out = (abi.Coefficients * max(n, 1))()
        st = (C.c_int32 * max(n, 1))()
        self._check(lib().pdsim_gpu_estimate_coefficients(self._h, C.byref(stats), n, rs, ss, C.byref(profile), dg,
                                                          len(degrees), total_gpus, out, st))
        return [(out[k], st[k]) for k in range(n)]

    def set_stream(self, cuda_stream_ptr):
        self._check(lib().pdsim_gpu_set_stream(self._h, C.c_void_p(cuda_stream_ptr or 0)))

    def run(self, trace, plan, profile, params, seed, records=True, itl=False):
        """Drop-in for pdsim::run: one replay on the GPU. With itl=True the
        per-token ITL samples are materialised too (SimResult::itl_samples)."""
        S, R = trace.n_sessions, trace.n_rounds
        out = abi.RunOutput()
        dec = ttft = sess = itls = None
        if records:
            dec = (abi.Decision * max(R, 1))()
            ttft = (abi.TtftSample * max(R, 1))()
            sess = (abi.SessionOutcome * max(S, 1))()
            out.decisions = C.cast(dec, C.POINTER(abi.Decision))
            out.ttft_samples = C.cast(ttft, C.POINTER(abi.TtftSample))
            out.sessions = C.cast(sess, C.POINTER(abi.SessionOutcome))
        if itl:
            cap = sum(max(trace.decode_len[k] - 1, 0) for k in range(R))  # one sample per token after the first
            itls = (abi.ItlSample * max(cap, 1))()
            out.itl_samples = C.cast(itls, C.POINTER(abi.ItlSample))
            out.itl_capacity = cap
        self._check(lib().pdsim_gpu_run(self._h, C.byref(trace), C.byref(plan), C.byref(profile),
                                        C.byref(params), seed, C.byref(out)))
        r = RunResult(out, dec, ttft, sess)
        r.itl_samples = [itls[k] for k in range(min(out.n_itl, out.itl_capacity))] if itl else []
        return r

    def _outputs(self, n_pairs, n_cand, report=False):
        att = (abi.Attainment * max(n_pairs, 1))()
        ctr = (abi.Counters * max(n_pairs, 1))()
        st = (C.c_int8 * max(n_pairs, 1))()
        cand = (C.c_int64 * max(n_cand, 1))()
        ev = (C.c_int64 * max(n_pairs, 1))()
        cy = (C.c_int64 * max(n_pairs, 1))()
        out = abi.SearchOutput(C.cast(att, C.POINTER(abi.Attainment)), C.cast(ctr, C.POINTER(abi.Counters)),
                               C.cast(st, C.POINTER(C.c_int8)), C.cast(cand, C.POINTER(C.c_int64)),
                               C.cast(ev, C.POINTER(C.c_int64)), C.cast(cy, C.POINTER(C.c_int64)))
        out._diag = (ev, cy)
        out._reports = None
        if report:
            reps = (abi.Report * max(n_pairs, 1))()
            out.pair_report = C.cast(reps, C.POINTER(abi.Report))
            out._reports = reps
        return out, att, ctr, st, cand

    def plan_search(self, traces, plans, profile, params, seed, pair_begin=0, pair_end=-1, report=False):
        """Replays every (candidate, replica) pair in [pair_begin, pair_end).
        report=True adds the reference's build_report of every pair
        (SearchResult.reports)."""
        inp = search_input(traces, plans, pair_begin, pair_end)
        end = len(traces) * len(plans) if pair_end < 0 else pair_end
        n = end - pair_begin
        out, att, ctr, st, cand = self._outputs(n, len(plans), report)
        self._check(lib().pdsim_gpu_plan_search(self._h, C.byref(inp), C.byref(profile), C.byref(params), seed,
                                                C.byref(out)))
        return SearchResult(out, att, ctr, st, cand, n)

    def sweep(self, traces, plan, profile, settings, seed, report=True):
        """Batched `pdsim sweep` (include/pdsim_gpu.h pdsim_gpu_sweep): `plan`
        on every trace under every scheduler setting; pair k * len(traces) + r
        is setting k on trace r. The settings stay staged (search_staged)."""
        tv = (abi.Trace * len(traces))(*traces)
        sv = (abi.SchedParams * len(settings))(*settings)
        n = len(traces) * len(settings)
        out, att, ctr, st, cand = self._outputs(n, len(settings), report)
        self._check(lib().pdsim_gpu_sweep(self._h, len(traces), tv, C.byref(plan), len(settings), sv,
                                          C.byref(profile), seed, C.byref(out)))
        self._staged = (len(traces), len(settings))
        return SearchResult(out, att, ctr, st, cand, n)

    def search_staged_list(self, seed, pairs, report=False):
        """Replays the staged pairs in `pairs` (global indices) in list order;
        per-pair outputs follow the list (include/pdsim_gpu.h)."""
        nt, nc = self._staged
        arr = (C.c_int64 * max(len(pairs), 1))(*pairs)
        out, att, ctr, st, cand = self._outputs(len(pairs), nc, report)
        self._check(lib().pdsim_gpu_search_staged_list(self._h, arr, len(pairs), seed, C.byref(out)))
        return SearchResult(out, att, ctr, st, cand, len(pairs))

    def set_global_sessions(self, total):
        """Sessions of the whole search this context is a shard of (ARGMAX bounds)."""
        self._check(lib().pdsim_gpu_set_global_sessions(self._h, int(total)))

    def comm_init(self, world, rank, unique_id):
        """Joins the NCCL communicator of a sharded search (one process per GPU)."""
        buf = (C.c_uint8 * 128)(*unique_id)
        self._check(lib().pdsim_gpu_comm_init(self._h, world, rank, buf))

    def set_search_mode(self, mode):
        """abi.SEARCH_FULL (default) or abi.SEARCH_ARGMAX (exact pruning:
        same best_candidate / best_slo_ok, pruned candidates report -2)."""
        self._check(lib().pdsim_gpu_set_search_mode(self._h, int(mode)))

    def set_kernel_build(self, build):
        """abi.BUILD_AUTO / BUILD_LATENCY / BUILD_THROUGHPUT (pdsim_gpu_set_kernel_build)."""
        self._check(lib().pdsim_gpu_set_kernel_build(self._h, int(build)))

    def last_kernel_build(self):
        return lib().pdsim_gpu_last_kernel_build(self._h)

    def set_profiling(self, enable):
        self._check(lib().pdsim_gpu_set_profiling(self._h, 1 if enable else 0))

    def profile_counters(self):
        """(cycles[28], counts[28], replayed_pairs) of the last search
        (bucket meanings: include/pdsim_gpu.h, PDSIM_PROF_BUCKETS)."""
        cy = (C.c_int64 * 28)()
        n = (C.c_int64 * 28)()
        rp = C.c_int64(0)
        self._check(lib().pdsim_gpu_profile_counters(self._h, cy, n, C.byref(rp)))
        return list(cy), list(n), rp.value

    def stage(self, traces, plans, profile, params):
        inp = search_input(traces, plans)
        self._check(lib().pdsim_gpu_stage(self._h, C.byref(inp), C.byref(profile), C.byref(params)))
        self._staged = (len(traces), len(plans))

    def search_staged(self, seed, pair_begin=0, pair_end=-1, report=False):
        nt, nc = self._staged
        end = nt * nc if pair_end < 0 else pair_end
        n = end - pair_begin
        out, att, ctr, st, cand = self._outputs(n, nc, report)
        self._check(lib().pdsim_gpu_search_staged(self._h, pair_begin, pair_end, seed, C.byref(out)))
        return SearchResult(out, att, ctr, st, cand, n)


def shard_pairs(traces, plans, world, rank):
    """This rank's pairs (global index c * len(traces) + r) in queue order:
    the library's cost-aware LPT split (pdsim_shard_pairs)."""
    rounds = (C.c_int64 * max(len(traces), 1))(*[int(t.n_rounds) for t in traces])
    pv = (abi.Plan * max(len(plans), 1))(*plans)
    n = lib().pdsim_shard_pairs(len(traces), rounds, len(plans), pv, world, rank, None, 0)
    if n < 0:
        _check(abi.ERR_CONFIG)
    out = (C.c_int64 * max(n, 1))()
    lib().pdsim_shard_pairs(len(traces), rounds, len(plans), pv, world, rank, out, n)
    return list(out)[:n]


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    _check(lib().pdsim_nccl_unique_id(buf))
    return bytes(buf)


def multi_plan_search(devices, traces, plans, profile, params, seed, mode=abi.SEARCH_FULL):
    """One host thread, several GPUs (pdsim_multi_plan_search): shards, replays,
    all-reduces over NCCL; outputs indexed by global pair."""
    inp = search_input(traces, plans)
    n = len(traces) * len(plans)
    dv = (C.c_int32 * len(devices))(*devices)
    out, att, ctr, st, cand = Context._outputs(None, n, len(plans), False)
    _check(lib().pdsim_multi_plan_search(len(devices), dv, C.byref(inp), C.byref(profile), C.byref(params), seed,
                                         int(mode), C.byref(out)))
    return SearchResult(out, att, ctr, st, cand, n)


def format_double(x):
    """std::to_chars(double) shortest round-trip text (the reference's CSV
    number format), from the library."""
    buf = C.create_string_buffer(64)
    n = lib().pdsim_format_double(float(x), buf, 64)
    if n < 0:
        raise PdsimError(abi.ERR_INTERNAL, "format_double: buffer too small")
    return buf.value.decode()


def argmax_candidates(candidate_slo_ok):
    """Max Σslo_ok, ties to the smallest index, negatives (invalid) skipped."""
    arr = (C.c_int64 * len(candidate_slo_ok))(*candidate_slo_ok)
    return lib().pdsim_argmax_candidates(arr, len(candidate_slo_ok))
