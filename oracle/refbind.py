"""ctypes loader for oracle/_ref/libpdsim_ref.so (TEST INFRASTRUCTURE ONLY).

The library is the unmodified reference simulator (/root/reference/proj/src)
plus oracle/ref_shim.cpp. It exists only as the checker for parity tests and as
the CPU baseline timed by bench.py; the product never loads it.
"""
import ctypes as C
import os

from paper_2602_14516_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libpdsim_ref.so")

_lib = None


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(
                f"{LIB_PATH} missing: build it with `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.ref_last_error.restype = C.c_char_p
        L.ref_synth_profile.argtypes = [P(abi.SynthSpec), C.c_uint64, P(abi.Profile)]
        L.ref_profile_hash.argtypes = [P(abi.Profile)]
        L.ref_profile_hash.restype = C.c_uint64
        L.ref_profile_validate.argtypes = [P(abi.Profile)]
        L.ref_preset_stats.argtypes = [C.c_char_p, P(abi.TraceStats)]
        L.ref_gen_trace.argtypes = [P(abi.TraceStats), C.c_char_p, C.c_double, C.c_int32, C.c_uint64]
        L.ref_gen_trace.restype = C.c_void_p
        L.ref_trace_view.argtypes = [C.c_void_p, P(abi.Trace)]
        L.ref_trace_free.argtypes = [C.c_void_p]
        L.ref_trace_hash.argtypes = [P(abi.Trace), C.c_char_p]
        L.ref_trace_hash.restype = C.c_uint64
        L.ref_trace_validate.argtypes = [P(abi.Trace)]
        L.ref_run.argtypes = [P(abi.Trace), P(abi.Plan), P(abi.Profile), P(abi.SchedParams), C.c_uint64,
                              P(abi.RunOutput), P(C.c_uint64), C.c_int64, P(C.c_int64), P(C.c_double),
                              P(C.c_double), P(C.c_int64)]
        L.ref_plan_search.argtypes = [P(abi.SearchInput), P(abi.Profile), P(abi.SchedParams), C.c_uint64,
                                      C.c_int32, P(abi.Attainment), P(C.c_int8), P(C.c_double)]
        L.ref_plan_search_list.argtypes = [P(abi.SearchInput), P(abi.Profile), P(abi.SchedParams), C.c_uint64,
                                           C.c_int32, P(C.c_int64), C.c_int64, P(abi.Attainment), P(C.c_int8),
                                           P(C.c_double)]
        L.ref_top_k_plans.argtypes = [P(C.c_int32), C.c_int32, C.c_int32, P(abi.Plan), C.c_int64]
        L.ref_top_k_plans.restype = C.c_int64
        L.ref_phase_sims.argtypes = [P(abi.Trace), P(abi.Profile), C.c_int32, P(abi.PhaseResult),
                                     P(abi.PhaseResult)]
        L.ref_estimate_coefficients.argtypes = [P(abi.TraceStats), C.c_char_p, C.c_double, P(abi.Profile),
                                                P(C.c_int32), C.c_int32, C.c_int32, C.c_uint64,
                                                P(abi.Coefficients)]
        L.ref_solve.argtypes = [P(abi.Coefficients), C.c_int32, P(abi.Plan), P(C.c_double), P(C.c_int32),
                                P(C.c_int32)]
        L.ref_top_k.argtypes = [P(abi.Coefficients), C.c_int32, C.c_int32, P(abi.Plan), P(C.c_double),
                                P(C.c_int32)]
        L.ref_top_k.restype = C.c_int64
        L.ref_report.argtypes = [P(abi.Trace), P(abi.Plan), P(abi.Profile), P(abi.SchedParams), C.c_uint64,
                                 P(abi.Report)]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def synth_profile(spec, seed):
    out = abi.Profile()
    _check(lib().ref_synth_profile(C.byref(spec), seed, C.byref(out)))
    return out


def profile_hash(profile):
    return lib().ref_profile_hash(C.byref(profile))


def preset_stats(name):
    out = abi.TraceStats()
    _check(lib().ref_preset_stats(name.encode(), C.byref(out)))
    return out


class RefTrace:
    """Owned reference-generated trace; .view is a pdsim_trace over its arrays."""

    def __init__(self, handle):
        self._h = handle
        self.view = abi.Trace()
        lib().ref_trace_view(handle, C.byref(self.view))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_trace_free(self._h)
            self._h = None


def gen_trace(stats, name, rate, n, seed):
    h = lib().ref_gen_trace(C.byref(stats), name.encode(), rate, n, seed)
    if not h:
        raise RefError(-1, lib().ref_last_error().decode())
    return RefTrace(h)


def trace_hash(view, name):
    return lib().ref_trace_hash(C.byref(view), name.encode())


def run(trace, plan, profile, params, seed, records=True, itl=False):
    """One reference replay. Returns (RunOutput, hashes[4], itl arrays|None)."""
    S, R = trace.n_sessions, trace.n_rounds
    out = abi.RunOutput()
    keep = []
    if records:
        d = (abi.Decision * max(R, 1))()
        t = (abi.TtftSample * max(R, 1))()
        s = (abi.SessionOutcome * max(S, 1))()
        keep += [d, t, s]
        out.decisions = C.cast(d, C.POINTER(abi.Decision))
        out.ttft_samples = C.cast(t, C.POINTER(abi.TtftSample))
        out.sessions = C.cast(s, C.POINTER(abi.SessionOutcome))
    hashes = (C.c_uint64 * 4)()
    n_itl = C.c_int64(0)
    itl_arrays = None
    if itl:
        # first call to size the ITL arrays
        _check(lib().ref_run(C.byref(trace), C.byref(plan), C.byref(profile), C.byref(params), seed, None,
                             None, 0, None, None, None, C.byref(n_itl)))
        n = max(n_itl.value, 1)
        ids = (C.c_int64 * (3 * n))()
        tm = (C.c_double * n)()
        vs = (C.c_double * n)()
        itl_arrays = (ids, tm, vs)
        _check(lib().ref_run(C.byref(trace), C.byref(plan), C.byref(profile), C.byref(params), seed,
                             C.byref(out), hashes, n, ids, tm, vs, C.byref(n_itl)))
    else:
        _check(lib().ref_run(C.byref(trace), C.byref(plan), C.byref(profile), C.byref(params), seed,
                             C.byref(out), hashes, 0, None, None, None, C.byref(n_itl)))
    out._keep = keep
    return out, list(hashes), itl_arrays, n_itl.value


def plan_search(traces, plans, profile, params, seed, n_threads=0, pair_begin=0, pair_end=-1):
    """Reference CPU plan search (thread pool over pairs). Returns (att, status, wall_s)."""
    tarr = (abi.Trace * len(traces))(*traces)
    parr = (abi.Plan * len(plans))(*plans)
    total = len(traces) * len(plans)
    end = total if pair_end < 0 else pair_end
    n = end - pair_begin
    inp = abi.SearchInput(len(traces), len(plans), tarr, parr, pair_begin, end)
    att = (abi.Attainment * max(n, 1))()
    st = (C.c_int8 * max(n, 1))()
    wall = C.c_double(0)
    _check(lib().ref_plan_search(C.byref(inp), C.byref(profile), C.byref(params), seed, n_threads, att, st,
                                 C.byref(wall)))
    return att, st, wall.value


def plan_search_list(traces, plans, profile, params, seed, pairs, n_threads=0):
    """The reference pool over an explicit pair list (pulled in list order).
    Returns (att, status, wall_s) indexed like `pairs`."""
    tarr = (abi.Trace * len(traces))(*traces)
    parr = (abi.Plan * len(plans))(*plans)
    inp = abi.SearchInput(len(traces), len(plans), tarr, parr, 0, -1)
    n = len(pairs)
    pl = (C.c_int64 * max(n, 1))(*pairs)
    att = (abi.Attainment * max(n, 1))()
    st = (C.c_int8 * max(n, 1))()
    wall = C.c_double(0)
    _check(lib().ref_plan_search_list(C.byref(inp), C.byref(profile), C.byref(params), seed, n_threads, pl, n,
                                      att, st, C.byref(wall)))
    return att, st, wall.value


def top_k_plans(degrees, total_gpus, capacity=1 << 20):
    ds = (C.c_int32 * len(degrees))(*degrees)
    n = lib().ref_top_k_plans(ds, len(degrees), total_gpus, None, 0)
    if n < 0:
        raise RefError(-1, lib().ref_last_error().decode())
    out = (abi.Plan * max(n, 1))()
    lib().ref_top_k_plans(ds, len(degrees), total_gpus, out, n)
    return list(out)[:n]


# ---- surrogate planner (reference planner.cpp:75-657) ----

def phase_sims(trace, profile, degree):
    """(prefill PhaseResult, decode PhaseResult) of the reference sims; a
    result's status carries the error the reference threw (0 = ok)."""
    pre, dec = abi.PhaseResult(), abi.PhaseResult()
    lib().ref_phase_sims(C.byref(trace), C.byref(profile), degree, C.byref(pre), C.byref(dec))
    return pre, dec


def estimate_coefficients(stats, rate, profile, degrees, total_gpus, seed, name="custom"):
    out = abi.Coefficients()
    dg = (C.c_int32 * len(degrees))(*degrees)
    rc = lib().ref_estimate_coefficients(C.byref(stats), name.encode(), rate, C.byref(profile), dg, len(degrees),
                                         total_gpus, seed, C.byref(out))
    return out, rc


def solve(coeffs, total_gpus):
    plan, z, g, f = abi.Plan(), C.c_double(), C.c_int32(), C.c_int32()
    _check(lib().ref_solve(C.byref(coeffs), total_gpus, C.byref(plan), C.byref(z), C.byref(g), C.byref(f)))
    return (plan, z.value, g.value) if f.value else None


def top_k(coeffs, total_gpus, k):
    plans = (abi.Plan * k)()
    zs = (C.c_double * k)()
    gs = (C.c_int32 * k)()
    n = lib().ref_top_k(C.byref(coeffs), total_gpus, k, plans, zs, gs)
    if n < 0:
        raise RefError(1, lib().ref_last_error().decode())
    return [(plans[i], zs[i], gs[i]) for i in range(n)]


def report(trace, plan, profile, params, seed):
    """build_report (metrics.cpp:138-190) of one reference replay."""
    out = abi.Report()
    _check(lib().ref_report(C.byref(trace), C.byref(plan), C.byref(profile), C.byref(params), seed, C.byref(out)))
    return out
