"""Parity helpers shared by the tests and __graft_entry__.smoke().

Checkers (TEST INFRASTRUCTURE): the reference simulator itself
(oracle/_ref/libpdsim_ref.so) when present, otherwise the plain-C
restatement (oracle/build/liboracle.so). Both share the C-ABI POD types.
"""
import ctypes as C
import os

from paper_2602_14516_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOSTSIM_PATH = os.path.join(ROOT, "tests", "native", "libhostsim.so")

_hostsim = None


def hostsim():
    """TEST-ONLY host build of the device engine (tests/native/hostsim.cpp)."""
    global _hostsim
    if _hostsim is None:
        L = C.CDLL(HOSTSIM_PATH)
        P = C.POINTER
        L.hostsim_run.argtypes = [P(abi.Trace), P(abi.Plan), P(abi.Profile), P(abi.SchedParams), C.c_uint64,
                                  P(abi.RunOutput)]
        L.hostsim_last_error.restype = C.c_char_p
        L.hostsim_run_counts.argtypes = L.hostsim_run.argtypes
        L.hostsim_fold_repeat.argtypes = [C.c_double, C.c_double, C.c_uint64]
        L.hostsim_fold_repeat.restype = C.c_double
        L.hostsim_run_report.argtypes = L.hostsim_run.argtypes[:5] + [P(abi.Report)]
        _hostsim = L
    return _hostsim


class Run:
    """Plain-Python view of a run's outputs, comparable field by field."""

    def __init__(self, out, dec, ttft, sess):
        self.counters = out.counters
        self.attainment = out.attainment
        self.n_decisions, self.n_ttft, self.n_sessions = out.n_decisions, out.n_ttft, out.n_sessions
        self.decisions = list(dec)[: out.n_decisions] if dec is not None else []
        self.ttft_samples = list(ttft)[: out.n_ttft] if ttft is not None else []
        self.sessions = list(sess)[: out.n_sessions] if sess is not None else []


def _alloc(trace):
    S, R = max(trace.n_sessions, 1), max(trace.n_rounds, 1)
    out = abi.RunOutput()
    dec, ttft, sess = (abi.Decision * R)(), (abi.TtftSample * R)(), (abi.SessionOutcome * S)()
    out.decisions = C.cast(dec, C.POINTER(abi.Decision))
    out.ttft_samples = C.cast(ttft, C.POINTER(abi.TtftSample))
    out.sessions = C.cast(sess, C.POINTER(abi.SessionOutcome))
    return out, dec, ttft, sess


class EngineError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def host_run(trace, plan, profile, params, seed):
    out, dec, ttft, sess = _alloc(trace)
    rc = hostsim().hostsim_run(C.byref(trace), C.byref(plan), C.byref(profile), C.byref(params), seed,
                               C.byref(out))
    if rc:
        raise EngineError(rc, hostsim().hostsim_last_error().decode())
    return Run(out, dec, ttft, sess)


def host_report(trace, plan, profile, params, seed):
    """Host engine build in search report mode: build_report of the replay."""
    out = abi.Report()
    rc = hostsim().hostsim_run_report(C.byref(trace), C.byref(plan), C.byref(profile), C.byref(params), seed,
                                      C.byref(out))
    if rc:
        raise EngineError(rc, hostsim().hostsim_last_error().decode())
    return out


def itl_capacity(trace):
    return max(sum(max(trace.decode_len[k] - 1, 0) for k in range(trace.n_rounds)), 1)


def host_run_itl(trace, plan, profile, params, seed):
    """Host engine build with materialised ITL samples."""
    out, dec, ttft, sess = _alloc(trace)
    cap = itl_capacity(trace)
    itls = (abi.ItlSample * cap)()
    out.itl_samples = C.cast(itls, C.POINTER(abi.ItlSample))
    out.itl_capacity = cap
    rc = hostsim().hostsim_run(C.byref(trace), C.byref(plan), C.byref(profile), C.byref(params), seed,
                               C.byref(out))
    if rc:
        raise EngineError(rc, hostsim().hostsim_last_error().decode())
    r = Run(out, dec, ttft, sess)
    r.itl_samples = [itl_tuple(itls[k]) for k in range(min(out.n_itl, cap))]
    r.n_itl = out.n_itl
    return r


def itl_tuple(x):
    return (x.session_id, x.round, x.token_index, x.completion_time, x.value)


def reference_itl(trace, plan, profile, params, seed):
    """The reference's SimResult::itl_samples as tuples (push order)."""
    from oracle import refbind
    _, _, arrays, n = refbind.run(trace, plan, profile, params, seed, records=True, itl=True)
    ids, tm, vs = arrays
    out = []
    for k in range(n):
        out.append((ids[3 * k], ids[3 * k + 1], ids[3 * k + 2], tm[k], vs[k]))
    return out


def to_chars(x):
    """std::to_chars(double) shortest round-trip form (metrics.cpp:32-36):
    the shorter of fixed and scientific notation, fixed on ties."""
    from decimal import Decimal
    x = float(x)
    if x == 0.0:
        return "-0" if str(x).startswith("-") else "0"
    sign, digits, exp = Decimal(repr(abs(x))).as_tuple()
    digits = list(digits)
    while len(digits) > 1 and digits[-1] == 0:
        digits.pop()
        exp += 1
    n = len(digits)
    ds = "".join(str(d) for d in digits)
    e10 = exp + n - 1
    sci = ds[0] + ("." + ds[1:] if n > 1 else "") + "e" + ("-" if e10 < 0 else "+") + f"{abs(e10):02d}"
    if exp >= 0:  # integral: libstdc++ prints the exact integer in fixed form
        fixed = str(int(abs(x)))
    elif -exp < n:
        fixed = ds[: n + exp] + "." + ds[n + exp:]
    else:
        fixed = "0." + "0" * (-exp - n) + ds
    out = fixed if len(fixed) <= len(sci) else sci
    return ("-" if x < 0 else "") + out


def itl_csv_fnv(samples):
    """FNV-1a of the reference's itl_samples.csv text (metrics.cpp:402-410)."""
    h = 1469598103934665603
    def feed(text):
        nonlocal h
        for c in text.encode():
            h ^= c
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    feed("session_id,round,token_index,completion_time,value\n")
    for sid, rnd, tok, t, v in samples:
        feed(f"{sid},{rnd},{tok},{to_chars(t)},{to_chars(v)}\n")
    return f"{h:016x}"


def diff_itl(got, want):
    if len(got) != len(want):
        return [f"itl_samples: {len(got)} != {len(want)}"]
    for k, (a, b) in enumerate(zip(got, want)):
        if a != b:
            return [f"itl_samples[{k}]: {a} != {b}"]
    return []


def host_run_counts(trace, plan, profile, params, seed):
    """Counts-only host replay (search mode: no records)."""
    out = abi.RunOutput()
    rc = hostsim().hostsim_run_counts(C.byref(trace), C.byref(plan), C.byref(profile), C.byref(params), seed,
                                      C.byref(out))
    if rc:
        raise EngineError(rc, hostsim().hostsim_last_error().decode())
    return Run(out, None, None, None)


def diff_counts(got, want):
    errs = []
    for f in CTR_FIELDS:
        if getattr(got.counters, f) != getattr(want.counters, f):
            errs.append(f"counter {f}: {getattr(got.counters, f)} != {getattr(want.counters, f)}")
    for f in ATT_FIELDS:
        if getattr(got.attainment, f) != getattr(want.attainment, f):
            errs.append(f"attainment {f}: {getattr(got.attainment, f)} != {getattr(want.attainment, f)}")
    return errs


def oracle_kind():
    from oracle import refbind
    return "reference" if refbind.available() else "c-oracle"


def oracle_run(trace, plan, profile, params, seed):
    """The checker's run(): the reference itself when built, else the C oracle."""
    from oracle import refbind
    if refbind.available():
        S, R = max(trace.n_sessions, 1), max(trace.n_rounds, 1)
        out, _, _, _ = refbind.run(trace, plan, profile, params, seed, records=True)
        dec = [out.decisions[i] for i in range(out.n_decisions)]
        ttft = [out.ttft_samples[i] for i in range(out.n_ttft)]
        sess = [out.sessions[i] for i in range(out.n_sessions)]
        r = Run(out, None, None, None)
        r.decisions, r.ttft_samples, r.sessions = dec, ttft, sess
        return r
    from oracle import cbind
    return cbind.run(trace, plan, profile, params, seed)


DEC_FIELDS = ("time", "session_id", "round", "local", "worker", "rationale", "has_estimate", "estimated_cost")
TTFT_FIELDS = ("session_id", "round", "kind", "local", "created_time", "completion_time", "value")
SESS_FIELDS = ("session_id", "arrival_time", "completion_time", "rounds", "admission_wait", "mean_itl",
               "ttft_ok", "itl_ok", "slo_ok")
CTR_FIELDS = ("tasks_created", "tasks_completed", "tokens_decoded", "kv_bytes_residual",
              "max_postpone_observed", "events_in_order")
ATT_FIELDS = ("sessions_completed", "slo_ok", "ttft_ok", "itl_ok")


def _tup(rec, fields):
    return tuple(getattr(rec, f) for f in fields)


def diff_runs(got, want):
    """Returns a list of human-readable mismatches (empty = bit-identical)."""
    errs = []
    for f in CTR_FIELDS:
        if getattr(got.counters, f) != getattr(want.counters, f):
            errs.append(f"counter {f}: {getattr(got.counters, f)} != {getattr(want.counters, f)}")
    for f in ATT_FIELDS:
        if getattr(got.attainment, f) != getattr(want.attainment, f):
            errs.append(f"attainment {f}: {getattr(got.attainment, f)} != {getattr(want.attainment, f)}")
    for name, fields in (("decisions", DEC_FIELDS), ("ttft_samples", TTFT_FIELDS), ("sessions", SESS_FIELDS)):
        a, b = getattr(got, name), getattr(want, name)
        if len(a) != len(b):
            errs.append(f"{name}: {len(a)} records != {len(b)}")
        for i, (x, y) in enumerate(zip(a, b)):
            tx, ty = _tup(x, fields), _tup(y, fields)
            if name == "decisions" and not x.has_estimate:
                tx, ty = tx[:-1], ty[:-1]
            if tx != ty:
                errs.append(f"{name}[{i}]: {tx} != {ty}")
                break
    return errs


def assert_same_run(got, want):
    errs = diff_runs(got, want)
    assert not errs, "\n".join(errs[:10])


# ---- canonical digests (golden fixtures) ------------------------------------

def _fnv(text):
    h = 1469598103934665603
    for c in text.encode():
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def _fmt(v):
    return float(v).hex() if isinstance(v, float) else str(int(v))


def record_lines(run):
    """Canonical text of every record (floats as exact hex)."""
    dec = []
    for d in run.decisions:
        f = [d.time, d.session_id, d.round, d.local, d.worker, d.rationale, d.has_estimate]
        if d.has_estimate:
            f.append(d.estimated_cost)
        dec.append(",".join(_fmt(x) for x in f))
    ttft = [",".join(_fmt(getattr(t, k)) for k in TTFT_FIELDS) for t in run.ttft_samples]
    sess = [",".join(_fmt(getattr(s, k)) for k in SESS_FIELDS) for s in run.sessions]
    return dec, ttft, sess


def digest(run):
    dec, ttft, sess = record_lines(run)
    return {
        "counters": {f: int(getattr(run.counters, f)) for f in CTR_FIELDS},
        "attainment": {f: int(getattr(run.attainment, f)) for f in ATT_FIELDS},
        "decisions": _fnv("\n".join(dec)),
        "ttft_samples": _fnv("\n".join(ttft)),
        "sessions": _fnv("\n".join(sess)),
    }


def trace_digest(view):
    import numpy as np
    S, R = view.n_sessions, view.n_rounds
    parts = [np.ctypeslib.as_array(view.session_id, (S,)).tobytes(),
             np.ctypeslib.as_array(view.arrival_time, (S,)).tobytes(),
             np.ctypeslib.as_array(view.round_offset, (S + 1,)).tobytes(),
             np.ctypeslib.as_array(view.incr_input_len, (R,)).tobytes(),
             np.ctypeslib.as_array(view.decode_len, (R,)).tobytes(),
             np.ctypeslib.as_array(view.interaction_delay, (R,)).tobytes()]
    import hashlib
    h = hashlib.sha256()
    for p in parts:
        h.update(p)
    h.update(float(view.ttft_thres).hex().encode() + float(view.itl_thres).hex().encode())
    return h.hexdigest()[:16]


def profile_digest(profile):
    import hashlib
    return hashlib.sha256(bytes(profile)).hexdigest()[:16]


# ---- golden case inputs ---------------------------------------------------------

def build_case(case):
    """Materialises a golden case's inputs with the product generators."""
    from paper_2602_14516_b200 import native
    spec = native.default_synth_spec()
    for k, v in case.get("spec", {}).items():
        if k == "degrees":
            spec.n_degrees = len(v)
            for i, d in enumerate(v):
                spec.degrees[i] = d
        else:
            setattr(spec, k, v)
    prof = native.synth_profile(spec, case["profile_seed"])
    if "sessions_manual" in case:
        trace = manual_trace(case["sessions_manual"], case["slo"])
    else:
        st = native.preset_stats(case["preset"])
        for k, v in case.get("stats", {}).items():
            setattr(st, k, v)
        trace = native.gen_trace(st, case["rate"], case["n"], case["gen_seed"])
    plan = abi.make_plan({int(k): v for k, v in case["x"].items()}, {int(k): v for k, v in case["y"].items()})
    params = abi.default_params(**case.get("params", {}))
    return trace, plan, prof, params


class ManualTrace:
    def __init__(self, sessions, slo):
        sid, arr, off, inc, dec, dl = [], [], [0], [], [], []
        for s in sessions:
            sid.append(s["id"])
            arr.append(s["arrival"])
            for r in s["rounds"]:
                inc.append(r[0])
                dec.append(r[1])
                dl.append(r[2])
            off.append(len(inc))
        self._arrays = [(C.c_int64 * max(len(sid), 1))(*sid), (C.c_double * max(len(arr), 1))(*arr),
                        (C.c_int64 * len(off))(*off), (C.c_int64 * max(len(inc), 1))(*inc),
                        (C.c_int64 * max(len(dec), 1))(*dec), (C.c_double * max(len(dl), 1))(*dl)]
        a = self._arrays
        self.view = abi.Trace(len(sid), len(inc), a[0], a[1], a[2], a[3], a[4], a[5], slo[0], slo[1])


def manual_trace(sessions, slo):
    return ManualTrace(sessions, slo)
