"""`pdsim sweep` as one batched GPU call (reference tools/pdsim.cpp:501-590).

The reference sweep generates one trace per arrival rate (gen_trace with the
sweep seed), then for every alpha x beta x window combination runs the plan
through `run()` (engine seed = the same seed) and writes one sweep.csv row of
build_report's figures. Here every (setting, rate) replay is a pair of a
single `pdsim_gpu_sweep` launch; the per-pair reports come back from the
device and the CSV text is assembled on the host exactly as the reference
formats it (std::to_chars numbers, rate-major row order).
"""
import ctypes as C

from . import abi, native

CSV_HEADER = ("rate,alpha,beta,window,slo_attainment,ttft_attainment,"
              "itl_attainment,ttft_initial_mean,ttft_initial_p95,ttft_incr_mean,"
              "ttft_incr_p95,itl_mean,itl_p95,e2e_mean,local_fraction\n")


def grid(base, alphas=None, betas=None, windows=None):
    """Settings in the reference's loop order (alpha, then beta, then window;
    an empty list keeps the base value, pdsim.cpp:537-539)."""
    out = []
    for a in alphas or [base.alpha]:
        for b in betas or [base.beta]:
            for w in windows or [base.window]:
                p = abi.SchedParams()
                C.memmove(C.byref(p), C.byref(base), C.sizeof(p))
                p.alpha, p.beta, p.window = float(a), float(b), int(w)
                out.append(p)
    return out


def sweep_csv(rates, settings, reports):
    """sweep.csv text; reports[k * len(rates) + r] is setting k at rate r."""
    f = native.format_double
    rows = [CSV_HEADER]
    for r, rate in enumerate(rates):
        for k, s in enumerate(settings):
            rep = reports[k * len(rates) + r]
            vals = [f(rate), f(s.alpha), f(s.beta), str(s.window)]
            vals += [f(v) for v in (rep.slo_attainment, rep.ttft_attainment, rep.itl_attainment,
                                    rep.ttft_initial.mean, rep.ttft_initial.p95, rep.ttft_incremental.mean,
                                    rep.ttft_incremental.p95, rep.itl.mean, rep.itl.p95, rep.e2e_mean,
                                    rep.local_fraction)]
            rows.append(",".join(vals) + "\n")
    return "".join(rows)


def run_sweep(ctx, preset, sessions, rates, plan, profile, base, seed, alphas=None, betas=None, windows=None):
    """The whole `pdsim sweep` (minus the per-combination experiment
    directories): returns (csv_text, settings, SearchResult)."""
    stats = native.preset_stats(preset)
    bufs = [native.gen_trace(stats, r, sessions, seed) for r in rates]
    settings = grid(base, alphas, betas, windows)
    res = ctx.sweep([b.view for b in bufs], plan, profile, settings, seed, report=True)
    return sweep_csv(rates, settings, res.reports), settings, res
