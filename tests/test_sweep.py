"""`pdsim sweep` as one batched GPU call (reference
tools/pdsim.cpp:501-590): the per-(rate, setting) Reports equal the
reference's build_report of run() on the same trace/plan/params/seed, and the
sweep.csv text equals the reference's formatting of those reports.

CPU tests: the std::to_chars formatter, the reference's grid order and the
CSV assembly. GPU tests: report parity, error behaviour, staged re-runs.
"""
import random
import struct

import pytest

from paper_2602_14516_b200 import abi, native, sweep
from tests import parity


def test_format_double_matches_to_chars():
    rng = random.Random(3)
    vals = [0.0, 1.0, 0.1, 1e-5, 123456789.0, 1e22, 1e21, 5e-324, 0.85, 0.9, 2.5e-3, 1.0 / 3.0, 100000.0]
    vals += [struct.unpack("<d", struct.pack("<Q", rng.getrandbits(63) & ~(0x7ff << 52) | (rng.randrange(900, 1150) << 52)))[0]
             for _ in range(3000)]
    vals += [rng.uniform(0, 50) for _ in range(2000)] + [float(rng.randrange(10 ** 7)) for _ in range(500)]
    for v in vals:
        assert native.format_double(v) == parity.to_chars(v), v


def test_grid_follows_reference_loop_order():
    base = abi.default_params(stat_window=7.0)
    g = sweep.grid(base, [0.5, 0.9], [0.85, 2.0], [1, 3, 8])
    assert [(p.alpha, p.beta, p.window) for p in g] == [(a, b, w) for a in (0.5, 0.9) for b in (0.85, 2.0)
                                                         for w in (1, 3, 8)]
    assert all(p.stat_window == 7.0 and p.routing == base.routing and p.reorder == base.reorder for p in g)
    one = sweep.grid(base)  # empty lists keep the base knobs (pdsim.cpp:537-539)
    assert [(p.alpha, p.beta, p.window) for p in one] == [(base.alpha, base.beta, base.window)]


def fake_report(k):
    r = abi.Report()
    r.slo_attainment, r.ttft_attainment, r.itl_attainment = 1.0 / (k + 3), 0.5, 1.0
    r.ttft_initial.mean, r.ttft_initial.p95 = 0.1 * k, 0.25
    r.ttft_incremental.mean, r.ttft_incremental.p95 = 1e-5 * k, 3e-4
    r.itl.mean, r.itl.p95 = 0.012345, 0.02
    r.e2e_mean, r.local_fraction = 123.5 + k, 0.0
    return r


def reference_csv(rates, settings, reports):
    """The reference's sweep.csv assembly (pdsim.cpp:541-586) with the
    checker's own to_chars."""
    f = parity.to_chars
    text = sweep.CSV_HEADER
    for r, rate in enumerate(rates):
        for k, s in enumerate(settings):
            rep = reports[k * len(rates) + r]
            text += ",".join([f(rate), f(s.alpha), f(s.beta), str(s.window), f(rep.slo_attainment),
                              f(rep.ttft_attainment), f(rep.itl_attainment), f(rep.ttft_initial.mean),
                              f(rep.ttft_initial.p95), f(rep.ttft_incremental.mean), f(rep.ttft_incremental.p95),
                              f(rep.itl.mean), f(rep.itl.p95), f(rep.e2e_mean), f(rep.local_fraction)]) + "\n"
    return text


def test_sweep_csv_assembly():
    rates = [2.0, 8.5, 16.0]
    settings = sweep.grid(abi.default_params(), [0.5, 0.9], [0.85], [1, 3])
    reports = [fake_report(k) for k in range(len(rates) * len(settings))]
    assert sweep.sweep_csv(rates, settings, reports) == reference_csv(rates, settings, reports)


# ---- GPU ---------------------------------------------------------------------

@pytest.mark.gpu
def test_sweep_reports_match_reference(ctx):
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    prof = native.synth_profile(native.default_synth_spec(), 7)
    plan = abi.make_plan({1: 2}, {1: 2})
    rates, seed = [4.0, 16.0, 40.0], 9
    base = abi.default_params()
    csv, settings, res = sweep.run_sweep(ctx, "toolbench", 300, rates, plan, prof, base, seed,
                                         alphas=[0.5, 0.9, 1.0], betas=[0.85, 0.3], windows=[1, 3, 8])
    stats = native.preset_stats("toolbench")
    trs = [native.gen_trace(stats, r, 300, seed) for r in rates]
    want = []
    for k, s in enumerate(settings):
        for r, tr in enumerate(trs):
            rep = refbind.report(tr.view, plan, prof, s, seed)
            assert res.reports[k * len(rates) + r].as_tuple() == rep.as_tuple(), (k, r)
            want.append(rep)
    assert csv == reference_csv(rates, settings, want)
    # the settings stay staged: a resident re-run gives the same counts
    again = ctx.search_staged(seed, report=True)
    assert [x.as_tuple() for x in again.reports] == [x.as_tuple() for x in res.reports]
    assert again.best_candidate == res.best_candidate


@pytest.mark.gpu
def test_sweep_mixed_routing_and_windows(ctx):
    """Settings that differ in more than the swept knobs (routing, reorder,
    statistics window) in one launch."""
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    prof = native.synth_profile(native.default_synth_spec(), 7)
    plan = abi.make_plan({2: 1, 1: 1}, {1: 1, 2: 1})
    trs = [native.gen_trace(native.preset_stats("hotpotqa"), 12.0, 200, s) for s in (1, 2)]
    settings = [abi.default_params(), abi.default_params(routing=abi.ROUTING_ALWAYS_REMOTE),
                abi.default_params(routing=abi.ROUTING_ALWAYS_LOCAL), abi.default_params(reorder=0),
                abi.default_params(window=5, stat_window=1.5), abi.default_params(stat_window=30.0)]
    res = ctx.sweep([t.view for t in trs], plan, prof, settings, 4)
    for k, s in enumerate(settings):
        for r, tr in enumerate(trs):
            assert res.reports[k * len(trs) + r].as_tuple() == refbind.report(tr.view, plan, prof, s, 4).as_tuple()


@pytest.mark.gpu
def test_sweep_rejects_bad_setting(ctx):
    prof = native.synth_profile(native.default_synth_spec(), 7)
    plan = abi.make_plan({1: 1}, {1: 1})
    tr = native.gen_trace(native.preset_stats("toolbench"), 4.0, 50, 1)
    with pytest.raises(native.ConfigError):  # reorder window > 8 (reorder.cpp:86-90)
        ctx.sweep([tr.view], plan, prof, [abi.default_params(), abi.default_params(window=9)], 1)
    with pytest.raises(native.ConfigError):  # SchedulerParams::validate (sim_engine.cpp:653-666)
        ctx.sweep([tr.view], plan, prof, [abi.default_params(alpha=-1.0)], 1)


@pytest.mark.gpu
def test_sweep_precheck_failure_is_config_error(ctx):
    """A trace whose first round cannot fit any decode worker makes the
    reference's run() throw inside the sweep loop (sim_engine.cpp:217-231,
    pdsim.cpp:567-570): the batched sweep raises the same ConfigError text,
    naming the first offending session of the first failing trace."""
    import numpy as np
    from oracle import refbind
    prof = native.synth_profile(native.default_synth_spec(), 7)
    plan = abi.make_plan({1: 1}, {1: 1})
    trs = [native.gen_trace(native.preset_stats("toolbench"), 4.0, 200, s) for s in (1, 2)]

    def first_rounds(v):
        off = np.ctypeslib.as_array(v.round_offset, shape=(v.n_sessions + 1,))
        return np.ctypeslib.as_array(v.incr_input_len, shape=(v.n_rounds,))[off[:-1]]

    m0, m1 = int(first_rounds(trs[0].view).max()), int(first_rounds(trs[1].view).max())
    assert m0 != m1
    lo, hi = sorted((m0, m1))
    prof.gpu_memory_capacity = (lo + hi) // 2 * prof.kv_bytes_per_token  # degree 1: one worker's capacity
    bad = 0 if m0 > m1 else 1
    settings = [abi.default_params(), abi.default_params(alpha=0.5)]
    with pytest.raises(native.ConfigError) as ei:
        ctx.sweep([t.view for t in trs], plan, prof, settings, 1)
    if refbind.available():
        with pytest.raises(refbind.RefError) as er:
            refbind.run(trs[bad].view, plan, prof, settings[0], 1)
        assert str(er.value).split("] ", 1)[1] in str(ei.value)
    sid = np.ctypeslib.as_array(trs[bad].view.session_id, shape=(trs[bad].view.n_sessions,))
    first = int(np.argmax(first_rounds(trs[bad].view) * prof.kv_bytes_per_token > prof.gpu_memory_capacity))
    assert f"session {int(sid[first])} first-round KV" in str(ei.value)
    # nothing stays staged after the failure
    ctx._staged = (len(trs), len(settings))
    with pytest.raises(native.ConfigError):
        ctx.search_staged(1)


@pytest.mark.gpu
def test_report_on_10k_session_trace(ctx):
    """Report mode on a trace with ~2M decode tokens: the ITL-gap histogram is
    sized from the staged traces (2x the decode tokens), so a long replay
    never overflows it, and every report equals the reference's."""
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    from paper_2602_14516_b200 import workloads
    prof = workloads.model_profile("llama3-8b")
    tr = native.gen_trace(native.preset_stats("toolbench"), 16.0, 10000, 5)
    plans = [abi.make_plan({4: 1}, {4: 1}), abi.make_plan({1: 2}, {2: 3})]
    res = ctx.plan_search([tr.view], plans, prof, abi.default_params(), 1, report=True)
    for c, plan in enumerate(plans):
        assert res.reports[c].as_tuple() == refbind.report(tr.view, plan, prof, abi.default_params(), 1).as_tuple(), c
