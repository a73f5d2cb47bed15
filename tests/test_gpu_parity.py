"""GPU parity: the CUDA replay engine vs the reference simulator on identical
inputs — bit-exact routing decisions, TTFT samples, session verdicts,
counters and attainment (north star: "bit-exact per-request routing
decisions, SLO-attainment counts and selected plan")."""
import pytest

from paper_2602_14516_b200 import abi, native
from tests import parity

pytestmark = pytest.mark.gpu

PLANS = {
    "P2xD2": ({1: 2}, {1: 2}),
    "mixed": ({2: 1, 4: 1}, {1: 1, 2: 1}),
    "decode-only": ({}, {1: 3}),
    "P1xD1": ({1: 1}, {1: 1}),
}
PARAMS = {
    "default": dict(),
    "always-remote": dict(routing=abi.ROUTING_ALWAYS_REMOTE),
    "always-local": dict(routing=abi.ROUTING_ALWAYS_LOCAL),
    "fifo": dict(reorder=0),
    "w5-short-window": dict(window=5, stat_window=1.5),
    "w8": dict(window=8, stat_window=2.0),
}


@pytest.fixture(scope="module")
def prof7():
    return native.synth_profile(native.default_synth_spec(), 7)


@pytest.mark.parametrize("preset", ["toolbench", "gaia", "hotpotqa", "dureader"])
@pytest.mark.parametrize("rate", [2.0, 12.0, 40.0])
@pytest.mark.parametrize("plan", list(PLANS))
def test_run_matches_oracle(ctx, prof7, preset, rate, plan):
    tr = native.gen_trace(native.preset_stats(preset), rate, 250, 11)
    p = abi.make_plan(*PLANS[plan])
    for name, kw in PARAMS.items():
        prm = abi.default_params(**kw)
        got = ctx.run(tr.view, p, prof7, prm, 3)
        want = parity.oracle_run(tr.view, p, prof7, prm, 3)
        errs = parity.diff_runs(got, want)
        assert not errs, f"{preset} rate={rate} plan={plan} params={name}: " + "; ".join(errs[:5])


def test_acceptance_saturating_scenario(ctx):
    """The reference acceptance scenario (acceptance_test.cpp:125-172): dureader
    4000 sessions @16/s seed 101, P:2x1,D:2x1, engine seed 2, w=4, stat window
    1.5 s, decode-heavy profile seed 42."""
    spec = native.default_synth_spec()
    spec.n_degrees = 1
    spec.degrees[0] = 1
    spec.decode_alpha_min, spec.decode_alpha_max = 0.01056, 0.01144
    spec.decode_beta_min, spec.decode_beta_max = 1.14e-4, 1.26e-4
    prof = native.synth_profile(spec, 42)
    tr = native.gen_trace(native.preset_stats("dureader"), 16.0, 4000, 101)
    plan = abi.make_plan({1: 2}, {1: 2})
    for routing in (abi.ROUTING_ADAPTIVE, abi.ROUTING_ALWAYS_REMOTE, abi.ROUTING_ALWAYS_LOCAL):
        for reorder in (0, 1):
            prm = abi.default_params(routing=routing, reorder=reorder, window=4, stat_window=1.5)
            got = ctx.run(tr.view, plan, prof, prm, 2)
            want = parity.oracle_run(tr.view, plan, prof, prm, 2)
            parity.assert_same_run(got, want)


def test_survey_fingerprint_scenario(ctx):
    """SURVEY.md §8(c) fingerprint inputs: dureader 4000 @16 seed 101,
    P:2x1,D:2x1, profile seed 7, engine seed 2, default params."""
    prof = native.synth_profile(native.default_synth_spec(), 7)
    tr = native.gen_trace(native.preset_stats("dureader"), 16.0, 4000, 101)
    plan = abi.make_plan({1: 2}, {1: 2})
    prm = abi.default_params()
    got = ctx.run(tr.view, plan, prof, prm, 2)
    parity.assert_same_run(got, parity.oracle_run(tr.view, plan, prof, prm, 2))


def test_plan_search_matches_reference_pool(ctx):
    """Batched search over all 169 N=8 candidates x 3 replicas: per-pair
    attainment, per-candidate sums and the argmax equal the reference's."""
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    prof = native.synth_profile(native.default_synth_spec(), 7)
    st = native.preset_stats("toolbench")
    trs = [native.gen_trace(st, 10.0, 400, s) for s in (1, 2, 3)]
    views = [t.view for t in trs]
    plans = native.enumerate_plans([1, 2, 4, 8], 8)
    prm = abi.default_params()
    res = ctx.plan_search(views, plans, prof, prm, 1)
    att, st_ref, _ = refbind.plan_search(views, plans, prof, prm, 1)
    n = len(views) * len(plans)
    sums = [0] * len(plans)
    for p in range(n):
        assert res.pair_status[p] == st_ref[p]
        for f in parity.ATT_FIELDS:
            assert getattr(res.pair_attainment[p], f) == getattr(att[p], f), (p, f)
        sums[p // len(views)] += att[p].slo_ok if st_ref[p] == 0 else 0
    assert [res.candidate_slo_ok[c] for c in range(len(plans))] == sums
    best = max(range(len(plans)), key=lambda c: (sums[c], -c))
    assert res.best_candidate == best
    assert res.best_slo_ok == sums[best]


def test_c2_headline_search_matches_reference(ctx):
    """The bench headline workload itself (C2: 169 N=8 plans, toolbench 10 000
    sessions @16/s): per-pair attainment, per-candidate sums and the argmax
    equal the unmodified reference's."""
    from oracle import refbind
    from paper_2602_14516_b200 import workloads
    if not refbind.available():
        pytest.skip("reference library not built")
    wl = workloads.c2()
    res = ctx.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed)
    att, st_ref, _ = refbind.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed)
    sums = []
    for p in range(wl.n_pairs):
        assert res.pair_status[p] == st_ref[p]
        for f in parity.ATT_FIELDS:
            assert getattr(res.pair_attainment[p], f) == getattr(att[p], f), (p, f)
        sums.append(att[p].slo_ok if st_ref[p] == 0 else -1)
    assert [res.candidate_slo_ok[c] for c in range(len(wl.plans))] == sums
    assert res.best_candidate == max(range(len(sums)), key=lambda c: (sums[c], -c))


def test_saturated_iterative_rag_pair_matches_reference(ctx):
    """C3's regime (qwen-32b cost model, hotpotqa 8 fixed rounds, overloaded):
    every record of a saturated replay is bit-identical, including the
    per-session mean ITL folds over thousands of concurrent decoders."""
    from paper_2602_14516_b200 import workloads
    prof = workloads.model_profile("qwen-32b")
    tr = native.gen_trace(workloads.trace_stats("hotpotqa-8fixed"), 20.0, 3000, 1)
    for x, y in (({1: 1}, {1: 1}), ({2: 1}, {1: 2, 2: 1})):
        plan = abi.make_plan(x, y)
        prm = abi.default_params()
        got = ctx.run(tr.view, plan, prof, prm, 1)
        parity.assert_same_run(got, parity.oracle_run(tr.view, plan, prof, prm, 1))


def test_run_itl_samples_match_reference(ctx):
    """Drop-in run() with materialised ITL samples: the survey fingerprint
    scenario's itl_samples.csv hash (1.79 M samples) and a mixed-plan run
    sample by sample."""
    from tests import golden_cases
    entry = [e for e in golden_cases.load() if e["case"]["name"] == "survey_fingerprint"][0]
    prof = native.synth_profile(native.default_synth_spec(), 7)
    tr = native.gen_trace(native.preset_stats("dureader"), 16.0, 4000, 101)
    plan = abi.make_plan({1: 2}, {1: 2})
    got = ctx.run(tr.view, plan, prof, abi.default_params(), 2, itl=True)
    assert got.n_itl == entry["itl_samples"]
    assert parity.itl_csv_fnv([parity.itl_tuple(x) for x in got.itl_samples]) == entry["reference_csv_fnv"]["itl"]
    tr2 = native.gen_trace(native.preset_stats("hotpotqa"), 12.0, 300, 5)
    plan2 = abi.make_plan({2: 1, 4: 1}, {1: 1, 2: 1})
    got2 = ctx.run(tr2.view, plan2, prof, abi.default_params(), 3, itl=True)
    want2 = parity.reference_itl(tr2.view, plan2, prof, abi.default_params(), 3)
    assert not parity.diff_itl([parity.itl_tuple(x) for x in got2.itl_samples], want2)


def test_search_reports_match_reference(ctx):
    """Per-pair Report in the batched search: every
    candidate x replica's build_report equals the reference's, and ranking
    candidates by it is exact (here: lowest P95 ITL among max attainment)."""
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    prof = native.synth_profile(native.default_synth_spec(), 7)
    trs = [native.gen_trace(native.preset_stats("hotpotqa"), 14.0, 300, s) for s in (1, 2)]
    plans = native.enumerate_plans([1, 2, 4], 4)
    prm = abi.default_params()
    res = ctx.plan_search([t.view for t in trs], plans, prof, prm, 1, report=True)
    for p in range(res.n_pairs):
        c, r = divmod(p, len(trs))
        want = refbind.report(trs[r].view, plans[c], prof, prm, 1)
        assert res.reports[p].as_tuple() == want.as_tuple(), (c, r)
    # attainment-only search is unchanged by report mode
    plain = ctx.plan_search([t.view for t in trs], plans, prof, prm, 1)
    assert [plain.candidate_slo_ok[c] for c in range(len(plans))] == [res.candidate_slo_ok[c] for c in range(len(plans))]
