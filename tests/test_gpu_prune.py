"""Search mode ARGMAX (exact pruning): the selected plan and
its count equal the full search's on every workload; a pruned candidate is
provably dominated by the winner (its full count is below the winner's, or
equal with a larger index); unpruned candidates keep their exact counts;
sharded runs combine to the same argmax."""
import pytest

from paper_2602_14516_b200 import abi, native, workloads

pytestmark = pytest.mark.gpu


def both_modes(ctx, traces, plans, prof, prm, seed, b=0, e=-1):
    ctx.set_search_mode(abi.SEARCH_FULL)
    full = ctx.plan_search(traces, plans, prof, prm, seed, b, e)
    ctx.set_search_mode(abi.SEARCH_ARGMAX)
    try:
        pr = ctx.plan_search(traces, plans, prof, prm, seed, b, e)
    finally:
        ctx.set_search_mode(abi.SEARCH_FULL)
    return full, pr


def check(full, pr, n_cand):
    assert pr.best_candidate == full.best_candidate
    assert pr.best_slo_ok == full.best_slo_ok
    best = full.best_candidate
    for c in range(n_cand):
        g, f = pr.candidate_slo_ok[c], full.candidate_slo_ok[c]
        if g == -2:
            assert f == -1 or f < full.best_slo_ok or (f == full.best_slo_ok and c > best), c
        else:
            assert g == f, c
    return sum(1 for c in range(n_cand) if pr.candidate_slo_ok[c] == -2)


WORKLOADS = [
    ("toolbench", 4.0, 300, 1),    # light: many candidates at full attainment
    ("hotpotqa", 14.0, 300, 2),    # loaded
    ("gaia", 40.0, 200, 3),        # saturated: most sessions miss TTFT
    ("dureader", 20.0, 250, 4),
]


@pytest.mark.parametrize("preset,rate,sessions,reps", WORKLOADS)
def test_argmax_mode_matches_full(ctx, preset, rate, sessions, reps):
    prof = workloads.model_profile("llama3-8b")
    trs = [native.gen_trace(native.preset_stats(preset), rate, sessions, 10 + s) for s in range(reps)]
    plans = native.enumerate_plans([1, 2, 4], 8)
    full, pr = both_modes(ctx, [t.view for t in trs], plans, prof, abi.default_params(), 7)
    check(full, pr, len(plans))


def test_argmax_mode_with_invalid_candidates(ctx):
    """Candidates whose KV precheck fails stay invalid (-1) and never become
    the incumbent."""
    spec = native.default_synth_spec()
    spec.gpu_memory_capacity = 200_000_000  # small KV: degree-1 decode workers cannot hold long first rounds
    prof = native.synth_profile(spec, 7)
    trs = [native.gen_trace(native.preset_stats("hotpotqa"), 6.0, 200, s) for s in (1, 2)]
    plans = native.enumerate_plans([1, 2, 4], 8)
    full, pr = both_modes(ctx, [t.view for t in trs], plans, prof, abi.default_params(), 3)
    check(full, pr, len(plans))


def test_argmax_mode_prunes_on_c2_small(ctx):
    wl = workloads.c2_small()
    full, pr = both_modes(ctx, wl.traces, wl.plans, wl.profile, wl.params, wl.seed)
    assert check(full, pr, len(wl.plans)) > 0  # C2-like: later all-attaining candidates are pruned


def test_argmax_mode_sharded(ctx):
    """Shards pruned independently, combined like the multi-GPU reduction
    (sum counts; any negative excludes the candidate), give the full argmax."""
    prof = workloads.model_profile("llama3-8b")
    trs = [native.gen_trace(native.preset_stats("toolbench"), 8.0, 200, s) for s in range(4)]
    plans = native.enumerate_plans([1, 2, 4], 8)
    views = [t.view for t in trs]
    ctx.set_search_mode(abi.SEARCH_FULL)
    full = ctx.plan_search(views, plans, prof, abi.default_params(), 5)
    total = len(plans) * len(trs)
    cuts = [0, total // 3, (2 * total) // 3 + 1, total]
    sums, bad = [0] * len(plans), [False] * len(plans)
    ctx.set_search_mode(abi.SEARCH_ARGMAX)
    try:
        for b, e in zip(cuts, cuts[1:]):
            part = ctx.plan_search(views, plans, prof, abi.default_params(), 5, b, e)
            for c in range(len(plans)):
                v = part.candidate_slo_ok[c]
                if v < 0:
                    bad[c] = True
                else:
                    sums[c] += v
    finally:
        ctx.set_search_mode(abi.SEARCH_FULL)
    key = [(sums[c], -c) for c in range(len(plans)) if not bad[c]]
    best = max(key)
    assert (-best[1], best[0]) == (full.best_candidate, full.best_slo_ok)


def test_search_mode_rejects_unknown(ctx):
    with pytest.raises(native.ConfigError):
        ctx.set_search_mode(7)
