"""Threading contract: one handle per device, calls on
distinct handles may run concurrently (the reference's run() is reentrant,
SPEC.md:381). Two contexts on the same GPU driven from two host threads give
the same results as sequential calls; a context's errors stay its own."""
import threading

import pytest

from paper_2602_14516_b200 import abi, native, workloads

pytestmark = pytest.mark.gpu


def _job(k):
    prof = workloads.model_profile("llama3-8b")
    trs = [native.gen_trace(native.preset_stats(("toolbench", "hotpotqa")[k % 2]), 8.0 + 4 * k, 300, 10 + k)]
    plans = native.enumerate_plans([1, 2, 4], 8)
    return trs, plans, prof


def _signature(res, n_cand):
    return (res.best_candidate, res.best_slo_ok, [res.candidate_slo_ok[c] for c in range(n_cand)],
            [res.pair_attainment[p].slo_ok for p in range(res.n_pairs)])


def test_two_contexts_two_threads_match_sequential(ctx):
    jobs = [_job(k) for k in range(2)]
    seq = []
    for trs, plans, prof in jobs:
        seq.append(_signature(ctx.plan_search([t.view for t in trs], plans, prof, abi.default_params(), 3),
                              len(plans)))
    out = [None, None]
    errs = []

    def worker(k):
        try:
            trs, plans, prof = jobs[k]
            with native.Context(0) as c:
                for _ in range(3):
                    r = c.plan_search([t.view for t in trs], plans, prof, abi.default_params(), 3)
                    sig = _signature(r, len(plans))
                    assert out[k] is None or out[k] == sig
                    out[k] = sig
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert out == seq


def test_errors_stay_on_their_context(ctx):
    with native.Context(0) as a, native.Context(0) as b:
        prof = workloads.model_profile("llama3-8b")
        tr = native.gen_trace(native.preset_stats("toolbench"), 4.0, 50, 1)
        with pytest.raises(native.ConfigError):
            a.plan_search([tr.view], [abi.make_plan({1: 1}, {1: 1})], prof, abi.default_params(alpha=-1.0), 1)
        r = b.plan_search([tr.view], [abi.make_plan({1: 1}, {1: 1})], prof, abi.default_params(), 1)
        assert r.best_candidate == 0


def _cost_model_job(model, k):
    prof = workloads.model_profile(model)
    trs = [native.gen_trace(native.preset_stats("toolbench"), 6.0 + 2 * k, 300, 20 + k)]
    plans = native.enumerate_plans([1, 2, 4], 8)
    return trs, plans, prof


def test_contexts_with_different_cost_models(ctx):
    """The cost model sits in a per-module __constant__ bank shared by every
    context on the device (engine.cuh c_profile). Contexts holding different
    profiles must never replay with each other's: concurrently from two
    threads, and in the sequence stage(A), stage(B), search_staged(A)."""
    jobs = [_cost_model_job("llama3-8b", 0), _cost_model_job("qwen-32b", 1)]
    seq = [_signature(ctx.plan_search([t.view for t in trs], plans, prof, abi.default_params(), 3), len(plans))
           for trs, plans, prof in jobs]
    assert seq[0] != seq[1]
    with native.Context(0) as a, native.Context(0) as b:
        (ta, pa, fa), (tb, pb, fb) = jobs
        a.stage([t.view for t in ta], pa, fa, abi.default_params())
        b.stage([t.view for t in tb], pb, fb, abi.default_params())
        assert _signature(a.search_staged(3), len(pa)) == seq[0]
        assert _signature(b.search_staged(3), len(pb)) == seq[1]
        assert _signature(a.search_staged(3), len(pa)) == seq[0]
    out, errs = [[], []], []

    def worker(k):
        try:
            trs, plans, prof = jobs[k]
            with native.Context(0) as c:
                for _ in range(4):
                    out[k].append(_signature(c.plan_search([t.view for t in trs], plans, prof,
                                                           abi.default_params(), 3), len(plans)))
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert all(s == seq[0] for s in out[0]) and all(s == seq[1] for s in out[1])
