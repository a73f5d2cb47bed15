"""Surrogate planner: the GPU phase simulations, the
batched coefficient estimation and the host assignment solver against the
unmodified reference (oracle/_ref: proj/src/planner.cpp:75-657).

Bars: P95 coefficients bit-exact (fp64 equality), sample counts and
infeasibility flags exact, error behaviour identical (the status a result
carries is the exception class the reference threw), solved plans and top-k
rankings identical.
"""
import random

import pytest

from oracle import refbind
from paper_2602_14516_b200 import abi, native, workloads
from tests import parity

pytestmark = pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")

PRESETS = ("toolbench", "gaia", "hotpotqa", "dureader")


def random_coefficients(rng, degrees):
    tau_pre, tau_dec, inf_pre, inf_dec = {}, {}, set(), set()
    pool = [rng.choice([0.05, 0.1, 0.2, 0.4, 0.8]) for _ in range(3)]  # repeated values exercise Z ties
    for d in degrees:
        if rng.random() < 0.15:
            inf_pre.add(d)
        else:
            tau_pre[d] = rng.choice(pool) if rng.random() < 0.5 else rng.uniform(0.01, 1.0)
        if rng.random() < 0.15:
            inf_dec.add(d)
        else:
            tau_dec[d] = rng.choice(pool) if rng.random() < 0.5 else rng.uniform(0.001, 0.2)
    return abi.make_coefficients(tau_pre, tau_dec, inf_pre, inf_dec)


def same_plan_list(a, b):
    assert len(a) == len(b)
    for (pa, za, ga), (pb, zb, gb) in zip(a, b):
        assert abi.plan_dict(pa) == abi.plan_dict(pb)
        assert za == zb and ga == gb


def test_solve_matches_reference_on_random_coefficients():
    rng = random.Random(11)
    for trial in range(400):
        degrees = sorted(rng.sample([1, 2, 3, 4, 6, 8], rng.randint(1, 5)))
        c = random_coefficients(rng, degrees)
        total = rng.randint(1, 20)
        got, want = native.solve(c, total), refbind.solve(c, total)
        assert (got is None) == (want is None), trial
        if got is not None:
            assert abi.plan_dict(got[0]) == abi.plan_dict(want[0]), trial
            assert got[1:] == want[1:], trial


def test_top_k_matches_reference_on_random_coefficients():
    rng = random.Random(12)
    for trial in range(120):
        degrees = sorted(rng.sample([1, 2, 4, 8], rng.randint(1, 4)))
        c = random_coefficients(rng, degrees)
        total = rng.randint(1, 12)
        same_plan_list(native.top_k(c, total, 25), refbind.top_k(c, total, 25))


def test_top_k_rank_one_is_solve():
    """planner.hpp:101-102: rank 1 equals solve's output."""
    c = abi.make_coefficients({1: 0.2, 2: 0.1, 4: 0.05, 8: 0.05}, {1: 0.03, 2: 0.02, 4: 0.02, 8: 0.01})
    best = native.top_k(c, 8, 1)[0]
    plan, z, g = native.solve(c, 8)
    assert abi.plan_dict(best[0]) == abi.plan_dict(plan) and best[1:] == (z, g)


def test_solver_errors_match_reference():
    bad = abi.make_coefficients({1: -1.0}, {1: 0.1})
    with pytest.raises(native.ConfigError):
        native.solve(bad, 4)
    with pytest.raises(refbind.RefError):
        refbind.solve(bad, 4)
    ok = abi.make_coefficients({1: 0.1}, {1: 0.1})
    with pytest.raises(native.ConfigError):
        native.solve(ok, 0)
    with pytest.raises(native.ConfigError):
        native.top_k(ok, 4, 0)
    # infeasible: no single replica pair fits
    assert native.solve(abi.make_coefficients({8: 0.1}, {8: 0.1}), 8) is None
    assert refbind.solve(abi.make_coefficients({8: 0.1}, {8: 0.1}), 8) is None


def test_reference_estimate_coefficients_is_deterministic():
    """The oracle path itself (planner.cpp:228-283): same seed, same table."""
    prof = workloads.model_profile("llama3-8b")
    st = native.preset_stats("toolbench")
    a, rc = refbind.estimate_coefficients(st, 16.0, prof, [1, 2, 4, 8], 8, 3)
    b, rc2 = refbind.estimate_coefficients(st, 16.0, prof, [1, 2, 4, 8], 8, 3)
    assert rc == rc2 == 0 and a.as_dict() == b.as_dict()


# ---- GPU: phase simulations and batched estimation -------------------------

def same_phase(got, want):
    assert got.status == want.status
    if want.status == 0:
        assert got.p95 == want.p95
        assert got.sample_count == want.sample_count
        assert got.infeasible == want.infeasible


def phase_cases():
    prof = workloads.model_profile("llama3-8b")
    cases = []
    for k, name in enumerate(PRESETS):
        st = native.preset_stats(name)
        for rate in (0.5, 4.0, 32.0):  # light, loaded, overloaded
            for n in (256, 37):
                cases.append((native.gen_trace(st, rate, n, 100 + 7 * k + n), prof))
    return cases


@pytest.mark.gpu
def test_phase_sims_match_reference(ctx):
    cases = phase_cases()
    traces, degrees, keep = [], [], []
    for tr, prof in cases:
        for d in (1, 2, 4, 8):
            traces.append(tr.view)
            degrees.append(d)
            keep.append((tr, prof, d))
    got = ctx.phase_sims(traces, degrees, cases[0][1])
    for (tr, prof, d), (gp, gd) in zip(keep, got):
        wp, wd = refbind.phase_sims(tr.view, prof, d)
        same_phase(gp, wp)
        same_phase(gd, wd)


@pytest.mark.gpu
def test_phase_sim_edge_cases(ctx):
    prof = workloads.model_profile("llama3-8b")
    slo = (5.0, 0.5)
    one = parity.manual_trace([{"id": 0, "arrival": 0.0, "rounds": [[100, 5, 0.2], [50, 7, 0.0]]}], slo)
    # every round decodes one token: no inter-token samples (ConfigError)
    single = parity.manual_trace([{"id": i, "arrival": 0.1 * i, "rounds": [[10, 1, 0.0]]} for i in range(4)], slo)
    # equal arrivals: span 0 (infeasible in both phases), ties in the sort
    tied = parity.manual_trace([{"id": i, "arrival": 1.0, "rounds": [[100 + i, 20, 0.5], [100 + i, 20, 0.0]]}
                                 for i in range(5)], slo)
    # unsorted ids, interleaved round offsets, an idle gap between sessions
    gap = parity.manual_trace([{"id": 9 - i, "arrival": 5.0 * i, "rounds": [[300, 40, 1.0], [20, 3, 0.0]]}
                               for i in range(6)], slo)
    for tr in (one, single, tied, gap):
        got = ctx.phase_sims([tr.view] * 2, [1, 4], prof)
        for d, (gp, gd) in zip((1, 4), got):
            wp, wd = refbind.phase_sims(tr.view, prof, d)
            same_phase(gp, wp)
            same_phase(gd, wd)


@pytest.mark.gpu
def test_phase_sims_unknown_degree_is_domain_error(ctx):
    prof = workloads.model_profile("llama3-8b")
    tr = native.gen_trace(native.preset_stats("toolbench"), 4.0, 16, 1)
    with pytest.raises(native.DomainError):
        ctx.phase_sims([tr.view], [3], prof)


@pytest.mark.gpu
def test_estimate_coefficients_match_reference(ctx):
    prof = workloads.model_profile("llama3-8b")
    for name in PRESETS:
        st = native.preset_stats(name)
        rates, seeds = [1.0, 8.0, 16.0, 64.0], [1, 2, 3, 4]
        got = ctx.estimate_coefficients(st, rates, seeds, prof, [8, 1, 4, 2], 8)
        for (c, status), r, s in zip(got, rates, seeds):
            want, rc = refbind.estimate_coefficients(st, r, prof, [8, 1, 4, 2], 8, s, name)
            assert status == rc, (name, r)
            if rc == 0:
                assert c.as_dict() == want.as_dict(), (name, r)
                got_plan, want_plan = native.solve(c, 8), refbind.solve(want, 8)
                assert (got_plan is None) == (want_plan is None)
                if got_plan:
                    assert abi.plan_dict(got_plan[0]) == abi.plan_dict(want_plan[0])
                    assert got_plan[1:] == want_plan[1:]


@pytest.mark.gpu
def test_estimate_coefficients_bad_rate_is_per_set(ctx):
    prof = workloads.model_profile("llama3-8b")
    st = native.preset_stats("gaia")
    got = ctx.estimate_coefficients(st, [4.0, -1.0], [1, 1], prof, [1, 2], 4)
    assert got[0][1] == 0 and got[1][1] == abi.ERR_CONFIG
    with pytest.raises(native.ConfigError):
        ctx.estimate_coefficients(st, [4.0], [1], prof, [1, 3], 4)  # degree 3 not in the profile
