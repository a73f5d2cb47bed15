"""Randomised batched searches against the unmodified reference: random cost
models, presets, rates, plan subsets and scheduler settings (routing mode,
reorder, window, statistics window, alpha, beta). Per-pair attainment and
status equal the reference's; the argmax search mode picks the same plan."""
import random

import pytest

from paper_2602_14516_b200 import abi, native
from tests import parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("build", [abi.BUILD_AUTO, abi.BUILD_THROUGHPUT])
@pytest.mark.parametrize("seed", range(24))
def test_random_search_matches_reference(ctx, seed, build):
    """Both kernel builds (the same engine source; THROUGHPUT keeps shared hot
    subroutines out of line) against the reference."""
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    rng = random.Random(1000 + seed)
    spec = native.default_synth_spec()
    prof = native.synth_profile(spec, rng.randrange(1, 10_000))
    preset = rng.choice(["toolbench", "gaia", "hotpotqa", "dureader"])
    trs = [native.gen_trace(native.preset_stats(preset), rng.choice([2.0, 8.0, 20.0, 45.0]),
                            rng.choice([150, 300]), rng.randrange(1 << 30)) for _ in range(rng.choice([1, 2, 3]))]
    views = [t.view for t in trs]
    allp = native.enumerate_plans([1, 2, 4, 8], 8)
    plans = [allp[k] for k in sorted(rng.sample(range(len(allp)), 24))]
    prm = abi.default_params(routing=rng.choice([0, 0, 1, 2]), reorder=rng.choice([0, 1, 1]),
                             window=rng.randint(1, 8), stat_window=rng.choice([0.5, 3.0, 10.0]),
                             alpha=rng.choice([0.5, 0.9, 1.0]), beta=rng.choice([0.3, 0.85, 1.0]))
    es = rng.randrange(1 << 62)
    ctx.set_kernel_build(build)
    try:
        res = ctx.plan_search(views, plans, prof, prm, es)
        assert ctx.last_kernel_build() == (abi.BUILD_THROUGHPUT if build == abi.BUILD_THROUGHPUT else abi.BUILD_LATENCY)
        ctx.set_search_mode(abi.SEARCH_ARGMAX)
        pr = ctx.plan_search(views, plans, prof, prm, es)
    finally:
        ctx.set_search_mode(abi.SEARCH_FULL)
        ctx.set_kernel_build(abi.BUILD_AUTO)
    att, st_ref, _ = refbind.plan_search(views, plans, prof, prm, es)
    for p in range(res.n_pairs):
        assert res.pair_status[p] == st_ref[p], p
        if st_ref[p] == 0:
            for f in parity.ATT_FIELDS:
                assert getattr(res.pair_attainment[p], f) == getattr(att[p], f), (p, f)
    assert (pr.best_candidate, pr.best_slo_ok) == (res.best_candidate, res.best_slo_ok)


def test_auto_build_switches_to_throughput_for_many_pairs(ctx):
    """AUTO launches the throughput build once a search replays more than 8
    pairs per SM; both builds return identical per-pair results there."""
    prof = native.synth_profile(native.default_synth_spec(), 3)
    trs = [native.gen_trace(native.preset_stats("toolbench"), 8.0, 40, 50 + k) for k in range(8)]
    views = [t.view for t in trs]
    plans = native.enumerate_plans([1, 2, 4, 8], 8)  # 169 x 8 = 1352 pairs > 8 x 148
    prm = abi.default_params()
    auto = ctx.plan_search(views, plans, prof, prm, 9)
    assert ctx.last_kernel_build() == abi.BUILD_THROUGHPUT
    ctx.set_kernel_build(abi.BUILD_LATENCY)
    try:
        lat = ctx.plan_search(views, plans, prof, prm, 9)
        assert ctx.last_kernel_build() == abi.BUILD_LATENCY
    finally:
        ctx.set_kernel_build(abi.BUILD_AUTO)
    assert auto.n_pairs == lat.n_pairs == 1352
    for p in range(auto.n_pairs):
        assert auto.pair_status[p] == lat.pair_status[p], p
        for f in parity.ATT_FIELDS:
            assert getattr(auto.pair_attainment[p], f) == getattr(lat.pair_attainment[p], f), (p, f)
    assert (auto.best_candidate, auto.best_slo_ok) == (lat.best_candidate, lat.best_slo_ok)


@pytest.mark.parametrize("build", [abi.BUILD_LATENCY, abi.BUILD_THROUGHPUT])
def test_candidate_affine_queues_equal_the_plain_queue(ctx, monkeypatch, build):
    """The per-SM candidate-affine queues (default with the throughput build)
    replay every pair exactly once: per-pair results, event counts and the
    argmax equal the plain atomic queue, for a whole search and for an LPT
    shard list (outputs follow the list)."""
    prof = native.synth_profile(native.default_synth_spec(), 5)
    trs = [native.gen_trace(native.preset_stats("hotpotqa"), 6.0, 60, 70 + k) for k in range(6)]
    views = [t.view for t in trs]
    plans = native.enumerate_plans([1, 2, 4, 8], 8)
    ctx.set_kernel_build(build)
    try:
        ctx.stage(views, plans, prof, abi.default_params())
        shard = native.shard_pairs(views, plans, 2, 1)
        got = {}
        for aff in ("0", "1"):
            monkeypatch.setenv("PDSIM_SM_AFFINITY", aff)
            got[aff] = (ctx.search_staged(3), ctx.search_staged_list(3, shard))
    finally:
        ctx.set_kernel_build(abi.BUILD_AUTO)
    for k in range(2):
        a, b = got["0"][k], got["1"][k]
        assert a.n_pairs == b.n_pairs > 0
        for p in range(a.n_pairs):
            assert a.pair_status[p] == b.pair_status[p], p
            assert a.pair_events[p] == b.pair_events[p], p
            for f in parity.ATT_FIELDS:
                assert getattr(a.pair_attainment[p], f) == getattr(b.pair_attainment[p], f), (p, f)
        assert (a.best_candidate, a.best_slo_ok) == (b.best_candidate, b.best_slo_ok)


@pytest.mark.parametrize("mode", [abi.SEARCH_FULL, abi.SEARCH_ARGMAX])
def test_affine_round_robin_groups_equal_the_plain_queue(ctx, monkeypatch, mode):
    """More pairs than resident warps (2 slots per SM): contiguous lists and
    round-robin groups replay every pair once; full-mode per-pair results and
    the argmax (both modes) equal the plain atomic queue."""
    prof = native.synth_profile(native.default_synth_spec(), 6)
    trs = [native.gen_trace(native.preset_stats("toolbench"), 10.0, 50, 90 + k) for k in range(4)]
    views = [t.view for t in trs]
    plans = native.enumerate_plans([1, 2, 4, 8], 8)  # 676 pairs > 2 x 148 slots
    monkeypatch.setenv("PDSIM_SLOTS_PER_SM", "2")
    ctx.set_kernel_build(abi.BUILD_THROUGHPUT)
    ctx.set_search_mode(mode)
    got = {}
    try:
        ctx.stage(views, plans, prof, abi.default_params())
        for name, env in (("plain", {"PDSIM_SM_AFFINITY": "0"}),
                          ("contiguous", {"PDSIM_SM_AFFINITY": "1", "PDSIM_SM_GROUP": "0"}),
                          ("round_robin", {"PDSIM_SM_AFFINITY": "1", "PDSIM_SM_GROUP": "1"})):
            for k, v in env.items():
                monkeypatch.setenv(k, v)
            got[name] = ctx.search_staged(4)
    finally:
        ctx.set_search_mode(abi.SEARCH_FULL)
        ctx.set_kernel_build(abi.BUILD_AUTO)
    a = got["plain"]
    for name in ("contiguous", "round_robin"):
        b = got[name]
        assert (a.best_candidate, a.best_slo_ok) == (b.best_candidate, b.best_slo_ok), name
        if mode == abi.SEARCH_FULL:
            for p in range(a.n_pairs):
                assert a.pair_status[p] == b.pair_status[p], (name, p)
                assert a.pair_events[p] == b.pair_events[p], (name, p)
