"""Sharded search on the GPU: pair-list launches, the
in-library NCCL reduction, the one-thread multi-device entry, and ARGMAX
soundness when each shard stages only some replicas.

The GPU box has one B200, so multi-rank layouts run as several contexts on
that device (each context is one "rank"); NCCL communicators are exercised
with world size 1. tests/test_multirank.py covers the N > 1 host logic over
gloo."""
import random

import pytest

from paper_2602_14516_b200 import abi, distributed, native, workloads

pytestmark = pytest.mark.gpu


def _small(model="llama3-8b", rates=(6.0, 14.0), sessions=250):
    prof = workloads.model_profile(model)
    trs = [native.gen_trace(native.preset_stats("toolbench"), r, sessions, 3 + k) for k, r in enumerate(rates)]
    plans = native.enumerate_plans([1, 2, 4], 8)
    return prof, trs, plans


def _pair_sig(res, k):
    a = res.pair_attainment[k]
    return (res.pair_status[k], a.sessions_total, a.sessions_completed, a.slo_ok, a.ttft_ok, a.itl_ok)


def test_pair_list_matches_range(ctx):
    prof, trs, plans = _small()
    views = [t.view for t in trs]
    full = ctx.plan_search(views, plans, prof, abi.default_params(), 2)
    n = full.n_pairs
    ctx.stage(views, plans, prof, abi.default_params())
    pairs = list(range(n))
    random.Random(5).shuffle(pairs)
    sub = pairs[: n // 2]
    res = ctx.search_staged_list(2, sub)
    for k, p in enumerate(sub):
        assert _pair_sig(res, k) == _pair_sig(full, p), p
    nt = len(views)
    want = [0] * len(plans)
    for p in sub:
        want[p // nt] += full.pair_attainment[p].slo_ok
    assert [res.candidate_slo_ok[c] for c in range(len(plans))] == want
    with pytest.raises(native.ConfigError):
        ctx.search_staged_list(2, [0, 0])
    with pytest.raises(native.ConfigError):
        ctx.search_staged_list(2, [n])


def test_shard_lists_cover_the_search_and_recombine(ctx):
    prof, trs, plans = _small()
    views = [t.view for t in trs]
    full = ctx.plan_search(views, plans, prof, abi.default_params(), 2)
    ctx.stage(views, plans, prof, abi.default_params())
    totals = None
    for rank in range(3):
        mine = native.shard_pairs(views, plans, 3, rank)
        r = ctx.search_staged_list(2, mine)
        part = [r.candidate_slo_ok[c] for c in range(len(plans))]
        totals = part if totals is None else [a + b for a, b in zip(totals, part)]
    assert totals == [full.candidate_slo_ok[c] for c in range(len(plans))]
    assert native.argmax_candidates(totals) == full.best_candidate


def test_nccl_communicator_world_one(ctx):
    """The in-library collective path (flags kernel + ncclAllReduce + argmax)
    with one rank leaves every output unchanged."""
    prof, trs, plans = _small()
    views = [t.view for t in trs]
    full = ctx.plan_search(views, plans, prof, abi.default_params(), 2)
    with native.Context(0) as c:
        c.comm_init(1, 0, native.nccl_unique_id())
        c.stage(views, plans, prof, abi.default_params())
        r = c.search_staged_list(2, native.shard_pairs(views, plans, 1, 0))
        assert [r.candidate_slo_ok[k] for k in range(len(plans))] == [full.candidate_slo_ok[k] for k in
                                                                          range(len(plans))]
        assert (r.best_candidate, r.best_slo_ok) == (full.best_candidate, full.best_slo_ok)
        c.set_search_mode(abi.SEARCH_ARGMAX)
        ra = c.search_staged_list(2, native.shard_pairs(views, plans, 1, 0))
        assert (ra.best_candidate, ra.best_slo_ok) == (full.best_candidate, full.best_slo_ok)


def test_multi_plan_search_one_device(ctx):
    prof, trs, plans = _small()
    views = [t.view for t in trs]
    full = ctx.plan_search(views, plans, prof, abi.default_params(), 2)
    for mode in (abi.SEARCH_FULL, abi.SEARCH_ARGMAX):
        m = native.multi_plan_search([0], views, plans, prof, abi.default_params(), 2, mode)
        assert (m.best_candidate, m.best_slo_ok) == (full.best_candidate, full.best_slo_ok)
        if mode == abi.SEARCH_FULL:
            assert [_pair_sig(m, p) for p in range(full.n_pairs)] == [_pair_sig(full, p) for p in range(full.n_pairs)]
            assert [m.candidate_slo_ok[c] for c in range(len(plans))] == [full.candidate_slo_ok[c] for c in
                                                                              range(len(plans))]


def test_argmax_replica_per_rank_uses_global_bound(ctx):
    """Replica-per-rank layout: rank k stages only
    replica k. On replica 0 every strong plan attains 300/300, so the global
    argmax (candidate 155, 439 over both replicas) merely ties there with a
    larger index than candidate 0. With the global session total the ARGMAX
    bounds stay sound: combining the ranks' pruned searches gives the FULL
    answer (the local total would let rank 0 prune candidate 155)."""
    prof, trs, plans = _small("qwen-32b", rates=(1.0, 20.0), sessions=300)
    views = [t.view for t in trs]
    full = ctx.plan_search(views, plans, prof, abi.default_params(), 1)
    assert full.best_candidate == 155 and full.best_slo_ok == 439
    total = sum(int(v.n_sessions) for v in views)
    per_rank = []
    for k in range(2):
        with native.Context(0) as c:
            c.stage([views[k]], plans, prof, abi.default_params())
            c.set_global_sessions(total)
            c.set_search_mode(abi.SEARCH_ARGMAX)
            r = c.search_staged(1)
            per_rank.append([r.candidate_slo_ok[i] for i in range(len(plans))])
    # the NCCL rule (counts summed, any negative excludes; invalid dominates)
    totals = []
    for a, b in zip(*per_rank):
        if -1 in (a, b):
            totals.append(-1)
        elif a < 0 or b < 0:
            totals.append(-2)
        else:
            totals.append(a + b)
    best = native.argmax_candidates(totals)
    assert best == full.best_candidate and totals[best] == full.best_slo_ok
    # the torch.distributed helper applies the same rule
    import torch
    assert distributed.argmax(torch.tensor(totals)) == (full.best_candidate, full.best_slo_ok)
