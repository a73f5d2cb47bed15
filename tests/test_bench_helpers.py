"""bench.py's sampling and reporting helpers (plain Python, no GPU): the CPU
baseline's stratified random sample and the candidate attainment spread."""
import types

import bench


def test_stratified_sample_one_random_replica_per_candidate():
    n_traces, n_cand = 16, 169
    s = bench.stratified_sample(n_traces, n_cand)
    assert len(s) == n_cand  # 6.25 % of C3's 2704 pairs, >= 1 %
    assert [p // n_traces for p in s] == list(range(n_cand))  # every candidate shape exactly once
    assert all(0 <= p % n_traces < n_traces for p in s)
    assert len({p % n_traces for p in s}) > 1  # replicas vary (random, not the first)
    assert s == bench.stratified_sample(n_traces, n_cand)  # fixed seed
    assert bench.stratified_sample(1, 5) == list(range(5))  # single-replica searches: every pair


def test_attainment_spread_counts_regimes():
    traces = [types.SimpleNamespace(n_sessions=100), types.SimpleNamespace(n_sessions=100)]
    wl = types.SimpleNamespace(traces=traces, plans=[0] * 5)
    res = types.SimpleNamespace(candidate_slo_ok=[200, 190, 10, -1, 100])
    got = bench.attainment_spread(res, wl)
    assert got["best"] == 1.0 and got["worst"] == 0.05
    assert got["candidates_ge_90pct"] == 2 and got["candidates_lt_10pct"] == 1
    assert got["valid_candidates"] == 4  # the invalid candidate (-1) is excluded
