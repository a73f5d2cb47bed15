"""The replay engine's logic (engine.cuh) compiled for the HOST (test-only
build tests/native/libhostsim.so) against the golden fixtures and the
oracle, so every CPU test run exercises the exact source the GPU runs."""
import ctypes as C
import math
import random

import pytest

from paper_2602_14516_b200 import abi, native
from tests import golden_cases, parity

CASES = golden_cases.load()


@pytest.mark.parametrize("entry", CASES, ids=golden_cases.ids())
def test_engine_matches_golden(entry):
    c = entry["case"]
    trace, plan, prof, params = parity.build_case(c)
    got = parity.host_run(trace.view, plan, prof, params, c["engine_seed"])
    assert parity.digest(got) == entry["expect"]
    if "records" in entry:
        dec, ttft, sess = parity.record_lines(got)
        assert dec == entry["records"]["decisions"]
        assert ttft == entry["records"]["ttft_samples"]
        assert sess == entry["records"]["sessions"]


@pytest.mark.parametrize("seed", range(6))
def test_engine_matches_oracle_random_configs(seed):
    rng = random.Random(seed)
    spec = native.default_synth_spec()
    prof = native.synth_profile(spec, rng.randrange(1, 1000))
    preset = rng.choice(["toolbench", "gaia", "hotpotqa", "dureader"])
    st = native.preset_stats(preset)
    tr = native.gen_trace(st, rng.choice([1.0, 6.0, 15.0, 35.0]), rng.choice([80, 200, 400]), rng.randrange(1 << 30))
    plans = native.enumerate_plans([1, 2, 4, 8], 8)
    for _ in range(4):
        plan = rng.choice(plans)
        prm = abi.default_params(routing=rng.choice([0, 0, 0, 1, 2]), reorder=rng.choice([0, 1, 1]),
                                 window=rng.randint(1, 6), stat_window=rng.choice([0.5, 2.0, 10.0]),
                                 alpha=rng.choice([0.5, 0.9, 1.0]), beta=rng.choice([0.3, 0.85, 1.0]))
        es = rng.randrange(1 << 62)
        a = parity.host_run(tr.view, plan, prof, prm, es)
        b = parity.oracle_run(tr.view, plan, prof, prm, es)
        parity.assert_same_run(a, b)
        c = parity.host_run_counts(tr.view, plan, prof, prm, es)
        assert not parity.diff_counts(c, b)


def naive_fold(s, g, n):
    for _ in range(n):
        s = s + g
    return s


def test_fold_repeat_is_exact():
    f = parity.hostsim().hostsim_fold_repeat
    rng = random.Random(5)
    for i in range(4000):
        s = 0.0 if i % 4 == 0 else math.ldexp(rng.random(), rng.randint(-20, 20))
        g = math.ldexp(rng.random(), rng.randint(-25, 5))
        if i % 5 == 0:
            g = math.ldexp(3.0, -rng.randint(0, 60))  # short mantissas: exact half-ulp ties
        if i % 7 == 0:
            g = s * 2.0 ** -rng.randint(50, 56)  # near-absorbed increments
        n = rng.randint(0, 3000)
        assert f(s, g, n) == naive_fold(s, g, n), (s, g, n)
    assert f(1.0, 0.0, 10) == 1.0
    assert f(0.0, 0.0, 10) == 0.0


def test_engine_config_errors_mirror_reference():
    prof = native.synth_profile(native.default_synth_spec(), 4)
    tr = native.gen_trace(native.preset_stats("toolbench"), 2.0, 20, 1)
    ok = abi.make_plan({1: 1}, {1: 1})
    cases = [
        (abi.make_plan({1: 1}, {}), abi.default_params()),          # no decode replica
        (abi.make_plan({1: 1}, {16: 1}), abi.default_params()),     # degree not in profile
        (ok, abi.default_params(alpha=0.0)),
        (ok, abi.default_params(beta=1.5)),
        (ok, abi.default_params(window=0)),
        (ok, abi.default_params(stat_window=0.0)),
        (ok, abi.default_params(window=9)),                         # reorder cap (reorder.cpp:86-90)
    ]
    for plan, prm in cases:
        with pytest.raises(parity.EngineError) as e:
            parity.host_run(tr.view, plan, prof, prm, 1)
        assert e.value.code == abi.ERR_CONFIG
        with pytest.raises(Exception):
            parity.oracle_run(tr.view, plan, prof, prm, 1)
    # window > 8 is fine without reordering
    parity.host_run(tr.view, ok, prof, abi.default_params(window=9, reorder=0), 1)


def test_kv_precheck_rejects_unfittable_first_round():
    """sim_engine_test.cpp:238-254."""
    spec = native.default_synth_spec()
    spec.n_degrees, spec.degrees[0] = 1, 1
    spec.kv_bytes_per_token, spec.gpu_memory_capacity = 1000, 50000
    prof = native.synth_profile(spec, 6)
    tr = parity.manual_trace([{"id": 0, "arrival": 0.0, "rounds": [[100, 5, 0.0]]}], (50.0, 5.0))
    with pytest.raises(parity.EngineError) as e:
        parity.host_run(tr.view, abi.make_plan({1: 1}, {1: 1}), prof, abi.default_params(), 1)
    assert e.value.code == abi.ERR_CONFIG


def test_admission_wait_and_resume():
    """sim_engine_test.cpp:209-236."""
    spec = native.default_synth_spec()
    spec.n_degrees, spec.degrees[0] = 1, 1
    spec.kv_bytes_per_token, spec.gpu_memory_capacity = 1000, 150000
    prof = native.synth_profile(spec, 6)
    tr = parity.manual_trace([{"id": i, "arrival": 0.05 * i, "rounds": [[100, 50, 0.0]]} for i in range(2)],
                             (50.0, 5.0))
    r = parity.host_run(tr.view, abi.make_plan({1: 1}, {1: 1}), prof, abi.default_params(), 2)
    assert r.sessions[0].admission_wait == 0.0
    assert r.sessions[1].admission_wait > 0.0
    assert r.sessions[1].completion_time > r.sessions[0].completion_time
    assert r.counters.kv_bytes_residual == 0


def test_engine_heap_spill_to_global_matches_golden():
    """With a one-entry shared-memory heap every session event spills to the
    global area; results must not change."""
    H = parity.hostsim()
    H.hostsim_set_smem_budget.argtypes = [C.c_size_t]
    H.hostsim_set_smem_budget(1)
    try:
        for entry in CASES[:12]:
            c = entry["case"]
            trace, plan, prof, params = parity.build_case(c)
            got = parity.host_run(trace.view, plan, prof, params, c["engine_seed"])
            assert parity.digest(got) == entry["expect"], c["name"]
    finally:
        H.hostsim_set_smem_budget(0)


@pytest.mark.parametrize("entry", CASES, ids=golden_cases.ids())
def test_engine_search_mode_counts_match_golden(entry):
    """Without record arrays the engine runs its search-mode paths (per-session
    ITL sums bracketed with directed rounding, certified verdicts); counters and
    attainment must still equal the reference's."""
    c = entry["case"]
    trace, plan, prof, params = parity.build_case(c)
    got = parity.host_run_counts(trace.view, plan, prof, params, c["engine_seed"])
    assert parity.digest(got)["counters"] == entry["expect"]["counters"]
    assert parity.digest(got)["attainment"] == entry["expect"]["attainment"]


@pytest.mark.parametrize("preset,rate,plan", [("toolbench", 6.0, ({1: 2}, {1: 2})), ("hotpotqa", 20.0, ({2: 1}, {1: 3})),
                                              ("dureader", 35.0, ({1: 1}, {1: 1, 2: 1})), ("gaia", 3.0, ({}, {1: 2}))])
def test_engine_itl_samples_match_reference(preset, rate, plan):
    """SimResult::itl_samples materialised from the step log and round spans
    (pack.hpp expand_itl) equal the reference's per-token push order."""
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    prof = native.synth_profile(native.default_synth_spec(), 7)
    tr = native.gen_trace(native.preset_stats(preset), rate, 150, 9)
    p = abi.make_plan(*plan)
    for prm in (abi.default_params(), abi.default_params(routing=abi.ROUTING_ALWAYS_LOCAL, window=5)):
        got = parity.host_run_itl(tr.view, p, prof, prm, 4)
        want = parity.reference_itl(tr.view, p, prof, prm, 4)
        assert got.n_itl == len(want)
        assert not parity.diff_itl(got.itl_samples, want)
        # the records stay bit-identical with ITL materialisation on (exact stepping)
        parity.assert_same_run(got, parity.oracle_run(tr.view, p, prof, prm, 4))


def test_itl_csv_hash_emulation_matches_reference():
    """parity.itl_csv_fnv reproduces the reference's itl_samples.csv bytes."""
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    prof = native.synth_profile(native.default_synth_spec(), 7)
    tr = native.gen_trace(native.preset_stats("gaia"), 5.0, 60, 3)
    p = abi.make_plan({1: 1}, {1: 2})
    _, hashes, _, _ = refbind.run(tr.view, p, prof, abi.default_params(), 1, records=True, itl=True)
    want = parity.reference_itl(tr.view, p, prof, abi.default_params(), 1)
    assert parity.itl_csv_fnv(want) == f"{hashes[3]:016x}"


@pytest.mark.parametrize("preset,rate,plan", [("toolbench", 6.0, ({1: 2}, {1: 2})), ("hotpotqa", 25.0, ({2: 1}, {1: 3})),
                                              ("dureader", 35.0, ({1: 1}, {1: 1, 2: 1})), ("gaia", 3.0, ({}, {1: 2})),
                                              ("toolbench", 60.0, ({1: 1}, {1: 1}))])
def test_engine_report_matches_reference(preset, rate, plan):
    """Search report mode: the reference's build_report (metrics.cpp:138-190)
    of the pair — in-order means, nearest-rank P95s (TTFT initial /
    incremental, ITL), attainment ratios, e2e mean, local fraction —
    bit-identical."""
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    prof = native.synth_profile(native.default_synth_spec(), 7)
    tr = native.gen_trace(native.preset_stats(preset), rate, 200, 13)
    p = abi.make_plan(*plan)
    for prm in (abi.default_params(), abi.default_params(routing=abi.ROUTING_ALWAYS_REMOTE)):
        got = parity.host_report(tr.view, p, prof, prm, 6)
        want = refbind.report(tr.view, p, prof, prm, 6)
        assert got.as_tuple() == want.as_tuple()
