"""Host generators are bit-identical to the reference's (north star: "traces
are generated on the host with the reference's own RNG so that inputs are
identical"), and candidate enumeration follows planner.cpp:582-657."""
import ctypes as C

import numpy as np
import pytest

from paper_2602_14516_b200 import abi, native

refbind = pytest.importorskip("oracle.refbind")
needs_ref = pytest.mark.skipif(not refbind.available(), reason="reference library not built")


def arrays(view):
    S, R = view.n_sessions, view.n_rounds
    a = lambda p, n: np.ctypeslib.as_array(p, (n,)).copy() if n else np.zeros(0)
    return dict(sid=a(view.session_id, S), arr=a(view.arrival_time, S), off=a(view.round_offset, S + 1),
                incr=a(view.incr_input_len, R), dec=a(view.decode_len, R), delay=a(view.interaction_delay, R),
                slo=(view.ttft_thres, view.itl_thres))


@needs_ref
@pytest.mark.parametrize("preset", ["toolbench", "gaia", "hotpotqa", "dureader"])
@pytest.mark.parametrize("rate,n,seed", [(0.5, 50, 1), (16.0, 2000, 101), (40.0, 500, 12345678901)])
def test_gen_trace_matches_reference(preset, rate, n, seed):
    st = native.preset_stats(preset)
    ours = native.gen_trace(st, rate, n, seed)
    ref = refbind.gen_trace(refbind.preset_stats(preset), preset, rate, n, seed)
    a, b = arrays(ours.view), arrays(ref.view)
    for k in a:
        if k == "slo":
            assert a[k] == b[k]
        else:
            assert a[k].dtype == b[k].dtype and np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k
    assert refbind.trace_hash(ours.view, preset) == refbind.trace_hash(ref.view, preset)


@needs_ref
def test_gen_trace_custom_stats_match_reference():
    st = native.preset_stats("toolbench")
    st.mean_rounds, st.fixed_rounds, st.length_cv, st.mean_interaction_delay = 1.0, 0, 0.0, 0.0
    for stats in (st,):
        ours = native.gen_trace(stats, 3.0, 300, 9)
        ref = refbind.gen_trace(stats, "custom", 3.0, 300, 9)
        assert refbind.trace_hash(ours.view, "x") == refbind.trace_hash(ref.view, "x")


@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 4, 7, 42, 2**63 + 5])
def test_synth_profile_matches_reference(seed):
    spec = native.default_synth_spec()
    ours = native.synth_profile(spec, seed)
    ref = refbind.synth_profile(spec, seed)
    assert bytes(ours) == bytes(ref)


@needs_ref
def test_model_presets_match_reference():
    from paper_2602_14516_b200 import workloads
    for name in workloads.MODEL_PRESETS:
        spec = workloads.model_spec(name)
        assert bytes(native.synth_profile(spec, 7)) == bytes(refbind.synth_profile(spec, 7))


@needs_ref
def test_survey_fingerprint_inputs():
    """profile daab0f5f25fc4a1d, trace 908379e3bd75387e."""
    prof = native.synth_profile(native.default_synth_spec(), 7)
    assert refbind.profile_hash(prof) == 0xdaab0f5f25fc4a1d
    tr = native.gen_trace(native.preset_stats("dureader"), 16.0, 4000, 101)
    assert refbind.trace_hash(tr.view, "dureader") == 0x908379e3bd75387e


def test_presets():
    tb = native.preset_stats("toolbench")
    assert (tb.mean_rounds, tb.fixed_rounds, tb.ttft_thres, tb.itl_thres) == (3.96, 0, 1.0, 0.05)
    du = native.preset_stats("dureader")
    assert (du.mean_rounds, du.fixed_rounds, du.ttft_thres) == (3.0, 1, 1.5)
    with pytest.raises(native.ConfigError):
        native.preset_stats("bogus")


def test_gen_trace_domain_errors():
    st = native.preset_stats("gaia")
    with pytest.raises(native.DomainError):
        native.gen_trace(st, 0.0, 10, 1)
    with pytest.raises(native.DomainError):
        native.gen_trace(st, 1.0, 0, 1)


def test_generated_trace_is_well_formed():
    tr = native.gen_trace(native.preset_stats("hotpotqa"), 5.0, 400, 3)
    a = arrays(tr.view)
    assert np.all(np.diff(a["arr"]) >= 0)
    assert np.all(np.diff(a["off"]) == 3)  # fixed 3 rounds
    assert np.all(a["incr"] >= 1) and np.all(a["dec"] >= 1)
    last = a["off"][1:] - 1
    assert np.all(a["delay"][last] == 0.0)


@pytest.mark.parametrize("n,count", [(1, 0), (2, 1), (4, 13), (8, 169), (16, 3389)])
def test_enumeration_counts(n, count):
    assert len(native.enumerate_plans([1, 2, 4, 8], n)) == count


def test_enumeration_order_is_reference_recursion():
    plans = [abi.plan_dict(p) for p in native.enumerate_plans([1, 2, 4, 8], 8)]
    # enumerate_counts recurses with the smallest degree outermost and counts
    # ascending: x={8:1} leaves no decode budget, so x={4:1} comes first and
    # its decode maps follow the same recursion under the remaining budget 4.
    assert plans[:9] == [({4: 1}, {4: 1}), ({4: 1}, {2: 1}), ({4: 1}, {2: 2}), ({4: 1}, {1: 1}),
                         ({4: 1}, {1: 1, 2: 1}), ({4: 1}, {1: 2}), ({4: 1}, {1: 2, 2: 1}), ({4: 1}, {1: 3}),
                         ({4: 1}, {1: 4})]
    xs = []
    for x, _ in plans:
        if not xs or xs[-1] != x:
            xs.append(x)
    key = lambda x: tuple(x.get(d, 0) for d in (1, 2, 4, 8))
    assert xs == sorted(xs, key=key), "x maps must be emitted in ascending count-vector order"
    assert len(set(map(key, xs))) == len(xs)


@needs_ref
@pytest.mark.parametrize("n", [4, 8, 16])
def test_enumeration_set_matches_reference_top_k(n):
    ours = native.enumerate_plans([1, 2, 4, 8], n)
    ref = refbind.top_k_plans([1, 2, 4, 8], n)
    canon = lambda p: (tuple(sorted(abi.plan_dict(p)[0].items())), tuple(sorted(abi.plan_dict(p)[1].items())))
    assert len(ours) == len(ref)
    assert set(map(canon, ours)) == set(map(canon, ref))


def test_profile_validation_rejects_malformed_curves():
    prof = native.synth_profile(native.default_synth_spec(), 1)
    assert native.lib().pdsim_profile_validate(C.byref(prof)) == 0
    bad = abi.Profile.from_buffer_copy(bytes(prof))
    bad.prefill[0].alpha[0] = -1.0
    assert native.lib().pdsim_profile_validate(C.byref(bad)) == abi.ERR_CONFIG
    bad = abi.Profile.from_buffer_copy(bytes(prof))
    bad.degrees[1] = 3
    assert native.lib().pdsim_profile_validate(C.byref(bad)) == abi.ERR_CONFIG
    bad = abi.Profile.from_buffer_copy(bytes(prof))
    bad.decode[0].breakpoints[0] = -5.0
    bad.decode[0].alpha[1] = 0.0
    bad.decode[0].beta[1] = 1e-9  # right segment far below the left limit
    assert native.lib().pdsim_profile_validate(C.byref(bad)) == abi.ERR_CONFIG


def test_batched_generation_is_bit_identical():
    """pdsim_gen_trace_batch (all host threads) equals
    separate gen_trace calls byte for byte."""
    st = native.preset_stats("toolbench")
    rates = [0.5 + 0.75 * k for k in range(24)]
    seeds = [7 * k + 1 for k in range(24)]
    batch = native.gen_traces(st, rates, 300, seeds)
    for tb, r, s in zip(batch, rates, seeds):
        one = native.gen_trace(st, r, 300, s)
        a, b = tb.view, one.view
        assert a.n_sessions == b.n_sessions and a.n_rounds == b.n_rounds
        for k in range(a.n_sessions):
            assert a.arrival_time[k] == b.arrival_time[k] and a.session_id[k] == b.session_id[k]
            assert a.round_offset[k + 1] == b.round_offset[k + 1]
        for k in range(a.n_rounds):
            assert (a.incr_input_len[k], a.decode_len[k], a.interaction_delay[k]) == \
                (b.incr_input_len[k], b.decode_len[k], b.interaction_delay[k])
    with pytest.raises(native.PdsimError):
        native.gen_traces(st, [1.0, -1.0], 10, [1, 2])
