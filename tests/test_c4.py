"""C4 (BASELINE.json configs[3]): llama3-70b, mixed toolbench + hotpotqa
traces merged by arrival time, an arrival-rate sweep.

CPU: the merge (workloads.merge_traces) is a valid reference Trace (the
reference's own Trace::validate via the oracle), sorted by arrival with
stable ties, ids renumbered, every session's rounds intact.
GPU: a C4 slice (all 169 N=8 plans x 3 rates of the sweep) replayed in one
search equals the unmodified reference per pair, per candidate and argmax.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2602_14516_b200 import abi, native, workloads
from tests import parity


def sessions_of(view):
    sid, arr, off, inc, dec, dly = workloads._arrays(view)
    return [(arr[k], [(int(inc[j]), int(dec[j]), float(dly[j])) for j in range(off[k], off[k + 1])])
            for k in range(len(sid))]


def test_merge_is_stable_and_keeps_rounds():
    a = native.gen_trace(workloads.trace_stats("toolbench"), 3.0, 300, 1)
    b = native.gen_trace(workloads.trace_stats("hotpotqa"), 3.0, 200, 2)
    m = workloads.merge_traces(a.view, b.view)
    assert m.view.n_sessions == 500 and m.view.n_rounds == a.view.n_rounds + b.view.n_rounds
    sid, arr, off, _, _, _ = workloads._arrays(m.view)
    assert list(sid) == list(range(500))
    assert np.all(np.diff(arr) >= 0)
    want = sessions_of(a.view) + sessions_of(b.view)
    order = sorted(range(len(want)), key=lambda k: (want[k][0], k))  # stable: a's sessions first on ties
    assert sessions_of(m.view) == [want[k] for k in order]
    assert native.lib().pdsim_trace_validate(C.byref(m.view)) == 0
    from oracle import refbind
    if refbind.available():  # the reference's own Trace::validate (workload.cpp:90-134)
        assert refbind.lib().ref_trace_validate(C.byref(m.view)) == 0


def test_merge_ties_keep_first_trace_first():
    slo = (1.0, 0.05)
    a = parity.manual_trace([{"id": 7, "arrival": 1.0, "rounds": [[10, 2, 0.0]]},
                             {"id": 9, "arrival": 2.0, "rounds": [[11, 3, 0.0]]}], slo)
    b = parity.manual_trace([{"id": 0, "arrival": 1.0, "rounds": [[20, 4, 0.1], [5, 5, 0.0]]}], slo)
    m = workloads.merge_traces(a.view, b.view)
    assert sessions_of(m.view) == [(1.0, [(10, 2, 0.0)]), (1.0, [(20, 4, 0.1), (5, 5, 0.0)]), (2.0, [(11, 3, 0.0)])]
    with pytest.raises(ValueError):
        workloads.merge_traces(a.view, parity.manual_trace([{"id": 0, "arrival": 0.0, "rounds": [[1, 1, 0.0]]}],
                                                            (2.0, 0.05)).view)


def test_merged_trace_runs_in_the_reference():
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    wl = workloads.c4(rates=[2.0], sessions=400)
    out = refbind.run(wl.traces[0], abi.make_plan({2: 1}, {2: 1}), wl.profile, wl.params, 1)[0]
    assert out.attainment.sessions_total == 400 and out.attainment.sessions_completed > 0


@pytest.mark.gpu
def test_c4_slice_search_matches_reference(ctx):
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    wl = workloads.c4(rates=[1.0, 4.0, 8.0], sessions=1500)
    res = ctx.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed)
    att, st_ref, _ = refbind.plan_search(wl.traces, wl.plans, wl.profile, wl.params, wl.seed)
    nt = len(wl.traces)
    sums = [0] * len(wl.plans)
    for p in range(wl.n_pairs):
        assert res.pair_status[p] == st_ref[p], p
        for f in parity.ATT_FIELDS:
            assert getattr(res.pair_attainment[p], f) == getattr(att[p], f), (p, f)
        c = p // nt
        sums[c] = -1 if (st_ref[p] != 0 or sums[c] < 0) else sums[c] + att[p].slo_ok
    assert [res.candidate_slo_ok[c] for c in range(len(wl.plans))] == sums
    assert res.best_candidate == max(range(len(sums)), key=lambda c: (sums[c], -c))
    # both regimes are covered: some pair saturates, some attains everything
    fr = [att[p].slo_ok / att[p].sessions_total for p in range(wl.n_pairs) if st_ref[p] == 0]
    assert min(fr) < 0.5 and max(fr) == 1.0


@pytest.mark.parametrize("case", ["dup-before-arrival", "arrival-before-dup", "dup-only", "bad-round-after-dup",
                                  "same-session-dup-and-arrival"])
def test_trace_validation_reports_the_reference_error(case):
    """pdsim_trace_validate finds duplicate ids by sorting (no per-session
    set) but must name the same first error as the reference's
    Trace::validate (workload.cpp:90-134), which checks each session's id
    before its other fields, in trace order."""
    from oracle import refbind
    if not refbind.available():
        pytest.skip("reference library not built")
    ok = lambda i, a: {"id": i, "arrival": a, "rounds": [[10, 2, 0.0]]}  # noqa: E731
    s = [ok(k, float(k)) for k in range(8)]
    if case == "dup-before-arrival":
        s[3]["id"] = 1
        s[5]["arrival"] = 0.5
    elif case == "arrival-before-dup":
        s[5]["id"] = 1
        s[3]["arrival"] = 0.5
    elif case == "dup-only":
        s[6]["id"] = 2
    elif case == "bad-round-after-dup":
        s[2]["id"] = 0
        s[4]["rounds"] = [[0, 2, 0.0]]
    else:
        s[4]["id"] = 0
        s[4]["arrival"] = 0.1
    tr = parity.manual_trace(s, (1.0, 0.05))
    rc = native.lib().pdsim_trace_validate(C.byref(tr.view))
    ours = native.lib().pdsim_last_error().decode()
    rrc = refbind.lib().ref_trace_validate(C.byref(tr.view))
    theirs = refbind.lib().ref_last_error().decode()
    assert rc != 0 and rrc != 0
    assert ours == theirs, (ours, theirs)
