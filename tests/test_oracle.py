"""Pins the checkers: the plain-C restatement (oracle/pdsim_oracle.c) must
reproduce the reference's outputs — against the committed golden fixtures
(always) and against the reference library itself (where it was built)."""
import pytest

from paper_2602_14516_b200 import abi, native
from tests import golden_cases, parity

cbind = pytest.importorskip("oracle.cbind")
from oracle import refbind  # noqa: E402

CASES = golden_cases.load()


@pytest.mark.parametrize("entry", CASES, ids=golden_cases.ids())
def test_c_oracle_matches_golden(entry):
    c = entry["case"]
    trace, plan, prof, params = parity.build_case(c)
    assert parity.trace_digest(trace.view) == entry["inputs"]["trace"], "generated inputs drifted"
    assert parity.profile_digest(prof) == entry["inputs"]["profile"]
    got = cbind.run(trace.view, plan, prof, params, c["engine_seed"])
    assert parity.digest(got) == entry["expect"]
    if "records" in entry:
        dec, ttft, sess = parity.record_lines(got)
        assert dec == entry["records"]["decisions"]
        assert ttft == entry["records"]["ttft_samples"]
        assert sess == entry["records"]["sessions"]


def test_survey_fingerprint_fixture():
    """The fixture's reference CSV hashes are SURVEY.md §8(c)'s fingerprint."""
    e = next(x for x in CASES if x["case"]["name"] == "survey_fingerprint")
    assert e["reference_csv_fnv"]["decisions"] == "665772a5ffd1e99f"
    assert e["reference_csv_fnv"]["ttft"] == "e4e6dd847853dbae"
    assert e["reference_csv_fnv"]["sessions"] == "2038a6a05715eebb"


@pytest.mark.skipif(not refbind.available(), reason="reference library not built")
@pytest.mark.parametrize("preset", ["toolbench", "gaia", "hotpotqa", "dureader"])
def test_c_oracle_matches_reference_library(preset):
    prof = native.synth_profile(native.default_synth_spec(), 11)
    tr = native.gen_trace(native.preset_stats(preset), 18.0, 200, 23)
    for x, y in (({1: 1}, {1: 1}), ({1: 3}, {2: 2}), ({4: 1}, {1: 1, 2: 1})):
        plan = abi.make_plan(x, y)
        for kw in (dict(), dict(routing=1), dict(reorder=0), dict(window=6, stat_window=1.0)):
            prm = abi.default_params(**kw)
            a = cbind.run(tr.view, plan, prof, prm, 4)
            b = parity.oracle_run(tr.view, plan, prof, prm, 4)
            parity.assert_same_run(a, b)


def test_c_oracle_config_errors():
    prof = native.synth_profile(native.default_synth_spec(), 4)
    tr = native.gen_trace(native.preset_stats("toolbench"), 2.0, 10, 1)
    with pytest.raises(cbind.OracleError):
        cbind.run(tr.view, abi.make_plan({1: 1}, {}), prof, abi.default_params(), 1)
    with pytest.raises(cbind.OracleError):
        cbind.run(tr.view, abi.make_plan({1: 1}, {16: 1}), prof, abi.default_params(), 1)
    with pytest.raises(cbind.OracleError):
        cbind.run(tr.view, abi.make_plan({1: 1}, {1: 1}), prof, abi.default_params(window=9), 1)


def test_reference_arm_builds_identical_inputs():
    """bench.py's reference arm builds its inputs through the reference alone
    (oracle/ref_workloads.py); they must be byte-identical to the product
    arm's: traces, cost model, candidate order (SURVEY.md §8(d) pinning)."""
    import numpy as np
    from oracle import ref_workloads, refbind
    from paper_2602_14516_b200 import specs, workloads
    if not refbind.available():
        pytest.skip("reference library not built")

    def arrays(v):
        return [np.ctypeslib.as_array(getattr(v, f), shape=(n,)).tobytes() for f, n in
                [("session_id", v.n_sessions), ("arrival_time", v.n_sessions), ("round_offset", v.n_sessions + 1),
                 ("incr_input_len", v.n_rounds), ("decode_len", v.n_rounds), ("interaction_delay", v.n_rounds)]]

    for sp in (specs.c1(), specs.c2(sessions=400), specs.c3(sessions=200, replicas=2),
               specs.c4(rates=[2.0, 6.0], sessions=500), specs.c5(rates=[4.0], seeds=2, sessions=100)):
        a, b = workloads.build(sp), ref_workloads.build(sp)
        assert bytes(a.profile) == bytes(b.profile), sp.name
        assert [bytes(x) for x in a.plans] == [bytes(x) for x in b.plans], sp.name
        assert len(a.traces) == len(b.traces)
        for x, y in zip(a.traces, b.traces):
            assert arrays(x) == arrays(y) and (x.ttft_thres, x.itl_thres) == (y.ttft_thres, y.itl_thres), sp.name
        assert specs.config_dict(sp)["pairs"] == a.n_pairs == b.n_pairs
