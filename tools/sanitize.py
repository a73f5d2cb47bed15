"""Small replays + a planner sweep for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402

prof = native.synth_profile(native.default_synth_spec(), 7)
tr = native.gen_trace(native.preset_stats("dureader"), 16.0, 120, 101)
with native.Context(0) as ctx:
    r = ctx.run(tr.view, abi.make_plan({1: 2}, {1: 2}), prof, abi.default_params(window=4, stat_window=1.5), 2)
    print("run ok", r.attainment.slo_ok, r.n_decisions)
    plans = native.enumerate_plans([1, 2, 4], 4)
    s = ctx.plan_search([tr.view], plans, prof, abi.default_params(), 1)
    print("search ok", s.best_candidate, s.best_slo_ok)
    st = native.preset_stats("toolbench")
    c = ctx.estimate_coefficients(st, [4.0, 8.0], [1, 2], prof, [1, 2, 4], 4)
    print("planner ok", [x[1] for x in c])
    trs = [native.gen_trace(native.preset_stats("hotpotqa"), 20.0, 80, k) for k in (1, 2)]
    ctx.set_search_mode(abi.SEARCH_ARGMAX)
    a = ctx.plan_search([t.view for t in trs], plans, prof, abi.default_params(), 1)
    ctx.set_search_mode(abi.SEARCH_FULL)
    print("argmax ok", a.best_candidate, a.best_slo_ok)
    settings = [abi.default_params(), abi.default_params(alpha=0.5, window=1), abi.default_params(reorder=0)]
    w = ctx.sweep([t.view for t in trs], abi.make_plan({1: 1}, {1: 2}), prof, settings, 3)
    print("sweep ok", [round(x.slo_attainment, 3) for x in w.reports])
