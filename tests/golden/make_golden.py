"""Generates tests/golden/replay_cases.json from the UNMODIFIED reference
simulator (oracle/_ref/libpdsim_ref.so, built from /root/reference by
oracle/Makefile). Run in the build container, where the reference exists:

    python tests/golden/make_golden.py

Each case records its generator parameters, digests of the generated inputs
(so input drift is detected), and digests of the reference's outputs:
counters, attainment, and FNV-1a of the canonical text of every decision,
TTFT sample and session outcome (floats as exact hex). Tiny cases also store
the full records. The reference's own CSV fingerprints (metrics.cpp:366-474)
are stored alongside for the SURVEY.md §8(c) scenario.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import refbind  # noqa: E402
from tests import parity  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "replay_cases.json")

SCENARIO_SPEC = {"degrees": [1], "decode_alpha_min": 0.01056, "decode_alpha_max": 0.01144,
                 "decode_beta_min": 1.14e-4, "decode_beta_max": 1.26e-4}


def cases():
    out = []
    # SURVEY fingerprint scenario (dureader 4000 @16, seed 101; P:2x1,D:2x1; profile 7; engine 2).
    out.append(dict(name="survey_fingerprint", preset="dureader", rate=16.0, n=4000, gen_seed=101,
                    profile_seed=7, x={1: 2}, y={1: 2}, params={}, engine_seed=2))
    # Acceptance saturating scenario (acceptance_test.cpp:125-172) in every routing/reorder mode.
    for routing in (0, 1, 2):
        for reorder in (0, 1):
            out.append(dict(name=f"acceptance_r{routing}_o{reorder}", preset="dureader", rate=16.0, n=4000,
                            gen_seed=101, profile_seed=42, spec=SCENARIO_SPEC, x={1: 2}, y={1: 2},
                            params=dict(routing=routing, reorder=reorder, window=4, stat_window=1.5),
                            engine_seed=2))
    # Preset x load x plan grid.
    plans = [({1: 2}, {1: 2}), ({2: 1, 4: 1}, {1: 1, 2: 1}), ({}, {1: 3}), ({1: 1}, {8: 1})]
    for preset in ("toolbench", "gaia", "hotpotqa", "dureader"):
        for rate in (3.0, 25.0):
            for k, (x, y) in enumerate(plans):
                out.append(dict(name=f"{preset}_{rate}_{k}", preset=preset, rate=rate, n=300, gen_seed=17,
                                profile_seed=4, x=x, y=y, params={}, engine_seed=5))
    # Parameter corners.
    for i, prm in enumerate([dict(window=1), dict(window=8, stat_window=2.0), dict(alpha=0.5, beta=0.3),
                             dict(alpha=1.0, beta=1.0), dict(stat_window=0.25), dict(reorder=0, routing=1)]):
        out.append(dict(name=f"params_{i}", preset="dureader", rate=20.0, n=300, gen_seed=14, profile_seed=7,
                        x={1: 2}, y={1: 2}, params=prm, engine_seed=7))
    # KV admission pressure (sim_engine_test.cpp:209-236 regime): tiny capacity.
    out.append(dict(name="admission_pressure", preset="toolbench", rate=30.0, n=400, gen_seed=3, profile_seed=6,
                    spec={"degrees": [1, 2], "kv_bytes_per_token": 1000, "gpu_memory_capacity": 2_000_000},
                    x={1: 1}, y={1: 1, 2: 1}, params={}, engine_seed=2))
    # Hand-built traces (sim_engine_test.cpp:45-55, 269-294): exact closed forms.
    single = [{"id": 0, "arrival": 0.0, "rounds": [[700, 3, 0.5], [250, 2, 0.0]]}]
    for routing in (0, 1, 2):
        out.append(dict(name=f"single_session_r{routing}", sessions_manual=single, slo=[5.0, 0.5], profile_seed=4,
                        x={1: 1}, y={1: 1}, params=dict(routing=routing), engine_seed=1, full=True))
    ties = [{"id": 10 - i, "arrival": 0.0 if i < 4 else 0.001 * i, "rounds": [[100 + 50 * (i % 3), 4, 0.1],
                                                                          [80, 3, 0.0]]} for i in range(8)]
    out.append(dict(name="equal_time_ties_unsorted_ids", sessions_manual=ties, slo=[0.5, 0.05], profile_seed=1,
                    x={1: 2}, y={1: 2}, params={}, engine_seed=9, full=True))
    return out


def main():
    result = []
    for c in cases():
        trace, plan, prof, params = parity.build_case(c)
        out, hashes, _, n_itl = refbind.run(trace.view, plan, prof, params, c["engine_seed"])
        run = parity.Run(out, None, None, None)
        run.decisions = [out.decisions[i] for i in range(out.n_decisions)]
        run.ttft_samples = [out.ttft_samples[i] for i in range(out.n_ttft)]
        run.sessions = [out.sessions[i] for i in range(out.n_sessions)]
        entry = dict(case=c, inputs=dict(trace=parity.trace_digest(trace.view), profile=parity.profile_digest(prof)),
                     expect=parity.digest(run),
                     reference_csv_fnv=dict(decisions=f"{hashes[0]:016x}", ttft=f"{hashes[1]:016x}",
                                            sessions=f"{hashes[2]:016x}", itl=f"{hashes[3]:016x}"),
                     itl_samples=n_itl)
        if c.get("full"):
            entry["records"] = dict(zip(("decisions", "ttft_samples", "sessions"), parity.record_lines(run)))
        result.append(entry)
        print(c["name"], entry["expect"]["attainment"], flush=True)
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "source": "reference pdsim (oracle/_ref)",
                   "cases": result}, f, indent=1)


if __name__ == "__main__":
    main()
