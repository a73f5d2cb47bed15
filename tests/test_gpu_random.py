"""Randomised batched searches against the unmodified reference: random cost
models, presets, rates, plan subsets and scheduler settings (routing mode,
reorder, window, statistics window, alpha, beta). Per-pair attainment and
status equal the reference's; the argmax search mode picks the same plan."""
import random

import pytest

from paper_2602_14516_b200 import abi, native
from tests import parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(24))
def test_random_search_matches_reference(ctx, seed):
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
    res = ctx.plan_search(views, plans, prof, prm, es)
    att, st_ref, _ = refbind.plan_search(views, plans, prof, prm, es)
    for p in range(res.n_pairs):
        assert res.pair_status[p] == st_ref[p], p
        if st_ref[p] == 0:
            for f in parity.ATT_FIELDS:
                assert getattr(res.pair_attainment[p], f) == getattr(att[p], f), (p, f)
    ctx.set_search_mode(abi.SEARCH_ARGMAX)
    try:
        pr = ctx.plan_search(views, plans, prof, prm, es)
    finally:
        ctx.set_search_mode(abi.SEARCH_FULL)
    assert (pr.best_candidate, pr.best_slo_ok) == (res.best_candidate, res.best_slo_ok)
