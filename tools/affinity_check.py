"""SM-affine queue experiment: results equal the plain queue (both builds)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2s"
wl = workloads.CONFIGS[cfg]()
with native.Context(0) as ctx:
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    for build in (abi.BUILD_LATENCY, abi.BUILD_THROUGHPUT):
        ctx.set_kernel_build(build)
        os.environ.pop("PDSIM_SM_AFFINITY", None)
        base = ctx.search_staged(wl.seed)
        os.environ["PDSIM_SM_AFFINITY"] = "1"
        try:
            aff = ctx.search_staged(wl.seed)
        except Exception as e:  # noqa: BLE001
            print("build", build, "affinity FAILED:", e, flush=True)
            raise
        same = all(base.pair_events[p] == aff.pair_events[p] for p in range(base.n_pairs))
        print("build", build, "base ms", base.kernel_ms, "affinity ms", aff.kernel_ms, "same events", same,
              "best", base.best_candidate, aff.best_candidate, flush=True)
