"""Kernel time of one GPU's shard of a search at N GPUs (pdsim_shard_pairs,
rank 0) with each kernel build: where AUTO should switch from the LATENCY
to the THROUGHPUT build.

usage: python tools/build_threshold.py [CONFIG] [WORLD ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402


def main(cfg="C3", *worlds):
    wl = workloads.CONFIGS[cfg]()
    with native.Context(0) as ctx:
        ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
        for w in [int(x) for x in (worlds or (1, 2, 4, 8))]:
            pairs = native.shard_pairs(wl.traces, wl.plans, w, 0)
            row = {"config": cfg, "world": w, "pairs": len(pairs)}
            for name, b in (("latency", abi.BUILD_LATENCY), ("throughput", abi.BUILD_THROUGHPUT)):
                ctx.set_kernel_build(b)
                ctx.search_staged_list(wl.seed, pairs)
                row[name + "_ms"] = min(ctx.search_staged_list(wl.seed, pairs).kernel_ms for _ in range(2))
            ctx.set_kernel_build(abi.BUILD_AUTO)
            ctx.search_staged_list(wl.seed, pairs)
            row["auto"] = {abi.BUILD_LATENCY: "latency", abi.BUILD_THROUGHPUT: "throughput"}[ctx.last_kernel_build()]
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
