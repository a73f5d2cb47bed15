"""Kernel time of one GPU's LPT shard of a search (world N, rank 0) per kernel
build, with the plain queue and the candidate-affine queues.

usage: python tools/shard_affinity.py CONFIG WORLD [WORLD ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import abi, native, workloads  # noqa: E402

cfg = sys.argv[1]
wl = workloads.CONFIGS[cfg]()
with native.Context(0) as ctx:
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    for world in map(int, sys.argv[2:]):
        shard = native.shard_pairs(wl.traces, wl.plans, world, 0)
        for build in (abi.BUILD_LATENCY, abi.BUILD_THROUGHPUT):
            ctx.set_kernel_build(build)
            for aff in ("0", "1"):
                os.environ["PDSIM_SM_AFFINITY"] = aff
                ctx.search_staged_list(wl.seed, shard)
                ms = min(ctx.search_staged_list(wl.seed, shard).kernel_ms for _ in range(2))
                print(json.dumps({"config": cfg, "world": world, "pairs": len(shard),
                                  "build": "latency" if build == abi.BUILD_LATENCY else "throughput",
                                  "affinity": aff, "kernel_ms": ms}), flush=True)
