"""Does sharing an SM slow a pair down? Per-pair cycles of the full C2 search
(169 pairs on 148 SMs) vs the first 148 pairs alone (one per SM)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_14516_b200 import native, workloads  # noqa: E402

wl = workloads.c2()
with native.Context(0) as ctx:
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    ctx.search_staged(wl.seed)
    full = ctx.search_staged(wl.seed)
    part = ctx.search_staged(wl.seed, 0, 148)
    a = [full.pair_cycles[p] for p in range(148)]
    b = [part.pair_cycles[p] for p in range(148)]
    print("full kernel_ms", round(full.kernel_ms, 1), "first-148 kernel_ms", round(part.kernel_ms, 1))
    print("max cycles full/part", max(a), max(b), "mean ratio", sum(x / y for x, y in zip(a, b)) / 148)
    worst = sorted(range(148), key=lambda p: a[p] / b[p])[-5:]
    print("most slowed", [(p, round(a[p] / b[p], 3)) for p in worst])
