"""World-size-2 gloo tests of the sharded search host logic. Each rank takes
its pairs from the library's cost-aware shard planner (C-ABI
pdsim_shard_pairs), replays them (the CPU checker stands in for the GPU
engine here; tests/test_gpu_multi.py runs the engine), the counts are
all-reduced with the flags rule of the NCCL path, and the C-ABI argmax
(pdsim_argmax_candidates) equals the single-process search."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_14516_b200 import abi, distributed, native


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    prof = native.synth_profile(native.default_synth_spec(), 7)
    traces = [native.gen_trace(native.preset_stats("toolbench"), 14.0, 120, s) for s in (1, 2)]
    plans = native.enumerate_plans([1, 2, 4, 8], 4)
    return prof, traces, plans


def _shard_counts(pairs, prof, traces, plans):
    """CPU checker for one shard: per-candidate slo_ok (-1 invalid)."""
    from tests import parity
    nt = len(traces)
    out = [0] * len(plans)
    for p in pairs:
        c, r = divmod(p, nt)
        try:
            run = parity.oracle_run(traces[r].view, plans[c], prof, abi.default_params(), 1)
            if out[c] >= 0:
                out[c] += run.attainment.slo_ok
        except Exception:
            out[c] = -1
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prof, traces, plans = _inputs()
    views = [t.view for t in traces]
    mine = distributed.shard(views, plans, rank, world)
    best, cnt, totals = distributed.sharded_search(
        lambda pairs: _shard_counts(pairs, prof, traces, plans), views, plans, rank, world)
    q.put((rank, best, cnt, totals.tolist(), mine))
    dist.destroy_process_group()


def test_two_rank_sharded_argmax_matches_single_process():
    prof, traces, plans = _inputs()
    n_pairs = len(traces) * len(plans)
    full = _shard_counts(range(n_pairs), prof, traces, plans)
    want_best = max(range(len(full)), key=lambda c: (full[c], -c))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = {}
    for rank, best, cnt, totals, mine in res:
        assert totals == full
        assert best == want_best
        assert cnt == full[want_best]
        shards[rank] = mine
    assert sorted(shards[0] + shards[1]) == list(range(n_pairs))  # a partition of the pairs


def test_shard_ranges_partition_the_pairs():
    for n in (1, 7, 169, 2704):
        for world in (1, 2, 3, 8):
            spans = [distributed.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_argmax_ties_and_invalid():
    t = torch.tensor([5, 7, -1, 7, 3])
    assert distributed.argmax(t) == (1, 7)
    assert distributed.argmax(torch.tensor([-1, -1])) == (-1, -1)


def _pruned_worker(rank, world, port, q):
    """Argmax-mode shards: each rank reports -2 for candidates its own bounds
    pruned; the reduction excludes every negative (include/pdsim_gpu.h)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local = [[-2, 5, 3, 7], [4, 6, -2, -1]][rank]
    totals = distributed.reduce_counts(local)
    q.put((rank, distributed.argmax(totals), totals.tolist()))
    dist.destroy_process_group()


def test_two_rank_reduction_excludes_pruned_candidates():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pruned_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, (best, cnt), totals in got:
        assert totals == [-2, 11, -2, -1]  # invalid anywhere wins over pruned
        assert (best, cnt) == (1, 11)


def test_shard_planner_is_a_balanced_lpt_partition():
    """pdsim_shard_pairs: every pair on exactly one rank; each rank's queue
    in non-increasing cost; the split equals LPT list scheduling restated
    here (cost = rounds x (workers + 2), ties to the lower pair / rank)."""
    prof, traces, plans = _inputs()
    views = [t.view for t in traces] + [native.gen_trace(native.preset_stats("gaia"), 3.0, 60, 9).view]
    nt = len(views)

    def cost(p):
        c, r = divmod(p, nt)
        x, y = abi.plan_dict(plans[c])
        return max(int(views[r].n_rounds), 1) * (sum(x.values()) + sum(y.values()) + 2)

    n = nt * len(plans)
    for world in (1, 2, 3, 8):
        order = sorted(range(n), key=lambda p: (-cost(p), p))
        load, want = [0] * world, [[] for _ in range(world)]
        for p in order:
            k = min(range(world), key=lambda j: (load[j], j))
            load[k] += cost(p)
            want[k].append(p)
        got = [distributed.shard(views, plans, r, world) for r in range(world)]
        assert got == want
        assert sorted(sum(got, [])) == list(range(n))
        assert max(load) - min(load) <= max(cost(p) for p in range(n))
