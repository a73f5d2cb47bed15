"""World-size-2 runs of the sharded search with the REAL engine: two
processes (one per rank, each with its own library context on the one GPU of
the box), each replaying its shard through the C-ABI
(pdsim_shard_pairs + pdsim_gpu_search_staged_list), counts reduced over gloo
with the NCCL path's rule (distributed.reduce_counts), argmax by the C-ABI.
The NCCL collective itself needs one GPU per rank; tests/test_gpu_multi.py
runs it at world size one and pdsim_multi_plan_search over the device list."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_14516_b200 import abi, distributed, native

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    spec = native.default_synth_spec()
    prof = native.synth_profile(spec, 11)
    trs = [native.gen_trace(native.preset_stats("hotpotqa"), r, 250, 40 + k) for k, r in enumerate((2.0, 16.0, 30.0))]
    plans = native.enumerate_plans([1, 2, 4, 8], 8)
    return prof, trs, plans


def _sharded_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prof, trs, plans = _inputs()
    views = [t.view for t in trs]
    with native.Context(0) as ctx:
        ctx.stage(views, plans, prof, abi.default_params())
        mine = distributed.shard(views, plans, rank, world)
        res = ctx.search_staged_list(3, mine)
        local = [res.candidate_slo_ok[c] for c in range(len(plans))]
        pairs = {p: (res.pair_status[k], res.pair_attainment[k].slo_ok) for k, p in enumerate(mine)}
    totals = distributed.reduce_counts(local)
    q.put((rank, distributed.argmax(totals), totals.tolist(), pairs))
    dist.destroy_process_group()


def test_two_process_sharded_search_matches_single_search(ctx):
    prof, trs, plans = _inputs()
    views = [t.view for t in trs]
    full = ctx.plan_search(views, plans, prof, abi.default_params(), 3)
    want = [full.candidate_slo_ok[c] for c in range(len(plans))]
    port = _free_port()
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    procs = [mctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    seen = {}
    for rank, (best, cnt), totals, pairs in got:
        assert totals == want
        assert (best, cnt) == (full.best_candidate, full.best_slo_ok)
        for p, (st, ok) in pairs.items():
            assert p not in seen
            seen[p] = True
            assert st == full.pair_status[p] and ok == full.pair_attainment[p].slo_ok, p
    assert len(seen) == full.n_pairs  # the two shards partition the search


def _replica_worker(rank, world, port, q):
    """Replica-per-rank layout in ARGMAX mode: rank k stages only replica k
    and declares the whole search's session total."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prof, trs, plans = _inputs()
    views = [t.view for t in trs][:world]
    with native.Context(0) as ctx:
        ctx.stage([views[rank]], plans, prof, abi.default_params())
        ctx.set_global_sessions(sum(int(v.n_sessions) for v in views))
        ctx.set_search_mode(abi.SEARCH_ARGMAX)
        res = ctx.search_staged(3)
        local = [res.candidate_slo_ok[c] for c in range(len(plans))]
    totals = distributed.reduce_counts(local)
    q.put((rank, distributed.argmax(totals)))
    dist.destroy_process_group()


def test_two_process_replica_per_rank_argmax(ctx):
    prof, trs, plans = _inputs()
    views = [t.view for t in trs][:2]
    full = ctx.plan_search(views, plans, prof, abi.default_params(), 3)
    port = _free_port()
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    procs = [mctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, (best, cnt) in got:
        assert (best, cnt) == (full.best_candidate, full.best_slo_ok)
