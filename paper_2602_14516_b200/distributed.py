"""Multi-GPU sharding of the plan search, torch.distributed
plumbing around the library's own shard planner and argmax.

One process per GPU. The (candidate, replica) pairs are independent replays:
rank r replays the pairs the library's cost-aware LPT split gives it
(pdsim_shard_pairs: pair cost rounds x (workers + 2), heaviest first, each to
the least-loaded rank; every rank computes the same split locally, so there is
no data-path communication). The only collective is the reduction of the
per-candidate SLO counts (int64 sum) and of the invalid / pruned flags (max),
followed by the argmax (pdsim_argmax_candidates: max Σslo_ok, ties to the
smallest enumeration index). On GPUs the library performs that reduction
itself over NCCL (pdsim_gpu_comm_init, see bench.py); this module's
torch.distributed path is the same rule for gloo / CPU callers and tests.
"""
import torch
import torch.distributed as dist

from . import native


def shard(traces, plans, rank, world):
    """This rank's pairs in queue order (C-ABI pdsim_shard_pairs)."""
    return native.shard_pairs(traces, plans, world, rank)


def shard_range(n_pairs, rank, world):
    """Contiguous candidate-major range (kept for pair-range callers)."""
    return n_pairs * rank // world, n_pairs * (rank + 1) // world


def reduce_counts(candidate_slo_ok, device="cpu"):
    """Combines this rank's per-candidate counts (-1 invalid, -2 pruned here)
    across ranks: counts summed, flags max-reduced with invalid dominating;
    returns the totals (-1 invalid, -2 pruned anywhere)."""
    cand = torch.as_tensor(list(candidate_slo_ok), dtype=torch.int64, device=device)
    flag = torch.where(cand == -1, torch.full_like(cand, 2), torch.where(cand < 0, torch.ones_like(cand),
                                                                          torch.zeros_like(cand)))
    cnt = torch.clamp(cand, min=0)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
    return torch.where(flag == 2, torch.full_like(cnt, -1), torch.where(flag == 1, torch.full_like(cnt, -2), cnt))


def argmax(totals):
    """Max count, ties to the smallest index; (-1, -1) if every candidate is
    excluded (C-ABI pdsim_argmax_candidates)."""
    vals = [int(x) for x in totals.tolist()]
    best = native.argmax_candidates(vals)
    return (best, vals[best]) if best >= 0 else (-1, -1)


def sharded_search(search_fn, traces, plans, rank, world, device="cpu"):
    """search_fn(pairs) -> per-candidate slo_ok over those pairs (-1 invalid,
    -2 pruned). Returns (best_candidate, best_slo_ok, totals)."""
    local = search_fn(shard(traces, plans, rank, world))
    totals = reduce_counts(local, device=device)
    best, cnt = argmax(totals)
    return best, cnt, totals
