"""Multi-GPU sharding of the plan search.

One process per GPU. The (candidate, replica) pairs are independent replays,
so rank r of N replays the contiguous range [P*r/N, P*(r+1)/N) of the
candidate-major pair index with no data-path communication. The only
collective is the reduction of per-candidate SLO counts (int64 sum) and of
the per-candidate invalid flags (max), followed by the argmax: max Σslo_ok,
ties to the smallest enumeration index. With the NCCL backend this is one
~C x 8 B all-reduce over NVLink; with gloo it runs on CPU (tests).
"""
import torch
import torch.distributed as dist


def shard_range(n_pairs, rank, world):
    return n_pairs * rank // world, n_pairs * (rank + 1) // world


def reduce_counts(candidate_slo_ok, device="cpu"):
    """Combines this rank's per-candidate counts (-1 = invalid here) across
    ranks; returns (totals tensor with -1 for invalid candidates)."""
    cand = torch.as_tensor(list(candidate_slo_ok), dtype=torch.int64, device=device)
    bad = (cand < 0).to(torch.int64)
    cnt = torch.clamp(cand, min=0)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
    return torch.where(bad > 0, torch.full_like(cnt, -1), cnt)


def argmax(totals):
    """Max count, ties to the smallest index; -1 if every candidate is invalid."""
    if int(torch.max(totals).item()) < 0:
        return -1, -1
    best = int(torch.argmax(totals).item())  # first maximal element
    return best, int(totals[best].item())


def sharded_search(search_fn, n_pairs, rank, world, device="cpu"):
    """search_fn(pair_begin, pair_end) -> per-candidate slo_ok of that shard
    (-1 invalid). Returns (best_candidate, best_slo_ok, totals)."""
    b, e = shard_range(n_pairs, rank, world)
    local = search_fn(b, e)
    totals = reduce_counts(local, device=device)
    best, cnt = argmax(totals)
    return best, cnt, totals
