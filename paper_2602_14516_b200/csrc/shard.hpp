// shard.hpp — cost-aware sharding of the (candidate, replica) pairs over GPUs
// and the per-GPU queue order. Host only, deterministic:
// every rank computes the whole assignment from the same inputs and keeps its
// own part, so sharding needs no communication.
//
// Cost model of a pair: the replay is a serial event loop whose length grows
// with the trace's rounds and with the plan's worker count (every worker adds
// decode steps, prefill completions and routing candidates), so
// cost(c, r) = rounds(r) * (P(c) + D(c) + 2). Pairs are taken in decreasing
// cost (ties: smaller pair index) and each goes to the least-loaded rank
// (ties: lower rank) — longest-processing-time-first list scheduling, which
// also interleaves the heavy candidates across GPUs. Within a rank the list
// keeps that order: the persistent kernel's atomic queue hands out the
// heaviest pairs first, so the last wave holds the short ones.
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "pdsim_gpu.h"

namespace pdg {

inline int64_t plan_workers(const pdsim_plan& p) {
  int64_t n = 0;
  for (int g = 0; g < p.n_prefill_groups && g < PDSIM_MAX_GROUPS; ++g) n += p.prefill_count[g];
  for (int g = 0; g < p.n_decode_groups && g < PDSIM_MAX_GROUPS; ++g) n += p.decode_count[g];
  return n;
}

// Pairs of `rank` (global index c * n_traces + r) in queue order.
inline std::vector<int64_t> shard_pairs(int32_t n_traces, const int64_t* trace_rounds, int32_t n_candidates,
                                        const pdsim_plan* candidates, int32_t world, int32_t rank) {
  const int64_t n = static_cast<int64_t>(n_traces) * n_candidates;
  std::vector<int64_t> cost(static_cast<size_t>(n));
  for (int32_t c = 0; c < n_candidates; ++c) {
    const int64_t w = plan_workers(candidates[c]) + 2;
    for (int32_t r = 0; r < n_traces; ++r) {
      cost[static_cast<size_t>(c) * n_traces + r] = std::max<int64_t>(trace_rounds[r], 1) * w;
    }
  }
  std::vector<int64_t> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return cost[static_cast<size_t>(a)] > cost[static_cast<size_t>(b)];
  });
  std::vector<int64_t> load(static_cast<size_t>(world), 0);
  std::vector<int64_t> mine;
  for (int64_t p : order) {
    int32_t best = 0;
    for (int32_t k = 1; k < world; ++k) {
      if (load[static_cast<size_t>(k)] < load[static_cast<size_t>(best)]) best = k;
    }
    load[static_cast<size_t>(best)] += cost[static_cast<size_t>(p)];
    if (best == rank) mine.push_back(p);
  }
  return mine;
}

}  // namespace pdg
