// pdsim/reorder.hpp — drop-in prefill-queue reordering (reference
// proj/include/pdsim/reorder.hpp:26-69; paper Alg. 2). Host utilities; the
// replay reorders on the GPU (engine.cuh: one lane per candidate
// permutation, REDUX.MAX winner).
#ifndef PDSIM_REORDER_HPP_
#define PDSIM_REORDER_HPP_

#include <deque>
#include <vector>

#include "pdsim/perf_model.hpp"
#include "pdsim/worker_state.hpp"

namespace pdsim {

struct ReorderParams {
  int window = 3;           // head-of-queue tasks considered per decision
  double ttft_thres = 5.0;  // seconds
};

struct ReorderOutcome {
  std::vector<int> chosen_order;  // chosen_order[k] = index into the head of the task served k-th
  int predicted_satisfied = 0;
  PrefillTask task;  // the dequeued head after reordering
};

// Completion offsets (from now) of `tasks` served back to back in `order`.
// Throws DomainError unless `order` is a permutation of the task indices.
std::vector<double> predict_completions(const std::vector<PrefillTask>& tasks, const std::vector<int>& order,
                                        const PerfProfile& profile, const ParallelismStrategy& theta);

// Tasks whose (now - enqueue_time) + predicted completion <= ttft_thres.
int count_satisfied(const std::vector<PrefillTask>& tasks, const std::vector<int>& order, double now,
                    double ttft_thres, const PerfProfile& profile, const ParallelismStrategy& theta);

// Reorders the first min(window, size) tasks to maximise count_satisfied
// (strict improvements over lexicographic permutation order; a task may not
// move back once postponed `window` times), bumps the postponement counts of
// the tasks moved back, and pops the new head.
ReorderOutcome reorder_and_dequeue(std::deque<PrefillTask>& queue, double now, const ReorderParams& params,
                                   const PerfProfile& profile, const ParallelismStrategy& theta);

}  // namespace pdsim

#endif  // PDSIM_REORDER_HPP_
