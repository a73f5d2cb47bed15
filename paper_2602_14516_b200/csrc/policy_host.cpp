// policy_host.cpp — the reference's routing and reordering API on host state
// (include/pdsim/coordinator.hpp, reorder.hpp, worker_state.hpp).
//
// The replay engine makes these decisions on the GPU with its own data
// structures; this file gives drop-in callers (and the reference's own unit
// and acceptance suites, relinked unmodified in tests/native/) the same
// functions over WorkerState / PrefillTask. Semantics follow
// coordinator.cpp:27-171 and reorder.cpp:44-146: the same fp64 operation
// order (so results are bit-identical), the same tie rules and the same
// error classes. The reorder search enumerates permutations by rank in the
// factorial number system (lexicographic, like the device engine's
// lane-parallel search) over costs evaluated once per decision.
#include <algorithm>
#include <cassert>
#include <cstdint>
#include <numeric>
#include <vector>

#include "pdsim/coordinator.hpp"
#include "pdsim/errors.hpp"
#include "pdsim/reorder.hpp"
#include "pdsim/worker_state.hpp"

namespace pdsim {

// ---- WindowedStat ---------------------------------------------------------------

void WindowedStat::add(double completion_time, double latency) {
  assert(times_.empty() || completion_time >= times_.back());
  times_.push_back(completion_time);
  values_.push_back(latency);
}

double WindowedStat::query(double now) const {
  // window (now - w, now]: first sample after the cutoff .. first after now
  const double cutoff = now - window_;
  const auto first = std::partition_point(times_.begin(), times_.end(), [&](double t) { return t <= cutoff; });
  const auto last = std::partition_point(first, times_.end(), [&](double t) { return t <= now; });
  const size_t lo = static_cast<size_t>(first - times_.begin());
  const size_t hi = static_cast<size_t>(last - times_.begin());
  if (lo == hi) return 0.0;
  double sum = 0.0;
  for (size_t k = lo; k < hi; ++k) sum += values_[k];
  return sum / static_cast<double>(hi - lo);
}

// ---- routing (paper Alg. 1) -------------------------------------------------------

int bind_session(const std::vector<WorkerState>& decode_workers) {
  if (decode_workers.empty()) throw ConfigError("bind_session: no decode workers available");
  size_t best = 0;
  for (size_t i = 1; i < decode_workers.size(); ++i) {
    if (decode_workers[i].kv_bytes_used < decode_workers[best].kv_bytes_used) best = i;
  }
  return static_cast<int>(best);
}

namespace {

// Sum of the queued tasks' prefill times on `theta`, in queue order.
double queue_cost(const std::deque<PrefillTask>& q, const PerfProfile& profile, ParallelismStrategy theta) {
  double s = 0.0;
  for (const PrefillTask& t : q) s += t_prefill(profile, t.l_hist, t.l_incr, theta);
  return s;
}

}  // namespace

double estimate_local(const PrefillTask& task, const WorkerState& decode_worker, const PerfProfile& profile) {
  // the task's own prefill first, then each queued task added in order
  double c = t_prefill(profile, task.l_hist, task.l_incr, decode_worker.theta);
  for (const PrefillTask& t : decode_worker.prefill_queue) c += t_prefill(profile, t.l_hist, t.l_incr, decode_worker.theta);
  return c;
}

double estimate_remote(const PrefillTask& task, const WorkerState& prefill_worker, const WorkerState& decode_worker,
                       const PerfProfile& profile) {
  const double compute = t_prefill(profile, task.l_hist, task.l_incr, prefill_worker.theta);
  const double read_history = t_kv(profile, task.l_hist, decode_worker.theta, prefill_worker.theta);
  const double write_back = t_kv(profile, task.l_incr, prefill_worker.theta, decode_worker.theta);
  const double transfers = read_history + write_back;
  const double waiting = queue_cost(prefill_worker.prefill_queue, profile, prefill_worker.theta);
  return compute + transfers + waiting;
}


Coordinator::Coordinator(RoutingParams params, std::uint64_t seed) : params_(params), rng_(seed) {
  if (!(params_.alpha > 0.0 && params_.alpha <= 1.0)) throw ConfigError("routing: alpha must be in (0, 1]");
  if (!(params_.beta > 0.0 && params_.beta <= 1.0)) throw ConfigError("routing: beta must be in (0, 1]");
  if (!(params_.ttft_thres > 0.0) || !(params_.itl_thres > 0.0)) {
    throw ConfigError("routing: SLO thresholds must be > 0");
  }
}

RoutingDecision Coordinator::route(const PrefillTask& task, const WorkerState& bound_decode_worker,
                                   const std::vector<WorkerState>& prefill_workers, const PerfProfile& profile,
                                   double now) {
  RoutingDecision d;
  const size_t n = prefill_workers.size();
  if (n > 0) {
    // (i) scan the prefill workers in a fresh random order (Fisher-Yates,
    // one draw per position from the back) for TTFT slack
    std::vector<int> scan(n);
    std::iota(scan.begin(), scan.end(), 0);
    for (size_t i = n - 1; i > 0; --i) {
      const size_t j = static_cast<size_t>(rng_() % static_cast<std::uint64_t>(i + 1));
      std::swap(scan[i], scan[j]);
    }
    const double ttft_slack = params_.alpha * params_.ttft_thres;
    for (int w : scan) {
      if (prefill_workers[static_cast<size_t>(w)].ttft_stat.query(now) <= ttft_slack) {
        d.local = false;
        d.prefill_worker = w;
        d.rationale = RouteRationale::kSlackRemote;
        return d;
      }
    }
  }
  // (ii) ITL slack on the bound decode worker
  if (bound_decode_worker.itl_stat.query(now) <= params_.beta * params_.itl_thres) {
    d.local = true;
    d.rationale = RouteRationale::kSlackLocal;
    return d;
  }
  // (iii) cheapest estimate; ties keep local, then the lowest worker index
  d.local = true;
  d.rationale = RouteRationale::kArgmin;
  double best = estimate_local(task, bound_decode_worker, profile);
  for (size_t i = 0; i < n; ++i) {
    const double c = estimate_remote(task, prefill_workers[i], bound_decode_worker, profile);
    if (c < best) {
      best = c;
      d.local = false;
      d.prefill_worker = static_cast<int>(i);
    }
  }
  d.estimated_cost = best;
  return d;
}

// ---- reordering (paper Alg. 2) ---------------------------------------------------

namespace {

void require_permutation(size_t n, const std::vector<int>& order) {
  if (order.size() != n) throw DomainError("reorder: order and task list sizes differ");
  std::vector<char> seen(n, 0);
  for (int k : order) {
    if (k < 0 || static_cast<size_t>(k) >= n || seen[static_cast<size_t>(k)]) {
      throw DomainError("reorder: order is not a permutation");
    }
    seen[static_cast<size_t>(k)] = 1;
  }
}

// Satisfied tasks when the tasks with costs `cost` are served in `order`.
int satisfied_in_order(const std::vector<PrefillTask>& tasks, const std::vector<double>& cost, const int* order,
                       size_t m, double now, double ttft_thres) {
  int ok = 0;
  double done = 0.0;
  for (size_t k = 0; k < m; ++k) {
    const size_t t = static_cast<size_t>(order[k]);
    done += cost[t];
    if ((now - tasks[t].enqueue_time) + done <= ttft_thres) ++ok;
  }
  return ok;
}

// The rank-th permutation of 0..m-1 in lexicographic order.
void permutation_of_rank(int64_t rank, size_t m, int* out) {
  int pool[8];
  int64_t fact = 1;
  for (size_t i = 0; i < m; ++i) {
    pool[i] = static_cast<int>(i);
    if (i > 0) fact *= static_cast<int64_t>(i);
  }
  size_t left = m;
  for (size_t i = 0; i < m; ++i) {
    const int64_t q = rank / fact;
    rank %= fact;
    out[i] = pool[q];
    for (size_t j = static_cast<size_t>(q); j + 1 < left; ++j) pool[j] = pool[j + 1];
    --left;
    if (left > 0) fact /= static_cast<int64_t>(left);
  }
}

}  // namespace

std::vector<double> predict_completions(const std::vector<PrefillTask>& tasks, const std::vector<int>& order,
                                        const PerfProfile& profile, const ParallelismStrategy& theta) {
  require_permutation(tasks.size(), order);
  std::vector<double> out;
  out.reserve(order.size());
  double done = 0.0;
  for (int k : order) {
    const PrefillTask& t = tasks[static_cast<size_t>(k)];
    done += t_prefill(profile, t.l_hist, t.l_incr, theta);
    out.push_back(done);
  }
  return out;
}

int count_satisfied(const std::vector<PrefillTask>& tasks, const std::vector<int>& order, double now,
                    double ttft_thres, const PerfProfile& profile, const ParallelismStrategy& theta) {
  const std::vector<double> done = predict_completions(tasks, order, profile, theta);
  int ok = 0;
  for (size_t k = 0; k < order.size(); ++k) {
    if ((now - tasks[static_cast<size_t>(order[k])].enqueue_time) + done[k] <= ttft_thres) ++ok;
  }
  return ok;
}

ReorderOutcome reorder_and_dequeue(std::deque<PrefillTask>& queue, double now, const ReorderParams& params,
                                   const PerfProfile& profile, const ParallelismStrategy& theta) {
  if (queue.empty()) throw DomainError("reorder: queue is empty");
  if (params.window < 1) throw ConfigError("reorder: window must be >= 1");
  if (params.window > 8) throw ConfigError("reorder: window must be <= 8");
  if (!(params.ttft_thres > 0.0)) throw ConfigError("reorder: ttft_thres must be > 0");
  const size_t m = std::min(static_cast<size_t>(params.window), queue.size());
  std::vector<PrefillTask> head(queue.begin(), queue.begin() + static_cast<std::ptrdiff_t>(m));
  std::vector<double> cost(m);
  for (size_t k = 0; k < m; ++k) cost[k] = t_prefill(profile, head[k].l_hist, head[k].l_incr, theta);

  int64_t n_perm = 1;
  for (size_t k = 2; k <= m; ++k) n_perm *= static_cast<int64_t>(k);
  int best[8], cand[8];
  std::iota(best, best + m, 0);
  int best_ok = satisfied_in_order(head, cost, best, m, now, params.ttft_thres);
  for (int64_t rank = 1; rank < n_perm; ++rank) {
    permutation_of_rank(rank, m, cand);
    // a task postponed `window` times may not be moved back again
    bool allowed = true;
    for (size_t k = 0; k < m && allowed; ++k) {
      const size_t p = static_cast<size_t>(cand[k]);
      allowed = !(k > p && head[p].postpone_count >= params.window);
    }
    if (!allowed) continue;
    const int ok = satisfied_in_order(head, cost, cand, m, now, params.ttft_thres);
    if (ok > best_ok) {  // strict: ties keep the earlier (less shuffled) order
      best_ok = ok;
      std::copy(cand, cand + m, best);
    }
  }
  for (size_t k = 0; k < m; ++k) {
    if (k > static_cast<size_t>(best[k])) ++head[static_cast<size_t>(best[k])].postpone_count;
  }
  for (size_t k = 0; k < m; ++k) queue[k] = head[static_cast<size_t>(best[k])];
  ReorderOutcome out;
  out.chosen_order.assign(best, best + m);
  out.predicted_satisfied = best_ok;
  out.task = queue.front();
  queue.pop_front();
  return out;
}

}  // namespace pdsim
