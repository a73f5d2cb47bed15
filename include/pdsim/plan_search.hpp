// pdsim/plan_search.hpp — the batched replay search (new; the reference has
// no batched API — its "batch" is the serial sweep loop, pdsim.cpp:547-586):
// every candidate x replica pair replayed on the GPU, SLO attainment scored
// per pair, argmax over candidates (max total slo_ok, ties -> smallest index).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "pdsim/metrics.hpp"
#include "pdsim/perf_model.hpp"
#include "pdsim/planner.hpp"
#include "pdsim/sim_engine.hpp"
#include "pdsim/workload.hpp"

namespace pdsim {

struct PairAttainment {
  std::int64_t sessions_total = 0;
  std::int64_t sessions_completed = 0;
  std::int64_t slo_ok = 0;
  std::int64_t ttft_ok = 0;
  std::int64_t itl_ok = 0;
  bool valid = true;  // false: run() would throw ConfigError (e.g. KV precheck)
};

struct SearchOptions {
  int device = -1;             // -1: $PDSIM_DEVICE or 0
  std::int64_t pair_begin = 0;  // shard [pair_begin, pair_end) of c * replicas + r
  std::int64_t pair_end = -1;
  bool report = false;  // per-pair build_report on the device (SearchResult::reports)
  // Argmax-only search (PDSIM_SEARCH_ARGMAX): candidates that provably cannot
  // win stop early; best_candidate / best_slo_ok are unchanged, pruned
  // candidates get candidate_slo_ok = -2 and pairs valid = false.
  bool prune = false;
  // Several GPUs of this process (pdsim_multi_plan_search): the whole search
  // is sharded over `devices` (cost-aware LPT split) and the per-candidate
  // counts all-reduced over NCCL; outputs as for one device. Needs the whole
  // pair range and no reports. Empty: one device (`device`).
  std::vector<int> devices;
};

struct SearchResult {
  int best_candidate = -1;  // argmax; -1 when no candidate is valid
  std::int64_t best_slo_ok = -1;
  std::vector<std::int64_t> candidate_slo_ok;  // -1 marks an invalid candidate
  std::vector<PairAttainment> pairs;
  double kernel_ms = 0.0;
  double device_ms = 0.0;
  std::vector<Report> reports;  // per pair, when SearchOptions::report
};

SearchResult plan_search(const std::vector<Trace>& replicas, const std::vector<DeploymentPlan>& candidates,
                         const PerfProfile& profile, const SchedulerParams& params, std::uint64_t engine_seed,
                         const SearchOptions& options = {});

// Batched `pdsim sweep` (pdsim.cpp:501-590): `plan` replayed on each trace
// (the sweep generates one trace per arrival rate) under every scheduler
// setting, all pairs in one GPU call. Returns build_report of each replay,
// indexed [setting * traces.size() + trace]. Every setting is validated
// first (ConfigError, like the reference's first failing combination).
std::vector<Report> sweep(const std::vector<Trace>& traces, const DeploymentPlan& plan, const PerfProfile& profile,
                          const std::vector<SchedulerParams>& settings, std::uint64_t seed,
                          const SearchOptions& options = {});

// The reference's sweep.csv text (pdsim.cpp:541-586): one row per (rate,
// setting) in rate-major order, numbers in std::to_chars form. `reports` as
// returned by sweep() for traces generated at `rates` (same order).
std::string sweep_csv(const std::vector<double>& rates, const std::vector<SchedulerParams>& settings,
                      const std::vector<Report>& reports);

}  // namespace pdsim
