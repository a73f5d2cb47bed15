// pdsim/planner.hpp — drop-in deployment plan type (reference
// proj/include/pdsim/planner.hpp:36-53), the candidate enumeration of
// top_k (planner.cpp:582-657) exposed as a function, and the reference's
// surrogate planner (planner.hpp:55-113): phase simulations and coefficient
// estimation run on the GPU, solve/top_k on the host.
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "pdsim/perf_model.hpp"
#include "pdsim/workload.hpp"

namespace pdsim {

struct DeploymentPlan {
  std::map<int, int> x;  // prefill replicas per degree
  std::map<int, int> y;  // decode replicas per degree
  double objective_z = 0.0;
  int gpus_used = 0;
  bool feasible = false;

  int prefill_replicas() const;
  int decode_replicas() const;
  int gpus() const;
  void validate(const std::string& where, int total_gpus = -1) const;  // throws ConfigError
};

bool operator==(const DeploymentPlan& a, const DeploymentPlan& b);

// Every (x, y) map with x, y non-empty and sum(degree*count) <= total_gpus,
// in the reference enumeration order (feasible = true, gpus_used set).
std::vector<DeploymentPlan> enumerate_plans(const std::vector<int>& degrees, int total_gpus);

// planner.hpp:55-66.
struct LatencyCoefficients {
  std::map<int, double> tau_pre;  // feasible degrees only, seconds
  std::map<int, double> tau_dec;
  std::set<int> infeasible_pre;
  std::set<int> infeasible_dec;
  std::string provenance;
};

struct PhaseSimResult {
  double p95 = 0.0;
  bool infeasible = false;
  std::int64_t sample_count = 0;
};

// planner.hpp:68-90 (GPU phase sims; throw ConfigError / DomainError as the
// reference does).
PhaseSimResult simulate_prefill_replica(const Trace& trace, const PerfProfile& profile, int degree);
PhaseSimResult simulate_decode_replica(const Trace& trace, const PerfProfile& profile, int degree);
LatencyCoefficients estimate_coefficients(const TraceStats& stats, double rate, const PerfProfile& profile,
                                          const std::vector<int>& degrees, int total_gpus, std::uint64_t seed);
// Batched form (no reference counterpart): one device launch for every
// (rates[s], seeds[s]) setting; throws on the first setting that would throw.
std::vector<LatencyCoefficients> estimate_coefficients_batch(const TraceStats& stats, const std::vector<double>& rates,
                                                             const std::vector<std::uint64_t>& seeds,
                                                             const PerfProfile& profile,
                                                             const std::vector<int>& degrees, int total_gpus);
// planner.hpp:92-108 (host).
DeploymentPlan solve(const LatencyCoefficients& coeffs, int total_gpus, const std::vector<int>& degrees);
std::vector<DeploymentPlan> top_k(const LatencyCoefficients& coeffs, int total_gpus, const std::vector<int>& degrees,
                                  int k);

std::string format_plan(const DeploymentPlan& plan);  // "P:<TP=4, DP=2>, D:<TP=8, DP=1>"

// plan_v1 JSON (planner.hpp:108-113). Canonical: plan_to_json(plan_from_json(
// plan_to_json(p))) == plan_to_json(p). plan_from_json throws ParseError.
std::string plan_to_json(const DeploymentPlan& plan);
DeploymentPlan plan_from_json(const std::string& text);
std::string coefficients_to_json(const LatencyCoefficients& coeffs);

}  // namespace pdsim
