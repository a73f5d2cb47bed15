// pdsim/planner.hpp — drop-in deployment plan type (reference
// proj/include/pdsim/planner.hpp:36-53) and the candidate enumeration of
// top_k (planner.cpp:582-657) exposed as a function.
#pragma once

#include <map>
#include <string>
#include <vector>

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

std::string format_plan(const DeploymentPlan& plan);  // "P:<TP=4, DP=2>, D:<TP=8, DP=1>"

}  // namespace pdsim
