// doc_io.cpp — JSON documents of the drop-in C++ API: perf_profile_v1,
// trace_v1, plan_v1 and coefficients_v1 (reference perf_model.hpp:143-146,
// workload.hpp:88-89, planner.hpp:108-113).
//
// Host document I/O (the files `pdsim profile / gen-trace / plan` write and
// the reference's suites round-trip), off the replay path. Layout and key
// order follow perf_model.cpp:279-433, workload.cpp:237-305 and
// planner.cpp:684-790 so documents are interchangeable with the reference:
// nlohmann dump(2) + newline, canonical (save(load(save(x))) == save(x)),
// loaders raise ParseError naming the offending path and validate the
// result (ConfigError -> ParseError).
#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "json.hpp"
#include "pdsim/errors.hpp"
#include "pdsim/perf_model.hpp"
#include "pdsim/planner.hpp"
#include "pdsim/workload.hpp"

namespace pdsim {

namespace {

using nlohmann::json;

constexpr const char* kProfileDoc = "perf_profile_v1";
constexpr const char* kTraceDoc = "trace_v1";
constexpr const char* kPlanDoc = "plan_v1";

json parse_document(const std::string& text, const char* where) {
  try {
    return json::parse(text);
  } catch (const json::parse_error& e) {
    throw ParseError(where, e.what());
  }
}

std::string require_version(const json& j, const char* expected) {
  if (!j.is_object() || !j.contains("version") || !j.at("version").is_string()) {
    throw ParseError("version", "missing version tag");
  }
  const std::string v = j.at("version").get<std::string>();
  if (v != expected) throw ParseError("version", "unknown version '" + v + "' (expected " + expected + ")");
  return v;
}

json curve_json(const PiecewiseAlphaBeta& c) {
  json segs = json::array();
  for (const AlphaBetaSegment& s : c.segments()) segs.push_back({{"alpha", s.alpha}, {"beta", s.beta}});
  json j;
  j["breakpoints"] = c.breakpoints();
  j["segments"] = std::move(segs);
  return j;
}

PiecewiseAlphaBeta curve_of(const json& j, const std::string& where) {
  if (!j.is_object() || !j.contains("breakpoints") || !j.contains("segments")) {
    throw ParseError(where, "expected object with breakpoints and segments");
  }
  std::vector<double> bps;
  for (const json& v : j.at("breakpoints")) {
    if (!v.is_number()) throw ParseError(where + ".breakpoints", "expected numbers");
    bps.push_back(v.get<double>());
  }
  std::vector<AlphaBetaSegment> segs;
  for (const json& v : j.at("segments")) {
    if (!v.is_object() || !v.contains("alpha") || !v.contains("beta")) {
      throw ParseError(where + ".segments[" + std::to_string(segs.size()) + "]", "expected object with alpha and beta");
    }
    segs.push_back({v.at("alpha").get<double>(), v.at("beta").get<double>()});
  }
  return PiecewiseAlphaBeta(std::move(bps), std::move(segs));
}

json counts_json(const std::map<int, int>& counts) {
  json a = json::array();
  for (const auto& [degree, n] : counts) a.push_back({{"degree", degree}, {"replicas", n}});
  return a;
}

std::map<int, int> counts_of(const json& j, const std::string& where) {
  if (!j.is_array()) throw ParseError(where, "expected an array");
  std::map<int, int> out;
  size_t k = 0;
  for (const json& e : j) {
    const std::string at = where + "[" + std::to_string(k++) + "]";
    if (!e.is_object() || !e.contains("degree") || !e.contains("replicas")) {
      throw ParseError(at, "expected object with degree and replicas");
    }
    const int degree = e.at("degree").get<int>();
    const int n = e.at("replicas").get<int>();
    if (degree < 1) throw ParseError(at + ".degree", "must be >= 1");
    if (n < 1) throw ParseError(at + ".replicas", "must be >= 1");
    if (!out.emplace(degree, n).second) throw ParseError(at + ".degree", "duplicate degree");
  }
  return out;
}

}  // namespace

// ---- perf_profile_v1 ---------------------------------------------------------

std::string save_profile(const PerfProfile& p) {
  json j;
  j["version"] = kProfileDoc;
  j["degrees"] = p.degrees;
  j["kv_bytes_per_token"] = p.kv_bytes_per_token;
  j["gpu_memory_capacity"] = p.gpu_memory_capacity;
  j["history_weight"] = p.history_weight;
  json pre = json::array(), dec = json::array(), kv = json::array();
  for (int d : p.degrees) {
    json a = curve_json(p.prefill_cost.at(d));
    a["degree"] = d;
    pre.push_back(std::move(a));
    json b = curve_json(p.decode_cost.at(d));
    b["degree"] = d;
    dec.push_back(std::move(b));
  }
  for (int s : p.degrees) {
    for (int d : p.degrees) {
      json c = curve_json(p.kv_cost.at({s, d}));
      c["src"] = s;
      c["dst"] = d;
      kv.push_back(std::move(c));
    }
  }
  j["prefill_cost"] = std::move(pre);
  j["decode_cost"] = std::move(dec);
  j["kv_cost"] = std::move(kv);
  return j.dump(2) + "\n";
}

PerfProfile load_profile(const std::string& text) {
  const json j = parse_document(text, "document");
  if (!j.is_object()) throw ParseError("document", "expected a JSON object");
  require_version(j, kProfileDoc);
  PerfProfile p;
  try {
    p.degrees = j.at("degrees").get<std::vector<int>>();
    p.kv_bytes_per_token = j.at("kv_bytes_per_token").get<std::int64_t>();
    p.gpu_memory_capacity = j.at("gpu_memory_capacity").get<std::int64_t>();
    p.history_weight = j.at("history_weight").get<double>();
  } catch (const json::exception& e) {
    throw ParseError("document", e.what());
  }
  for (const auto& [key, table] : {std::make_pair("prefill_cost", &p.prefill_cost),
                                   std::make_pair("decode_cost", &p.decode_cost)}) {
    if (!j.contains(key) || !j.at(key).is_array()) throw ParseError(key, "expected an array of per-degree curves");
    size_t k = 0;
    for (const json& e : j.at(key)) {
      const std::string at = std::string(key) + "[" + std::to_string(k++) + "]";
      if (!e.contains("degree")) throw ParseError(at, "missing degree");
      const int degree = e.at("degree").get<int>();
      if (!table->emplace(degree, curve_of(e, at)).second) throw ParseError(at, "duplicate degree " + std::to_string(degree));
    }
  }
  if (!j.contains("kv_cost") || !j.at("kv_cost").is_array()) {
    throw ParseError("kv_cost", "expected an array of per-pair curves");
  }
  size_t k = 0;
  for (const json& e : j.at("kv_cost")) {
    const std::string at = "kv_cost[" + std::to_string(k++) + "]";
    if (!e.contains("src") || !e.contains("dst")) throw ParseError(at, "missing src/dst degrees");
    const int s = e.at("src").get<int>(), d = e.at("dst").get<int>();
    if (!p.kv_cost.emplace(std::make_pair(s, d), curve_of(e, at)).second) {
      throw ParseError(at, "duplicate pair (" + std::to_string(s) + ", " + std::to_string(d) + ")");
    }
  }
  try {
    p.validate();
  } catch (const ConfigError& e) {
    throw ParseError("validation", e.what());
  }
  return p;
}

// ---- trace_v1 ----------------------------------------------------------------

std::string save_trace(const Trace& t) {
  json sessions = json::array();
  for (const SessionSpec& s : t.sessions) {
    json rounds = json::array();
    for (const Round& r : s.rounds) {
      rounds.push_back({{"incr_input_len", r.incr_input_len}, {"decode_len", r.decode_len},
                        {"interaction_delay", r.interaction_delay}});
    }
    sessions.push_back({{"session_id", s.session_id}, {"arrival_time", s.arrival_time}, {"rounds", std::move(rounds)}});
  }
  json j;
  j["version"] = kTraceDoc;
  j["name"] = t.name;
  j["slo"] = {{"ttft_thres", t.slo.ttft_thres}, {"itl_thres", t.slo.itl_thres}};
  j["sessions"] = std::move(sessions);
  return j.dump(2) + "\n";
}

Trace load_trace(const std::string& text) {
  const json j = parse_document(text, "document");
  require_version(j, kTraceDoc);
  Trace t;
  try {
    t.name = j.at("name").get<std::string>();
    t.slo.ttft_thres = j.at("slo").at("ttft_thres").get<double>();
    t.slo.itl_thres = j.at("slo").at("itl_thres").get<double>();
    for (const json& js : j.at("sessions")) {
      SessionSpec s;
      s.session_id = js.at("session_id").get<std::int64_t>();
      s.arrival_time = js.at("arrival_time").get<double>();
      for (const json& jr : js.at("rounds")) {
        s.rounds.push_back(Round{jr.at("incr_input_len").get<TokenCount>(), jr.at("decode_len").get<TokenCount>(),
                                 jr.at("interaction_delay").get<double>()});
      }
      t.sessions.push_back(std::move(s));
    }
  } catch (const json::exception& e) {
    throw ParseError("document", e.what());
  }
  try {
    t.validate();
  } catch (const ConfigError& e) {
    throw ParseError("validate", e.what());
  }
  return t;
}

// ---- plan_v1 / coefficients_v1 ---------------------------------------------------

std::string plan_to_json(const DeploymentPlan& plan) {
  json j;
  j["version"] = kPlanDoc;
  j["feasible"] = plan.feasible;
  j["objective_z"] = plan.objective_z;
  j["gpus_used"] = plan.gpus_used;
  j["x"] = counts_json(plan.x);
  j["y"] = counts_json(plan.y);
  return j.dump(2) + "\n";
}

DeploymentPlan plan_from_json(const std::string& text) {
  const json j = parse_document(text, "plan");
  if (!j.is_object()) throw ParseError("plan", "expected a JSON object");
  if (!j.contains("version") || j.at("version") != kPlanDoc) {
    throw ParseError("plan.version", std::string("expected \"") + kPlanDoc + "\"");
  }
  for (const char* key : {"feasible", "objective_z", "gpus_used", "x", "y"}) {
    if (!j.contains(key)) throw ParseError(std::string("plan.") + key, "missing field");
  }
  DeploymentPlan plan;
  plan.feasible = j.at("feasible").get<bool>();
  plan.objective_z = j.at("objective_z").get<double>();
  plan.gpus_used = j.at("gpus_used").get<int>();
  plan.x = counts_of(j.at("x"), "plan.x");
  plan.y = counts_of(j.at("y"), "plan.y");
  try {
    plan.validate("plan");
  } catch (const ConfigError& e) {
    throw ParseError("plan", e.what());
  }
  return plan;
}

std::string coefficients_to_json(const LatencyCoefficients& c) {
  auto taus = [](const std::map<int, double>& tau) {
    json a = json::array();
    for (const auto& [degree, seconds] : tau) a.push_back({{"degree", degree}, {"seconds", seconds}});
    return a;
  };
  json j;
  j["version"] = "coefficients_v1";
  j["provenance"] = c.provenance;
  j["tau_pre"] = taus(c.tau_pre);
  j["tau_dec"] = taus(c.tau_dec);
  j["infeasible_pre"] = c.infeasible_pre;
  j["infeasible_dec"] = c.infeasible_dec;
  return j.dump(2) + "\n";
}

}  // namespace pdsim
