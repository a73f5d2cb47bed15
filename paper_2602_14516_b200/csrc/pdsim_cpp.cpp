// pdsim_cpp.cpp — the reference's C++ API (include/pdsim/*.hpp) implemented
// over the C-ABI (include/pdsim_gpu.h). Host code stays C++; every replay
// goes to the GPU through pdsim_gpu_run / pdsim_gpu_plan_search. Compiled into
// libpdsim_gpu.so with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pdsim/errors.hpp"
#include "pdsim/metrics.hpp"
#include "pdsim/perf_model.hpp"
#include "pdsim/plan_search.hpp"
#include "pdsim/planner.hpp"
#include "pdsim/sim_engine.hpp"
#include "pdsim/workload.hpp"
#include "pdsim_gpu.h"

namespace pdsim {
namespace {

[[noreturn]] void raise(int code, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (code) {
    case PDSIM_ERR_CONFIG: throw ConfigError(m);
    case PDSIM_ERR_DOMAIN: throw DomainError(m);
    case PDSIM_ERR_PARSE: throw ParseError("document", m);
    default: throw DeviceError(m);
  }
}

void check(int rc) {
  if (rc != PDSIM_OK) raise(rc, pdsim_last_error());
}

void check_ctx(int rc, pdsim_gpu_ctx* ctx) {
  if (rc != PDSIM_OK) raise(rc, pdsim_gpu_last_error(ctx));
}

int default_device() {
  const char* e = std::getenv("PDSIM_DEVICE");
  return e ? std::atoi(e) : 0;
}

// One context per (thread, device), created lazily.
pdsim_gpu_ctx* context(int device) {
  struct Holder {
    std::vector<std::pair<int, pdsim_gpu_ctx*>> ctxs;
    ~Holder() {
      for (auto& c : ctxs) pdsim_gpu_destroy(c.second);
    }
  };
  thread_local Holder h;
  for (auto& c : h.ctxs)
    if (c.first == device) return c.second;
  pdsim_gpu_ctx* ctx = nullptr;
  check(pdsim_gpu_create(device, &ctx));
  h.ctxs.emplace_back(device, ctx);
  return ctx;
}

pdsim_curve curve_to_pod(const PiecewiseAlphaBeta& c) {
  if (c.breakpoints().size() > PDSIM_MAX_BREAKPOINTS || c.segments().size() != c.breakpoints().size() + 1) {
    throw ConfigError("cost curve exceeds the engine's " + std::to_string(PDSIM_MAX_BREAKPOINTS) +
                      "-breakpoint layout or is malformed");
  }
  pdsim_curve out;
  std::memset(&out, 0, sizeof(out));
  out.n_breakpoints = static_cast<int32_t>(c.breakpoints().size());
  for (size_t i = 0; i < c.breakpoints().size(); ++i) out.breakpoints[i] = c.breakpoints()[i];
  for (size_t i = 0; i < c.segments().size(); ++i) {
    out.alpha[i] = c.segments()[i].alpha;
    out.beta[i] = c.segments()[i].beta;
  }
  return out;
}

PiecewiseAlphaBeta curve_from_pod(const pdsim_curve& c) {
  std::vector<double> bps(c.breakpoints, c.breakpoints + c.n_breakpoints);
  std::vector<AlphaBetaSegment> segs;
  for (int i = 0; i <= c.n_breakpoints; ++i) segs.push_back({c.alpha[i], c.beta[i]});
  return PiecewiseAlphaBeta(bps, segs);
}

void profile_to_pod(const PerfProfile& p, pdsim_profile* out) {
  std::memset(out, 0, sizeof(*out));
  if (p.degrees.size() > PDSIM_MAX_DEGREES) throw ConfigError("degrees: more than 8 parallelism degrees");
  out->n_degrees = static_cast<int32_t>(p.degrees.size());
  for (size_t i = 0; i < p.degrees.size(); ++i) {
    const int d = p.degrees[i];
    out->degrees[i] = d;
    auto pit = p.prefill_cost.find(d);
    auto dit = p.decode_cost.find(d);
    if (pit == p.prefill_cost.end()) throw ConfigError("prefill_cost: missing entry for degree " + std::to_string(d));
    if (dit == p.decode_cost.end()) throw ConfigError("decode_cost: missing entry for degree " + std::to_string(d));
    out->prefill[i] = curve_to_pod(pit->second);
    out->decode[i] = curve_to_pod(dit->second);
    for (size_t j = 0; j < p.degrees.size(); ++j) {
      auto kit = p.kv_cost.find({d, p.degrees[j]});
      if (kit == p.kv_cost.end()) {
        throw ConfigError("kv_cost: missing entry for pair (" + std::to_string(d) + ", " +
                          std::to_string(p.degrees[j]) + ")");
      }
      out->kv[i][j] = curve_to_pod(kit->second);
    }
  }
  if (p.prefill_cost.size() != p.degrees.size() || p.decode_cost.size() != p.degrees.size() ||
      p.kv_cost.size() != p.degrees.size() * p.degrees.size()) {
    throw ConfigError("cost tables contain entries for unknown degrees");
  }
  out->kv_bytes_per_token = p.kv_bytes_per_token;
  out->gpu_memory_capacity = p.gpu_memory_capacity;
  out->history_weight = p.history_weight;
}

PerfProfile profile_from_pod(const pdsim_profile& p) {
  PerfProfile out;
  out.degrees.assign(p.degrees, p.degrees + p.n_degrees);
  out.kv_bytes_per_token = p.kv_bytes_per_token;
  out.gpu_memory_capacity = p.gpu_memory_capacity;
  out.history_weight = p.history_weight;
  for (int i = 0; i < p.n_degrees; ++i) {
    out.prefill_cost.emplace(p.degrees[i], curve_from_pod(p.prefill[i]));
    out.decode_cost.emplace(p.degrees[i], curve_from_pod(p.decode[i]));
    for (int j = 0; j < p.n_degrees; ++j) {
      out.kv_cost.emplace(std::make_pair(p.degrees[i], p.degrees[j]), curve_from_pod(p.kv[i][j]));
    }
  }
  return out;
}

// SoA view of a Trace (arrays owned by this object).
struct TraceArrays {
  std::vector<int64_t> sid, off, incr, dec;
  std::vector<double> arr, delay;
  pdsim_trace view{};
  explicit TraceArrays(const Trace& t) {
    off.push_back(0);
    for (const SessionSpec& s : t.sessions) {
      sid.push_back(s.session_id);
      arr.push_back(s.arrival_time);
      for (const Round& r : s.rounds) {
        incr.push_back(r.incr_input_len);
        dec.push_back(r.decode_len);
        delay.push_back(r.interaction_delay);
      }
      off.push_back(static_cast<int64_t>(incr.size()));
    }
    view.n_sessions = static_cast<int64_t>(sid.size());
    view.n_rounds = static_cast<int64_t>(incr.size());
    view.session_id = sid.data();
    view.arrival_time = arr.data();
    view.round_offset = off.data();
    view.incr_input_len = incr.data();
    view.decode_len = dec.data();
    view.interaction_delay = delay.data();
    view.ttft_thres = t.slo.ttft_thres;
    view.itl_thres = t.slo.itl_thres;
  }
};

pdsim_plan plan_to_pod(const DeploymentPlan& p) {
  pdsim_plan out;
  std::memset(&out, 0, sizeof(out));
  if (p.x.size() > PDSIM_MAX_GROUPS || p.y.size() > PDSIM_MAX_GROUPS) {
    throw ConfigError("plan: more than 8 degree groups per phase");
  }
  for (const auto& [d, c] : p.x) {
    out.prefill_degree[out.n_prefill_groups] = d;
    out.prefill_count[out.n_prefill_groups++] = c;
  }
  for (const auto& [d, c] : p.y) {
    out.decode_degree[out.n_decode_groups] = d;
    out.decode_count[out.n_decode_groups++] = c;
  }
  return out;
}

pdsim_sched_params params_to_pod(const SchedulerParams& s) {
  pdsim_sched_params p;
  std::memset(&p, 0, sizeof(p));
  p.routing = static_cast<int32_t>(s.routing);
  p.reorder = s.reorder ? 1 : 0;
  p.alpha = s.alpha;
  p.beta = s.beta;
  p.window = s.window;
  p.stat_window = s.stat_window;
  return p;
}

bool all_within(const std::vector<double>& v, double limit) {
  for (double x : v)
    if (x > limit) return false;
  return true;
}

}  // namespace

// ---- perf_model (perf_model.cpp:43-205) ----
double PiecewiseAlphaBeta::eval(double load) const {
  size_t i = 0;
  while (i < breakpoints_.size() && !(load < breakpoints_[i])) ++i;
  const AlphaBetaSegment& s = segments_[i];
  return s.alpha + s.beta * load;
}

void PiecewiseAlphaBeta::validate(const std::string& where) const {
  if (segments_.empty()) throw ConfigError(where + ": at least one segment required");
  if (segments_.size() != breakpoints_.size() + 1) {
    throw ConfigError(where + ": expected " + std::to_string(breakpoints_.size() + 1) + " segments for " +
                      std::to_string(breakpoints_.size()) + " breakpoints, got " + std::to_string(segments_.size()));
  }
  for (size_t i = 0; i + 1 < breakpoints_.size(); ++i) {
    if (!(breakpoints_[i] < breakpoints_[i + 1])) {
      throw ConfigError(where + ".breakpoints[" + std::to_string(i + 1) + "]: breakpoints must be strictly ascending");
    }
  }
  for (size_t i = 0; i < segments_.size(); ++i) {
    const AlphaBetaSegment& s = segments_[i];
    const std::string a = where + ".segments[" + std::to_string(i) + "]";
    if (!(s.alpha >= 0.0) || !std::isfinite(s.alpha)) throw ConfigError(a + ".alpha: must be finite and >= 0");
    if (!(s.beta >= 0.0) || !std::isfinite(s.beta)) throw ConfigError(a + ".beta: must be finite and >= 0");
    if (s.alpha == 0.0 && s.beta == 0.0) throw ConfigError(a + ": degenerate segment (alpha and beta both 0)");
  }
  for (size_t i = 0; i < breakpoints_.size(); ++i) {
    const double bp = breakpoints_[i];
    const double left = segments_[i].alpha + segments_[i].beta * bp;
    const double right = segments_[i + 1].alpha + segments_[i + 1].beta * bp;
    if (right + 1e-9 * std::max(1.0, std::abs(left)) < left) {
      throw ConfigError(where + ".breakpoints[" + std::to_string(i) + "]: non-monotone transition");
    }
  }
}

bool PerfProfile::has_degree(int degree) const {
  return std::find(degrees.begin(), degrees.end(), degree) != degrees.end();
}

void PerfProfile::validate() const {
  pdsim_profile pod;
  profile_to_pod(*this, &pod);
  check(pdsim_profile_validate(&pod));
}

double t_prefill(const PerfProfile& profile, TokenCount l_hist, TokenCount l_incr, ParallelismStrategy theta) {
  if (l_incr < 1) throw DomainError("t_prefill: l_incr must be >= 1 (a prefill task has non-empty input)");
  if (l_hist < 0) throw DomainError("t_prefill: l_hist must be >= 0");
  auto it = profile.prefill_cost.find(theta.degree);
  if (it == profile.prefill_cost.end()) throw DomainError("t_prefill: unknown degree " + std::to_string(theta.degree));
  const double load = static_cast<double>(l_incr) + profile.history_weight * static_cast<double>(l_hist);
  return it->second.eval(load);
}

double t_decode(const PerfProfile& profile, int batch_size, ParallelismStrategy theta) {
  if (batch_size < 1) throw DomainError("t_decode: batch_size must be >= 1");
  auto it = profile.decode_cost.find(theta.degree);
  if (it == profile.decode_cost.end()) throw DomainError("t_decode: unknown degree " + std::to_string(theta.degree));
  return it->second.eval(static_cast<double>(batch_size));
}

double t_kv(const PerfProfile& profile, TokenCount l_ctx, ParallelismStrategy src, ParallelismStrategy dst) {
  if (l_ctx < 0) throw DomainError("t_kv: l_ctx must be >= 0");
  auto it = profile.kv_cost.find({src.degree, dst.degree});
  if (it == profile.kv_cost.end()) {
    throw DomainError("t_kv: unknown degree pair (" + std::to_string(src.degree) + ", " +
                      std::to_string(dst.degree) + ")");
  }
  if (l_ctx == 0) return 0.0;
  return it->second.eval(static_cast<double>(l_ctx));
}

PerfProfile synth_profile(const SynthProfileSpec& spec, std::uint64_t seed) {
  pdsim_synth_spec s;
  std::memset(&s, 0, sizeof(s));
  if (spec.degrees.size() > PDSIM_MAX_DEGREES || spec.prefill_breakpoints.size() > PDSIM_MAX_BREAKPOINTS ||
      spec.decode_breakpoints.size() > PDSIM_MAX_BREAKPOINTS) {
    throw ConfigError("synth_profile: spec exceeds the C-ABI table sizes");
  }
  s.n_degrees = static_cast<int32_t>(spec.degrees.size());
  for (size_t i = 0; i < spec.degrees.size(); ++i) s.degrees[i] = spec.degrees[i];
  s.prefill_alpha_min = spec.prefill_alpha_min;
  s.prefill_alpha_max = spec.prefill_alpha_max;
  s.prefill_beta_min = spec.prefill_beta_min;
  s.prefill_beta_max = spec.prefill_beta_max;
  s.n_prefill_breakpoints = static_cast<int32_t>(spec.prefill_breakpoints.size());
  for (size_t i = 0; i < spec.prefill_breakpoints.size(); ++i) s.prefill_breakpoints[i] = spec.prefill_breakpoints[i];
  s.decode_alpha_min = spec.decode_alpha_min;
  s.decode_alpha_max = spec.decode_alpha_max;
  s.decode_beta_min = spec.decode_beta_min;
  s.decode_beta_max = spec.decode_beta_max;
  s.n_decode_breakpoints = static_cast<int32_t>(spec.decode_breakpoints.size());
  for (size_t i = 0; i < spec.decode_breakpoints.size(); ++i) s.decode_breakpoints[i] = spec.decode_breakpoints[i];
  s.segment_growth_min = spec.segment_growth_min;
  s.segment_growth_max = spec.segment_growth_max;
  s.scaling_exponent = spec.scaling_exponent;
  s.kv_bandwidth_bytes_per_sec = spec.kv_bandwidth_bytes_per_sec;
  s.kv_latency_seconds = spec.kv_latency_seconds;
  s.kv_reshard_penalty = spec.kv_reshard_penalty;
  s.kv_bytes_per_token = spec.kv_bytes_per_token;
  s.gpu_memory_capacity = spec.gpu_memory_capacity;
  s.history_weight = spec.history_weight;
  pdsim_profile out;
  check(pdsim_synth_profile(&s, seed, &out));
  return profile_from_pod(out);
}

// ---- workload ----
TokenCount SessionSpec::total_prefill() const {
  TokenCount t = 0;
  for (const Round& r : rounds) t += r.incr_input_len;
  return t;
}

TokenCount SessionSpec::total_decode() const {
  TokenCount t = 0;
  for (const Round& r : rounds) t += r.decode_len;
  return t;
}

void Trace::validate() const {
  TraceArrays a(*this);
  check(pdsim_trace_validate(&a.view));
}

TraceStats preset_stats(const std::string& name) {
  pdsim_trace_stats s;
  check(pdsim_preset_stats(name.c_str(), &s));
  TraceStats out;
  out.name = name;
  out.mean_rounds = s.mean_rounds;
  out.fixed_rounds = s.fixed_rounds != 0;
  out.mean_prefill_len = s.mean_prefill_len;
  out.mean_decode_len = s.mean_decode_len;
  out.length_cv = s.length_cv;
  out.first_round_fraction = s.first_round_fraction;
  out.mean_interaction_delay = s.mean_interaction_delay;
  out.slo = {s.ttft_thres, s.itl_thres};
  return out;
}

Trace gen_trace(const TraceStats& stats, double arrival_rate, int num_sessions, std::uint64_t seed) {
  pdsim_trace_stats s;
  std::memset(&s, 0, sizeof(s));
  s.mean_rounds = stats.mean_rounds;
  s.fixed_rounds = stats.fixed_rounds ? 1 : 0;
  s.mean_prefill_len = stats.mean_prefill_len;
  s.mean_decode_len = stats.mean_decode_len;
  s.length_cv = stats.length_cv;
  s.first_round_fraction = stats.first_round_fraction;
  s.mean_interaction_delay = stats.mean_interaction_delay;
  s.ttft_thres = stats.slo.ttft_thres;
  s.itl_thres = stats.slo.itl_thres;
  pdsim_trace_buf* buf = nullptr;
  check(pdsim_gen_trace(&s, arrival_rate, num_sessions, seed, &buf));
  std::unique_ptr<pdsim_trace_buf, void (*)(pdsim_trace_buf*)> owner(buf, pdsim_trace_buf_free);
  pdsim_trace v;
  check(pdsim_trace_buf_view(buf, &v));
  Trace t;
  t.name = stats.name;
  t.slo = stats.slo;
  t.sessions.resize(static_cast<size_t>(v.n_sessions));
  for (int64_t i = 0; i < v.n_sessions; ++i) {
    SessionSpec& s2 = t.sessions[static_cast<size_t>(i)];
    s2.session_id = v.session_id[i];
    s2.arrival_time = v.arrival_time[i];
    for (int64_t r = v.round_offset[i]; r < v.round_offset[i + 1]; ++r) {
      s2.rounds.push_back({v.incr_input_len[r], v.decode_len[r], v.interaction_delay[r]});
    }
  }
  return t;
}

// ---- planner ----
int DeploymentPlan::prefill_replicas() const {
  int t = 0;
  for (const auto& [d, c] : x) t += c;
  return t;
}
int DeploymentPlan::decode_replicas() const {
  int t = 0;
  for (const auto& [d, c] : y) t += c;
  return t;
}
int DeploymentPlan::gpus() const {
  int t = 0;
  for (const auto& [d, c] : x) t += d * c;
  for (const auto& [d, c] : y) t += d * c;
  return t;
}
void DeploymentPlan::validate(const std::string& where, int total_gpus) const {
  for (const auto& [d, c] : x)
    if (d < 1 || c < 1) throw ConfigError(where + ": x entries need degree >= 1 and count >= 1");
  for (const auto& [d, c] : y)
    if (d < 1 || c < 1) throw ConfigError(where + ": y entries need degree >= 1 and count >= 1");
  if (gpus_used != gpus()) throw ConfigError(where + ": gpus_used does not match replica totals");
  if (total_gpus >= 0 && gpus() > total_gpus) throw ConfigError(where + ": plan exceeds the GPU budget");
}
bool operator==(const DeploymentPlan& a, const DeploymentPlan& b) {
  return a.x == b.x && a.y == b.y && a.objective_z == b.objective_z && a.gpus_used == b.gpus_used &&
         a.feasible == b.feasible;
}

std::vector<DeploymentPlan> enumerate_plans(const std::vector<int>& degrees, int total_gpus) {
  std::vector<int32_t> ds(degrees.begin(), degrees.end());
  const int64_t n = pdsim_enumerate_plans(ds.data(), static_cast<int32_t>(ds.size()), total_gpus, nullptr, 0);
  if (n < 0) throw ConfigError("planner: degrees must be >= 1");
  std::vector<pdsim_plan> pods(static_cast<size_t>(n));
  pdsim_enumerate_plans(ds.data(), static_cast<int32_t>(ds.size()), total_gpus, pods.data(), n);
  std::vector<DeploymentPlan> out;
  for (const pdsim_plan& p : pods) {
    DeploymentPlan d;
    for (int i = 0; i < p.n_prefill_groups; ++i) d.x[p.prefill_degree[i]] = p.prefill_count[i];
    for (int i = 0; i < p.n_decode_groups; ++i) d.y[p.decode_degree[i]] = p.decode_count[i];
    d.gpus_used = d.gpus();
    d.feasible = true;
    out.push_back(d);
  }
  return out;
}

namespace {

pdsim_trace_stats stats_to_pod(const TraceStats& stats) {
  pdsim_trace_stats s;
  std::memset(&s, 0, sizeof(s));
  s.mean_rounds = stats.mean_rounds;
  s.fixed_rounds = stats.fixed_rounds ? 1 : 0;
  s.mean_prefill_len = stats.mean_prefill_len;
  s.mean_decode_len = stats.mean_decode_len;
  s.length_cv = stats.length_cv;
  s.first_round_fraction = stats.first_round_fraction;
  s.mean_interaction_delay = stats.mean_interaction_delay;
  s.ttft_thres = stats.slo.ttft_thres;
  s.itl_thres = stats.slo.itl_thres;
  return s;
}

// Only the listed degrees enter the table (the reference's check_coefficients
// requires each of them to be known).
pdsim_coefficients coeffs_to_pod(const LatencyCoefficients& c, const std::vector<int>& degrees) {
  std::vector<int> ts = degrees;
  std::sort(ts.begin(), ts.end());
  ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
  if (ts.empty() || ts.front() < 1) throw ConfigError("planner: degrees must be >= 1");
  if (ts.size() > PDSIM_MAX_DEGREES) throw ConfigError("planner: too many degrees");
  pdsim_coefficients p;
  std::memset(&p, 0, sizeof(p));
  p.n_degrees = static_cast<int32_t>(ts.size());
  for (size_t k = 0; k < ts.size(); ++k) {
    const int n = ts[k];
    p.degrees[k] = n;
    const bool pre = c.tau_pre.count(n) != 0, dec = c.tau_dec.count(n) != 0;
    if ((!pre && !c.infeasible_pre.count(n)) || (!dec && !c.infeasible_dec.count(n))) {
      throw ConfigError("planner: no coefficient for degree " + std::to_string(n));
    }
    p.infeasible_pre[k] = pre ? 0 : 1;
    p.infeasible_dec[k] = dec ? 0 : 1;
    p.tau_pre[k] = pre ? c.tau_pre.at(n) : 0.0;
    p.tau_dec[k] = dec ? c.tau_dec.at(n) : 0.0;
  }
  return p;
}

DeploymentPlan plan_from_pod(const pdsim_plan& p, double z, int gpus) {
  DeploymentPlan d;
  for (int i = 0; i < p.n_prefill_groups; ++i) d.x[p.prefill_degree[i]] = p.prefill_count[i];
  for (int i = 0; i < p.n_decode_groups; ++i) d.y[p.decode_degree[i]] = p.decode_count[i];
  d.objective_z = z;
  d.gpus_used = gpus;
  d.feasible = true;
  return d;
}

PhaseSimResult phase(const Trace& trace, const PerfProfile& profile, int degree, bool prefill) {
  profile.validate();
  TraceArrays ta(trace);
  pdsim_profile prof;
  profile_to_pod(profile, &prof);
  pdsim_gpu_ctx* ctx = context(default_device());
  const int32_t deg = degree;
  pdsim_phase_result pre, dec;
  check_ctx(pdsim_gpu_phase_sims(ctx, 1, &ta.view, &deg, &prof, &pre, &dec), ctx);
  const pdsim_phase_result& r = prefill ? pre : dec;
  if (r.status != PDSIM_OK) {
    raise(r.status, prefill ? "planner: reference trace has no prefill tasks"
                            : (trace.sessions.empty() ? "planner: reference trace has no sessions"
                                                      : "planner: reference trace produced no inter-token samples"));
  }
  PhaseSimResult out;
  out.p95 = r.p95;
  out.infeasible = r.infeasible != 0;
  out.sample_count = r.sample_count;
  return out;
}

}  // namespace

PhaseSimResult simulate_prefill_replica(const Trace& trace, const PerfProfile& profile, int degree) {
  return phase(trace, profile, degree, true);
}

PhaseSimResult simulate_decode_replica(const Trace& trace, const PerfProfile& profile, int degree) {
  return phase(trace, profile, degree, false);
}

std::vector<LatencyCoefficients> estimate_coefficients_batch(const TraceStats& stats, const std::vector<double>& rates,
                                                             const std::vector<std::uint64_t>& seeds,
                                                             const PerfProfile& profile,
                                                             const std::vector<int>& degrees, int total_gpus) {
  if (rates.size() != seeds.size()) throw ConfigError("planner: rates and seeds differ in length");
  pdsim_profile prof;
  profile_to_pod(profile, &prof);
  const pdsim_trace_stats st = stats_to_pod(stats);
  std::vector<int32_t> ds(degrees.begin(), degrees.end());
  pdsim_gpu_ctx* ctx = context(default_device());
  std::vector<pdsim_coefficients> pods(rates.size());
  std::vector<int32_t> status(rates.size(), PDSIM_OK);
  check_ctx(pdsim_gpu_estimate_coefficients(ctx, &st, static_cast<int32_t>(rates.size()), rates.data(), seeds.data(),
                                            &prof, ds.data(), static_cast<int32_t>(ds.size()), total_gpus,
                                            pods.data(), status.data()),
            ctx);
  std::vector<LatencyCoefficients> out;
  for (size_t s = 0; s < rates.size(); ++s) {
    if (status[s] != PDSIM_OK) raise(status[s], pdsim_gpu_last_error(ctx));
    LatencyCoefficients c;
    const pdsim_coefficients& p = pods[s];
    std::string degs;
    for (int k = 0; k < p.n_degrees; ++k) {
      const int n = p.degrees[k];
      if (p.infeasible_pre[k]) c.infeasible_pre.insert(n); else c.tau_pre[n] = p.tau_pre[k];
      if (p.infeasible_dec[k]) c.infeasible_dec.insert(n); else c.tau_dec[n] = p.tau_dec[k];
      degs += (k ? "," : "") + std::to_string(n);
    }
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%g", rates[s]);
    c.provenance = std::string("rate=") + buf + " sessions=256 gpus=" + std::to_string(total_gpus) +
                   " seed=" + std::to_string(seeds[s]) + " degrees=[" + degs + "]";  // planner.cpp:273-281
    out.push_back(std::move(c));
  }
  return out;
}

LatencyCoefficients estimate_coefficients(const TraceStats& stats, double rate, const PerfProfile& profile,
                                          const std::vector<int>& degrees, int total_gpus, std::uint64_t seed) {
  return estimate_coefficients_batch(stats, {rate}, {seed}, profile, degrees, total_gpus).front();
}

DeploymentPlan solve(const LatencyCoefficients& coeffs, int total_gpus, const std::vector<int>& degrees) {
  const pdsim_coefficients c = coeffs_to_pod(coeffs, degrees);
  pdsim_plan p;
  double z = 0.0;
  int32_t gpus = 0, feasible = 0;
  check(pdsim_solve(&c, total_gpus, &p, &z, &gpus, &feasible));
  if (!feasible) return DeploymentPlan{};
  return plan_from_pod(p, z, gpus);
}

std::vector<DeploymentPlan> top_k(const LatencyCoefficients& coeffs, int total_gpus, const std::vector<int>& degrees,
                                  int k) {
  const pdsim_coefficients c = coeffs_to_pod(coeffs, degrees);
  if (k < 1) throw ConfigError("top_k: k must be >= 1");
  std::vector<pdsim_plan> plans(static_cast<size_t>(k));
  std::vector<double> z(static_cast<size_t>(k));
  std::vector<int32_t> g(static_cast<size_t>(k));
  const int64_t n = pdsim_top_k(&c, total_gpus, k, plans.data(), z.data(), g.data());
  if (n < 0) raise(PDSIM_ERR_CONFIG, pdsim_last_error());
  std::vector<DeploymentPlan> out;
  for (int64_t i = 0; i < n; ++i) out.push_back(plan_from_pod(plans[static_cast<size_t>(i)], z[static_cast<size_t>(i)], g[static_cast<size_t>(i)]));
  return out;
}

// ---- Report aggregation (metrics.cpp:108-190), host restatement ----
namespace {
double mean_in_order(const std::vector<double>& v) {
  if (v.empty()) return 0.0;
  double s = 0.0;
  for (double x : v) s += x;
  return s / static_cast<double>(v.size());
}
MetricStat stat_of(const std::vector<double>& v) {
  MetricStat m;
  m.count = static_cast<std::int64_t>(v.size());
  m.mean = mean_in_order(v);
  m.p95 = percentile_nearest_rank(v, 0.95);
  return m;
}
}  // namespace

double percentile_nearest_rank(std::vector<double> values, double q) {
  if (!(q > 0.0 && q <= 1.0)) throw DomainError("percentile: q must be in (0, 1]");
  if (values.empty()) return 0.0;
  const std::size_t n = values.size();
  std::size_t rank = static_cast<std::size_t>(std::ceil(q * static_cast<double>(n)));
  if (rank < 1) rank = 1;
  std::nth_element(values.begin(), values.begin() + static_cast<std::ptrdiff_t>(rank - 1), values.end());
  return values[rank - 1];
}

Report build_report_from_samples(const std::string& trace_name, std::int64_t sessions_total,
                                 const std::vector<TtftSample>& ttft, const std::vector<ItlSample>& itl,
                                 const std::vector<SessionOutcome>& sessions) {
  Report r;
  r.trace_name = trace_name;
  r.sessions_total = sessions_total;
  r.sessions_completed = static_cast<std::int64_t>(sessions.size());
  if (sessions.empty() && ttft.empty() && itl.empty()) {
    r.empty = true;
    return r;
  }
  std::vector<double> initial, incremental;
  std::int64_t local = 0;
  for (const TtftSample& s : ttft) {
    (s.kind == TaskKind::kInitial ? initial : incremental).push_back(s.value);
    if (s.local) ++local;
  }
  r.ttft_initial = stat_of(initial);
  r.ttft_incremental = stat_of(incremental);
  if (!ttft.empty()) r.local_fraction = static_cast<double>(local) / static_cast<double>(ttft.size());
  std::vector<double> gaps;
  gaps.reserve(itl.size());
  for (const ItlSample& s : itl) gaps.push_back(s.value);
  r.itl = stat_of(gaps);
  if (!sessions.empty()) {
    std::int64_t slo = 0, t_ok = 0, i_ok = 0;
    std::vector<double> e2e;
    e2e.reserve(sessions.size());
    for (const SessionOutcome& s : sessions) {
      slo += s.slo_ok;
      t_ok += s.ttft_ok;
      i_ok += s.itl_ok;
      e2e.push_back(s.completion_time - s.arrival_time);
    }
    const double denom = static_cast<double>(sessions.size());
    r.slo_attainment = static_cast<double>(slo) / denom;
    r.ttft_attainment = static_cast<double>(t_ok) / denom;
    r.itl_attainment = static_cast<double>(i_ok) / denom;
    r.e2e_mean = mean_in_order(e2e);
  }
  return r;
}

Report build_report(const SimResult& result) {
  return build_report_from_samples(result.trace_name, result.total_sessions, result.ttft_samples,
                                   result.itl_samples, result.sessions);
}

std::string format_plan(const DeploymentPlan& plan) {
  if (!plan.feasible) return "infeasible";
  auto phase = [](const std::map<int, int>& counts) {
    if (counts.empty()) return std::string("<none>");
    std::string out;
    for (const auto& [d, c] : counts) {
      if (!out.empty()) out += " + ";
      out += "<TP=" + std::to_string(d) + ", DP=" + std::to_string(c) + ">";
    }
    return out;
  };
  return "P:" + phase(plan.x) + ", D:" + phase(plan.y);
}

// ---- coordinator / sim_engine enums and helpers ----
const char* to_string(RouteRationale r) {
  switch (r) {
    case RouteRationale::kSlackRemote: return "slack_remote";
    case RouteRationale::kSlackLocal: return "slack_local";
    case RouteRationale::kArgmin: return "argmin";
    case RouteRationale::kForcedRemote: return "forced_remote";
    case RouteRationale::kForcedLocal: return "forced_local";
  }
  return "unknown";
}

const char* to_string(RoutingMode m) {
  switch (m) {
    case RoutingMode::kAdaptive: return "adaptive";
    case RoutingMode::kAlwaysRemote: return "always-remote";
    case RoutingMode::kAlwaysLocal: return "always-local";
  }
  return "unknown";
}

RoutingMode routing_mode_from_string(const std::string& text) {
  if (text == "adaptive") return RoutingMode::kAdaptive;
  if (text == "always-remote") return RoutingMode::kAlwaysRemote;
  if (text == "always-local") return RoutingMode::kAlwaysLocal;
  throw ConfigError("routing: unknown mode '" + text + "' (expected adaptive, always-remote, or always-local)");
}

void SchedulerParams::validate() const {
  if (!(alpha > 0.0 && alpha <= 1.0)) throw ConfigError("scheduler: alpha must be in (0, 1]");
  if (!(beta > 0.0 && beta <= 1.0)) throw ConfigError("scheduler: beta must be in (0, 1]");
  if (window < 1) throw ConfigError("scheduler: window must be >= 1");
  if (!(stat_window > 0.0)) throw ConfigError("scheduler: stat_window must be > 0");
}

bool slo_verdict(const std::vector<double>& ttft_values, const std::vector<double>& itl_values, const SloSpec& slo) {
  double sum = 0.0;
  for (double v : itl_values) sum += v;
  const bool itl_ok = itl_values.empty() || sum / static_cast<double>(itl_values.size()) <= slo.itl_thres;
  return all_within(ttft_values, slo.ttft_thres) && itl_ok;
}

// ---- run(): one replay on the GPU ----
SimResult run(const Trace& trace, const DeploymentPlan& plan, const PerfProfile& profile,
              const SchedulerParams& params, std::uint64_t seed) {
  params.validate();
  plan.validate("plan");
  pdsim_profile prof;
  profile_to_pod(profile, &prof);
  TraceArrays arrays(trace);
  const pdsim_plan pplan = plan_to_pod(plan);
  const pdsim_sched_params pparams = params_to_pod(params);
  const size_t R = static_cast<size_t>(std::max<int64_t>(arrays.view.n_rounds, 1));
  const size_t S = static_cast<size_t>(std::max<int64_t>(arrays.view.n_sessions, 1));
  std::vector<pdsim_decision> dec(R);
  std::vector<pdsim_ttft_sample> ttft(R);
  std::vector<pdsim_session_outcome> sess(S);
  pdsim_run_output out;
  std::memset(&out, 0, sizeof(out));
  out.decisions = dec.data();
  out.ttft_samples = ttft.data();
  out.sessions = sess.data();
  // SimResult::itl_samples, as the reference produces them (one per token
  // after a round's first; PDSIM_RUN_ITL=0 skips the materialisation).
  std::vector<pdsim_itl_sample> itl;
  const char* itl_env = std::getenv("PDSIM_RUN_ITL");
  if (!(itl_env && itl_env[0] == '0')) {
    int64_t cap = 0;
    for (int64_t k = 0; k < arrays.view.n_rounds; ++k) cap += std::max<int64_t>(arrays.view.decode_len[k] - 1, 0);
    itl.resize(static_cast<size_t>(std::max<int64_t>(cap, 1)));
    out.itl_samples = itl.data();
    out.itl_capacity = cap;
  }
  pdsim_gpu_ctx* ctx = context(default_device());
  check_ctx(pdsim_gpu_run(ctx, &arrays.view, &pplan, &prof, &pparams, seed, &out), ctx);
  if (out.itl_samples && out.n_itl > out.itl_capacity) throw DeviceError("run: ITL sample capacity exceeded");

  SimResult r;
  r.trace_name = trace.name;
  r.slo = trace.slo;
  r.total_sessions = static_cast<std::int64_t>(trace.sessions.size());
  for (int64_t k = 0; k < out.n_decisions; ++k) {
    const pdsim_decision& d = dec[static_cast<size_t>(k)];
    DecisionRecord x;
    x.time = d.time;
    x.session_id = d.session_id;
    x.round = d.round;
    x.local = d.local != 0;
    x.worker = d.worker;
    x.rationale = static_cast<RouteRationale>(d.rationale);
    if (d.has_estimate) x.estimated_cost = d.estimated_cost;
    r.decisions.push_back(x);
  }
  if (out.itl_samples) {
    r.itl_samples.reserve(static_cast<size_t>(out.n_itl));
    for (int64_t k = 0; k < out.n_itl; ++k) {
      const pdsim_itl_sample& x = itl[static_cast<size_t>(k)];
      r.itl_samples.push_back({x.session_id, x.round, x.token_index, x.completion_time, x.value});
    }
  }
  for (int64_t k = 0; k < out.n_ttft; ++k) {
    const pdsim_ttft_sample& t = ttft[static_cast<size_t>(k)];
    r.ttft_samples.push_back({t.session_id, t.round, t.kind == 0 ? TaskKind::kInitial : TaskKind::kIncremental,
                              t.local != 0, t.created_time, t.completion_time, t.value});
  }
  for (int64_t k = 0; k < out.n_sessions; ++k) {
    const pdsim_session_outcome& s = sess[static_cast<size_t>(k)];
    r.sessions.push_back({s.session_id, s.arrival_time, s.completion_time, s.rounds, s.admission_wait, s.mean_itl,
                          s.ttft_ok != 0, s.itl_ok != 0, s.slo_ok != 0});
  }
  r.counters.tasks_created = out.counters.tasks_created;
  r.counters.tasks_completed = out.counters.tasks_completed;
  r.counters.tokens_decoded = out.counters.tokens_decoded;
  r.counters.kv_bytes_residual = out.counters.kv_bytes_residual;
  r.counters.max_postpone_observed = out.counters.max_postpone_observed;
  r.counters.events_in_order = out.counters.events_in_order != 0;
  return r;
}

Report report_from_pod(const pdsim_report& p, const std::string& name) {
  Report x;
  x.trace_name = name;
  x.empty = p.empty != 0;
  x.sessions_total = p.sessions_total;
  x.sessions_completed = p.sessions_completed;
  x.slo_attainment = p.slo_attainment;
  x.ttft_attainment = p.ttft_attainment;
  x.itl_attainment = p.itl_attainment;
  x.ttft_initial = {p.ttft_initial.mean, p.ttft_initial.p95, p.ttft_initial.count};
  x.ttft_incremental = {p.ttft_incremental.mean, p.ttft_incremental.p95, p.ttft_incremental.count};
  x.itl = {p.itl.mean, p.itl.p95, p.itl.count};
  x.e2e_mean = p.e2e_mean;
  x.local_fraction = p.local_fraction;
  return x;
}

// ---- raw-sample CSV writers (metrics.cpp:350-474) ----
namespace {
std::string num(double v) {
  char buf[64];
  const int32_t n = pdsim_format_double(v, buf, sizeof(buf));
  return std::string(buf, static_cast<size_t>(std::max(n, 0)));
}
const char* flag(bool b) { return b ? "1" : "0"; }
}  // namespace

std::string ttft_csv(const std::vector<TtftSample>& samples) {
  std::string out = "session_id,round,kind,local,created_time,completion_time,value\n";
  for (const TtftSample& s : samples) {
    out += std::to_string(s.session_id) + ',' + std::to_string(s.round) + ',' +
           (s.kind == TaskKind::kInitial ? "initial" : "incremental") + ',' + flag(s.local) + ',' +
           num(s.created_time) + ',' + num(s.completion_time) + ',' + num(s.value) + '\n';
  }
  return out;
}

std::string itl_csv(const std::vector<ItlSample>& samples) {
  std::string out = "session_id,round,token_index,completion_time,value\n";
  for (const ItlSample& s : samples) {
    out += std::to_string(s.session_id) + ',' + std::to_string(s.round) + ',' + std::to_string(s.token_index) + ',' +
           num(s.completion_time) + ',' + num(s.value) + '\n';
  }
  return out;
}

std::string sessions_csv(const std::vector<SessionOutcome>& sessions) {
  std::string out = "session_id,arrival_time,completion_time,rounds,admission_wait,mean_itl,ttft_ok,itl_ok,slo_ok\n";
  for (const SessionOutcome& s : sessions) {
    out += std::to_string(s.session_id) + ',' + num(s.arrival_time) + ',' + num(s.completion_time) + ',' +
           std::to_string(s.rounds) + ',' + num(s.admission_wait) + ',' + num(s.mean_itl) + ',' + flag(s.ttft_ok) +
           ',' + flag(s.itl_ok) + ',' + flag(s.slo_ok) + '\n';
  }
  return out;
}

std::string decisions_csv(const std::vector<DecisionRecord>& decisions) {
  std::string out = "time,session_id,round,local,worker,rationale,estimated_cost\n";
  for (const DecisionRecord& d : decisions) {
    out += num(d.time) + ',' + std::to_string(d.session_id) + ',' + std::to_string(d.round) + ',' + flag(d.local) +
           ',' + std::to_string(d.worker) + ',' + to_string(d.rationale) + ',';
    if (d.estimated_cost) out += num(*d.estimated_cost);
    out += '\n';
  }
  return out;
}

// ---- sweep(): pdsim sweep as one batched GPU call ----
std::vector<Report> sweep(const std::vector<Trace>& traces, const DeploymentPlan& plan, const PerfProfile& profile,
                          const std::vector<SchedulerParams>& settings, std::uint64_t seed,
                          const SearchOptions& options) {
  if (traces.empty() || settings.empty()) throw ConfigError("sweep: need at least one trace and one setting");
  for (const SchedulerParams& s : settings) s.validate();
  plan.validate("plan");
  pdsim_profile prof;
  profile_to_pod(profile, &prof);
  std::vector<std::unique_ptr<TraceArrays>> arrays;
  std::vector<pdsim_trace> views;
  for (const Trace& t : traces) {
    arrays.emplace_back(new TraceArrays(t));
    views.push_back(arrays.back()->view);
  }
  std::vector<pdsim_sched_params> sets;
  for (const SchedulerParams& s : settings) sets.push_back(params_to_pod(s));
  const pdsim_plan pp = plan_to_pod(plan);
  const size_t n = traces.size() * settings.size();
  std::vector<pdsim_report> reps(n);
  std::vector<int64_t> cand(settings.size());
  pdsim_search_output out;
  std::memset(&out, 0, sizeof(out));
  out.pair_report = reps.data();
  out.candidate_slo_ok = cand.data();
  pdsim_gpu_ctx* ctx = context(options.device >= 0 ? options.device : default_device());
  check_ctx(pdsim_gpu_sweep(ctx, static_cast<int32_t>(views.size()), views.data(), &pp,
                            static_cast<int32_t>(sets.size()), sets.data(), &prof, seed, &out),
            ctx);
  std::vector<Report> r;
  r.reserve(n);
  for (size_t k = 0; k < n; ++k) r.push_back(report_from_pod(reps[k], traces[k % traces.size()].name));
  return r;
}

std::string sweep_csv(const std::vector<double>& rates, const std::vector<SchedulerParams>& settings,
                      const std::vector<Report>& reports) {
  if (reports.size() != rates.size() * settings.size()) throw ConfigError("sweep_csv: reports do not match the grid");
  auto f = [](double v) {
    char buf[64];
    const int32_t n = pdsim_format_double(v, buf, sizeof(buf));
    return std::string(buf, static_cast<size_t>(std::max(n, 0)));
  };
  std::string csv =
      "rate,alpha,beta,window,slo_attainment,ttft_attainment,"
      "itl_attainment,ttft_initial_mean,ttft_initial_p95,ttft_incr_mean,"
      "ttft_incr_p95,itl_mean,itl_p95,e2e_mean,local_fraction\n";
  for (size_t r = 0; r < rates.size(); ++r) {
    for (size_t k = 0; k < settings.size(); ++k) {
      const Report& rep = reports[k * rates.size() + r];
      const SchedulerParams& s = settings[k];
      csv += f(rates[r]) + "," + f(s.alpha) + "," + f(s.beta) + "," + std::to_string(s.window) + "," +
             f(rep.slo_attainment) + "," + f(rep.ttft_attainment) + "," + f(rep.itl_attainment) + "," +
             f(rep.ttft_initial.mean) + "," + f(rep.ttft_initial.p95) + "," + f(rep.ttft_incremental.mean) + "," +
             f(rep.ttft_incremental.p95) + "," + f(rep.itl.mean) + "," + f(rep.itl.p95) + "," + f(rep.e2e_mean) +
             "," + f(rep.local_fraction) + "\n";
    }
  }
  return csv;
}

// ---- plan_search(): the batched GPU search ----
SearchResult plan_search(const std::vector<Trace>& replicas, const std::vector<DeploymentPlan>& candidates,
                         const PerfProfile& profile, const SchedulerParams& params, std::uint64_t engine_seed,
                         const SearchOptions& options) {
  params.validate();
  pdsim_profile prof;
  profile_to_pod(profile, &prof);
  std::vector<std::unique_ptr<TraceArrays>> arrays;
  std::vector<pdsim_trace> views;
  for (const Trace& t : replicas) {
    arrays.emplace_back(new TraceArrays(t));
    views.push_back(arrays.back()->view);
  }
  std::vector<pdsim_plan> plans;
  for (const DeploymentPlan& p : candidates) {
    p.validate("plan");
    plans.push_back(plan_to_pod(p));
  }
  const pdsim_sched_params pparams = params_to_pod(params);
  pdsim_search_input in;
  std::memset(&in, 0, sizeof(in));
  in.n_traces = static_cast<int32_t>(views.size());
  in.n_candidates = static_cast<int32_t>(plans.size());
  in.traces = views.data();
  in.candidates = plans.data();
  in.pair_begin = options.pair_begin;
  const int64_t total = static_cast<int64_t>(views.size()) * static_cast<int64_t>(plans.size());
  in.pair_end = options.pair_end < 0 ? total : options.pair_end;
  const int64_t n = in.pair_end - in.pair_begin;
  std::vector<pdsim_attainment> att(static_cast<size_t>(std::max<int64_t>(n, 1)));
  std::vector<int8_t> status(static_cast<size_t>(std::max<int64_t>(n, 1)));
  SearchResult r;
  r.candidate_slo_ok.assign(plans.size(), 0);
  pdsim_search_output out;
  std::memset(&out, 0, sizeof(out));
  out.pair_attainment = att.data();
  out.pair_status = status.data();
  out.candidate_slo_ok = r.candidate_slo_ok.data();
  std::vector<pdsim_report> reps;
  if (options.report) {
    reps.resize(static_cast<size_t>(std::max<int64_t>(n, 1)));
    out.pair_report = reps.data();
  }
  if (!options.devices.empty()) {
    if (options.report) raise(PDSIM_ERR_CONFIG, "plan_search: reports are single-device");
    check(pdsim_multi_plan_search(static_cast<int32_t>(options.devices.size()), options.devices.data(), &in, &prof,
                                  &pparams, engine_seed, options.prune ? PDSIM_SEARCH_ARGMAX : PDSIM_SEARCH_FULL,
                                  &out));
  } else {
    pdsim_gpu_ctx* ctx = context(options.device >= 0 ? options.device : default_device());
    check_ctx(pdsim_gpu_set_search_mode(ctx, options.prune && !options.report ? PDSIM_SEARCH_ARGMAX : PDSIM_SEARCH_FULL),
              ctx);
    const int rc = pdsim_gpu_plan_search(ctx, &in, &prof, &pparams, engine_seed, &out);
    pdsim_gpu_set_search_mode(ctx, PDSIM_SEARCH_FULL);
    check_ctx(rc, ctx);
  }
  if (options.report) {
    for (int64_t k = 0; k < n; ++k) {
      r.reports.push_back(report_from_pod(
          reps[static_cast<size_t>(k)],
          replicas[static_cast<size_t>((in.pair_begin + k) % static_cast<int64_t>(replicas.size()))].name));
    }
  }
  r.best_candidate = out.best_candidate;
  r.best_slo_ok = out.best_slo_ok;
  r.kernel_ms = out.kernel_ms;
  r.device_ms = out.device_ms;
  for (int64_t k = 0; k < n; ++k) {
    const pdsim_attainment& a = att[static_cast<size_t>(k)];
    r.pairs.push_back({a.sessions_total, a.sessions_completed, a.slo_ok, a.ttft_ok, a.itl_ok,
                       status[static_cast<size_t>(k)] == PDSIM_PAIR_OK});
  }
  return r;
}

}  // namespace pdsim
