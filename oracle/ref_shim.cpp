// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" shim over the UNMODIFIED reference simulator, compiled
// from the sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libpdsim_ref.so. It converts the POD types of include/pdsim_gpu.h
// into the reference's C++ types, calls the reference entry points and
// converts the results back, so that tests and bench.py's CPU legs can run the
// reference path on the same inputs as the GPU path:
//   - pdsim::run           (proj/src/sim_engine.cpp:676-681)
//   - pdsim::gen_trace     (proj/src/workload.cpp:170-229)
//   - pdsim::synth_profile (proj/src/perf_model.cpp:207-273)
//   - pdsim::top_k         (proj/src/planner.cpp:605-657, enumeration pinning)
//   - the surrogate planner: simulate_prefill_replica / simulate_decode_replica
//     / estimate_coefficients / solve / top_k (proj/src/planner.cpp:75-657)
//   - the CSV writers      (proj/src/metrics.cpp:366-474, FNV-1a fingerprints)
// plus a std::thread pool replaying (candidate, replica) pairs: the reference's
// CPU plan-search baseline.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "pdsim/errors.hpp"
#include "pdsim/metrics.hpp"
#include "pdsim/perf_model.hpp"
#include "pdsim/planner.hpp"
#include "pdsim/sim_engine.hpp"
#include "pdsim/workload.hpp"
#include "pdsim_gpu.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PDSIM_OK;
  } catch (const pdsim::ParseError& e) {
    return fail(PDSIM_ERR_PARSE, e.what());
  } catch (const pdsim::ConfigError& e) {
    return fail(PDSIM_ERR_CONFIG, e.what());
  } catch (const pdsim::DomainError& e) {
    return fail(PDSIM_ERR_DOMAIN, e.what());
  } catch (const std::exception& e) {
    return fail(PDSIM_ERR_INTERNAL, e.what());
  }
}

std::uint64_t fnv1a(const std::string& s) {
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

pdsim::PiecewiseAlphaBeta curve_from_pod(const pdsim_curve& c) {
  std::vector<double> bps(c.breakpoints, c.breakpoints + c.n_breakpoints);
  std::vector<pdsim::AlphaBetaSegment> segs;
  for (int i = 0; i <= c.n_breakpoints; ++i) segs.push_back({c.alpha[i], c.beta[i]});
  return pdsim::PiecewiseAlphaBeta(bps, segs);
}

void curve_to_pod(const pdsim::PiecewiseAlphaBeta& c, pdsim_curve* out) {
  std::memset(out, 0, sizeof(*out));
  if (c.breakpoints().size() > PDSIM_MAX_BREAKPOINTS ||
      c.segments().size() != c.breakpoints().size() + 1) {
    throw pdsim::ConfigError("shim: curve does not fit the POD layout");
  }
  out->n_breakpoints = static_cast<int32_t>(c.breakpoints().size());
  for (std::size_t i = 0; i < c.breakpoints().size(); ++i) out->breakpoints[i] = c.breakpoints()[i];
  for (std::size_t i = 0; i < c.segments().size(); ++i) {
    out->alpha[i] = c.segments()[i].alpha;
    out->beta[i] = c.segments()[i].beta;
  }
}

pdsim::PerfProfile profile_from_pod(const pdsim_profile& p) {
  pdsim::PerfProfile out;
  out.degrees.assign(p.degrees, p.degrees + p.n_degrees);
  out.kv_bytes_per_token = p.kv_bytes_per_token;
  out.gpu_memory_capacity = p.gpu_memory_capacity;
  out.history_weight = p.history_weight;
  for (int i = 0; i < p.n_degrees; ++i) {
    out.prefill_cost.emplace(p.degrees[i], curve_from_pod(p.prefill[i]));
    out.decode_cost.emplace(p.degrees[i], curve_from_pod(p.decode[i]));
    for (int j = 0; j < p.n_degrees; ++j) {
      out.kv_cost.emplace(std::make_pair(p.degrees[i], p.degrees[j]),
                          curve_from_pod(p.kv[i][j]));
    }
  }
  return out;
}

void profile_to_pod(const pdsim::PerfProfile& p, pdsim_profile* out) {
  std::memset(out, 0, sizeof(*out));
  if (p.degrees.size() > PDSIM_MAX_DEGREES) throw pdsim::ConfigError("shim: too many degrees");
  out->n_degrees = static_cast<int32_t>(p.degrees.size());
  for (std::size_t i = 0; i < p.degrees.size(); ++i) {
    const int d = p.degrees[i];
    out->degrees[i] = d;
    curve_to_pod(p.prefill_cost.at(d), &out->prefill[i]);
    curve_to_pod(p.decode_cost.at(d), &out->decode[i]);
    for (std::size_t j = 0; j < p.degrees.size(); ++j) {
      curve_to_pod(p.kv_cost.at({d, p.degrees[j]}), &out->kv[i][j]);
    }
  }
  out->kv_bytes_per_token = p.kv_bytes_per_token;
  out->gpu_memory_capacity = p.gpu_memory_capacity;
  out->history_weight = p.history_weight;
}

pdsim::Trace trace_from_pod(const pdsim_trace& t) {
  pdsim::Trace out;
  out.name = "pod";
  out.slo = {t.ttft_thres, t.itl_thres};
  out.sessions.resize(static_cast<std::size_t>(t.n_sessions));
  for (int64_t i = 0; i < t.n_sessions; ++i) {
    pdsim::SessionSpec& s = out.sessions[static_cast<std::size_t>(i)];
    s.session_id = t.session_id[i];
    s.arrival_time = t.arrival_time[i];
    for (int64_t r = t.round_offset[i]; r < t.round_offset[i + 1]; ++r) {
      s.rounds.push_back({t.incr_input_len[r], t.decode_len[r], t.interaction_delay[r]});
    }
  }
  return out;
}

pdsim::DeploymentPlan plan_from_pod(const pdsim_plan& p) {
  pdsim::DeploymentPlan out;
  for (int i = 0; i < p.n_prefill_groups; ++i) out.x[p.prefill_degree[i]] = p.prefill_count[i];
  for (int i = 0; i < p.n_decode_groups; ++i) out.y[p.decode_degree[i]] = p.decode_count[i];
  out.gpus_used = out.gpus();
  out.feasible = true;
  return out;
}

void plan_to_pod(const pdsim::DeploymentPlan& p, pdsim_plan* out) {
  std::memset(out, 0, sizeof(*out));
  for (const auto& [d, c] : p.x) {
    out->prefill_degree[out->n_prefill_groups] = d;
    out->prefill_count[out->n_prefill_groups++] = c;
  }
  for (const auto& [d, c] : p.y) {
    out->decode_degree[out->n_decode_groups] = d;
    out->decode_count[out->n_decode_groups++] = c;
  }
}

pdsim::SchedulerParams params_from_pod(const pdsim_sched_params& p) {
  pdsim::SchedulerParams out;
  out.routing = static_cast<pdsim::RoutingMode>(p.routing);
  out.reorder = p.reorder != 0;
  out.alpha = p.alpha;
  out.beta = p.beta;
  out.window = p.window;
  out.stat_window = p.stat_window;
  return out;
}

pdsim::TraceStats stats_from_pod(const pdsim_trace_stats& s, const char* name) {
  pdsim::TraceStats out;
  out.name = name ? name : "custom";
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

// Owned SoA copy of a reference trace.
struct RefTrace {
  pdsim::Trace trace;
  std::vector<int64_t> sid, off, incr, dec;
  std::vector<double> arr, delay;
  void flatten() {
    sid.clear(); off.assign(1, 0); incr.clear(); dec.clear(); arr.clear(); delay.clear();
    for (const auto& s : trace.sessions) {
      sid.push_back(s.session_id);
      arr.push_back(s.arrival_time);
      for (const auto& r : s.rounds) {
        incr.push_back(r.incr_input_len);
        dec.push_back(r.decode_len);
        delay.push_back(r.interaction_delay);
      }
      off.push_back(static_cast<int64_t>(incr.size()));
    }
  }
};

void attain_of(const pdsim::SimResult& r, pdsim_attainment* a) {
  a->sessions_total = r.total_sessions;
  a->sessions_completed = static_cast<int64_t>(r.sessions.size());
  a->slo_ok = a->ttft_ok = a->itl_ok = 0;
  for (const auto& s : r.sessions) {
    a->slo_ok += s.slo_ok;
    a->ttft_ok += s.ttft_ok;
    a->itl_ok += s.itl_ok;
  }
}

void counters_of(const pdsim::SimResult& r, pdsim_counters* c) {
  c->tasks_created = r.counters.tasks_created;
  c->tasks_completed = r.counters.tasks_completed;
  c->tokens_decoded = r.counters.tokens_decoded;
  c->kv_bytes_residual = r.counters.kv_bytes_residual;
  c->max_postpone_observed = r.counters.max_postpone_observed;
  c->events_in_order = r.counters.events_in_order;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_synth_profile(const pdsim_synth_spec* spec, uint64_t seed, pdsim_profile* out) {
  return guarded([&] {
    pdsim::SynthProfileSpec s;
    s.degrees.assign(spec->degrees, spec->degrees + spec->n_degrees);
    s.prefill_alpha_min = spec->prefill_alpha_min;
    s.prefill_alpha_max = spec->prefill_alpha_max;
    s.prefill_beta_min = spec->prefill_beta_min;
    s.prefill_beta_max = spec->prefill_beta_max;
    s.prefill_breakpoints.assign(spec->prefill_breakpoints,
                                 spec->prefill_breakpoints + spec->n_prefill_breakpoints);
    s.decode_alpha_min = spec->decode_alpha_min;
    s.decode_alpha_max = spec->decode_alpha_max;
    s.decode_beta_min = spec->decode_beta_min;
    s.decode_beta_max = spec->decode_beta_max;
    s.decode_breakpoints.assign(spec->decode_breakpoints,
                                spec->decode_breakpoints + spec->n_decode_breakpoints);
    s.segment_growth_min = spec->segment_growth_min;
    s.segment_growth_max = spec->segment_growth_max;
    s.scaling_exponent = spec->scaling_exponent;
    s.kv_bandwidth_bytes_per_sec = spec->kv_bandwidth_bytes_per_sec;
    s.kv_latency_seconds = spec->kv_latency_seconds;
    s.kv_reshard_penalty = spec->kv_reshard_penalty;
    s.kv_bytes_per_token = spec->kv_bytes_per_token;
    s.gpu_memory_capacity = spec->gpu_memory_capacity;
    s.history_weight = spec->history_weight;
    profile_to_pod(pdsim::synth_profile(s, seed), out);
  });
}

// The reference's default SynthProfileSpec (perf_model.hpp:110-139) as POD.
int ref_synth_spec_default(pdsim_synth_spec* out) {
  return guarded([&] {
    const pdsim::SynthProfileSpec s;
    std::memset(out, 0, sizeof(*out));
    if (s.degrees.size() > PDSIM_MAX_DEGREES || s.prefill_breakpoints.size() > PDSIM_MAX_BREAKPOINTS ||
        s.decode_breakpoints.size() > PDSIM_MAX_BREAKPOINTS) {
      throw pdsim::ConfigError("synth spec default exceeds the POD capacity");
    }
    out->n_degrees = static_cast<int32_t>(s.degrees.size());
    for (std::size_t i = 0; i < s.degrees.size(); ++i) out->degrees[i] = s.degrees[i];
    out->prefill_alpha_min = s.prefill_alpha_min;
    out->prefill_alpha_max = s.prefill_alpha_max;
    out->prefill_beta_min = s.prefill_beta_min;
    out->prefill_beta_max = s.prefill_beta_max;
    out->n_prefill_breakpoints = static_cast<int32_t>(s.prefill_breakpoints.size());
    for (std::size_t i = 0; i < s.prefill_breakpoints.size(); ++i) out->prefill_breakpoints[i] = s.prefill_breakpoints[i];
    out->decode_alpha_min = s.decode_alpha_min;
    out->decode_alpha_max = s.decode_alpha_max;
    out->decode_beta_min = s.decode_beta_min;
    out->decode_beta_max = s.decode_beta_max;
    out->n_decode_breakpoints = static_cast<int32_t>(s.decode_breakpoints.size());
    for (std::size_t i = 0; i < s.decode_breakpoints.size(); ++i) out->decode_breakpoints[i] = s.decode_breakpoints[i];
    out->segment_growth_min = s.segment_growth_min;
    out->segment_growth_max = s.segment_growth_max;
    out->scaling_exponent = s.scaling_exponent;
    out->kv_bandwidth_bytes_per_sec = s.kv_bandwidth_bytes_per_sec;
    out->kv_latency_seconds = s.kv_latency_seconds;
    out->kv_reshard_penalty = s.kv_reshard_penalty;
    out->kv_bytes_per_token = s.kv_bytes_per_token;
    out->gpu_memory_capacity = s.gpu_memory_capacity;
    out->history_weight = s.history_weight;
  });
}

uint64_t ref_profile_hash(const pdsim_profile* p) {
  try {
    return fnv1a(pdsim::save_profile(profile_from_pod(*p)));
  } catch (...) {
    return 0;
  }
}

int ref_profile_validate(const pdsim_profile* p) {
  return guarded([&] { profile_from_pod(*p).validate(); });
}

int ref_preset_stats(const char* name, pdsim_trace_stats* out) {
  return guarded([&] {
    const pdsim::TraceStats s = pdsim::preset_stats(name);
    out->mean_rounds = s.mean_rounds;
    out->fixed_rounds = s.fixed_rounds;
    out->mean_prefill_len = s.mean_prefill_len;
    out->mean_decode_len = s.mean_decode_len;
    out->length_cv = s.length_cv;
    out->first_round_fraction = s.first_round_fraction;
    out->mean_interaction_delay = s.mean_interaction_delay;
    out->ttft_thres = s.slo.ttft_thres;
    out->itl_thres = s.slo.itl_thres;
  });
}

// Returns an owned RefTrace (free with ref_trace_free) or NULL on error.
void* ref_gen_trace(const pdsim_trace_stats* stats, const char* name, double rate,
                    int32_t n, uint64_t seed) {
  RefTrace* t = new RefTrace();
  const int rc = guarded([&] {
    t->trace = pdsim::gen_trace(stats_from_pod(*stats, name), rate, n, seed);
    t->flatten();
  });
  if (rc != PDSIM_OK) {
    delete t;
    return nullptr;
  }
  return t;
}

void ref_trace_view(void* h, pdsim_trace* v) {
  RefTrace* t = static_cast<RefTrace*>(h);
  v->n_sessions = static_cast<int64_t>(t->sid.size());
  v->n_rounds = static_cast<int64_t>(t->incr.size());
  v->session_id = t->sid.data();
  v->arrival_time = t->arr.data();
  v->round_offset = t->off.data();
  v->incr_input_len = t->incr.data();
  v->decode_len = t->dec.data();
  v->interaction_delay = t->delay.data();
  v->ttft_thres = t->trace.slo.ttft_thres;
  v->itl_thres = t->trace.slo.itl_thres;
}

void ref_trace_free(void* h) { delete static_cast<RefTrace*>(h); }

// FNV-1a of save_trace() of a POD trace (name forced to `name`).
uint64_t ref_trace_hash(const pdsim_trace* v, const char* name) {
  try {
    pdsim::Trace t = trace_from_pod(*v);
    t.name = name ? name : "pod";
    return fnv1a(pdsim::save_trace(t));
  } catch (...) {
    return 0;
  }
}

int ref_trace_validate(const pdsim_trace* v) {
  return guarded([&] { trace_from_pod(*v).validate(); });
}

// One reference replay. Record arrays in `out` are optional. hashes (optional,
// 4 entries): FNV-1a of decisions_csv, ttft_csv, sessions_csv, itl_csv.
// itl (optional): [itl_cap] x {session_id, round, token_index} int64 triples
// and values/completion times.
int ref_run(const pdsim_trace* tr, const pdsim_plan* plan, const pdsim_profile* prof,
            const pdsim_sched_params* params, uint64_t seed, pdsim_run_output* out,
            uint64_t* hashes, int64_t itl_cap, int64_t* itl_ids, double* itl_times,
            double* itl_values, int64_t* n_itl) {
  return guarded([&] {
    const pdsim::SimResult r =
        pdsim::run(trace_from_pod(*tr), plan_from_pod(*plan), profile_from_pod(*prof),
                   params_from_pod(*params), seed);
    if (out) {
      out->n_decisions = static_cast<int64_t>(r.decisions.size());
      out->n_ttft = static_cast<int64_t>(r.ttft_samples.size());
      out->n_sessions = static_cast<int64_t>(r.sessions.size());
      counters_of(r, &out->counters);
      attain_of(r, &out->attainment);
      if (out->decisions) {
        for (std::size_t i = 0; i < r.decisions.size(); ++i) {
          const auto& d = r.decisions[i];
          pdsim_decision& o = out->decisions[i];
          std::memset(&o, 0, sizeof(o));
          o.time = d.time;
          o.session_id = d.session_id;
          o.round = d.round;
          o.worker = d.worker;
          o.local = d.local;
          o.rationale = static_cast<int8_t>(d.rationale);
          o.has_estimate = d.estimated_cost.has_value();
          o.estimated_cost = d.estimated_cost.value_or(0.0);
        }
      }
      if (out->ttft_samples) {
        for (std::size_t i = 0; i < r.ttft_samples.size(); ++i) {
          const auto& s = r.ttft_samples[i];
          pdsim_ttft_sample& o = out->ttft_samples[i];
          std::memset(&o, 0, sizeof(o));
          o.session_id = s.session_id;
          o.round = s.round;
          o.kind = s.kind == pdsim::TaskKind::kInitial ? 0 : 1;
          o.local = s.local;
          o.created_time = s.created_time;
          o.completion_time = s.completion_time;
          o.value = s.value;
        }
      }
      if (out->sessions) {
        for (std::size_t i = 0; i < r.sessions.size(); ++i) {
          const auto& s = r.sessions[i];
          pdsim_session_outcome& o = out->sessions[i];
          std::memset(&o, 0, sizeof(o));
          o.session_id = s.session_id;
          o.arrival_time = s.arrival_time;
          o.completion_time = s.completion_time;
          o.admission_wait = s.admission_wait;
          o.mean_itl = s.mean_itl;
          o.rounds = s.rounds;
          o.ttft_ok = s.ttft_ok;
          o.itl_ok = s.itl_ok;
          o.slo_ok = s.slo_ok;
        }
      }
    }
    if (hashes) {
      hashes[0] = fnv1a(pdsim::decisions_csv(r.decisions));
      hashes[1] = fnv1a(pdsim::ttft_csv(r.ttft_samples));
      hashes[2] = fnv1a(pdsim::sessions_csv(r.sessions));
      hashes[3] = fnv1a(pdsim::itl_csv(r.itl_samples));
    }
    if (n_itl) *n_itl = static_cast<int64_t>(r.itl_samples.size());
    if (itl_ids || itl_times || itl_values) {
      const int64_t n = std::min<int64_t>(itl_cap, static_cast<int64_t>(r.itl_samples.size()));
      for (int64_t i = 0; i < n; ++i) {
        const auto& s = r.itl_samples[static_cast<std::size_t>(i)];
        if (itl_ids) {
          itl_ids[3 * i] = s.session_id;
          itl_ids[3 * i + 1] = s.round;
          itl_ids[3 * i + 2] = s.token_index;
        }
        if (itl_times) itl_times[i] = s.completion_time;
        if (itl_values) itl_values[i] = s.value;
      }
    }
  });
}

// The reference CPU plan search: a std::thread pool of
// `n_threads` workers pulls pairs p in [pair_begin, pair_end) (p = c *
// n_traces + r) from an atomic counter and calls pdsim::run on each. Traces,
// plans and the profile are converted to reference types before the clock
// starts; *wall_s covers the pool only. A ConfigError marks the pair invalid.
// Pair k of the pool is pairs[k] when `pairs` is given (a sample of the
// search, outputs indexed by k), else pair_begin + k.
static int plan_search_impl(const pdsim_search_input* in, const pdsim_profile* prof,
                            const pdsim_sched_params* params, uint64_t seed, int32_t n_threads,
                            const int64_t* pairs, int64_t n_pairs, pdsim_attainment* pair_att,
                            int8_t* pair_status, double* wall_s) {
  return guarded([&] {
    std::vector<pdsim::Trace> traces;
    for (int i = 0; i < in->n_traces; ++i) traces.push_back(trace_from_pod(in->traces[i]));
    std::vector<pdsim::DeploymentPlan> plans;
    for (int i = 0; i < in->n_candidates; ++i) plans.push_back(plan_from_pod(in->candidates[i]));
    const pdsim::PerfProfile profile = profile_from_pod(*prof);
    const pdsim::SchedulerParams sp = params_from_pod(*params);
    const int64_t total = static_cast<int64_t>(in->n_traces) * in->n_candidates;
    const int64_t b = pairs ? 0 : in->pair_begin;
    const int64_t e = pairs ? n_pairs : (in->pair_end < 0 ? total : in->pair_end);
    std::atomic<int64_t> next{b};
    auto worker = [&] {
      for (;;) {
        const int64_t k = next.fetch_add(1);
        if (k >= e) return;
        const int64_t p = pairs ? pairs[k] : k;
        const int c = static_cast<int>(p / in->n_traces);
        const int r = static_cast<int>(p % in->n_traces);
        pdsim_attainment a{};
        int8_t st = PDSIM_PAIR_OK;
        try {
          const pdsim::SimResult res = pdsim::run(traces[r], plans[c], profile, sp, seed);
          attain_of(res, &a);
        } catch (const pdsim::ConfigError&) {
          st = PDSIM_PAIR_INVALID;
        } catch (...) {
          st = PDSIM_PAIR_ERROR;
        }
        if (pair_att) pair_att[k - b] = a;
        if (pair_status) pair_status[k - b] = st;
      }
    };
    const int nt = n_threads > 0 ? n_threads
                                 : static_cast<int>(std::thread::hardware_concurrency());
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int i = 0; i < nt; ++i) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    if (wall_s) *wall_s = std::chrono::duration<double>(t1 - t0).count();
  });
}

int ref_plan_search(const pdsim_search_input* in, const pdsim_profile* prof,
                    const pdsim_sched_params* params, uint64_t seed, int32_t n_threads,
                    pdsim_attainment* pair_att, int8_t* pair_status, double* wall_s) {
  return plan_search_impl(in, prof, params, seed, n_threads, nullptr, 0, pair_att, pair_status, wall_s);
}

// The same pool over an explicit list of pairs (bench.py's sampled CPU
// baseline); the pool pulls them in list order.
int ref_plan_search_list(const pdsim_search_input* in, const pdsim_profile* prof,
                         const pdsim_sched_params* params, uint64_t seed, int32_t n_threads,
                         const int64_t* pairs, int64_t n_pairs, pdsim_attainment* pair_att,
                         int8_t* pair_status, double* wall_s) {
  return plan_search_impl(in, prof, params, seed, n_threads, pairs, n_pairs, pair_att, pair_status, wall_s);
}

// Every plan top_k ranks (k = capacity), in plan_ranks_before order — used to
// pin the SET of enumerated candidates. Coefficients are all 1.0.
int64_t ref_top_k_plans(const int32_t* degrees, int32_t n_degrees, int32_t total_gpus,
                        pdsim_plan* out, int64_t capacity) {
  int64_t n = -1;
  guarded([&] {
    std::vector<int> ds(degrees, degrees + n_degrees);
    pdsim::LatencyCoefficients c;
    for (int d : ds) {
      c.tau_pre[d] = 1.0;
      c.tau_dec[d] = 1.0;
    }
    const auto plans = pdsim::top_k(c, total_gpus, ds, 1 << 30);
    n = static_cast<int64_t>(plans.size());
    for (std::size_t i = 0; out && i < plans.size() && static_cast<int64_t>(i) < capacity; ++i) {
      plan_to_pod(plans[i], &out[i]);
    }
  });
  return n;
}


// ---- surrogate planner (planner.cpp:75-657) ----
namespace {
pdsim::LatencyCoefficients coeffs_from_pod(const pdsim_coefficients& c) {
  pdsim::LatencyCoefficients out;
  for (int i = 0; i < c.n_degrees; ++i) {
    if (c.infeasible_pre[i]) out.infeasible_pre.insert(c.degrees[i]); else out.tau_pre[c.degrees[i]] = c.tau_pre[i];
    if (c.infeasible_dec[i]) out.infeasible_dec.insert(c.degrees[i]); else out.tau_dec[c.degrees[i]] = c.tau_dec[i];
  }
  return out;
}
std::vector<int> coeff_degrees(const pdsim_coefficients& c) {
  return std::vector<int>(c.degrees, c.degrees + c.n_degrees);
}
}  // namespace

int ref_phase_sims(const pdsim_trace* tr, const pdsim_profile* prof, int32_t degree, pdsim_phase_result* pre,
                   pdsim_phase_result* dec) {
  const pdsim::Trace t = trace_from_pod(*tr);
  const pdsim::PerfProfile p = profile_from_pod(*prof);
  const int rc1 = guarded([&] {
    const pdsim::PhaseSimResult r = pdsim::simulate_prefill_replica(t, p, degree);
    *pre = pdsim_phase_result{r.p95, r.sample_count, r.infeasible ? 1 : 0, PDSIM_OK};
  });
  if (rc1 != PDSIM_OK) *pre = pdsim_phase_result{0.0, 0, 0, rc1};
  const int rc2 = guarded([&] {
    const pdsim::PhaseSimResult r = pdsim::simulate_decode_replica(t, p, degree);
    *dec = pdsim_phase_result{r.p95, r.sample_count, r.infeasible ? 1 : 0, PDSIM_OK};
  });
  if (rc2 != PDSIM_OK) *dec = pdsim_phase_result{0.0, 0, 0, rc2};
  return PDSIM_OK;
}

int ref_estimate_coefficients(const pdsim_trace_stats* stats, const char* name, double rate,
                              const pdsim_profile* prof, const int32_t* degrees, int32_t n_degrees,
                              int32_t total_gpus, uint64_t seed, pdsim_coefficients* out) {
  return guarded([&] {
    const std::vector<int> ds(degrees, degrees + n_degrees);
    const pdsim::LatencyCoefficients c = pdsim::estimate_coefficients(stats_from_pod(*stats, name), rate,
                                                                      profile_from_pod(*prof), ds, total_gpus, seed);
    std::memset(out, 0, sizeof(*out));
    std::vector<int> ts = ds;
    std::sort(ts.begin(), ts.end());
    ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
    out->n_degrees = static_cast<int32_t>(ts.size());
    for (std::size_t k = 0; k < ts.size(); ++k) {
      const int n = ts[k];
      out->degrees[k] = n;
      out->infeasible_pre[k] = c.infeasible_pre.count(n) ? 1 : 0;
      out->infeasible_dec[k] = c.infeasible_dec.count(n) ? 1 : 0;
      out->tau_pre[k] = c.tau_pre.count(n) ? c.tau_pre.at(n) : 0.0;
      out->tau_dec[k] = c.tau_dec.count(n) ? c.tau_dec.at(n) : 0.0;
    }
  });
}

int ref_solve(const pdsim_coefficients* c, int32_t total_gpus, pdsim_plan* plan, double* z, int32_t* gpus,
              int32_t* feasible) {
  return guarded([&] {
    const pdsim::DeploymentPlan p = pdsim::solve(coeffs_from_pod(*c), total_gpus, coeff_degrees(*c));
    *feasible = p.feasible ? 1 : 0;
    if (p.feasible) {
      plan_to_pod(p, plan);
      *z = p.objective_z;
      *gpus = p.gpus_used;
    }
  });
}

int64_t ref_top_k(const pdsim_coefficients* c, int32_t total_gpus, int32_t k, pdsim_plan* plans, double* z,
                  int32_t* gpus) {
  int64_t n = -1;
  guarded([&] {
    const auto ps = pdsim::top_k(coeffs_from_pod(*c), total_gpus, coeff_degrees(*c), k);
    n = static_cast<int64_t>(ps.size());
    for (std::size_t i = 0; i < ps.size(); ++i) {
      plan_to_pod(ps[i], &plans[i]);
      z[i] = ps[i].objective_z;
      gpus[i] = ps[i].gpus_used;
    }
  });
  return n;
}

// build_report (metrics.cpp:138-190) of one reference replay.
int ref_report(const pdsim_trace* tr, const pdsim_plan* plan, const pdsim_profile* prof,
               const pdsim_sched_params* params, uint64_t seed, pdsim_report* out) {
  return guarded([&] {
    const pdsim::SimResult res = pdsim::run(trace_from_pod(*tr), plan_from_pod(*plan), profile_from_pod(*prof),
                                            params_from_pod(*params), seed);
    const pdsim::Report r = pdsim::build_report(res);
    std::memset(out, 0, sizeof(*out));
    out->sessions_total = r.sessions_total;
    out->sessions_completed = r.sessions_completed;
    out->slo_attainment = r.slo_attainment;
    out->ttft_attainment = r.ttft_attainment;
    out->itl_attainment = r.itl_attainment;
    out->ttft_initial = pdsim_metric_stat{r.ttft_initial.mean, r.ttft_initial.p95, r.ttft_initial.count};
    out->ttft_incremental = pdsim_metric_stat{r.ttft_incremental.mean, r.ttft_incremental.p95, r.ttft_incremental.count};
    out->itl = pdsim_metric_stat{r.itl.mean, r.itl.p95, r.itl.count};
    out->e2e_mean = r.e2e_mean;
    out->local_fraction = r.local_fraction;
    out->empty = r.empty ? 1 : 0;
  });
}

}  // extern "C"
