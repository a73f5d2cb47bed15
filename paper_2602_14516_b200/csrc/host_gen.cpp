// host_gen.cpp — host-side input generation and candidate enumeration.
//
// The north star keeps trace generation on the host "with the reference's own
// RNG so that inputs are identical". These functions restate the reference
// generators with the same std::mt19937_64 draws and the same glibc libm calls
// in the same order; tests/test_generators.py checks them byte-for-byte against
// the reference built in oracle/_ref. Compiled with -ffp-contract=off: the
// reference's `lo + (hi - lo) * u` must round twice.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "common.cuh"
#include "pack.hpp"
#include "pdsim_gpu.h"

namespace pdg {
void set_last_error(const std::string& msg);  // capi.cu: backs pdsim_last_error()
}

namespace {

int host_fail(int code, const std::string& msg) {
  pdg::set_last_error(msg);
  return code;
}

struct Rng {
  uint64_t mt[pdg::Mt64::kN];
  uint32_t idx;
  explicit Rng(uint64_t seed) { pdg::mt64_seed(mt, &idx, seed); }
  uint64_t operator()() { return pdg::mt64_next(mt, &idx); }
};

// uniform() / uniform01() draw the top 53 bits (perf_model.cpp:36-39,
// workload.cpp:32-34).
double uniform01(Rng& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
double uniform(Rng& rng, double lo, double hi) { return lo + (hi - lo) * uniform01(rng); }

// workload.cpp:37-40
double exponential(Rng& rng, double rate) { return -std::log1p(-uniform01(rng)) / rate; }

// workload.cpp:43-47 (Box-Muller, two uniforms)
double standard_normal(Rng& rng) {
  const double u1 = 1.0 - uniform01(rng);
  const double u2 = uniform01(rng);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// workload.cpp:51-58
double lognormal_mean_cv(Rng& rng, double mean, double cv) {
  if (cv <= 0.0) return mean;
  const double sigma2 = std::log1p(cv * cv);
  const double mu = std::log(mean) - 0.5 * sigma2;
  return std::exp(mu + std::sqrt(sigma2) * standard_normal(rng));
}

// workload.cpp:61-70
int64_t draw_round_count(Rng& rng, double mean_rounds, bool fixed) {
  if (fixed || mean_rounds <= 1.0) return std::max<int64_t>(1, std::llround(mean_rounds));
  const double p = 1.0 / mean_rounds;
  const double u = uniform01(rng);
  const double failures = std::floor(std::log1p(-u) / std::log1p(-p));
  return 1 + static_cast<int64_t>(failures);
}

int64_t positive_tokens(double x) { return std::max<int64_t>(1, std::llround(x)); }

void set_curve(pdsim_curve* c, const std::vector<double>& bps, const std::vector<double>& alpha,
               const std::vector<double>& beta) {
  std::memset(c, 0, sizeof(*c));
  c->n_breakpoints = static_cast<int32_t>(bps.size());
  for (size_t i = 0; i < bps.size(); ++i) c->breakpoints[i] = bps[i];
  for (size_t i = 0; i < alpha.size(); ++i) {
    c->alpha[i] = alpha[i];
    c->beta[i] = beta[i];
  }
}

}  // namespace

struct pdsim_trace_buf {
  std::vector<int64_t> sid, off, incr, dec;
  std::vector<double> arr, delay;
  double ttft = 0, itl = 0;
};

extern "C" {

void pdsim_synth_spec_default(pdsim_synth_spec* s) {
  // SynthProfileSpec{} (perf_model.hpp:110-139).
  std::memset(s, 0, sizeof(*s));
  s->n_degrees = 4;
  s->degrees[0] = 1;
  s->degrees[1] = 2;
  s->degrees[2] = 4;
  s->degrees[3] = 8;
  s->prefill_alpha_min = 0.008;
  s->prefill_alpha_max = 0.015;
  s->prefill_beta_min = 1.5e-5;
  s->prefill_beta_max = 3.0e-5;
  s->n_prefill_breakpoints = 2;
  s->prefill_breakpoints[0] = 2048.0;
  s->prefill_breakpoints[1] = 8192.0;
  s->decode_alpha_min = 0.004;
  s->decode_alpha_max = 0.008;
  s->decode_beta_min = 3.0e-4;
  s->decode_beta_max = 6.0e-4;
  s->n_decode_breakpoints = 1;
  s->decode_breakpoints[0] = 64.0;
  s->segment_growth_min = 1.05;
  s->segment_growth_max = 1.30;
  s->scaling_exponent = 0.7;
  s->kv_bandwidth_bytes_per_sec = 2.0e10;
  s->kv_latency_seconds = 0.002;
  s->kv_reshard_penalty = 1.25;
  s->kv_bytes_per_token = 163840;
  s->gpu_memory_capacity = 96LL * 1000 * 1000 * 1000;
  s->history_weight = 0.1;
}

// synth_profile (perf_model.cpp:207-273).
int pdsim_synth_profile(const pdsim_synth_spec* spec, uint64_t seed, pdsim_profile* out) {
  if (!spec || !out) return host_fail(PDSIM_ERR_CONFIG, "null argument");
  if (spec->n_degrees <= 0) return host_fail(PDSIM_ERR_CONFIG, "synth_profile: degree set is empty");
  if (spec->n_degrees > PDSIM_MAX_DEGREES || spec->n_prefill_breakpoints < 0 ||
      spec->n_prefill_breakpoints > PDSIM_MAX_BREAKPOINTS || spec->n_decode_breakpoints < 0 ||
      spec->n_decode_breakpoints > PDSIM_MAX_BREAKPOINTS) {
    return host_fail(PDSIM_ERR_CONFIG, "synth_profile: spec exceeds the C-ABI table sizes");
  }
  Rng rng(seed);
  std::memset(out, 0, sizeof(*out));
  std::vector<int> degrees(spec->degrees, spec->degrees + spec->n_degrees);
  std::sort(degrees.begin(), degrees.end());
  out->n_degrees = spec->n_degrees;
  for (int i = 0; i < spec->n_degrees; ++i) out->degrees[i] = degrees[static_cast<size_t>(i)];
  out->kv_bytes_per_token = spec->kv_bytes_per_token;
  out->gpu_memory_capacity = spec->gpu_memory_capacity;
  out->history_weight = spec->history_weight;

  struct Base {
    std::vector<double> bps, alpha, beta;
  };
  auto draw = [&](double amin, double amax, double bmin, double bmax, const double* bps, int nbp) {
    Base b;
    const double alpha = uniform(rng, amin, amax);
    const double beta = uniform(rng, bmin, bmax);
    b.bps.assign(bps, bps + nbp);
    double cur = beta;
    b.alpha.push_back(alpha);
    b.beta.push_back(cur);
    for (int i = 0; i < nbp; ++i) {
      cur *= uniform(rng, spec->segment_growth_min, spec->segment_growth_max);
      b.alpha.push_back(alpha);
      b.beta.push_back(cur);
    }
    return b;
  };
  const Base pre = draw(spec->prefill_alpha_min, spec->prefill_alpha_max, spec->prefill_beta_min,
                        spec->prefill_beta_max, spec->prefill_breakpoints, spec->n_prefill_breakpoints);
  const Base dec = draw(spec->decode_alpha_min, spec->decode_alpha_max, spec->decode_beta_min,
                        spec->decode_beta_max, spec->decode_breakpoints, spec->n_decode_breakpoints);
  for (int i = 0; i < out->n_degrees; ++i) {
    const double f = std::pow(static_cast<double>(out->degrees[i]), -spec->scaling_exponent);
    std::vector<double> a, b;
    for (size_t k = 0; k < pre.alpha.size(); ++k) {
      a.push_back(pre.alpha[k] * f);
      b.push_back(pre.beta[k] * f);
    }
    set_curve(&out->prefill[i], pre.bps, a, b);
    a.clear();
    b.clear();
    for (size_t k = 0; k < dec.alpha.size(); ++k) {
      a.push_back(dec.alpha[k] * f);
      b.push_back(dec.beta[k] * f);
    }
    set_curve(&out->decode[i], dec.bps, a, b);
  }
  const double kv_beta = static_cast<double>(spec->kv_bytes_per_token) / spec->kv_bandwidth_bytes_per_sec;
  for (int i = 0; i < out->n_degrees; ++i) {
    for (int j = 0; j < out->n_degrees; ++j) {
      const double penalty = i == j ? 1.0 : spec->kv_reshard_penalty;
      const double jitter = uniform(rng, 0.95, 1.05);
      set_curve(&out->kv[i][j], {}, {spec->kv_latency_seconds * penalty}, {kv_beta * penalty * jitter});
    }
  }
  pdg::HostError err;
  if (!pdg::validate_profile(*out, &err)) return host_fail(err.code, err.msg);
  return PDSIM_OK;
}

int pdsim_profile_validate(const pdsim_profile* p) {
  if (!p) return host_fail(PDSIM_ERR_CONFIG, "null profile");
  pdg::HostError err;
  if (!pdg::validate_profile(*p, &err)) return host_fail(err.code, err.msg);
  return PDSIM_OK;
}

// preset_stats (workload.cpp:136-168).
int pdsim_preset_stats(const char* name, pdsim_trace_stats* out) {
  if (!name || !out) return host_fail(PDSIM_ERR_CONFIG, "null argument");
  std::memset(out, 0, sizeof(*out));
  // TraceStats{} defaults (workload.hpp:66-76).
  out->length_cv = 0.5;
  out->first_round_fraction = 0.5;
  out->mean_interaction_delay = 0.5;
  const std::string n(name);
  if (n == "toolbench") {
    out->mean_rounds = 3.96;
    out->fixed_rounds = 0;
    out->mean_prefill_len = 703.79;
    out->mean_decode_len = 50.39;
    out->ttft_thres = 1.0;
    out->itl_thres = 0.05;
  } else if (n == "gaia") {
    out->mean_rounds = 11.32;
    out->fixed_rounds = 0;
    out->mean_prefill_len = 6161.02;
    out->mean_decode_len = 528.76;
    out->ttft_thres = 2.5;
    out->itl_thres = 0.06;
  } else if (n == "hotpotqa") {
    out->mean_rounds = 3.0;
    out->fixed_rounds = 1;
    out->mean_prefill_len = 1569.8;
    out->mean_decode_len = 80.03;
    out->ttft_thres = 1.0;
    out->itl_thres = 0.05;
  } else if (n == "dureader") {
    out->mean_rounds = 3.0;
    out->fixed_rounds = 1;
    out->mean_prefill_len = 3081.23;
    out->mean_decode_len = 150.10;
    out->ttft_thres = 1.5;
    out->itl_thres = 0.05;
  } else {
    return host_fail(PDSIM_ERR_CONFIG,
                     "unknown trace preset '" + n + "' (expected toolbench|gaia|hotpotqa|dureader)");
  }
  return PDSIM_OK;
}

// gen_trace (workload.cpp:170-229).
int pdsim_gen_trace(const pdsim_trace_stats* st, double rate, int32_t num_sessions, uint64_t seed,
                    pdsim_trace_buf** out) {
  if (!st || !out) return host_fail(PDSIM_ERR_CONFIG, "null argument");
  *out = nullptr;
  if (!(rate > 0.0)) return host_fail(PDSIM_ERR_DOMAIN, "gen_trace: arrival_rate must be > 0");
  if (num_sessions < 1) return host_fail(PDSIM_ERR_DOMAIN, "gen_trace: num_sessions must be >= 1");
  if (!(st->mean_rounds >= 1.0) || !(st->mean_prefill_len >= 1.0) || !(st->mean_decode_len >= 1.0)) {
    return host_fail(PDSIM_ERR_DOMAIN, "gen_trace: stats means must be >= 1");
  }
  Rng rng(seed);
  auto* buf = new pdsim_trace_buf();
  buf->ttft = st->ttft_thres;
  buf->itl = st->itl_thres;
  buf->off.push_back(0);
  double clock = 0.0;
  std::vector<int64_t> incr, dec;
  std::vector<double> delay;
  for (int i = 0; i < num_sessions; ++i) {
    clock += exponential(rng, rate);
    buf->sid.push_back(i);
    buf->arr.push_back(clock);
    const int64_t n = draw_round_count(rng, st->mean_rounds, st->fixed_rounds != 0);
    const double total_prefill = lognormal_mean_cv(rng, st->mean_prefill_len, st->length_cv);
    incr.assign(static_cast<size_t>(n), 0);
    dec.assign(static_cast<size_t>(n), 0);
    delay.assign(static_cast<size_t>(n), 0.0);
    if (n == 1) {
      incr[0] = positive_tokens(total_prefill);
    } else {
      const double first = st->first_round_fraction * total_prefill;
      const double rest = (total_prefill - first) / static_cast<double>(n - 1);
      incr[0] = positive_tokens(first);
      for (int64_t r = 1; r < n; ++r) incr[static_cast<size_t>(r)] = positive_tokens(rest);
    }
    for (int64_t r = 0; r < n; ++r) {
      dec[static_cast<size_t>(r)] = positive_tokens(lognormal_mean_cv(rng, st->mean_decode_len, st->length_cv));
    }
    for (int64_t r = 0; r + 1 < n; ++r) {
      delay[static_cast<size_t>(r)] =
          st->mean_interaction_delay > 0.0 ? exponential(rng, 1.0 / st->mean_interaction_delay) : 0.0;
    }
    buf->incr.insert(buf->incr.end(), incr.begin(), incr.end());
    buf->dec.insert(buf->dec.end(), dec.begin(), dec.end());
    buf->delay.insert(buf->delay.end(), delay.begin(), delay.end());
    buf->off.push_back(static_cast<int64_t>(buf->incr.size()));
  }
  pdsim_trace view;
  pdsim_trace_buf_view(buf, &view);
  pdg::PackedTrace scratch;
  pdg::HostError err;
  if (!pdg::pack_trace(view, &scratch, &err)) {  // trace.validate()
    delete buf;
    return host_fail(err.code, err.msg);
  }
  *out = buf;
  return PDSIM_OK;
}

int pdsim_gen_trace_batch(const pdsim_trace_stats* st, int32_t n, const double* rates, int32_t num_sessions,
                          const uint64_t* seeds, pdsim_trace_buf** out) {
  if (!st || !out || n < 0 || (n > 0 && (!rates || !seeds))) return host_fail(PDSIM_ERR_CONFIG, "null argument");
  std::vector<int> rc(static_cast<size_t>(n), PDSIM_OK);
  std::vector<std::string> msg(static_cast<size_t>(n));
  pdg::parallel_for(static_cast<size_t>(n), [&](size_t k) {
    out[k] = nullptr;
    rc[k] = pdsim_gen_trace(st, rates[k], num_sessions, seeds[k], &out[k]);
    if (rc[k] != PDSIM_OK) msg[k] = pdsim_last_error();
  });
  for (int32_t k = 0; k < n; ++k) {
    if (rc[static_cast<size_t>(k)] != PDSIM_OK) {
      for (int32_t j = 0; j < n; ++j) {
        pdsim_trace_buf_free(out[j]);
        out[j] = nullptr;
      }
      return host_fail(rc[static_cast<size_t>(k)], msg[static_cast<size_t>(k)].c_str());
    }
  }
  return PDSIM_OK;
}

int pdsim_trace_buf_view(const pdsim_trace_buf* b, pdsim_trace* v) {
  if (!b || !v) return host_fail(PDSIM_ERR_CONFIG, "null argument");
  v->n_sessions = static_cast<int64_t>(b->sid.size());
  v->n_rounds = static_cast<int64_t>(b->incr.size());
  v->session_id = b->sid.data();
  v->arrival_time = b->arr.data();
  v->round_offset = b->off.data();
  v->incr_input_len = b->incr.data();
  v->decode_len = b->dec.data();
  v->interaction_delay = b->delay.data();
  v->ttft_thres = b->ttft;
  v->itl_thres = b->itl;
  return PDSIM_OK;
}

void pdsim_trace_buf_free(pdsim_trace_buf* b) { delete b; }

int pdsim_trace_validate(const pdsim_trace* t) {
  if (!t) return host_fail(PDSIM_ERR_CONFIG, "null trace");
  pdg::PackedTrace scratch;
  pdg::HostError err;
  if (!pdg::pack_trace(*t, &scratch, &err)) return host_fail(err.code, err.msg);
  return PDSIM_OK;
}

// enumerate_counts / top_k emission order (planner.cpp:582-601, 625-655):
// prefill count vectors over ascending degrees with counts ascending (first
// degree outermost), each followed by every decode vector under the remaining
// budget; empty phases are skipped.
int64_t pdsim_enumerate_plans(const int32_t* degrees, int32_t n_degrees, int32_t total_gpus, pdsim_plan* out,
                              int64_t capacity) {
  if (!degrees || n_degrees <= 0 || total_gpus < 1) return 0;
  std::vector<int> ds(degrees, degrees + n_degrees);
  std::sort(ds.begin(), ds.end());
  ds.erase(std::unique(ds.begin(), ds.end()), ds.end());
  if (ds.front() < 1 || static_cast<int>(ds.size()) > PDSIM_MAX_GROUPS) return -1;
  const size_t nd = ds.size();
  int64_t count = 0;
  std::vector<int> xs(nd, 0), ys(nd, 0);
  std::function<void(size_t, int, std::vector<int>&, const std::function<void()>&)> rec =
      [&](size_t j, int budget, std::vector<int>& cur, const std::function<void()>& emit) {
        if (j == nd) {
          emit();
          return;
        }
        for (int c = 0; c * ds[j] <= budget; ++c) {
          cur[j] = c;
          rec(j + 1, budget - c * ds[j], cur, emit);
        }
        cur[j] = 0;
      };
  rec(0, total_gpus, xs, [&] {
    int xg = 0, xn = 0;
    for (size_t j = 0; j < nd; ++j) {
      xg += ds[j] * xs[j];
      xn += xs[j];
    }
    if (xn == 0) return;
    rec(0, total_gpus - xg, ys, [&] {
      int yn = 0;
      for (size_t j = 0; j < nd; ++j) yn += ys[j];
      if (yn == 0) return;
      if (out && count < capacity) {
        pdsim_plan& p = out[count];
        std::memset(&p, 0, sizeof(p));
        for (size_t j = 0; j < nd; ++j) {
          if (xs[j]) {
            p.prefill_degree[p.n_prefill_groups] = ds[j];
            p.prefill_count[p.n_prefill_groups++] = xs[j];
          }
          if (ys[j]) {
            p.decode_degree[p.n_decode_groups] = ds[j];
            p.decode_count[p.n_decode_groups++] = ys[j];
          }
        }
      }
      ++count;
    });
  });
  return count;
}

int32_t pdsim_format_double(double value, char* buf, int32_t cap) {
  char tmp[64];
  const auto res = std::to_chars(tmp, tmp + sizeof(tmp), value);
  const int32_t n = static_cast<int32_t>(res.ptr - tmp);
  if (!buf || cap < n + 1) return -1;
  memcpy(buf, tmp, static_cast<size_t>(n));
  buf[n] = '\0';
  return n;
}

int32_t pdsim_argmax_candidates(const int64_t* v, int32_t n) {
  int32_t best = -1;
  for (int32_t c = 0; c < n; ++c) {
    if (v[c] < 0) continue;
    if (best < 0 || v[c] > v[best]) best = c;
  }
  return best;
}

}  // extern "C"
