// pack.hpp — host-side validation and packing of C-ABI inputs into the
// device layouts of engine.cuh. Validation mirrors the checks the reference
// Engine constructor runs before simulating (sim_engine.cpp:109-122):
// Coordinator ctor (coordinator.cpp:102-113), SchedulerParams::validate
// (sim_engine.cpp:653-666), Trace::validate (workload.cpp:90-134),
// PerfProfile::validate (perf_model.cpp:91-153), build_workers
// (sim_engine.cpp:175-203) and precheck_sessions (sim_engine.cpp:217-231).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <set>
#include <queue>
#include <functional>
#include <string>
#include <unordered_set>
#include <thread>
#include <vector>

#include "engine.cuh"
#include "pdsim_gpu.h"

namespace pdg {

struct HostError {
  int code = PDSIM_OK;
  std::string msg;
  bool set(int c, const std::string& m) {
    code = c;
    msg = m;
    return false;
  }
};

inline int64_t pow2_at_least(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// ---- PiecewiseAlphaBeta::validate (perf_model.cpp:54-89) ----
inline bool validate_curve(const pdsim_curve& c, const std::string& where, HostError* err) {
  if (c.n_breakpoints < 0 || c.n_breakpoints > PDSIM_MAX_BREAKPOINTS) {
    return err->set(PDSIM_ERR_CONFIG, where + ": unsupported breakpoint count");
  }
  const int nseg = c.n_breakpoints + 1;
  for (int i = 0; i + 1 < c.n_breakpoints; ++i) {
    if (!(c.breakpoints[i] < c.breakpoints[i + 1])) {
      return err->set(PDSIM_ERR_CONFIG, where + ".breakpoints[" + std::to_string(i + 1) +
                                            "]: breakpoints must be strictly ascending");
    }
  }
  for (int i = 0; i < nseg; ++i) {
    const std::string anchor = where + ".segments[" + std::to_string(i) + "]";
    if (!(c.alpha[i] >= 0.0) || !std::isfinite(c.alpha[i])) {
      return err->set(PDSIM_ERR_CONFIG, anchor + ".alpha: must be finite and >= 0");
    }
    if (!(c.beta[i] >= 0.0) || !std::isfinite(c.beta[i])) {
      return err->set(PDSIM_ERR_CONFIG, anchor + ".beta: must be finite and >= 0");
    }
    if (c.alpha[i] == 0.0 && c.beta[i] == 0.0) {
      return err->set(PDSIM_ERR_CONFIG, anchor + ": degenerate segment (alpha and beta both 0)");
    }
  }
  for (int i = 0; i < c.n_breakpoints; ++i) {
    const double bp = c.breakpoints[i];
    const double left = dadd(c.alpha[i], dmul(c.beta[i], bp));
    const double right = dadd(c.alpha[i + 1], dmul(c.beta[i + 1], bp));
    const double slack = 1e-9 * std::max(1.0, std::abs(left));
    if (right + slack < left) {
      return err->set(PDSIM_ERR_CONFIG, where + ".breakpoints[" + std::to_string(i) +
                                            "]: non-monotone transition");
    }
  }
  return true;
}

// ---- PerfProfile::validate (perf_model.cpp:95-153) ----
inline bool validate_profile(const pdsim_profile& p, HostError* err) {
  if (p.n_degrees <= 0) return err->set(PDSIM_ERR_CONFIG, "degrees: the supported degree set is empty");
  if (p.n_degrees > PDSIM_MAX_DEGREES) return err->set(PDSIM_ERR_CONFIG, "degrees: too many degrees");
  for (int i = 0; i < p.n_degrees; ++i) {
    const int d = p.degrees[i];
    if (!(d > 0 && (d & (d - 1)) == 0)) {
      return err->set(PDSIM_ERR_CONFIG, "degrees[" + std::to_string(i) + "]: " + std::to_string(d) +
                                            " is not a power of 2");
    }
    if (i > 0 && d <= p.degrees[i - 1]) return err->set(PDSIM_ERR_CONFIG, "degrees: must be strictly ascending");
  }
  if (p.kv_bytes_per_token <= 0) return err->set(PDSIM_ERR_CONFIG, "kv_bytes_per_token: must be > 0");
  if (p.gpu_memory_capacity <= 0) return err->set(PDSIM_ERR_CONFIG, "gpu_memory_capacity: must be > 0");
  if (!(p.history_weight >= 0.0) || !std::isfinite(p.history_weight)) {
    return err->set(PDSIM_ERR_CONFIG, "history_weight: must be finite and >= 0");
  }
  for (int i = 0; i < p.n_degrees; ++i) {
    const std::string d = std::to_string(p.degrees[i]);
    if (!validate_curve(p.prefill[i], "prefill_cost[degree=" + d + "]", err)) return false;
    if (!validate_curve(p.decode[i], "decode_cost[degree=" + d + "]", err)) return false;
  }
  for (int i = 0; i < p.n_degrees; ++i) {
    for (int j = 0; j < p.n_degrees; ++j) {
      if (!validate_curve(p.kv[i][j], "kv_cost[src=" + std::to_string(p.degrees[i]) +
                                          ", dst=" + std::to_string(p.degrees[j]) + "]",
                          err))
        return false;
    }
  }
  return true;
}

inline int degree_index(const pdsim_profile& p, int degree) {
  for (int i = 0; i < p.n_degrees; ++i)
    if (p.degrees[i] == degree) return i;
  return -1;
}

// ---- Coordinator ctor + SchedulerParams::validate ----
inline bool validate_params(const pdsim_sched_params& s, double ttft_thres, double itl_thres,
                            HostError* err) {
  if (!(s.alpha > 0.0 && s.alpha <= 1.0)) return err->set(PDSIM_ERR_CONFIG, "routing: alpha must be in (0, 1]");
  if (!(s.beta > 0.0 && s.beta <= 1.0)) return err->set(PDSIM_ERR_CONFIG, "routing: beta must be in (0, 1]");
  if (!(ttft_thres > 0.0) || !(itl_thres > 0.0)) {
    return err->set(PDSIM_ERR_CONFIG, "routing: SLO thresholds must be > 0");
  }
  if (s.routing < 0 || s.routing > 2) return err->set(PDSIM_ERR_CONFIG, "routing: unknown mode");
  if (s.window < 1) return err->set(PDSIM_ERR_CONFIG, "scheduler: window must be >= 1");
  if (!(s.stat_window > 0.0)) return err->set(PDSIM_ERR_CONFIG, "scheduler: stat_window must be > 0");
  return true;
}

// Packed (device-layout) copy of one trace.
struct PackedTrace {
  int32_t S = 0, R = 0, max_dec = 0, max_incr = 0;
  int64_t total_decode = 0;
  double ttft_thres = 0, itl_thres = 0;
  std::vector<double> arrival, delay;
  std::vector<int32_t> round_off, incr, dec, rank, by_rank;
  std::vector<int64_t> sid;
  std::vector<int64_t> first_round_incr;  // for the KV precheck
  int64_t max_first_incr = 0;              // its maximum: the precheck of a plan is one comparison
  // the replay engine's record tables (engine.cuh SessTr / RoundTr)
  std::vector<SessTr> stab;   // [sess_table_len(S)]
  std::vector<RoundTr> rtab;  // [R]
  size_t device_bytes() const {  // what the replay engine reads from HBM
    return stab.size() * sizeof(SessTr) + rtab.size() * sizeof(RoundTr) + by_rank.size() * 4 + sid.size() * 8;
  }
};

// ---- Trace::validate (workload.cpp:90-134) + packing ----
inline bool pack_trace(const pdsim_trace& t, PackedTrace* out, HostError* err) {
  if (!(t.ttft_thres > 0.0) || !(t.itl_thres > 0.0)) {
    return err->set(PDSIM_ERR_CONFIG, "trace: slo thresholds must be > 0");
  }
  if (t.n_sessions < 0 || t.n_sessions > INT32_MAX / 2) return err->set(PDSIM_ERR_CONFIG, "trace: bad session count");
  const int64_t S = t.n_sessions;
  if (S > 0 && (!t.session_id || !t.arrival_time || !t.round_offset)) {
    return err->set(PDSIM_ERR_CONFIG, "trace: null array");
  }
  if (S > 0 && t.round_offset[0] != 0) return err->set(PDSIM_ERR_CONFIG, "trace: round_offset[0] must be 0");
  const int64_t R = S > 0 ? t.round_offset[S] : 0;
  if (R != t.n_rounds || R < 0 || R > INT32_MAX / 2) return err->set(PDSIM_ERR_CONFIG, "trace: bad round count");
  if (R > 0 && (!t.incr_input_len || !t.decode_len || !t.interaction_delay)) {
    return err->set(PDSIM_ERR_CONFIG, "trace: null array");
  }
  out->S = static_cast<int32_t>(S);
  out->R = static_cast<int32_t>(R);
  out->ttft_thres = t.ttft_thres;
  out->itl_thres = t.itl_thres;
  out->arrival.assign(t.arrival_time, t.arrival_time + S);
  out->sid.assign(t.session_id, t.session_id + S);
  out->round_off.resize(static_cast<size_t>(S + 1));
  out->incr.resize(static_cast<size_t>(R));
  out->dec.resize(static_cast<size_t>(R));
  out->delay.assign(t.interaction_delay, t.interaction_delay + R);
  out->first_round_incr.resize(static_cast<size_t>(S));
  out->max_dec = 0;
  out->max_first_incr = 0;
  out->max_incr = 0;
  out->total_decode = 0;
  // Duplicate ids are found after the id sort below (adjacent equal ids).
  // The reference checks them first for each session in trace order
  // (workload.cpp:90-134), so an error at session i (or a duplicate found
  // by the sort) reports the first session j <= i whose id repeats, if any.
  auto dup_error = [&](int64_t upto) -> bool {
    std::unordered_set<int64_t> seen;
    for (int64_t j = 0; j <= upto && j < S; ++j) {
      if (!seen.insert(t.session_id[j]).second) {
        err->set(PDSIM_ERR_CONFIG, "trace: session[" + std::to_string(j) + "] (id " + std::to_string(t.session_id[j]) +
                                       "): duplicate session_id");
        return true;
      }
    }
    return false;
  };
  auto fail_at = [&](int64_t i, const std::string& msg) -> bool {
    if (dup_error(i)) return false;
    return err->set(PDSIM_ERR_CONFIG, msg);
  };
  double prev_arrival = 0.0;
  for (int64_t i = 0; i < S; ++i) {
    // error texts are built only on the failing path (the loop runs per round)
    auto where = [&] { return "session[" + std::to_string(i) + "] (id " + std::to_string(t.session_id[i]) + ")"; };
    if (t.arrival_time[i] < 0.0) return fail_at(i, "trace: " + where() + ": arrival_time must be >= 0");
    if (i > 0 && t.arrival_time[i] < prev_arrival) {
      return fail_at(i, "trace: " + where() + ": sessions must be sorted by arrival_time");
    }
    prev_arrival = t.arrival_time[i];
    const int64_t b = t.round_offset[i], e = t.round_offset[i + 1];
    if (e <= b) return fail_at(i, "trace: " + where() + ": rounds must be non-empty");
    if (e > R) return fail_at(i, "trace: " + where() + ": round_offset out of range");
    if (e - b > 32000) return fail_at(i, "trace: " + where() + ": too many rounds for the device layout");
    int64_t ctx = 0;
    for (int64_t r = b; r < e; ++r) {
      auto ra = [&] { return where() + ".rounds[" + std::to_string(r - b) + "]"; };
      const int64_t inc = t.incr_input_len[r], dl = t.decode_len[r];
      if (inc < 1) return fail_at(i, "trace: " + ra() + ": incr_input_len must be >= 1");
      if (dl < 1) return fail_at(i, "trace: " + ra() + ": decode_len must be >= 1");
      if (t.interaction_delay[r] < 0.0) return fail_at(i, "trace: " + ra() + ": interaction_delay must be >= 0");
      if (r + 1 == e && t.interaction_delay[r] != 0.0) {
        return fail_at(i, "trace: " + ra() + ": final round must have interaction_delay 0");
      }
      ctx += inc + dl;
      if (ctx > INT32_MAX / 2) return fail_at(i, "trace: " + where() + ": context too long for the device layout");
      out->incr[static_cast<size_t>(r)] = static_cast<int32_t>(inc);
      out->dec[static_cast<size_t>(r)] = static_cast<int32_t>(dl);
      out->max_dec = std::max<int32_t>(out->max_dec, static_cast<int32_t>(dl));
      out->max_incr = std::max<int32_t>(out->max_incr, static_cast<int32_t>(inc));
      out->total_decode += dl;
    }
    out->round_off[static_cast<size_t>(i)] = static_cast<int32_t>(b);
    out->first_round_incr[static_cast<size_t>(i)] = t.incr_input_len[b];
    out->max_first_incr = std::max<int64_t>(out->max_first_incr, t.incr_input_len[b]);
  }
  if (S > 0 && t.round_offset[S] != R) return err->set(PDSIM_ERR_CONFIG, "trace: round_offset end mismatch");
  out->round_off[static_cast<size_t>(S)] = static_cast<int32_t>(R);
  // Rank of each session id: cohorts run in ascending id order
  // (decode_batch is sorted by id, sim_engine.cpp:482, 515-516).
  out->by_rank.resize(static_cast<size_t>(S));
  std::iota(out->by_rank.begin(), out->by_rank.end(), 0);
  std::sort(out->by_rank.begin(), out->by_rank.end(),
            [&](int32_t a, int32_t b) { return t.session_id[a] < t.session_id[b]; });
  for (int64_t k = 1; k < S; ++k) {
    if (t.session_id[out->by_rank[static_cast<size_t>(k)]] == t.session_id[out->by_rank[static_cast<size_t>(k - 1)]]) {
      dup_error(S - 1);
      return false;
    }
  }
  out->rank.resize(static_cast<size_t>(S));
  for (int32_t k = 0; k < static_cast<int32_t>(S); ++k) out->rank[static_cast<size_t>(out->by_rank[k])] = k;
  out->stab.assign(static_cast<size_t>(sess_table_len(S)), SessTr{0.0, static_cast<int32_t>(R), 0});
  for (int64_t i = 0; i < S; ++i) {
    out->stab[static_cast<size_t>(i)] = SessTr{out->arrival[static_cast<size_t>(i)], out->round_off[static_cast<size_t>(i)],
                                              out->rank[static_cast<size_t>(i)]};
  }
  out->rtab.resize(static_cast<size_t>(R));
  for (int64_t r = 0; r < R; ++r) {
    out->rtab[static_cast<size_t>(r)] = RoundTr{out->incr[static_cast<size_t>(r)], out->dec[static_cast<size_t>(r)],
                                               out->delay[static_cast<size_t>(r)]};
  }
  return true;
}

// ---- DeploymentPlan::validate + build_workers (planner.cpp:304-321,
// sim_engine.cpp:175-203) ----
inline bool pack_plan(const pdsim_plan& p, const pdsim_profile& prof, DevPlan* out, HostError* err) {
  if (p.n_prefill_groups < 0 || p.n_prefill_groups > PDSIM_MAX_GROUPS || p.n_decode_groups < 0 ||
      p.n_decode_groups > PDSIM_MAX_GROUPS) {
    return err->set(PDSIM_ERR_CONFIG, "plan: bad group count");
  }
  for (int i = 0; i < p.n_prefill_groups; ++i) {
    if (p.prefill_degree[i] < 1 || p.prefill_count[i] < 1) {
      return err->set(PDSIM_ERR_CONFIG, "plan: x entries need degree >= 1 and count >= 1");
    }
    if (i > 0 && p.prefill_degree[i] <= p.prefill_degree[i - 1]) {
      return err->set(PDSIM_ERR_CONFIG, "plan: x degrees must be distinct and ascending");
    }
  }
  for (int i = 0; i < p.n_decode_groups; ++i) {
    if (p.decode_degree[i] < 1 || p.decode_count[i] < 1) {
      return err->set(PDSIM_ERR_CONFIG, "plan: y entries need degree >= 1 and count >= 1");
    }
    if (i > 0 && p.decode_degree[i] <= p.decode_degree[i - 1]) {
      return err->set(PDSIM_ERR_CONFIG, "plan: y degrees must be distinct and ascending");
    }
  }
  int P = 0, D = 0;
  for (int i = 0; i < p.n_prefill_groups; ++i) {
    const int di = degree_index(prof, p.prefill_degree[i]);
    if (di < 0) {
      return err->set(PDSIM_ERR_CONFIG, "plan: prefill degree " + std::to_string(p.prefill_degree[i]) +
                                            " not covered by profile");
    }
    for (int k = 0; k < p.prefill_count[i]; ++k) {
      if (P >= PDSIM_MAX_WORKERS) return err->set(PDSIM_ERR_CONFIG, "plan: too many prefill replicas");
      out->pdeg[P++] = static_cast<int8_t>(di);
    }
  }
  for (int i = 0; i < p.n_decode_groups; ++i) {
    const int di = degree_index(prof, p.decode_degree[i]);
    if (di < 0) {
      return err->set(PDSIM_ERR_CONFIG, "plan: decode degree " + std::to_string(p.decode_degree[i]) +
                                            " not covered by profile");
    }
    for (int k = 0; k < p.decode_count[i]; ++k) {
      if (D >= PDSIM_MAX_WORKERS || P + D >= 2 * PDSIM_MAX_WORKERS) {
        return err->set(PDSIM_ERR_CONFIG, "plan: too many decode replicas");
      }
      out->ddeg[D++] = static_cast<int8_t>(di);
    }
  }
  if (D == 0) return err->set(PDSIM_ERR_CONFIG, "plan: at least one decode replica is required");
  if (P + D > PDSIM_MAX_WORKERS) return err->set(PDSIM_ERR_CONFIG, "plan: more than PDSIM_MAX_WORKERS replicas");
  if (D + 2 * P > kMaxSlots) {
    return err->set(PDSIM_ERR_CONFIG, "plan: decode + 2 x prefill replicas exceeds the engine's 64 event slots");
  }
  out->P = P;
  out->D = D;
  return true;
}

// precheck_sessions (sim_engine.cpp:217-231): true when every session's
// first round fits the largest decode worker.
inline bool precheck(const PackedTrace& t, const DevPlan& plan, const pdsim_profile& prof) {
  int64_t max_cap = 0;
  for (int d = 0; d < plan.D; ++d) {
    max_cap = std::max<int64_t>(max_cap, static_cast<int64_t>(prof.degrees[plan.ddeg[d]]) * prof.gpu_memory_capacity);
  }
  // some session's first round exceeds every decode worker <=> the largest
  // one does (kv_bytes_per_token > 0, validated)
  return !(t.max_first_incr * prof.kv_bytes_per_token > max_cap);
}

// Index of the first session (trace order) precheck_sessions would reject,
// -1 when none; and the reference's ConfigError text for it
// (sim_engine.cpp:217-231).
inline int64_t precheck_violator(const PackedTrace& t, const DevPlan& plan, const pdsim_profile& prof) {
  int64_t max_cap = 0;
  for (int d = 0; d < plan.D; ++d) {
    max_cap = std::max<int64_t>(max_cap, static_cast<int64_t>(prof.degrees[plan.ddeg[d]]) * prof.gpu_memory_capacity);
  }
  for (size_t i = 0; i < t.first_round_incr.size(); ++i) {
    if (t.first_round_incr[i] * prof.kv_bytes_per_token > max_cap) return static_cast<int64_t>(i);
  }
  return -1;
}

inline std::string precheck_message(const PackedTrace& t, int64_t i) {
  return "trace: session " + std::to_string(t.sid[static_cast<size_t>(i)]) +
         " first-round KV exceeds every decode worker's capacity";
}

inline DevParams to_dev_params(const pdsim_sched_params& s) {
  DevParams d;
  d.routing = s.routing;
  d.reorder = s.reorder != 0;
  d.window = s.window;
  d.reserved = 0;
  d.alpha = s.alpha;
  d.beta = s.beta;
  d.stat_window = s.stat_window;
  return d;
}

// Smallest value of a piecewise curve over loads >= lo: each segment is
// non-decreasing (beta >= 0), so the minimum sits at a segment's left end.
inline double curve_min_from(const pdsim_curve& c, double lo) {
  double m = INFINITY;
  for (int i = 0; i <= c.n_breakpoints; ++i) {
    const double left = i == 0 ? lo : std::max(lo, c.breakpoints[i - 1]);
    if (i < c.n_breakpoints && c.breakpoints[i] <= lo) continue;  // segment entirely below lo
    m = std::min(m, c.alpha[i] + c.beta[i] * left);
  }
  return m;
}

inline double curve_max_upto(const pdsim_curve& c, double hi) {
  double m = 0.0;
  for (int i = 0; i <= c.n_breakpoints; ++i) m = std::max(m, c.alpha[i] + c.beta[i] * hi);
  return m;
}

// Workspace capacities: provable upper bounds for every ring and heap of a
// replay.
// `dres`/`pres` (0: dmax/pmax) are the worker entries reserved in shared
// memory; the device picks them from a few compiled layouts.
inline Caps compute_caps(const std::vector<const PackedTrace*>& traces, int pmax, int dmax,
                         const pdsim_profile& prof, const pdsim_sched_params& prm, size_t smem_budget = 0,
                         int dres = 0, int pres = 0) {
  Caps c{};
  int64_t S = 1, R = 1, maxdec = 1, maxincr = 1, tdec = 1;
  for (const PackedTrace* t : traces) {
    S = std::max<int64_t>(S, t->S);
    R = std::max<int64_t>(R, t->R);
    maxdec = std::max<int64_t>(maxdec, t->max_dec);
    maxincr = std::max<int64_t>(maxincr, t->max_incr);
    tdec = std::max<int64_t>(tdec, t->total_decode);
  }
  double min_pre = INFINITY, min_dec = INFINITY, max_kv = 0.0;
  for (int i = 0; i < prof.n_degrees; ++i) {
    min_pre = std::min(min_pre, curve_min_from(prof.prefill[i], 1.0));
    min_dec = std::min(min_dec, curve_min_from(prof.decode[i], 1.0));
    for (int j = 0; j < prof.n_degrees; ++j) max_kv = std::max(max_kv, curve_max_upto(prof.kv[i][j], static_cast<double>(maxincr)));
  }
  const double W = prm.stat_window;
  int64_t tw = R + 2;
  if (min_pre > 0.0 && std::isfinite(min_pre)) {
    const double b = std::ceil((W + max_kv * 1.01) / (min_pre * (1.0 - 1e-6))) + 4.0;
    if (b < static_cast<double>(tw)) tw = static_cast<int64_t>(b);
  }
  int64_t iw = tdec + 2;
  if (min_dec > 0.0 && std::isfinite(min_dec)) {
    const double b = std::ceil(W / (min_dec * (1.0 - 1e-6))) + 4.0;
    if (b < static_cast<double>(iw)) iw = static_cast<int64_t>(b);
  }
  c.S = static_cast<int32_t>(S);
  c.pmax = std::max(pmax, 0);
  c.dmax = std::max(dmax, 1);
  c.dres = std::max(dres, c.dmax);
  c.pres = std::max(pres, std::max(c.pmax, 1));
  c.hcap = static_cast<int32_t>(S + 2 * c.pmax + c.dmax + 8);
  // Session-event heap entries kept in shared memory (the rest spills).
  c.hs = 1;
  {
    Caps probe = c;
    probe.hs = 0;
    const size_t fixed = smem_slot_bytes(probe, nullptr, nullptr);
    const size_t budget = smem_budget ? smem_budget : (size_t(48) << 10);
    const size_t room = budget > fixed ? (budget - fixed) / sizeof(HEv) : 1;
    c.hs = static_cast<int32_t>(std::max<size_t>(1, std::min<size_t>(room, static_cast<size_t>(c.hcap))));
  }
  c.qcap = static_cast<int32_t>(pow2_at_least(std::max<int64_t>(S, 2)));
  c.fcap = static_cast<int32_t>(std::max<int64_t>(S, 2));
  // Windows are trimmed lazily (at queries, or when full): twice the
  // in-window bound keeps forced trims rare.
  c.twcap = static_cast<int32_t>(pow2_at_least(std::max<int64_t>(2 * tw + 2, 4)));
  // Step segments retained: those in the ITL window (<= one per step in it)
  // plus those a running round may still fold (rounds span <= maxdec steps).
  c.segcap = static_cast<int32_t>(pow2_at_least(std::max<int64_t>(iw + maxdec + 16, 16)));
  c.maxdec = static_cast<int32_t>(maxdec);
  return c;
}

// Expands a records-mode replay's step log and round spans into the
// reference's per-token ItlSample stream (sim_engine.cpp:536-556): for each
// decode step in event order, every member of that worker's batch that is
// past its round's first token, in cohort order (ascending session id), with
// token_index = step - join + 1 and the step's gap. Returns the number of
// samples (writes at most `cap`).
inline int64_t expand_itl(const StepRec* steps, int64_t n_steps, const SpanRec* spans, int64_t n_spans,
                          const PackedTrace& t, int n_workers, pdsim_itl_sample* out, int64_t cap) {
  struct Lane {
    std::vector<int32_t> order;  // span indices by (first ITL step, rank)
    size_t next = 0;
    std::set<std::pair<int32_t, int32_t>> active;  // (rank, span)
    std::priority_queue<std::pair<int32_t, int32_t>, std::vector<std::pair<int32_t, int32_t>>,
                        std::greater<std::pair<int32_t, int32_t>>>
        ends;  // (end step, span)
  };
  std::vector<Lane> w(static_cast<size_t>(std::max(n_workers, 1)));
  for (int64_t j = 0; j < n_spans; ++j) {
    const SpanRec& sp = spans[j];
    if (sp.end < sp.join + 1 || sp.d < 0 || sp.d >= n_workers) continue;  // one-token rounds emit nothing
    w[static_cast<size_t>(sp.d)].order.push_back(static_cast<int32_t>(j));
  }
  for (Lane& l : w) {
    std::sort(l.order.begin(), l.order.end(), [&](int32_t a, int32_t b) {
      const int32_t sa = spans[a].join + 1, sb = spans[b].join + 1;
      if (sa != sb) return sa < sb;
      return t.rank[static_cast<size_t>(spans[a].sess)] < t.rank[static_cast<size_t>(spans[b].sess)];
    });
  }
  int64_t n = 0;
  for (int64_t q = 0; q < n_steps; ++q) {
    const StepRec& st = steps[q];
    if (st.d < 0 || st.d >= n_workers) continue;
    Lane& l = w[static_cast<size_t>(st.d)];
    while (l.next < l.order.size() && spans[l.order[l.next]].join + 1 <= st.k) {
      const int32_t j = l.order[l.next++];
      l.active.insert({t.rank[static_cast<size_t>(spans[j].sess)], j});
      l.ends.push({spans[j].end, j});
    }
    while (!l.ends.empty() && l.ends.top().first < st.k) {
      const int32_t j = l.ends.top().second;
      l.ends.pop();
      l.active.erase({t.rank[static_cast<size_t>(spans[j].sess)], j});
    }
    for (const auto& a : l.active) {
      const SpanRec& sp = spans[a.second];
      if (n < cap && out) {
        pdsim_itl_sample& o = out[n];
        o.session_id = t.sid[static_cast<size_t>(sp.sess)];
        o.round = sp.round;
        o.token_index = st.k - sp.join + 1;
        o.completion_time = st.t;
        o.value = st.gap;
      }
      ++n;
    }
  }
  return n;
}

// Runs f(0..n-1) on all host threads (static interleave; small n runs inline).
template <class F>
inline void parallel_for(size_t n, F&& f) {
  const size_t nt = std::min<size_t>(n, std::max(1u, std::thread::hardware_concurrency()));
  if (nt <= 1 || n < 16) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  for (size_t t = 0; t < nt; ++t) {
    pool.emplace_back([&, t] {
      for (size_t i = t; i < n; i += nt) f(i);
    });
  }
  for (auto& th : pool) th.join();
}

// Host-side sort of session outcomes by id (sim_engine.cpp:165-168).
inline void sort_outcomes(pdsim_session_outcome* s, int64_t n) {
  std::sort(s, s + n, [](const pdsim_session_outcome& a, const pdsim_session_outcome& b) {
    return a.session_id < b.session_id;
  });
}

}  // namespace pdg
