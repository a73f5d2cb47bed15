// tests/native/hostsim.cpp — TEST-ONLY host build of the device replay engine.
//
// Compiles paper_2602_14516_b200/csrc/engine.cuh for the CPU so the engine's
// logic can be compared with the reference on every CPU test run (this
// container has no GPU). It is not part of the product: nothing in the
// package loads libhostsim.so, and the product's C-ABI has no CPU path.
#include <cstring>
#include <string>
#include <vector>

#include "engine.cuh"
#include "pack.hpp"
#include "pdsim_gpu.h"

namespace {
thread_local std::string g_err;
size_t g_smem_budget = 0;  // 0: the device default; small values force heap spills
thread_local pdsim_report* g_report_out = nullptr;  // hostsim_run_report: report mode
int fail(const pdg::HostError& e) {
  g_err = e.msg;
  return e.code;
}
}  // namespace

extern "C" {

const char* hostsim_last_error(void) { return g_err.c_str(); }

// Same contract as pdsim_gpu_run.
int hostsim_run(const pdsim_trace* trace, const pdsim_plan* plan, const pdsim_profile* prof,
                const pdsim_sched_params* params, uint64_t seed, pdsim_run_output* out) {
  pdg::HostError err;
  if (!pdg::validate_params(*params, trace->ttft_thres, trace->itl_thres, &err)) return fail(err);
  pdg::PackedTrace t;
  if (!pdg::pack_trace(*trace, &t, &err)) return fail(err);
  if (!pdg::validate_profile(*prof, &err)) return fail(err);
  if (params->reorder && params->window > 8 && t.S > 0) {
    err.set(PDSIM_ERR_CONFIG, "reorder: window must be <= 8");
    return fail(err);
  }
  pdg::DevPlan dp;
  std::memset(&dp, 0, sizeof(dp));
  if (!pdg::pack_plan(*plan, *prof, &dp, &err)) return fail(err);
  if (!pdg::precheck(t, dp, *prof)) {
    err.set(PDSIM_ERR_CONFIG, "trace: a session's first-round KV exceeds every decode worker's capacity");
    return fail(err);
  }
  pdg::Caps caps = pdg::compute_caps({&t}, dp.P, dp.D, *prof, *params, g_smem_budget);
  if (g_report_out) {
    caps.rep_r = std::max<int32_t>(t.R, 1);
    caps.rep_gapcap = 1 << 16;
  }
  std::vector<char> gws(pdg::global_slot_bytes(caps, nullptr, nullptr) + 256);
  std::vector<char> sws(pdg::smem_slot_bytes(caps, nullptr, nullptr) + 256);
  auto align = [](std::vector<char>& v) {
    return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(v.data()) + 255) & ~uintptr_t(255));
  };
  pdg::GlobalSlot gslot;
  pdg::global_slot_bytes(caps, &gslot, align(gws));
  pdg::SmemSlot sslot;
  pdg::smem_slot_bytes(caps, &sslot, align(sws));
  pdg::DevTrace dt;
  dt.S = t.S;
  dt.R = t.R;
  dt.max_dec = t.max_dec;
  dt.rank_is_index = 1;
  for (size_t k = 0; k < t.by_rank.size(); ++k) dt.rank_is_index &= t.by_rank[k] == static_cast<int32_t>(k) ? 1 : 0;
  dt.ttft_thres = t.ttft_thres;
  dt.itl_thres = t.itl_thres;
  dt.ss = t.stab.data();
  dt.rr = t.rtab.data();
  dt.sid = t.sid.data();
  dt.by_rank = t.by_rank.data();
  const pdg::DevParams dprm = pdg::to_dev_params(*params);
  pdg::Records rec{out->decisions, out->ttft_samples, out->sessions, nullptr, nullptr, 0};
  std::vector<pdg::StepRec> steps;
  std::vector<pdg::SpanRec> spans;
  if (out->itl_samples) {
    steps.resize(static_cast<size_t>(std::max<int64_t>(t.total_decode, 1)));
    spans.resize(static_cast<size_t>(std::max<int32_t>(t.R, 1)));
    rec.steps = steps.data();
    rec.spans = spans.data();
    rec.steps_cap = static_cast<int64_t>(steps.size());
  }
  pdg::host_profile() = prof;
  pdg::Engine eng(sslot.es, dt, dp, dprm, caps, sslot, gslot, rec, seed);
  pdg::PairResult res;
  std::memset(&res, 0, sizeof(res));
  eng.run(&res);
  if (g_report_out) eng.build_report(g_report_out);
  if (res.status != PDSIM_PAIR_OK) {
    err.set(PDSIM_ERR_INTERNAL, "engine capacity or invariant violated");
    return fail(err);
  }
  out->n_decisions = res.n_decisions;
  out->n_ttft = res.n_ttft;
  out->n_sessions = res.att.sessions_completed;
  out->counters = res.ctr;
  out->attainment = res.att;
  if (out->sessions) pdg::sort_outcomes(out->sessions, out->n_sessions);
  out->n_itl = 0;
  if (out->itl_samples) {
    out->n_itl = pdg::expand_itl(steps.data(), res.n_steps, spans.data(), res.n_spans, t, dp.D, out->itl_samples,
                                 out->itl_capacity);
  }
  return PDSIM_OK;
}

}  // extern "C"

extern "C" void hostsim_set_smem_budget(size_t bytes) { g_smem_budget = bytes; }

extern "C" double hostsim_fold_repeat(double s, double g, uint64_t count) {
  return pdg::fold_repeat(s, g, count);
}

// Counts only (no record arrays): exercises the search-mode paths (certified
// per-session ITL verdicts) exactly as the batched GPU search runs them.
extern "C" int hostsim_run_counts(const pdsim_trace* trace, const pdsim_plan* plan, const pdsim_profile* prof,
                                  const pdsim_sched_params* params, uint64_t seed, pdsim_run_output* out) {
  pdsim_run_output o = *out;
  o.decisions = nullptr;
  o.ttft_samples = nullptr;
  o.sessions = nullptr;
  o.itl_samples = nullptr;
  const int rc = hostsim_run(trace, plan, prof, params, seed, &o);
  out->n_decisions = o.n_decisions;
  out->n_ttft = o.n_ttft;
  out->n_sessions = o.n_sessions;
  out->counters = o.counters;
  out->attainment = o.attainment;
  return rc;
}

// Report mode (search pair_report path): build_report of the replay.
extern "C" int hostsim_run_report(const pdsim_trace* trace, const pdsim_plan* plan, const pdsim_profile* prof,
                                  const pdsim_sched_params* params, uint64_t seed, pdsim_report* report) {
  pdsim_run_output o;
  std::memset(&o, 0, sizeof(o));
  g_report_out = report;
  const int rc = hostsim_run(trace, plan, prof, params, seed, &o);
  g_report_out = nullptr;
  return rc;
}
