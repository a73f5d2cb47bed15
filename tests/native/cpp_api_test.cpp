// tests/native/cpp_api_test.cpp — exercises the C++ drop-in API
// (include/pdsim/*.hpp) the way the reference's own suites do
// (proj/tests/sim_engine_test.cpp): closed-form timelines, conservation,
// determinism, config errors, and a small batched search. Needs a B200.
#include <cmath>
#include <cstdio>
#include <map>
#include <cstdlib>
#include <string>

#include "pdsim/errors.hpp"
#include "pdsim/metrics.hpp"
#include "pdsim/plan_search.hpp"
#include "pdsim/planner.hpp"
#include "pdsim/sim_engine.hpp"
#include "pdsim/workload.hpp"

using namespace pdsim;

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                  \
    }                                                              \
  } while (0)

static bool near(double a, double b) { return std::fabs(a - b) <= 1e-12 * std::max(1.0, std::fabs(b)); }

static std::uint64_t fnv1a(const std::string& text) {
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : text) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

static DeploymentPlan simple_plan(int prefill, int decode, int degree = 1) {
  DeploymentPlan plan;
  if (prefill > 0) plan.x[degree] = prefill;
  plan.y[degree] = decode;
  plan.feasible = true;
  plan.gpus_used = plan.gpus();
  return plan;
}

int main() {
  const PerfProfile p = synth_profile(SynthProfileSpec{}, 4);
  Trace t;
  t.name = "manual";
  t.slo = {5.0, 0.5};
  SessionSpec s;
  s.session_id = 0;
  s.arrival_time = 0.0;
  s.rounds = {{700, 3, 0.5}, {250, 2, 0.0}};
  t.sessions.push_back(s);

  // Remote path timeline (sim_engine_test.cpp:75-119).
  SchedulerParams remote;
  remote.routing = RoutingMode::kAlwaysRemote;
  const SimResult r = run(t, simple_plan(1, 1), p, remote, 1);
  const ParallelismStrategy th{1};
  const double td = t_decode(p, 1, th);
  const double t1 = t_prefill(p, 0, 700, th) + t_kv(p, 700, th, th);
  const double i1 = t1 + 3.0 * td + 0.5;
  const double t2 = t_kv(p, 703, th, th) + t_prefill(p, 703, 250, th) + t_kv(p, 250, th, th);
  const double end = i1 + t2 + 2.0 * td;
  CHECK(r.ttft_samples.size() == 2);
  CHECK(near(r.ttft_samples[0].value, t1));
  CHECK(near(r.ttft_samples[1].value, t2));
  CHECK(r.sessions.size() == 1 && near(r.sessions[0].completion_time, end));
  CHECK(r.counters.tokens_decoded == 5 && r.counters.kv_bytes_residual == 0);

  // Idle-cluster TTFT equals the estimate exactly (sim_engine_test.cpp:269-294).
  Trace one = t;
  one.sessions[0].rounds = {{500, 2, 0.0}};
  const SimResult rr = run(one, simple_plan(1, 1), p, remote, 1);
  CHECK(rr.ttft_samples[0].value == t_prefill(p, 0, 500, th) + t_kv(p, 500, th, th));

  // Conservation on a generated workload (sim_engine_test.cpp:141-167).
  const Trace gen = gen_trace(preset_stats("toolbench"), 6.0, 300, 21);
  std::int64_t rounds = 0, decode = 0;
  for (const SessionSpec& x : gen.sessions) {
    rounds += static_cast<std::int64_t>(x.rounds.size());
    decode += x.total_decode();
  }
  for (RoutingMode mode : {RoutingMode::kAdaptive, RoutingMode::kAlwaysRemote, RoutingMode::kAlwaysLocal}) {
    SchedulerParams prm;
    prm.routing = mode;
    const SimResult g = run(gen, simple_plan(2, 2), p, prm, 5);
    CHECK(g.sessions.size() == 300);
    CHECK(g.counters.tasks_created == rounds && g.counters.tasks_completed == rounds);
    CHECK(g.counters.tokens_decoded == decode && g.counters.kv_bytes_residual == 0);
    CHECK(static_cast<std::int64_t>(g.decisions.size()) == rounds);
  }

  // Determinism (sim_engine_test.cpp:169-179).
  const Trace gaia = gen_trace(preset_stats("gaia"), 4.0, 150, 8);
  const SimResult a = run(gaia, simple_plan(2, 2), p, SchedulerParams{}, 33);
  const SimResult b = run(gaia, simple_plan(2, 2), p, SchedulerParams{}, 33);
  CHECK(a.decisions.size() == b.decisions.size());
  for (size_t k = 0; k < a.decisions.size() && k < b.decisions.size(); ++k) {
    CHECK(a.decisions[k].time == b.decisions[k].time && a.decisions[k].worker == b.decisions[k].worker);
  }

  // Validation (sim_engine_test.cpp:306-331).
  bool threw = false;
  try {
    DeploymentPlan no_decode;
    no_decode.x[1] = 1;
    no_decode.feasible = true;
    no_decode.gpus_used = 1;
    run(t, no_decode, p, SchedulerParams{}, 1);
  } catch (const ConfigError&) {
    threw = true;
  }
  CHECK(threw);

  // Batched search over the 13 N=4 candidates.
  const std::vector<DeploymentPlan> cands = enumerate_plans({1, 2, 4, 8}, 4);
  CHECK(cands.size() == 13);
  const SearchResult sr = plan_search({gen}, cands, p, SchedulerParams{}, 1);
  CHECK(sr.best_candidate >= 0 && sr.pairs.size() == 13);
  std::int64_t best = -1;
  for (size_t c = 0; c < cands.size(); ++c) {
    const SimResult one_run = run(gen, cands[c], p, SchedulerParams{}, 1);
    std::int64_t ok = 0;
    for (const SessionOutcome& o : one_run.sessions) ok += o.slo_ok;
    CHECK(ok == sr.candidate_slo_ok[c]);
    if (ok > best) best = ok;
  }
  CHECK(sr.best_slo_ok == best);

  // SimResult::itl_samples: one per token after each round's first, and every
  // session's mean_itl is the sequential mean of its samples in push order
  // (sim_engine.cpp:544-556, 602).
  {
    const SimResult r = run(gen, simple_plan(2, 2), p, SchedulerParams{}, 5);
    std::map<std::int64_t, std::pair<double, std::int64_t>> acc;
    for (const ItlSample& x : r.itl_samples) {
      auto& a = acc[x.session_id];
      a.first += x.value;
      a.second += 1;
      CHECK(x.token_index >= 2 && x.value > 0.0);
    }
    std::int64_t expect = 0;
    for (const SessionOutcome& o : r.sessions) {
      const auto it = acc.find(o.session_id);
      const double mean = it == acc.end() ? 0.0 : it->second.first / static_cast<double>(it->second.second);
      CHECK(mean == o.mean_itl);
      for (const SessionSpec& ss : gen.sessions)
        if (ss.session_id == o.session_id)
          for (const Round& rd : ss.rounds) expect += rd.decode_len - 1;
    }
    CHECK(static_cast<std::int64_t>(r.itl_samples.size()) == expect);
  }

  // Report (metrics.cpp:138-190): the device's per-pair report in the search
  // equals build_report over the drop-in run()'s full SimResult.
  {
    SearchOptions so;
    so.report = true;
    const std::vector<DeploymentPlan> few = {simple_plan(1, 1), simple_plan(2, 2)};
    const SearchResult sr2 = plan_search({gen}, few, p, SchedulerParams{}, 3, so);
    CHECK(sr2.reports.size() == 2);
    for (size_t c = 0; c < few.size() && c < sr2.reports.size(); ++c) {
      const Report want = build_report(run(gen, few[c], p, SchedulerParams{}, 3));
      const Report& got = sr2.reports[c];
      CHECK(got.sessions_completed == want.sessions_completed && got.slo_attainment == want.slo_attainment);
      CHECK(got.ttft_initial.mean == want.ttft_initial.mean && got.ttft_initial.p95 == want.ttft_initial.p95);
      CHECK(got.ttft_incremental.mean == want.ttft_incremental.mean &&
            got.ttft_incremental.p95 == want.ttft_incremental.p95);
      CHECK(got.itl.mean == want.itl.mean && got.itl.p95 == want.itl.p95 && got.itl.count == want.itl.count);
      CHECK(got.e2e_mean == want.e2e_mean && got.local_fraction == want.local_fraction);
    }
  }

  // `pdsim simulate`'s raw-sample CSVs (metrics.cpp:350-474) of the survey
  // fingerprint scenario: dureader 4000 sessions @16 seed
  // 101, P:2x1 D:2x1, profile seed 7, engine seed 2 -> the reference's FNV-1a
  // hashes of decisions / ttft / sessions / itl CSV text.
  {
    const PerfProfile fp = synth_profile(SynthProfileSpec{}, 7);
    const Trace ft = gen_trace(preset_stats("dureader"), 16.0, 4000, 101);
    const SimResult fr = run(ft, simple_plan(2, 2), fp, SchedulerParams{}, 2);
    CHECK(fnv1a(decisions_csv(fr.decisions)) == 0x665772a5ffd1e99full);
    CHECK(fnv1a(ttft_csv(fr.ttft_samples)) == 0xe4e6dd847853dbaeull);
    CHECK(fnv1a(sessions_csv(fr.sessions)) == 0x2038a6a05715eebbull);
    CHECK(fnv1a(itl_csv(fr.itl_samples)) == 0xbd3adf1d08563504ull);
  }

  // SearchOptions::prune (argmax mode): same winner and count as the full search.
  {
    const std::vector<DeploymentPlan> cands = enumerate_plans({1, 2, 4}, 8);
    const SearchResult full = plan_search({gen}, cands, p, SchedulerParams{}, 3);
    SearchOptions so;
    so.prune = true;
    const SearchResult pr = plan_search({gen}, cands, p, SchedulerParams{}, 3, so);
    CHECK(pr.best_candidate == full.best_candidate && pr.best_slo_ok == full.best_slo_ok);
    for (size_t c = 0; c < cands.size(); ++c) {
      CHECK(pr.candidate_slo_ok[c] == -2 || pr.candidate_slo_ok[c] == full.candidate_slo_ok[c]);
    }
  }

  // SearchOptions::devices (pdsim_multi_plan_search: shards over the listed
  // GPUs, NCCL all-reduce of the counts): the same search result.
  {
    const std::vector<DeploymentPlan> cands = enumerate_plans({1, 2, 4}, 8);
    const Trace gen3 = gen_trace(preset_stats("hotpotqa"), 12.0, 150, 21);
    const SearchResult one = plan_search({gen, gen3}, cands, p, SchedulerParams{}, 3);
    SearchOptions so;
    so.devices = {0};
    const SearchResult md = plan_search({gen, gen3}, cands, p, SchedulerParams{}, 3, so);
    CHECK(md.best_candidate == one.best_candidate && md.best_slo_ok == one.best_slo_ok);
    CHECK(md.candidate_slo_ok == one.candidate_slo_ok);
    CHECK(md.pairs.size() == one.pairs.size());
    for (size_t k = 0; k < md.pairs.size(); ++k) {
      CHECK(md.pairs[k].slo_ok == one.pairs[k].slo_ok && md.pairs[k].valid == one.pairs[k].valid);
    }
  }

  // sweep() (pdsim sweep, pdsim.cpp:501-590): one launch over traces x
  // settings; each report equals build_report of run() under that setting.
  {
    SchedulerParams a, b;
    a.alpha = 0.5;
    b.beta = 0.3;
    b.window = 1;
    const std::vector<SchedulerParams> sets = {a, b};
    const Trace gen2 = gen_trace(preset_stats("toolbench"), 16.0, 120, 5);
    const std::vector<Trace> trs = {gen, gen2};
    const std::vector<Report> reps = sweep(trs, simple_plan(1, 1), p, sets, 3);
    CHECK(reps.size() == 4);
    for (size_t k = 0; k < sets.size(); ++k) {
      for (size_t r = 0; r < trs.size() && reps.size() == 4; ++r) {
        const Report want = build_report(run(trs[r], simple_plan(1, 1), p, sets[k], 3));
        const Report& got = reps[k * trs.size() + r];
        CHECK(got.slo_attainment == want.slo_attainment && got.itl.p95 == want.itl.p95 &&
              got.ttft_initial.p95 == want.ttft_initial.p95 && got.e2e_mean == want.e2e_mean);
      }
    }
    const std::string csv = sweep_csv({8.0, 16.0}, sets, reps);
    CHECK(csv.rfind("rate,alpha,beta,window,", 0) == 0);
    CHECK(csv.find("\n8,0.5,0.85,3,") != std::string::npos && csv.find("\n16,0.9,0.3,1,") != std::string::npos);
    bool threw = false;
    try {
      SchedulerParams bad;
      bad.alpha = -1.0;
      sweep(trs, simple_plan(1, 1), p, {bad}, 3);
    } catch (const ConfigError&) {
      threw = true;
    }
    CHECK(threw);
  }

  // Surrogate planner (planner.hpp:55-113): the coefficient pipeline and the
  // solver behave like the reference's planner_test properties.
  {
    const std::vector<int> ds = {1, 2, 4, 8};
    const LatencyCoefficients c1 = estimate_coefficients(preset_stats("toolbench"), 8.0, p, ds, 8, 42);
    const LatencyCoefficients c2 = estimate_coefficients(preset_stats("toolbench"), 8.0, p, ds, 8, 42);
    CHECK(c1.tau_pre == c2.tau_pre && c1.tau_dec == c2.tau_dec);  // deterministic per seed
    CHECK(c1.provenance == "rate=8 sessions=256 gpus=8 seed=42 degrees=[1,2,4,8]");
    for (const auto& [d, tau] : c1.tau_pre) CHECK(tau > 0.0);
    const std::vector<LatencyCoefficients> batch =
        estimate_coefficients_batch(preset_stats("toolbench"), {8.0, 8.0}, {42, 42}, p, ds, 8);
    CHECK(batch.size() == 2 && batch[1].tau_dec == c1.tau_dec);
    const DeploymentPlan best = solve(c1, 8, ds);
    const std::vector<DeploymentPlan> ranked = top_k(c1, 8, ds, 5);
    CHECK(!ranked.empty() && ranked.front() == best);
    CHECK(best.gpus() <= 8 && best.prefill_replicas() >= 1 && best.decode_replicas() >= 1);
    bool bad = false;
    try {
      LatencyCoefficients missing;
      missing.tau_pre[1] = 0.1;
      solve(missing, 8, {1});  // no decode coefficient for degree 1
    } catch (const ConfigError&) {
      bad = true;
    }
    CHECK(bad);
    const PhaseSimResult pr = simulate_prefill_replica(gen, p, 2);
    const PhaseSimResult dr = simulate_decode_replica(gen, p, 2);
    std::int64_t rounds = 0;
    for (const SessionSpec& ss : gen.sessions) rounds += static_cast<std::int64_t>(ss.rounds.size());
    CHECK(pr.p95 > 0.0 && dr.p95 > 0.0 && pr.sample_count == rounds);
  }

  std::printf("cpp_api_test: %s (%d failures)\n", failures ? "FAIL" : "ok", failures);
  return failures ? 1 : 0;
}
