// pdsim/metrics.hpp — drop-in Report types and build_report (reference
// proj/include/pdsim/metrics.hpp:32-60, proj/src/metrics.cpp:108-190).
// The raw-sample CSV writers of `pdsim simulate` (byte-identical, std::to_chars
// numbers), their parsers, and the report text / JSON / comparison formats
// (metrics.cpp:198-474) are host document I/O over the same types. The
// batched search can compute the Report per pair on the device
// (SearchOptions::report).
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "pdsim/sim_engine.hpp"

namespace pdsim {

struct MetricStat {
  double mean = 0.0;
  double p95 = 0.0;
  std::int64_t count = 0;
};

struct Report {
  std::string trace_name;
  bool empty = false;  // no sessions and no samples
  std::int64_t sessions_total = 0;
  std::int64_t sessions_completed = 0;
  double slo_attainment = 0.0;
  double ttft_attainment = 0.0;
  double itl_attainment = 0.0;
  MetricStat ttft_initial;
  MetricStat ttft_incremental;
  MetricStat itl;
  double e2e_mean = 0.0;
  double local_fraction = 0.0;
};

// Nearest-rank percentile: index ceil(q*n) on the 1-based sorted list; empty
// input yields 0 (metrics.cpp:125-136). Throws DomainError for q outside (0, 1].
double percentile_nearest_rank(std::vector<double> values, double q);

// Raw-sample CSVs (metrics.cpp:350-474): header line, one row per record.
std::string ttft_csv(const std::vector<TtftSample>& samples);
std::string itl_csv(const std::vector<ItlSample>& samples);
std::string sessions_csv(const std::vector<SessionOutcome>& sessions);
std::string decisions_csv(const std::vector<DecisionRecord>& decisions);

// Parsers of the three sample CSVs (ParseError naming file, line and column);
// text -> records -> text is the identity.
std::vector<TtftSample> parse_ttft_csv(const std::string& text);
std::vector<ItlSample> parse_itl_csv(const std::string& text);
std::vector<SessionOutcome> parse_sessions_csv(const std::string& text);

// Human-readable report (fixed, 4 digits) and report_v1 JSON.
std::string format_report(const Report& report);
std::string report_to_json(const Report& report);

// Side-by-side comparison of named reports: aligned text table, and CSV.
std::string comparison_table(const std::vector<std::pair<std::string, Report>>& reports);
std::string comparison_csv(const std::vector<std::pair<std::string, Report>>& reports);

Report build_report(const SimResult& result);
Report build_report_from_samples(const std::string& trace_name, std::int64_t sessions_total,
                                 const std::vector<TtftSample>& ttft, const std::vector<ItlSample>& itl,
                                 const std::vector<SessionOutcome>& sessions);

}  // namespace pdsim
