// metrics_io.cpp — Report text / JSON formatting, side-by-side comparisons
// and the raw-sample CSV parsers of the drop-in C++ API
// (include/pdsim/metrics.hpp; reference metrics.hpp:62-91).
//
// Host document I/O, off the replay path: `pdsim simulate`/`compare` write
// these files, and the reference's metrics_test rebuilds a Report from the
// CSV text to check bit identity. Formats follow metrics.cpp:198-474:
// fixed 4-digit report text, report_v1 JSON (nlohmann dump(2)), CSV numbers
// as std::to_chars shortest round-trip (parsed back with std::from_chars, so
// text -> value -> text is the identity), ParseError naming file and line.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <functional>
#include <iomanip>
#include <sstream>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "json.hpp"
#include "pdsim/errors.hpp"
#include "pdsim/metrics.hpp"

namespace pdsim {

namespace {

std::string shortest(double v) {
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, r.ptr);
}

std::string fixed4(double v) {
  std::ostringstream s;
  s << std::fixed << std::setprecision(4) << v;
  return s.str();
}

// One CSV document: exact header line, then rows of exactly `width` fields
// (blank lines skipped). Fields are comma-separated, no quoting.
class CsvReader {
 public:
  CsvReader(const std::string& text, std::string file, std::string_view header, size_t width)
      : text_(text), file_(std::move(file)), width_(width) {
    std::string first;
    if (!next_line(&first)) throw ParseError(file_, "empty file");
    if (first != header) throw ParseError(file_ + " line 1", "unexpected header '" + first + "'");
  }

  // Next non-empty row; false at the end.
  bool row(std::vector<std::string>* fields) {
    std::string line;
    while (next_line(&line)) {
      if (line.empty()) continue;
      where_ = file_ + " line " + std::to_string(line_no_);
      fields->clear();
      size_t start = 0;
      for (;;) {
        const size_t comma = line.find(',', start);
        fields->push_back(line.substr(start, comma == std::string::npos ? std::string::npos : comma - start));
        if (comma == std::string::npos) break;
        start = comma + 1;
      }
      if (fields->size() != width_) {
        throw ParseError(where_, "expected " + std::to_string(width_) + " fields, got " +
                                     std::to_string(fields->size()));
      }
      return true;
    }
    return false;
  }

  const std::string& where() const { return where_; }

  double number(const std::string& f, const char* col) const {
    double v = 0.0;
    const auto r = std::from_chars(f.data(), f.data() + f.size(), v);
    if (r.ec != std::errc() || r.ptr != f.data() + f.size()) {
      throw ParseError(where_ + " " + col, "expected a number, got '" + f + "'");
    }
    return v;
  }

  std::int64_t integer(const std::string& f, const char* col) const {
    std::int64_t v = 0;
    const auto r = std::from_chars(f.data(), f.data() + f.size(), v);
    if (r.ec != std::errc() || r.ptr != f.data() + f.size()) {
      throw ParseError(where_ + " " + col, "expected an integer, got '" + f + "'");
    }
    return v;
  }

  bool flag(const std::string& f, const char* col) const {
    if (f == "1") return true;
    if (f == "0") return false;
    throw ParseError(where_ + " " + col, "expected 0 or 1, got '" + f + "'");
  }

 private:
  bool next_line(std::string* out) {
    if (pos_ > text_.size() || (pos_ == text_.size())) return false;
    const size_t nl = text_.find('\n', pos_);
    *out = text_.substr(pos_, nl == std::string::npos ? std::string::npos : nl - pos_);
    pos_ = nl == std::string::npos ? text_.size() : nl + 1;
    ++line_no_;
    return true;
  }

  const std::string& text_;
  std::string file_;
  size_t width_;
  size_t pos_ = 0;
  size_t line_no_ = 0;
  std::string where_;
};

constexpr std::string_view kTtftHeader = "session_id,round,kind,local,created_time,completion_time,value";
constexpr std::string_view kItlHeader = "session_id,round,token_index,completion_time,value";
constexpr std::string_view kSessionsHeader =
    "session_id,arrival_time,completion_time,rounds,admission_wait,mean_itl,ttft_ok,itl_ok,slo_ok";

}  // namespace

std::vector<TtftSample> parse_ttft_csv(const std::string& text) {
  CsvReader in(text, "ttft_samples.csv", kTtftHeader, 7);
  std::vector<TtftSample> out;
  std::vector<std::string> f;
  while (in.row(&f)) {
    TtftSample s;
    s.session_id = in.integer(f[0], "session_id");
    s.round = static_cast<int>(in.integer(f[1], "round"));
    if (f[2] == "initial") {
      s.kind = TaskKind::kInitial;
    } else if (f[2] == "incremental") {
      s.kind = TaskKind::kIncremental;
    } else {
      throw ParseError(in.where() + " kind", "unknown kind '" + f[2] + "'");
    }
    s.local = in.flag(f[3], "local");
    s.created_time = in.number(f[4], "created_time");
    s.completion_time = in.number(f[5], "completion_time");
    s.value = in.number(f[6], "value");
    out.push_back(s);
  }
  return out;
}

std::vector<ItlSample> parse_itl_csv(const std::string& text) {
  CsvReader in(text, "itl_samples.csv", kItlHeader, 5);
  std::vector<ItlSample> out;
  std::vector<std::string> f;
  while (in.row(&f)) {
    ItlSample s;
    s.session_id = in.integer(f[0], "session_id");
    s.round = static_cast<int>(in.integer(f[1], "round"));
    s.token_index = static_cast<int>(in.integer(f[2], "token_index"));
    s.completion_time = in.number(f[3], "completion_time");
    s.value = in.number(f[4], "value");
    out.push_back(s);
  }
  return out;
}

std::vector<SessionOutcome> parse_sessions_csv(const std::string& text) {
  CsvReader in(text, "sessions.csv", kSessionsHeader, 9);
  std::vector<SessionOutcome> out;
  std::vector<std::string> f;
  while (in.row(&f)) {
    SessionOutcome s;
    s.session_id = in.integer(f[0], "session_id");
    s.arrival_time = in.number(f[1], "arrival_time");
    s.completion_time = in.number(f[2], "completion_time");
    s.rounds = static_cast<int>(in.integer(f[3], "rounds"));
    s.admission_wait = in.number(f[4], "admission_wait");
    s.mean_itl = in.number(f[5], "mean_itl");
    s.ttft_ok = in.flag(f[6], "ttft_ok");
    s.itl_ok = in.flag(f[7], "itl_ok");
    s.slo_ok = in.flag(f[8], "slo_ok");
    out.push_back(s);
  }
  return out;
}

std::string format_report(const Report& r) {
  std::ostringstream o;
  o << std::fixed << std::setprecision(4);
  o << "trace:             " << r.trace_name << "\n";
  if (r.empty) {
    o << "(empty result)\n";
    return o.str();
  }
  o << "sessions:          " << r.sessions_completed << "/" << r.sessions_total << " completed\n";
  o << "slo_attainment:    " << r.slo_attainment << "  (ttft " << r.ttft_attainment << ", itl " << r.itl_attainment
    << ")\n";
  const std::pair<const char*, const MetricStat*> stats[] = {
      {"ttft_initial:      ", &r.ttft_initial}, {"ttft_incremental:  ", &r.ttft_incremental}, {"itl:               ", &r.itl}};
  for (const auto& [label, s] : stats) {
    o << label << "mean " << s->mean << "s  p95 " << s->p95 << "s  (n=" << s->count << ")\n";
  }
  o << "e2e_mean:          " << r.e2e_mean << "s\n";
  o << "local_fraction:    " << r.local_fraction << "\n";
  return o.str();
}

std::string report_to_json(const Report& r) {
  auto stat = [](const MetricStat& s) { return nlohmann::json{{"mean", s.mean}, {"p95", s.p95}, {"count", s.count}}; };
  nlohmann::json j;
  j["version"] = "report_v1";
  j["trace_name"] = r.trace_name;
  j["empty"] = r.empty;
  j["sessions_total"] = r.sessions_total;
  j["sessions_completed"] = r.sessions_completed;
  j["slo_attainment"] = r.slo_attainment;
  j["ttft_attainment"] = r.ttft_attainment;
  j["itl_attainment"] = r.itl_attainment;
  j["ttft_initial"] = stat(r.ttft_initial);
  j["ttft_incremental"] = stat(r.ttft_incremental);
  j["itl"] = stat(r.itl);
  j["e2e_mean"] = r.e2e_mean;
  j["local_fraction"] = r.local_fraction;
  return j.dump(2) + "\n";
}

namespace {

using Cell = std::function<std::string(const Report&)>;

std::vector<std::pair<const char*, Cell>> comparison_cells() {
  auto num = [](double Report::*field) { return Cell([field](const Report& r) { return fixed4(r.*field); }); };
  auto stat = [](MetricStat Report::*s, double MetricStat::*f) {
    return Cell([s, f](const Report& r) { return fixed4((r.*s).*f); });
  };
  return {{"trace", [](const Report& r) { return r.trace_name; }},
          {"slo_attainment", num(&Report::slo_attainment)},
          {"ttft_attainment", num(&Report::ttft_attainment)},
          {"itl_attainment", num(&Report::itl_attainment)},
          {"ttft_initial_mean", stat(&Report::ttft_initial, &MetricStat::mean)},
          {"ttft_initial_p95", stat(&Report::ttft_initial, &MetricStat::p95)},
          {"ttft_incr_mean", stat(&Report::ttft_incremental, &MetricStat::mean)},
          {"ttft_incr_p95", stat(&Report::ttft_incremental, &MetricStat::p95)},
          {"itl_mean", stat(&Report::itl, &MetricStat::mean)},
          {"itl_p95", stat(&Report::itl, &MetricStat::p95)},
          {"e2e_mean", num(&Report::e2e_mean)},
          {"local_fraction", num(&Report::local_fraction)}};
}

}  // namespace

std::string comparison_table(const std::vector<std::pair<std::string, Report>>& reports) {
  std::ostringstream o;
  for (const auto& nr : reports) {
    if (nr.second.trace_name != reports.front().second.trace_name) {
      o << "warning: reports cover different traces\n";
      break;
    }
  }
  const auto cells = comparison_cells();
  size_t label_w = 0;
  for (const auto& c : cells) label_w = std::max(label_w, std::string(c.first).size());
  std::vector<size_t> col_w;
  for (const auto& [name, rep] : reports) {
    size_t w = name.size();
    for (const auto& c : cells) w = std::max(w, c.second(rep).size());
    col_w.push_back(w);
  }
  auto pad = [&](const std::string& s, size_t w) { o << std::left << std::setw(static_cast<int>(w) + 2) << s; };
  pad("metric", label_w);
  for (size_t i = 0; i < reports.size(); ++i) pad(reports[i].first, col_w[i]);
  o << "\n";
  for (const auto& c : cells) {
    pad(c.first, label_w);
    for (size_t i = 0; i < reports.size(); ++i) pad(c.second(reports[i].second), col_w[i]);
    o << "\n";
  }
  return o.str();
}

std::string comparison_csv(const std::vector<std::pair<std::string, Report>>& reports) {
  std::string out =
      "name,trace,sessions_completed,sessions_total,slo_attainment,ttft_attainment,itl_attainment,"
      "ttft_initial_mean,ttft_initial_p95,ttft_incr_mean,ttft_incr_p95,itl_mean,itl_p95,e2e_mean,local_fraction\n";
  for (const auto& [name, r] : reports) {
    const double nums[] = {r.slo_attainment,          r.ttft_attainment,     r.itl_attainment, r.ttft_initial.mean,
                           r.ttft_initial.p95,        r.ttft_incremental.mean, r.ttft_incremental.p95, r.itl.mean,
                           r.itl.p95,                 r.e2e_mean,            r.local_fraction};
    out += name + "," + r.trace_name + "," + std::to_string(r.sessions_completed) + "," +
           std::to_string(r.sessions_total);
    for (double v : nums) out += "," + shortest(v);
    out += "\n";
  }
  return out;
}

}  // namespace pdsim
