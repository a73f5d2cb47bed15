// planner_host.cpp — host C++ restatement of the reference's exact assignment
// solver and top-k ranking over latency coefficients:
//   solve   (proj/src/planner.cpp:482-578; tables 360-425)
//   top_k   (proj/src/planner.cpp:582-657)
//   plan_ranks_before / compare_counts (planner.cpp:329-356)
// These are tiny integer/table computations over a handful of degrees; the
// costly part of the surrogate planner — the phase simulations behind the
// coefficients — runs on the GPU (planner.cuh).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "pdsim_gpu.h"

namespace pdg {
void set_last_error(const std::string& msg);
}

namespace {

constexpr int64_t kTopKEnumerationCap = 2000000;  // planner.cpp:34

struct Plan {
  std::vector<int> x, y;  // counts per degree (index into the sorted degree list)
  double z = 0.0;
  int gpus = 0;
};

int fail(int code, const std::string& msg) {
  pdg::set_last_error(msg);
  return code;
}

struct Coeffs {
  std::vector<int> deg;  // sorted unique
  std::vector<double> tau_pre, tau_dec;
  std::vector<char> has_pre, has_dec;
};

// sorted_unique + check_coefficients (planner.cpp:437-478).
bool load(const pdsim_coefficients* c, Coeffs* out, std::string* err) {
  if (!c || c->n_degrees < 0 || c->n_degrees > PDSIM_MAX_DEGREES) {
    *err = "planner: bad coefficient table";
    return false;
  }
  std::vector<int> order(static_cast<size_t>(c->n_degrees));
  for (int i = 0; i < c->n_degrees; ++i) order[static_cast<size_t>(i)] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return c->degrees[a] < c->degrees[b]; });
  for (int i : order) {
    if (!out->deg.empty() && out->deg.back() == c->degrees[i]) continue;
    out->deg.push_back(c->degrees[i]);
    out->has_pre.push_back(c->infeasible_pre[i] ? 0 : 1);
    out->has_dec.push_back(c->infeasible_dec[i] ? 0 : 1);
    out->tau_pre.push_back(c->tau_pre[i]);
    out->tau_dec.push_back(c->tau_dec[i]);
  }
  if (out->deg.empty() || out->deg.front() < 1) {
    *err = "planner: degrees must be >= 1";
    return false;
  }
  for (size_t j = 0; j < out->deg.size(); ++j) {
    if (out->has_pre[j] && !(out->tau_pre[j] > 0.0)) {
      *err = "planner: tau_pre must be > 0 for degree " + std::to_string(out->deg[j]);
      return false;
    }
    if (out->has_dec[j] && !(out->tau_dec[j] > 0.0)) {
      *err = "planner: tau_dec must be > 0 for degree " + std::to_string(out->deg[j]);
      return false;
    }
  }
  return true;
}

int replicas(const Plan& p) {
  int r = 0;
  for (int c : p.x) r += c;
  for (int c : p.y) r += c;
  return r;
}

int cmp_counts(const std::vector<int>& a, const std::vector<int>& b) {
  for (size_t j = 0; j < a.size(); ++j)
    if (a[j] != b[j]) return a[j] < b[j] ? -1 : 1;
  return 0;
}

// plan_ranks_before (planner.cpp:346-356).
bool ranks_before(const Plan& a, const Plan& b) {
  if (a.z != b.z) return a.z < b.z;
  const int ra = replicas(a), rb = replicas(b);
  if (ra != rb) return ra > rb;
  if (a.gpus != b.gpus) return a.gpus > b.gpus;
  const int cx = cmp_counts(a.x, b.x);
  if (cx != 0) return cx < 0;
  return cmp_counts(a.y, b.y) < 0;
}

// replica_table (planner.cpp:360-373): most replicas spending exactly b GPUs.
std::vector<int> replica_table(const std::vector<int>& ds, int budget) {
  std::vector<int> best(static_cast<size_t>(budget) + 1, -1);
  best[0] = 0;
  for (int b = 1; b <= budget; ++b)
    for (int n : ds)
      if (n <= b && best[static_cast<size_t>(b - n)] >= 0)
        best[static_cast<size_t>(b)] = std::max(best[static_cast<size_t>(b)], best[static_cast<size_t>(b - n)] + 1);
  return best;
}

// lex_min_counts over exact_table (planner.cpp:377-425): the lexicographically
// smallest count vector over `ds` (ascending) hitting exactly (budget, count).
std::vector<int> lex_min_counts(const std::vector<int>& ds, int budget, int count) {
  const size_t nd = ds.size();
  const size_t B = static_cast<size_t>(budget) + 1, Cn = static_cast<size_t>(count) + 1;
  std::vector<char> ex((nd + 1) * B * Cn, 0);
  auto at = [&](size_t j, int b, int c) -> char& { return ex[(j * B + static_cast<size_t>(b)) * Cn + static_cast<size_t>(c)]; };
  at(nd, 0, 0) = 1;
  for (size_t j = nd; j-- > 0;)
    for (int b = 0; b <= budget; ++b)
      for (int c = 0; c <= count; ++c)
        if (at(j + 1, b, c) || (b >= ds[j] && c >= 1 && at(j, b - ds[j], c - 1))) at(j, b, c) = 1;
  std::vector<int> out(nd, 0);
  size_t j = 0;
  int b = budget, c = count;
  while (j < nd) {
    if (at(j + 1, b, c)) {
      ++j;
      continue;
    }
    ++out[j];
    b -= ds[j];
    c -= 1;
  }
  return out;
}

void to_pod(const Plan& p, const std::vector<int>& deg, pdsim_plan* out) {
  std::memset(out, 0, sizeof(*out));
  for (size_t j = 0; j < deg.size(); ++j) {
    if (p.x[j]) {
      out->prefill_degree[out->n_prefill_groups] = deg[j];
      out->prefill_count[out->n_prefill_groups++] = p.x[j];
    }
    if (p.y[j]) {
      out->decode_degree[out->n_decode_groups] = deg[j];
      out->decode_count[out->n_decode_groups++] = p.y[j];
    }
  }
}

// Expands counts over an admissible subset back onto the full degree list.
std::vector<int> spread(const std::vector<int>& sub_counts, const std::vector<int>& sub, const std::vector<int>& deg) {
  std::vector<int> out(deg.size(), 0);
  for (size_t k = 0; k < sub.size(); ++k) {
    const size_t j = static_cast<size_t>(std::find(deg.begin(), deg.end(), sub[k]) - deg.begin());
    out[j] = sub_counts[k];
  }
  return out;
}

}  // namespace

extern "C" {

int pdsim_solve(const pdsim_coefficients* coeffs, int32_t total_gpus, pdsim_plan* plan, double* objective_z,
                int32_t* gpus_used, int32_t* feasible) {
  Coeffs c;
  std::string err;
  if (!load(coeffs, &c, &err)) return fail(PDSIM_ERR_CONFIG, err);
  if (total_gpus < 1) return fail(PDSIM_ERR_CONFIG, "planner: total_gpus must be >= 1");
  if (feasible) *feasible = 0;
  std::vector<int> pre_all, dec_all;
  for (size_t j = 0; j < c.deg.size(); ++j) {
    if (c.has_pre[j]) pre_all.push_back(static_cast<int>(j));
    if (c.has_dec[j]) dec_all.push_back(static_cast<int>(j));
  }
  if (pre_all.empty() || dec_all.empty()) return PDSIM_OK;
  // Candidate objectives: the coefficient values (planner.cpp:500-528).
  std::vector<double> cand;
  for (int j : pre_all) cand.push_back(c.tau_pre[static_cast<size_t>(j)]);
  for (int j : dec_all) cand.push_back(c.tau_dec[static_cast<size_t>(j)]);
  std::sort(cand.begin(), cand.end());
  cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
  std::vector<int> pre_adm, dec_adm;
  double z_star = 0.0;
  bool found = false;
  for (double z : cand) {
    pre_adm.clear();
    dec_adm.clear();
    for (int j : pre_all)
      if (c.tau_pre[static_cast<size_t>(j)] <= z) pre_adm.push_back(c.deg[static_cast<size_t>(j)]);
    for (int j : dec_all)
      if (c.tau_dec[static_cast<size_t>(j)] <= z) dec_adm.push_back(c.deg[static_cast<size_t>(j)]);
    if (!pre_adm.empty() && !dec_adm.empty() && pre_adm.front() + dec_adm.front() <= total_gpus) {
      z_star = z;
      found = true;
      break;
    }
  }
  if (!found) return PDSIM_OK;
  const std::vector<int> fp = replica_table(pre_adm, total_gpus), fd = replica_table(dec_adm, total_gpus);
  int best_count = -1, best_gpus = -1;
  for (int bp = 0; bp <= total_gpus; ++bp) {
    if (fp[static_cast<size_t>(bp)] < 1) continue;
    for (int bd = 0; bd + bp <= total_gpus; ++bd) {
      if (fd[static_cast<size_t>(bd)] < 1) continue;
      const int count = fp[static_cast<size_t>(bp)] + fd[static_cast<size_t>(bd)], used = bp + bd;
      if (count > best_count || (count == best_count && used > best_gpus)) {
        best_count = count;
        best_gpus = used;
      }
    }
  }
  Plan best;
  bool have = false;
  for (int bp = 0; bp <= total_gpus; ++bp) {
    if (fp[static_cast<size_t>(bp)] < 1) continue;
    const int bd = best_gpus - bp;
    if (bd < 0 || bd > total_gpus || fd[static_cast<size_t>(bd)] < 1) continue;
    if (fp[static_cast<size_t>(bp)] + fd[static_cast<size_t>(bd)] != best_count) continue;
    Plan p;
    p.x = spread(lex_min_counts(pre_adm, bp, fp[static_cast<size_t>(bp)]), pre_adm, c.deg);
    p.y = spread(lex_min_counts(dec_adm, bd, fd[static_cast<size_t>(bd)]), dec_adm, c.deg);
    p.z = z_star;
    p.gpus = best_gpus;
    if (!have || ranks_before(p, best)) {
      best = p;
      have = true;
    }
  }
  if (!have) return PDSIM_OK;
  if (plan) to_pod(best, c.deg, plan);
  if (objective_z) *objective_z = best.z;
  if (gpus_used) *gpus_used = best.gpus;
  if (feasible) *feasible = 1;
  return PDSIM_OK;
}

int64_t pdsim_top_k(const pdsim_coefficients* coeffs, int32_t total_gpus, int32_t k, pdsim_plan* plans,
                    double* objective_z, int32_t* gpus_used) {
  if (k < 1) return fail(PDSIM_ERR_CONFIG, "top_k: k must be >= 1"), -1;
  Coeffs c;
  std::string err;
  if (!load(coeffs, &c, &err)) return fail(PDSIM_ERR_CONFIG, err), -1;
  if (total_gpus < 1) return fail(PDSIM_ERR_CONFIG, "planner: total_gpus must be >= 1"), -1;
  std::vector<size_t> pre, dec;
  for (size_t j = 0; j < c.deg.size(); ++j) {
    if (c.has_pre[j]) pre.push_back(j);
    if (c.has_dec[j]) dec.push_back(j);
  }
  if (pre.empty() || dec.empty()) return 0;
  std::vector<Plan> best;
  int64_t visited = 0;
  bool capped = false;
  const size_t nd = c.deg.size();
  std::vector<int> xs(nd, 0), ys(nd, 0);
  // enumerate_counts (planner.cpp:582-601) over the usable degrees.
  std::function<void(const std::vector<size_t>&, size_t, int, std::vector<int>&, const std::function<void()>&)> rec =
      [&](const std::vector<size_t>& use, size_t j, int budget, std::vector<int>& cur, const std::function<void()>& emit) {
        if (capped) return;
        if (j == use.size()) {
          if (++visited > kTopKEnumerationCap) {
            capped = true;
            return;
          }
          emit();
          return;
        }
        const int n = c.deg[use[j]];
        for (int cnt = 0; cnt * n <= budget && !capped; ++cnt) {
          cur[use[j]] = cnt;
          rec(use, j + 1, budget - cnt * n, cur, emit);
        }
        cur[use[j]] = 0;
      };
  rec(pre, 0, total_gpus, xs, [&] {
    int xg = 0, xn = 0;
    for (size_t j = 0; j < nd; ++j) {
      xg += c.deg[j] * xs[j];
      xn += xs[j];
    }
    if (xn == 0) return;
    rec(dec, 0, total_gpus - xg, ys, [&] {
      int yn = 0, yg = 0;
      for (size_t j = 0; j < nd; ++j) {
        yn += ys[j];
        yg += c.deg[j] * ys[j];
      }
      if (yn == 0) return;
      Plan p;
      p.x = xs;
      p.y = ys;
      double z = 0.0;  // plan_objective (planner.cpp:427-436)
      for (size_t j = 0; j < nd; ++j) {
        if (xs[j]) z = std::max(z, c.tau_pre[j]);
        if (ys[j]) z = std::max(z, c.tau_dec[j]);
      }
      p.z = z;
      p.gpus = xg + yg;
      auto pos = std::lower_bound(best.begin(), best.end(), p, [](const Plan& a, const Plan& b) { return ranks_before(a, b); });
      if (pos - best.begin() < static_cast<std::ptrdiff_t>(k)) {
        best.insert(pos, p);
        if (best.size() > static_cast<size_t>(k)) best.pop_back();
      }
    });
  });
  if (capped) return fail(PDSIM_ERR_CONFIG, "top_k: instance too large for exhaustive ranking"), -1;
  for (size_t i = 0; i < best.size(); ++i) {
    if (plans) to_pod(best[i], c.deg, &plans[i]);
    if (objective_z) objective_z[i] = best[i].z;
    if (gpus_used) gpus_used[i] = best[i].gpus;
  }
  return static_cast<int64_t>(best.size());
}

}  // extern "C"
