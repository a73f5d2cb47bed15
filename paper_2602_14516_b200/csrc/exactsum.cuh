// exactsum.cuh — certified comparisons for order-sensitive fp64 folds.
//
// The reference evaluates windowed means (coordinator.cpp:32-47) and queue
// cost estimates (coordinator.cpp:74-100) as left-to-right fp64 folds, then
// only COMPARES the results (slack tests `mean <= alpha*thres`, argmin
// `cost < best`). The engine keeps an exact running sum of every window and
// queue in 128-bit fixed point (LSB 2^-80), updated in O(1) on insert/remove.
// For a fold of n non-negative terms the classic bound
//     |fold - exact| <= gamma_{n-1} * exact,   gamma_k = k*u / (1 - k*u)
// brackets the reference's value; when the bracket decides the comparison the
// answer is exact, otherwise the caller re-runs the sequential fold. Margins
// are 16x the bound to absorb the rounding of the bracket arithmetic itself.
#pragma once

#include "common.cuh"

namespace pdg {

typedef __int128 fx_t;

constexpr int kFxFrac = 80;                 // fixed-point fraction bits
constexpr int64_t kFxMaxTerms = 1ll << 22;  // sums of <= 2^22 terms of < 2^24 fit in 127 bits

// Exact fixed-point image of x >= 0 (round toward zero). Returns false when x
// is not exactly representable (negative, tiny, >= 2^24, or non-finite).
PDG_HD bool to_fx(double x, fx_t* out) {
  if (x == 0.0) {
    *out = 0;
    return true;
  }
  const uint64_t b = dbits(x);
  const int E = static_cast<int>((b >> 52) & 0x7ff);
  if ((b >> 63) || E == 0 || E == 0x7ff || E >= 1023 + 24) {
    *out = 0;
    return false;
  }
  const uint64_t M = (b & ((1ull << 52) - 1)) | (1ull << 52);
  const int sh = E - 1075 + kFxFrac;
  if (sh >= 0) {
    *out = static_cast<fx_t>(M) << sh;
    return true;
  }
  const int r = -sh;
  if (r >= 53) {
    *out = 0;
    return false;
  }
  *out = static_cast<fx_t>(M >> r);
  return (M & ((1ull << r) - 1)) == 0;
}

// Approximate double of a fixed-point value (relative error <= ~2u).
PDG_HD double fx_to_double(fx_t v) {
  const bool neg = v < 0;
  const unsigned __int128 a = neg ? static_cast<unsigned __int128>(-v) : static_cast<unsigned __int128>(v);
  const double hi = static_cast<double>(static_cast<uint64_t>(a >> 64));
  const double lo = static_cast<double>(static_cast<uint64_t>(a));
  const double d = (hi * 18446744073709551616.0 + lo) * 0x1p-80;
  return neg ? -d : d;
}

// Running exact sum of a multiset of non-negative doubles.
struct ExactSum {
  fx_t sum;
  int64_t terms;    // number of scalar terms (runs count with multiplicity)
  int32_t inexact;  // members without an exact fixed-point image
  int32_t reserved;

  PDG_HD void clear() {
    sum = 0;
    terms = 0;
    inexact = 0;
    reserved = 0;
  }
  PDG_HD void add(double x, int64_t count = 1) {
    fx_t f;
    if (!to_fx(x, &f)) ++inexact;
    sum += f * static_cast<fx_t>(count);
    terms += count;
  }
  PDG_HD void remove(double x, int64_t count = 1) {
    fx_t f;
    if (!to_fx(x, &f)) --inexact;
    sum -= f * static_cast<fx_t>(count);
    terms -= count;
  }
  PDG_HD bool exact() const { return inexact == 0 && terms < kFxMaxTerms; }
};

// Relative half-width of the bracket around a fold of n non-negative terms.
PDG_HD double fold_margin(int64_t n) { return (static_cast<double>(n) + 8.0) * 0x1p-49; }

// Decides fl(fold(x_1..x_n) / n) <= thr from the exact sum of the x_i.
// Returns 1 (true), 0 (false) or -1 (undecided: run the sequential fold).
PDG_HD int mean_le_certified(const ExactSum& s, double thr) {
  if (!s.exact() || s.terms <= 0) return -1;
  const double x = fx_to_double(s.sum);
  const double nt = static_cast<double>(s.terms) * thr;
  const double m = fold_margin(s.terms);
  if (x * (1.0 + m) <= nt * (1.0 - m)) return 1;
  if (x * (1.0 - m) >= nt * (1.0 + m)) return 0;
  return -1;
}

// ---- directed rounding (rigorous brackets). Host (test) builds move one
// ulp outward from round-to-nearest, a valid and slightly looser bound.
PDG_HD double add_rd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rd(a, b);
#else
  return __builtin_nextafter(a + b, -__builtin_huge_val());
#endif
}
PDG_HD double add_ru(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_ru(a, b);
#else
  return __builtin_nextafter(a + b, __builtin_huge_val());
#endif
}
PDG_HD double sub_rd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rd(a, b);
#else
  return __builtin_nextafter(a - b, -__builtin_huge_val());
#endif
}
PDG_HD double sub_ru(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_ru(a, b);
#else
  return __builtin_nextafter(a - b, __builtin_huge_val());
#endif
}
PDG_HD double mul_rd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rd(a, b);
#else
  return __builtin_nextafter(a * b, -__builtin_huge_val());
#endif
}
PDG_HD double mul_ru(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_ru(a, b);
#else
  return __builtin_nextafter(a * b, __builtin_huge_val());
#endif
}

// Decides fl(fold(x_1..x_n) / n) <= thr for non-negative terms whose exact
// sum S is known to lie in [lo, hi]: the fold lies in
// [lo (1 - gamma), hi (1 + gamma)]; the margin is 16x gamma_{n-1} plus slack
// for the rounding of these products. 1 true, 0 false, -1 undecided.
PDG_HD int mean_le_bracket(double lo, double hi, int64_t n, double thr) {
  if (n <= 0 || n >= (1ll << 40) || !(hi < 1e300)) return -1;
  const double nt = static_cast<double>(n) * thr;
  const double m = fold_margin(n);
  if (hi * (1.0 + m) <= nt * (1.0 - m)) return 1;
  if (lo * (1.0 - m) >= nt * (1.0 + m)) return 0;
  return -1;
}

// Running prefix of a lazily trimmed window: the window's exact sum is the
// difference of two prefixes. Sums wrap modulo 2^128 (unsigned arithmetic),
// which keeps every in-window difference exact.
typedef unsigned __int128 ufx_t;

struct Pfx {
  ufx_t sum;
  int64_t terms;
  int32_t inexact;
  int32_t reserved;

  PDG_HD void clear() {
    sum = 0;
    terms = 0;
    inexact = 0;
    reserved = 0;
  }
  PDG_HD void add(double x, int64_t count) {
    fx_t f;
    if (!to_fx(x, &f)) ++inexact;
    sum += static_cast<ufx_t>(f) * static_cast<ufx_t>(count);
    terms += count;
  }
};

// Decides fl(fold / n) <= thr for the window [head, tail) given both prefixes.
PDG_HD int window_mean_le(const Pfx& tail, const Pfx& head, double thr) {
  ExactSum s;
  s.sum = static_cast<fx_t>(tail.sum - head.sum);
  s.terms = tail.terms - head.terms;
  s.inexact = tail.inexact - head.inexact;
  s.reserved = 0;
  return mean_le_certified(s, thr);
}

}  // namespace pdg
