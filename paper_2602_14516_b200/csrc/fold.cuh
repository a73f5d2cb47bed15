// fold.cuh — exact emulation of a left-to-right fp64 fold over a run of
// identical addends, in O(binades) instead of O(count).
//
// The reference's WindowedStat::query (coordinator.cpp:32-47) sums every ITL
// sample of the window one by one. All ITL samples produced by one decode step
// carry the same value (SURVEY.md §8(a) note A), so the device stores the ITL
// window as runs (time, gap, count) and reproduces the reference's sequential
// sum bit-for-bit with fold_repeat().
//
// Why it is exact: while the running sum s stays inside one binade
// [2^e, 2^(e+1)) with ulp u, fl(s + g) = s + d*u where d = round-half-even of
// g/u, evaluated against the parity of s/u. For a non-tie g/u the increment d
// is the same at every step; for an exact tie the first step makes s/u even,
// after which d = k + (k & 1) is constant. So a whole stretch of steps inside
// the binade is one integer multiply-add on the significand. Steps that may
// leave the binade, and any s < g step, are done with one real fp64 add.
#pragma once

#include "common.cuh"

namespace pdg {

// Returns fl(...fl(fl(s + g) + g)... + g) with `count` additions of g, exactly
// as a sequential loop (round-to-nearest-even, no FMA). Requires s >= 0,
// g >= 0 (the engine only folds non-negative latencies).
PDG_HD double fold_repeat(double s, double g, uint64_t count) {
  if (count <= 16) {  // short folds: plain adds beat the binade arithmetic
    for (uint64_t k = 0; k < count; ++k) s = dadd(s, g);
    return s;
  }
  const uint64_t kMant = (1ull << 52) - 1;
  const uint64_t kTop = (1ull << 53) - 2;  // stay strictly inside the binade
  while (count > 0) {
    if (!(g > 0.0) || !(s >= g) || !(s < 1.0e300)) {
      // g == 0 leaves s unchanged except for signed-zero details: take one
      // real add. s < g: one real add always ends with s >= g.
      s = dadd(s, g);
      --count;
      if (g == 0.0) return s;  // further adds of +0 are identities
      continue;
    }
    const uint64_t sb = dbits(s);
    const uint64_t gb = dbits(g);
    const int es = static_cast<int>((sb >> 52) & 0x7ff);
    const int eg = static_cast<int>((gb >> 52) & 0x7ff);
    if (es == 0 || eg == 0) {  // subnormal operands: take the slow path
      s = dadd(s, g);
      --count;
      continue;
    }
    uint64_t S = (sb & kMant) | (1ull << 52);
    const uint64_t G = (gb & kMant) | (1ull << 52);
    const int sh = es - eg;  // >= 0 because g <= s
    uint64_t k, rem, half;
    if (sh == 0) {
      k = G;
      rem = 0;
      half = 1;
    } else if (sh < 64) {
      k = G >> sh;
      rem = G & ((1ull << sh) - 1);
      half = 1ull << (sh - 1);
    } else {
      k = 0;
      rem = 1;  // nonzero, far below half
      half = 2;
    }
    uint64_t d;
    if (rem == 0 || rem < half) {
      d = k;
    } else if (rem > half) {
      d = k + 1;
    } else {  // exact tie: parity of the result decides
      if (S & 1ull) {
        s = dadd(s, g);
        --count;
        continue;
      }
      d = k + (k & 1ull);
    }
    if (d == 0) return s;  // g is absorbed by s at every remaining step
    if (S + d > kTop) {    // the next step may cross into the next binade
      s = dadd(s, g);
      --count;
      continue;
    }
    uint64_t n = udiv53(kTop - S, d);
    if (n > count) n = count;
    S += n * d;
    count -= n;
    s = bitsd((static_cast<uint64_t>(es) << 52) | (S & kMant));
  }
  return s;
}

// Number m >= 0 of consecutive steps after a step ending at e0 whose ends
// E_1 = e0 + g (given, = fl(e0 + dur)), E_2 = fl(E_1 + dur), ... all add
// exactly g, stay below t, and number at most max_m. Within one binade of
// the end time the rounded increment of fl(E + dur) is the same integer
// number of ulps unless dur/ulp is an exact half (then it is constant once
// the significand is even) — the same argument as fold_repeat (fold.cuh).
PDG_HD int64_t stable_run(double e0, double dur, double g, double t, int64_t max_m) {
  const double e1 = dadd(e0, g);
  if (!(e1 < t) || max_m <= 0) return 0;
  const uint64_t eb = dbits(e1), db = dbits(dur);
  const int es = static_cast<int>((eb >> 52) & 0x7ff);
  const int ed = static_cast<int>((db >> 52) & 0x7ff);
  if (es == 0 || ed == 0 || es >= 0x7fe || ed > es || es < 53 + 1) return 1;
  const uint64_t kMant = (1ull << 52) - 1;
  const uint64_t kTop = (1ull << 53) - 2;
  const uint64_t S1 = (eb & kMant) | (1ull << 52);
  const uint64_t G = (db & kMant) | (1ull << 52);
  const int sh = es - ed;
  uint64_t k, rem, half;
  if (sh == 0) {
    k = G;
    rem = 0;
    half = 1;
  } else if (sh < 64) {
    k = G >> sh;
    rem = G & ((1ull << sh) - 1);
    half = 1ull << (sh - 1);
  } else {
    k = 0;
    rem = 1;
    half = 2;
  }
  uint64_t dstep;
  if (rem == 0 || rem < half) {
    dstep = k;
  } else if (rem > half) {
    dstep = k + 1;
  } else {
    if (S1 & 1ull) return 1;  // tie with an odd significand: one step at a time
    dstep = k + (k & 1ull);
  }
  if (dstep == 0) return 1;
  // the stable increment must be the gap we were given
  const double ulp = bitsd(static_cast<uint64_t>(es - 52) << 52);
  if (dmul(static_cast<double>(dstep), ulp) != g) return 1;
  if (S1 > kTop) return 1;
  int64_t m = 1 + static_cast<int64_t>(udiv53(kTop - S1, dstep));
  const uint64_t tb = dbits(t);
  const int et = static_cast<int>((tb >> 52) & 0x7ff);
  if (et == es) {  // t in the same binade: S1 + (j-1) d < T
    const uint64_t T = (tb & kMant) | (1ull << 52);
    const int64_t mt = 1 + static_cast<int64_t>(udiv53(T - S1 - 1, dstep));
    if (mt < m) m = mt;
  }
  if (max_m < m) m = max_m;
  return m;
}

}  // namespace pdg
