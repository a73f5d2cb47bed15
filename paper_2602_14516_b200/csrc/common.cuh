// common.cuh — numerics shared by the device replay engine and the host
// generators: separately-rounded fp64 ops (no FMA contraction, SURVEY §8(a)
// R1), std::mt19937_64, and the piecewise alpha-beta cost curves.
#pragma once

#include <stdint.h>
#include <string.h>

#include "pdsim_gpu.h"

#if defined(__CUDACC__)
#define PDG_HD __host__ __device__ __forceinline__
#define PDG_COLD __host__ __device__ __noinline__  // cold paths: keep the hot loop small
#else
#define PDG_HD inline
#define PDG_COLD inline
#endif

namespace pdg {

// ---- separately rounded fp64 (reference evaluates a*b+c as two roundings;
// perf_model.cpp:51, 172-173). Host code is compiled with -ffp-contract=off.
PDG_HD double dadd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
PDG_HD double dsub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
PDG_HD double dmul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
PDG_HD double ddiv(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
PDG_HD uint64_t dbits(double x) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
#endif
}
PDG_HD double bitsd(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}

// ---- exact integer helpers without the u64 division subroutine ----
// floor(a / d) for a < 2^53, 1 <= d < 2^53 without a division subroutine:
// a hardware reciprocal estimate refined by two Newton steps gives the
// quotient to within one; one exact integer check on each side fixes it.
PDG_HD uint64_t udiv53(uint64_t a, uint64_t d) {
#if defined(__CUDA_ARCH__)
  const double dd = static_cast<double>(d);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(dd));
  r = __fma_rn(__fma_rn(-dd, r, 1.0), r, r);
  r = __fma_rn(__fma_rn(-dd, r, 1.0), r, r);
  uint64_t q = static_cast<uint64_t>(__dmul_rz(static_cast<double>(a), r));
  if (q * d > a) {
    --q;
  } else if ((q + 1) * d <= a) {
    ++q;
  }
  return q;
#else
  return a / d;
#endif
}
// x mod m for 2 <= m < 2^16 (the routing scan's `rng() % (i + 1)`,
// coordinator.cpp:124-130), from three 32-bit remainders.
PDG_HD uint32_t umod64_small(uint64_t x, uint32_t m) {
#if defined(__CUDA_ARCH__)
  const uint32_t hi = static_cast<uint32_t>(x >> 32), lo = static_cast<uint32_t>(x);
  const uint32_t c = (0xffffffffu % m + 1u) % m;  // 2^32 mod m
  return ((hi % m) * c + lo % m) % m;
#else
  return static_cast<uint32_t>(x % m);
#endif
}

// ---- std::mt19937_64 (the reference's engine for routing scan order,
// coordinator.hpp:84, coordinator.cpp:124-130, and for trace/profile
// generation, workload.cpp:32-74, perf_model.cpp:36-39). Parameters are the
// ones fixed by the C++ standard for mt19937_64.
struct Mt64 {
  static constexpr int kN = 312;
  static constexpr int kM = 156;
  static constexpr uint64_t kMatrix = 0xB5026F5AA96619E9ull;
  static constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull;
  static constexpr uint64_t kLower = 0x000000007FFFFFFFull;
};

PDG_HD void mt64_seed(uint64_t* mt, uint32_t* idx, uint64_t seed) {
  mt[0] = seed;
  for (int i = 1; i < Mt64::kN; ++i) {
    mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + static_cast<uint64_t>(i);
  }
  *idx = Mt64::kN;
}

PDG_HD void mt64_twist(uint64_t* mt) {
  for (int i = 0; i < Mt64::kN; ++i) {
    const uint64_t x = (mt[i] & Mt64::kUpper) | (mt[(i + 1) % Mt64::kN] & Mt64::kLower);
    uint64_t xa = x >> 1;
    if (x & 1ull) xa ^= Mt64::kMatrix;
    mt[i] = mt[(i + Mt64::kM) % Mt64::kN] ^ xa;
  }
}

PDG_HD uint64_t mt64_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

PDG_HD uint64_t mt64_next(uint64_t* mt, uint32_t* idx) {
  if (*idx >= static_cast<uint32_t>(Mt64::kN)) {
    mt64_twist(mt);
    *idx = 0;
  }
  return mt64_temper(mt[(*idx)++]);
}

// ---- PiecewiseAlphaBeta::eval (perf_model.cpp:43-52): the segment index is
// the number of breakpoints <= load (right-closed), then alpha + beta*load
// with two roundings.
PDG_HD double curve_eval(const pdsim_curve& c, double load) {
  int i = 0;
  while (i < c.n_breakpoints && !(load < c.breakpoints[i])) ++i;
  return dadd(c.alpha[i], dmul(c.beta[i], load));
}

}  // namespace pdg
