// planner.cuh — the reference's surrogate planner phase simulations on the GPU
// (SURVEY.md §8(f)1).
//
// Behavioural restatement, for B200, of
//   simulate_prefill_replica (proj/src/planner.cpp:75-104, flattening 55-72)
//   simulate_decode_replica  (proj/src/planner.cpp:106-226)
//   nearest_rank_p95         (proj/src/planner.cpp:36-42)
// used by estimate_coefficients (planner.cpp:228-283). One CTA (256 threads)
// replays one (trace, degree) job; jobs are pulled from an atomic queue, so a
// rates x seeds x degrees coefficient sweep is one launch.
//
// Layout choices (not a translation of the reference loops):
//  * prefill: the flattened tasks are sorted by (arrival, flattened index) —
//    the reference's stable_sort — with a CTA bitonic sort; the FIFO recurrence
//    start = max(arrival, free_at), free_at = start + service is inherently
//    sequential and runs on one thread over precomputed service times.
//  * decode: one thread per session; batch size and ITL sample counts are
//    CTA reductions. All ITL samples of one step are now - (previous step
//    end) (a member decodes in consecutive steps within a round), so the
//    sample multiset is stored as (value, count) runs instead of one entry
//    per token, and a quiet stretch of steps (no finish, no admission, end
//    times in one binade) is advanced in one go as a single run.
//  * P95: nearest rank (ceil(0.95 n)) by an exact 8-pass radix select over
//    the fp64 bit patterns (non-negative values order like their bits),
//    weighted by run counts — no sort of the samples.
// Every fp64 operation is the reference's, separately rounded (common.cuh).
#pragma once

#include "common.cuh"
#include "fold.cuh"

namespace pdg {

struct PhaseJob {
  int32_t trace;   // index into the packed trace table
  int32_t deg;     // profile degree index
};

struct PhaseOut {
  double pre_p95;
  double dec_p95;
  int64_t pre_samples;
  int64_t dec_samples;
  int32_t pre_infeasible;
  int32_t dec_infeasible;
  int32_t pre_status;  // PDSIM_OK or PDSIM_ERR_CONFIG (the reference throws)
  int32_t dec_status;
};

struct PhaseTrace {
  int32_t S, R;
  int64_t total_decode;
  const double* arrival;     // [S]
  const int32_t* round_off;  // [S+1]
  const int32_t* incr;       // [R]
  const int32_t* dec;        // [R]
  const double* delay;       // [R]
};

struct PhaseArgs {
  const PhaseTrace* traces;
  const PhaseJob* jobs;
  int32_t n_jobs;
  int32_t sort_cap;      // power of two >= max R (prefill sort scratch)
  int32_t max_s;         // >= max sessions (decode sim state)
  int64_t run_cap;       // >= max steps of any decode sim (<= max total decode)
  char* scratch;         // per-CTA scratch
  size_t scratch_bytes;  // per CTA
  unsigned long long* next_job;
  PhaseOut* out;
  const pdsim_profile* profile;  // device copy
};

constexpr int kPhaseThreads = 256;

#if defined(__CUDACC__)

// Per-CTA scratch layout.
struct PhaseScratch {
  uint64_t* key;     // [sort_cap] arrival bits (then latency bits)
  uint32_t* idx;     // [sort_cap] flattened task index
  double* service;   // [sort_cap] by flattened index
  int64_t* hist;     // [sort_cap] by flattened index (l_hist)
  uint64_t* run_v;   // [run_cap] ITL run value bits
  int64_t* run_n;    // [run_cap] ITL run sample counts
  int32_t* remaining;  // [S] decode sim session state
  int32_t* emitted;
  int32_t* round;
  int32_t* state;      // 0 not arrived, 1 active, 2 blocked, 3 done
  double* unblock;
};

__host__ __device__ inline size_t phase_scratch_bytes(int32_t sort_cap, int64_t run_cap, int32_t max_s) {
  const size_t n = static_cast<size_t>(sort_cap), r = static_cast<size_t>(run_cap), s = static_cast<size_t>(max_s);
  auto a = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
  return a(8 * n) + a(4 * n) + a(8 * n) + a(8 * n) + a(8 * r) + a(8 * r) + 4 * a(4 * s) + a(8 * s) + 256;
}

__device__ inline PhaseScratch phase_scratch(char* base, int32_t sort_cap, int64_t run_cap, int32_t max_s) {
  const size_t n = static_cast<size_t>(sort_cap), r = static_cast<size_t>(run_cap), s = static_cast<size_t>(max_s);
  auto a = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
  PhaseScratch p;
  size_t off = 0;
  p.key = reinterpret_cast<uint64_t*>(base + off);
  off += a(8 * n);
  p.idx = reinterpret_cast<uint32_t*>(base + off);
  off += a(4 * n);
  p.service = reinterpret_cast<double*>(base + off);
  off += a(8 * n);
  p.hist = reinterpret_cast<int64_t*>(base + off);
  off += a(8 * n);
  p.run_v = reinterpret_cast<uint64_t*>(base + off);
  off += a(8 * r);
  p.run_n = reinterpret_cast<int64_t*>(base + off);
  off += a(8 * r);
  p.remaining = reinterpret_cast<int32_t*>(base + off);
  off += a(4 * s);
  p.emitted = reinterpret_cast<int32_t*>(base + off);
  off += a(4 * s);
  p.round = reinterpret_cast<int32_t*>(base + off);
  off += a(4 * s);
  p.state = reinterpret_cast<int32_t*>(base + off);
  off += a(4 * s);
  p.unblock = reinterpret_cast<double*>(base + off);
  return p;
}

// CTA bitonic sort of (key, idx) pairs ascending, n a power of two.
__device__ inline void cta_bitonic_sort(uint64_t* key, uint32_t* idx, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const uint64_t ki = key[i], kl = key[l];
          const uint32_t ii = idx[i], il = idx[l];
          const bool up = (i & k) == 0;
          const bool gt = ki > kl || (ki == kl && ii > il);
          if (gt == up) {
            key[i] = kl;
            key[l] = ki;
            idx[i] = il;
            idx[l] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
}

// k-th smallest (1-based rank) of n keys with optional weights: 8 passes over
// 8-bit digits from the top. Exact for any multiset of u64 keys.
__device__ inline uint64_t cta_radix_select(const uint64_t* keys, const int64_t* weights, int64_t n, int64_t rank) {
  __shared__ unsigned long long hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int64_t s_rank;
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_rank = rank;
  }
  __syncthreads();
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    const uint64_t mask_hi = shift == 56 ? 0ull : (~0ull << (shift + 8));
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t k = keys[i];
      if ((k & mask_hi) == prefix) {
        atomicAdd(&hist[(k >> shift) & 255u], static_cast<unsigned long long>(weights ? weights[i] : 1));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t r = s_rank;
      int b = 0;
      for (; b < 255; ++b) {
        const int64_t c = static_cast<int64_t>(hist[b]);
        if (r <= c) break;
        r -= c;
      }
      s_rank = r;
      s_prefix = prefix | (static_cast<uint64_t>(b) << shift);
    }
    __syncthreads();
  }
  return s_prefix;
}

__device__ inline double cta_min(double v) {
  __shared__ double red[32];
  for (int m = 16; m > 0; m >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, v, m);
    v = o < v ? o : v;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) r = red[w] < r ? red[w] : r;
  __syncthreads();
  return r;
}

__device__ inline double cta_max(double v) { return -cta_min(-v); }

// Sum of per-thread counts; one barrier when every thread holds 0 or 1.
__device__ inline long long cta_count(int v, bool unit) {
  if (unit) return __syncthreads_count(v != 0);
  return 0;
}

__device__ inline long long cta_sum(long long v) {
  __shared__ long long red[32];
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  long long r = 0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) r += red[w];
  __syncthreads();
  return r;
}

// nearest_rank_p95 (planner.cpp:36-42): rank = ceil(0.95 * n).
__device__ inline int64_t p95_rank(int64_t n) {
  return static_cast<int64_t>(ceil(__dmul_rn(0.95, static_cast<double>(n))));
}

// simulate_prefill_replica (planner.cpp:75-104).
__device__ inline void prefill_sim(const PhaseTrace& T, int deg, const pdsim_profile& prof, const PhaseScratch& w,
                                   int32_t sort_cap, PhaseOut* o) {
  const int R = T.R;
  if (R == 0) {  // "planner: reference trace has no prefill tasks"
    if (threadIdx.x == 0) o->pre_status = PDSIM_ERR_CONFIG;
    return;
  }
  // Flattening (planner.cpp:55-72): task index = round_offset[i] + r.
  for (int i = threadIdx.x; i < T.S; i += blockDim.x) {
    double off = T.arrival[i];
    int64_t hist = 0;
    for (int k = T.round_off[i]; k < T.round_off[i + 1]; ++k) {
      w.key[k] = dbits(off);  // arrival >= 0: bits order like values
      w.idx[k] = static_cast<uint32_t>(k);
      w.hist[k] = hist;
      hist += static_cast<int64_t>(T.incr[k]) + T.dec[k];
      off = dadd(off, T.delay[k]);
    }
  }
  for (int k = R + threadIdx.x; k < sort_cap; k += blockDim.x) {
    w.key[k] = ~0ull;
    w.idx[k] = 0xffffffffu;
  }
  __syncthreads();
  // t_prefill (perf_model.cpp:158-175) per task, by flattened index.
  for (int k = threadIdx.x; k < R; k += blockDim.x) {
    const double load = dadd(static_cast<double>(T.incr[k]), dmul(prof.history_weight, static_cast<double>(w.hist[k])));
    w.service[k] = curve_eval(prof.prefill[deg], load);
  }
  int n = 1;
  while (n < R) n <<= 1;
  cta_bitonic_sort(w.key, w.idx, n);  // stable_sort by arrival (ties: flattened order)
  // FIFO single server, in sorted order (sequential recurrence).
  if (threadIdx.x == 0) {
    double total_service = 0.0, free_at = 0.0;
    for (int j = 0; j < R; ++j) {
      const double arrival = bitsd(w.key[j]);
      const double service = w.service[w.idx[j]];
      total_service = dadd(total_service, service);
      const double start = arrival < free_at ? free_at : arrival;  // std::max(arrival, free_at)
      free_at = dadd(start, service);
      w.hist[j] = static_cast<int64_t>(dbits(dsub(free_at, arrival)));  // latency bits, reuse
    }
    const double span = dsub(bitsd(w.key[R - 1]), bitsd(w.key[0]));
    o->pre_infeasible = (R >= 2 && (span <= 0.0 || ddiv(total_service, span) >= 1.0)) ? 1 : 0;
    o->pre_samples = R;
  }
  __syncthreads();
  const uint64_t v = cta_radix_select(reinterpret_cast<const uint64_t*>(w.hist), nullptr, R, p95_rank(R));
  if (threadIdx.x == 0) {
    o->pre_p95 = bitsd(v);
    o->pre_status = PDSIM_OK;
  }
  __syncthreads();
}

// simulate_decode_replica (planner.cpp:106-226).
__device__ inline void decode_sim(const PhaseTrace& T, int deg, const pdsim_profile& prof, const PhaseScratch& w,
                                  int64_t run_cap, PhaseOut* o) {
  const int S = T.S;
  if (S == 0) {  // "planner: reference trace has no sessions"
    if (threadIdx.x == 0) o->dec_status = PDSIM_ERR_CONFIG;
    return;
  }
  double amin = __builtin_huge_val(), amax = -__builtin_huge_val();
  for (int i = threadIdx.x; i < S; i += blockDim.x) {
    amin = T.arrival[i] < amin ? T.arrival[i] : amin;
    amax = T.arrival[i] > amax ? T.arrival[i] : amax;
    w.remaining[i] = T.dec[T.round_off[i]];
    w.emitted[i] = 0;
    w.round[i] = 0;
    w.state[i] = 0;
    w.unblock[i] = 0.0;
  }
  amin = cta_min(amin);
  amax = cta_max(amax);
  const pdsim_curve& dc = prof.decode[deg];
  const double beta_last = dc.beta[dc.n_breakpoints];
  if (threadIdx.x == 0) {
    int infeasible = 0;
    if (S >= 2) {
      const double span = dsub(amax, amin);  // sorted back - front
      if (span <= 0.0) {
        infeasible = 1;
      } else if (beta_last > 0.0 && ddiv(static_cast<double>(T.total_decode), span) >= ddiv(0.98, beta_last)) {
        infeasible = 1;  // demand at or past the asymptotic token throughput
      }
    }
    o->dec_infeasible = infeasible;
  }
  __shared__ double s_now;
  __shared__ int64_t s_runs, s_samples;
  __shared__ int s_overflow;
  if (threadIdx.x == 0) {
    s_now = 0.0;
    s_runs = 0;
    s_samples = 0;
    s_overflow = 0;
  }
  __syncthreads();
  int active = 0;
  const bool unit = S <= static_cast<int>(blockDim.x);  // one session per thread
  for (;;) {
    double now = s_now;
    if (active == 0) {
      // Idle: jump to the next arrival or unblock (planner.cpp:181-190).
      double wake = __builtin_huge_val();
      for (int i = threadIdx.x; i < S; i += blockDim.x) {
        const int st = w.state[i];
        const double t = st == 0 ? T.arrival[i] : st == 2 ? w.unblock[i] : __builtin_huge_val();
        wake = t < wake ? t : wake;
      }
      wake = cta_min(wake);
      if (wake == __builtin_huge_val()) break;  // no arrival, nothing blocked, nothing active
      now = now < wake ? wake : now;            // std::max(now, wake)
    }
    // admit_ready(now) (planner.cpp:164-174): the admitted SET is what matters.
    int mine = 0;
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
      int st = w.state[i];
      if ((st == 0 && T.arrival[i] <= now) || (st == 2 && w.unblock[i] <= now)) {
        st = 1;
        w.state[i] = 1;
      }
      mine += st == 1;
    }
    active = static_cast<int>(unit ? cta_count(mine, true) : cta_sum(mine));
    if (active == 0) {
      if (threadIdx.x == 0) s_now = now;
      __syncthreads();
      continue;
    }
    const double step = curve_eval(dc, static_cast<double>(active));  // t_decode (perf_model.cpp:177-188)
    const double prev = now;
    now = dadd(now, step);
    int samples = 0, still = 0;
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
      if (w.state[i] != 1) continue;
      const int rem = w.remaining[i] - 1;
      const int em = w.emitted[i] + 1;
      if (em >= 2) ++samples;  // itl sample now - last_token (= prev)
      if (rem > 0) {
        w.remaining[i] = rem;
        w.emitted[i] = em;
        ++still;
        continue;
      }
      const int r = w.round[i];
      const int k = T.round_off[i] + r;
      if (T.round_off[i] + r + 1 < T.round_off[i + 1]) {
        w.round[i] = r + 1;
        w.remaining[i] = T.dec[k + 1];
        w.emitted[i] = 0;
        w.state[i] = 2;
        w.unblock[i] = dadd(now, T.delay[k]);
      } else {
        w.state[i] = 3;
      }
    }
    const long long ns = unit ? cta_count(samples, true) : cta_sum(samples);
    const int before = active;
    active = static_cast<int>(unit ? cta_count(still, true) : cta_sum(still));
    if (threadIdx.x == 0) {
      s_now = now;
      if (ns > 0) {
        if (s_runs < run_cap) {
          w.run_v[s_runs] = dbits(dsub(now, prev));
          w.run_n[s_runs] = ns;
          ++s_runs;
        } else {
          s_overflow = 1;
        }
        s_samples += ns;
      }
    }
    __syncthreads();
    if (s_overflow) break;
    // Quiet stretch: nobody finished and nobody is admitted until time T, so
    // the next steps keep this batch, each yields `active` samples (every
    // member is past its first token) of the same gap while the end times
    // stay in one binade (stable_run, fold.cuh). They are advanced together
    // — the reference loop would take them one by one with identical results.
    if (active == before && active > 0) {
      double tn = __builtin_huge_val(), mfin = __builtin_huge_val();
      for (int i = threadIdx.x; i < S; i += blockDim.x) {
        const int st = w.state[i];
        const double t = st == 0 ? T.arrival[i] : st == 2 ? w.unblock[i] : __builtin_huge_val();
        tn = t < tn ? t : tn;
        if (st == 1) mfin = static_cast<double>(w.remaining[i]) < mfin ? static_cast<double>(w.remaining[i]) : mfin;
      }
      tn = cta_min(tn);
      mfin = cta_min(mfin);
      int64_t m2 = 0;
      double g = 0.0, end = now;
      if (now < tn && mfin > 1.0) {
        const double e2 = dadd(now, step);
        g = dsub(e2, now);
        m2 = stable_run(now, step, g, tn, static_cast<int64_t>(mfin) - 1);
        if (m2 > 0) end = dadd(e2, dmul(static_cast<double>(m2 - 1), g));
      }
      if (m2 > 0) {
        for (int i = threadIdx.x; i < S; i += blockDim.x) {
          if (w.state[i] != 1) continue;
          w.remaining[i] -= static_cast<int32_t>(m2);
          w.emitted[i] += static_cast<int32_t>(m2);
        }
        if (threadIdx.x == 0) {
          s_now = end;
          if (s_runs < run_cap) {
            w.run_v[s_runs] = dbits(g);
            w.run_n[s_runs] = static_cast<int64_t>(active) * m2;
            ++s_runs;
          } else {
            s_overflow = 1;
          }
          s_samples += static_cast<int64_t>(active) * m2;
        }
        __syncthreads();
        if (s_overflow) break;
      }
    }
  }
  __syncthreads();
  const int64_t runs = s_runs, total = s_samples;
  if (s_overflow) {
    if (threadIdx.x == 0) o->dec_status = PDSIM_ERR_INTERNAL;
    return;
  }
  if (total == 0) {  // "planner: reference trace produced no inter-token samples"
    if (threadIdx.x == 0) o->dec_status = PDSIM_ERR_CONFIG;
    return;
  }
  const uint64_t v = cta_radix_select(w.run_v, w.run_n, runs, p95_rank(total));
  if (threadIdx.x == 0) {
    o->dec_p95 = bitsd(v);
    o->dec_samples = total;
    o->dec_status = PDSIM_OK;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kPhaseThreads) phase_sim_kernel(PhaseArgs a) {
  __shared__ unsigned long long s_job;
  const PhaseScratch w = phase_scratch(a.scratch + static_cast<size_t>(blockIdx.x) * a.scratch_bytes, a.sort_cap,
                                       a.run_cap, a.max_s);
  for (;;) {
    if (threadIdx.x == 0) s_job = atomicAdd(a.next_job, 1ull);
    __syncthreads();
    const unsigned long long j = s_job;
    __syncthreads();
    if (j >= static_cast<unsigned long long>(a.n_jobs)) break;
    const PhaseJob job = a.jobs[j];
    const PhaseTrace T = a.traces[job.trace];
    PhaseOut* o = &a.out[j];
    prefill_sim(T, job.deg, *a.profile, w, a.sort_cap, o);
    __syncthreads();
    decode_sim(T, job.deg, *a.profile, w, a.run_cap, o);
    __syncthreads();
  }
}

#endif  // __CUDACC__

}  // namespace pdg
