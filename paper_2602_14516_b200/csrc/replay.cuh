// replay.cuh — the persistent replay kernel (one warp per workspace slot
// pulling (candidate, replica) pairs from an atomic queue; engine.cuh replays
// each pair; SLO counts folded into per-candidate integer sums) and its
// launch table. The kernels of each shared-memory layout are compiled in
// their own translation unit (replay_l0/l1/l2.cu) so they build in parallel;
// each unit owns its copy of the __constant__ cost model.
#pragma once

#include <cuda_runtime.h>

#include "engine.cuh"

namespace pdg {

struct KernelArgs {
  const DevTrace* traces;
  const DevPlan* plans;
  const int8_t* pair_invalid;  // [n_candidates * n_traces]
  int32_t n_traces;
  int32_t reserved;
  int64_t pair_begin;
  int64_t pair_end;
  DevParams params;
  const DevParams* cand_params;  // optional per-candidate settings (sweep); null: `params` for all
  Caps caps;
  char* ws;
  size_t slot_bytes;
  size_t smem_bytes;
  unsigned long long* next_pair;
  PairResult* results;            // [pair_end - pair_begin], by launch item
  unsigned long long* cand_sum;        // [n_candidates]
  int* cand_bad;                       // [n_candidates]
  Records rec;                    // single-run records (one pair only)
  pdsim_report* reports;               // optional per-pair reports [pair_end - pair_begin]
  uint64_t seed;
  int32_t profile;                     // per-phase clock64 instrumentation
  int32_t reserved3;
  unsigned long long* best_key;        // prune: incumbent key
  int32_t* pair_fail;                  // prune: [n_candidates * n_traces], by global pair
  int32_t* pair_ok;                    // prune: [n_candidates * n_traces], by global pair
  const int8_t* cand_invalid;          // prune: [n_candidates] any pair of c invalid (whole search)
  int64_t total_sessions;              // prune: sum of S over ALL replicas of the search (every shard)
  const int64_t* pair_list;            // optional: the launch replays pair_list[0 .. pair_end - pair_begin)
  // optional SM-affine queues: list s = sm_items[sm_off[s] .. sm_off[s+1]) of
  // launch items, taken first by warps on SM (smid % n_lists), then stolen
  const int64_t* sm_items;
  const int32_t* sm_off;               // [n_lists + 1]
  unsigned int* sm_next;               // [n_lists], zeroed per launch
  int32_t n_lists;
  int32_t reserved4;
};

// Next launch item of a warp on an SM-affine queue set: its home list first,
// then the other lists in ring order; -1 when every list is exhausted. The
// warp stays converged (lane 0 takes the tickets, broadcast by shuffle).
__device__ __forceinline__ int64_t take_sm_affine(const int64_t* items, const int32_t* off, unsigned* next, int L,
                                                  unsigned smid) {
  int s = static_cast<int>(smid % static_cast<unsigned>(L));
  for (int k = 0; k < L; ++k) {
    const int32_t lo = off[s];
    const unsigned cnt = static_cast<unsigned>(off[s + 1] - lo);
    unsigned t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(&next[s], 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t < cnt) return items[lo + t];
    s = s + 1 == L ? 0 : s + 1;
  }
  return -1;
}

// Result of a pair that is not replayed (pruned / invalid), field by field.
__device__ __forceinline__ void write_empty_result(PairResult* out, int32_t status, int64_t sessions) {
  out->att.sessions_total = sessions;
  out->att.sessions_completed = out->att.slo_ok = out->att.ttft_ok = out->att.itl_ok = 0;
  out->ctr.tasks_created = out->ctr.tasks_completed = out->ctr.tokens_decoded = out->ctr.kv_bytes_residual = 0;
  out->ctr.max_postpone_observed = out->ctr.events_in_order = 0;
  out->n_decisions = out->n_ttft = out->n_steps = out->n_spans = out->events = out->cycles = out->exact_folds = 0;
  out->status = status;
  out->attempts = 0;
  for (int j = 0; j < PDSIM_PROF_BUCKETS; ++j) out->prof_cycles[j] = out->prof_count[j] = 0;
}
__device__ __forceinline__ void write_empty_report(pdsim_report* rep, int64_t sessions) {
  pdsim_report z;
  memset(&z, 0, sizeof(z));
  z.sessions_total = sessions;
  z.empty = 1;
  *rep = z;
}

// One warp per block; the warp replays pairs pulled from an atomic queue.
// kD/kP: DecodeW/PrefillW entries reserved in shared memory; the engine
// addresses slot state at compile-time offsets (engine.cuh smem_off).
// PDG_MIN_BLOCKS: resident-warp target handed to ptxas (register budget per
// lane = 64K / (32 * PDG_MIN_BLOCKS)); 1 = unconstrained.
#ifndef PDG_MIN_BLOCKS
#define PDG_MIN_BLOCKS 1
#endif
template <bool kProf, int kD, int kP, bool kRec, bool kPrune = false>
__global__ void __launch_bounds__(32, PDG_MIN_BLOCKS) replay_kernel(KernelArgs a) {
  const int slot_id = blockIdx.x;
  GlobalSlot gslot;
  global_slot_bytes(a.caps, &gslot, a.ws + static_cast<size_t>(slot_id) * a.slot_bytes);
  SmemSlot sslot;
  smem_slot_bytes(a.caps, &sslot, pdg_smem);  // EngState first (engine.cuh)
  {
    constexpr SmemOff off = smem_off(kD, kP);
    if (a.caps.dres != kD || a.caps.pres != kP || reinterpret_cast<char*>(sslot.dw) != pdg_smem + off.dw ||
        reinterpret_cast<char*>(sslot.pw) != pdg_smem + off.pw || reinterpret_cast<char*>(sslot.heap) != pdg_smem + off.heap) {
      __trap();  // host/device slot layouts disagree: never replay on a wrong layout
    }
  }
  const int lane = threadIdx.x & 31;
  unsigned smid = 0;
  if (a.sm_items) asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  for (;;) {
    // Item `idx` of the launch: pair_begin + idx, or pair_list[idx] (a shard
    // of the search in cost order, pdsim_shard_pairs). Per-pair outputs are
    // indexed by item; argmax-mode bounds by global pair (c * n_traces + r).
    int64_t idx;
    if (a.sm_items) {
      idx = take_sm_affine(a.sm_items, a.sm_off, a.sm_next, a.n_lists, smid);
      if (idx < 0) break;
    } else {
      unsigned long long ticket = 0;
      if (lane == 0) ticket = atomicAdd(a.next_pair, 1ull);
      ticket = __shfl_sync(0xffffffffu, ticket, 0);
      idx = static_cast<int64_t>(ticket);
      if (idx >= a.pair_end - a.pair_begin) break;
    }
    const int64_t pair = a.pair_list ? a.pair_list[idx] : a.pair_begin + idx;
    const int32_t c = static_cast<int32_t>(pair / a.n_traces);
    const int32_t r = static_cast<int32_t>(pair % a.n_traces);
    // Per-pair result: written straight to a.results[idx] by lane 0 (no
    // local copy); the counters the reduction needs are read back after.
    PairResult* out = a.results + idx;
    if (kPrune) {  // a dead candidate's remaining replicas are not replayed
      const unsigned long long key = *reinterpret_cast<volatile unsigned long long*>(a.best_key);
      if ((*reinterpret_cast<volatile int*>(&a.cand_bad[c]) & 2) || prune_dominated(a.total_sessions, key, c)) {
        if (lane == 0) write_empty_result(out, PDSIM_PAIR_PRUNED, a.traces[r].S);
        goto reduce;
      }
    }
    if (a.pair_invalid[pair]) {
      if (lane == 0) {
        write_empty_result(out, PDSIM_PAIR_INVALID, a.traces[r].S);
        if (a.reports) write_empty_report(a.reports + idx, a.traces[r].S);
      }
    } else {
      const DevTrace tr = a.traces[r];
      const DevPlan pl = a.plans[c];
      const long long t0 = clock64();
      const DevParams prm = a.cand_params ? a.cand_params[c] : a.params;
      Prune prn;
      memset(&prn, 0, sizeof(prn));
      if (kPrune) {
        prn.best = a.best_key;
        prn.pair_fail = a.pair_fail;
        prn.pair_ok = a.pair_ok;
        prn.c_invalid = a.cand_invalid[c];
        prn.cand_bad = a.cand_bad;
        prn.total_sessions = a.total_sessions;
        // Bounds over every replica of c: replicas outside this launch (or
        // on another GPU) read as 0 failures / 0 attained, which keeps the
        // upper bound (total_sessions of the whole search - failures) and
        // the lower bound (attained so far) valid for the global argmax.
        prn.self = pair;
        prn.fail_base = static_cast<int64_t>(c) * a.n_traces;
        prn.r_lo = 0;
        prn.r_hi = a.n_traces;
        prn.c = c;
      }
      EngineT<kProf, kD, kP, kRec, true, kPrune> eng(sslot.es, tr, pl, prm, a.caps, sslot, gslot, a.rec, a.seed, kProf ? 1 : 0,
                                       &prn);
      eng.run(out);
      if (lane == 0) out->cycles = clock64() - t0;
      if (kRec && a.reports) {
        pdsim_report rep;
        eng.build_report(&rep);
        if (lane == 0) a.reports[idx] = rep;
      }
    }
  reduce:
    __syncwarp();
    if (lane == 0) {
      const int32_t status = out->status;
      const int64_t slo_ok = out->att.slo_ok, total = out->att.sessions_total;
      if (status == PDSIM_PAIR_PRUNED) {
        atomicOr(&a.cand_bad[c], 2);
      } else if (status != PDSIM_PAIR_OK) {
        atomicOr(&a.cand_bad[c], 1);
      } else {
        const unsigned long long old = atomicAdd(&a.cand_sum[c], static_cast<unsigned long long>(slo_ok));
        if (kPrune) {  // final counts join the replicas' bounds
          atomicMax(&a.pair_ok[pair], static_cast<int32_t>(slo_ok));
          atomicMax(&a.pair_fail[pair], static_cast<int32_t>(total - slo_ok));
        }
        if (kPrune && !a.cand_invalid[c]) {  // completed replicas: a lower bound of c's count
          const unsigned long long lb = old + static_cast<unsigned long long>(slo_ok);
          atomicMax(a.best_key, ((lb + 1ull) << 32) | (0xffffffffull - static_cast<unsigned>(c)));
        }
      }
    }
    __syncwarp();
  }
}


using ReplayKernel = void (*)(KernelArgs);

// Kernel of layout (0: <8,8>, 1: <16,16>, 2: <64,32>) and variant (0 search,
// 1 diagnostics, 2 records/reports); defined across replay_l*.cu.
ReplayKernel replay_kernel_for(int layout, int variant);
// Copies the cost model into every translation unit's __constant__ bank.
cudaError_t replay_set_profile(const pdsim_profile* profile, cudaStream_t stream);

ReplayKernel replay_kernels_l0(int variant);
ReplayKernel replay_kernels_l1(int variant);
ReplayKernel replay_kernels_l2(int variant);
cudaError_t replay_set_profile_l0(const pdsim_profile* profile, cudaStream_t stream);
cudaError_t replay_set_profile_l1(const pdsim_profile* profile, cudaStream_t stream);
cudaError_t replay_set_profile_l2(const pdsim_profile* profile, cudaStream_t stream);

}  // namespace pdg
