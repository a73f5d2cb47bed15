// capi.cu — C-ABI implementation (include/pdsim_gpu.h) and the replay kernels.
//
// Drop-in for pdsim::run (reference proj/src/sim_engine.cpp:676-681) and the
// batched candidate x replica search composed from it. All
// replays execute on the GPU; there is no host execution path: a missing or
// non-sm_100 device is a PDSIM_ERR_CUDA failure.
//
// Kernels
//   replay_kernel  : persistent; one warp per workspace slot pulls
//                    (candidate, replica) pairs from an atomic queue and replays
//                    each with pdg::Engine (engine.cuh); SLO counts are folded
//                    into per-candidate int64 sums with integer atomics
//                    (deterministic).
//   argmax_kernel  : one warp; max Σslo_ok over valid candidates, ties to the
//                    smallest enumeration index.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "engine.cuh"
#include "nccl_dl.hpp"
#include "pack.hpp"
#include "shard.hpp"
#include "planner.cuh"
#include "replay.cuh"
#include "pdsim_gpu.h"

// Throughput build of the search kernels (replay_tp_l*.o, Makefile): the same
// sources compiled in namespace pdg_tp with the shared hot subroutines kept
// out of line — a smaller instruction footprint when many warps share an SM
// (DESIGN.md §3.1). Its KernelArgs is pdg::KernelArgs (same source, same
// layout); only the search variants (0, 3) exist there.
namespace pdg_tp {
struct KernelArgs;
using ReplayKernel = void (*)(KernelArgs);
ReplayKernel replay_kernel_for(int layout, int variant);
cudaError_t replay_set_profile(const pdsim_profile* profile, cudaStream_t stream);
}  // namespace pdg_tp

namespace {

thread_local std::string g_last_error;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t reserve(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace

namespace pdg {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace pdg

struct pdsim_gpu_ctx {
  int device = 0;
  int sm_count = 0;
  int kernel_build = PDSIM_BUILD_AUTO;
  int last_build = 0;  // build of the last replay launch
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

  // staged inputs
  bool staged = false;
  int32_t n_traces = 0, n_candidates = 0;
  pdsim_profile profile{};
  pdsim_sched_params params{};
  std::vector<pdg::DevParams> cand_params;  // sweep: scheduler settings per candidate (empty: `params`)
  std::vector<pdg::PackedTrace> packed;
  std::vector<pdg::DevPlan> plans;
  std::vector<int8_t> pair_invalid;  // [n_candidates * n_traces], host precheck
  pdg::Caps caps{};
  size_t slot_bytes = 0;   // global workspace per slot
  size_t smem_bytes = 0;   // dynamic shared memory per slot (one warp / block)
  DevBuf d_trace_data, d_traces, d_plans, d_invalid, d_cand_params, d_cand_inv;
  std::vector<int8_t> cand_invalid;  // [n_candidates]: some pair of c is invalid (whole search)
  int64_t total_sessions = 0;        // sum of S over the staged traces
  int64_t global_sessions = 0;       // > 0: sum of S over every replica of a sharded search (argmax bounds)
  DevBuf d_pair_list;                // launch pair list (sharded / cost-ordered searches)
  DevBuf d_sm_items, d_sm_off, d_sm_next;  // candidate-affine per-SM queues (throughput build)
  std::vector<int64_t> h_sm_items;         // their host staging (asynchronous copies)
  std::vector<int32_t> h_sm_off;
  ncclComm_t comm = nullptr;         // set: every search all-reduces its candidate counts over it
  int32_t comm_world = 1, comm_rank = 0;
  int search_mode = 0;               // PDSIM_SEARCH_*
  DevBuf d_pair_fail, d_pair_ok, d_best_key;  // argmax mode (pruning) state
  // per-search buffers
  DevBuf d_ws, d_results, d_cand_sum, d_cand_bad, d_counter, d_best;
  // single-run records
  DevBuf d_dec, d_ttft, d_sess, d_steps, d_spans, d_reports;
  // surrogate-planner phase sims
  DevBuf d_ph_data, d_ph_traces, d_ph_jobs, d_ph_out, d_ph_scratch, d_ph_counter, d_ph_profile;
  // diagnostics
  int profiling = 0;
  int layout = 0;  // index of the compiled shared-memory layout (stage_impl)
  int64_t prof_cycles[PDSIM_PROF_BUCKETS] = {0};
  int64_t prof_count[PDSIM_PROF_BUCKETS] = {0};
  int64_t attempts2 = 0;
};

namespace {

int set_err(pdsim_gpu_ctx* ctx, int code, const std::string& msg) {
  g_last_error = msg;
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_err(pdsim_gpu_ctx* ctx, cudaError_t e, const char* what) {
  return set_err(ctx, PDSIM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CU(ctx, expr)                                  \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return cuda_err(ctx, _e, #expr); \
  } while (0)

// ---------------------------------------------------------------------------
// Kernels

// Packed key: (slo_ok + 1) << 32 | (0xffffffff - c); 0 = invalid. One max
// reduction yields max count with ties to the smallest index.
__global__ void argmax_kernel(const unsigned long long* cand_sum, const int* cand_bad, int n,
                              unsigned long long* best) {
  unsigned long long key = 0;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    if (!cand_bad[c]) {
      const unsigned long long k = ((cand_sum[c] + 1ull) << 32) | (0xffffffffull - static_cast<unsigned>(c));
      key = k > key ? k : key;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_down_sync(0xffffffffu, key, o);
    key = other > key ? other : key;
  }
  __shared__ unsigned long long warp_best[32];
  if ((threadIdx.x & 31) == 0) warp_best[threadIdx.x >> 5] = key;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long k = 0;
    for (int w = 0; w < static_cast<int>((blockDim.x + 31) / 32); ++w) k = warp_best[w] > k ? warp_best[w] : k;
    *best = k;
  }
}

// ---------------------------------------------------------------------------
// The cost model lives in one __constant__ bank per module (engine.cuh
// c_profile): every context on a device shares it. A context uploads its
// profile and launches under a per-device lease; leases on the same profile
// run concurrently, a different profile waits until the device's running
// searches have finished, then replaces the bank. The lease ends after the
// search's stream synchronisation, so a kernel never sees another context's
// cost model.
struct ProfileGate {
  std::mutex m;
  std::condition_variable cv;
  bool loaded = false;
  pdsim_profile cur{};
  int active = 0;
};

ProfileGate& profile_gate(int device) {
  static ProfileGate gates[64];
  return gates[device & 63];
}

class ProfileLease {
 public:
  explicit ProfileLease(pdsim_gpu_ctx* ctx) : ctx_(ctx) {}
  ProfileLease(const ProfileLease&) = delete;
  ProfileLease& operator=(const ProfileLease&) = delete;
  cudaError_t acquire();
  ~ProfileLease();

 private:
  pdsim_gpu_ctx* ctx_;
  bool held_ = false;
};

cudaError_t ProfileLease::acquire() {
  ProfileGate& g = profile_gate(ctx_->device);
  std::unique_lock<std::mutex> lk(g.m);
  auto same = [&] { return g.loaded && memcmp(&g.cur, &ctx_->profile, sizeof(pdsim_profile)) == 0; };
  g.cv.wait(lk, [&] { return g.active == 0 || same(); });
  if (!same()) {
    cudaError_t e = pdg::replay_set_profile(&ctx_->profile, ctx_->stream);
    if (e == cudaSuccess) e = pdg_tp::replay_set_profile(&ctx_->profile, ctx_->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx_->stream);
    if (e != cudaSuccess) {
      g.loaded = false;
      return e;
    }
    g.cur = ctx_->profile;
    g.loaded = true;
  }
  ++g.active;
  held_ = true;
  return cudaSuccess;
}

ProfileLease::~ProfileLease() {
  if (!held_) return;
  cudaStreamSynchronize(ctx_->stream);  // error paths: the kernel must be done before the bank may change
  ProfileGate& g = profile_gate(ctx_->device);
  {
    std::lock_guard<std::mutex> lk(g.m);
    --g.active;
  }
  g.cv.notify_all();
}

// Candidate flags before the cross-GPU max-reduction: bit 0 = invalid on
// this GPU, bit 1 = pruned here. Invalid anywhere must win over pruned, so
// invalid becomes 3 (both bits): max() then keeps bit 0 whenever any rank
// saw the candidate invalid, and bit 1 alone means pruned somewhere.
__global__ void flags_for_max_kernel(int* cand_bad, int n) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (cand_bad[c] & 1) cand_bad[c] = 3;
  }
}

// ---------------------------------------------------------------------------
// Host orchestration

int check_ctx(pdsim_gpu_ctx* ctx) {
  if (!ctx) return set_err(nullptr, PDSIM_ERR_CONFIG, "null context");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_err(ctx, e, "cudaSetDevice");
  return PDSIM_OK;
}

// `cand_params` (sweep; may be null) gives candidate c its own scheduler
// settings; `params` then only supplies defaults for unset fields (none).
int stage_impl(pdsim_gpu_ctx* ctx, const pdsim_search_input* in, const pdsim_profile* profile,
               const pdsim_sched_params* params, int64_t* h2d_bytes, const pdsim_sched_params* cand_params = nullptr) {
  if (!in || !profile || !params) return set_err(ctx, PDSIM_ERR_CONFIG, "null argument");
  if (in->n_traces < 1 || in->n_candidates < 1 || !in->traces || !in->candidates) {
    return set_err(ctx, PDSIM_ERR_CONFIG, "search: need at least one trace and one candidate");
  }
  ctx->staged = false;
  pdg::HostError err;
  // Reference validation order (sim_engine.cpp:115-122): every setting
  // against every trace, settings in order (the reference sweep throws at
  // the first invalid combination, pdsim.cpp:547-559).
  const int n_set = cand_params ? in->n_candidates : 1;
  const pdsim_sched_params* sets = cand_params ? cand_params : params;
  for (int k = 0; k < n_set; ++k) {
    for (int r = 0; r < in->n_traces; ++r) {
      if (!pdg::validate_params(sets[k], in->traces[r].ttft_thres, in->traces[r].itl_thres, &err)) {
        return set_err(ctx, err.code, err.msg);
      }
    }
  }
  ctx->packed.assign(static_cast<size_t>(in->n_traces), pdg::PackedTrace());
  bool any_sessions = false;
  {
    // Replicas are validated and packed on all host threads; the first
    // failing trace in input order is reported.
    const int nt = in->n_traces;
    std::vector<pdg::HostError> errs(static_cast<size_t>(nt));
    std::vector<char> ok(static_cast<size_t>(nt), 1);
    auto pack = [&](int r) {
      ok[static_cast<size_t>(r)] =
          pdg::pack_trace(in->traces[r], &ctx->packed[static_cast<size_t>(r)], &errs[static_cast<size_t>(r)]) ? 1 : 0;
    };
    const int nth = std::min<int>(nt, static_cast<int>(std::max(1u, std::thread::hardware_concurrency())));
    if (nth > 1) {
      std::atomic<int> next{0};
      std::vector<std::thread> pool;
      for (int k = 0; k < nth; ++k) {
        pool.emplace_back([&] {
          for (int r = next++; r < nt; r = next++) pack(r);
        });
      }
      for (auto& t : pool) t.join();
    } else {
      for (int r = 0; r < nt; ++r) pack(r);
    }
    for (int r = 0; r < nt; ++r) {
      if (!ok[static_cast<size_t>(r)]) return set_err(ctx, errs[static_cast<size_t>(r)].code, errs[static_cast<size_t>(r)].msg);
      any_sessions |= ctx->packed[static_cast<size_t>(r)].S > 0;
    }
  }
  if (!pdg::validate_profile(*profile, &err)) return set_err(ctx, err.code, err.msg);
  for (int k = 0; k < n_set; ++k) {
    if (sets[k].reorder && sets[k].window > 8 && any_sessions) {
      // reorder_and_dequeue throws at the first dequeue (reorder.cpp:86-90).
      return set_err(ctx, PDSIM_ERR_CONFIG, "reorder: window must be <= 8");
    }
  }
  // Window ring capacities follow the longest statistics window of any setting.
  pdsim_sched_params cap_params = sets[0];
  for (int k = 1; k < n_set; ++k) cap_params.stat_window = std::max(cap_params.stat_window, sets[k].stat_window);
  ctx->cand_params.clear();
  if (cand_params) {
    for (int k = 0; k < n_set; ++k) ctx->cand_params.push_back(pdg::to_dev_params(sets[k]));
  }
  ctx->plans.assign(static_cast<size_t>(in->n_candidates), pdg::DevPlan());
  int pmax = 0, dmax = 1;
  for (int c = 0; c < in->n_candidates; ++c) {
    pdg::DevPlan& p = ctx->plans[static_cast<size_t>(c)];
    memset(&p, 0, sizeof(p));
    if (!pdg::pack_plan(in->candidates[c], *profile, &p, &err)) return set_err(ctx, err.code, err.msg);
    pmax = std::max(pmax, p.P);
    dmax = std::max(dmax, p.D);
  }
  ctx->pair_invalid.assign(static_cast<size_t>(in->n_candidates) * in->n_traces, 0);
  for (int c = 0; c < in->n_candidates; ++c)
    for (int r = 0; r < in->n_traces; ++r)
      ctx->pair_invalid[static_cast<size_t>(c) * in->n_traces + r] =
          pdg::precheck(ctx->packed[static_cast<size_t>(r)], ctx->plans[static_cast<size_t>(c)], *profile) ? 0 : 1;

  ctx->cand_invalid.assign(static_cast<size_t>(in->n_candidates), 0);
  for (int c = 0; c < in->n_candidates; ++c)
    for (int r = 0; r < in->n_traces; ++r)
      ctx->cand_invalid[static_cast<size_t>(c)] |= ctx->pair_invalid[static_cast<size_t>(c) * in->n_traces + r];
  ctx->total_sessions = 0;
  for (const auto& t : ctx->packed) ctx->total_sessions += t.S;
  // Argmax / pruning keys pack (count + 1) into 32 bits (argmax_kernel).
  if (ctx->total_sessions >= static_cast<int64_t>(0xfffffffeLL)) {
    return set_err(ctx, PDSIM_ERR_CONFIG, "search: the replicas hold 2^32-2 or more sessions (argmax key range)");
  }

  std::vector<const pdg::PackedTrace*> tp;
  for (auto& t : ctx->packed) tp.push_back(&t);
  // Shared-memory budget per slot: generous when few pairs run at once.
  const int64_t pairs = static_cast<int64_t>(in->n_traces) * in->n_candidates;
  size_t smem_budget = pairs <= 2 * ctx->sm_count ? (size_t(96) << 10)
                       : pairs <= 8 * ctx->sm_count ? (size_t(24) << 10)
                                                    : size_t(9216);  // 24 warps/SM (the throughput build's register budget)
  if (pairs > 8 * ctx->sm_count && pairs < 22 * static_cast<int64_t>(ctx->sm_count)) {
    // Every pair resident at once (C3: 18.3 per SM): the largest slot that
    // still fits ceil(pairs / SMs) blocks per SM (228 KB shared memory per
    // SM, 1 KB reserved per block): C3s 10-11 KB vs 9 KB -2 %
    // (profiles/round2/ab_smem_budget_v24.log).
    const int64_t per_sm = (pairs + ctx->sm_count - 1) / ctx->sm_count;
    const size_t fit = ((size_t(228) << 10) / static_cast<size_t>(per_sm) - 1024) & ~size_t(511);
    smem_budget = std::max(smem_budget, std::min(fit, size_t(24) << 10));
  }
  if (const char* v = getenv("PDSIM_SMEM_BUDGET")) smem_budget = static_cast<size_t>(atoll(v));  // tuning only
  // Compiled shared-memory layouts (replay_kernel<.., kD, kP>): N <= 8 plans
  // fit <8, 8>, N <= 16 plans <16, 16>; D + 2P <= 64 bounds the rest.
  const int lay = (dmax <= 8 && pmax <= 8) ? 0 : (dmax <= 16 && pmax <= 16) ? 1 : 2;
  static const int kLayD[3] = {8, 16, 64}, kLayP[3] = {8, 16, 32};
  ctx->layout = lay;
  ctx->caps = pdg::compute_caps(tp, pmax, dmax, *profile, cap_params, smem_budget, kLayD[lay], kLayP[lay]);
  ctx->slot_bytes = pdg::global_slot_bytes(ctx->caps, nullptr, nullptr);
  ctx->smem_bytes = pdg::smem_slot_bytes(ctx->caps, nullptr, nullptr);
  ctx->profile = *profile;
  ctx->params = *params;
  ctx->n_traces = in->n_traces;
  ctx->n_candidates = in->n_candidates;

  // H2D: trace arrays (one contiguous buffer), DevTrace table, plans, flags.
  size_t total = 0;
  for (auto& t : ctx->packed) total += pdg::align_up(t.device_bytes() + 8 * 256);
  CU(ctx, ctx->d_trace_data.reserve(std::max<size_t>(total, 256)));
  std::vector<pdg::DevTrace> dt(static_cast<size_t>(in->n_traces));
  std::vector<char> host(std::max<size_t>(total, 256));
  size_t off = 0;
  char* dbase = ctx->d_trace_data.as<char>();
  auto put = [&](const void* src, size_t bytes) -> void* {
    void* dst = dbase + off;
    if (bytes) memcpy(host.data() + off, src, bytes);
    off = pdg::align_up(off + bytes);
    return dst;
  };
  for (size_t r = 0; r < ctx->packed.size(); ++r) {
    const pdg::PackedTrace& t = ctx->packed[r];
    pdg::DevTrace& d = dt[r];
    d.S = t.S;
    d.R = t.R;
    d.max_dec = t.max_dec;
    d.rank_is_index = 1;
    for (size_t k = 0; k < t.by_rank.size(); ++k) {
      if (t.by_rank[k] != static_cast<int32_t>(k)) {
        d.rank_is_index = 0;
        break;
      }
    }
    d.ttft_thres = t.ttft_thres;
    d.itl_thres = t.itl_thres;
    d.ss = static_cast<const pdg::SessTr*>(put(t.stab.data(), t.stab.size() * sizeof(pdg::SessTr)));
    d.rr = static_cast<const pdg::RoundTr*>(put(t.rtab.data(), t.rtab.size() * sizeof(pdg::RoundTr)));
    d.sid = static_cast<const int64_t*>(put(t.sid.data(), t.sid.size() * 8));
    d.by_rank = static_cast<const int32_t*>(put(t.by_rank.data(), t.by_rank.size() * 4));
  }
  CU(ctx, cudaMemcpyAsync(ctx->d_trace_data.p, host.data(), off, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, ctx->d_traces.reserve(sizeof(pdg::DevTrace) * dt.size()));
  CU(ctx, cudaMemcpyAsync(ctx->d_traces.p, dt.data(), sizeof(pdg::DevTrace) * dt.size(), cudaMemcpyHostToDevice,
                          ctx->stream));
  CU(ctx, ctx->d_plans.reserve(sizeof(pdg::DevPlan) * ctx->plans.size()));
  CU(ctx, cudaMemcpyAsync(ctx->d_plans.p, ctx->plans.data(), sizeof(pdg::DevPlan) * ctx->plans.size(),
                          cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, ctx->d_invalid.reserve(ctx->pair_invalid.size()));
  CU(ctx, cudaMemcpyAsync(ctx->d_invalid.p, ctx->pair_invalid.data(), ctx->pair_invalid.size(),
                          cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, ctx->d_cand_inv.reserve(ctx->cand_invalid.size()));
  CU(ctx, cudaMemcpyAsync(ctx->d_cand_inv.p, ctx->cand_invalid.data(), ctx->cand_invalid.size(), cudaMemcpyHostToDevice,
                          ctx->stream));
  if (!ctx->cand_params.empty()) {
    CU(ctx, ctx->d_cand_params.reserve(sizeof(pdg::DevParams) * ctx->cand_params.size()));
    CU(ctx, cudaMemcpyAsync(ctx->d_cand_params.p, ctx->cand_params.data(),
                            sizeof(pdg::DevParams) * ctx->cand_params.size(), cudaMemcpyHostToDevice, ctx->stream));
  }
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  if (h2d_bytes) {
    *h2d_bytes = static_cast<int64_t>(off + sizeof(pdg::DevTrace) * dt.size() +
                                      sizeof(pdg::DevPlan) * ctx->plans.size() + ctx->pair_invalid.size() +
                                      sizeof(pdg::DevParams) * ctx->cand_params.size() + sizeof(pdsim_profile));
  }
  ctx->staged = true;
  return PDSIM_OK;
}

// Replays pairs [b, e) of the staged inputs; results land in host buffers.
// With `list` (n_list entries), the launch replays those pairs in list order
// instead of the range; per-pair outputs follow the list.
int search_impl(pdsim_gpu_ctx* ctx, int64_t b, int64_t e, uint64_t seed, pdsim_search_output* out,
                pdg::Records rec, pdg::PairResult* single_result, const int64_t* list = nullptr,
                int64_t n_list = 0) {
  if (!ctx->staged) return set_err(ctx, PDSIM_ERR_CONFIG, "search: nothing staged");
  const int64_t total = static_cast<int64_t>(ctx->n_traces) * ctx->n_candidates;
  if (list) {
    if (n_list < 0) return set_err(ctx, PDSIM_ERR_CONFIG, "search: negative pair-list length");
    std::vector<uint8_t> seen(static_cast<size_t>(total), 0);
    for (int64_t k = 0; k < n_list; ++k) {
      if (list[k] < 0 || list[k] >= total) return set_err(ctx, PDSIM_ERR_CONFIG, "search: pair index out of range");
      if (seen[static_cast<size_t>(list[k])]++) return set_err(ctx, PDSIM_ERR_CONFIG, "search: duplicate pair in list");
    }
    b = 0;
    e = n_list;
  }
  if (e < 0) e = total;
  if (b < 0 || b > e || (!list && e > total)) return set_err(ctx, PDSIM_ERR_CONFIG, "search: bad pair range");
  const int64_t n = e - b;
  const int C = ctx->n_candidates;
  // Report mode widens the global workspace layout (the shared-memory layout
  // is unchanged): TTFT values, e2e latencies and the ITL gap histogram.
  const bool report = out && out->pair_report;
  pdg::Caps caps = ctx->caps;
  if (report) {
    int32_t max_r = 1;
    for (const auto& t : ctx->packed) max_r = std::max(max_r, t.R);
    caps.rep_r = max_r;
    // Distinct ITL gaps <= decode steps <= decode tokens: 2x the largest
    // trace's token count (load factor <= 1/2) guarantees room; capped at
    // 2^24 entries (256 MiB per slot). Beyond the cap a full table is a loud
    // PDSIM_PAIR_ERROR, never a silent miscount.
    int64_t max_tok = 1;
    for (const auto& t : ctx->packed) max_tok = std::max<int64_t>(max_tok, t.total_decode);
    int32_t cap = 1 << 12;
    while (cap < (1 << 24) && static_cast<int64_t>(cap) < 2 * max_tok) cap <<= 1;
    caps.rep_gapcap = cap;
  }
  const size_t slot_bytes = pdg::global_slot_bytes(caps, nullptr, nullptr);

  // Workspace slots: one warp each, at most 32 resident per SM, bounded by a
  // memory budget.
  size_t free_b = 0, total_b = 0;
  CU(ctx, cudaMemGetInfo(&free_b, &total_b));
  const size_t budget = std::min<size_t>(free_b / 2 + ctx->d_ws.bytes / 2, size_t(64) << 30);
  int64_t per_sm = std::max<int64_t>(
      1, std::min<int64_t>(32, static_cast<int64_t>((size_t(227) << 10) / std::max<size_t>(ctx->smem_bytes, 1))));
  if (const char* v = getenv("PDSIM_SLOTS_PER_SM")) per_sm = std::max<int64_t>(1, std::min<int64_t>(per_sm, atoll(v)));  // tuning only
  int64_t slots = std::min<int64_t>(std::max<int64_t>(n, 1), static_cast<int64_t>(ctx->sm_count) * per_sm);
  slots = std::min<int64_t>(slots, static_cast<int64_t>(budget / std::max<size_t>(slot_bytes, 1)));
  if (slots < 1) return set_err(ctx, PDSIM_ERR_CUDA, "search: workspace of one slot exceeds device memory");
  CU(ctx, ctx->d_ws.reserve(slot_bytes * static_cast<size_t>(slots)));
  if (report) CU(ctx, ctx->d_reports.reserve(sizeof(pdsim_report) * static_cast<size_t>(std::max<int64_t>(n, 1))));
  CU(ctx, ctx->d_results.reserve(sizeof(pdg::PairResult) * static_cast<size_t>(std::max<int64_t>(n, 1))));
  CU(ctx, ctx->d_cand_sum.reserve(8 * static_cast<size_t>(C)));
  CU(ctx, ctx->d_cand_bad.reserve(4 * static_cast<size_t>(C)));
  CU(ctx, ctx->d_counter.reserve(8));
  CU(ctx, ctx->d_best.reserve(8));

  CU(ctx, cudaEventRecord(ctx->ev[0], ctx->stream));
  CU(ctx, cudaMemsetAsync(ctx->d_cand_sum.p, 0, 8 * static_cast<size_t>(C), ctx->stream));
  CU(ctx, cudaMemsetAsync(ctx->d_cand_bad.p, 0, 4 * static_cast<size_t>(C), ctx->stream));
  CU(ctx, cudaMemsetAsync(ctx->d_counter.p, 0, 8, ctx->stream));

  pdg::KernelArgs a;
  memset(&a, 0, sizeof(a));
  a.traces = ctx->d_traces.as<pdg::DevTrace>();
  a.plans = ctx->d_plans.as<pdg::DevPlan>();
  a.pair_invalid = ctx->d_invalid.as<int8_t>();
  a.n_traces = ctx->n_traces;
  a.pair_begin = b;
  a.pair_end = e;
  a.params = pdg::to_dev_params(ctx->params);
  a.cand_params = ctx->cand_params.empty() ? nullptr : ctx->d_cand_params.as<pdg::DevParams>();
  a.caps = caps;
  a.ws = ctx->d_ws.as<char>();
  a.slot_bytes = slot_bytes;
  a.reports = report ? ctx->d_reports.as<pdsim_report>() : nullptr;
  a.smem_bytes = ctx->smem_bytes;
  a.next_pair = ctx->d_counter.as<unsigned long long>();
  a.results = ctx->d_results.as<pdg::PairResult>();
  a.cand_sum = ctx->d_cand_sum.as<unsigned long long>();
  a.cand_bad = ctx->d_cand_bad.as<int>();
  a.rec = rec;
  a.seed = seed;
  a.profile = ctx->profiling;
  const bool with_rec0 = a.reports || rec.decisions || rec.ttft || rec.sessions || rec.steps;
  // (a single candidate is its own argmax: nothing to prune)
  const bool prune = ctx->search_mode == PDSIM_SEARCH_ARGMAX && !with_rec0 && !ctx->profiling && n > 0 && C > 1;
  if (list && n > 0) {
    CU(ctx, ctx->d_pair_list.reserve(8 * static_cast<size_t>(n)));
    CU(ctx, cudaMemcpyAsync(ctx->d_pair_list.p, list, 8 * static_cast<size_t>(n), cudaMemcpyHostToDevice, ctx->stream));
    a.pair_list = ctx->d_pair_list.as<int64_t>();
  }
  // Build choice (needed by the queue policy below): many warps per SM (more
  // than 4 pairs per SM in this launch; measured crossover,
  // tools/build_threshold.py, profiles/round2/build_threshold_v20.jsonl) run
  // the throughput build; few pairs the inlined build (lowest latency per event).
  const bool with_rec = a.reports || rec.decisions || rec.ttft || rec.sessions || rec.steps;
  // variant 0: attainment-only search, 1: diagnostics (clock64 phases; N <= 8
  // layout only), 2: record / report outputs (drop-in run(), ITL samples, pair
  // reports), 3: attainment-only search in argmax mode (Prune, engine.cuh).
  const int variant = with_rec ? 2 : ctx->profiling ? 1 : prune ? 3 : 0;
  const bool search_only = variant == 0 || variant == 3;
  const bool tp = search_only && (ctx->kernel_build == PDSIM_BUILD_THROUGHPUT ||
                                  (ctx->kernel_build == PDSIM_BUILD_AUTO && n > 4 * static_cast<int64_t>(ctx->sm_count)));
  // Candidate-affine queues (throughput build): one list per SM holding a
  // contiguous run of the launch items grouped by candidate (launch order kept
  // within a candidate), taken first by the warps of that SM, then stolen in
  // ring order. Co-resident warps then replay the same plan, whose handler mix
  // shares the instruction cache: the throughput regime is bound by
  // instruction fetch; measured C3s -8.7 %, C5 slice -4 %
  // (profiles/round2/ab_sm_affinity_v22.log). It pays from about 8 pairs per
  // SM (C3s shards, profiles/round2/shard_affinity_c3s_v23.jsonl: 9 per SM
  // -7 %, 4.6 per SM +3 %, 2.3 per SM neutral). PDSIM_SM_AFFINITY=0/1 forces it.
  const char* aff_env = getenv("PDSIM_SM_AFFINITY");
  const bool affine = n > 0 && n < (int64_t(1) << 31) &&  // (int32 list offsets)
                     (aff_env ? atoi(aff_env) > 0 : tp && n > 8 * static_cast<int64_t>(ctx->sm_count));
  if (affine) {
    const int L = ctx->sm_count;
    auto& items = ctx->h_sm_items;
    auto& off = ctx->h_sm_off;
    std::vector<int64_t> start(static_cast<size_t>(C) + 1, 0);  // counting sort by candidate
    for (int64_t i = 0; i < n; ++i) ++start[static_cast<size_t>((list ? list[i] : b + i) / ctx->n_traces) + 1];
    for (int64_t c = 0; c < C; ++c) start[static_cast<size_t>(c) + 1] += start[static_cast<size_t>(c)];
    std::vector<int64_t> srt(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) srt[static_cast<size_t>(start[static_cast<size_t>((list ? list[i] : b + i) / ctx->n_traces)]++)] = i;
    off.resize(static_cast<size_t>(L) + 1);
    // One contiguous chunk per SM. In argmax mode with more pairs than
    // resident warps, groups of one SM's resident warps are dealt round-robin
    // instead (list s = groups s, s+L, ...): each SM still works on one group
    // at a time, but the search as a whole advances in launch order, so the
    // incumbent rises as early as with the plain queue (C5 grid, argmax:
    // contiguous 89.3 s, plain 59.8 s, round-robin 55.9 s; full mode on the
    // C5 slice: contiguous -4.4 %, round-robin -2.5 % vs plain;
    // profiles/round2/ab_sm_affinity_v22.log).
    const int64_t per_sm = (slots + L - 1) / L;
    const char* gv = getenv("PDSIM_SM_GROUP");  // A/B: 0 contiguous, 1 round-robin
    const bool round_robin = gv ? atoi(gv) == 1 : prune;
    if (n <= slots || !round_robin) {
      items.swap(srt);
      for (int s = 0; s <= L; ++s) off[static_cast<size_t>(s)] = static_cast<int32_t>(n * s / L);
    } else {
      const int64_t G = std::max<int64_t>(1, per_sm), ng = (n + G - 1) / G;
      items.clear();
      items.reserve(static_cast<size_t>(n));
      for (int s = 0; s < L; ++s) {
        off[static_cast<size_t>(s)] = static_cast<int32_t>(items.size());
        for (int64_t g = s; g < ng; g += L) {
          for (int64_t k = g * G; k < std::min(n, (g + 1) * G); ++k) items.push_back(srt[static_cast<size_t>(k)]);
        }
      }
      off[static_cast<size_t>(L)] = static_cast<int32_t>(n);
    }
    CU(ctx, ctx->d_sm_items.reserve(8 * static_cast<size_t>(n)));
    CU(ctx, ctx->d_sm_off.reserve(4 * off.size()));
    CU(ctx, ctx->d_sm_next.reserve(4 * static_cast<size_t>(L)));
    // (host vectors live in the context: the copies are asynchronous)
    CU(ctx, cudaMemcpyAsync(ctx->d_sm_items.p, items.data(), 8 * items.size(), cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, cudaMemcpyAsync(ctx->d_sm_off.p, off.data(), 4 * off.size(), cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, cudaMemsetAsync(ctx->d_sm_next.p, 0, 4 * static_cast<size_t>(L), ctx->stream));
    a.sm_items = ctx->d_sm_items.as<int64_t>();
    a.sm_off = ctx->d_sm_off.as<int32_t>();
    a.sm_next = ctx->d_sm_next.as<unsigned>();
    a.n_lists = L;
  }
  if (prune) {
    // bounds are indexed by global pair (every replica of a candidate)
    const size_t nb = 4 * static_cast<size_t>(total);
    CU(ctx, ctx->d_pair_fail.reserve(nb));
    CU(ctx, ctx->d_pair_ok.reserve(nb));
    CU(ctx, cudaMemsetAsync(ctx->d_pair_ok.p, 0, nb, ctx->stream));
    CU(ctx, ctx->d_best_key.reserve(8));
    CU(ctx, cudaMemsetAsync(ctx->d_pair_fail.p, 0, nb, ctx->stream));
    CU(ctx, cudaMemsetAsync(ctx->d_best_key.p, 0, 8, ctx->stream));
    a.best_key = ctx->d_best_key.as<unsigned long long>();
    a.pair_fail = ctx->d_pair_fail.as<int32_t>();
    a.pair_ok = ctx->d_pair_ok.as<int32_t>();
    a.cand_invalid = ctx->d_cand_inv.as<int8_t>();
    // A shard of a larger search (replicas staged on other GPUs) bounds
    // candidates by the sessions of the WHOLE search (set_global_sessions):
    // the local staged total would prune a candidate that merely loses on
    // this GPU's replicas.
    a.total_sessions = ctx->global_sessions > 0 ? ctx->global_sessions : ctx->total_sessions;
  }
  int64_t launches = 0;
  ProfileLease lease(ctx);  // held until this search's stream synchronisation
  CU(ctx, lease.acquire());
  CU(ctx, cudaEventRecord(ctx->ev[1], ctx->stream));
  if (n > 0) {
    // The diagnostics build (per-phase clock64 counters) is a separate
    // instantiation so the product kernel carries no instrumentation. Each
    // layout's kernels live in their own translation unit (replay_l*.cu).
    pdg::ReplayKernel kern = pdg::replay_kernel_for(ctx->layout, variant);
    if (tp) kern = reinterpret_cast<pdg::ReplayKernel>(pdg_tp::replay_kernel_for(ctx->layout, variant));
    ctx->last_build = tp ? PDSIM_BUILD_THROUGHPUT : PDSIM_BUILD_LATENCY;
    CU(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ctx->smem_bytes)));
    kern<<<static_cast<unsigned>(slots), 32, ctx->smem_bytes, ctx->stream>>>(a);
    ++launches;
    CU(ctx, cudaGetLastError());
  }
  CU(ctx, cudaEventRecord(ctx->ev[2], ctx->stream));
  if (ctx->comm) {
    // The one collective of a sharded search: per-candidate
    // counts summed and flags max-reduced over every GPU's shard, in place,
    // on this search's stream; the argmax below then sees the whole search.
    flags_for_max_kernel<<<1, 256, 0, ctx->stream>>>(ctx->d_cand_bad.as<int>(), C);
    ++launches;
    CU(ctx, cudaGetLastError());
    const pdg::NcclApi& nc = pdg::nccl();
    ncclResult_t r = nc.GroupStart();
    if (r == ncclSuccess) {
      r = nc.AllReduce(ctx->d_cand_sum.p, ctx->d_cand_sum.p, static_cast<size_t>(C), ncclUint64, ncclSum, ctx->comm,
                       ctx->stream);
    }
    if (r == ncclSuccess) {
      r = nc.AllReduce(ctx->d_cand_bad.p, ctx->d_cand_bad.p, static_cast<size_t>(C), ncclInt32, ncclMax, ctx->comm,
                       ctx->stream);
    }
    const ncclResult_t r2 = nc.GroupEnd();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) return set_err(ctx, PDSIM_ERR_CUDA, "ncclAllReduce: " + pdg::nccl_error(r));
  }
  argmax_kernel<<<1, 256, 0, ctx->stream>>>(ctx->d_cand_sum.as<unsigned long long>(), ctx->d_cand_bad.as<int>(), C,
                                          ctx->d_best.as<unsigned long long>());
  ++launches;
  CU(ctx, cudaGetLastError());
  CU(ctx, cudaEventRecord(ctx->ev[3], ctx->stream));

  // D2H
  std::vector<pdg::PairResult> res(static_cast<size_t>(n));
  std::vector<unsigned long long> csum(static_cast<size_t>(C));
  std::vector<int> cbad(static_cast<size_t>(C));
  unsigned long long best = 0;
  if (n > 0) {
    CU(ctx, cudaMemcpyAsync(res.data(), ctx->d_results.p, sizeof(pdg::PairResult) * static_cast<size_t>(n),
                            cudaMemcpyDeviceToHost, ctx->stream));
  }
  CU(ctx, cudaMemcpyAsync(csum.data(), ctx->d_cand_sum.p, 8 * static_cast<size_t>(C), cudaMemcpyDeviceToHost,
                          ctx->stream));
  CU(ctx, cudaMemcpyAsync(cbad.data(), ctx->d_cand_bad.p, 4 * static_cast<size_t>(C), cudaMemcpyDeviceToHost,
                          ctx->stream));
  CU(ctx, cudaMemcpyAsync(&best, ctx->d_best.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (report && n > 0) {
    CU(ctx, cudaMemcpyAsync(out->pair_report, ctx->d_reports.p, sizeof(pdsim_report) * static_cast<size_t>(n),
                            cudaMemcpyDeviceToHost, ctx->stream));
  }
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  float k_ms = 0, d_ms = 0;
  CU(ctx, cudaEventElapsedTime(&k_ms, ctx->ev[1], ctx->ev[2]));
  CU(ctx, cudaEventElapsedTime(&d_ms, ctx->ev[0], ctx->ev[3]));

  bool engine_error = false;
  for (int j = 0; j < PDSIM_PROF_BUCKETS; ++j) ctx->prof_cycles[j] = ctx->prof_count[j] = 0;
  ctx->attempts2 = 0;
  for (const auto& r : res) {
    engine_error |= r.status == PDSIM_PAIR_ERROR;
    ctx->attempts2 += r.attempts > 1 ? 1 : 0;
    for (int j = 0; j < PDSIM_PROF_BUCKETS; ++j) {
      ctx->prof_cycles[j] += r.prof_cycles[j];
      ctx->prof_count[j] += r.prof_count[j];
    }
  }
  if (out) {
    for (int64_t k = 0; k < n; ++k) {
      if (out->pair_attainment) out->pair_attainment[k] = res[static_cast<size_t>(k)].att;
      if (out->pair_counters) out->pair_counters[k] = res[static_cast<size_t>(k)].ctr;
      if (out->pair_status) out->pair_status[k] = static_cast<int8_t>(res[static_cast<size_t>(k)].status);
      if (out->pair_events) out->pair_events[k] = res[static_cast<size_t>(k)].events;
      if (out->pair_cycles) out->pair_cycles[k] = res[static_cast<size_t>(k)].cycles;
    }
    if (out->candidate_slo_ok) {
      for (int c = 0; c < C; ++c) {
        out->candidate_slo_ok[c] = (cbad[c] & 1) ? -1 : (cbad[c] & 2) ? -2 : static_cast<int64_t>(csum[c]);
      }
    }
    out->best_candidate = best ? static_cast<int32_t>(0xffffffffull - (best & 0xffffffffull)) : -1;
    out->best_slo_ok = best ? static_cast<int64_t>((best >> 32) - 1) : -1;
    out->kernel_ms = k_ms;
    out->device_ms = d_ms;
    out->kernel_launches = launches;
    out->d2h_bytes = static_cast<int64_t>(sizeof(pdg::PairResult) * static_cast<size_t>(n) + 12 * C + 8);
  }
  if (single_result && n == 1) *single_result = res[0];
  if (engine_error) {
    return set_err(ctx, PDSIM_ERR_INTERNAL, "engine capacity or invariant violated in at least one pair");
  }
  return PDSIM_OK;
}

// Surrogate-planner phase sims (planner.cuh) for jobs (trace, degree index).
int phase_impl(pdsim_gpu_ctx* ctx, const std::vector<const pdsim_trace*>& traces, const std::vector<int>& trace_of,
               const std::vector<int>& deg_idx, const pdsim_profile& profile, std::vector<pdg::PhaseOut>* out) {
  pdg::HostError err;
  if (!pdg::validate_profile(profile, &err)) return set_err(ctx, err.code, err.msg);
  const size_t nt = traces.size(), nj = trace_of.size();
  std::vector<pdg::PackedTrace> packed(nt);
  int32_t max_r = 1, max_s = 1;
  int64_t max_tok = 1;
  size_t total = 0;
  std::vector<pdg::HostError> perr(nt);
  std::vector<char> pok(nt, 1);
  pdg::parallel_for(nt, [&](size_t k) { pok[k] = pdg::pack_trace(*traces[k], &packed[k], &perr[k]) ? 1 : 0; });
  for (size_t k = 0; k < nt; ++k) {
    if (!pok[k]) return set_err(ctx, perr[k].code, perr[k].msg);
    max_r = std::max(max_r, packed[k].R);
    max_s = std::max(max_s, packed[k].S);
    max_tok = std::max(max_tok, packed[k].total_decode);
    total += pdg::align_up(packed[k].arrival.size() * 8 + 256) + pdg::align_up(packed[k].round_off.size() * 4 + 256) +
             pdg::align_up(packed[k].incr.size() * 4 + 256) * 2 + pdg::align_up(packed[k].delay.size() * 8 + 256);
  }
  CU(ctx, ctx->d_ph_data.reserve(std::max<size_t>(total, 256)));
  std::vector<char> host(std::max<size_t>(total, 256));
  std::vector<pdg::PhaseTrace> pt(nt);
  size_t off = 0;
  char* dbase = ctx->d_ph_data.as<char>();
  auto put = [&](const void* src, size_t bytes) -> void* {
    void* dst = dbase + off;
    if (bytes) memcpy(host.data() + off, src, bytes);
    off = pdg::align_up(off + bytes + 1);
    return dst;
  };
  for (size_t k = 0; k < nt; ++k) {
    const pdg::PackedTrace& t = packed[k];
    pt[k].S = t.S;
    pt[k].R = t.R;
    pt[k].total_decode = t.total_decode;
    pt[k].arrival = static_cast<const double*>(put(t.arrival.data(), t.arrival.size() * 8));
    pt[k].round_off = static_cast<const int32_t*>(put(t.round_off.data(), t.round_off.size() * 4));
    pt[k].incr = static_cast<const int32_t*>(put(t.incr.data(), t.incr.size() * 4));
    pt[k].dec = static_cast<const int32_t*>(put(t.dec.data(), t.dec.size() * 4));
    pt[k].delay = static_cast<const double*>(put(t.delay.data(), t.delay.size() * 8));
  }
  std::vector<pdg::PhaseJob> jobs(nj);
  for (size_t j = 0; j < nj; ++j) {
    jobs[j].trace = trace_of[j];
    jobs[j].deg = deg_idx[j];
  }
  int32_t sort_cap = 1;
  while (sort_cap < max_r) sort_cap <<= 1;
  const size_t per_cta = pdg::phase_scratch_bytes(sort_cap, max_tok, max_s);
  // Up to 8 resident 256-thread CTAs per SM; each job is a serial event loop
  // with CTA-wide reductions, so occupancy hides the barrier latency.
  int threads = pdg::kPhaseThreads, per_sm = 8;
  if (const char* v = getenv("PDSIM_PHASE_THREADS")) threads = atoi(v);      // tuning only
  if (const char* v = getenv("PDSIM_PHASE_CTAS_PER_SM")) per_sm = atoi(v);  // tuning only
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(nj), per_sm * ctx->sm_count));
  CU(ctx, ctx->d_ph_traces.reserve(sizeof(pdg::PhaseTrace) * nt));
  CU(ctx, ctx->d_ph_jobs.reserve(sizeof(pdg::PhaseJob) * std::max<size_t>(nj, 1)));
  CU(ctx, ctx->d_ph_out.reserve(sizeof(pdg::PhaseOut) * std::max<size_t>(nj, 1)));
  CU(ctx, ctx->d_ph_scratch.reserve(per_cta * static_cast<size_t>(ctas)));
  CU(ctx, ctx->d_ph_counter.reserve(8));
  CU(ctx, ctx->d_ph_profile.reserve(sizeof(pdsim_profile)));
  CU(ctx, cudaMemcpyAsync(ctx->d_ph_data.p, host.data(), off, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMemcpyAsync(ctx->d_ph_traces.p, pt.data(), sizeof(pdg::PhaseTrace) * nt, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMemcpyAsync(ctx->d_ph_jobs.p, jobs.data(), sizeof(pdg::PhaseJob) * nj, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMemcpyAsync(ctx->d_ph_profile.p, &profile, sizeof(pdsim_profile), cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMemsetAsync(ctx->d_ph_counter.p, 0, 8, ctx->stream));
  CU(ctx, cudaMemsetAsync(ctx->d_ph_out.p, 0, sizeof(pdg::PhaseOut) * nj, ctx->stream));
  pdg::PhaseArgs a;
  a.traces = ctx->d_ph_traces.as<pdg::PhaseTrace>();
  a.jobs = ctx->d_ph_jobs.as<pdg::PhaseJob>();
  a.n_jobs = static_cast<int32_t>(nj);
  a.sort_cap = sort_cap;
  a.max_s = max_s;
  a.run_cap = max_tok;
  a.scratch = ctx->d_ph_scratch.as<char>();
  a.scratch_bytes = per_cta;
  a.next_job = ctx->d_ph_counter.as<unsigned long long>();
  a.out = ctx->d_ph_out.as<pdg::PhaseOut>();
  a.profile = ctx->d_ph_profile.as<pdsim_profile>();
  if (nj > 0) {
    pdg::phase_sim_kernel<<<static_cast<unsigned>(ctas), static_cast<unsigned>(threads), 0, ctx->stream>>>(a);
    CU(ctx, cudaGetLastError());
  }
  out->assign(nj, pdg::PhaseOut());
  CU(ctx, cudaMemcpyAsync(out->data(), ctx->d_ph_out.p, sizeof(pdg::PhaseOut) * nj, cudaMemcpyDeviceToHost, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  for (const auto& o : *out) {
    if (o.pre_status == PDSIM_ERR_INTERNAL || o.dec_status == PDSIM_ERR_INTERNAL) {
      return set_err(ctx, PDSIM_ERR_INTERNAL, "phase sim: scratch capacity violated");
    }
  }
  return PDSIM_OK;
}

const char* phase_error_text(int which) {
  return which == 0 ? "planner: reference trace has no prefill tasks"
         : which == 1 ? "planner: reference trace has no sessions"
                      : "planner: reference trace produced no inter-token samples";
}

}  // namespace

extern "C" {

int pdsim_abi_version(void) { return PDSIM_ABI_VERSION; }

const char* pdsim_last_error(void) { return g_last_error.c_str(); }

int pdsim_gpu_create(int device, pdsim_gpu_ctx** out) {
  if (!out) return set_err(nullptr, PDSIM_ERR_CONFIG, "null output pointer");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    return set_err(nullptr, PDSIM_ERR_CUDA,
                   std::string("no CUDA device available (the replay engine has no CPU path): ") +
                       (e != cudaSuccess ? cudaGetErrorString(e) : "device count 0"));
  }
  if (device < 0 || device >= n) return set_err(nullptr, PDSIM_ERR_CUDA, "device index out of range");
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return set_err(nullptr, PDSIM_ERR_CUDA, cudaGetErrorString(e));
  if (prop.major != 10) {
    return set_err(nullptr, PDSIM_ERR_CUDA,
                   "device " + std::to_string(device) + " is sm_" + std::to_string(prop.major) +
                       std::to_string(prop.minor) + "; this build targets sm_100a only");
  }
  std::unique_ptr<pdsim_gpu_ctx> ctx(new pdsim_gpu_ctx());
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  CU(ctx.get(), cudaSetDevice(device));
  CU(ctx.get(), cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
  ctx->stream = ctx->own_stream;
  for (auto& ev : ctx->ev) CU(ctx.get(), cudaEventCreate(&ev));
  *out = ctx.release();
  return PDSIM_OK;
}

void pdsim_gpu_destroy(pdsim_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) pdg::nccl().CommDestroy(ctx->comm);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

const char* pdsim_gpu_last_error(const pdsim_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

int pdsim_gpu_set_stream(pdsim_gpu_ctx* ctx, void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return PDSIM_OK;
}

int pdsim_gpu_set_search_mode(pdsim_gpu_ctx* ctx, int mode) {
  if (int rc = check_ctx(ctx)) return rc;
  if (mode != PDSIM_SEARCH_FULL && mode != PDSIM_SEARCH_ARGMAX) return set_err(ctx, PDSIM_ERR_CONFIG, "unknown search mode");
  ctx->search_mode = mode;
  return PDSIM_OK;
}

int pdsim_gpu_set_kernel_build(pdsim_gpu_ctx* ctx, int build) {
  if (int rc = check_ctx(ctx)) return rc;
  if (build != PDSIM_BUILD_AUTO && build != PDSIM_BUILD_LATENCY && build != PDSIM_BUILD_THROUGHPUT) {
    return set_err(ctx, PDSIM_ERR_CONFIG, "unknown kernel build");
  }
  ctx->kernel_build = build;
  return PDSIM_OK;
}

int pdsim_gpu_last_kernel_build(const pdsim_gpu_ctx* ctx) { return ctx ? ctx->last_build : 0; }

int pdsim_gpu_set_profiling(pdsim_gpu_ctx* ctx, int enable) {
  if (int rc = check_ctx(ctx)) return rc;
  ctx->profiling = enable ? 1 : 0;
  return PDSIM_OK;
}

int pdsim_gpu_profile_counters(const pdsim_gpu_ctx* ctx, int64_t* cycles, int64_t* counts, int64_t* replayed) {
  if (!ctx) return set_err(nullptr, PDSIM_ERR_CONFIG, "null context");
  for (int j = 0; j < PDSIM_PROF_BUCKETS; ++j) {
    if (cycles) cycles[j] = ctx->prof_cycles[j];
    if (counts) counts[j] = ctx->prof_count[j];
  }
  if (replayed) *replayed = ctx->attempts2;
  return PDSIM_OK;
}

int pdsim_gpu_stage(pdsim_gpu_ctx* ctx, const pdsim_search_input* in, const pdsim_profile* profile,
                    const pdsim_sched_params* params) {
  if (int rc = check_ctx(ctx)) return rc;
  return stage_impl(ctx, in, profile, params, nullptr);
}

int pdsim_gpu_search_staged(pdsim_gpu_ctx* ctx, int64_t pair_begin, int64_t pair_end, uint64_t seed,
                            pdsim_search_output* out) {
  if (int rc = check_ctx(ctx)) return rc;
  pdg::Records rec{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  const int rc = search_impl(ctx, pair_begin, pair_end, seed, out, rec, nullptr);
  if (out && rc == PDSIM_OK) out->h2d_bytes = 0;
  return rc;
}

int pdsim_gpu_plan_search(pdsim_gpu_ctx* ctx, const pdsim_search_input* in, const pdsim_profile* profile,
                          const pdsim_sched_params* params, uint64_t seed, pdsim_search_output* out) {
  if (int rc = check_ctx(ctx)) return rc;
  int64_t h2d = 0;
  if (int rc = stage_impl(ctx, in, profile, params, &h2d)) return rc;
  pdg::Records rec{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  const int rc = search_impl(ctx, in->pair_begin, in->pair_end, seed, out, rec, nullptr);
  if (out) out->h2d_bytes = h2d;
  return rc;
}

int pdsim_gpu_search_staged_list(pdsim_gpu_ctx* ctx, const int64_t* pairs, int64_t n_pairs, uint64_t seed,
                                 pdsim_search_output* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!pairs && n_pairs > 0) return set_err(ctx, PDSIM_ERR_CONFIG, "search: null pair list");
  static const int64_t kNone = 0;
  pdg::Records rec{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  const int rc = search_impl(ctx, 0, 0, seed, out, rec, nullptr, pairs ? pairs : &kNone, n_pairs);
  if (out && rc == PDSIM_OK) out->h2d_bytes = 8 * n_pairs;
  return rc;
}

int pdsim_gpu_set_global_sessions(pdsim_gpu_ctx* ctx, int64_t total_sessions) {
  if (int rc = check_ctx(ctx)) return rc;
  if (total_sessions < 0 || total_sessions >= static_cast<int64_t>(0xfffffffeLL)) {
    return set_err(ctx, PDSIM_ERR_CONFIG, "search: global session total out of range");
  }
  ctx->global_sessions = total_sessions;
  return PDSIM_OK;
}

int64_t pdsim_shard_pairs(int32_t n_traces, const int64_t* trace_rounds, int32_t n_candidates,
                          const pdsim_plan* candidates, int32_t world, int32_t rank, int64_t* out,
                          int64_t capacity) {
  if (n_traces < 0 || n_candidates < 0 || (n_traces > 0 && !trace_rounds) || (n_candidates > 0 && !candidates) ||
      world < 1 || rank < 0 || rank >= world) {
    set_err(nullptr, PDSIM_ERR_CONFIG, "shard_pairs: bad arguments");
    return -1;
  }
  const std::vector<int64_t> mine = pdg::shard_pairs(n_traces, trace_rounds, n_candidates, candidates, world, rank);
  if (out) {
    for (size_t k = 0; k < mine.size() && static_cast<int64_t>(k) < capacity; ++k) out[k] = mine[k];
  }
  return static_cast<int64_t>(mine.size());
}

int pdsim_nccl_unique_id(uint8_t id[128]) {
  const pdg::NcclApi& nc = pdg::nccl();
  if (!nc.error.empty()) return set_err(nullptr, PDSIM_ERR_CUDA, nc.error);
  ncclUniqueId u;
  const ncclResult_t r = nc.GetUniqueId(&u);
  if (r != ncclSuccess) return set_err(nullptr, PDSIM_ERR_CUDA, "ncclGetUniqueId: " + pdg::nccl_error(r));
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  memcpy(id, &u, sizeof(u));
  return PDSIM_OK;
}

int pdsim_gpu_comm_init(pdsim_gpu_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[128]) {
  if (int rc = check_ctx(ctx)) return rc;
  if (world < 1 || rank < 0 || rank >= world || !id) return set_err(ctx, PDSIM_ERR_CONFIG, "comm_init: bad arguments");
  const pdg::NcclApi& nc = pdg::nccl();
  if (!nc.error.empty()) return set_err(ctx, PDSIM_ERR_CUDA, nc.error);
  if (ctx->comm) {
    nc.CommDestroy(ctx->comm);
    ctx->comm = nullptr;
  }
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  const ncclResult_t r = nc.CommInitRank(&ctx->comm, world, u, rank);
  if (r != ncclSuccess) {
    ctx->comm = nullptr;
    return set_err(ctx, PDSIM_ERR_CUDA, "ncclCommInitRank: " + pdg::nccl_error(r));
  }
  ctx->comm_world = world;
  ctx->comm_rank = rank;
  return PDSIM_OK;
}

int pdsim_multi_plan_search(int32_t n_devices, const int32_t* devices, const pdsim_search_input* in,
                            const pdsim_profile* profile, const pdsim_sched_params* params, uint64_t seed,
                            int32_t search_mode, pdsim_search_output* out) {
  if (n_devices < 1 || !devices || !in || !profile || !params) {
    return set_err(nullptr, PDSIM_ERR_CONFIG, "multi_plan_search: bad arguments");
  }
  if (in->n_traces < 1 || in->n_candidates < 1 || !in->traces || !in->candidates) {
    return set_err(nullptr, PDSIM_ERR_CONFIG, "search: need at least one trace and one candidate");
  }
  const int64_t total = static_cast<int64_t>(in->n_traces) * in->n_candidates;
  if (in->pair_begin != 0 || (in->pair_end >= 0 && in->pair_end != total)) {
    return set_err(nullptr, PDSIM_ERR_CONFIG, "multi_plan_search: shards the whole search (pair range must be all)");
  }
  const pdg::NcclApi& nc = pdg::nccl();
  if (!nc.error.empty()) return set_err(nullptr, PDSIM_ERR_CUDA, nc.error);
  std::vector<pdsim_gpu_ctx*> ctxs(static_cast<size_t>(n_devices), nullptr);
  auto cleanup = [&]() {
    for (auto* c : ctxs) pdsim_gpu_destroy(c);
  };
  for (int32_t k = 0; k < n_devices; ++k) {
    if (int rc = pdsim_gpu_create(devices[k], &ctxs[static_cast<size_t>(k)])) {
      cleanup();
      return rc;
    }
  }
  std::vector<ncclComm_t> comms(static_cast<size_t>(n_devices), nullptr);
  const ncclResult_t r = nc.CommInitAll(comms.data(), n_devices, devices);
  if (r != ncclSuccess) {
    cleanup();
    return set_err(nullptr, PDSIM_ERR_CUDA, "ncclCommInitAll: " + pdg::nccl_error(r));
  }
  std::vector<int64_t> rounds(static_cast<size_t>(in->n_traces));
  int64_t sessions = 0;
  for (int32_t t = 0; t < in->n_traces; ++t) {
    rounds[static_cast<size_t>(t)] = in->traces[t].n_rounds;
    sessions += in->traces[t].n_sessions;
  }
  const int C = in->n_candidates;
  std::vector<std::vector<int64_t>> lists(static_cast<size_t>(n_devices));
  std::vector<int> rcs(static_cast<size_t>(n_devices), PDSIM_OK);
  std::vector<pdsim_search_output> outs(static_cast<size_t>(n_devices));
  std::vector<std::vector<pdsim_attainment>> att(static_cast<size_t>(n_devices));
  std::vector<std::vector<pdsim_counters>> ctr(static_cast<size_t>(n_devices));
  std::vector<std::vector<int8_t>> st(static_cast<size_t>(n_devices));
  std::vector<std::vector<int64_t>> ev(static_cast<size_t>(n_devices)), cy(static_cast<size_t>(n_devices));
  std::vector<std::vector<int64_t>> cand(static_cast<size_t>(n_devices), std::vector<int64_t>(static_cast<size_t>(C)));
  std::vector<int64_t> h2d(static_cast<size_t>(n_devices), 0);
  std::vector<std::thread> th;
  for (int32_t k = 0; k < n_devices; ++k) {
    th.emplace_back([&, k]() {
      const size_t K = static_cast<size_t>(k);
      pdsim_gpu_ctx* c = ctxs[K];
      c->comm = comms[K];
      c->comm_world = n_devices;
      c->comm_rank = k;
      lists[K] = pdg::shard_pairs(in->n_traces, rounds.data(), C, in->candidates, n_devices, k);
      const size_t m = std::max<size_t>(lists[K].size(), 1);
      att[K].resize(m);
      ctr[K].resize(m);
      st[K].resize(m);
      ev[K].resize(m);
      cy[K].resize(m);
      pdsim_search_output& o = outs[K];
      memset(&o, 0, sizeof(o));
      o.pair_attainment = att[K].data();
      o.pair_counters = ctr[K].data();
      o.pair_status = st[K].data();
      o.pair_events = ev[K].data();
      o.pair_cycles = cy[K].data();
      o.candidate_slo_ok = cand[K].data();
      int rc = check_ctx(c);
      if (rc == PDSIM_OK) rc = stage_impl(c, in, profile, params, &h2d[K]);
      if (rc == PDSIM_OK) rc = pdsim_gpu_set_global_sessions(c, sessions);
      if (rc == PDSIM_OK) rc = pdsim_gpu_set_search_mode(c, search_mode);
      pdg::Records rec{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
      static const int64_t kNone = 0;
      // every rank reaches the collective inside search_impl, even with an
      // empty shard; a rank that failed before it would hang the others,
      // so staging errors are validated identically on every rank first.
      if (rc == PDSIM_OK) {
        rc = search_impl(c, 0, 0, seed, &o, rec, nullptr, lists[K].empty() ? &kNone : lists[K].data(),
                         static_cast<int64_t>(lists[K].size()));
      }
      rcs[K] = rc;
    });
  }
  for (auto& t : th) t.join();
  int rc = PDSIM_OK;
  std::string msg;
  for (int32_t k = 0; k < n_devices && rc == PDSIM_OK; ++k) {
    if (rcs[static_cast<size_t>(k)] != PDSIM_OK) {
      rc = rcs[static_cast<size_t>(k)];
      msg = ctxs[static_cast<size_t>(k)]->err;
    }
  }
  if (rc == PDSIM_OK && out) {
    const pdsim_search_output& o0 = outs[0];
    double kms = 0, dms = 0;
    int64_t launches = 0, d2h = 0, h2d_all = 0;
    for (int32_t k = 0; k < n_devices; ++k) {
      const size_t K = static_cast<size_t>(k);
      for (size_t j = 0; j < lists[K].size(); ++j) {
        const int64_t p = lists[K][j];
        if (out->pair_attainment) out->pair_attainment[p] = att[K][j];
        if (out->pair_counters) out->pair_counters[p] = ctr[K][j];
        if (out->pair_status) out->pair_status[p] = st[K][j];
        if (out->pair_events) out->pair_events[p] = ev[K][j];
        if (out->pair_cycles) out->pair_cycles[p] = cy[K][j];
      }
      kms = std::max(kms, outs[K].kernel_ms);
      dms = std::max(dms, outs[K].device_ms);
      launches += outs[K].kernel_launches;
      d2h += outs[K].d2h_bytes;
      h2d_all += h2d[K];
    }
    if (out->candidate_slo_ok) memcpy(out->candidate_slo_ok, cand[0].data(), 8 * static_cast<size_t>(C));
    out->best_candidate = o0.best_candidate;
    out->best_slo_ok = o0.best_slo_ok;
    out->kernel_ms = kms;
    out->device_ms = dms;
    out->kernel_launches = launches;
    out->d2h_bytes = d2h;
    out->h2d_bytes = h2d_all;
  }
  cleanup();  // destroys the communicators with the contexts
  if (rc != PDSIM_OK) return set_err(nullptr, rc, msg);
  return PDSIM_OK;
}

int pdsim_gpu_sweep(pdsim_gpu_ctx* ctx, int32_t n_traces, const pdsim_trace* traces, const pdsim_plan* plan,
                    int32_t n_settings, const pdsim_sched_params* settings, const pdsim_profile* profile,
                    uint64_t seed, pdsim_search_output* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!plan || !settings || n_settings < 1) return set_err(ctx, PDSIM_ERR_CONFIG, "sweep: need a plan and at least one setting");
  // Candidates are the settings, all on the one plan: pair k * n_traces + r.
  std::vector<pdsim_plan> plans(static_cast<size_t>(n_settings), *plan);
  pdsim_search_input in;
  memset(&in, 0, sizeof(in));
  in.n_traces = n_traces;
  in.n_candidates = n_settings;
  in.traces = traces;
  in.candidates = plans.data();
  in.pair_begin = 0;
  in.pair_end = -1;
  int64_t h2d = 0;
  if (int rc = stage_impl(ctx, &in, profile, &settings[0], &h2d, settings)) return rc;
  // The reference sweep replays rate-major (pdsim.cpp:547-586) and run()'s
  // precheck throws at the first trace with an oversized first round; the
  // plan is the same for every setting, so that trace fails them all.
  for (int32_t r = 0; r < n_traces; ++r) {
    if (ctx->pair_invalid[static_cast<size_t>(r)]) {
      ctx->staged = false;
      const int64_t i = pdg::precheck_violator(ctx->packed[static_cast<size_t>(r)], ctx->plans[0], ctx->profile);
      return set_err(ctx, PDSIM_ERR_CONFIG, pdg::precheck_message(ctx->packed[static_cast<size_t>(r)], i));
    }
  }
  pdg::Records rec{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  const int rc = search_impl(ctx, 0, -1, seed, out, rec, nullptr);
  // The settings stay staged: pdsim_gpu_search_staged() re-runs the sweep
  // with inputs resident; the next stage()/run() replaces them.
  if (out) out->h2d_bytes = h2d;
  return rc;
}

int pdsim_gpu_run(pdsim_gpu_ctx* ctx, const pdsim_trace* trace, const pdsim_plan* plan,
                  const pdsim_profile* profile, const pdsim_sched_params* params, uint64_t seed,
                  pdsim_run_output* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!trace || !plan || !out) return set_err(ctx, PDSIM_ERR_CONFIG, "null argument");
  pdsim_search_input in;
  memset(&in, 0, sizeof(in));
  in.n_traces = 1;
  in.n_candidates = 1;
  in.traces = trace;
  in.candidates = plan;
  in.pair_begin = 0;
  in.pair_end = 1;
  if (int rc = stage_impl(ctx, &in, profile, params, nullptr)) return rc;
  if (ctx->pair_invalid[0]) {
    const int64_t i = pdg::precheck_violator(ctx->packed[0], ctx->plans[0], ctx->profile);
    return set_err(ctx, PDSIM_ERR_CONFIG, pdg::precheck_message(ctx->packed[0], i));
  }
  const pdg::PackedTrace& t = ctx->packed[0];
  pdg::Records rec{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  const size_t R = static_cast<size_t>(std::max(t.R, 1)), S = static_cast<size_t>(std::max(t.S, 1));
  if (out->decisions) {
    CU(ctx, ctx->d_dec.reserve(sizeof(pdsim_decision) * R));
    rec.decisions = ctx->d_dec.as<pdsim_decision>();
  }
  if (out->ttft_samples) {
    CU(ctx, ctx->d_ttft.reserve(sizeof(pdsim_ttft_sample) * R));
    rec.ttft = ctx->d_ttft.as<pdsim_ttft_sample>();
  }
  if (out->sessions) {
    CU(ctx, ctx->d_sess.reserve(sizeof(pdsim_session_outcome) * S));
    rec.sessions = ctx->d_sess.as<pdsim_session_outcome>();
  }
  if (out->itl_samples) {  // materialised ITL samples: step log + round spans
    const size_t cap = static_cast<size_t>(std::max<int64_t>(t.total_decode, 1));
    CU(ctx, ctx->d_steps.reserve(sizeof(pdg::StepRec) * cap));
    CU(ctx, ctx->d_spans.reserve(sizeof(pdg::SpanRec) * R));
    rec.steps = ctx->d_steps.as<pdg::StepRec>();
    rec.spans = ctx->d_spans.as<pdg::SpanRec>();
    rec.steps_cap = static_cast<int64_t>(cap);
  }
  pdg::PairResult res;
  memset(&res, 0, sizeof(res));
  if (int rc = search_impl(ctx, 0, 1, seed, nullptr, rec, &res)) return rc;
  out->n_decisions = res.n_decisions;
  out->n_ttft = res.n_ttft;
  out->n_sessions = res.att.sessions_completed;
  out->counters = res.ctr;
  out->attainment = res.att;
  if (out->decisions && res.n_decisions > 0) {
    CU(ctx, cudaMemcpyAsync(out->decisions, rec.decisions, sizeof(pdsim_decision) * res.n_decisions,
                            cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (out->ttft_samples && res.n_ttft > 0) {
    CU(ctx, cudaMemcpyAsync(out->ttft_samples, rec.ttft, sizeof(pdsim_ttft_sample) * res.n_ttft,
                            cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (out->sessions && out->n_sessions > 0) {
    CU(ctx, cudaMemcpyAsync(out->sessions, rec.sessions, sizeof(pdsim_session_outcome) * out->n_sessions,
                            cudaMemcpyDeviceToHost, ctx->stream));
  }
  out->n_itl = 0;
  std::vector<pdg::StepRec> steps;
  std::vector<pdg::SpanRec> spans;
  if (out->itl_samples) {
    if (res.n_steps > rec.steps_cap) return set_err(ctx, PDSIM_ERR_INTERNAL, "run: step log capacity exceeded");
    steps.resize(static_cast<size_t>(res.n_steps));
    spans.resize(static_cast<size_t>(res.n_spans));
    if (res.n_steps > 0) {
      CU(ctx, cudaMemcpyAsync(steps.data(), rec.steps, sizeof(pdg::StepRec) * steps.size(), cudaMemcpyDeviceToHost,
                              ctx->stream));
    }
    if (res.n_spans > 0) {
      CU(ctx, cudaMemcpyAsync(spans.data(), rec.spans, sizeof(pdg::SpanRec) * spans.size(), cudaMemcpyDeviceToHost,
                              ctx->stream));
    }
  }
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  if (out->sessions) pdg::sort_outcomes(out->sessions, out->n_sessions);
  if (out->itl_samples) {
    out->n_itl = pdg::expand_itl(steps.data(), res.n_steps, spans.data(), res.n_spans, t,
                                 ctx->plans[0].D, out->itl_samples, out->itl_capacity);
  }
  return PDSIM_OK;
}

int pdsim_gpu_phase_sims(pdsim_gpu_ctx* ctx, int32_t n_jobs, const pdsim_trace* traces, const int32_t* degrees,
                         const pdsim_profile* profile, pdsim_phase_result* prefill, pdsim_phase_result* decode) {
  if (int rc = check_ctx(ctx)) return rc;
  if (n_jobs < 0 || (n_jobs > 0 && (!traces || !degrees)) || !profile) {
    return set_err(ctx, PDSIM_ERR_CONFIG, "phase_sims: bad arguments");
  }
  std::vector<const pdsim_trace*> tv;
  std::vector<int> trace_of, deg_idx;
  for (int32_t j = 0; j < n_jobs; ++j) {
    const int di = pdg::degree_index(*profile, degrees[j]);
    if (di < 0) return set_err(ctx, PDSIM_ERR_DOMAIN, "t_prefill: unknown degree " + std::to_string(degrees[j]));
    tv.push_back(&traces[j]);
    trace_of.push_back(j);
    deg_idx.push_back(di);
  }
  std::vector<pdg::PhaseOut> out;
  if (int rc = phase_impl(ctx, tv, trace_of, deg_idx, *profile, &out)) return rc;
  for (int32_t j = 0; j < n_jobs; ++j) {
    const pdg::PhaseOut& o = out[static_cast<size_t>(j)];
    if (prefill) prefill[j] = pdsim_phase_result{o.pre_p95, o.pre_samples, o.pre_infeasible, o.pre_status};
    if (decode) decode[j] = pdsim_phase_result{o.dec_p95, o.dec_samples, o.dec_infeasible, o.dec_status};
  }
  return PDSIM_OK;
}

int pdsim_gpu_estimate_coefficients(pdsim_gpu_ctx* ctx, const pdsim_trace_stats* stats, int32_t n_sets,
                                    const double* rates, const uint64_t* seeds, const pdsim_profile* profile,
                                    const int32_t* degrees, int32_t n_degrees, int32_t total_gpus,
                                    pdsim_coefficients* out, int32_t* set_status) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!stats || !profile || !out || n_sets < 0 || (n_sets > 0 && (!rates || !seeds))) {
    return set_err(ctx, PDSIM_ERR_CONFIG, "estimate_coefficients: bad arguments");
  }
  // Argument checks in the reference order (planner.cpp:232-249).
  if (total_gpus < 1) return set_err(ctx, PDSIM_ERR_CONFIG, "planner: total_gpus must be >= 1");
  if (!degrees || n_degrees < 1) return set_err(ctx, PDSIM_ERR_CONFIG, "planner: degree set is empty");
  std::vector<int> ts(degrees, degrees + n_degrees);
  std::sort(ts.begin(), ts.end());
  ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
  if (ts.size() > PDSIM_MAX_DEGREES) return set_err(ctx, PDSIM_ERR_CONFIG, "planner: too many degrees");
  std::vector<int> di(ts.size());
  for (size_t k = 0; k < ts.size(); ++k) {
    di[k] = pdg::degree_index(*profile, ts[k]);
    if (di[k] < 0) return set_err(ctx, PDSIM_ERR_CONFIG, "planner: degree " + std::to_string(ts[k]) + " not covered by profile");
  }
  // Reference-load traces on the host RNG (workload.cpp:170-229).
  const size_t nd = ts.size();
  std::vector<pdsim_trace_buf*> bufs(static_cast<size_t>(n_sets) * nd, nullptr);
  std::vector<pdsim_trace> views(bufs.size());
  std::vector<int> status(static_cast<size_t>(n_sets), PDSIM_OK);
  std::vector<std::string> msgs(static_cast<size_t>(n_sets));
  std::vector<const pdsim_trace*> tv;
  std::vector<int> trace_of, deg_idx, job_slot;
  for (int32_t s = 0; s < n_sets; ++s) {
    if (!(rates[s] > 0.0)) {
      status[static_cast<size_t>(s)] = PDSIM_ERR_CONFIG;
      msgs[static_cast<size_t>(s)] = "planner: arrival rate must be > 0";
    }
  }
  // Host generation (libm-bound, must stay on the CPU) on all host threads.
  std::vector<int> gen_rc(bufs.size(), PDSIM_OK);
  std::vector<std::string> gen_msg(bufs.size());
  pdg::parallel_for(bufs.size(), [&](size_t slot) {
    const size_t s = slot / nd, k = slot % nd;
    if (status[s] != PDSIM_OK) return;
    const double share = rates[s] * static_cast<double>(ts[k]) / static_cast<double>(total_gpus);
    const uint64_t seed = seeds[s] + 0x9E3779B97F4A7C15ull * static_cast<uint64_t>(ts[k]);
    pdsim_trace_buf* b = nullptr;
    gen_rc[slot] = pdsim_gen_trace(stats, share, 256, seed, &b);  // kCoefficientSessions (planner.cpp:33)
    if (gen_rc[slot] != PDSIM_OK) {
      gen_msg[slot] = pdsim_last_error();
      return;
    }
    bufs[slot] = b;
    pdsim_trace_buf_view(b, &views[slot]);
  });
  for (size_t slot = 0; slot < bufs.size(); ++slot) {  // first failing degree of each set, in order
    const size_t s = slot / nd;
    if (status[s] == PDSIM_OK && gen_rc[slot] != PDSIM_OK) {
      status[s] = gen_rc[slot];
      msgs[s] = gen_msg[slot];
    }
  }
  for (size_t slot = 0; slot < bufs.size(); ++slot) {
    if (!bufs[slot] || status[slot / nd] != PDSIM_OK) continue;
    trace_of.push_back(static_cast<int>(tv.size()));
    tv.push_back(&views[slot]);
    deg_idx.push_back(di[slot % nd]);
    job_slot.push_back(static_cast<int>(slot));
  }
  std::vector<pdg::PhaseOut> po;
  const int rc = phase_impl(ctx, tv, trace_of, deg_idx, *profile, &po);
  for (auto* b : bufs) pdsim_trace_buf_free(b);
  if (rc) return rc;
  for (int32_t s = 0; s < n_sets; ++s) {
    pdsim_coefficients& c = out[s];
    memset(&c, 0, sizeof(c));
    c.n_degrees = static_cast<int32_t>(nd);
    for (size_t k = 0; k < nd; ++k) c.degrees[k] = ts[k];
  }
  for (size_t j = 0; j < po.size(); ++j) {
    const size_t slot = static_cast<size_t>(job_slot[j]), s = slot / nd, k = slot % nd;
    const pdg::PhaseOut& o = po[j];
    if (status[s] != PDSIM_OK) continue;
    // The reference runs degrees in ascending order and throws at the first
    // failing sim (prefill before decode).
    if (o.pre_status != PDSIM_OK || o.dec_status != PDSIM_OK) {
      status[s] = PDSIM_ERR_CONFIG;
      msgs[s] = phase_error_text(o.pre_status != PDSIM_OK ? 0 : 2);
      continue;
    }
    pdsim_coefficients& c = out[s];
    c.infeasible_pre[k] = static_cast<int8_t>(o.pre_infeasible);
    c.infeasible_dec[k] = static_cast<int8_t>(o.dec_infeasible);
    c.tau_pre[k] = o.pre_infeasible ? 0.0 : o.pre_p95;
    c.tau_dec[k] = o.dec_infeasible ? 0.0 : o.dec_p95;
  }
  for (int32_t s = 0; s < n_sets; ++s) {
    if (set_status) set_status[s] = status[static_cast<size_t>(s)];
    if (status[static_cast<size_t>(s)] != PDSIM_OK && !msgs[static_cast<size_t>(s)].empty()) {
      ctx->err = msgs[static_cast<size_t>(s)];
    }
  }
  return PDSIM_OK;
}

}  // extern "C"
