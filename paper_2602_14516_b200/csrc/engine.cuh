// engine.cuh — the replay of one (candidate plan, trace replica) pair by one
// warp.
//
// Behavioural restatement, for B200, of the reference discrete-event engine
// (proj/src/sim_engine.cpp:107-632) and of the routing
// (proj/src/coordinator.cpp:27-171) and reordering (proj/src/reorder.cpp:44-146)
// policies it calls. Every observable — routing decisions, TTFT samples,
// session verdicts, counters — is reproduced bit-for-bit. The data layout is
// re-designed for the GPU:
//
//  * Warp-uniform execution. All 32 lanes run the event loop in lock-step on
//    identical scalar state (kept in registers); lanes split only where the
//    work is parallel: the next-event reduction, window trimming (ballot),
//    the reorder permutation search, routing estimates, the RNG twist.
//    Shared/global stores of warp-uniform state are issued by lane 0 between
//    __syncwarp()s.
//  * Worker events (decode step / local prefill done, prefill compute done,
//    history read) live in registers: slot s is owned by lane s % 32; the next
//    event is a 5-step shuffle min over (time, kind<<58 | seq<<6 | slot).
//    Only session events (interaction done, write-back) use a binary heap, in
//    shared memory with a global-memory spill area.
//  * Arrivals are read in trace order and merged (kind 0 wins ties).
//  * A task is identified by its session (at most one task in flight each).
//    The admission queue is the index range [adm_head, next_arrival).
//  * Decode batches are never materialised: a member finishes its round at
//    step join + decode_len - 1, so a per-worker min-heap keyed by
//    (end_step, session-id rank) yields the finishing cohort members in cohort
//    order; per-session ITL sums are folded at round end from a ring of step
//    end times (every ITL gap of a step is now - previous step end).
//  * Windowed statistics are lazily trimmed rings with exact 128-bit prefix
//    sums, so `mean <= threshold` is decided in O(1) (exactsum.cuh); the
//    sequential fold (fold.cuh for ITL runs) runs only inside the error band.
//
// The same source compiles for the GPU (the product; PDG_NL = 32 lanes) and,
// in tests only, for the host (PDG_NL = 1) so the logic can be checked against
// the reference without a device.
#pragma once

#include <math.h>

#include "common.cuh"
#include "exactsum.cuh"
#include "fold.cuh"

namespace pdg {

#if defined(__CUDA_ARCH__)
#define PDG_NL 32
#else
#define PDG_NL 1
#endif

// Address-space hints. Engine state lives in shared memory and the workspace
// in global memory, but the pointers to them are stored in (shared) engine
// state, which makes them generic; generic loads are tracked on the long
// scoreboard and pay an extra address-space check. The hints let ptxas emit
// LDS/LDG instead.
#if defined(__CUDACC__)
extern __shared__ __align__(16) char pdg_smem[];
#endif
#if defined(__CUDA_ARCH__)
template <class T>
__device__ __forceinline__ T* SHP(T* p) {
  __builtin_assume(__isShared(p));
  return p;
}
template <class T>
__device__ __forceinline__ T* GLP(T* p) {
  __builtin_assume(__isGlobal(p));
  return p;
}
#else
template <class T>
inline T* SHP(T* p) {
  return p;
}
template <class T>
inline T* GLP(T* p) {
  return p;
}
#endif

// Shared-or-inlined hot subroutines (I-cache footprint): a
// routine inlined at several call sites occupies instruction-cache lines once
// per copy; a PDG_SHARE_<NAME> build keeps one out-of-line copy instead.
#if defined(PDG_SHARE_SEG_APPEND) || defined(PDG_SHARE_ALL)
#define PDG_A_SEG_APPEND PDG_COLD
#else
#define PDG_A_SEG_APPEND PDG_HD
#endif
#if defined(PDG_SHARE_CATCH_UP_WORKER) || defined(PDG_SHARE_ALL)
#define PDG_A_CATCH_UP_WORKER PDG_COLD
#else
#define PDG_A_CATCH_UP_WORKER PDG_HD
#endif
#if defined(PDG_SHARE_TRY_STAGE) || defined(PDG_SHARE_ALL)
#define PDG_A_TRY_STAGE PDG_COLD
#else
#define PDG_A_TRY_STAGE PDG_HD
#endif
#if defined(PDG_SHARE_COMPLETE_TASK) || defined(PDG_SHARE_ALL)
#define PDG_A_COMPLETE_TASK PDG_COLD
#else
#define PDG_A_COMPLETE_TASK PDG_HD
#endif
#if defined(PDG_SHARE_HEAP_PUSH) || defined(PDG_SHARE_ALL)
#define PDG_A_HEAP_PUSH PDG_COLD
#else
#define PDG_A_HEAP_PUSH PDG_HD
#endif
#if defined(PDG_SHARE_SELECT_NEXT) || defined(PDG_SHARE_ALL)
#define PDG_A_SELECT_NEXT PDG_COLD
#else
#define PDG_A_SELECT_NEXT PDG_HD
#endif
#if defined(PDG_SHARE_FH_PUSH) || defined(PDG_SHARE_ALL)
#define PDG_A_FH_PUSH PDG_COLD
#else
#define PDG_A_FH_PUSH PDG_HD
#endif
#if defined(PDG_SHARE_FH_POP) || defined(PDG_SHARE_ALL)
#define PDG_A_FH_POP PDG_COLD
#else
#define PDG_A_FH_POP PDG_HD
#endif
#if defined(PDG_SHARE_ADVANCE_DECODE) || defined(PDG_SHARE_ALL)
#define PDG_A_ADVANCE_DECODE PDG_COLD
#else
#define PDG_A_ADVANCE_DECODE PDG_HD
#endif
#if defined(PDG_SHARE_START_ROUND) || defined(PDG_SHARE_ALL)
#define PDG_A_START_ROUND PDG_COLD
#else
#define PDG_A_START_ROUND PDG_HD
#endif
#if defined(PDG_SHARE_TTFT_HAS_SLACK) || defined(PDG_SHARE_ALL)
#define PDG_A_TTFT_HAS_SLACK PDG_COLD
#else
#define PDG_A_TTFT_HAS_SLACK PDG_HD
#endif

// Route slack scan on the device: 0 sequential (worker by worker, warp-
// collective trims; the latency build), 1 all workers in parallel (lane per
// worker; the throughput build, Makefile), 2 the first worker alone, then
// the rest in parallel. Same decisions in every mode (tests/test_gpu_random.py
// runs both builds); A/B on one B200 (profiles/round2/ab_route_fh_v14.log):
// mode 1 -2 % on C3s/C5, +2 % on C2.
#ifndef PDG_ROUTE_SCAN
#define PDG_ROUTE_SCAN 0
#endif
// Finisher heap arity (2 or 32; 32 measured neutral, the binary heap kept).
#ifndef PDG_FH_ARITY
#define PDG_FH_ARITY 2
#endif

// Branch hints for the rare paths (capacity failures, lazy-mode aborts,
// exact-fold fallbacks): keeps them off the fall-through path of the hot
// code (instruction fetch).
#define PDG_UNLIKELY(x) __builtin_expect(!!(x), 0)
#define PDG_LIKELY(x) __builtin_expect(!!(x), 1)

constexpr int kMaxSlots = 64;
constexpr int32_t kSmallHeap = 64;
constexpr int32_t kShortBulk = 16;  // silent stretches up to this long are stepped with plain fp64 adds  // session events kept unordered (lanes scan them) up to this count
constexpr int kSlotsPerLane = kMaxSlots / PDG_NL;
constexpr double kInf = __builtin_huge_val();

PDG_HD int lane_id() {
#if defined(__CUDA_ARCH__)
  return static_cast<int>(threadIdx.x & 31u);
#else
  return 0;
#endif
}
PDG_HD void warp_sync() {
#if defined(__CUDA_ARCH__)
  __syncwarp();
#endif
}
PDG_HD uint64_t shfl_xor_u64(uint64_t v, int m) {
#if defined(__CUDA_ARCH__)
  return __shfl_xor_sync(0xffffffffu, static_cast<unsigned long long>(v), m);
#else
  (void)m;
  return v;
#endif
}
PDG_HD uint64_t shfl_u64(uint64_t v, int src) {
#if defined(__CUDA_ARCH__)
  return __shfl_sync(0xffffffffu, static_cast<unsigned long long>(v), src);
#else
  (void)src;
  return v;
#endif
}
PDG_HD double shfl_d(double v, int src) {
#if defined(__CUDA_ARCH__)
  return __shfl_sync(0xffffffffu, v, src);
#else
  (void)src;
  return v;
#endif
}
PDG_HD int shfl_i(int v, int src) {
#if defined(__CUDA_ARCH__)
  return __shfl_sync(0xffffffffu, v, src);
#else
  (void)src;
  return v;
#endif
}
PDG_HD uint32_t ballot(bool p) {
#if defined(__CUDA_ARCH__)
  return __ballot_sync(0xffffffffu, p);
#else
  return p ? 1u : 0u;
#endif
}
PDG_HD int popc(uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __popc(b);
#else
  return __builtin_popcount(b);
#endif
}
PDG_HD int first_zero(uint32_t bits) {  // index of the lowest clear bit (32 if none)
  if (bits == 0xffffffffu) return 32;
#if defined(__CUDA_ARCH__)
  return __ffs(~bits) - 1;
#else
  return __builtin_ctz(~bits);
#endif
}
PDG_HD double warp_min(double v) {
  for (int m = PDG_NL / 2; m > 0; m >>= 1) {
    const double o = bitsd(shfl_xor_u64(dbits(v), m));
    if (o < v) v = o;
  }
  return v;
}

enum EventKind : uint32_t {
  kArrival = 0,
  kInteractionDone = 1,
  kKvTransferDone = 2,
  kPrefillDone = 3,
  kDecodeStep = 4,
};

// Event order key (sim_engine.cpp:68-74): time first, then kind, then the
// scheduling sequence number; the slot id rides in the low bits (never
// decisive because seq is unique).
PDG_HD uint64_t mk_key(uint32_t kind, uint64_t seq, uint32_t slot) {
  return (static_cast<uint64_t>(kind) << 58) | (seq << 6) | slot;
}
PDG_HD bool before(double ta, uint64_t ka, double tb, uint64_t kb) { return ta < tb || (ta == tb && ka < kb); }

// Session event (interaction done: a = session; write-back: a = session, b = prefill worker).
struct HEv {
  double t;
  uint64_t key;
  uint32_t a;
  uint32_t b;
};

// Trace records, one 128-bit load each (workload.hpp:28-39 re-laid for the
// device). Per session: arrival time, offset of its first round, rank of its
// id among all ids. Per round: the Round's three fields.
struct alignas(16) SessTr {
  double arrival;
  int32_t round_off;
  int32_t rank;
};
struct alignas(16) RoundTr {
  int32_t incr;
  int32_t dec;
  double delay;
};
static_assert(sizeof(SessTr) == 16 && sizeof(RoundTr) == 16, "trace records are one 128-bit load");

// Session-table length: S + 1 entries (entry S holds the round count as its
// round_off, so session i's rounds are [ss[i].round_off, ss[i+1].round_off)).
PDG_HD int64_t sess_table_len(int64_t S) { return S + 1; }

// Packed read-only trace (one per replica, shared by all candidates).
struct DevTrace {
  int32_t S;
  int32_t R;
  int32_t max_dec;
  int32_t rank_is_index;     // by_rank[k] == k for every k (generated traces): skip the lookup
  double ttft_thres;
  double itl_thres;
  const SessTr* ss;          // [sess_table_len(S)]; entry S: round_off = R
  const RoundTr* rr;         // [R]
  const int64_t* sid;        // [S]
  const int32_t* by_rank;    // [S] session of each id rank
};

// Worker layout of a candidate (sim_engine.cpp:175-203): prefill workers
// 0..P-1 then decode workers P..P+D-1, each with its profile degree index.
struct DevPlan {
  int32_t P;
  int32_t D;
  int8_t pdeg[PDSIM_MAX_WORKERS];
  int8_t ddeg[PDSIM_MAX_WORKERS];
};

struct DevParams {
  int32_t routing;
  int32_t reorder;
  int32_t window;
  int32_t reserved;
  double alpha;
  double beta;
  double stat_window;
};

// Per-session runtime state (SessionRt + the one PrefillTask in flight),
// split by access frequency. SessRt is what every mode touches on every
// event of the session: 64 B, so one record is half a 128-byte line and two
// 32-byte sectors (the throughput configs keep millions of these in DRAM,
// profiles/traffic_C3.json). SessCold holds what only the exact engine and
// the record outputs read.
struct alignas(64) SessRt {
  double itl_lo;     // search mode: bracket [itl_lo, itl_hi] of the exact sum of this
  double itl_hi;     //   session's ITL samples (directed rounding)
  double t_enq;      // enqueue time of the current task (== created for r >= 2)
  double e_join;     // lazy search mode: end time of step `join` (stamped when it starts)
  int32_t itl_cnt;
  int32_t next_pend; // lazy search mode: next session waiting for its round's first step
  int32_t join;      // step index at which the current round joined the batch
  int32_t ctx;       // context_len
  int32_t roff;      // index of its first round in the round table (cached at admission)
  int16_t round;     // 1-based current round
  int16_t nround;    // the session's round count (cached at admission)
  int8_t bound;      // decode worker index
  int8_t postpone;   // PrefillTask::postpone_count
  int8_t ttft_bad;   // some TTFT > threshold
  int8_t reserved;
  int32_t reserved2;
};
static_assert(sizeof(SessRt) == 64, "SessRt layout");
struct SessCold {
  double itl_sum;    // exact mode: sequential fold of this session's ITL samples
  double bind_time;  // admission time (records)
  int32_t seg_hint;  // exact mode: bound worker's open-segment index when the round joined
  int32_t reserved;
};
static_assert(sizeof(SessCold) == 24, "SessCold layout");

// A worker's task queue (global ring) + exact sum of the queued costs.
struct TaskQueue {
  ExactSum sum;
  uint32_t qh, qt;
  uint32_t reserved[2];
};

// Lazily trimmed window ring (global storage) + running prefix at the tail.
// Bracket [lo, hi] of an exact running sum (directed rounding).
struct Brk {
  double lo;
  double hi;
};

// Lazily trimmed window ring (global storage) + running prefix at the tail.
struct WinState {
  Brk tail;  // prefix bracket after the newest sample
  uint32_t head, end;
  uint32_t reserved[2];
};

struct PrefillW {  // shared memory
  TaskQueue q;
  WinState tw;  // TTFT window
  int32_t deg;
  int32_t cur, stg;
  int8_t computing, staged, pending, reserved;
  double cur_cost, stg_cost;
  double staged_ready;
};

// A run of consecutive decode steps of one worker with the same ITL gap and
// the same ITL sample count per step: step j (first <= j < first + n) ends
// at t0 + (j - first) * gap exactly (each step adds exactly `gap`).
struct Seg {
  double plo;     // bracket [plo, phi] of the exact ITL-sample sum over every
  double phi;     //   step before this segment (directed rounding)
  int64_t pterms; // ITL samples before this segment
  double t0;     // end time of step `first`
  double gap;    // every step's ITL gap (end - previous end)
  int32_t first; // first step index
  int32_t n;     // steps
  uint32_t cnt;  // ITL samples per step after the first (cohort members past their first token)
  uint32_t cnt_first;  // ITL samples of step `first` (differs from cnt when a run starts with joiners)
};

struct DecodeW {  // shared memory
  TaskQueue q;  // local prefill queue
  Seg sg;       // the open (newest) segment of the step log
  int64_t kv_used;
  int64_t kv_cap;
  uint64_t fh_top;     // cached finisher-heap minimum (valid when fh_n > 0)
  double cur_cost;
  double last_step_t;  // end time of the previous step
  double cur_end;      // end time of the step in flight (valid while stepping)
  int32_t run_b;       // lazy mode: the in-flight run's next explicit step index
  int32_t run_pad;
  double dur;          // cached t_decode(dur_cohort)
  int32_t dur_cohort;
  int32_t deg;
  int32_t cur;
  int32_t batch_n, n_new, cohort_n, first_n;
  int32_t steps;  // steps started
  int32_t fh_n;   // finisher-heap size
  int8_t stepping, prefilling, reserved[2];
  // closed segments live in the global ring [seg_keep, seg_end); the open
  // segment has index seg_end. ITL window head: segment seg_head with its
  // first seg_off steps expired.
  int32_t seg_end;
  int32_t seg_keep;
  int32_t seg_head;
  int32_t seg_off;
  int32_t pend_head;  // lazy search mode: sessions whose round starts with the next step
  int32_t pend_pad;
};

// Capacities (host-computed provable upper bounds, see pack.hpp).
struct Caps {
  int32_t S;      // sessions
  int32_t hcap;   // session-event heap (global spill capacity)
  int32_t hs;     // session-event heap entries kept in shared memory
  int32_t qcap;   // per-worker task queue (power of 2)
  int32_t fcap;   // per-decode-worker finisher heap
  int32_t twcap;  // TTFT window ring (power of 2)
  int32_t segcap;  // per-decode-worker step-segment ring (power of 2)
  int32_t maxdec;  // longest decode round (steps a per-session fold may reach back)
  int32_t pmax;
  int32_t dmax;
  int32_t pres;    // PrefillW / DecodeW entries reserved in shared memory (>= pmax, dmax);
  int32_t dres;    // the device engine addresses them at compile-time offsets (EngineT<.., kD, kP>)
  int32_t rep_r;      // report mode: TTFT value slots (max rounds); 0 = no report
  int32_t rep_gapcap; // report mode: ITL gap histogram entries (power of two)
};

struct EngState;

// Shared-memory part of a workspace slot.
struct SmemSlot {
  EngState* es;
  PrefillW* pw;
  DecodeW* dw;
  uint64_t* mt;    // 312 words
  HEv* heap;       // [hs]
  int32_t* order;  // [kMaxSlots] routing scan order scratch
};

// Global-memory part of a workspace slot.
struct GlobalSlot {
  SessRt* sess;
  SessCold* sess_cold;
  HEv* heap;  // spill area [hcap]
  int32_t* pq_s;
  double* pq_c;
  int32_t* dq_s;
  double* dq_c;
  double* tw_t;
  double* tw_v;
  Brk* tw_p;  // prefix bracket before each TTFT sample
  Seg* seg;  // [dmax][segcap]
  uint64_t* fh;
  double* rep_ttft;    // report mode: [rep_r] TTFT values in push order (incremental negated)
  double* rep_e2e;     // report mode: [S] e2e latency by session-id rank (NaN = not completed)
  uint64_t* rep_gkey;  // report mode: ITL gap histogram keys (value bits, 0 = empty)
  int64_t* rep_gcnt;   //   and sample counts
  unsigned long long* rep_hist;  // report mode: [256] radix-select digit histogram
};

PDG_HD size_t align_up(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }
PDG_HD size_t align16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

constexpr size_t kEngStateBytes = 2560;  // >= sizeof(EngState), checked below

// Shared-memory layout of a slot: EngState, DecodeW[dres], PrefillW[pres],
// the mt19937_64 state, the routing-order scratch, then the session-event
// heap (the only variable-size part, last). smem_off() gives the same offsets
// as compile-time constants for the device engine.
PDG_HD constexpr size_t smem_a16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }
struct SmemOff {
  size_t dw, pw, mt, order, heap;
};
PDG_HD constexpr SmemOff smem_off(size_t dres, size_t pres) {
  return SmemOff{smem_a16(kEngStateBytes),
                 smem_a16(kEngStateBytes) + smem_a16(sizeof(DecodeW) * dres),
                 smem_a16(kEngStateBytes) + smem_a16(sizeof(DecodeW) * dres) + smem_a16(sizeof(PrefillW) * pres),
                 smem_a16(kEngStateBytes) + smem_a16(sizeof(DecodeW) * dres) + smem_a16(sizeof(PrefillW) * pres) +
                     smem_a16(8 * 312),
                 smem_a16(kEngStateBytes) + smem_a16(sizeof(DecodeW) * dres) + smem_a16(sizeof(PrefillW) * pres) +
                     smem_a16(8 * 312) + smem_a16(4 * kMaxSlots)};
}

PDG_HD size_t smem_slot_bytes(const Caps& c, SmemSlot* s, char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + off : nullptr;
    off = align16(off + bytes);
    return p;
  };
  SmemSlot t;
  t.es = reinterpret_cast<EngState*>(take(kEngStateBytes));
  t.dw = reinterpret_cast<DecodeW*>(take(sizeof(DecodeW) * static_cast<size_t>(c.dres)));
  t.pw = reinterpret_cast<PrefillW*>(take(sizeof(PrefillW) * static_cast<size_t>(c.pres)));
  t.mt = reinterpret_cast<uint64_t*>(take(8 * 312));
  t.order = reinterpret_cast<int32_t*>(take(4 * kMaxSlots));
  t.heap = reinterpret_cast<HEv*>(take(sizeof(HEv) * static_cast<size_t>(c.hs)));
  if (s) *s = t;
  return off;
}

PDG_HD size_t global_slot_bytes(const Caps& c, GlobalSlot* s, char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + off : nullptr;
    off = align_up(off + bytes);
    return p;
  };
  const size_t P = static_cast<size_t>(c.pmax > 0 ? c.pmax : 1), D = static_cast<size_t>(c.dmax);
  GlobalSlot t;
  t.sess = reinterpret_cast<SessRt*>(take(sizeof(SessRt) * static_cast<size_t>(c.S)));
  t.sess_cold = reinterpret_cast<SessCold*>(take(sizeof(SessCold) * static_cast<size_t>(c.S)));
  t.heap = reinterpret_cast<HEv*>(take(sizeof(HEv) * static_cast<size_t>(c.hcap)));
  t.pq_s = reinterpret_cast<int32_t*>(take(4 * P * static_cast<size_t>(c.qcap)));
  t.pq_c = reinterpret_cast<double*>(take(8 * P * static_cast<size_t>(c.qcap)));
  t.dq_s = reinterpret_cast<int32_t*>(take(4 * D * static_cast<size_t>(c.qcap)));
  t.dq_c = reinterpret_cast<double*>(take(8 * D * static_cast<size_t>(c.qcap)));
  t.tw_t = reinterpret_cast<double*>(take(8 * P * static_cast<size_t>(c.twcap)));
  t.tw_v = reinterpret_cast<double*>(take(8 * P * static_cast<size_t>(c.twcap)));
  t.tw_p = reinterpret_cast<Brk*>(take(sizeof(Brk) * P * static_cast<size_t>(c.twcap)));
  t.seg = reinterpret_cast<Seg*>(take(sizeof(Seg) * D * static_cast<size_t>(c.segcap)));
  t.fh = reinterpret_cast<uint64_t*>(take(8 * D * static_cast<size_t>(c.fcap)));
  const bool rep = c.rep_gapcap > 0;
  t.rep_ttft = reinterpret_cast<double*>(take(rep ? 8 * static_cast<size_t>(c.rep_r) : 0));
  t.rep_e2e = reinterpret_cast<double*>(take(rep ? 8 * static_cast<size_t>(c.S) : 0));
  t.rep_gkey = reinterpret_cast<uint64_t*>(take(rep ? 8 * static_cast<size_t>(c.rep_gapcap) : 0));
  t.rep_gcnt = reinterpret_cast<int64_t*>(take(rep ? 8 * static_cast<size_t>(c.rep_gapcap) : 0));
  t.rep_hist = reinterpret_cast<unsigned long long*>(take(rep ? 8 * 256 : 0));
  if (s) *s = t;
  return off;
}

// Optional per-pair record outputs (drop-in SimResult vectors).
// ITL materialisation (records mode): decode steps in event order and the
// step interval of every decoded round; the host expands them into the
// reference's per-token ItlSample stream (pack.hpp expand_itl).
struct StepRec {
  double t;    // step end time
  double gap;  // the step's ITL value (end - previous step end)
  int32_t d;   // decode worker
  int32_t k;   // step index on that worker
};
struct SpanRec {
  int32_t sess;   // session index
  int32_t round;  // 1-based
  int32_t d;      // decode worker
  int32_t join;   // step of the round's first token
  int32_t end;    // step of its last token
  int32_t reserved;
};

struct Records {
  pdsim_decision* decisions;        // [R]
  pdsim_ttft_sample* ttft;          // [R]
  pdsim_session_outcome* sessions;  // [S], termination order
  StepRec* steps;                   // [steps_cap] (optional: ITL materialisation)
  SpanRec* spans;                   // [R]
  int64_t steps_cap;
};

// Exact argmax pruning (search mode), shared by the pairs of
// one launch. A candidate c is dead once its upper bound (total sessions over
// its replicas minus sessions already known to miss the SLO) is below the
// incumbent's lower bound (slo_ok summed over its completed replicas), or
// equal to it with c after the incumbent in enumeration order: c can then
// never be the argmax (max count, ties to the smallest index).
struct Prune {
  unsigned long long* best;  // incumbent key ((lb + 1) << 32) | (0xffffffff - c); 0 = none; null = off
  int32_t* pair_fail;        // [pairs of the launch] failures seen per pair (max over attempts)
  int32_t* pair_ok;          // [pairs of the launch] sessions attaining the SLO so far (max over attempts)
  int* cand_bad;             // [C] bit 1 = pruned (bit 0 = invalid)
  int64_t total_sessions;    // sum of S over all replicas
  int64_t self;              // this pair's index in pair_fail
  int64_t fail_base;         // index of (c, replica 0) in pair_fail (may be negative)
  int32_t c;                 // this pair's candidate
  int32_t r_lo, r_hi;        // replicas of c inside the launch
  int32_t c_invalid;         // some pair of c is invalid: c never becomes the incumbent
};

PDG_HD bool prune_dominated(int64_t ub, unsigned long long key, int32_t c) {
  if (key == 0) return false;
  const int64_t lb = static_cast<int64_t>(key >> 32) - 1;
  const int32_t cs = static_cast<int32_t>(0xffffffffull - (key & 0xffffffffull));
  if (cs == c) return false;
  return ub < lb || (ub == lb && c > cs);
}

struct PairResult {
  pdsim_attainment att;
  pdsim_counters ctr;
  int64_t n_decisions;
  int64_t n_ttft;
  int64_t n_steps;      // ITL materialisation records written
  int64_t n_spans;
  int64_t events;       // dynamic events processed (diagnostics)
  int64_t cycles;       // device clock64() ticks for this pair (0 on host)
  int64_t exact_folds;  // certified comparisons that fell back to a fold
  int32_t status;       // PDSIM_PAIR_*
  int32_t attempts;     // 1, or 2 when the lazy/search-mode attempt was replayed exactly
  int64_t prof_cycles[PDSIM_PROF_BUCKETS];  // optional per-phase SM cycles (kProf*), 0 unless profiling
  int64_t prof_count[PDSIM_PROF_BUCKETS];
};

// Per-phase instrumentation buckets (enabled by KernelArgs::profile).
enum ProfBucket { kProfSelect = 0, kProfArrival, kProfInteraction, kProfWriteback, kProfDecodeStep,
                  kProfLocalPrefill, kProfPrefillDone, kProfHistory,
                  // inclusive sub-scopes
                  kProfRoute, kProfEnqueue, kProfCatchUp, kProfFinisher, kProfAdvance, kProfComplete,
                  kProfHeap, kProfDequeue };

PDG_HD int64_t pdg_clock() {
#if defined(__CUDA_ARCH__)
  return clock64();
#else
  return 0;
#endif
}

struct RouteOut {
  int32_t local;
  int32_t p;
  int32_t rationale;
  int32_t has_est;
  double est;
};

// k-th (0-based) lexicographic permutation of 0..m-1 (factorial number system).
PDG_HD void unrank_perm(int64_t k, int m, int* perm) {
  int avail[8];
  int64_t fact[9];
  fact[0] = 1;
  for (int i = 1; i <= m; ++i) fact[i] = fact[i - 1] * i;
  for (int i = 0; i < m; ++i) avail[i] = i;
  int n = m;
  for (int i = 0; i < m; ++i) {
    const int64_t f = fact[m - 1 - i];
    const int q = static_cast<int>(k / f);
    k -= q * f;
    perm[i] = avail[q];
    for (int j = q; j + 1 < n; ++j) avail[j] = avail[j + 1];
    --n;
  }
}

// All mutable engine state of one warp-slot lives in shared memory (one
// instance per warp); the Engine object itself is a single pointer, so the
// compiler keeps nothing of it on the stack. Warp-uniform fields are written
// with the same value by every lane.
struct EngState {
  DevTrace T;
  DevPlan PL;
  DevParams PR;
  Caps C;
  SmemSlot SM;
  GlobalSlot G;
  Records REC;
  uint64_t seed_;
  double now_;
  double next_arr_t_;
  uint64_t seq_;
  int32_t next_arr_roff_;  // round offset of the next arrival
  int32_t next_arr_pad_;
  int32_t hn_;
  int32_t heap_spilled_;
  int32_t hsmall_;  // session events form an unordered set of <= kSmallHeap entries in shared memory
  int32_t next_arr_;
  int32_t adm_head_;
  int32_t rr_next_;
  uint32_t mt_idx_;
  int32_t failed_;
  int32_t nslots_;
  int32_t lazy_;   // lazy decode stepping enabled for this attempt
  int32_t profile_;
  int32_t attempts_;
  int64_t prof_c_[PDSIM_PROF_BUCKETS];
  int64_t prof_n_[PDSIM_PROF_BUCKETS];
  int32_t exact_itl_;  // per-session ITL means by sequential fold (records / retry)
  uint32_t cur_kind_;  // kind of the event being processed (catch-up tie rule)
  int32_t abort_;  // lazy attempt hit an ambiguous tie: replay exactly
  pdsim_attainment att_;
  pdsim_counters ctr_;
  int64_t n_dec_;
  int64_t n_ttft_;
  int64_t n_steps_;
  int64_t n_spans_;
  // report mode (metrics.cpp:138-190): in-order folds and counts
  double rep_init_sum_;
  double rep_incr_sum_;
  double rep_itl_sum_;
  int64_t rep_n_init_;
  int64_t rep_n_incr_;
  int64_t rep_n_local_;
  int64_t rep_n_itl_;
  int64_t events_;
  int64_t folds_;
  double st_[kMaxSlots];    // worker-event slot times (+inf when empty)
  uint64_t sk_[kMaxSlots];  // worker-event slot keys
  // argmax search mode (kPrune engines only)
  Prune PRN;
  int32_t pruned_;    // the candidate can no longer be the argmax
  int32_t fails_;     // sessions of this attempt known to miss the SLO
  int32_t prn_pub_;   // fails_ last published to Prune::pair_fail
  int32_t prn_ok_pub_;  // att_.slo_ok last published to Prune::pair_ok
  uint32_t prn_tick_;
};

#if defined(__CUDACC__)
__constant__ pdsim_profile c_profile;  // the cost model, broadcast from the constant cache
#endif
inline const pdsim_profile*& host_profile() {  // host (test) builds only
  static thread_local const pdsim_profile* p = nullptr;
  return p;
}
#if defined(__CUDA_ARCH__)
#define PDG_PROF c_profile
#else
#define PDG_PROF (*host_profile())
#endif

static_assert(sizeof(EngState) <= kEngStateBytes, "EngState outgrew its shared-memory reservation");


static_assert(kEngStateBytes % 16 == 0, "slot layout alignment");

#if defined(__CUDA_ARCH__)
#define s_ (reinterpret_cast<EngState*>(pdg_smem))
#endif

// kProf compiles in the per-phase clock64 instrumentation (diagnostics
// kernel only); the product kernel is EngineT<false>.
// kRec compiles in the record / report outputs (drop-in run(), ITL
// materialisation, per-pair reports); the attainment-only search kernel is
// built without them.
struct EngineAttach {};

// kLazy: lazy decode stepping (silent steps are not events). The exact
// engine (kLazy = false) replays a pair whose lazy attempt hit an ambiguous
// tie, and runs record modes that need every step as an event.
// kPrune: argmax search mode (Prune): failures are counted and the
// candidate is tested against the incumbent every 128 events.
template <bool kProf, int kD = 0, int kP = 0, bool kRec = true, bool kLazy = true, bool kPrune = false>
class EngineT {
  template <bool, int, int, bool, bool, bool>
  friend class EngineT;
  static constexpr SmemOff kOff = smem_off(static_cast<size_t>(kD), static_cast<size_t>(kP));

 public:
  // `es` must point at this warp's EngState (shared memory on the device).
  // On the device `es` must be the EngState at the start of the block's
  // dynamic shared memory (one warp per block): the engine addresses it
  // directly from the shared-memory base, so `this` carries no state.
  PDG_HD EngineT(EngState* es, const DevTrace& tr, const DevPlan& plan, const DevParams& prm, const Caps& caps,
                const SmemSlot& sm, const GlobalSlot& gm, Records rec, uint64_t seed, int profile = 0,
                const Prune* prn = nullptr)
#if !defined(__CUDA_ARCH__)
      : s_(es)
#endif
  {
    (void)es;
    s_->profile_ = profile;
    s_->T = tr;
    s_->PL = plan;
    s_->PR = prm;
    s_->C = caps;
    s_->SM = sm;
    s_->G = gm;
    s_->REC = rec;
    s_->seed_ = seed;
    if (prn) {
      s_->PRN = *prn;
    } else {
      memset(&s_->PRN, 0, sizeof(Prune));
    }
    s_->pruned_ = 0;
    s_->prn_pub_ = 0;
    s_->prn_ok_pub_ = 0;
    s_->prn_tick_ = 0;
    warp_sync();
  }

  PDG_HD void run(PairResult* out) {
    // Lazy decode stepping first; an ambiguous equal-time ordering between a
    // lazily advanced decode step and another decode step aborts the attempt,
    // and the pair is replayed by the exact engine with every step an event.
    // Materialised ITL samples and reports need every step as an event too.
    const bool exact_first = kRec && (s_->REC.steps || s_->C.rep_gapcap > 0);
    if (kLazy && !exact_first) {
      attempt(0);
      if (!s_->abort_ || s_->pruned_) {
        finish_result(out);
        return;
      }
    }
    EngineT<kProf, kD, kP, kRec, false, kPrune> exact{EngineAttach{}};
#if !defined(__CUDA_ARCH__)
    exact.s_ = s_;
#endif
    exact.attempt(kLazy && !exact_first ? 1 : 0);
    exact.finish_result(out);
  }

  // Attaches to an engine state already set up by the full constructor.
  PDG_HD explicit EngineT(EngineAttach) {}

  PDG_HD void attempt(int a) {
    init();
    s_->attempts_ = a + 1;
    s_->lazy_ = kLazy ? 1 : 0;
    s_->exact_itl_ = (!kLazy || (kRec && s_->REC.sessions)) ? 1 : 0;
    event_loop();
  }

  PDG_HD void event_loop() {
    const int D = s_->PL.D, P = s_->PL.P;
    const int nslots = s_->nslots_;
    constexpr bool prof = kProf;
    int64_t tp = prof ? pdg_clock() : 0;
    int bucket = -1;
    const int32_t n_sess = s_->T.S;
    while (!s_->failed_ && !s_->abort_) {
      warp_sync();  // re-converge once per event (handlers store uniform values)
      if (kPrune && ((++s_->prn_tick_ & 127u) == 0) && prune_check()) {
        s_->pruned_ = 1;
        return;
      }
      if (prof) {
        const int64_t now_c = pdg_clock();
        if (bucket >= 0) {
          s_->prof_c_[bucket] += now_c - tp;
          s_->prof_n_[bucket] += 1;
        }
        tp = now_c;
        bucket = kProfSelect;
      }
      // Arrival cursor read ahead of the slot reduction (overlaps its latency).
      const int32_t next_arr = s_->next_arr_;
      const double next_arr_t = s_->next_arr_t_;
      // Next worker event: min over the slot table (lanes split the slots).
      double bt;
      uint64_t bk;
      bool slot_tie;
      int wid;
      next_slot_event(nslots, &bt, &bk, &slot_tie, &wid);
      int src = bk == ~0ull ? -1 : (wid >= kMaxSlots ? 1 : 0);  // 0 slot, 1 session event, 2 arrival
      if (!s_->hsmall_ && s_->hn_ > 0) {
        double ht;
        uint64_t hk;
        heap_top(&ht, &hk);
        if (src < 0 || before(ht, hk, bt, bk)) {
          bt = ht;
          bk = hk;
          src = 1;
        }
      }
      // Arrivals carry kind 0 and seq = index: they precede every dynamic
      // event at an equal time (sim_engine.cpp:137-143).
      if (next_arr < n_sess && (src < 0 || next_arr_t <= bt)) src = 2;
      if (src < 0) {
        if (kLazy) catch_up(kInf, 0);  // drain silent steps (none remain)
        break;
      }
      if (src == 2) {
        const int32_t i = next_arr;
        const double t = next_arr_t;
        const int32_t roff = s_->next_arr_roff_;
        // the next cursor entry (one 128-bit load): its round offset also
        // ends session i's round range
        const SessTr nx = sess_tr(i + 1);
        s_->next_arr_ = i + 1;
        s_->next_arr_t_ = nx.arrival;
        s_->next_arr_roff_ = nx.round_off;
        s_->cur_kind_ = kArrival;
        if (prof) prof_switch(&tp, &bucket, kProfArrival);
        advance_to(t);
        on_arrival(i, roff, nx.round_off - roff);
        continue;
      }
      const uint32_t kind = static_cast<uint32_t>(bk >> 58);
      // Two decode-step events at the same time: their order is the
      // scheduling order, which lazily materialised steps do not carry.
      if (PDG_UNLIKELY(kLazy && src == 0 && kind == kDecodeStep && slot_tie)) {
        s_->abort_ = 1;
        return;
      }
      s_->cur_kind_ = kind;
      ++s_->events_;
      advance_to(bt);
      if (prof) prof_switch(&tp, &bucket, src == 1 ? (kind == kInteractionDone ? kProfInteraction : kProfWriteback)
                                           : (static_cast<int>(bk & 63u) < D ? (kind == kDecodeStep ? kProfDecodeStep : kProfLocalPrefill)
                                              : (static_cast<int>(bk & 63u) < D + P ? kProfPrefillDone : kProfHistory)));
      if (src == 1) {
        const HEv e = wid >= kMaxSlots ? heap_take(wid - kMaxSlots) : heap_pop();
        if (kind == kInteractionDone) {
          on_interaction_done(static_cast<int32_t>(e.a));
        } else {
          on_writeback(static_cast<int32_t>(e.a), static_cast<int>(e.b));
        }
        continue;
      }
      const int s = static_cast<int>(bk & 63u);
      clear_slot(s);
      if (s < D) {
        if (kind == kDecodeStep) {
          on_decode_step(s);
        } else {
          on_local_prefill_done(s);
        }
      } else if (s < D + P) {
        on_prefill_done(s - D);
      } else {
        on_history_read(s - D - P);
      }
    }
  }

  // ---- per-pair Report (metrics.cpp:108-190) ----
  // One decode step's ITL samples: cnt identical values g in push order.
  PDG_HD void report_itl_step(double g, int32_t cnt) {
    s_->rep_itl_sum_ = fold_repeat(s_->rep_itl_sum_, g, static_cast<uint64_t>(cnt));
    s_->rep_n_itl_ += cnt;
    uint64_t* keys = GLP(s_->G.rep_gkey);
    int64_t* cnts = GLP(s_->G.rep_gcnt);
    const uint64_t key = dbits(g);  // g > 0: never the empty key 0
    const uint32_t mask = static_cast<uint32_t>(s_->C.rep_gapcap - 1);
    uint32_t h = static_cast<uint32_t>((key * 0x9E3779B97F4A7C15ull) >> 32) & mask;
    bool placed = false;
    for (uint32_t probe = 0; probe <= mask; ++probe) {  // warp-uniform probe sequence
      const uint64_t k = keys[h];
      if (k == key || k == 0) {
        warp_sync();
        if (lane_id() == 0) {
          keys[h] = key;
          cnts[h] = (k == 0 ? 0 : cnts[h]) + cnt;
        }
        warp_sync();
        placed = true;
        break;
      }
      h = (h + 1) & mask;
    }
    if (PDG_UNLIKELY(!placed)) fail();  // histogram capacity exceeded: loud failure
  }

  // k-th smallest (1-based) of the keys item(i) yields for i < n (items
  // returning false are skipped), weighted: 8 radix passes over 8-bit digits.
  template <class F>
  PDG_HD uint64_t report_select(int64_t n, int64_t rank, F item) {
    unsigned long long* hist = GLP(s_->G.rep_hist);
    uint64_t prefix = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
      warp_sync();
      for (int b = lane_id(); b < 256; b += PDG_NL) hist[b] = 0;
      warp_sync();
      const uint64_t mask_hi = shift == 56 ? 0ull : (~0ull << (shift + 8));
      for (int64_t i = lane_id(); i < n; i += PDG_NL) {
        uint64_t key;
        int64_t w;
        if (!item(i, &key, &w) || (key & mask_hi) != prefix) continue;
#if defined(__CUDA_ARCH__)
        atomicAdd(&hist[(key >> shift) & 255u], static_cast<unsigned long long>(w));
#else
        hist[(key >> shift) & 255u] += static_cast<unsigned long long>(w);
#endif
      }
      warp_sync();
#if defined(__CUDA_ARCH__)
      __threadfence_block();
#endif
      int b = 0;
      for (; b < 255; ++b) {  // every lane scans the same histogram: uniform result
        const int64_t c = static_cast<int64_t>(hist[b]);
        if (rank <= c) break;
        rank -= c;
      }
      prefix |= static_cast<uint64_t>(b) << shift;
    }
    warp_sync();
    return prefix;
  }

  PDG_HD static int64_t p95_rank(int64_t n) {  // percentile_nearest_rank (metrics.cpp:125-136)
    int64_t r = static_cast<int64_t>(ceil(dmul(0.95, static_cast<double>(n))));
    return r < 1 ? 1 : r;
  }

  // build_report_from_samples (metrics.cpp:138-190) of the pair just replayed.
  PDG_HD void build_report(pdsim_report* out) {
    pdsim_report r;
    memset(&r, 0, sizeof(r));
    const int64_t completed = s_->att_.sessions_completed, nt = s_->n_ttft_, ni = s_->rep_n_itl_;
    r.sessions_total = s_->T.S;
    r.sessions_completed = completed;
    if (completed == 0 && nt == 0 && ni == 0) {
      r.empty = 1;
      *out = r;
      return;
    }
    const double* tv = GLP(s_->G.rep_ttft);
    const int64_t ntv = nt < s_->C.rep_r ? nt : s_->C.rep_r;
    for (int kind = 0; kind < 2; ++kind) {
      pdsim_metric_stat& m = kind == 0 ? r.ttft_initial : r.ttft_incremental;
      const int64_t c = kind == 0 ? s_->rep_n_init_ : s_->rep_n_incr_;
      const double sum = kind == 0 ? s_->rep_init_sum_ : s_->rep_incr_sum_;
      m.count = c;
      m.mean = c > 0 ? ddiv(sum, static_cast<double>(c)) : 0.0;
      m.p95 = c > 0 ? bitsd(report_select(ntv, p95_rank(c), [&](int64_t i, uint64_t* key, int64_t* w) {
                const uint64_t b = dbits(tv[i]);
                if ((b >> 63) != static_cast<uint64_t>(kind)) return false;
                *key = b & ~(1ull << 63);
                *w = 1;
                return true;
              }))
                    : 0.0;
    }
    if (nt > 0) r.local_fraction = ddiv(static_cast<double>(s_->rep_n_local_), static_cast<double>(nt));
    r.itl.count = ni;
    r.itl.mean = ni > 0 ? ddiv(s_->rep_itl_sum_, static_cast<double>(ni)) : 0.0;
    if (ni > 0) {
      const uint64_t* keys = GLP(s_->G.rep_gkey);
      const int64_t* cnts = GLP(s_->G.rep_gcnt);
      r.itl.p95 = bitsd(report_select(s_->C.rep_gapcap, p95_rank(ni), [&](int64_t i, uint64_t* key, int64_t* w) {
        if (keys[i] == 0) return false;
        *key = keys[i];
        *w = cnts[i];
        return true;
      }));
    }
    if (completed > 0) {
      const double denom = static_cast<double>(completed);
      r.slo_attainment = ddiv(static_cast<double>(s_->att_.slo_ok), denom);
      r.ttft_attainment = ddiv(static_cast<double>(s_->att_.ttft_ok), denom);
      r.itl_attainment = ddiv(static_cast<double>(s_->att_.itl_ok), denom);
      double sum = 0.0;  // mean_in_order over sessions sorted by id
      const double* e2e = GLP(s_->G.rep_e2e);
      for (int32_t k = 0; k < s_->T.S; ++k) {
        const double v = e2e[k];
        if (v == v) sum = dadd(sum, v);
      }
      r.e2e_mean = ddiv(sum, denom);
    }
    *out = r;
  }

  // Inclusive sub-scope timers (no code unless kProf).
  PDG_HD int64_t pb() const { return kProf ? pdg_clock() : 0; }
  PDG_HD void pe(int k, int64_t t0) {
    if (kProf) {
      s_->prof_c_[k] += pdg_clock() - t0;
      s_->prof_n_[k] += 1;
    }
  }

  PDG_HD void prof_switch(int64_t* tp, int* bucket, int next) {
    const int64_t c = pdg_clock();
    s_->prof_c_[*bucket] += c - *tp;
    s_->prof_n_[*bucket] += 1;
    *tp = c;
    *bucket = next;
  }

  // Writes this pair's result to *out (global memory on the device; lane 0
  // stores, the warp re-converges after).
  PDG_HD void finish_result(PairResult* out) {
    int64_t kv_res = s_->ctr_.kv_bytes_residual;
    for (int d = 0; d < s_->PL.D; ++d) kv_res += DW(d).kv_used;
    warp_sync();
    if (lane_id() == 0) {
      out->att = s_->att_;
      out->att.sessions_total = s_->T.S;
      out->ctr = s_->ctr_;
      out->ctr.kv_bytes_residual = kv_res;
      out->n_decisions = s_->n_dec_;
      out->n_ttft = s_->n_ttft_;
      out->n_steps = s_->n_steps_;
      out->n_spans = s_->n_spans_;
      out->events = s_->events_;
      out->exact_folds = s_->folds_;
      out->status = s_->failed_ ? PDSIM_PAIR_ERROR : s_->pruned_ ? PDSIM_PAIR_PRUNED : PDSIM_PAIR_OK;
      out->attempts = s_->attempts_;
      out->cycles = 0;
      for (int j = 0; j < PDSIM_PROF_BUCKETS; ++j) {
        out->prof_cycles[j] = kProf ? s_->prof_c_[j] : 0;
        out->prof_count[j] = kProf ? s_->prof_n_[j] : 0;
      }
    }
    warp_sync();
  }

 private:
#if !defined(__CUDA_ARCH__)
  EngState* s_;
#endif

  PDG_HD void fail() { s_->failed_ = 1; }

  // Publishes this pair's failures, then tests the candidate against the
  // incumbent (Prune). Failures seen in an aborted lazy attempt are real
  // (everything before the abort equals the exact replay), hence max().
  PDG_COLD bool prune_check() {
    const Prune& p = s_->PRN;
    const int32_t f_own = s_->fails_;
    const int32_t ok_own = static_cast<int32_t>(s_->att_.slo_ok);
#if defined(__CUDA_ARCH__)
    if (lane_id() == 0) {
      if (f_own > s_->prn_pub_) atomicMax(&p.pair_fail[p.self], f_own);
      if (ok_own > s_->prn_ok_pub_) atomicMax(&p.pair_ok[p.self], ok_own);
    }
    warp_sync();
    // Bounds of this candidate over its replicas in the launch: published
    // values are real (max over attempts); this pair's own counts join by max.
    long long f = 0, ok = 0;
    for (int32_t r = p.r_lo + lane_id(); r < p.r_hi; r += 32) {
      const int64_t j = p.fail_base + r;
      int32_t vf = *reinterpret_cast<volatile int32_t*>(&p.pair_fail[j]);
      int32_t vo = *reinterpret_cast<volatile int32_t*>(&p.pair_ok[j]);
      if (j == p.self) {
        vf = vf > f_own ? vf : f_own;
        vo = vo > ok_own ? vo : ok_own;
      }
      f += vf > 0 ? vf : 0;
      ok += vo > 0 ? vo : 0;
    }
    for (int o = 16; o > 0; o >>= 1) {
      f += __shfl_xor_sync(0xffffffffu, f, o);
      ok += __shfl_xor_sync(0xffffffffu, ok, o);
    }
    // Sessions already attaining the SLO are final: a running candidate's
    // partial count is a lower bound too (valid candidates only).
    if (!p.c_invalid && ok > 0 && lane_id() == 0) {
      atomicMax(p.best, (static_cast<unsigned long long>(ok + 1) << 32) | (0xffffffffull - static_cast<unsigned>(p.c)));
    }
    const unsigned long long key = *reinterpret_cast<volatile unsigned long long*>(p.best);
    const bool dead = (*reinterpret_cast<volatile int*>(&p.cand_bad[p.c]) & 2) ||
                      prune_dominated(p.total_sessions - f, key, p.c);
    warp_sync();
    // warp-uniform stores
    if (f_own > s_->prn_pub_) s_->prn_pub_ = f_own;
    if (ok_own > s_->prn_ok_pub_) s_->prn_ok_pub_ = ok_own;
    if (dead && lane_id() == 0) atomicOr(&p.cand_bad[p.c], 2);
    return dead;
#else
    return false;
#endif
  }

  // Slot arrays in shared memory: fixed offsets from the dynamic shared
  // memory base on the device (one LDS/STS per field, no pointer load).
#if defined(__CUDA_ARCH__)
  PDG_HD DecodeW& DW(int d) const { return reinterpret_cast<DecodeW*>(pdg_smem + kOff.dw)[d]; }
  PDG_HD PrefillW& PW(int p) const { return reinterpret_cast<PrefillW*>(pdg_smem + kOff.pw)[p]; }
  PDG_HD uint64_t* MT() const { return reinterpret_cast<uint64_t*>(pdg_smem + kOff.mt); }
  PDG_HD int32_t* ORD() const { return reinterpret_cast<int32_t*>(pdg_smem + kOff.order); }
  PDG_HD HEv* SHEAP() const { return reinterpret_cast<HEv*>(pdg_smem + kOff.heap); }
#else
  DecodeW& DW(int d) const { return s_->SM.dw[d]; }
  PrefillW& PW(int p) const { return s_->SM.pw[p]; }
  uint64_t* MT() const { return s_->SM.mt; }
  int32_t* ORD() const { return s_->SM.order; }
  HEv* SHEAP() const { return s_->SM.heap; }
#endif

  // ---- trace records (one 128-bit read-only load each) ----
  PDG_HD static SessTr ld_sess(const SessTr* p) {
#if defined(__CUDA_ARCH__)
    const int4 v = __ldg(reinterpret_cast<const int4*>(p));
    SessTr r;
    r.arrival = __hiloint2double(v.y, v.x);
    r.round_off = v.z;
    r.rank = v.w;
    return r;
#else
    return *p;
#endif
  }
  PDG_HD static RoundTr ld_round(const RoundTr* p) {
#if defined(__CUDA_ARCH__)
    const int4 v = __ldg(reinterpret_cast<const int4*>(p));
    RoundTr r;
    r.incr = v.x;
    r.dec = v.y;
    r.delay = __hiloint2double(v.w, v.z);
    return r;
#else
    return *p;
#endif
  }
  PDG_HD SessTr sess_tr(int32_t i) const { return ld_sess(GLP(s_->T.ss) + i); }
  PDG_HD RoundTr round_tr(int32_t ridx) const { return ld_round(GLP(s_->T.rr) + ridx); }
  // Round `round` (1-based) of admitted session i (its round offset is cached in SessRt).
  PDG_HD RoundTr round_of(int32_t i, int round) const { return round_tr(GLP(s_->G.sess)[i].roff + round - 1); }


  PDG_HD void advance_to(double t) {
    if (t < s_->now_) s_->ctr_.events_in_order = 0;  // sim_engine.cpp:148-150
    s_->now_ = t;
  }

  PDG_COLD void init() {
    s_->now_ = 0.0;
    s_->seq_ = static_cast<uint64_t>(s_->T.S);  // arrivals took seq 0..S-1
    s_->hn_ = 0;
    s_->heap_spilled_ = false;
    s_->hsmall_ = 1;
    s_->next_arr_ = 0;
    {
      const SessTr e0 = sess_tr(0);
      s_->next_arr_t_ = s_->T.S > 0 ? e0.arrival : 0.0;
      s_->next_arr_roff_ = e0.round_off;
    }
    s_->adm_head_ = 0;
    s_->rr_next_ = 0;
    s_->ctr_.events_in_order = 1;
    s_->nslots_ = s_->PL.D + 2 * s_->PL.P;
    s_->failed_ = 0;
    s_->abort_ = 0;
    s_->fails_ = 0;
    s_->heap_spilled_ = 0;
    s_->mt_idx_ = 0;
    s_->att_ = pdsim_attainment{};
    s_->ctr_ = pdsim_counters{};
    s_->n_dec_ = 0;
    s_->n_ttft_ = 0;
    s_->n_steps_ = 0;
    s_->n_spans_ = 0;
    s_->rep_init_sum_ = s_->rep_incr_sum_ = s_->rep_itl_sum_ = 0.0;
    s_->rep_n_init_ = s_->rep_n_incr_ = s_->rep_n_local_ = s_->rep_n_itl_ = 0;
    if (kRec && s_->C.rep_gapcap > 0) {
      for (int k = lane_id(); k < s_->T.S; k += PDG_NL) GLP(s_->G.rep_e2e)[k] = __builtin_nan("");
      for (int k = lane_id(); k < s_->C.rep_gapcap; k += PDG_NL) {
        GLP(s_->G.rep_gkey)[k] = 0;
        GLP(s_->G.rep_gcnt)[k] = 0;
      }
      warp_sync();
    }
    s_->events_ = 0;
    s_->folds_ = 0;
    s_->ctr_.events_in_order = 1;
    for (int j = 0; j < PDSIM_PROF_BUCKETS; ++j) {
      s_->prof_c_[j] = 0;
      s_->prof_n_[j] = 0;
    }
    for (int j = lane_id(); j < kMaxSlots; j += PDG_NL) {
      s_->st_[j] = kInf;
      s_->sk_[j] = ~0ull;
    }
    {  // warp-uniform stores (every lane writes the same values)
      uint32_t idx;
      mt64_seed(MT(), &idx, s_->seed_);
      for (int p = 0; p < s_->PL.P; ++p) {
        PrefillW& w = PW(p);
        w.q.sum.clear();
        w.q.qh = w.q.qt = 0;
        w.tw.tail.lo = w.tw.tail.hi = 0.0;
        w.tw.head = w.tw.end = 0;
        w.deg = s_->PL.pdeg[p];
        w.cur = w.stg = -1;
        w.computing = w.staged = w.pending = 0;
        w.cur_cost = w.stg_cost = 0.0;
        w.staged_ready = 0.0;
      }
      for (int d = 0; d < s_->PL.D; ++d) {
        DecodeW& w = DW(d);
        w.q.sum.clear();
        w.q.qh = w.q.qt = 0;
        w.sg.plo = 0.0;
        w.sg.phi = 0.0;
        w.sg.pterms = 0;
        w.sg.t0 = 0.0;
        w.sg.gap = 0.0;
        w.sg.first = 0;
        w.sg.n = 0;
        w.sg.cnt = 0;
        w.sg.cnt_first = 0;
        w.seg_end = w.seg_keep = w.seg_head = w.seg_off = 0;
        w.kv_used = 0;
        w.kv_cap = static_cast<int64_t>(PDG_PROF.degrees[s_->PL.ddeg[d]]) * PDG_PROF.gpu_memory_capacity;
        w.fh_top = 0;
        w.cur_cost = 0.0;
        w.last_step_t = 0.0;
        w.dur = 0.0;
        w.dur_cohort = -1;
        w.deg = s_->PL.ddeg[d];
        w.cur = -1;
        w.batch_n = w.n_new = w.cohort_n = w.first_n = 0;
        w.steps = 0;
        w.fh_n = 0;
        w.stepping = w.prefilling = 0;
        w.cur_end = 0.0;
        w.run_b = 0;
        w.run_pad = 0;
        w.pend_head = -1;
        w.pend_pad = 0;
      }
    }
    s_->mt_idx_ = Mt64::kN;
    warp_sync();
  }

  // ---- cost model (perf_model.cpp:158-205) ----
  PDG_HD double t_prefill(int32_t l_hist, int32_t l_incr, int deg) const {
    const double load = dadd(static_cast<double>(l_incr), dmul(PDG_PROF.history_weight, static_cast<double>(l_hist)));
    return curve_eval(PDG_PROF.prefill[deg], load);
  }
  PDG_HD double t_kv(int32_t l, int src, int dst) const {
    if (l == 0) return 0.0;
    return curve_eval(PDG_PROF.kv[src][dst], static_cast<double>(l));
  }

  PDG_HD int32_t l_incr_of(int32_t i) const {
    const SessRt& s = GLP(s_->G.sess)[i];
    return round_tr(s.roff + s.round - 1).incr;
  }

  // ---- RNG (coordinator.cpp:124-130): std::mt19937_64 in shared memory ----
  PDG_COLD uint64_t rng_next() {
    if (s_->mt_idx_ >= static_cast<uint32_t>(Mt64::kN)) {
#if defined(__CUDA_ARCH__)
      // Warp-parallel twist in three dependency phases: elements below 156
      // read only old words; 156..310 read updated words i-156; 311 reads
      // updated words 0 and 155.
      uint64_t* mt = MT();
      const int lane = lane_id();
      for (int base = 0; base < 156; base += 32) {
        const int i = base + lane;
        uint64_t v = 0;
        if (i < 156) {
          const uint64_t x = (mt[i] & Mt64::kUpper) | (mt[i + 1] & Mt64::kLower);
          v = mt[i + 156] ^ (x >> 1) ^ ((x & 1ull) ? Mt64::kMatrix : 0ull);
        }
        __syncwarp();
        if (i < 156) mt[i] = v;
        __syncwarp();
      }
      for (int base = 156; base < 311; base += 32) {
        const int i = base + lane;
        uint64_t v = 0;
        if (i < 311) {
          const uint64_t x = (mt[i] & Mt64::kUpper) | (mt[i + 1] & Mt64::kLower);
          v = mt[i - 156] ^ (x >> 1) ^ ((x & 1ull) ? Mt64::kMatrix : 0ull);
        }
        __syncwarp();
        if (i < 311) mt[i] = v;
        __syncwarp();
      }
      {
        const uint64_t x = (mt[311] & Mt64::kUpper) | (mt[0] & Mt64::kLower);
        const uint64_t v = mt[155] ^ (x >> 1) ^ ((x & 1ull) ? Mt64::kMatrix : 0ull);
        __syncwarp();
        if (lane == 0) mt[311] = v;
        __syncwarp();
      }
#else
      mt64_twist(MT());
#endif
      s_->mt_idx_ = 0;
    }
    return mt64_temper(MT()[s_->mt_idx_++]);
  }

  // ---- worker-event slots (registers) ----
  // Minimum (time, key) over the slot table. Times are >= 0 (or +inf), so
  // their bit patterns order like unsigned integers: two warp REDUX.MIN on
  // the 32-bit halves find the earliest time; equal times (rare) are broken
  // by the key the same way.
  // Earliest pending event among the worker slots and, while the session
  // events are a small unordered set, those too: one warp reduction over
  // (time, key). *id_out is the slot index, or kMaxSlots + the session-event
  // entry. Times are >= 0 (or +inf), so their bit patterns order like
  // unsigned integers: two REDUX.MIN on the 32-bit halves find the earliest
  // time; equal times (rare) are broken by the key the same way.
  PDG_HD void next_slot_event(int nslots, double* bt_out, uint64_t* bk_out, bool* tie_out, int* id_out) const {
    const int hn = s_->hsmall_ ? s_->hn_ : 0;
#if defined(__CUDA_ARCH__)
    const int lane = lane_id();
    uint64_t tb = 0x7ff0000000000000ull;  // +inf
    uint64_t kb = ~0ull;
    int id = -1;
    if (lane < nslots) {
      tb = dbits(s_->st_[lane]);
      kb = s_->sk_[lane];
      id = lane;
    }
    if (lane + 32 < nslots) {
      const uint64_t t2 = dbits(s_->st_[lane + 32]);
      const uint64_t k2 = s_->sk_[lane + 32];
      const bool take = (t2 < tb) | ((t2 == tb) & (k2 < kb));  // branch-free select
      tb = take ? t2 : tb;
      kb = take ? k2 : kb;
      id = take ? lane + 32 : id;
    }
    static_assert(kSmallHeap <= 64, "two small-set entries per lane");
    const HEv* h = SHEAP();
    if (lane < hn) {
      const uint64_t t2 = dbits(h[lane].t);
      const uint64_t k2 = h[lane].key;
      const bool take = (t2 < tb) | ((t2 == tb) & (k2 < kb));  // branch-free select
      tb = take ? t2 : tb;
      kb = take ? k2 : kb;
      id = take ? kMaxSlots + lane : id;
    }
    if (lane + 32 < hn) {
      const uint64_t t2 = dbits(h[lane + 32].t);
      const uint64_t k2 = h[lane + 32].key;
      const bool take = (t2 < tb) | ((t2 == tb) & (k2 < kb));  // branch-free select
      tb = take ? t2 : tb;
      kb = take ? k2 : kb;
      id = take ? kMaxSlots + lane + 32 : id;
    }
    const uint32_t hi = static_cast<uint32_t>(tb >> 32);
    const uint32_t mhi = __reduce_min_sync(0xffffffffu, hi);
    const uint32_t lo = hi == mhi ? static_cast<uint32_t>(tb) : 0xffffffffu;
    const uint32_t mlo = __reduce_min_sync(0xffffffffu, lo);
    const bool at = hi == mhi && static_cast<uint32_t>(tb) == mlo;
    uint32_t b = __ballot_sync(0xffffffffu, at);
    *tie_out = __popc(b) > 1 && mhi != 0x7ff00000u;
    if (__popc(b) > 1) {  // several entries share the earliest time: smallest key
      const uint32_t khi = at ? static_cast<uint32_t>(kb >> 32) : 0xffffffffu;
      const uint32_t mkhi = __reduce_min_sync(0xffffffffu, khi);
      const uint32_t klo = (at && khi == mkhi) ? static_cast<uint32_t>(kb) : 0xffffffffu;
      const uint32_t mklo = __reduce_min_sync(0xffffffffu, klo);
      b = __ballot_sync(0xffffffffu, at && khi == mkhi && static_cast<uint32_t>(kb) == mklo);
    }
    const int src = __ffs(b) - 1;
    *bt_out = bitsd((static_cast<uint64_t>(mhi) << 32) | mlo);
    *bk_out = __shfl_sync(0xffffffffu, static_cast<unsigned long long>(kb), src);
    *id_out = __shfl_sync(0xffffffffu, id, src);
#else
    double bt = kInf;
    uint64_t bk = ~0ull;
    int ties = 0, id = -1;
    auto take = [&](double t, uint64_t k, int j) {
      if (t == bt) ++ties;
      if (before(t, k, bt, bk)) {
        if (t < bt) ties = 1;
        bt = t;
        bk = k;
        id = j;
      }
    };
    for (int j = 0; j < nslots; ++j) take(s_->st_[j], s_->sk_[j], j);
    for (int j = 0; j < hn; ++j) take(SHEAP()[j].t, SHEAP()[j].key, kMaxSlots + j);
    *bt_out = bt;
    *bk_out = bk;
    *tie_out = ties > 1 && bt != kInf;
    *id_out = id;
#endif
  }

  PDG_HD void set_slot(int s, double t, uint32_t kind) {
    const uint64_t seq = s_->seq_;
    const uint64_t key = mk_key(kind, seq, static_cast<uint32_t>(s));
    s_->seq_ = seq + 1;
    s_->st_[s] = t;
    s_->sk_[s] = key;
  }
  PDG_HD void clear_slot(int s) {
    s_->st_[s] = kInf;
    s_->sk_[s] = ~0ull;
  }
  PDG_HD int slot_compute(int p) const { return s_->PL.D + p; }
  PDG_HD int slot_history(int p) const { return s_->PL.D + s_->PL.P + p; }

  // ---- session-event heap (shared memory, global spill) ----
  PDG_HD HEv* heap_base() const { return s_->heap_spilled_ ? s_->G.heap : s_->SM.heap; }
  // Earliest session event (requires hn_ > 0).
  PDG_HD void heap_top(double* t, uint64_t* key) const {
    if (s_->heap_spilled_) {
      const HEv* h = GLP(s_->G.heap);
      *t = h[0].t;
      *key = h[0].key;
    } else {
      const HEv* h = SHEAP();
      *t = h[0].t;
      *key = h[0].key;
    }
  }

  PDG_A_HEAP_PUSH void heap_push(double t, uint32_t kind, uint32_t a, uint32_t b) {
    const int64_t t0 = pb();
    heap_push_(t, kind, a, b);
    pe(kProfHeap, t0);
  }
  PDG_HD void heap_push_(double t, uint32_t kind, uint32_t a, uint32_t b) {
    HEv e;
    e.t = t;
    e.key = mk_key(kind, s_->seq_++, 0);
    e.a = a;
    e.b = b;
    if (s_->hsmall_) {
      const int32_t n = s_->hn_;
      const int32_t cap = s_->C.hs < kSmallHeap ? s_->C.hs : kSmallHeap;
      if (n < cap) {
        warp_sync();
        SHEAP()[n] = e;  // warp-uniform store
        s_->hn_ = n + 1;
        return;
      }
      heapify(SHEAP(), n);  // the set outgrew the lane scan: order it as a binary heap
      s_->hsmall_ = 0;
    }
    if (!s_->heap_spilled_ && s_->hn_ >= s_->C.hs) {
      HEv* gh = GLP(s_->G.heap);
      const HEv* sh = SHEAP();
      for (int k = lane_id(); k < s_->hn_; k += PDG_NL) gh[k] = sh[k];
      warp_sync();
      s_->heap_spilled_ = true;
    }
    if (PDG_UNLIKELY(s_->hn_ >= s_->C.hcap)) {
      fail();
      return;
    }
    const int32_t n = s_->hn_++;
    if (s_->heap_spilled_) {
      heap_sift_up(GLP(s_->G.heap), n, e);
    } else {
      heap_sift_up(SHEAP(), n, e);
    }
  }
  PDG_HD static void heap_sift_up(HEv* h, int32_t i, const HEv& e) {
    while (i > 0) {
      const int32_t par = (i - 1) >> 1;
      const HEv pe = h[par];
      if (!before(e.t, e.key, pe.t, pe.key)) break;
      h[i] = pe;  // warp-uniform store
      i = par;
    }
    h[i] = e;  // warp-uniform store
  }

  PDG_HD HEv heap_pop() {
    const int64_t t0 = pb();
    const HEv top = heap_pop_();
    pe(kProfHeap, t0);
    return top;
  }
  PDG_HD HEv heap_pop_() {
    const int32_t n = --s_->hn_;
    const HEv top = s_->heap_spilled_ ? heap_sift_down(GLP(s_->G.heap), n) : heap_sift_down(SHEAP(), n);
    if (n == 0) s_->heap_spilled_ = false;
    if (!s_->heap_spilled_ && n <= kSmallHeap / 2) s_->hsmall_ = 1;  // a heap is also a valid unordered set
    return top;
  }
  // Removes entry j of the small unordered set (the last entry fills the hole).
  PDG_HD HEv heap_take(int32_t j) {
    HEv* h = SHEAP();
    const int32_t n = s_->hn_ - 1;
    const HEv e = h[j];
    const HEv last = h[n];
    warp_sync();
    if (j != n && lane_id() == 0) h[j] = last;
    s_->hn_ = n;
    warp_sync();
    return e;
  }
  PDG_HD static void heapify(HEv* h, int32_t n) {
    for (int32_t r = n / 2 - 1; r >= 0; --r) {
      const HEv x = h[r];
      int32_t i = r;
      for (;;) {
        int32_t c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && before(h[c + 1].t, h[c + 1].key, h[c].t, h[c].key)) ++c;
        if (!before(h[c].t, h[c].key, x.t, x.key)) break;
        const HEv hc = h[c];
        warp_sync();
        h[i] = hc;  // warp-uniform store
        i = c;
      }
      warp_sync();
      h[i] = x;  // warp-uniform store
      warp_sync();
    }
  }
  // Removes h[0] from a heap that now holds n entries (h[n] is the last).
  PDG_HD static HEv heap_sift_down(HEv* h, int32_t n) {
    const HEv top = h[0];
    const HEv last = h[n];
    int32_t i = 0;
    for (;;) {
      int32_t c = 2 * i + 1;
      if (c >= n) break;
      HEv ce = h[c];
      if (c + 1 < n) {
        const HEv c2 = h[c + 1];
        if (before(c2.t, c2.key, ce.t, ce.key)) {
          ++c;
          ce = c2;
        }
      }
      if (!before(ce.t, ce.key, last.t, last.key)) break;
      h[i] = ce;  // warp-uniform store
      i = c;
    }
    warp_sync();
    if (n > 0 && lane_id() == 0) h[i] = last;
    warp_sync();
    return top;
  }

  // ---- admission (sim_engine.cpp:240-267; bind_session coordinator.cpp:60-72) ----
  PDG_HD void on_arrival(int32_t i, int32_t roff, int32_t nround) {
    if (s_->adm_head_ < i) return;  // queue non-empty: park behind the head
    if (!try_admit(i, roff, nround)) return;  // parked: s_->adm_head_ == i
    s_->adm_head_ = i + 1;
  }

  // Least KV bytes, lowest index on ties (coordinator.cpp:60-72). In lazy
  // mode a worker's KV bytes include the silent steps of its in-flight run
  // that end before now; lanes project them per worker without advancing
  // the run (the step log is materialised when the worker is next observed).
  PDG_HD int bind_session(int64_t* kv_best) {
    const int64_t tc0_ = pb();
    const int D = s_->PL.D;
    const double t = s_->now_;
    const uint32_t kind = s_->cur_kind_;
    constexpr bool lazy = kLazy;
    const int64_t kvb = PDG_PROF.kv_bytes_per_token;
    uint64_t key = ~0ull;
    bool ab = false;
    for (int base = 0; base < D; base += PDG_NL) {
      const int d = base + lane_id();
      if (d < D) {
        const DecodeW& w = DW(d);
        int64_t kv = w.kv_used;
        if (lazy) kv += static_cast<int64_t>(w.cohort_n) * silent_done(w, t, kind, &ab) * kvb;
        const uint64_t k = (static_cast<uint64_t>(kv) << 6) | static_cast<uint64_t>(d);
        if (k < key) key = k;
      }
    }
    for (int m = PDG_NL / 2; m > 0; m >>= 1) {
      const uint64_t o = shfl_xor_u64(key, m);
      if (o < key) key = o;
    }
    if (ballot(ab)) s_->abort_ = 1;
    *kv_best = static_cast<int64_t>(key >> 6);
    pe(27, tc0_);
    return static_cast<int>(key & 63u);
  }

  // Silent steps of w's in-flight run that end before t: exactly the steps
  // catch_up_worker(d, t, kind) would advance, without advancing them.
  PDG_HD int64_t silent_done(const DecodeW& w, double t, uint32_t kind, bool* abort) const {
    if (!w.stepping) return 0;
    const int32_t run_b = w.run_b;
    int32_t k = w.steps - 1;
    double e = w.cur_end;
    const double dur = w.dur;
    int64_t total = 0;
    while (k < run_b) {
      if (e > t) break;
      if (e == t) {
        if (kind == kDecodeStep) *abort = true;
        break;
      }
      int32_t done = 1;
      double end = e;
      double next = dadd(e, dur);
      if (!(next > e)) {
        *abort = true;
        break;
      }
      const int32_t room = run_b - (k + 1);
      if (room > 0 && next < t) {
        const double g = dsub(next, e);
        if (room <= kShortBulk) {  // same stepping as catch_up_worker_
          int32_t m = 0;
          double last_end = e, nxt = next;
          while (m < room && nxt < t && dsub(nxt, last_end) == g) {
            ++m;
            last_end = nxt;
            nxt = dadd(nxt, dur);
          }
          if (m > 0) {
            end = last_end;
            done += m;
            next = nxt;
            if (!(next > end)) {
              *abort = true;
              break;
            }
          }
        } else {
          const int64_t m = stable_run(e, dur, g, t, room);
          if (m > 0) {
            end = dadd(next, dmul(static_cast<double>(m - 1), g));
            done += static_cast<int32_t>(m);
            next = dadd(end, dur);
            if (!(next > end)) {
              *abort = true;
              break;
            }
          }
        }
      }
      total += done;
      k += done;
      e = next;
    }
    return total;
  }

  PDG_COLD bool try_admit(int32_t i, int32_t roff, int32_t nround) {
    int64_t kv_best;
    const RoundTr r1 = round_tr(roff);
    const int best = bind_session(&kv_best);
    const DecodeW& w = DW(best);
    const int64_t first = static_cast<int64_t>(r1.incr) * PDG_PROF.kv_bytes_per_token;
    if (kv_best + first > w.kv_cap) return false;
    SessRt& s = GLP(s_->G.sess)[i];
    {  // warp-uniform stores (every lane writes the same values)
      s.roff = roff;
      s.nround = static_cast<int16_t>(nround);
      s.bound = static_cast<int8_t>(best);
      s.round = 1;
      s.ctx = 0;
      s.itl_lo = 0.0;
      s.itl_hi = 0.0;
      s.itl_cnt = 0;
      s.join = 0;
      s.postpone = 0;
      s.ttft_bad = 0;
    }
    if (!kLazy || kRec) {  // the exact engine and the records only
      SessCold& c = GLP(s_->G.sess_cold)[i];
      c.bind_time = s_->now_;  // warp-uniform stores
      c.itl_sum = 0.0;
    }
    start_round(i, 1, best, 0, r1.incr);
    return true;
  }

  PDG_HD void admit_waiting() {
    while (s_->adm_head_ < s_->next_arr_) {
      const int32_t i = s_->adm_head_;
      const int32_t roff = sess_tr(i).round_off;
      if (!try_admit(i, roff, sess_tr(i + 1).round_off - roff)) break;
      ++s_->adm_head_;
    }
  }

  // ---- task creation and routing (sim_engine.cpp:271-333) ----
  PDG_A_START_ROUND void start_round(int32_t i, int round, int bound, int32_t ctx, int32_t incr) {
    SessRt& s = GLP(s_->G.sess)[i];
    {  // warp-uniform stores (every lane writes the same values)
      s.t_enq = s_->now_;
      s.postpone = 0;
    }
    ++s_->ctr_.tasks_created;
    const int64_t tr0 = pb();
    const RouteOut r = decide(i, bound, ctx, incr);
    pe(kProfRoute, tr0);
    if (kRec && s_->REC.decisions && lane_id() == 0) {
      pdsim_decision& d = s_->REC.decisions[s_->n_dec_];
      d.time = s_->now_;
      d.session_id = GLP(s_->T.sid)[i];
      d.round = round;
      d.worker = r.local ? s_->PL.P + bound : r.p;
      d.local = static_cast<int8_t>(r.local);
      d.rationale = static_cast<int8_t>(r.rationale);
      d.has_estimate = static_cast<int8_t>(r.has_est);
      for (int k = 0; k < 5; ++k) d.reserved[k] = 0;
      d.estimated_cost = r.has_est ? r.est : 0.0;
    }
    ++s_->n_dec_;
    const int64_t te0 = pb();
    if (r.local) {
      enqueue_local(bound, i, ctx, incr);
    } else {
      enqueue_remote(r.p, i, ctx, incr);
    }
    pe(kProfEnqueue, te0);
  }

  PDG_HD RouteOut decide(int32_t i, int bound, int32_t ctx, int32_t incr) {
    RouteOut r;
    r.local = 1;
    r.p = -1;
    r.has_est = 0;
    r.est = 0.0;
    if (s_->PR.routing == PDSIM_ROUTING_ALWAYS_LOCAL) {
      r.rationale = PDSIM_RATIONALE_FORCED_LOCAL;
      return r;
    }
    if (s_->PR.routing == PDSIM_ROUTING_ALWAYS_REMOTE) {
      if (s_->PL.P == 0) {
        r.rationale = PDSIM_RATIONALE_FORCED_LOCAL;
        return r;
      }
      r.local = 0;
      r.p = s_->rr_next_;
      s_->rr_next_ = (s_->rr_next_ + 1) % s_->PL.P;
      r.rationale = PDSIM_RATIONALE_FORCED_REMOTE;
      return r;
    }
    return route(bound, ctx, incr);
  }

  // Coordinator::route (coordinator.cpp:115-171).
  // Returns the decision by value (registers across the call: no stack).
  PDG_COLD RouteOut route(int bound, int32_t ctx, int32_t incr) {
    RouteOut r;
    r.has_est = 0;
    r.est = 0.0;
    const int n = s_->PL.P;
    if (n > 0) {
#if defined(__CUDA_ARCH__)
      const uint32_t idx = s_->mt_idx_;
      const bool packed = n <= 16 && idx + static_cast<uint32_t>(n - 1) <= static_cast<uint32_t>(Mt64::kN);
#else
      const bool packed = false;
#endif
      uint64_t perm = 0;  // packed scan order, 4 bits per position (n <= 16)
      int32_t* order = ORD();
      if (packed) {
#if defined(__CUDA_ARCH__)
        // The n-1 draws of one route are consecutive engine outputs with no
        // twist in between: lane t tempers word idx+t and reduces it mod
        // n-t (draw t belongs to k = n-1-t); the swaps then run on a
        // register-packed permutation.
        const int lane = lane_id();
        uint32_t j = 0;
        if (lane < n - 1) j = umod64_small(mt64_temper(MT()[idx + lane]), static_cast<uint32_t>(n - lane));
        const uint32_t jlo = __reduce_or_sync(0xffffffffu, lane < 8 ? j << (4 * lane) : 0u);
        const uint32_t jhi = __reduce_or_sync(0xffffffffu, (lane >= 8 && lane < 16) ? j << (4 * (lane - 8)) : 0u);
        const uint64_t js = (static_cast<uint64_t>(jhi) << 32) | jlo;
        s_->mt_idx_ = idx + static_cast<uint32_t>(n - 1);
        perm = 0xfedcba9876543210ull;
        for (int t = 0; t < n - 1; ++t) {
          const int k = n - 1 - t;
          const int jj = static_cast<int>((js >> (4 * t)) & 15u);
          const uint64_t x = ((perm >> (4 * k)) ^ (perm >> (4 * jj))) & 15u;
          perm ^= (x << (4 * k)) | (x << (4 * jj));
        }
#endif
      } else {
        {  // warp-uniform stores (every lane writes the same values)
          for (int k = 0; k < n; ++k) order[k] = k;
        }
        for (int k = n - 1; k > 0; --k) {
          const int j = static_cast<int>(umod64_small(rng_next(), static_cast<uint32_t>(k + 1)));
          const int a = order[k], b = order[j];
          {  // warp-uniform stores (every lane writes the same values)
            order[k] = b;
            order[j] = a;
          }
        }
      }
      const double thr = dmul(s_->PR.alpha, s_->T.ttft_thres);
#if defined(__CUDA_ARCH__) && PDG_ROUTE_SCAN > 0
#if PDG_ROUTE_SCAN == 2
      // The first worker of the scan alone (warp-collective trim); the rest,
      // when it has no slack, in parallel.
      const int p0 = packed ? static_cast<int>(perm & 15u) : order[0];
      const int p = ttft_has_slack(p0, thr) ? p0 : n > 1 ? slack_scan(thr, perm, packed, n, p0) : -1;
#else
      const int p = slack_scan(thr, perm, packed, n, -1);
#endif
      if (p >= 0) {
        r.local = 0;
        r.p = p;
        r.rationale = PDSIM_RATIONALE_SLACK_REMOTE;
        return r;
      }
#else
      for (int k = 0; k < n; ++k) {
        const int p = packed ? static_cast<int>((perm >> (4 * k)) & 15u) : order[k];
        if (ttft_has_slack(p, thr)) {
          r.local = 0;
          r.p = p;
          r.rationale = PDSIM_RATIONALE_SLACK_REMOTE;
          return r;
        }
      }
#endif
    }
    if (itl_has_slack(bound, dmul(s_->PR.beta, s_->T.itl_thres))) {
      r.local = 1;
      r.p = -1;
      r.rationale = PDSIM_RATIONALE_SLACK_LOCAL;
      return r;
    }
    r = argmin_route(bound, ctx, incr);
    r.rationale = PDSIM_RATIONALE_ARGMIN;
    return r;
  }

#if defined(__CUDA_ARCH__)
  // The slack scan of Coordinator::route (coordinator.cpp:139-150): the first
  // prefill worker in the shuffled scan order whose windowed TTFT mean is
  // <= thr (worker `skip`, already found without slack, excluded). Lane p
  // tests worker p (its own window, trimmed by that lane), all at once; the
  // winner is the lowest scan position with slack. Trimming a
  // window the sequential scan would not have reached changes nothing: its
  // expired samples are expired at every later query too (queries only move
  // forward in time), and the ring only gains room.
  PDG_HD int slack_scan(double thr, uint64_t perm, bool packed, int n, int skip) {
    warp_sync();  // the scan order (ORD) was written by the whole warp
    const int lane = lane_id();
    bool slack = false, folded = false;
    if (lane < n && lane != skip) {
      PrefillW& w = PW(lane);
      const size_t base = static_cast<size_t>(lane) * s_->C.twcap;
      const uint32_t mask = static_cast<uint32_t>(s_->C.twcap - 1);
      const double* times = GLP(s_->G.tw_t) + base;
      const double cutoff = dsub(s_->now_, s_->PR.stat_window);
      uint32_t head = w.tw.head;
      const uint32_t end = w.tw.end;
      while (head != end && times[head & mask] <= cutoff) ++head;
      const Brk tail = w.tw.tail;
      w.tw.head = head;  // this lane's own worker
      if (head == end) {
        slack = 0.0 <= thr;  // an empty window reads 0
      } else {
        const Brk hp = GLP(s_->G.tw_p)[base + (head & mask)];
        double lo = sub_rd(tail.lo, hp.hi);
        const double hi = sub_ru(tail.hi, hp.lo);
        if (lo < 0.0) lo = 0.0;
        const int dec = mean_le_bracket(lo, hi, static_cast<int64_t>(end - head), thr);
        if (PDG_LIKELY(dec >= 0)) {
          slack = dec == 1;
        } else {  // inside the error band: the reference's sequential fold
          folded = true;
          const double* v = GLP(s_->G.tw_v) + base;
          double sum = 0.0;
          for (uint32_t k = head; k != end; ++k) sum = dadd(sum, v[k & mask]);
          slack = ddiv(sum, static_cast<double>(end - head)) <= thr;
        }
      }
    }
    const uint32_t nf = ballot(folded);
    const int pk = lane < n ? (packed ? static_cast<int>((perm >> (4 * lane)) & 15u) : ORD()[lane]) : 0;
    const bool sk = shfl_i(slack ? 1 : 0, pk) != 0;
    const uint32_t b = ballot(lane < n && sk);
    warp_sync();
    if (nf) s_->folds_ += popc(nf);  // warp-uniform store
    if (!b) return -1;
    return shfl_i(pk, __ffs(b) - 1);
  }
#endif

  // ---- routing estimates (coordinator.cpp:74-100) ----
  PDG_HD double fold_queue(const TaskQueue& q, const double* qc, double init) const {
    const uint32_t mask = static_cast<uint32_t>(s_->C.qcap - 1);
    double c = init;
    for (uint32_t k = q.qh; k != q.qt; ++k) c = dadd(c, qc[k & mask]);
    return c;
  }
  // Estimate of candidate c (-1 local, else prefill worker c): the exact
  // reference value, or a certified bracket [lo, hi] around it.
  PDG_HD void estimate(int d, int32_t ctx, int32_t incr, int c, bool force_exact, double* lo, double* hi,
                       bool* exact) const {
    if (c < 0) {
      const DecodeW& w = DW(d);
      const uint32_t len = w.q.qt - w.q.qh;
      const double own = t_prefill(ctx, incr, w.deg);
      if (force_exact || len <= 2 || !w.q.sum.exact()) {
        *lo = *hi = fold_queue(w.q, GLP(s_->G.dq_c) + static_cast<size_t>(d) * s_->C.qcap, own);
        *exact = true;
        return;
      }
      const double v = dadd(own, fx_to_double(w.q.sum.sum));
      const double m = fold_margin(static_cast<int64_t>(len) + 1);
      *lo = v * (1.0 - m);
      *hi = v * (1.0 + m);
      *exact = false;
      return;
    }
    const PrefillW& w = PW(c);
    const int pd = w.deg, dd = DW(d).deg;
    const uint32_t len = w.q.qt - w.q.qh;
    const double head = dadd(t_prefill(ctx, incr, pd), dadd(t_kv(ctx, dd, pd), t_kv(incr, pd, dd)));
    if (force_exact || len <= 2 || !w.q.sum.exact()) {
      *lo = *hi = dadd(head, fold_queue(w.q, GLP(s_->G.pq_c) + static_cast<size_t>(c) * s_->C.qcap, 0.0));
      *exact = true;
      return;
    }
    const double v = dadd(head, fx_to_double(w.q.sum.sum));
    const double m = fold_margin(static_cast<int64_t>(len));
    *lo = v * (1.0 - m);
    *hi = v * (1.0 + m);
    *exact = false;
  }

  // Lines 6-9 of Alg. 1: best = local; for i: if (cost_i < best) take i.
  // The strict-< scan ends on the FIRST candidate (local first, then the
  // lowest worker index) holding the minimum value. Lanes estimate remote
  // candidates in parallel; a candidate whose bracket starts above the
  // smallest upper bound cannot win, and exact folds run only when two or
  // more candidates remain in contention.
  PDG_COLD RouteOut argmin_route(int d, int32_t ctx, int32_t incr) {
    // prefill candidates per lane: the compiled layout bounds P by kP
    constexpr int kPer = ((kP > 0 ? kP : kMaxSlots) + PDG_NL - 1) / PDG_NL;
    const int n = s_->PL.P;
    const int lane = lane_id();
    double llo, lhi;
    bool lex;
    estimate(d, ctx, incr, -1, false, &llo, &lhi, &lex);
    double rlo[kPer], rhi[kPer];
    bool rex[kPer];
    double min_hi = lhi;
    for (int k = 0; k < kPer; ++k) {
      const int c = lane + k * PDG_NL;
      rlo[k] = kInf;
      rhi[k] = kInf;
      rex[k] = true;
      if (c < n) estimate(d, ctx, incr, c, false, &rlo[k], &rhi[k], &rex[k]);
      if (rhi[k] < min_hi) min_hi = rhi[k];
    }
    min_hi = warp_min(min_hi);
    const bool lcan = llo <= min_hi;
    int count = lcan ? 1 : 0;
    bool can[kPer];
    for (int k = 0; k < kPer; ++k) {
      can[k] = (lane + k * PDG_NL) < n && rlo[k] <= min_hi;
      count += popc(ballot(can[k]));
    }
    int winner;
    double est;
    bool est_exact;
    if (count >= 2) {
      if (lcan && !lex) {
        ++s_->folds_;
        estimate(d, ctx, incr, -1, true, &llo, &lhi, &lex);
      }
      double v = lcan ? llo : kInf;
      for (int k = 0; k < kPer; ++k) {
        if (can[k] && !rex[k]) estimate(d, ctx, incr, lane + k * PDG_NL, true, &rlo[k], &rhi[k], &rex[k]);
        if (can[k] && rlo[k] < v) v = rlo[k];
      }
      v = warp_min(v);
      winner = -2;
      if (lcan && llo == v) winner = -1;
      for (int k = 0; k < kPer && winner == -2; ++k) {
        const uint32_t b = ballot(can[k] && rlo[k] == v);
        if (b) winner = k * PDG_NL + first_zero(~b);
      }
      est = v;
      est_exact = true;
    } else if (lcan) {
      winner = -1;
      est = llo;
      est_exact = lex;
    } else {
      winner = -2;
      for (int k = 0; k < kPer && winner == -2; ++k) {
        const uint32_t b = ballot(can[k]);
        if (b) winner = k * PDG_NL + first_zero(~b);
      }
      if (winner < 0) {  // no contender at all: impossible, keep state consistent
        fail();
        winner = -1;
      }
      const int owner = winner % PDG_NL, kk = winner / PDG_NL;
      double lo = kInf;
      int ex = 1;
      for (int k = 0; k < kPer; ++k) {
        if (k == kk) {
          lo = rlo[k];
          ex = rex[k] ? 1 : 0;
        }
      }
      est = shfl_d(lo, owner);
      est_exact = shfl_i(ex, owner) != 0;
    }
    if (kRec && !est_exact && s_->REC.decisions) {
      double a, b;
      bool e;
      estimate(d, ctx, incr, winner, true, &a, &b, &e);
      est = a;
    }
    RouteOut r;
    r.local = winner < 0 ? 1 : 0;
    r.p = winner < 0 ? -1 : winner;
    r.rationale = PDSIM_RATIONALE_ARGMIN;
    r.has_est = 1;
    r.est = est;
    return r;
  }

  // ---- windowed statistics (coordinator.cpp:27-47) ----
  // Drops entries with time <= now - window from the head (times are
  // non-decreasing, so expired entries form a prefix): one ballot per 32.
  PDG_HD void window_trim(WinState& w, const double* times, uint32_t mask, double now) {
    const double cutoff = dsub(now, s_->PR.stat_window);
    uint32_t head = w.head;
    const uint32_t end = w.end;
    while (head != end) {
      const uint32_t off = static_cast<uint32_t>(lane_id());
      const bool in = off < end - head;
      const bool expired = in && times[(head + off) & mask] <= cutoff;
      const int n = first_zero(ballot(expired));
      head += static_cast<uint32_t>(n);
      if (n < PDG_NL) break;
    }
    w.head = head;  // warp-uniform store
  }

  PDG_HD bool window_room(WinState& w, const double* times, uint32_t cap, double now) {
    if (w.end - w.head >= cap - 1) {
      window_trim(w, times, cap - 1, now);
      if (PDG_UNLIKELY(w.end - w.head >= cap - 1)) {
        fail();
        return false;
      }
    }
    return true;
  }

    PDG_HD void ttft_add(int p, double v) {
    const int64_t t0_ = pb();
    ttft_add_(p, v);
    pe(18, t0_);
  }
  PDG_HD void ttft_add_(int p, double v) {
    PrefillW& w = PW(p);
    const size_t base = static_cast<size_t>(p) * s_->C.twcap;
    const uint32_t mask = static_cast<uint32_t>(s_->C.twcap - 1);
    if (!window_room(w.tw, GLP(s_->G.tw_t) + base, static_cast<uint32_t>(s_->C.twcap), s_->now_)) return;
    const uint32_t k = w.tw.end & mask;
    const Brk cur = w.tw.tail;
    Brk next;
    next.lo = add_rd(cur.lo, v);
    next.hi = add_ru(cur.hi, v);
    {  // warp-uniform stores (every lane writes the same values)
      GLP(s_->G.tw_t)[base + k] = s_->now_;
      GLP(s_->G.tw_v)[base + k] = v;
      GLP(s_->G.tw_p)[base + k] = cur;
      w.tw.tail = next;
      ++w.tw.end;
    }
  }

  // query(now) <= thr with the sequential windowed mean's semantics.
    PDG_A_TTFT_HAS_SLACK bool ttft_has_slack(int p, double thr) {
    const int64_t t0_ = pb();
    const bool r_ = ttft_has_slack_(p, thr);
    pe(20, t0_);
    return r_;
  }
  PDG_HD bool ttft_has_slack_(int p, double thr) {
    PrefillW& w = PW(p);
    const size_t base = static_cast<size_t>(p) * s_->C.twcap;
    const uint32_t mask = static_cast<uint32_t>(s_->C.twcap - 1);
    window_trim(w.tw, GLP(s_->G.tw_t) + base, mask, s_->now_);
    const uint32_t head = w.tw.head, end = w.tw.end;
    if (head == end) return 0.0 <= thr;  // an empty window reads 0
    // Window sum bracket = tail prefix - head prefix (TTFT values are >= 0);
    // the reference's fold is within gamma_{n-1} of the exact sum.
    const Brk hp = GLP(s_->G.tw_p)[base + (head & mask)];
    double lo = sub_rd(w.tw.tail.lo, hp.hi);
    const double hi = sub_ru(w.tw.tail.hi, hp.lo);
    if (lo < 0.0) lo = 0.0;
    const int dec = mean_le_bracket(lo, hi, static_cast<int64_t>(end - head), thr);
    if (PDG_LIKELY(dec >= 0)) return dec == 1;
    ++s_->folds_;
    double sum = 0.0;
    for (uint32_t k = head; k != end; ++k) sum = dadd(sum, GLP(s_->G.tw_v)[base + (k & mask)]);
    return ddiv(sum, static_cast<double>(end - head)) <= thr;
  }

  // ---- step-segment log: ITL window + per-session ITL folds ----
  PDG_HD Seg* seg_ring(int d) const { return GLP(s_->G.seg) + static_cast<size_t>(d) * s_->C.segcap; }
  // Segment i of worker d (i == seg_end is the open one, in shared memory).
  PDG_HD Seg seg_at(int d, int32_t i) const {
    const DecodeW& w = DW(d);
    if (i == w.seg_end) return w.sg;
    return seg_ring(d)[static_cast<uint32_t>(i) & static_cast<uint32_t>(s_->C.segcap - 1)];
  }
  // Exact end time of step j of segment g (the progression is exact).
  PDG_HD static double seg_time(const Seg& g, int32_t j) {
    return dadd(g.t0, dmul(static_cast<double>(j - g.first), g.gap));
  }

  // Appends n consecutive steps (first index `first`, first end time t0,
  // each with ITL gap `gap` and `cnt` ITL samples) to worker d's log.
    PDG_A_SEG_APPEND void seg_append(int d, int32_t first, int32_t n, double t0, double gap, uint32_t cnt) {
    const int64_t t0_ = pb();
    seg_append_(d, first, n, t0, gap, cnt);
    pe(16, t0_);
  }
  PDG_HD void seg_append_(int d, int32_t first, int32_t n, double t0, double gap, uint32_t cnt) {
    DecodeW& w = DW(d);
    if (w.sg.n > 0 && gap == w.sg.gap && first == w.sg.first + w.sg.n) {
      if (cnt == w.sg.cnt) {
        w.sg.n = w.sg.n + n;  // extends the open segment (t0 continues the progression)
        return;
      }
      if (w.sg.n == 1) {  // a run's first step (joiners emit no sample yet) heads the same segment
        w.sg.cnt_first = w.sg.cnt;
        w.sg.cnt = cnt;
        w.sg.n = 1 + n;
        return;
      }
    }
    if (w.sg.n > 0) {
      // close the open segment into the ring
      const int32_t end = w.seg_end;
      if (end - w.seg_keep >= s_->C.segcap) {
        seg_trim(d, t0);  // later queries are at >= t0
        seg_reclaim(d, first);
        if (PDG_UNLIKELY(end - w.seg_keep >= s_->C.segcap)) {
          fail();
          return;
        }
      }
      const Seg c = w.sg;
      seg_ring(d)[static_cast<uint32_t>(end) & static_cast<uint32_t>(s_->C.segcap - 1)] = c;
      w.seg_end = end + 1;
      const int64_t k = seg_samples(c, 0, c.n);
      w.sg.plo = add_rd(c.plo, mul_rd(static_cast<double>(k), c.gap));
      w.sg.phi = add_ru(c.phi, mul_ru(static_cast<double>(k), c.gap));
      w.sg.pterms = c.pterms + k;
    }
    w.sg.t0 = t0;
    w.sg.gap = gap;
    w.sg.first = first;
    w.sg.n = n;
    w.sg.cnt = cnt;
    w.sg.cnt_first = cnt;
  }
  // ITL samples of steps [first + a, first + b) of segment g.
  PDG_HD static int64_t seg_samples(const Seg& g, int32_t a, int32_t b) {
    if (b > g.n) b = g.n;
    if (b <= a) return 0;
    return a == 0 ? static_cast<int64_t>(g.cnt_first) + static_cast<int64_t>(g.cnt) * (b - 1)
                  : static_cast<int64_t>(g.cnt) * (b - a);
  }

  // Frees ring slots no longer needed: behind the ITL window head and before
  // any step an active round can still fold (rounds span <= maxdec steps).
  PDG_HD void seg_reclaim(int d, int32_t cur_step) {
    DecodeW& w = DW(d);
    const int32_t oldest_needed = cur_step - s_->C.maxdec - 1;
    int32_t keep = w.seg_keep;
    while (keep < w.seg_head && keep < w.seg_end) {
      const Seg g = seg_ring(d)[static_cast<uint32_t>(keep) & static_cast<uint32_t>(s_->C.segcap - 1)];
      if (g.first + g.n - 1 >= oldest_needed) break;
      ++keep;
    }
    w.seg_keep = keep;
  }

  // Advances the ITL window head past steps that ended at or before
  // now - window (coordinator.cpp:32-40: the interval is (now - w, now]).
  PDG_HD void seg_trim(int d, double now) {
    DecodeW& w = DW(d);
    const double cutoff = dsub(now, s_->PR.stat_window);
    int32_t h = w.seg_head, off = w.seg_off;
    for (;;) {
      const Seg g = seg_at(d, h);
      if (g.n == 0 || off >= g.n) {  // empty open segment, or fully expired
        if (h == w.seg_end) break;
        ++h;
        off = 0;
        continue;
      }
      if (seg_time(g, g.first + g.n - 1) <= cutoff) {  // the whole segment expired
        if (h == w.seg_end) {
          off = g.n;
          break;
        }
        ++h;
        off = 0;
        continue;
      }
      // partially expired: steps first .. first+q-1 end at or before cutoff
      int32_t q = 0;
      if (g.t0 <= cutoff) {
        const double est = floor(ddiv(dsub(cutoff, g.t0), g.gap));
        q = static_cast<int32_t>(est < 0.0 ? 0.0 : (est > g.n ? g.n : est)) + 1;
        while (q > 1 && seg_time(g, g.first + q - 1) > cutoff) --q;
        while (q < g.n && seg_time(g, g.first + q) <= cutoff) ++q;
      }
      if (q > off) off = q;
      break;
    }
    w.seg_head = h;
    w.seg_off = off;
  }

  // Windowed ITL mean <= thr (coordinator.cpp:32-47 over run-length steps).
    PDG_HD bool itl_has_slack(int d, double thr) {
    const int64_t t0_ = pb();
    const bool r_ = itl_has_slack_(d, thr);
    pe(19, t0_);
    return r_;
  }
  PDG_HD bool itl_has_slack_(int d, double thr) {
    if (kLazy) catch_up_worker(d, s_->now_, s_->cur_kind_);
    seg_trim(d, s_->now_);
    const DecodeW& w = DW(d);
    // Exact window sum S = sum over in-window steps of cnt * gap, bracketed
    // by the difference of two directed-rounding prefix brackets: after the
    // open segment (tail) and before the first in-window step (head). The
    // reference's fold differs from S by <= gamma_{n-1} S.
    const Seg& o = w.sg;
    const int64_t ko = seg_samples(o, 0, o.n);
    const double tlo = add_rd(o.plo, mul_rd(static_cast<double>(ko), o.gap));
    const double thi = add_ru(o.phi, mul_ru(static_cast<double>(ko), o.gap));
    const Seg h = seg_at(d, w.seg_head);
    const int64_t kh = seg_samples(h, 0, w.seg_off);
    const double hlo = add_rd(h.plo, mul_rd(static_cast<double>(kh), h.gap));
    const double hhi = add_ru(h.phi, mul_ru(static_cast<double>(kh), h.gap));
    const int64_t terms = o.pterms + ko - (h.pterms + kh);
    double lo = sub_rd(tlo, hhi);
    const double hi = sub_ru(thi, hlo);
    if (lo < 0.0) lo = 0.0;
    if (terms == 0) return 0.0 <= thr;  // an empty window reads 0
    const int dec = mean_le_bracket(lo, hi, terms, thr);
    if (PDG_LIKELY(dec >= 0)) return dec == 1;
    ++s_->folds_;
    double sum = 0.0;
    for (int32_t i = w.seg_head; i <= w.seg_end; ++i) {
      const Seg g = seg_at(d, i);
      const int32_t skip = i == w.seg_head ? w.seg_off : 0;
      if (g.n > skip) {
        sum = fold_repeat(sum, g.gap, static_cast<uint64_t>(seg_samples(g, skip, g.n)));
      }
    }
    return ddiv(sum, static_cast<double>(terms)) <= thr;
  }

  // Bracket [lo, hi] of the sum of the ITL gaps of steps (j0, k] of worker
  // d (one sample per step), where step k is the step ending now. Every gap
  // is fl(e_j - e_{j-1}) of consecutive step end times, so the sum is within
  // a relative u of e_k - e_j0 (exactly equal when the subtractions are
  // exact); e_j0 comes from the segment holding step j0, at or after `hint`
  // (the open-segment index when the round joined).
  PDG_HD void seg_span(int d, int32_t j0, int32_t hint, double* lo, double* hi) {
    const int64_t t0_ = pb();
    seg_span_(d, j0, hint, lo, hi);
    pe(22, t0_);
  }
  PDG_HD void seg_span_(int d, int32_t j0, int32_t hint, double* lo, double* hi) {
    const DecodeW& w = DW(d);
    if (PDG_UNLIKELY(hint < w.seg_keep)) {  // the needed steps were reclaimed: capacity bound broken
      fail();
      *lo = *hi = 0.0;
      return;
    }
    const int32_t gi = seg_find(d, j0, hint);
    if (PDG_UNLIKELY(gi < 0)) {
      fail();
      *lo = *hi = 0.0;
      return;
    }
    const Seg g = seg_at(d, gi);
    const double ej = seg_time(g, j0);
    const double now = s_->now_;
    *lo = mul_rd(sub_rd(now, ej), 1.0 - 0x1p-51);
    *hi = mul_ru(sub_ru(now, ej), 1.0 + 0x1p-51);
    if (*lo < 0.0) *lo = 0.0;
  }

  // Index of the first segment at or after `hint` that holds step j (i.e.
  // j < first + n; the open segment has index seg_end), or -1. Segments are
  // ordered by first step; lanes test 32 candidates per ballot.
  PDG_HD int32_t seg_find(int d, int32_t j, int32_t hint) const {
    const DecodeW& w = DW(d);
    const int32_t end = w.seg_end;
    const Seg* ring = seg_ring(d);
    const uint32_t mask = static_cast<uint32_t>(s_->C.segcap - 1);
#if defined(__CUDA_ARCH__)
    for (int32_t base = hint; base <= end; base += 32) {
      const int32_t i = base + lane_id();
      bool hit = false;
      if (i < end) {
        const Seg& g = ring[static_cast<uint32_t>(i) & mask];
        hit = j < g.first + g.n;
      } else if (i == end) {
        hit = j < w.sg.first + w.sg.n;
      }
      const uint32_t b = ballot(hit);
      if (b) return base + __ffs(b) - 1;
    }
    return -1;
#else
    for (int32_t i = hint; i <= end; ++i) {
      const Seg& g = i == end ? w.sg : ring[static_cast<uint32_t>(i) & mask];
      if (j < g.first + g.n) return i;
    }
    return -1;
#endif
  }

  // Sequential fold of the ITL gaps of steps [a, k] of worker d onto s
  // (one sample per step: a session's own tokens, sim_engine.cpp:544-555).
  // `hint` is the open-segment index when the round joined: the segment
  // holding step a is at or after it.
  PDG_HD double seg_fold(int d, int32_t a, int32_t k, double s, int32_t hint) {
    const DecodeW& w = DW(d);
    if (a > k) return s;
    if (PDG_UNLIKELY(hint < w.seg_keep)) {  // the needed steps were reclaimed: capacity bound broken
      fail();
      return s;
    }
    const Seg* ring = seg_ring(d);
    const uint32_t mask = static_cast<uint32_t>(s_->C.segcap - 1);
    const int32_t from = seg_find(d, a, hint);
    if (from < 0) return s;
    for (int32_t i = from; i <= w.seg_end; ++i) {
      const Seg& g = i == w.seg_end ? w.sg : ring[static_cast<uint32_t>(i) & mask];
      const int32_t gfirst = g.first, gn = g.n;
      const int32_t lo = a > gfirst ? a : gfirst;
      const int32_t hi = k < gfirst + gn - 1 ? k : gfirst + gn - 1;
      if (hi < lo) {
        if (gfirst > k) break;
        continue;
      }
      const double gap = g.gap;
      const int32_t cnt = hi - lo + 1;
      if (cnt <= 4) {
        for (int32_t c = 0; c < cnt; ++c) s = dadd(s, gap);
      } else {
        s = fold_repeat(s, gap, static_cast<uint64_t>(cnt));
      }
      if (hi == k) break;
    }
    return s;
  }

  // ---- queues + reorder (reorder.cpp:76-146; select_next sim_engine.cpp:335-350) ----
  PDG_HD bool queue_push(TaskQueue& q, int32_t* qs, double* qc, int32_t i, double cost) {
    const uint32_t qh = q.qh, qt = q.qt;
    if (PDG_UNLIKELY(qt - qh >= static_cast<uint32_t>(s_->C.qcap))) {
      fail();
      return false;
    }
    const uint32_t mask = static_cast<uint32_t>(s_->C.qcap - 1);
    ExactSum ns = q.sum;
    ns.add(cost);
    {  // warp-uniform stores (every lane writes the same values)
      qs[qt & mask] = i;
      qc[qt & mask] = cost;
      q.sum = ns;
      q.qt = qt + 1;
    }
    return true;
  }

  // Dequeues the next task (after reordering the head window).
  PDG_A_SELECT_NEXT int32_t select_next(TaskQueue& q, int32_t* qs, double* qc, double* cost) {
    const int64_t t0 = pb();
    const int32_t i = select_next_(q, qs, qc, cost);
    pe(kProfDequeue, t0);
    return i;
  }
  PDG_HD int32_t select_next_(TaskQueue& q, int32_t* qs, double* qc, double* cost) {
    const uint32_t mask = static_cast<uint32_t>(s_->C.qcap - 1);
    const uint32_t qh = q.qh;
    if (s_->PR.reorder) {
      const uint32_t len = q.qt - qh;
      const int m = static_cast<int>(len < static_cast<uint32_t>(s_->PR.window) ? len : static_cast<uint32_t>(s_->PR.window));
      if (m > 1) reorder_head(qs, qc, qh, m);
    }
    const int32_t i = qs[qh & mask];
    *cost = qc[qh & mask];
    ExactSum ns = q.sum;
    ns.remove(*cost);
    const int32_t pc = GLP(s_->G.sess)[i].postpone;
    {  // warp-uniform stores (every lane writes the same values)
      q.sum = ns;
      q.qh = qh + 1;
    }
    if (pc > s_->ctr_.max_postpone_observed) s_->ctr_.max_postpone_observed = pc;
    return i;
  }

  // Exhaustive search over the lexicographic permutations of the first m
  // queued tasks with strict improvements only: the winner is the
  // lexicographically first permutation with the maximum count among the
  // allowed ones (the identity is always allowed); capped tasks cannot be
  // pushed back (reorder.cpp:93-138). Lanes evaluate permutations in parallel.
#if defined(__CUDA_ARCH__)
  // Device form: lane k holds queued task k (session, cost, wait, postpone
  // count) in registers; permutations are packed 4 bits per position and
  // read the task fields with shuffles, so nothing goes to local memory.
  // Lanes scan ranks base+lane in warp-uniform rounds; one REDUX.MAX over
  // (count << 16 | ~rank) picks the largest count, ties to the smallest rank
  // (the identity, rank 0, wins every tie: strict improvements only).
  PDG_COLD void reorder_head(int32_t* qs, double* qc, uint32_t qh, int m) {
    const uint32_t mask = static_cast<uint32_t>(s_->C.qcap - 1);
    const int lane = lane_id();
    int32_t ms = 0;
    double mc = 0.0, mw = 0.0;
    int mp = 0;
    if (lane < m) {
      ms = qs[(qh + lane) & mask];
      mc = qc[(qh + lane) & mask];
      const SessRt& s = GLP(s_->G.sess)[ms];
      mw = dsub(s_->now_, s.t_enq);
      mp = s.postpone;
    }
    const double thres = s_->T.ttft_thres;
    int id_sat = 0;
    {
      double el = 0.0;
      for (int k = 0; k < m; ++k) {
        el = dadd(el, shfl_d(mc, k));
        if (dadd(shfl_d(mw, k), el) <= thres) ++id_sat;
      }
    }
    if (id_sat == m) return;  // the identity already satisfies every task
    const uint32_t capped = ballot(lane < m && mp >= s_->PR.window);
    uint32_t nperm = 1;
    for (int k = 2; k <= m; ++k) nperm *= static_cast<uint32_t>(k);
    uint32_t best = (static_cast<uint32_t>(id_sat) << 16) | 0xffffu;
    for (uint32_t base = 0; base < nperm; base += 32) {
      const uint32_t r = base + static_cast<uint32_t>(lane);
      const bool valid = r >= 1 && r < nperm;
      const uint32_t pk = unrank_packed(valid ? r : 0u, m);
      bool allowed = valid;
      double el = 0.0;
      int sat = 0;
      for (int k = 0; k < m; ++k) {
        const int p = static_cast<int>((pk >> (4 * k)) & 15u);
        if (k > p && ((capped >> p) & 1u)) allowed = false;
        el = dadd(el, shfl_d(mc, p));
        if (dadd(shfl_d(mw, p), el) <= thres) ++sat;
      }
      if (allowed) {
        const uint32_t key = (static_cast<uint32_t>(sat) << 16) | (0xffffu - r);
        if (key > best) best = key;
      }
    }
    best = __reduce_max_sync(0xffffffffu, best);
    const uint32_t best_r = 0xffffu - (best & 0xffffu);
    if (best_r == 0) return;
    const uint32_t pk = unrank_packed(best_r, m);
    const int p = lane < m ? static_cast<int>((pk >> (4 * lane)) & 15u) : 0;
    const int32_t ns = shfl_i(ms, p);
    const double nc = shfl_d(mc, p);
    if (lane < m) {
      qs[(qh + lane) & mask] = ns;
      qc[(qh + lane) & mask] = nc;
      if (lane > p) ++GLP(s_->G.sess)[ns].postpone;
    }
    warp_sync();
  }

  // k-th (0-based) lexicographic permutation of 0..m-1, 4 bits per position.
  PDG_HD static uint32_t unrank_packed(uint32_t k, int m) {
    uint64_t avail = 0x76543210ull;
    uint32_t out = 0;
    uint32_t f = 1;
    for (int i = 2; i < m; ++i) f *= static_cast<uint32_t>(i);  // (m-1)!
    for (int i = 0; i < m; ++i) {
      const uint32_t q = k / f;
      k -= q * f;
      const uint32_t sh = 4 * q;
      out |= static_cast<uint32_t>((avail >> sh) & 15u) << (4 * i);
      avail = (avail & ((1ull << sh) - 1ull)) | ((avail >> (sh + 4)) << sh);
      const int rest = m - 1 - i;
      if (rest > 0) f /= static_cast<uint32_t>(rest);
    }
    return out;
  }
#else
  PDG_COLD void reorder_head(int32_t* qs, double* qc, uint32_t qh, int m) {
    const uint32_t mask = static_cast<uint32_t>(s_->C.qcap - 1);
    int32_t hs[8];
    double hc[8], wait[8];
    int pc[8];
    for (int k = 0; k < m; ++k) {
      hs[k] = qs[(qh + k) & mask];
      hc[k] = qc[(qh + k) & mask];
      const SessRt& s = GLP(s_->G.sess)[hs[k]];
      wait[k] = dsub(s_->now_, s.t_enq);
      pc[k] = s.postpone;
    }
    const double thres = s_->T.ttft_thres;
    int perm[8];
    for (int k = 0; k < m; ++k) perm[k] = k;
    const int id_sat = count_satisfied(perm, m, hc, wait, thres);
    if (id_sat == m) return;  // the identity already satisfies every task
    int64_t nperm = 1;
    for (int k = 2; k <= m; ++k) nperm *= k;
    int best_sat = id_sat;
    int64_t best_r = 0;
    for (int64_t r = 1 + lane_id(); r < nperm; r += PDG_NL) {
      unrank_perm(r, m, perm);
      bool allowed = true;
      for (int k = 0; k < m; ++k) {
        if (k > perm[k] && pc[perm[k]] >= s_->PR.window) {
          allowed = false;
          break;
        }
      }
      if (!allowed) continue;
      const int sat = count_satisfied(perm, m, hc, wait, thres);
      if (sat > best_sat) {  // per lane: smallest rank with a strict maximum
        best_sat = sat;
        best_r = r;
      }
    }
    for (int s = PDG_NL / 2; s > 0; s >>= 1) {
      const int os = shfl_i(best_sat, lane_id() ^ s);
      const int64_t orr = static_cast<int64_t>(shfl_u64(static_cast<uint64_t>(best_r), lane_id() ^ s));
      if (os > best_sat || (os == best_sat && orr < best_r)) {
        best_sat = os;
        best_r = orr;
      }
    }
    if (best_r == 0) return;
    unrank_perm(best_r, m, perm);
    {  // warp-uniform stores (every lane writes the same values)
      for (int k = 0; k < m; ++k) {
        const int p = perm[k];
        if (k > p) ++GLP(s_->G.sess)[hs[p]].postpone;
        qs[(qh + k) & mask] = hs[p];
        qc[(qh + k) & mask] = hc[p];
      }
    }
  }

#endif

  PDG_HD static int count_satisfied(const int* perm, int m, const double* hc, const double* wait, double thres) {
    double elapsed = 0.0;
    int sat = 0;
    for (int k = 0; k < m; ++k) {
      elapsed = dadd(elapsed, hc[perm[k]]);
      if (dadd(wait[perm[k]], elapsed) <= thres) ++sat;
    }
    return sat;
  }

  // ---- prefill workers (sim_engine.cpp:354-453) ----
  PDG_HD void enqueue_remote(int p, int32_t i, int32_t ctx, int32_t incr) {
    PrefillW& w = PW(p);
    const double cost = t_prefill(ctx, incr, w.deg);
    if (!queue_push(w.q, GLP(s_->G.pq_s) + static_cast<size_t>(p) * s_->C.qcap, GLP(s_->G.pq_c) + static_cast<size_t>(p) * s_->C.qcap, i, cost))
      return;
    try_stage(p);
    try_start_compute(p);
  }

    PDG_A_TRY_STAGE void try_stage(int p) {
    const int64_t t0_ = pb();
    try_stage_(p);
    pe(23, t0_);
  }
  PDG_HD void try_stage_(int p) {
    PrefillW& w = PW(p);
    if (w.staged || w.q.qh == w.q.qt) return;
    double cost;
    const int32_t stg = select_next(w.q, GLP(s_->G.pq_s) + static_cast<size_t>(p) * s_->C.qcap,
                                    GLP(s_->G.pq_c) + static_cast<size_t>(p) * s_->C.qcap, &cost);
    const int32_t hist = GLP(s_->G.sess)[stg].ctx;
    double ready = s_->now_;
    bool event = false;
    if (hist > 0) {
      // Lazy history read from the bound decode worker (sim_engine.cpp:368-383).
      const int dd = DW(GLP(s_->G.sess)[stg].bound).deg;
      ready = dadd(s_->now_, t_kv(hist, dd, w.deg));
      // The read's completion event only clears the pending flag and retries
      // the compute start (sim_engine.cpp:438-443). While the worker computes
      // until done >= ready, that retry is a no-op and the start happens at
      // done (on_prefill_done), where staged_ready <= now holds: the event is
      // not scheduled. (Sequence numbers of later events shift uniformly, so
      // their order is unchanged.)
      event = !(w.computing && s_->st_[slot_compute(p)] >= ready);
    }
    {  // warp-uniform stores (every lane writes the same values)
      w.stg = stg;
      w.stg_cost = cost;
      w.staged = 1;
      w.staged_ready = ready;
      w.pending = event ? 1 : 0;
    }
    if (event) set_slot(slot_history(p), ready, kKvTransferDone);
  }

  PDG_HD void try_start_compute(int p) {
    PrefillW& w = PW(p);
    if (w.computing || !w.staged || w.pending || w.staged_ready > s_->now_) return;
    const double done = dadd(s_->now_, w.stg_cost);
    {  // warp-uniform stores (every lane writes the same values)
      w.cur = w.stg;
      w.cur_cost = w.stg_cost;
      w.staged = 0;
      w.computing = 1;
    }
    set_slot(slot_compute(p), done, kPrefillDone);
    try_stage(p);  // the next task's history read overlaps this compute
  }

  PDG_HD void on_prefill_done(int p) {
    PrefillW& w = PW(p);
    const int32_t i = w.cur;
    w.computing = 0;  // warp-uniform store
    const int dd = DW(GLP(s_->G.sess)[i].bound).deg;
    heap_push(dadd(s_->now_, t_kv(l_incr_of(i), w.deg, dd)), kKvTransferDone, static_cast<uint32_t>(i),
              static_cast<uint32_t>(p));
    try_stage(p);
    try_start_compute(p);
  }

  PDG_HD void on_history_read(int p) {
    PW(p).pending = 0;  // warp-uniform store
    try_start_compute(p);
  }

  PDG_HD void on_writeback(int32_t i, int p) {
    const int d = GLP(s_->G.sess)[i].bound;
    complete_task(i, false, p, d);
    advance_decode(d);
  }

  // complete_task (sim_engine.cpp:458-484).
  PDG_A_COMPLETE_TASK void complete_task(int32_t i, bool local, int p, int d) {
    const int64_t t0 = pb();
    complete_task_(i, local, p, d);
    pe(kProfComplete, t0);
  }
  PDG_HD void complete_task_(int32_t i, bool local, int p, int d) {
    SessRt& s = GLP(s_->G.sess)[i];
    const int round = s.round;
    const SessTr st = sess_tr(i);
    const RoundTr rt = round_tr(s.roff + round - 1);
    const double created = round == 1 ? st.arrival : s.t_enq;
    const double value = dsub(s_->now_, created);
    if (!local) ttft_add(p, value);  // decode workers' TTFT windows are never queried
    if (kRec && s_->REC.ttft && lane_id() == 0) {
      pdsim_ttft_sample& o = s_->REC.ttft[s_->n_ttft_];
      o.session_id = GLP(s_->T.sid)[i];
      o.round = round;
      o.kind = round == 1 ? 0 : 1;
      o.local = local ? 1 : 0;
      o.reserved[0] = o.reserved[1] = 0;
      o.created_time = created;
      o.completion_time = s_->now_;
      o.value = value;
    }
    if (kRec && s_->C.rep_gapcap > 0) {  // report mode: TTFT value and in-order folds (metrics.cpp:152-161)
      const int64_t nt = s_->n_ttft_;
      if (nt < s_->C.rep_r && lane_id() == 0) GLP(s_->G.rep_ttft)[nt] = round == 1 ? value : -value;
      if (round == 1) {
        s_->rep_init_sum_ = dadd(s_->rep_init_sum_, value);
        ++s_->rep_n_init_;
      } else {
        s_->rep_incr_sum_ = dadd(s_->rep_incr_sum_, value);
        ++s_->rep_n_incr_;
      }
      if (local) ++s_->rep_n_local_;
    }
    ++s_->n_ttft_;
    const int32_t incr = rt.incr;
    const int32_t dec = rt.dec;
    DecodeW& w = DW(d);
    interrupt_run(d);
    const int32_t join = w.steps;  // first token in the next step started
    const uint64_t key =
        (static_cast<uint64_t>(static_cast<uint32_t>(join + dec - 1)) << 32) | static_cast<uint32_t>(st.rank);
    warp_sync();
    const int32_t hint = w.seg_end;
    if (kPrune) {
      const bool newly_bad = value > s_->T.ttft_thres && !s.ttft_bad;  // read by every lane before lane 0 writes
      warp_sync();
      if (newly_bad) s_->fails_ += 1;  // warp-uniform store
    }
    if ((!kLazy || kRec) && lane_id() == 0) GLP(s_->G.sess_cold)[i].seg_hint = hint;
    if (lane_id() == 0) {
      if (value > s_->T.ttft_thres) s.ttft_bad = 1;
      s.ctx += incr;
      s.join = join;
      if (kLazy) {
        s.next_pend = w.pend_head;
        w.pend_head = i;
      }
      w.kv_used += static_cast<int64_t>(incr) * PDG_PROF.kv_bytes_per_token;
      ++w.batch_n;
      ++w.n_new;
    }
    warp_sync();
    fh_push(d, key);
    ++s_->ctr_.tasks_completed;
  }

  // ---- decode workers (sim_engine.cpp:488-583) ----
  PDG_HD void enqueue_local(int d, int32_t i, int32_t ctx, int32_t incr) {
    DecodeW& w = DW(d);
    const double cost = t_prefill(ctx, incr, w.deg);
    if (!queue_push(w.q, GLP(s_->G.dq_s) + static_cast<size_t>(d) * s_->C.qcap, GLP(s_->G.dq_c) + static_cast<size_t>(d) * s_->C.qcap, i, cost))
      return;
    interrupt_run(d);
    advance_decode(d);
  }

  PDG_A_ADVANCE_DECODE void advance_decode(int d) {
    const int64_t t0 = pb();
    advance_decode_(d);
    pe(kProfAdvance, t0);
  }
  PDG_HD void advance_decode_(int d) {
    DecodeW& w = DW(d);
    if (w.stepping || w.prefilling) return;
    if (w.q.qh != w.q.qt) {
      // Local prefill preempts decoding until the queue drains.
      double cost;
      const int32_t cur = select_next(w.q, GLP(s_->G.dq_s) + static_cast<size_t>(d) * s_->C.qcap,
                                      GLP(s_->G.dq_c) + static_cast<size_t>(d) * s_->C.qcap, &cost);
      {  // warp-uniform stores (every lane writes the same values)
        w.cur = cur;
        w.cur_cost = cost;
        w.prefilling = 1;
      }
      set_slot(d, dadd(s_->now_, cost), kPrefillDone);
      return;
    }
    const int32_t batch = w.batch_n;
    if (batch > 0) {
      double dur = w.dur;
      if (w.dur_cohort != batch) dur = curve_eval(PDG_PROF.decode[w.deg], static_cast<double>(batch));
      const int32_t first = w.n_new;
      const int32_t steps = w.steps;  // index of the step starting now
      const double end = dadd(s_->now_, dur);
      if (kLazy) {  // stamp the end of this step on the rounds starting with it (their e_join)
        for (int32_t j = w.pend_head; j >= 0;) {
          SessRt& q = GLP(s_->G.sess)[j];
          const int32_t nx = q.next_pend;
          warp_sync();
          if (lane_id() == 0) q.e_join = end;
          j = nx;
        }
        w.pend_head = -1;
      }
      // Lazy mode: steps before the next round end of a batch member are
      // "silent" (no state outside this worker changes) and are advanced by
      // catch_up(); only the step where a member finishes is an event.
      int32_t b = steps;
      double b_end = end;
      if (kLazy && w.fh_n > 0) {
        const int32_t fin = static_cast<int32_t>(w.fh_top >> 32);
        if (fin > steps) {
          b = fin;
          b_end = fold_repeat(end, dur, static_cast<uint64_t>(fin - steps));
        }
      }
      // warp-uniform stores (every lane writes the same values)
      w.dur = dur;
      w.dur_cohort = batch;
      w.cohort_n = batch;
      w.first_n = first;
      w.n_new = 0;
      w.steps = steps + 1;
      w.stepping = 1;
      w.cur_end = end;
      w.run_b = b;
      set_slot(d, b_end, kDecodeStep);
    }
  }

  // ---- lazy decode stepping ----
  // Advances every decode worker's silent steps that end strictly before the
  // event about to run at time t. A silent step ending exactly at t comes
  // after an event of kind < 4 (kinds order equal-time events), so it stays
  // pending; against another decode step (kind 4) the order is the
  // scheduling order, which lazy steps do not carry: abort to exact mode.
  PDG_HD void catch_up(double t, uint32_t kind) {
    const int D = s_->PL.D;
    for (int base = 0; base < D; base += PDG_NL) {
      // lanes test their workers in parallel; only flagged workers advance
      const int mine = base + lane_id();
      bool need = false;
      if (mine < D) {
        const DecodeW& w = DW(mine);
        need = w.stepping && w.steps - 1 < w.run_b && w.cur_end <= t;
      }
      uint32_t m = ballot(need);
      while (m) {
        const int d = base + first_zero(~m);
        m &= m - 1;
        catch_up_worker(d, t, kind);
        if (s_->failed_ || s_->abort_) return;
      }
    }
  }

  PDG_A_CATCH_UP_WORKER void catch_up_worker(int d, double t, uint32_t kind) {
    const int64_t t0 = pb();
    catch_up_worker_(d, t, kind);
    pe(kProfCatchUp, t0);
  }
  PDG_HD void catch_up_worker_(int d, double t, uint32_t kind) {
    DecodeW& w = DW(d);
    const int64_t kvb = PDG_PROF.kv_bytes_per_token;
    if (kProf && !(w.stepping && w.steps - 1 < w.run_b && w.cur_end <= t)) pe(24, pdg_clock());
    while (w.stepping && w.steps - 1 < w.run_b) {
      const double e = w.cur_end;
      if (e > t) break;
      if (kProf) pe(26, pdg_clock());
      if (e == t) {
        if (kind == kDecodeStep) s_->abort_ = 1;
        break;
      }
      // The in-flight step k ends at e (a silent step: no member finishes).
      const int32_t k = w.steps - 1;
      const int32_t cohort = w.cohort_n;
      const double dur = w.dur;
      const double last = w.last_step_t;
      const int64_t kv = w.kv_used;
      const int64_t tokens = s_->ctr_.tokens_decoded;
      seg_append(d, k, 1, e, dsub(e, last), static_cast<uint32_t>(cohort - w.first_n));
      double end = e;
      int32_t done = 1;
      double next = dadd(e, dur);
      if (PDG_UNLIKELY(!(next > e))) {  // a zero-length step cannot be advanced lazily
        s_->abort_ = 1;
        return;
      }
      // Bulk: the following steps add exactly the same gap while the end
      // time stays in one binade; complete all of them that end before t.
      const int32_t room = w.run_b - (k + 1);
      const int64_t tb0_ = pb();
      if (room > 0 && next < t) {
        const double g = dsub(next, e);
        const int64_t ts0_ = pb();
        int64_t m = 0;
        double last_end = e, nxt = next;
        if (room <= kShortBulk) {
          // Short stretch: step explicitly while each end adds exactly g (two
          // fp64 ops a step, cheaper than the binade arithmetic).
          while (m < room && nxt < t && dsub(nxt, last_end) == g) {
            ++m;
            last_end = nxt;
            nxt = dadd(nxt, dur);
          }
        } else {
          m = stable_run(e, dur, g, t, room);
          if (m > 0) {
            last_end = dadd(next, dmul(static_cast<double>(m - 1), g));
            nxt = dadd(last_end, dur);
          }
        }
        pe(25, ts0_);
        if (m > 0) {
          seg_append(d, k + 1, static_cast<int32_t>(m), next, g, static_cast<uint32_t>(cohort));
          end = last_end;
          done += static_cast<int32_t>(m);
          next = nxt;
          if (PDG_UNLIKELY(!(next > end))) {
            s_->abort_ = 1;
            return;
          }
        }
      }
      pe(21, tb0_);
      // warp-uniform stores
      w.last_step_t = end;
      w.kv_used = kv + static_cast<int64_t>(cohort) * done * kvb;
      s_->ctr_.tokens_decoded = tokens + static_cast<int64_t>(cohort) * done;
      w.first_n = 0;  // no joins inside a run (a join ends the run)
      w.steps = k + 1 + done;
      w.cur_end = next;
      if (s_->failed_) return;
    }
  }



  // A join or a local prefill on a worker whose in-flight step is silent:
  // that step's end becomes an explicit event (its successor differs).
  PDG_HD void interrupt_run(int d) {
    DecodeW& w = DW(d);
    if (!kLazy || !w.stepping) return;
    catch_up_worker(d, s_->now_, s_->cur_kind_);
    const int32_t k = w.steps - 1;
    if (w.run_b <= k) return;
    const double end = w.cur_end;
    w.run_b = k;
    set_slot(d, end, kDecodeStep);
  }

  PDG_HD void on_local_prefill_done(int d) {
    DecodeW& w = DW(d);
    const int32_t i = w.cur;
    w.prefilling = 0;  // warp-uniform store
    complete_task(i, true, -1, d);
    advance_decode(d);
  }

  PDG_HD void on_decode_step(int d) {
    DecodeW& w = DW(d);
    if (kLazy) catch_up_worker(d, s_->now_, kDecodeStep);
    const int32_t k = w.steps - 1;  // index of the step that just ended
    const int32_t cohort = w.cohort_n;
    const int32_t n_itl = cohort - w.first_n;
    const double prev = w.last_step_t;
    const double now = s_->now_;
    const int64_t kv = w.kv_used;
    const int64_t tokens = s_->ctr_.tokens_decoded;
    seg_append(d, k, 1, now, dsub(now, prev), static_cast<uint32_t>(n_itl));
    if (kRec && s_->C.rep_gapcap > 0 && n_itl > 0) report_itl_step(dsub(now, prev), n_itl);
    if (kRec && s_->REC.steps) {
      const int64_t ns = s_->n_steps_;
      if (ns < s_->REC.steps_cap && lane_id() == 0) {
        StepRec& r = s_->REC.steps[ns];
        r.t = now;
        r.gap = dsub(now, prev);
        r.d = d;
        r.k = k;
      }
      s_->n_steps_ = ns + 1;  // warp-uniform store
    }
    // warp-uniform stores
    w.stepping = 0;
    w.last_step_t = now;
    w.kv_used = kv + static_cast<int64_t>(cohort) * PDG_PROF.kv_bytes_per_token;
    s_->ctr_.tokens_decoded = tokens + cohort;

    bool any_terminated = false;
    while (!s_->failed_ && w.fh_n > 0 && static_cast<int32_t>(w.fh_top >> 32) <= k) {
      if (PDG_UNLIKELY(static_cast<int32_t>(w.fh_top >> 32) < k)) {  // a round end was missed
        fail();
        return;
      }
      const int64_t tf0 = pb();
      const uint32_t rank = static_cast<uint32_t>(w.fh_top);
      fh_pop(d);
      const int32_t i = s_->T.rank_is_index ? static_cast<int32_t>(rank) : GLP(s_->T.by_rank)[rank];
      SessRt& s = GLP(s_->G.sess)[i];
      const RoundTr rt = round_tr(s.roff + s.round - 1);
      const int32_t dec = rt.dec;
      // This round's ITL samples, in token order (sim_engine.cpp:544-555).
      double ilo = s.itl_lo, ihi = s.itl_hi;
      if (!kLazy || (kRec && s_->exact_itl_)) {
        SessCold& c = GLP(s_->G.sess_cold)[i];
        const double sum = seg_fold(d, s.join + 1, k, c.itl_sum, c.seg_hint);
        warp_sync();
        c.itl_sum = sum;  // warp-uniform store
      } else if (dec > 1) {
        // ITL samples at steps join+1..k sum to within a relative u of
        // e_k - e_join (every sample is fl(e_j - e_{j-1})).
        const double now = s_->now_, ej = s.e_join;
        double rlo = mul_rd(sub_rd(now, ej), 1.0 - 0x1p-51);
        const double rhi = mul_ru(sub_ru(now, ej), 1.0 + 0x1p-51);
        if (rlo < 0.0) rlo = 0.0;
        ilo = add_rd(ilo, rlo);
        ihi = add_ru(ihi, rhi);
      }
      if (kRec && s_->REC.spans) {
        const int64_t nsp = s_->n_spans_;
        if (lane_id() == 0) {
          SpanRec& r = s_->REC.spans[nsp];
          r.sess = i;
          r.round = s.round;
          r.d = d;
          r.join = s.join;
          r.end = k;
          r.reserved = 0;
        }
        s_->n_spans_ = nsp + 1;  // warp-uniform store
      }
      const bool last = s.round == s.nround;
      {  // warp-uniform stores (every lane writes the same values)
        s.itl_lo = ilo;
        s.itl_hi = ihi;
        s.itl_cnt += dec - 1;
        s.ctx += dec;
        --w.batch_n;
      }
      if (last) {
        terminate_session(i, d);
        any_terminated = true;
      } else {
        heap_push(dadd(s_->now_, rt.delay), kInteractionDone, static_cast<uint32_t>(i), 0u);
      }
      pe(kProfFinisher, tf0);
    }
    if (any_terminated) admit_waiting();
    advance_decode(d);
  }

  PDG_HD void on_interaction_done(int32_t i) {
    SessRt& s = GLP(s_->G.sess)[i];
    const int round = s.round + 1;
    const int bound = s.bound;
    const int32_t ctx = s.ctx;
    const int32_t incr = round_tr(s.roff + round - 1).incr;
    s.round = static_cast<int16_t>(round);  // warp-uniform store
    start_round(i, round, bound, ctx, incr);
  }

  // terminate_session + slo_verdict (sim_engine.cpp:591-607, 668-674).
  PDG_COLD void terminate_session(int32_t i, int d) {
    SessRt& s = GLP(s_->G.sess)[i];
    const int32_t ctx = s.ctx;
    const int32_t cnt = s.itl_cnt;
    // the exact sequential fold exists only where the exact engine or the
    // records ran (SessCold); search mode decides on the bracket below
    const double mean_itl =
        (!kLazy || kRec) && cnt > 0 ? ddiv(GLP(s_->G.sess_cold)[i].itl_sum, static_cast<double>(cnt)) : 0.0;
    const bool ttft_ok = !s.ttft_bad;
    bool itl_ok;
    if (!kLazy || (kRec && s_->exact_itl_) || cnt == 0) {
      itl_ok = cnt == 0 || mean_itl <= s_->T.itl_thres;
    } else {
      // search mode: certified decision of fl(fold / cnt) <= itl_thres
      const int dec = mean_le_bracket(s.itl_lo, s.itl_hi, cnt, s_->T.itl_thres);
      if (PDG_UNLIKELY(dec < 0)) {  // inside the error band: replay this pair with exact folds
        s_->abort_ = 1;
        return;
      }
      itl_ok = dec == 1;
    }
    const bool slo_ok = ttft_ok && itl_ok;
    {  // warp-uniform stores (every lane writes the same values)
      DW(d).kv_used -= static_cast<int64_t>(ctx) * PDG_PROF.kv_bytes_per_token;
      if (kRec && s_->C.rep_gapcap > 0 && lane_id() == 0) {
        const SessTr st = sess_tr(i);
        GLP(s_->G.rep_e2e)[st.rank] = dsub(s_->now_, st.arrival);
      }
      if (kRec && s_->REC.sessions) {
        pdsim_session_outcome& o = s_->REC.sessions[s_->att_.sessions_completed];
        const double arrival = sess_tr(i).arrival;
        o.session_id = GLP(s_->T.sid)[i];
        o.arrival_time = arrival;
        o.completion_time = s_->now_;
        o.admission_wait = dsub(GLP(s_->G.sess_cold)[i].bind_time, arrival);
        o.mean_itl = mean_itl;
        o.rounds = s.nround;
        o.ttft_ok = ttft_ok;
        o.itl_ok = itl_ok;
        o.slo_ok = slo_ok;
        o.reserved = 0;
      }
    }
    ++s_->att_.sessions_completed;
    if (kPrune && ttft_ok && !itl_ok) s_->fails_ += 1;  // TTFT misses were counted when they happened
    s_->att_.slo_ok += slo_ok;
    s_->att_.ttft_ok += ttft_ok;
    s_->att_.itl_ok += itl_ok;
  }

  // ---- finisher heap (global): u64 keys (end_step << 32 | id rank) ----
    PDG_A_FH_PUSH void fh_push(int d, uint64_t key) {
    const int64_t t0_ = pb();
    fh_push_(d, key);
    pe(17, t0_);
  }
#if PDG_FH_ARITY == 32
  // A 32-ary min-heap: the children of entry i are 32i+1 .. 32i+32, so a pop
  // reads one level's children with one coalesced warp load and picks the
  // smallest with two REDUX.MIN — depth log32(n) instead of log2(n)
  // dependent loads. Keys are unique (one entry per session).
  PDG_HD void fh_push_(int d, uint64_t key) {
    DecodeW& w = DW(d);
    const int32_t n = w.fh_n;
    if (PDG_UNLIKELY(n >= s_->C.fcap)) {
      fail();
      return;
    }
    uint64_t* h = GLP(s_->G.fh) + static_cast<size_t>(d) * s_->C.fcap;
    const uint64_t top = w.fh_top;
    int32_t i = n;
    while (i > 0) {
      const int32_t par = (i - 1) >> 5;
      const uint64_t pv = h[par];
      if (pv <= key) break;
      warp_sync();
      if (lane_id() == 0) h[i] = pv;
      i = par;
    }
    warp_sync();
    if (lane_id() == 0) h[i] = key;
    // warp-uniform stores
    w.fh_n = n + 1;
    if (n == 0 || key < top) w.fh_top = key;
    warp_sync();
  }

#else
  PDG_HD void fh_push_(int d, uint64_t key) {
    DecodeW& w = DW(d);
    const int32_t n = w.fh_n;
    if (PDG_UNLIKELY(n >= s_->C.fcap)) {
      fail();
      return;
    }
    uint64_t* h = GLP(s_->G.fh) + static_cast<size_t>(d) * s_->C.fcap;
    const uint64_t top = w.fh_top;
    {  // warp-uniform stores (every lane writes the same values)
      int32_t i = n;
      while (i > 0) {
        const int32_t par = (i - 1) >> 1;
        const uint64_t pv = h[par];
        if (pv <= key) break;
        h[i] = pv;
        i = par;
      }
      h[i] = key;
      w.fh_n = n + 1;
      if (n == 0 || key < top) w.fh_top = key;
    }
  }

#endif
    PDG_A_FH_POP void fh_pop(int d) {
    const int64_t t0_ = pb();
    fh_pop_(d);
    pe(17, t0_);
  }
#if PDG_FH_ARITY == 32
  PDG_HD void fh_pop_(int d) {
    DecodeW& w = DW(d);
    uint64_t* h = GLP(s_->G.fh) + static_cast<size_t>(d) * s_->C.fcap;
    const int32_t n = w.fh_n - 1;
    const uint64_t last = h[n];
    int32_t i = 0;
    for (;;) {
      const int32_t c0 = 32 * i + 1;
      if (c0 >= n) break;
#if defined(__CUDA_ARCH__)
      const int32_t c = c0 + lane_id();
      const uint64_t v = c < n ? h[c] : ~0ull;
      const uint32_t hi = static_cast<uint32_t>(v >> 32);
      const uint32_t mhi = __reduce_min_sync(0xffffffffu, hi);
      const uint32_t mlo = __reduce_min_sync(0xffffffffu, hi == mhi ? static_cast<uint32_t>(v) : 0xffffffffu);
      const uint64_t m = (static_cast<uint64_t>(mhi) << 32) | mlo;
      if (m >= last) break;
      const int am = __ffs(__ballot_sync(0xffffffffu, v == m)) - 1;
#else
      uint64_t m = ~0ull;
      int am = 0;
      for (int k = 0; k < 32 && c0 + k < n; ++k) {
        if (h[c0 + k] < m) {
          m = h[c0 + k];
          am = k;
        }
      }
      if (m >= last) break;
#endif
      if (lane_id() == 0) h[i] = m;
      i = c0 + am;
    }
    warp_sync();
    if (n > 0 && lane_id() == 0) h[i] = last;
    warp_sync();
    // warp-uniform stores
    w.fh_n = n;
    w.fh_top = n > 0 ? h[0] : 0;
    warp_sync();
  }
#else
  PDG_HD void fh_pop_(int d) {
    DecodeW& w = DW(d);
    uint64_t* h = GLP(s_->G.fh) + static_cast<size_t>(d) * s_->C.fcap;
    {  // warp-uniform stores (every lane writes the same values)
      const int32_t n = w.fh_n - 1;
      const uint64_t last = h[n];
      int32_t i = 0;
      for (;;) {
        int32_t c = 2 * i + 1;
        if (c >= n) break;
        uint64_t cv = h[c];
        if (c + 1 < n) {
          const uint64_t cv2 = h[c + 1];
          if (cv2 < cv) {
            ++c;
            cv = cv2;
          }
        }
        if (cv >= last) break;
        h[i] = cv;
        i = c;
      }
      if (n > 0) h[i] = last;
      w.fh_n = n;
      w.fh_top = n > 0 ? h[0] : 0;
    }
  }
#endif


};

using Engine = EngineT<false>;  // host (test) build: pointer-based slot layout

#if defined(__CUDA_ARCH__)
#undef s_
#endif

}  // namespace pdg
