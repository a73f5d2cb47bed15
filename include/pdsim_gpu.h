/* pdsim_gpu.h — C-ABI of the B200 plan-search replay engine.
 *
 * This is the drop-in boundary for the reference simulator's hot path:
 *   SimResult pdsim::run(const Trace&, const DeploymentPlan&,
 *                        const PerfProfile&, const SchedulerParams&, uint64_t)
 *     (reference: proj/include/pdsim/sim_engine.hpp:125-127,
 *                 proj/src/sim_engine.cpp:676-681)
 * plus the batched candidate x trace-replica search that composes it with the
 * reference candidate enumerator (proj/src/planner.cpp:582-657) and SLO scoring
 * (proj/src/sim_engine.cpp:591-607, proj/src/metrics.cpp:171-186).
 *
 * Conventions
 *  - Plain C types only. No allocation crosses the ABI: every output buffer is
 *    caller-allocated. Device memory is owned by the context.
 *  - Every entry point returns a status code (PDSIM_OK or PDSIM_ERR_*). The
 *    error classes mirror the reference exception taxonomy
 *    (proj/include/pdsim/errors.hpp:25-46): ConfigError -> PDSIM_ERR_CONFIG,
 *    DomainError -> PDSIM_ERR_DOMAIN. No C++ exception crosses the ABI; the
 *    message is available from pdsim_gpu_last_error() (per context) or
 *    pdsim_last_error() (thread-local, for context-free calls).
 *  - A context is bound to one CUDA device. Calls on distinct contexts may run
 *    concurrently; calls on one context must be serialized by the caller.
 */
#ifndef PDSIM_GPU_H_
#define PDSIM_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDSIM_ABI_VERSION 3

#define PDSIM_MAX_DEGREES 8     /* profile degree set size */
#define PDSIM_MAX_BREAKPOINTS 7 /* per piecewise curve; segments = bps + 1 */
#define PDSIM_MAX_SEGMENTS (PDSIM_MAX_BREAKPOINTS + 1)
#define PDSIM_MAX_GROUPS 8      /* distinct degrees per phase in a plan */
#define PDSIM_MAX_WORKERS 64    /* prefill + decode replicas in one plan */

/* Status codes (errors.hpp:25-46 mapping). */
enum {
  PDSIM_OK = 0,
  PDSIM_ERR_CONFIG = 1,   /* pdsim::ConfigError */
  PDSIM_ERR_DOMAIN = 2,   /* pdsim::DomainError */
  PDSIM_ERR_CUDA = 3,     /* device / driver failure, or no usable device */
  PDSIM_ERR_INTERNAL = 4, /* engine invariant or capacity violated */
  PDSIM_ERR_PARSE = 5     /* pdsim::ParseError (document I/O helpers) */
};

/* RoutingMode (sim_engine.hpp:37-41). */
enum {
  PDSIM_ROUTING_ADAPTIVE = 0,
  PDSIM_ROUTING_ALWAYS_REMOTE = 1,
  PDSIM_ROUTING_ALWAYS_LOCAL = 2
};

/* RouteRationale (coordinator.hpp:27-33). */
enum {
  PDSIM_RATIONALE_SLACK_REMOTE = 0,
  PDSIM_RATIONALE_SLACK_LOCAL = 1,
  PDSIM_RATIONALE_ARGMIN = 2,
  PDSIM_RATIONALE_FORCED_REMOTE = 3,
  PDSIM_RATIONALE_FORCED_LOCAL = 4
};

/* Per-pair status in a search. */
enum {
  PDSIM_PAIR_OK = 0,
  PDSIM_PAIR_INVALID = 1, /* run() would throw ConfigError (e.g. KV precheck,
                             sim_engine.cpp:217-231); the candidate is invalid */
  PDSIM_PAIR_ERROR = 2,   /* engine capacity/invariant failure (never expected) */
  PDSIM_PAIR_PRUNED = 3   /* search mode "argmax": stopped once it could no longer win */
};

/* ---- inputs --------------------------------------------------------------- */

/* PiecewiseAlphaBeta (perf_model.hpp:48-74): segment i covers
 * [bp[i-1], bp[i]); a load exactly on a breakpoint belongs to the right
 * segment. eval(load) = alpha[i] + beta[i] * load, separately rounded. */
typedef struct pdsim_curve {
  int32_t n_breakpoints; /* 0..PDSIM_MAX_BREAKPOINTS */
  int32_t reserved;
  double breakpoints[PDSIM_MAX_BREAKPOINTS];
  double alpha[PDSIM_MAX_SEGMENTS];
  double beta[PDSIM_MAX_SEGMENTS];
} pdsim_curve;

/* PerfProfile (perf_model.hpp:76-91). Tables are indexed by the position of a
 * degree in `degrees` (ascending); kv[src][dst]. */
typedef struct pdsim_profile {
  int32_t n_degrees;
  int32_t degrees[PDSIM_MAX_DEGREES];
  int32_t reserved;
  pdsim_curve prefill[PDSIM_MAX_DEGREES];
  pdsim_curve decode[PDSIM_MAX_DEGREES];
  pdsim_curve kv[PDSIM_MAX_DEGREES][PDSIM_MAX_DEGREES];
  int64_t kv_bytes_per_token;
  int64_t gpu_memory_capacity;
  double history_weight;
} pdsim_profile;

/* Trace (workload.hpp:28-62) as a structure of arrays. Round r of session i
 * is element round_offset[i] + r. Caller-owned, read-only for the call. */
typedef struct pdsim_trace {
  int64_t n_sessions;
  int64_t n_rounds;                 /* == round_offset[n_sessions] */
  const int64_t* session_id;        /* [n_sessions] */
  const double* arrival_time;       /* [n_sessions], non-decreasing */
  const int64_t* round_offset;      /* [n_sessions + 1], round_offset[0] == 0 */
  const int64_t* incr_input_len;    /* [n_rounds] */
  const int64_t* decode_len;        /* [n_rounds] */
  const double* interaction_delay;  /* [n_rounds] */
  double ttft_thres;                /* SloSpec (workload.hpp:46-50) */
  double itl_thres;
} pdsim_trace;

/* DeploymentPlan (planner.hpp:36-53): replica groups in ascending degree
 * order (std::map iteration order). Worker ids: prefill replicas 0..P-1 in
 * group order, decode replicas P..P+D-1 (sim_engine.cpp:175-203). */
typedef struct pdsim_plan {
  int32_t n_prefill_groups;
  int32_t n_decode_groups;
  int32_t prefill_degree[PDSIM_MAX_GROUPS];
  int32_t prefill_count[PDSIM_MAX_GROUPS];
  int32_t decode_degree[PDSIM_MAX_GROUPS];
  int32_t decode_count[PDSIM_MAX_GROUPS];
} pdsim_plan;

/* SchedulerParams (sim_engine.hpp:46-54). */
typedef struct pdsim_sched_params {
  int32_t routing;  /* PDSIM_ROUTING_* */
  int32_t reorder;  /* bool */
  double alpha;
  double beta;
  int32_t window;
  int32_t reserved;
  double stat_window;
} pdsim_sched_params;

/* ---- outputs -------------------------------------------------------------- */

/* DecisionRecord (sim_engine.hpp:86-94). */
typedef struct pdsim_decision {
  double time;
  int64_t session_id;
  int32_t round;
  int32_t worker;
  int8_t local;
  int8_t rationale;
  int8_t has_estimate;
  int8_t reserved[5];
  double estimated_cost;
} pdsim_decision;

/* TtftSample (sim_engine.hpp:56-64). kind: 0 initial, 1 incremental. */
typedef struct pdsim_ttft_sample {
  int64_t session_id;
  int32_t round;
  int8_t kind;
  int8_t local;
  int8_t reserved[2];
  double created_time;
  double completion_time;
  double value;
} pdsim_ttft_sample;

/* SessionOutcome (sim_engine.hpp:74-84). */
typedef struct pdsim_session_outcome {
  int64_t session_id;
  double arrival_time;
  double completion_time;
  double admission_wait;
  double mean_itl;
  int32_t rounds;
  int8_t ttft_ok;
  int8_t itl_ok;
  int8_t slo_ok;
  int8_t reserved;
} pdsim_session_outcome;

/* SimCounters (sim_engine.hpp:96-103). */
typedef struct pdsim_counters {
  int64_t tasks_created;
  int64_t tasks_completed;
  int64_t tokens_decoded;
  int64_t kv_bytes_residual;
  int32_t max_postpone_observed;
  int32_t events_in_order;
} pdsim_counters;

/* Attainment numerators and denominator (metrics.cpp:171-186). */
typedef struct pdsim_attainment {
  int64_t sessions_total;
  int64_t sessions_completed;
  int64_t slo_ok;
  int64_t ttft_ok;
  int64_t itl_ok;
} pdsim_attainment;

/* Output of one replay (the SimResult of run()). Record arrays are optional
 * (NULL to skip); when given they must hold n_rounds decisions / TTFT samples
 * and n_sessions outcomes. Decisions and TTFT samples come in the reference
 * push order; sessions are sorted by session id (sim_engine.cpp:165-168). */
/* ItlSample (sim_engine.hpp:66-72). */
typedef struct pdsim_itl_sample {
  int64_t session_id;
  int32_t round;        /* 1-based */
  int32_t token_index;  /* position within the round (>= 2) */
  double completion_time;
  double value;
} pdsim_itl_sample;

typedef struct pdsim_run_output {
  pdsim_decision* decisions;
  pdsim_ttft_sample* ttft_samples;
  pdsim_session_outcome* sessions;
  int64_t n_decisions;   /* out */
  int64_t n_ttft;        /* out */
  int64_t n_sessions;    /* out: completed sessions */
  pdsim_counters counters;     /* out */
  pdsim_attainment attainment; /* out */
  /* Optional per-token ITL samples in the reference's push order
   * (sim_engine.cpp:536-556): NULL skips them. At most itl_capacity are
   * written; n_itl is the total (sum over rounds of decode_len - 1 bounds it). */
  pdsim_itl_sample* itl_samples;
  int64_t itl_capacity;
  int64_t n_itl;         /* out */
} pdsim_run_output;

/* Batched search: pairs are (candidate c, trace replica r), pair index
 * p = c * n_traces + r. Only pairs in [pair_begin, pair_end) are replayed
 * (the shard of this device); pair_end < 0 means all pairs. */
typedef struct pdsim_search_input {
  int32_t n_traces;
  int32_t n_candidates;
  const pdsim_trace* traces;     /* [n_traces] */
  const pdsim_plan* candidates;  /* [n_candidates] */
  int64_t pair_begin;
  int64_t pair_end;
} pdsim_search_input;

/* Search results. Arrays are caller-allocated; any may be NULL.
 *  pair_attainment / pair_counters / pair_status: [pair_end - pair_begin].
 *  candidate_slo_ok: [n_candidates], sum of slo_ok over this call's pairs;
 *    -1 for a candidate with any invalid pair in this call.
 * best_candidate = argmax candidate_slo_ok, ties -> smallest index (-1 when no
 * candidate is valid). Timings are device (CUDA event) milliseconds. */
/* MetricStat / Report (metrics.hpp:32-51): build_report (metrics.cpp:138-190)
 * of one replay — in-order means, nearest-rank P95s, attainment ratios. */
typedef struct pdsim_metric_stat {
  double mean;
  double p95;
  int64_t count;
} pdsim_metric_stat;

typedef struct pdsim_report {
  int64_t sessions_total;
  int64_t sessions_completed;
  double slo_attainment;
  double ttft_attainment;
  double itl_attainment;
  pdsim_metric_stat ttft_initial;
  pdsim_metric_stat ttft_incremental;
  pdsim_metric_stat itl;
  double e2e_mean;
  double local_fraction;
  int32_t empty;
  int32_t reserved;
} pdsim_report;

typedef struct pdsim_search_output {
  pdsim_attainment* pair_attainment;
  pdsim_counters* pair_counters;
  int8_t* pair_status;
  int64_t* candidate_slo_ok;
  int64_t* pair_events;   /* diagnostics: dynamic events replayed per pair */
  int64_t* pair_cycles;   /* diagnostics: SM clock ticks spent per pair */
  int32_t best_candidate;
  int32_t reserved;
  int64_t best_slo_ok;
  double kernel_ms;     /* replay kernel(s) only */
  double device_ms;     /* whole device-side search incl. reductions */
  int64_t kernel_launches;
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  /* Optional per-pair Report (NULL: attainment only). Requesting it replays
   * every decode step as an event (in-order ITL folds) and keeps per-pair
   * TTFT values, e2e latencies and an ITL gap histogram on the device; the
   * report is reduced on the device right after each replay. */
  pdsim_report* pair_report;
} pdsim_search_output;

/* ---- context -------------------------------------------------------------- */

typedef struct pdsim_gpu_ctx pdsim_gpu_ctx;

int pdsim_abi_version(void);
const char* pdsim_last_error(void); /* thread-local message of the last failure */

/* Creates a context on CUDA device `device`. Fails with PDSIM_ERR_CUDA when no
 * sm_100 device is present: there is no CPU fallback. */
int pdsim_gpu_create(int device, pdsim_gpu_ctx** out);
void pdsim_gpu_destroy(pdsim_gpu_ctx* ctx);
const char* pdsim_gpu_last_error(const pdsim_gpu_ctx* ctx);
/* Launch subsequent work on this cudaStream_t (NULL = the context's own). */
int pdsim_gpu_set_stream(pdsim_gpu_ctx* ctx, void* cuda_stream);

/* Drop-in for pdsim::run (sim_engine.hpp:125-127): one replay, full records. */
int pdsim_gpu_run(pdsim_gpu_ctx* ctx, const pdsim_trace* trace,
                  const pdsim_plan* plan, const pdsim_profile* profile,
                  const pdsim_sched_params* params, uint64_t seed,
                  pdsim_run_output* out);

/* Batched replay search: host inputs, host outputs (H2D + kernels + D2H). */
int pdsim_gpu_plan_search(pdsim_gpu_ctx* ctx, const pdsim_search_input* in,
                          const pdsim_profile* profile,
                          const pdsim_sched_params* params, uint64_t seed,
                          pdsim_search_output* out);

/* Batched `pdsim sweep` (pdsim.cpp:501-590): one plan replayed on n_traces
 * traces (the sweep's one trace per arrival rate) under n_settings scheduler
 * settings (its alpha x beta x window grid, any order). Candidates are the
 * settings: pair p = k * n_traces + r is setting k on trace r, and every
 * per-pair / per-candidate output of pdsim_search_output is indexed that way
 * (pair_report gives the sweep.csv row of each combination; best_candidate is
 * the setting with the most slo_ok sessions over the traces). Every setting
 * is validated against every trace before launch (ConfigError, as the
 * reference's first failing combination would throw). The settings stay
 * staged for pdsim_gpu_search_staged(). */
int pdsim_gpu_sweep(pdsim_gpu_ctx* ctx, int32_t n_traces, const pdsim_trace* traces,
                    const pdsim_plan* plan, int32_t n_settings,
                    const pdsim_sched_params* settings, const pdsim_profile* profile,
                    uint64_t seed, pdsim_search_output* out);

/* Resident variant: pdsim_gpu_stage() copies traces + candidates into HBM
 * once; pdsim_gpu_search_staged() replays them with inputs already resident
 * (outputs still land in caller host buffers). */
int pdsim_gpu_stage(pdsim_gpu_ctx* ctx, const pdsim_search_input* in,
                    const pdsim_profile* profile,
                    const pdsim_sched_params* params);
int pdsim_gpu_search_staged(pdsim_gpu_ctx* ctx, int64_t pair_begin,
                            int64_t pair_end, uint64_t seed,
                            pdsim_search_output* out);

/* Diagnostics: per-phase SM-cycle instrumentation of the replay kernel,
 * PDSIM_PROF_BUCKETS buckets summed over the pairs of the last search.
 * Exclusive handler phases: 0 event selection, 1 arrival, 2 interaction done,
 * 3 write-back, 4 decode step, 5 local prefill done, 6 prefill compute done,
 * 7 history read. Inclusive sub-scopes (nested inside the phases): 8 routing
 * decision, 9 task enqueue, 10 lazy decode catch-up, 11 finishing-member
 * fold, 12 advance_decode, 13 complete_task, 14 session-event heap,
 * 15 queue dequeue (reorder), 16 step-log append, 17 finisher heap,
 * 18 TTFT window add, 19 ITL slack test, 20 TTFT slack test, 21 bulk silent
 * steps, 22 per-round ITL sum, 23 prefill staging, 24 catch-up calls with
 * nothing to do (count), 25 stable_run, 26 catch-up iterations (count),
 * 27 admission catch-up over all decode workers. `replayed` counts pairs
 * whose fast attempt was replayed in exact mode. */
#define PDSIM_PROF_BUCKETS 28

/* Search modes. FULL (default) replays every pair to completion: every
 * per-pair and per-candidate output is exact. ARGMAX stops a candidate's
 * replays once it provably cannot be the argmax (SURVEY.md §8(e) pruning):
 * its upper bound — the sessions of all its replicas minus those already
 * known to miss the SLO (a TTFT over threshold is final; an ITL miss is known
 * at session end) — is below the incumbent's lower bound (slo_ok summed over
 * the incumbent's completed replicas), or equal with a larger enumeration
 * index. best_candidate and best_slo_ok are identical to FULL mode; pruned
 * pairs report PDSIM_PAIR_PRUNED and pruned candidates candidate_slo_ok = -2.
 * Record/report searches always run FULL. Sharded callers reduce
 * candidate_slo_ok with the same rule as invalid candidates (any negative
 * excludes the candidate): the global argmax is never pruned on any shard,
 * PROVIDED the upper bound counts the sessions of the whole search — a shard
 * that stages only some replicas must declare the global total with
 * pdsim_gpu_set_global_sessions(), or it would prune a candidate that merely
 * loses on its own replicas. */
enum { PDSIM_SEARCH_FULL = 0, PDSIM_SEARCH_ARGMAX = 1 };
int pdsim_gpu_set_search_mode(pdsim_gpu_ctx* ctx, int mode);
/* Kernel build of attainment-only searches (both builds compile the same
 * engine source and return identical results). LATENCY inlines every hot
 * subroutine (fewest instructions per event: few pairs per SM); THROUGHPUT
 * keeps the subroutines shared by several handlers out of line (smaller
 * instruction footprint: many warps per SM, where instruction fetch binds,
 * DESIGN.md §3.1). AUTO (default): THROUGHPUT when a launch replays more than
 * 4 pairs per SM. Record, report and diagnostics searches use LATENCY. */
enum { PDSIM_BUILD_AUTO = 0, PDSIM_BUILD_LATENCY = 1, PDSIM_BUILD_THROUGHPUT = 2 };
int pdsim_gpu_set_kernel_build(pdsim_gpu_ctx* ctx, int build);
/* Build the context's last replay launch used (LATENCY or THROUGHPUT; 0 before any). */
int pdsim_gpu_last_kernel_build(const pdsim_gpu_ctx* ctx);
/* Sessions of every replica of the search this context is a shard of (0 =
 * the staged replicas are the whole search). Used only by ARGMAX bounds. */
int pdsim_gpu_set_global_sessions(pdsim_gpu_ctx* ctx, int64_t total_sessions);

/* ---- multi-GPU (replaces the reference's serial sweep
 * loop pdsim.cpp:547-586 over run() calls, sim_engine.cpp:676-681) -------- */

/* Cost-aware shard of the pairs c * n_traces + r over `world` GPUs: pair cost
 * rounds(r) x (workers(c) + 2), longest first, each to the least-loaded rank
 * (deterministic; every rank computes the same split without communicating).
 * Writes rank's pairs in queue order (heaviest first) to out[0..capacity) and
 * returns their count (-1 on bad arguments). */
int64_t pdsim_shard_pairs(int32_t n_traces, const int64_t* trace_rounds,
                          int32_t n_candidates, const pdsim_plan* candidates,
                          int32_t world, int32_t rank, int64_t* out,
                          int64_t capacity);

/* Replays the staged pairs listed in `pairs` (global indices, no duplicates)
 * in list order: the persistent kernel's queue hands them out in that order
 * (with more than 8 pairs per SM, per-SM queues keep the pairs of one
 * candidate together on an SM, list order kept within a candidate).
 * Per-pair outputs follow the list; per-candidate outputs cover the pairs
 * replayed (or, with a communicator, the whole sharded search). */
int pdsim_gpu_search_staged_list(pdsim_gpu_ctx* ctx, const int64_t* pairs,
                                 int64_t n_pairs, uint64_t seed,
                                 pdsim_search_output* out);

/* NCCL (loaded at first use from the process's libnccl.so.2). One process per
 * GPU: rank 0 calls pdsim_nccl_unique_id(), the caller broadcasts the 128
 * bytes, every rank calls pdsim_gpu_comm_init(). From then on every search
 * of the context ends with the only collective of the path: an in-place
 * ncclAllReduce of the per-candidate counts (sum, uint64) and flags (max)
 * on the search's stream, then the argmax — candidate_slo_ok, best_candidate
 * and best_slo_ok describe the whole sharded search on every rank. */
int pdsim_nccl_unique_id(uint8_t id[128]);
int pdsim_gpu_comm_init(pdsim_gpu_ctx* ctx, int32_t world, int32_t rank,
                        const uint8_t id[128]);

/* One host thread driving several GPUs of this process: stages the whole
 * search on every device, shards it with pdsim_shard_pairs, replays the
 * shards concurrently and all-reduces the counts over a communicator made by
 * ncclCommInitAll. Outputs are indexed by global pair like
 * pdsim_gpu_plan_search (the pair range must be the whole search);
 * kernel_ms / device_ms are the maximum over devices. */
int pdsim_multi_plan_search(int32_t n_devices, const int32_t* devices,
                            const pdsim_search_input* in,
                            const pdsim_profile* profile,
                            const pdsim_sched_params* params, uint64_t seed,
                            int32_t search_mode, pdsim_search_output* out);
int pdsim_gpu_set_profiling(pdsim_gpu_ctx* ctx, int enable);
int pdsim_gpu_profile_counters(const pdsim_gpu_ctx* ctx, int64_t* cycles, int64_t* counts,
                               int64_t* replayed);

/* ---- host-side helpers (reference generators; host C++, libm) ------------ */

/* SynthProfileSpec (perf_model.hpp:110-139). */
typedef struct pdsim_synth_spec {
  int32_t n_degrees;
  int32_t degrees[PDSIM_MAX_DEGREES];
  int32_t n_prefill_breakpoints;
  int32_t n_decode_breakpoints;
  double prefill_alpha_min, prefill_alpha_max;
  double prefill_beta_min, prefill_beta_max;
  double prefill_breakpoints[PDSIM_MAX_BREAKPOINTS];
  double decode_alpha_min, decode_alpha_max;
  double decode_beta_min, decode_beta_max;
  double decode_breakpoints[PDSIM_MAX_BREAKPOINTS];
  double segment_growth_min, segment_growth_max;
  double scaling_exponent;
  double kv_bandwidth_bytes_per_sec;
  double kv_latency_seconds;
  double kv_reshard_penalty;
  int64_t kv_bytes_per_token;
  int64_t gpu_memory_capacity;
  double history_weight;
} pdsim_synth_spec;

/* TraceStats (workload.hpp:66-76); name is informational. */
typedef struct pdsim_trace_stats {
  double mean_rounds;
  int32_t fixed_rounds;
  int32_t reserved;
  double mean_prefill_len;
  double mean_decode_len;
  double length_cv;
  double first_round_fraction;
  double mean_interaction_delay;
  double ttft_thres;
  double itl_thres;
} pdsim_trace_stats;

/* Owned trace produced by the generator. */
typedef struct pdsim_trace_buf pdsim_trace_buf;

void pdsim_synth_spec_default(pdsim_synth_spec* spec);
int pdsim_synth_profile(const pdsim_synth_spec* spec, uint64_t seed,
                        pdsim_profile* out);
int pdsim_profile_validate(const pdsim_profile* profile);
int pdsim_preset_stats(const char* name, pdsim_trace_stats* out);
int pdsim_gen_trace(const pdsim_trace_stats* stats, double arrival_rate,
                    int32_t num_sessions, uint64_t seed, pdsim_trace_buf** out);
/* Batched gen_trace on all host threads: trace k is
 * gen_trace(stats, rates[k], num_sessions, seeds[k]), bit-identical to n
 * separate calls. out[k] receives an owned buffer (free each with
 * pdsim_trace_buf_free); on error every out[k] is NULL and the first failing
 * k's status is returned. */
int pdsim_gen_trace_batch(const pdsim_trace_stats* stats, int32_t n, const double* rates, int32_t num_sessions,
                          const uint64_t* seeds, pdsim_trace_buf** out);
/* Fills a view whose arrays stay owned by `buf`. */
int pdsim_trace_buf_view(const pdsim_trace_buf* buf, pdsim_trace* view);
void pdsim_trace_buf_free(pdsim_trace_buf* buf);
int pdsim_trace_validate(const pdsim_trace* trace);

/* Candidate enumeration in the reference order (planner.cpp:582-601,
 * 625-655): every (x, y) degree->count map with x, y non-empty and
 * sum(degree * count) <= total_gpus. Returns the count; writes up to
 * `capacity` plans into `out` (may be NULL to query the count). */
int64_t pdsim_enumerate_plans(const int32_t* degrees, int32_t n_degrees,
                              int32_t total_gpus, pdsim_plan* out,
                              int64_t capacity);

/* ---- surrogate planner -------------------------------- */

/* PhaseSimResult (planner.hpp:62-66); status is PDSIM_OK or the error the
 * reference would throw (PDSIM_ERR_CONFIG: no prefill tasks / no sessions /
 * no inter-token samples). */
typedef struct pdsim_phase_result {
  double p95;
  int64_t sample_count;
  int32_t infeasible;
  int32_t status;
} pdsim_phase_result;

/* Batched single-replica phase simulations on the device, one CTA per job:
 * job k = simulate_prefill_replica(traces[k], profile, degrees[k])
 * (planner.cpp:75-104) and simulate_decode_replica(traces[k], profile,
 * degrees[k]) (planner.cpp:106-226). A degree missing from the profile is a
 * PDSIM_ERR_DOMAIN for the whole call (t_prefill/t_decode, perf_model.cpp
 * :158-188). */
int pdsim_gpu_phase_sims(pdsim_gpu_ctx* ctx, int32_t n_jobs, const pdsim_trace* traces,
                         const int32_t* degrees, const pdsim_profile* profile,
                         pdsim_phase_result* prefill, pdsim_phase_result* decode);

/* LatencyCoefficients (planner.hpp:55-60) over the sorted unique degree list:
 * degree i is feasible for a phase when infeasible_* [i] == 0 (tau_* [i] is
 * then its P95 coefficient). */
typedef struct pdsim_coefficients {
  int32_t n_degrees;
  int32_t degrees[PDSIM_MAX_DEGREES];
  int32_t reserved;
  double tau_pre[PDSIM_MAX_DEGREES];
  double tau_dec[PDSIM_MAX_DEGREES];
  int8_t infeasible_pre[PDSIM_MAX_DEGREES];
  int8_t infeasible_dec[PDSIM_MAX_DEGREES];
} pdsim_coefficients;

/* estimate_coefficients (planner.cpp:228-283) for n_sets (rate, seed)
 * settings in ONE device launch: for set s and degree n the host generates
 * gen_trace(stats, rates[s] * n / total_gpus, 256, seeds[s] + 0x9E37...15 * n)
 * with the reference RNG, and both phase sims of every (set, degree) run on
 * the GPU. set_status[s] is the first error the reference would throw for
 * set s (PDSIM_OK otherwise); argument errors fail the whole call. */
int pdsim_gpu_estimate_coefficients(pdsim_gpu_ctx* ctx, const pdsim_trace_stats* stats, int32_t n_sets,
                                    const double* rates, const uint64_t* seeds, const pdsim_profile* profile,
                                    const int32_t* degrees, int32_t n_degrees, int32_t total_gpus,
                                    pdsim_coefficients* out, int32_t* set_status);

/* solve (planner.cpp:482-578), host C++: the exact min-Z assignment with the
 * reference tie-break chain. plan/objective_z/gpus_used are written when
 * *feasible is 1. Errors: PDSIM_ERR_CONFIG as check_coefficients/solve. */
int pdsim_solve(const pdsim_coefficients* coeffs, int32_t total_gpus, pdsim_plan* plan, double* objective_z,
                int32_t* gpus_used, int32_t* feasible);

/* top_k (planner.cpp:605-657), host C++: the k best plans in solve order.
 * Returns the number written (<= k) or -1 on error (pdsim_last_error). */
int64_t pdsim_top_k(const pdsim_coefficients* coeffs, int32_t total_gpus, int32_t k, pdsim_plan* plans,
                    double* objective_z, int32_t* gpus_used);

/* std::to_chars(double) shortest round-trip text: the reference's CSV number
 * format (metrics.cpp:32-36; fmt_double, pdsim.cpp:84-88). Writes the text
 * NUL-terminated; returns its length, or -1 when `cap` is too small. */
int32_t pdsim_format_double(double value, char* buf, int32_t cap);

/* Device-free CPU argmax helper used by multi-rank callers after the NCCL
 * reduction: max count, ties -> smallest index, negative = invalid. */
int32_t pdsim_argmax_candidates(const int64_t* candidate_slo_ok,
                                int32_t n_candidates);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* PDSIM_GPU_H_ */
