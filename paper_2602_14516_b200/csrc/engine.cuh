// engine.cuh — the replay of one (candidate plan, trace replica) pair.
//
// Behavioural restatement, for B200, of the reference discrete-event engine
// (proj/src/sim_engine.cpp:107-632) together with the routing
// (proj/src/coordinator.cpp:27-171) and reordering (proj/src/reorder.cpp:44-146)
// policies it calls. Every observable — routing decisions, TTFT samples,
// session verdicts, counters — is reproduced bit-for-bit; the data structures
// are re-designed for a GPU:
//  * a task is identified by its session (each session has at most one task
//    in flight), so queues and events carry 32-bit session indices;
//  * the admission queue is the index range [adm_head, next_arrival) because
//    sessions park in arrival order (sim_engine.cpp:240-267);
//  * arrivals are not heap events: they are read in trace order and merged
//    with the dynamic-event heap (kind 0 wins ties, sim_engine.cpp:48-74);
//  * decode batches are never materialised: a session in the batch finishes
//    its round at step join + decode_len - 1, so a per-worker min-heap keyed
//    by (end_step, session-id rank) yields exactly the finishing cohort
//    members in cohort order (sim_engine.cpp:514-517, 536-577) at O(log n)
//    per round instead of O(batch) per token;
//  * per-session ITL sums are folded at round end from a ring of step end
//    times (every ITL gap of a step equals now - previous step end);
//  * the ITL window keeps one (time, gap, count) run per step and folds it
//    with fold_repeat() (fold.cuh), exact to the last bit.
// The same source is compiled for the GPU (the product) and, in tests only,
// for the host so the engine logic can be checked without a device.
#pragma once

#include "common.cuh"
#include "exactsum.cuh"
#include "fold.cuh"

namespace pdg {

enum EventKind : uint32_t {
  kArrival = 0,
  kInteractionDone = 1,
  kKvTransferDone = 2,
  kPrefillDone = 3,
  kDecodeStep = 4,
};

struct Event {
  double t;
  uint64_t key;  // kind << 56 | seq  (sim_engine.cpp:68-74 total order)
  uint32_t a;    // session index or worker id
  uint32_t b;    // writeback: session index | 1<<31 ; history read: 0
};

PDG_HD bool ev_less(const Event& x, const Event& y) {
  return x.t < y.t || (x.t == y.t && x.key < y.key);
}

// Packed read-only trace (one per replica, shared by all candidates).
struct DevTrace {
  int32_t S;
  int32_t R;
  int32_t max_dec;
  int32_t reserved;
  double ttft_thres;
  double itl_thres;
  const double* arrival;     // [S]
  const int32_t* round_off;  // [S+1]
  const int32_t* incr;       // [R]
  const int32_t* dec;        // [R]
  const double* delay;       // [R]
  const int64_t* sid;        // [S]
  const int32_t* rank;       // [S] rank of session_id among all ids
  const int32_t* by_rank;    // [S] inverse of rank
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

// Per-session runtime state (SessionRt + the one PrefillTask in flight).
struct SessRt {
  double t_enq;      // enqueue time of the current task (== created for r >= 2)
  double itl_sum;    // sequential fold of this session's ITL samples
  double bind_time;  // admission time
  int32_t itl_cnt;
  int32_t join;      // step index at which the current round joined the batch
  int32_t ctx;       // context_len
  int16_t round;     // 1-based current round
  int8_t bound;      // decode worker index
  int8_t postpone;   // PrefillTask::postpone_count
  int8_t ttft_bad;   // some TTFT > threshold
  int8_t reserved[7];
};

// A worker's task queue: ring counters + exact sum of the queued costs.
struct TaskQueue {
  ExactSum sum;
  uint32_t qh, qt;
  uint32_t reserved[2];
};

struct PrefillW {
  TaskQueue q;
  ExactSum tw;      // exact sum of the TTFT window
  int32_t deg;
  int32_t cur, stg;
  uint32_t th, tt;  // TTFT window ring counters
  int8_t computing, staged, pending, reserved;
  double cur_cost, stg_cost;
  double staged_ready;
};

struct DecodeW {
  TaskQueue q;      // local prefill queue
  ExactSum iw;      // exact sum of the ITL window (terms = samples)
  int32_t deg;
  int32_t cur;
  double cur_cost;
  int64_t kv_used;
  int64_t kv_cap;
  int8_t stepping, prefilling, reserved[2];
  int32_t batch_n, n_new, cohort_n, first_n;
  int32_t steps;  // steps started
  int32_t fh_n;   // finisher-heap size
  uint32_t ih, it;  // ITL-run ring counters
};

// Capacities of one workspace slot (host-computed upper bounds).
struct Caps {
  int32_t S;      // sessions
  int32_t hcap;   // event heap
  int32_t qcap;   // per-worker task queue (power of 2)
  int32_t fcap;   // per-decode-worker finisher heap
  int32_t twcap;  // TTFT window ring (power of 2)
  int32_t iwcap;  // ITL-run ring (power of 2)
  int32_t lcap;   // step-log ring (power of 2)
  int32_t pmax;
  int32_t dmax;
  int32_t reserved;
};

// Pointers into one workspace slot.
struct Slot {
  SessRt* sess;
  Event* heap;
  uint64_t* mt;
  PrefillW* pw;
  DecodeW* dw;
  int32_t* pq_s;
  double* pq_c;
  double* tw_t;
  double* tw_v;
  int32_t* dq_s;
  double* dq_c;
  uint64_t* fh;
  double* slog;
  double* iw_t;
  double* iw_g;
  uint32_t* iw_c;
};

PDG_HD size_t align_up(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// Bytes of one slot and the carving of a base pointer into a Slot.
PDG_HD size_t slot_bytes(const Caps& c, Slot* s, char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + off : nullptr;
    off = align_up(off + bytes);
    return p;
  };
  const size_t P = static_cast<size_t>(c.pmax), D = static_cast<size_t>(c.dmax);
  Slot t;
  t.sess = reinterpret_cast<SessRt*>(take(sizeof(SessRt) * static_cast<size_t>(c.S)));
  t.heap = reinterpret_cast<Event*>(take(sizeof(Event) * static_cast<size_t>(c.hcap)));
  t.mt = reinterpret_cast<uint64_t*>(take(8 * 313));
  t.pw = reinterpret_cast<PrefillW*>(take(sizeof(PrefillW) * (P ? P : 1)));
  t.dw = reinterpret_cast<DecodeW*>(take(sizeof(DecodeW) * D));
  t.pq_s = reinterpret_cast<int32_t*>(take(4 * P * static_cast<size_t>(c.qcap)));
  t.pq_c = reinterpret_cast<double*>(take(8 * P * static_cast<size_t>(c.qcap)));
  t.tw_t = reinterpret_cast<double*>(take(8 * P * static_cast<size_t>(c.twcap)));
  t.tw_v = reinterpret_cast<double*>(take(8 * P * static_cast<size_t>(c.twcap)));
  t.dq_s = reinterpret_cast<int32_t*>(take(4 * D * static_cast<size_t>(c.qcap)));
  t.dq_c = reinterpret_cast<double*>(take(8 * D * static_cast<size_t>(c.qcap)));
  t.fh = reinterpret_cast<uint64_t*>(take(8 * D * static_cast<size_t>(c.fcap)));
  t.slog = reinterpret_cast<double*>(take(8 * D * static_cast<size_t>(c.lcap)));
  t.iw_t = reinterpret_cast<double*>(take(8 * D * static_cast<size_t>(c.iwcap)));
  t.iw_g = reinterpret_cast<double*>(take(8 * D * static_cast<size_t>(c.iwcap)));
  t.iw_c = reinterpret_cast<uint32_t*>(take(4 * D * static_cast<size_t>(c.iwcap)));
  if (s) *s = t;
  return off;
}

// Optional per-pair record outputs (drop-in SimResult vectors).
struct Records {
  pdsim_decision* decisions;      // [R]
  pdsim_ttft_sample* ttft;        // [R]
  pdsim_session_outcome* sessions;  // [S], termination order
};


struct PairResult {
  pdsim_attainment att;
  pdsim_counters ctr;
  int64_t n_decisions;
  int64_t n_ttft;
  int64_t events;        // dynamic events processed (diagnostics)
  int64_t cycles;        // device clock64() ticks for this pair (0 on host)
  int64_t exact_folds;   // certified comparisons that fell back to a fold
  int32_t status;        // PDSIM_PAIR_*
  int32_t reserved;
};

struct RouteOut {
  int32_t local;
  int32_t p;
  int32_t rationale;
  int32_t has_est;
  double est;
};

// A routing cost estimate: exact value, or a certified bracket around the
// reference's fold (exactsum.cuh).
struct Est {
  double lo, hi;
  int32_t exact;
  int32_t who;  // -1 local, else prefill worker index
};

class Engine {
 public:
  PDG_HD Engine(const DevTrace& tr, const DevPlan& plan, const pdsim_profile& prof,
                const DevParams& prm, const Caps& caps, const Slot& slot, Records rec,
                uint64_t seed)
      : T(tr), PL(plan), PF(prof), PR(prm), C(caps), W(slot), REC(rec), seed_(seed) {}

  PDG_HD void run(PairResult* out) {
    init();
    while (!failed_) {
      const bool has_arr = next_arr_ < T.S;
      const bool has_ev = hn_ > 0;
      if (!has_arr && !has_ev) break;
      if (has_arr && (!has_ev || T.arrival[next_arr_] <= W.heap[0].t)) {
        // Arrivals carry kind 0 and seq = index, so they precede every dynamic
        // event at an equal time (sim_engine.cpp:137-143, 68-74).
        const int32_t i = next_arr_++;
        advance_to(T.arrival[i]);
        on_arrival(i);
        continue;
      }
      const Event ev = heap_pop();
      ++events_;
      advance_to(ev.t);
      const uint32_t kind = static_cast<uint32_t>(ev.key >> 56);
      switch (kind) {
        case kInteractionDone: on_interaction_done(static_cast<int32_t>(ev.a)); break;
        case kKvTransferDone: on_kv_transfer_done(ev); break;
        case kPrefillDone: on_prefill_done(static_cast<int32_t>(ev.a)); break;
        case kDecodeStep: on_decode_step(static_cast<int32_t>(ev.a) - PL.P); break;
        default: fail(); break;
      }
    }
    for (int d = 0; d < PL.D; ++d) ctr_.kv_bytes_residual += W.dw[d].kv_used;
    out->att = att_;
    out->att.sessions_total = T.S;
    out->ctr = ctr_;
    out->n_decisions = n_dec_;
    out->n_ttft = n_ttft_;
    out->events = events_;
    out->exact_folds = folds_;
    out->status = failed_ ? PDSIM_PAIR_ERROR : PDSIM_PAIR_OK;
  }

 private:
  const DevTrace& T;
  const DevPlan& PL;
  const pdsim_profile& PF;
  const DevParams& PR;
  const Caps& C;
  const Slot& W;
  Records REC;
  uint64_t seed_;

  double now_ = 0.0;
  uint64_t seq_ = 0;
  int32_t hn_ = 0;
  int32_t next_arr_ = 0;
  int32_t adm_head_ = 0;
  int32_t rr_next_ = 0;
  uint32_t mt_idx_ = 0;
  bool failed_ = false;
  pdsim_attainment att_{};
  pdsim_counters ctr_{};
  int64_t n_dec_ = 0;
  int64_t n_ttft_ = 0;
  int64_t events_ = 0;
  int64_t folds_ = 0;

  PDG_HD void fail() { failed_ = true; }

  PDG_HD void advance_to(double t) {
    if (t < now_) ctr_.events_in_order = 0;  // sim_engine.cpp:148-150
    now_ = t;
  }

  PDG_HD void init() {
    now_ = 0.0;
    seq_ = static_cast<uint64_t>(T.S);  // arrivals took seq 0..S-1
    hn_ = 0;
    next_arr_ = 0;
    adm_head_ = 0;
    rr_next_ = 0;
    ctr_.events_in_order = 1;
    mt64_seed(W.mt, &mt_idx_, seed_);
    for (int p = 0; p < PL.P; ++p) {
      PrefillW& w = W.pw[p];
      w.q.sum.clear();
      w.q.qh = w.q.qt = 0;
      w.tw.clear();
      w.deg = PL.pdeg[p];
      w.cur = w.stg = -1;
      w.th = w.tt = 0;
      w.computing = w.staged = w.pending = 0;
      w.cur_cost = w.stg_cost = 0.0;
      w.staged_ready = 0.0;
    }
    for (int d = 0; d < PL.D; ++d) {
      DecodeW& w = W.dw[d];
      w.q.sum.clear();
      w.q.qh = w.q.qt = 0;
      w.iw.clear();
      w.deg = PL.ddeg[d];
      w.cur = -1;
      w.cur_cost = 0.0;
      w.kv_used = 0;
      w.kv_cap = static_cast<int64_t>(PF.degrees[w.deg]) * PF.gpu_memory_capacity;
      w.stepping = w.prefilling = 0;
      w.batch_n = w.n_new = w.cohort_n = w.first_n = 0;
      w.steps = 0;
      w.fh_n = 0;
      w.ih = w.it = 0;
    }
  }

  // ---- cost model (perf_model.cpp:158-205) ----
  PDG_HD double t_prefill(int32_t l_hist, int32_t l_incr, int deg) const {
    const double load = dadd(static_cast<double>(l_incr),
                             dmul(PF.history_weight, static_cast<double>(l_hist)));
    return curve_eval(PF.prefill[deg], load);
  }
  PDG_HD double t_decode(int32_t batch, int deg) const {
    return curve_eval(PF.decode[deg], static_cast<double>(batch));
  }
  PDG_HD double t_kv(int32_t l, int src, int dst) const {
    if (l == 0) return 0.0;
    return curve_eval(PF.kv[src][dst], static_cast<double>(l));
  }

  PDG_HD int32_t round_index(int32_t i) const { return T.round_off[i] + W.sess[i].round - 1; }
  PDG_HD int32_t l_incr_of(int32_t i) const { return T.incr[round_index(i)]; }
  PDG_HD double created_of(int32_t i) const {
    return W.sess[i].round == 1 ? T.arrival[i] : W.sess[i].t_enq;  // sim_engine.cpp:258, 283, 588
  }

  // ---- event heap ----
  PDG_HD void schedule(double t, uint32_t kind, uint32_t a, uint32_t b) {
    if (hn_ >= C.hcap) {
      fail();
      return;
    }
    Event e;
    e.t = t;
    e.key = (static_cast<uint64_t>(kind) << 56) | seq_++;
    e.a = a;
    e.b = b;
    int32_t i = hn_++;
    while (i > 0) {
      const int32_t par = (i - 1) >> 1;
      if (!ev_less(e, W.heap[par])) break;
      W.heap[i] = W.heap[par];
      i = par;
    }
    W.heap[i] = e;
  }

  PDG_HD Event heap_pop() {
    const Event top = W.heap[0];
    const Event last = W.heap[--hn_];
    int32_t i = 0;
    for (;;) {
      int32_t c = 2 * i + 1;
      if (c >= hn_) break;
      if (c + 1 < hn_ && ev_less(W.heap[c + 1], W.heap[c])) ++c;
      if (!ev_less(W.heap[c], last)) break;
      W.heap[i] = W.heap[c];
      i = c;
    }
    if (hn_ > 0) W.heap[i] = last;
    return top;
  }

  // ---- admission (sim_engine.cpp:240-267; bind_session coordinator.cpp:60-72) ----
  PDG_HD void on_arrival(int32_t i) {
    if (adm_head_ < i) return;  // queue non-empty: park behind the head
    if (!try_admit(i)) return;  // parked: adm_head_ == i
    adm_head_ = i + 1;
  }

  PDG_HD bool try_admit(int32_t i) {
    int best = 0;
    for (int d = 1; d < PL.D; ++d) {
      if (W.dw[d].kv_used < W.dw[best].kv_used) best = d;
    }
    const DecodeW& w = W.dw[best];
    const int64_t first = static_cast<int64_t>(T.incr[T.round_off[i]]) * PF.kv_bytes_per_token;
    if (w.kv_used + first > w.kv_cap) return false;
    SessRt& s = W.sess[i];
    s.bound = static_cast<int8_t>(best);
    s.bind_time = now_;
    s.round = 1;
    s.ctx = 0;
    s.itl_sum = 0.0;
    s.itl_cnt = 0;
    s.join = 0;
    s.postpone = 0;
    s.ttft_bad = 0;
    start_round(i);
    return true;
  }

  PDG_HD void admit_waiting() {
    while (adm_head_ < next_arr_ && try_admit(adm_head_)) ++adm_head_;
  }

  // ---- task creation and routing (sim_engine.cpp:271-333) ----
  PDG_HD void start_round(int32_t i) {
    SessRt& s = W.sess[i];
    s.t_enq = now_;
    s.postpone = 0;
    ++ctr_.tasks_created;
    const RouteOut r = decide(i);
    if (REC.decisions) {
      pdsim_decision& d = REC.decisions[n_dec_];
      d.time = now_;
      d.session_id = T.sid[i];
      d.round = s.round;
      d.worker = r.local ? PL.P + s.bound : r.p;
      d.local = static_cast<int8_t>(r.local);
      d.rationale = static_cast<int8_t>(r.rationale);
      d.has_estimate = static_cast<int8_t>(r.has_est);
      for (int k = 0; k < 5; ++k) d.reserved[k] = 0;
      d.estimated_cost = r.has_est ? r.est : 0.0;
    }
    ++n_dec_;
    if (r.local) {
      enqueue_local(s.bound, i);
    } else {
      enqueue_remote(r.p, i);
    }
  }

  PDG_HD RouteOut decide(int32_t i) {
    RouteOut r;
    r.local = 1;
    r.p = -1;
    r.has_est = 0;
    r.est = 0.0;
    if (PR.routing == PDSIM_ROUTING_ALWAYS_LOCAL) {
      r.rationale = PDSIM_RATIONALE_FORCED_LOCAL;
      return r;
    }
    if (PR.routing == PDSIM_ROUTING_ALWAYS_REMOTE) {
      if (PL.P == 0) {
        r.rationale = PDSIM_RATIONALE_FORCED_LOCAL;
        return r;
      }
      r.local = 0;
      r.p = rr_next_;
      rr_next_ = (rr_next_ + 1) % PL.P;
      r.rationale = PDSIM_RATIONALE_FORCED_REMOTE;
      return r;
    }
    return route(i);
  }

  // Coordinator::route (coordinator.cpp:115-171).
  PDG_HD RouteOut route(int32_t i) {
    const SessRt& s = W.sess[i];
    const int n = PL.P;
    RouteOut r;
    r.has_est = 0;
    r.est = 0.0;
    if (n > 0) {
      int order[PDSIM_MAX_WORKERS];
      for (int k = 0; k < n; ++k) order[k] = k;
      for (int k = n - 1; k > 0; --k) {
        const int j = static_cast<int>(mt64_next(W.mt, &mt_idx_) % static_cast<uint64_t>(k + 1));
        const int tmp = order[k];
        order[k] = order[j];
        order[j] = tmp;
      }
      const double thr = dmul(PR.alpha, T.ttft_thres);
      for (int k = 0; k < n; ++k) {
        if (ttft_has_slack(order[k], thr)) {
          r.local = 0;
          r.p = order[k];
          r.rationale = PDSIM_RATIONALE_SLACK_REMOTE;
          return r;
        }
      }
    }
    if (itl_has_slack(s.bound, dmul(PR.beta, T.itl_thres))) {
      r.local = 1;
      r.p = -1;
      r.rationale = PDSIM_RATIONALE_SLACK_LOCAL;
      return r;
    }
    // Cost comparison; ties prefer local, then the lowest worker index.
    r.local = 1;
    r.p = -1;
    r.rationale = PDSIM_RATIONALE_ARGMIN;
    Est best = est_local(i, s.bound);
    for (int p = 0; p < n; ++p) {
      Est c = est_remote(i, p, s.bound);
      if (est_less(c, best, i, s.bound)) {
        best = c;
        r.local = 0;
        r.p = p;
      }
    }
    r.has_est = 1;
    if (REC.decisions && !best.exact) resolve(best, i, s.bound);
    r.est = best.lo;
    return r;
  }

  // ---- routing estimates (coordinator.cpp:74-100) ----
  // Exact sequential folds (the reference's arithmetic).
  PDG_HD double fold_queue(const TaskQueue& q, const double* qc, double init) const {
    const uint32_t mask = static_cast<uint32_t>(C.qcap - 1);
    double c = init;
    for (uint32_t k = q.qh; k != q.qt; ++k) c = dadd(c, qc[k & mask]);
    return c;
  }
  PDG_HD double local_exact(int32_t i, int d) {
    ++folds_;
    const DecodeW& w = W.dw[d];
    return fold_queue(w.q, W.dq_c + static_cast<size_t>(d) * C.qcap, t_prefill(W.sess[i].ctx, l_incr_of(i), w.deg));
  }
  PDG_HD double remote_head(int32_t i, int p, int d) const {
    const int pd = W.pw[p].deg, dd = W.dw[d].deg;
    const int32_t hist = W.sess[i].ctx;
    const int32_t incr = l_incr_of(i);
    return dadd(t_prefill(hist, incr, pd), dadd(t_kv(hist, dd, pd), t_kv(incr, pd, dd)));
  }
  PDG_HD double remote_exact(int32_t i, int p, int d) {
    ++folds_;
    const double tq = fold_queue(W.pw[p].q, W.pq_c + static_cast<size_t>(p) * C.qcap, 0.0);
    return dadd(remote_head(i, p, d), tq);
  }
  PDG_HD static Est exact_est(double v, int who) {
    Est e;
    e.lo = e.hi = v;
    e.exact = 1;
    e.who = who;
    return e;
  }
  // head + fold(queue) of `len` non-negative terms, with exact queue sum.
  PDG_HD static Est bracket_est(double head, const ExactSum& qs, int64_t nterms, int who) {
    Est e;
    const double v = dadd(head, fx_to_double(qs.sum));
    const double m = fold_margin(nterms);
    e.lo = v * (1.0 - m);
    e.hi = v * (1.0 + m);
    e.exact = 0;
    e.who = who;
    return e;
  }
  PDG_HD Est est_local(int32_t i, int d) {
    const DecodeW& w = W.dw[d];
    const uint32_t len = w.q.qt - w.q.qh;
    const double own = t_prefill(W.sess[i].ctx, l_incr_of(i), w.deg);
    if (len <= 2 || !w.q.sum.exact()) {
      return exact_est(fold_queue(w.q, W.dq_c + static_cast<size_t>(d) * C.qcap, own), -1);
    }
    return bracket_est(own, w.q.sum, static_cast<int64_t>(len) + 1, -1);
  }
  PDG_HD Est est_remote(int32_t i, int p, int d) {
    const PrefillW& w = W.pw[p];
    const uint32_t len = w.q.qt - w.q.qh;
    const double head = remote_head(i, p, d);
    if (len <= 2 || !w.q.sum.exact()) {
      return exact_est(dadd(head, fold_queue(w.q, W.pq_c + static_cast<size_t>(p) * C.qcap, 0.0)), p);
    }
    return bracket_est(head, w.q.sum, static_cast<int64_t>(len), p);
  }
  PDG_HD void resolve(Est& e, int32_t i, int d) {
    if (e.exact) return;
    const double v = e.who < 0 ? local_exact(i, d) : remote_exact(i, e.who, d);
    e = exact_est(v, e.who);
  }
  // `c < b` on the reference's values.
  PDG_HD bool est_less(Est& c, Est& b, int32_t i, int d) {
    if (!(c.exact && b.exact)) {
      if (c.hi < b.lo) return true;
      if (c.lo >= b.hi) return false;
      resolve(c, i, d);
      resolve(b, i, d);
    }
    return c.lo < b.lo;
  }

  // ---- windowed statistics (coordinator.cpp:27-47) ----
  PDG_HD void ttft_trim(PrefillW& w, const double* tt, const double* tv) {
    const uint32_t mask = static_cast<uint32_t>(C.twcap - 1);
    const double cutoff = dsub(now_, PR.stat_window);
    while (w.th != w.tt && tt[w.th & mask] <= cutoff) {
      w.tw.remove(tv[w.th & mask]);
      ++w.th;
    }
  }

  PDG_HD void ttft_add(int p, double v) {
    PrefillW& w = W.pw[p];
    const uint32_t mask = static_cast<uint32_t>(C.twcap - 1);
    double* tt = W.tw_t + static_cast<size_t>(p) * C.twcap;
    double* tv = W.tw_v + static_cast<size_t>(p) * C.twcap;
    ttft_trim(w, tt, tv);
    if (w.tt - w.th >= static_cast<uint32_t>(C.twcap)) {
      fail();
      return;
    }
    tt[w.tt & mask] = now_;
    tv[w.tt & mask] = v;
    ++w.tt;
    w.tw.add(v);
  }

  // query(now) <= thr, where query is the sequential windowed mean.
  PDG_HD bool ttft_has_slack(int p, double thr) {
    PrefillW& w = W.pw[p];
    const double* tt = W.tw_t + static_cast<size_t>(p) * C.twcap;
    const double* tv = W.tw_v + static_cast<size_t>(p) * C.twcap;
    ttft_trim(w, tt, tv);
    if (w.th == w.tt) return 0.0 <= thr;  // empty window reads 0
    const int dec = mean_le_certified(w.tw, thr);
    if (dec >= 0) return dec == 1;
    ++folds_;
    const uint32_t mask = static_cast<uint32_t>(C.twcap - 1);
    double sum = 0.0;
    for (uint32_t k = w.th; k != w.tt; ++k) sum = dadd(sum, tv[k & mask]);
    return ddiv(sum, static_cast<double>(w.tt - w.th)) <= thr;
  }

  PDG_HD void itl_trim(DecodeW& w, const double* it, const double* ig, const uint32_t* ic) {
    const uint32_t mask = static_cast<uint32_t>(C.iwcap - 1);
    const double cutoff = dsub(now_, PR.stat_window);
    while (w.ih != w.it && it[w.ih & mask] <= cutoff) {
      w.iw.remove(ig[w.ih & mask], ic[w.ih & mask]);
      ++w.ih;
    }
  }

  PDG_HD void itl_add(int d, double gap, uint32_t count) {
    DecodeW& w = W.dw[d];
    const uint32_t mask = static_cast<uint32_t>(C.iwcap - 1);
    double* it = W.iw_t + static_cast<size_t>(d) * C.iwcap;
    double* ig = W.iw_g + static_cast<size_t>(d) * C.iwcap;
    uint32_t* ic = W.iw_c + static_cast<size_t>(d) * C.iwcap;
    itl_trim(w, it, ig, ic);
    if (w.it - w.ih >= static_cast<uint32_t>(C.iwcap)) {
      fail();
      return;
    }
    it[w.it & mask] = now_;
    ig[w.it & mask] = gap;
    ic[w.it & mask] = count;
    ++w.it;
    w.iw.add(gap, count);
  }

  PDG_HD bool itl_has_slack(int d, double thr) {
    DecodeW& w = W.dw[d];
    const double* it = W.iw_t + static_cast<size_t>(d) * C.iwcap;
    const double* ig = W.iw_g + static_cast<size_t>(d) * C.iwcap;
    const uint32_t* ic = W.iw_c + static_cast<size_t>(d) * C.iwcap;
    itl_trim(w, it, ig, ic);
    if (w.ih == w.it) return 0.0 <= thr;
    const int dec = mean_le_certified(w.iw, thr);
    if (dec >= 0) return dec == 1;
    ++folds_;
    const uint32_t mask = static_cast<uint32_t>(C.iwcap - 1);
    double sum = 0.0;
    for (uint32_t k = w.ih; k != w.it; ++k) sum = fold_repeat(sum, ig[k & mask], ic[k & mask]);
    return ddiv(sum, static_cast<double>(w.iw.terms)) <= thr;
  }

  // ---- queues + reorder (reorder.cpp:76-146; select_next sim_engine.cpp:335-350) ----
  PDG_HD bool queue_push(TaskQueue& q, int32_t* qs, double* qc, int32_t i, double cost) {
    if (q.qt - q.qh >= static_cast<uint32_t>(C.qcap)) {
      fail();
      return false;
    }
    const uint32_t mask = static_cast<uint32_t>(C.qcap - 1);
    qs[q.qt & mask] = i;
    qc[q.qt & mask] = cost;
    ++q.qt;
    q.sum.add(cost);
    return true;
  }

  // Dequeues the next task (after reordering the head window).
  PDG_HD int32_t select_next(TaskQueue& q, int32_t* qs, double* qc, double* cost) {
    const uint32_t mask = static_cast<uint32_t>(C.qcap - 1);
    if (PR.reorder) {
      const uint32_t len = q.qt - q.qh;
      const int m = static_cast<int>(len < static_cast<uint32_t>(PR.window) ? len : PR.window);
      if (m > 1) reorder_head(qs, qc, q.qh, m);
    }
    const int32_t i = qs[q.qh & mask];
    *cost = qc[q.qh & mask];
    ++q.qh;
    q.sum.remove(*cost);
    const int32_t pc = W.sess[i].postpone;
    if (pc > ctr_.max_postpone_observed) ctr_.max_postpone_observed = pc;
    return i;
  }

  // Exhaustive search over the lexicographic permutations of the first m
  // queued tasks; strict improvements only; capped tasks cannot be pushed
  // back (reorder.cpp:93-138).
  PDG_HD void reorder_head(int32_t* qs, double* qc, uint32_t qh, int m) {
    const uint32_t mask = static_cast<uint32_t>(C.qcap - 1);
    int32_t hs[8];
    double hc[8], wait[8];
    int8_t pc[8];
    for (int k = 0; k < m; ++k) {
      hs[k] = qs[(qh + k) & mask];
      hc[k] = qc[(qh + k) & mask];
      wait[k] = dsub(now_, W.sess[hs[k]].t_enq);
      pc[k] = W.sess[hs[k]].postpone;
    }
    const double thres = T.ttft_thres;
    int perm[8], best[8];
    for (int k = 0; k < m; ++k) perm[k] = best[k] = k;
    int best_sat = count_satisfied(perm, m, hc, wait, thres);
    if (best_sat == m) return;  // identity already satisfies every task: no strict improvement exists
    while (next_permutation(perm, m)) {
      bool allowed = true;
      for (int k = 0; k < m; ++k) {
        if (k > perm[k] && pc[perm[k]] >= PR.window) {
          allowed = false;
          break;
        }
      }
      if (!allowed) continue;
      const int sat = count_satisfied(perm, m, hc, wait, thres);
      if (sat > best_sat) {
        best_sat = sat;
        for (int k = 0; k < m; ++k) best[k] = perm[k];
        if (best_sat == m) break;  // cannot be strictly improved upon
      }
    }
    for (int k = 0; k < m; ++k) {
      const int p = best[k];
      if (k > p) ++W.sess[hs[p]].postpone;
      qs[(qh + k) & mask] = hs[p];
      qc[(qh + k) & mask] = hc[p];
    }
  }

  PDG_HD static int count_satisfied(const int* perm, int m, const double* hc,
                                    const double* wait, double thres) {
    double elapsed = 0.0;
    int sat = 0;
    for (int k = 0; k < m; ++k) {
      elapsed = dadd(elapsed, hc[perm[k]]);
      if (dadd(wait[perm[k]], elapsed) <= thres) ++sat;
    }
    return sat;
  }

  PDG_HD static bool next_permutation(int* a, int n) {
    int i = n - 2;
    while (i >= 0 && a[i] >= a[i + 1]) --i;
    if (i < 0) return false;
    int j = n - 1;
    while (a[j] <= a[i]) --j;
    int t = a[i];
    a[i] = a[j];
    a[j] = t;
    for (int l = i + 1, r = n - 1; l < r; ++l, --r) {
      t = a[l];
      a[l] = a[r];
      a[r] = t;
    }
    return true;
  }

  // ---- prefill workers (sim_engine.cpp:354-453) ----
  PDG_HD void enqueue_remote(int p, int32_t i) {
    PrefillW& w = W.pw[p];
    const double cost = t_prefill(W.sess[i].ctx, l_incr_of(i), w.deg);
    if (!queue_push(w.q, W.pq_s + static_cast<size_t>(p) * C.qcap, W.pq_c + static_cast<size_t>(p) * C.qcap, i,
                    cost))
      return;
    try_stage(p);
    try_start_compute(p);
  }

  PDG_HD void try_stage(int p) {
    PrefillW& w = W.pw[p];
    if (w.staged || w.q.qh == w.q.qt) return;
    w.stg = select_next(w.q, W.pq_s + static_cast<size_t>(p) * C.qcap, W.pq_c + static_cast<size_t>(p) * C.qcap,
                        &w.stg_cost);
    w.staged = 1;
    const int32_t hist = W.sess[w.stg].ctx;
    if (hist > 0) {
      // Lazy history read from the bound decode worker (sim_engine.cpp:368-383).
      const int dd = W.dw[W.sess[w.stg].bound].deg;
      w.staged_ready = dadd(now_, t_kv(hist, dd, w.deg));
      w.pending = 1;
      schedule(w.staged_ready, kKvTransferDone, static_cast<uint32_t>(p), 0u);
    } else {
      w.staged_ready = now_;
      w.pending = 0;
    }
  }

  PDG_HD void try_start_compute(int p) {
    PrefillW& w = W.pw[p];
    if (w.computing || !w.staged || w.pending || w.staged_ready > now_) return;
    w.cur = w.stg;
    w.cur_cost = w.stg_cost;
    w.staged = 0;
    w.computing = 1;
    schedule(dadd(now_, w.cur_cost), kPrefillDone, static_cast<uint32_t>(p), 0u);
    try_stage(p);  // the next task's history read overlaps this compute
  }

  PDG_HD void on_prefill_done(int32_t worker) {
    if (worker < PL.P) {
      const int p = worker;
      PrefillW& w = W.pw[p];
      w.computing = 0;
      const int32_t i = w.cur;
      const int dd = W.dw[W.sess[i].bound].deg;
      schedule(dadd(now_, t_kv(l_incr_of(i), w.deg, dd)), kKvTransferDone, static_cast<uint32_t>(p),
               static_cast<uint32_t>(i) | 0x80000000u);
      try_stage(p);
      try_start_compute(p);
    } else {
      const int d = worker - PL.P;
      DecodeW& w = W.dw[d];
      w.prefilling = 0;
      complete_task(w.cur, true, -1, d);
      advance_decode(d);
    }
  }

  PDG_HD void on_kv_transfer_done(const Event& ev) {
    const int p = static_cast<int>(ev.a);
    if (!(ev.b & 0x80000000u)) {  // history read landed
      W.pw[p].pending = 0;
      try_start_compute(p);
      return;
    }
    const int32_t i = static_cast<int32_t>(ev.b & 0x7fffffffu);
    const int d = W.sess[i].bound;
    complete_task(i, false, p, d);
    advance_decode(d);
  }

  // complete_task (sim_engine.cpp:458-484).
  PDG_HD void complete_task(int32_t i, bool local, int p, int d) {
    SessRt& s = W.sess[i];
    const double created = created_of(i);
    const double value = dsub(now_, created);
    if (!local) ttft_add(p, value);  // decode workers' TTFT windows are never queried
    if (REC.ttft) {
      pdsim_ttft_sample& o = REC.ttft[n_ttft_];
      o.session_id = T.sid[i];
      o.round = s.round;
      o.kind = s.round == 1 ? 0 : 1;
      o.local = local ? 1 : 0;
      o.reserved[0] = o.reserved[1] = 0;
      o.created_time = created;
      o.completion_time = now_;
      o.value = value;
    }
    ++n_ttft_;
    if (value > T.ttft_thres) s.ttft_bad = 1;
    const int32_t incr = l_incr_of(i);
    s.ctx += incr;
    DecodeW& w = W.dw[d];
    w.kv_used += static_cast<int64_t>(incr) * PF.kv_bytes_per_token;
    // Join the decode batch: first token in the next step started.
    s.join = w.steps;
    const int32_t dec = T.dec[round_index(i)];
    fh_push(d, (static_cast<uint64_t>(static_cast<uint32_t>(w.steps + dec - 1)) << 32) |
                   static_cast<uint32_t>(T.rank[i]));
    ++w.batch_n;
    ++w.n_new;
    ++ctr_.tasks_completed;
  }

  // ---- decode workers (sim_engine.cpp:488-583) ----
  PDG_HD void enqueue_local(int d, int32_t i) {
    DecodeW& w = W.dw[d];
    const double cost = t_prefill(W.sess[i].ctx, l_incr_of(i), w.deg);
    if (!queue_push(w.q, W.dq_s + static_cast<size_t>(d) * C.qcap, W.dq_c + static_cast<size_t>(d) * C.qcap, i,
                    cost))
      return;
    advance_decode(d);
  }

  PDG_HD void advance_decode(int d) {
    DecodeW& w = W.dw[d];
    if (w.stepping || w.prefilling) return;
    if (w.q.qh != w.q.qt) {
      // Local prefill preempts decoding until the queue drains.
      w.cur = select_next(w.q, W.dq_s + static_cast<size_t>(d) * C.qcap, W.dq_c + static_cast<size_t>(d) * C.qcap,
                          &w.cur_cost);
      w.prefilling = 1;
      schedule(dadd(now_, w.cur_cost), kPrefillDone, static_cast<uint32_t>(PL.P + d), 0u);
      return;
    }
    if (w.batch_n > 0) {
      w.cohort_n = w.batch_n;
      w.first_n = w.n_new;
      w.n_new = 0;
      ++w.steps;
      w.stepping = 1;
      schedule(dadd(now_, t_decode(w.cohort_n, w.deg)), kDecodeStep, static_cast<uint32_t>(PL.P + d), 0u);
    }
  }

  PDG_HD void on_decode_step(int d) {
    DecodeW& w = W.dw[d];
    w.stepping = 0;
    const int32_t k = w.steps - 1;  // index of the step that just ended
    const uint32_t lmask = static_cast<uint32_t>(C.lcap - 1);
    double* slog = W.slog + static_cast<size_t>(d) * C.lcap;
    slog[static_cast<uint32_t>(k) & lmask] = now_;
    const int32_t n_itl = w.cohort_n - w.first_n;
    if (n_itl > 0) {
      const double gap = dsub(now_, slog[static_cast<uint32_t>(k - 1) & lmask]);
      itl_add(d, gap, static_cast<uint32_t>(n_itl));
    }
    ctr_.tokens_decoded += w.cohort_n;
    w.kv_used += static_cast<int64_t>(w.cohort_n) * PF.kv_bytes_per_token;

    bool any_terminated = false;
    uint64_t* fh = W.fh + static_cast<size_t>(d) * C.fcap;
    while (w.fh_n > 0 && static_cast<int32_t>(fh[0] >> 32) <= k) {
      if (static_cast<int32_t>(fh[0] >> 32) < k) {  // a round end was missed: invariant broken
        fail();
        return;
      }
      const uint32_t rank = static_cast<uint32_t>(fh[0]);
      fh_pop(d);
      const int32_t i = T.by_rank[rank];
      SessRt& s = W.sess[i];
      const int32_t ridx = round_index(i);
      const int32_t dec = T.dec[ridx];
      // This round's ITL samples, in token order (sim_engine.cpp:544-555).
      double sum = s.itl_sum;
      for (int32_t j = s.join + 1; j <= k; ++j) {
        sum = dadd(sum, dsub(slog[static_cast<uint32_t>(j) & lmask], slog[static_cast<uint32_t>(j - 1) & lmask]));
      }
      s.itl_sum = sum;
      s.itl_cnt += dec - 1;
      s.ctx += dec;
      --w.batch_n;
      if (s.round == T.round_off[i + 1] - T.round_off[i]) {
        terminate_session(i, d);
        any_terminated = true;
      } else {
        schedule(dadd(now_, T.delay[ridx]), kInteractionDone, static_cast<uint32_t>(i), 0u);
      }
    }
    if (any_terminated) admit_waiting();
    advance_decode(d);
  }

  PDG_HD void on_interaction_done(int32_t i) {
    ++W.sess[i].round;
    start_round(i);
  }

  // terminate_session + slo_verdict (sim_engine.cpp:591-607, 668-674).
  PDG_HD void terminate_session(int32_t i, int d) {
    SessRt& s = W.sess[i];
    W.dw[d].kv_used -= static_cast<int64_t>(s.ctx) * PF.kv_bytes_per_token;
    const double mean_itl = s.itl_cnt > 0 ? ddiv(s.itl_sum, static_cast<double>(s.itl_cnt)) : 0.0;
    const bool ttft_ok = !s.ttft_bad;
    const bool itl_ok = s.itl_cnt == 0 || mean_itl <= T.itl_thres;
    const bool slo_ok = ttft_ok && itl_ok;
    if (REC.sessions) {
      pdsim_session_outcome& o = REC.sessions[att_.sessions_completed];
      o.session_id = T.sid[i];
      o.arrival_time = T.arrival[i];
      o.completion_time = now_;
      o.admission_wait = dsub(s.bind_time, T.arrival[i]);
      o.mean_itl = mean_itl;
      o.rounds = T.round_off[i + 1] - T.round_off[i];
      o.ttft_ok = ttft_ok;
      o.itl_ok = itl_ok;
      o.slo_ok = slo_ok;
      o.reserved = 0;
    }
    ++att_.sessions_completed;
    att_.slo_ok += slo_ok;
    att_.ttft_ok += ttft_ok;
    att_.itl_ok += itl_ok;
  }

  // ---- finisher heap: u64 keys (end_step << 32 | id rank), min at [0] ----
  PDG_HD void fh_push(int d, uint64_t key) {
    DecodeW& w = W.dw[d];
    if (w.fh_n >= C.fcap) {
      fail();
      return;
    }
    uint64_t* h = W.fh + static_cast<size_t>(d) * C.fcap;
    int32_t i = w.fh_n++;
    while (i > 0) {
      const int32_t par = (i - 1) >> 1;
      if (h[par] <= key) break;
      h[i] = h[par];
      i = par;
    }
    h[i] = key;
  }

  PDG_HD void fh_pop(int d) {
    DecodeW& w = W.dw[d];
    uint64_t* h = W.fh + static_cast<size_t>(d) * C.fcap;
    const uint64_t last = h[--w.fh_n];
    const int32_t n = w.fh_n;
    int32_t i = 0;
    for (;;) {
      int32_t c = 2 * i + 1;
      if (c >= n) break;
      if (c + 1 < n && h[c + 1] < h[c]) ++c;
      if (h[c] >= last) break;
      h[i] = h[c];
      i = c;
    }
    if (n > 0) h[i] = last;
  }
};

}  // namespace pdg
