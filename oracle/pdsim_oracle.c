/* oracle/pdsim_oracle.c — TEST INFRASTRUCTURE ONLY: the plain-C restatement
 * of the reference replay (pdsim::run), used as a checker.
 *
 * It follows the reference algorithm literally — a binary heap of full events
 * with task payloads, per-sample windowed statistics summed from the first
 * in-window sample, a materialised sorted decode batch stepped token by token,
 * and exhaustive permutation reordering — with none of the GPU engine's
 * restructurings (finisher heaps, run-length ITL windows, certified folds).
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/proj). Parity of this restatement with the reference itself
 * is pinned by tests/test_oracle.py (against oracle/_ref, and against the
 * committed fixtures in tests/golden when the reference library is absent).
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off (oracle/Makefile). No FMA
 * contraction: every a*b+c of the reference rounds twice.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pdsim_gpu.h"

static char g_err[512];
const char* oracle_last_error(void) { return g_err; }

static int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

/* ---- std::mt19937_64 (coordinator.hpp:84) -------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} Mt64;

static void mt_seed(Mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t mt_next(Mt64* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ull) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* ---- cost model (src/perf_model.cpp:43-52, 158-205) ---------------------- */
static double eval_curve(const pdsim_curve* c, double load) {
  int i = 0; /* upper_bound: number of breakpoints <= load */
  while (i < c->n_breakpoints && !(load < c->breakpoints[i])) ++i;
  return c->alpha[i] + c->beta[i] * load;
}

typedef struct {
  const pdsim_profile* pf;
} Cost;

static int deg_index(const pdsim_profile* p, int degree) {
  for (int i = 0; i < p->n_degrees; ++i)
    if (p->degrees[i] == degree) return i;
  return -1;
}

static double t_prefill(const pdsim_profile* p, int64_t l_hist, int64_t l_incr, int di) {
  const double load = (double)l_incr + p->history_weight * (double)l_hist;
  return eval_curve(&p->prefill[di], load);
}
static double t_decode(const pdsim_profile* p, int64_t batch, int di) { return eval_curve(&p->decode[di], (double)batch); }
static double t_kv(const pdsim_profile* p, int64_t l, int s, int d) {
  if (l == 0) return 0.0;
  return eval_curve(&p->kv[s][d], (double)l);
}

/* ---- PrefillTask (include/pdsim/worker_state.hpp:30-43) ------------------ */
typedef struct {
  int64_t session_id;
  int round;
  int kind; /* 0 initial, 1 incremental */
  int64_t l_hist, l_incr;
  double created_time, enqueue_time;
  int postpone_count;
} Task;

typedef struct {
  Task* v;
  int64_t head, len, cap;
} Deque;

static void dq_push(Deque* q, Task t) {
  if (q->len == q->cap) {
    int64_t nc = q->cap ? q->cap * 2 : 16;
    Task* nv = (Task*)malloc(sizeof(Task) * (size_t)nc);
    for (int64_t k = 0; k < q->len; ++k) nv[k] = q->v[(q->head + k) % q->cap];
    free(q->v);
    q->v = nv;
    q->head = 0;
    q->cap = nc;
  }
  q->v[(q->head + q->len) % q->cap] = t;
  ++q->len;
}
static Task* dq_at(Deque* q, int64_t k) { return &q->v[(q->head + k) % q->cap]; }
static Task dq_pop(Deque* q) {
  Task t = q->v[q->head];
  q->head = (q->head + 1) % q->cap;
  --q->len;
  return t;
}

/* ---- WindowedStat (src/coordinator.cpp:27-47) ---------------------------- */
typedef struct {
  double* t;
  double* v;
  int64_t n, cap;
  double window;
} Window;

static void win_add(Window* w, double t, double v) {
  if (w->n == w->cap) {
    w->cap = w->cap ? w->cap * 2 : 64;
    w->t = (double*)realloc(w->t, sizeof(double) * (size_t)w->cap);
    w->v = (double*)realloc(w->v, sizeof(double) * (size_t)w->cap);
  }
  w->t[w->n] = t;
  w->v[w->n] = v;
  ++w->n;
}

static double win_query(const Window* w, double now) {
  const double cutoff = now - w->window;
  int64_t lo = 0, hi = w->n; /* lower_bound(completion_time <= cutoff) */
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (w->t[mid] <= cutoff) lo = mid + 1; else hi = mid;
  }
  int64_t b = lo;
  lo = b;
  hi = w->n; /* upper_bound(now < completion_time) */
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (!(now < w->t[mid])) lo = mid + 1; else hi = mid;
  }
  int64_t e = lo;
  if (b == e) return 0.0;
  double sum = 0.0;
  for (int64_t k = b; k < e; ++k) sum += w->v[k];
  return sum / (double)(e - b);
}

/* ---- events (src/sim_engine.cpp:48-74) ----------------------------------- */
enum { K_ARRIVAL = 0, K_INTERACTION = 1, K_KV = 2, K_PREFILL_DONE = 3, K_DECODE_STEP = 4 };
typedef struct {
  double time;
  int kind;
  uint64_t seq;
  int64_t session;
  int worker;
  int transfer; /* 0 history read, 1 writeback */
  Task task;
} Event;

static int ev_after(const Event* a, const Event* b) {
  if (a->time != b->time) return a->time > b->time;
  if (a->kind != b->kind) return a->kind > b->kind;
  return a->seq > b->seq;
}

typedef struct {
  Event* v;
  int64_t n, cap;
} Heap;

static void heap_push(Heap* h, Event e) {
  if (h->n == h->cap) {
    h->cap = h->cap ? h->cap * 2 : 64;
    h->v = (Event*)realloc(h->v, sizeof(Event) * (size_t)h->cap);
  }
  int64_t i = h->n++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!ev_after(&h->v[p], &e)) break;
    h->v[i] = h->v[p];
    i = p;
  }
  h->v[i] = e;
}

static Event heap_pop(Heap* h) {
  Event top = h->v[0];
  Event last = h->v[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= h->n) break;
    if (c + 1 < h->n && ev_after(&h->v[c], &h->v[c + 1])) ++c;
    if (!ev_after(&last, &h->v[c])) break;
    h->v[i] = h->v[c];
    i = c;
  }
  if (h->n > 0) h->v[i] = last;
  return top;
}

/* ---- engine state (src/sim_engine.cpp:76-105, 613-631) ------------------- */
typedef struct {
  int id, phase, di;
  Deque queue;
  int64_t* batch; /* sorted session ids */
  int64_t batch_n, batch_cap;
  int64_t kv_used, kv_cap;
  Window ttft, itl;
} Worker;

typedef struct {
  int computing;
  Task current;
  double current_done;
  int staged;
  Task staged_task;
  double staged_ready;
  int transfer_pending;
} PrefillExec;

typedef struct {
  int stepping, prefilling;
  Task current;
  int64_t* cohort;
  int64_t cohort_n, cohort_cap;
} DecodeExec;

typedef struct {
  int bound, current_round;
  int64_t context_len, decoded_in_round;
  double last_token_time, bind_time;
  double itl_sum; /* sequential fold of the itl_values vector */
  int64_t itl_n;
  int ttft_bad;
} SessionRt;

typedef struct {
  const pdsim_trace* tr;
  const pdsim_profile* pf;
  const pdsim_sched_params* prm;
  int P, D;
  Worker* pw;
  Worker* dw;
  PrefillExec* pe;
  DecodeExec* de;
  SessionRt* s;
  int64_t* id_sorted_idx; /* for id -> index lookups */
  int64_t* adm;
  int64_t adm_head, adm_n;
  Heap ev;
  uint64_t next_seq;
  double now;
  int rr_next;
  Mt64 rng;
  pdsim_run_output* out;
  int64_t n_dec, n_ttft, n_sess;
  int failed;
} Engine;

static int64_t index_of(const Engine* e, int64_t sid) {
  int64_t lo = 0, hi = e->tr->n_sessions;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (e->tr->session_id[e->id_sorted_idx[mid]] < sid) lo = mid + 1; else hi = mid;
  }
  return e->id_sorted_idx[lo];
}

static void schedule(Engine* e, Event ev) { /* src/sim_engine.cpp:233-236 */
  ev.seq = e->next_seq++;
  heap_push(&e->ev, ev);
}

static Event mk_event(double t, int kind) {
  Event ev;
  memset(&ev, 0, sizeof(ev));
  ev.time = t;
  ev.kind = kind;
  ev.session = -1;
  ev.worker = -1;
  return ev;
}

static void start_round(Engine* e, int64_t sidx, double created);
static void advance_decode(Engine* e, int d);
static void try_stage(Engine* e, int p);
static void try_start_compute(Engine* e, int p);

/* bind_session (src/coordinator.cpp:60-72) */
static int bind_session(const Engine* e) {
  int best = 0;
  for (int i = 1; i < e->D; ++i)
    if (e->dw[i].kv_used < e->dw[best].kv_used) best = i;
  return best;
}

/* try_admit / admit_waiting / on_arrival (src/sim_engine.cpp:240-267) */
static int try_admit(Engine* e, int64_t sidx) {
  SessionRt* s = &e->s[sidx];
  const int cand = bind_session(e);
  const Worker* w = &e->dw[cand];
  const int64_t r0 = e->tr->round_offset[sidx];
  const int64_t first = e->tr->incr_input_len[r0] * e->pf->kv_bytes_per_token;
  if (w->kv_used + first > w->kv_cap) return 0;
  s->bound = cand;
  s->bind_time = e->now;
  s->current_round = 1;
  start_round(e, sidx, e->tr->arrival_time[sidx]);
  return 1;
}

static void admit_waiting(Engine* e) {
  while (e->adm_n > 0 && try_admit(e, e->adm[e->adm_head])) {
    ++e->adm_head;
    --e->adm_n;
  }
}

static void on_arrival(Engine* e, int64_t sidx) {
  if (e->adm_n > 0 || !try_admit(e, sidx)) {
    e->adm[e->adm_head + e->adm_n] = sidx;
    ++e->adm_n;
  }
}

/* estimate_local / estimate_remote (src/coordinator.cpp:74-100) */
static double estimate_local(Engine* e, const Task* t, Worker* d) {
  double c = t_prefill(e->pf, t->l_hist, t->l_incr, d->di);
  for (int64_t k = 0; k < d->queue.len; ++k) {
    const Task* q = dq_at(&d->queue, k);
    c += t_prefill(e->pf, q->l_hist, q->l_incr, d->di);
  }
  return c;
}

static double estimate_remote(Engine* e, const Task* t, Worker* p, const Worker* d) {
  const double t_pre = t_prefill(e->pf, t->l_hist, t->l_incr, p->di);
  const double legs = t_kv(e->pf, t->l_hist, d->di, p->di) + t_kv(e->pf, t->l_incr, p->di, d->di);
  double tq = 0.0;
  for (int64_t k = 0; k < p->queue.len; ++k) {
    const Task* q = dq_at(&p->queue, k);
    tq += t_prefill(e->pf, q->l_hist, q->l_incr, p->di);
  }
  return t_pre + legs + tq;
}

typedef struct {
  int local, worker, rationale, has_est;
  double est;
} Decision;

/* Coordinator::route (src/coordinator.cpp:115-171) */
static Decision route(Engine* e, const Task* t, int bound) {
  Decision d;
  memset(&d, 0, sizeof(d));
  const int n = e->P;
  if (n > 0) {
    int order[PDSIM_MAX_WORKERS];
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int i = n - 1; i > 0; --i) {
      const int j = (int)(mt_next(&e->rng) % (uint64_t)(i + 1));
      const int tmp = order[i];
      order[i] = order[j];
      order[j] = tmp;
    }
    for (int k = 0; k < n; ++k) {
      if (win_query(&e->pw[order[k]].ttft, e->now) <= e->prm->alpha * e->tr->ttft_thres) {
        d.local = 0;
        d.worker = order[k];
        d.rationale = PDSIM_RATIONALE_SLACK_REMOTE;
        return d;
      }
    }
  }
  if (win_query(&e->dw[bound].itl, e->now) <= e->prm->beta * e->tr->itl_thres) {
    d.local = 1;
    d.rationale = PDSIM_RATIONALE_SLACK_LOCAL;
    return d;
  }
  d.local = 1;
  d.rationale = PDSIM_RATIONALE_ARGMIN;
  double best = estimate_local(e, t, &e->dw[bound]);
  for (int i = 0; i < n; ++i) {
    const double c = estimate_remote(e, t, &e->pw[i], &e->dw[bound]);
    if (c < best) {
      best = c;
      d.local = 0;
      d.worker = i;
    }
  }
  d.has_est = 1;
  d.est = best;
  return d;
}

/* decide (src/sim_engine.cpp:307-333) */
static Decision decide(Engine* e, const Task* t, const SessionRt* s) {
  Decision d;
  memset(&d, 0, sizeof(d));
  if (e->prm->routing == PDSIM_ROUTING_ALWAYS_LOCAL) {
    d.local = 1;
    d.rationale = PDSIM_RATIONALE_FORCED_LOCAL;
    return d;
  }
  if (e->prm->routing == PDSIM_ROUTING_ALWAYS_REMOTE) {
    if (e->P == 0) {
      d.local = 1;
      d.rationale = PDSIM_RATIONALE_FORCED_LOCAL;
      return d;
    }
    d.local = 0;
    d.worker = e->rr_next;
    e->rr_next = (e->rr_next + 1) % e->P;
    d.rationale = PDSIM_RATIONALE_FORCED_REMOTE;
    return d;
  }
  return route(e, t, s->bound);
}

/* count_satisfied (src/reorder.cpp:44-74) */
static int count_satisfied(Engine* e, const Task* tasks, const int* order, int m, int di) {
  double elapsed = 0.0;
  int sat = 0;
  for (int k = 0; k < m; ++k) {
    const Task* t = &tasks[order[k]];
    elapsed += t_prefill(e->pf, t->l_hist, t->l_incr, di);
    const double waited = e->now - t->enqueue_time;
    if (waited + elapsed <= e->tr->ttft_thres) ++sat;
  }
  return sat;
}

static int next_perm(int* a, int n) {
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) return 0;
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
  return 1;
}

/* reorder_and_dequeue (src/reorder.cpp:76-146) + select_next (src/sim_engine.cpp:335-350) */
static Task select_next(Engine* e, Deque* q, int di, int32_t* max_postpone) {
  Task task;
  if (e->prm->reorder) {
    const int w = e->prm->window;
    const int m = (int)(q->len < w ? q->len : w);
    Task head[8];
    for (int k = 0; k < m; ++k) head[k] = *dq_at(q, k);
    int best[8], perm[8];
    for (int k = 0; k < m; ++k) best[k] = perm[k] = k;
    int best_sat = count_satisfied(e, head, best, m, di);
    while (next_perm(perm, m)) {
      int allowed = 1;
      for (int k = 0; k < m; ++k) {
        const int p = perm[k];
        if (k > p && head[p].postpone_count >= w) {
          allowed = 0;
          break;
        }
      }
      if (!allowed) continue;
      const int sat = count_satisfied(e, head, perm, m, di);
      if (sat > best_sat) {
        best_sat = sat;
        memcpy(best, perm, sizeof(int) * (size_t)m);
      }
    }
    for (int k = 0; k < m; ++k)
      if (k > best[k]) ++head[best[k]].postpone_count;
    for (int k = 0; k < m; ++k) *dq_at(q, k) = head[best[k]];
  }
  task = dq_pop(q);
  if (task.postpone_count > *max_postpone) *max_postpone = task.postpone_count;
  return task;
}

/* start_round (src/sim_engine.cpp:271-305) */
static void start_round(Engine* e, int64_t sidx, double created) {
  SessionRt* s = &e->s[sidx];
  const int64_t ridx = e->tr->round_offset[sidx] + s->current_round - 1;
  Task t;
  memset(&t, 0, sizeof(t));
  t.session_id = e->tr->session_id[sidx];
  t.round = s->current_round;
  t.kind = s->current_round == 1 ? 0 : 1;
  t.l_hist = s->context_len;
  t.l_incr = e->tr->incr_input_len[ridx];
  t.created_time = created;
  t.enqueue_time = e->now;
  ++e->out->counters.tasks_created;
  const Decision d = decide(e, &t, s);
  if (e->out->decisions) {
    pdsim_decision* r = &e->out->decisions[e->n_dec];
    memset(r, 0, sizeof(*r));
    r->time = e->now;
    r->session_id = t.session_id;
    r->round = t.round;
    r->local = (int8_t)d.local;
    r->worker = d.local ? e->P + s->bound : d.worker;
    r->rationale = (int8_t)d.rationale;
    r->has_estimate = (int8_t)d.has_est;
    r->estimated_cost = d.has_est ? d.est : 0.0;
  }
  ++e->n_dec;
  if (d.local) {
    dq_push(&e->dw[s->bound].queue, t); /* enqueue_local (488-491) */
    advance_decode(e, s->bound);
  } else {
    dq_push(&e->pw[d.worker].queue, t); /* enqueue_remote (354-358) */
    try_stage(e, d.worker);
    try_start_compute(e, d.worker);
  }
}

/* try_stage (src/sim_engine.cpp:360-388) */
static void try_stage(Engine* e, int p) {
  Worker* w = &e->pw[p];
  PrefillExec* x = &e->pe[p];
  if (x->staged || w->queue.len == 0) return;
  x->staged_task = select_next(e, &w->queue, w->di, &e->out->counters.max_postpone_observed);
  x->staged = 1;
  if (x->staged_task.l_hist > 0) {
    const SessionRt* s = &e->s[index_of(e, x->staged_task.session_id)];
    const Worker* d = &e->dw[s->bound];
    x->staged_ready = e->now + t_kv(e->pf, x->staged_task.l_hist, d->di, w->di);
    x->transfer_pending = 1;
    Event ev = mk_event(x->staged_ready, K_KV);
    ev.worker = w->id;
    ev.transfer = 0;
    schedule(e, ev);
  } else {
    x->staged_ready = e->now;
    x->transfer_pending = 0;
  }
}

/* try_start_compute (src/sim_engine.cpp:390-410) */
static void try_start_compute(Engine* e, int p) {
  Worker* w = &e->pw[p];
  PrefillExec* x = &e->pe[p];
  if (x->computing || !x->staged || x->transfer_pending || x->staged_ready > e->now) return;
  x->current = x->staged_task;
  x->staged = 0;
  x->computing = 1;
  x->current_done = e->now + t_prefill(e->pf, x->current.l_hist, x->current.l_incr, w->di);
  Event ev = mk_event(x->current_done, K_PREFILL_DONE);
  ev.worker = w->id;
  schedule(e, ev);
  try_stage(e, p);
}

/* complete_task (src/sim_engine.cpp:458-484) */
static void complete_task(Engine* e, const Task* t, int local, int d, Window* serving) {
  const double value = e->now - t->created_time;
  win_add(serving, e->now, value);
  if (e->out->ttft_samples) {
    pdsim_ttft_sample* o = &e->out->ttft_samples[e->n_ttft];
    memset(o, 0, sizeof(*o));
    o->session_id = t->session_id;
    o->round = t->round;
    o->kind = (int8_t)t->kind;
    o->local = (int8_t)local;
    o->created_time = t->created_time;
    o->completion_time = e->now;
    o->value = value;
  }
  ++e->n_ttft;
  SessionRt* s = &e->s[index_of(e, t->session_id)];
  if (value > e->tr->ttft_thres) s->ttft_bad = 1;
  s->context_len += t->l_incr;
  s->decoded_in_round = 0;
  Worker* w = &e->dw[d];
  w->kv_used += t->l_incr * e->pf->kv_bytes_per_token;
  /* sorted insert of the session id into the decode batch */
  if (w->batch_n == w->batch_cap) {
    w->batch_cap = w->batch_cap ? w->batch_cap * 2 : 16;
    w->batch = (int64_t*)realloc(w->batch, sizeof(int64_t) * (size_t)w->batch_cap);
  }
  int64_t pos = w->batch_n;
  while (pos > 0 && w->batch[pos - 1] > t->session_id) {
    w->batch[pos] = w->batch[pos - 1];
    --pos;
  }
  w->batch[pos] = t->session_id;
  ++w->batch_n;
  ++e->out->counters.tasks_completed;
}

/* advance_decode (src/sim_engine.cpp:493-528) */
static void advance_decode(Engine* e, int d) {
  Worker* w = &e->dw[d];
  DecodeExec* x = &e->de[d];
  if (x->stepping || x->prefilling) return;
  if (w->queue.len > 0) {
    x->current = select_next(e, &w->queue, w->di, &e->out->counters.max_postpone_observed);
    x->prefilling = 1;
    Event ev = mk_event(e->now + t_prefill(e->pf, x->current.l_hist, x->current.l_incr, w->di), K_PREFILL_DONE);
    ev.worker = w->id;
    schedule(e, ev);
    return;
  }
  if (w->batch_n > 0) {
    if (w->batch_n > x->cohort_cap) {
      x->cohort_cap = w->batch_n * 2;
      x->cohort = (int64_t*)realloc(x->cohort, sizeof(int64_t) * (size_t)x->cohort_cap);
    }
    for (int64_t k = 0; k < w->batch_n; ++k) x->cohort[k] = index_of(e, w->batch[k]);
    x->cohort_n = w->batch_n;
    x->stepping = 1;
    Event ev = mk_event(e->now + t_decode(e->pf, x->cohort_n, w->di), K_DECODE_STEP);
    ev.worker = w->id;
    schedule(e, ev);
  }
}

/* terminate_session (src/sim_engine.cpp:591-607) */
static void terminate_session(Engine* e, int64_t sidx, int d) {
  SessionRt* s = &e->s[sidx];
  e->dw[d].kv_used -= s->context_len * e->pf->kv_bytes_per_token;
  const double mean_itl = s->itl_n ? s->itl_sum / (double)s->itl_n : 0.0;
  const int ttft_ok = !s->ttft_bad;
  const int itl_ok = s->itl_n == 0 || mean_itl <= e->tr->itl_thres;
  const int slo_ok = ttft_ok && itl_ok;
  if (e->out->sessions) {
    pdsim_session_outcome* o = &e->out->sessions[e->n_sess];
    memset(o, 0, sizeof(*o));
    o->session_id = e->tr->session_id[sidx];
    o->arrival_time = e->tr->arrival_time[sidx];
    o->completion_time = e->now;
    o->rounds = (int32_t)(e->tr->round_offset[sidx + 1] - e->tr->round_offset[sidx]);
    o->admission_wait = s->bind_time - e->tr->arrival_time[sidx];
    o->mean_itl = mean_itl;
    o->ttft_ok = (int8_t)ttft_ok;
    o->itl_ok = (int8_t)itl_ok;
    o->slo_ok = (int8_t)slo_ok;
  }
  ++e->n_sess;
  e->out->attainment.slo_ok += slo_ok;
  e->out->attainment.ttft_ok += ttft_ok;
  e->out->attainment.itl_ok += itl_ok;
}

/* on_decode_step (src/sim_engine.cpp:530-583): token by token, in cohort order */
static void on_decode_step(Engine* e, int d) {
  Worker* w = &e->dw[d];
  DecodeExec* x = &e->de[d];
  x->stepping = 0;
  int any_terminated = 0;
  for (int64_t c = 0; c < x->cohort_n; ++c) {
    const int64_t sidx = x->cohort[c];
    SessionRt* s = &e->s[sidx];
    const int64_t ridx = e->tr->round_offset[sidx] + s->current_round - 1;
    ++s->decoded_in_round;
    ++e->out->counters.tokens_decoded;
    if (s->decoded_in_round >= 2) {
      const double gap = e->now - s->last_token_time;
      win_add(&w->itl, e->now, gap);
      s->itl_sum += gap;
      ++s->itl_n;
    }
    s->last_token_time = e->now;
    s->context_len += 1;
    w->kv_used += e->pf->kv_bytes_per_token;
    if (s->decoded_in_round == e->tr->decode_len[ridx]) {
      const int64_t sid = e->tr->session_id[sidx];
      int64_t pos = 0;
      while (w->batch[pos] != sid) ++pos;
      memmove(&w->batch[pos], &w->batch[pos + 1], sizeof(int64_t) * (size_t)(w->batch_n - pos - 1));
      --w->batch_n;
      if (s->current_round == (int)(e->tr->round_offset[sidx + 1] - e->tr->round_offset[sidx])) {
        terminate_session(e, sidx, d);
        any_terminated = 1;
      } else {
        Event ev = mk_event(e->now + e->tr->interaction_delay[ridx], K_INTERACTION);
        ev.session = sidx;
        schedule(e, ev);
      }
    }
  }
  x->cohort_n = 0;
  if (any_terminated) admit_waiting(e);
  advance_decode(e, d);
}

/* on_prefill_done (src/sim_engine.cpp:412-438) */
static void on_prefill_done(Engine* e, int worker) {
  if (worker < e->P) {
    const int p = worker;
    PrefillExec* x = &e->pe[p];
    x->computing = 0;
    const Task t = x->current;
    const SessionRt* s = &e->s[index_of(e, t.session_id)];
    Event ev = mk_event(e->now + t_kv(e->pf, t.l_incr, e->pw[p].di, e->dw[s->bound].di), K_KV);
    ev.worker = e->pw[p].id;
    ev.transfer = 1;
    ev.task = t;
    schedule(e, ev);
    try_stage(e, p);
    try_start_compute(e, p);
  } else {
    const int d = worker - e->P;
    DecodeExec* x = &e->de[d];
    x->prefilling = 0;
    complete_task(e, &x->current, 1, d, &e->dw[d].ttft);
    advance_decode(e, d);
  }
}

/* on_kv_transfer_done (src/sim_engine.cpp:440-453) */
static void on_kv(Engine* e, const Event* ev) {
  const int p = ev->worker;
  if (ev->transfer == 0) {
    e->pe[p].transfer_pending = 0;
    try_start_compute(e, p);
    return;
  }
  const SessionRt* s = &e->s[index_of(e, ev->task.session_id)];
  const int d = s->bound;
  complete_task(e, &ev->task, 0, d, &e->pw[p].ttft);
  advance_decode(e, d);
}

/* on_interaction_done (src/sim_engine.cpp:585-589) */
static void on_interaction(Engine* e, int64_t sidx) {
  ++e->s[sidx].current_round;
  start_round(e, sidx, e->now);
}

static int cmp_outcome(const void* a, const void* b) {
  const pdsim_session_outcome* x = (const pdsim_session_outcome*)a;
  const pdsim_session_outcome* y = (const pdsim_session_outcome*)b;
  return x->session_id < y->session_id ? -1 : x->session_id > y->session_id;
}

static const pdsim_trace* g_sort_tr;
static int cmp_idx_by_id(const void* a, const void* b) {
  const int64_t x = g_sort_tr->session_id[*(const int64_t*)a];
  const int64_t y = g_sort_tr->session_id[*(const int64_t*)b];
  return x < y ? -1 : x > y;
}

/* Validation the reference Engine ctor performs (src/sim_engine.cpp:109-122,
 * 175-231; src/coordinator.cpp:102-113; src/workload.cpp:90-134). The profile
 * is assumed valid here (its validation is pinned by the product tests). */
static int validate(const pdsim_trace* tr, const pdsim_plan* plan, const pdsim_profile* pf,
                    const pdsim_sched_params* prm) {
  if (!(prm->alpha > 0.0 && prm->alpha <= 1.0) || !(prm->beta > 0.0 && prm->beta <= 1.0))
    return set_err(PDSIM_ERR_CONFIG, "routing: alpha/beta must be in (0, 1]");
  if (!(tr->ttft_thres > 0.0) || !(tr->itl_thres > 0.0)) return set_err(PDSIM_ERR_CONFIG, "SLO thresholds must be > 0");
  if (prm->window < 1 || !(prm->stat_window > 0.0)) return set_err(PDSIM_ERR_CONFIG, "scheduler: bad window");
  for (int64_t i = 0; i < tr->n_sessions; ++i) {
    if (tr->arrival_time[i] < 0.0 || (i > 0 && tr->arrival_time[i] < tr->arrival_time[i - 1]))
      return set_err(PDSIM_ERR_CONFIG, "trace: arrivals");
    if (tr->round_offset[i + 1] <= tr->round_offset[i]) return set_err(PDSIM_ERR_CONFIG, "trace: empty rounds");
    for (int64_t r = tr->round_offset[i]; r < tr->round_offset[i + 1]; ++r) {
      if (tr->incr_input_len[r] < 1 || tr->decode_len[r] < 1 || tr->interaction_delay[r] < 0.0)
        return set_err(PDSIM_ERR_CONFIG, "trace: round fields");
      if (r + 1 == tr->round_offset[i + 1] && tr->interaction_delay[r] != 0.0)
        return set_err(PDSIM_ERR_CONFIG, "trace: final round must have interaction_delay 0");
    }
  }
  int P = 0, D = 0;
  for (int g = 0; g < plan->n_prefill_groups; ++g) {
    if (deg_index(pf, plan->prefill_degree[g]) < 0) return set_err(PDSIM_ERR_CONFIG, "plan: prefill degree");
    P += plan->prefill_count[g];
  }
  for (int g = 0; g < plan->n_decode_groups; ++g) {
    if (deg_index(pf, plan->decode_degree[g]) < 0) return set_err(PDSIM_ERR_CONFIG, "plan: decode degree");
    D += plan->decode_count[g];
  }
  if (D == 0) return set_err(PDSIM_ERR_CONFIG, "plan: at least one decode replica is required");
  if (P + D > PDSIM_MAX_WORKERS) return set_err(PDSIM_ERR_CONFIG, "plan: too many replicas");
  if (prm->reorder && prm->window > 8 && tr->n_sessions > 0) return set_err(PDSIM_ERR_CONFIG, "reorder: window must be <= 8");
  int64_t max_cap = 0; /* precheck_sessions (src/sim_engine.cpp:217-231) */
  for (int g = 0; g < plan->n_decode_groups; ++g) {
    const int64_t cap = (int64_t)plan->decode_degree[g] * pf->gpu_memory_capacity;
    if (cap > max_cap) max_cap = cap;
  }
  for (int64_t i = 0; i < tr->n_sessions; ++i) {
    if (tr->incr_input_len[tr->round_offset[i]] * pf->kv_bytes_per_token > max_cap)
      return set_err(PDSIM_ERR_CONFIG, "trace: first-round KV exceeds every decode worker's capacity");
  }
  return PDSIM_OK;
}

/* pdsim::run (src/sim_engine.cpp:109-170, 676-681) */
int oracle_run(const pdsim_trace* tr, const pdsim_plan* plan, const pdsim_profile* pf, const pdsim_sched_params* prm,
               uint64_t seed, pdsim_run_output* out) {
  int rc = validate(tr, plan, pf, prm);
  if (rc) return rc;
  Engine e;
  memset(&e, 0, sizeof(e));
  e.tr = tr;
  e.pf = pf;
  e.prm = prm;
  e.out = out;
  memset(&out->counters, 0, sizeof(out->counters));
  memset(&out->attainment, 0, sizeof(out->attainment));
  out->counters.events_in_order = 1;
  mt_seed(&e.rng, seed);
  for (int g = 0; g < plan->n_prefill_groups; ++g) e.P += plan->prefill_count[g];
  for (int g = 0; g < plan->n_decode_groups; ++g) e.D += plan->decode_count[g];
  e.pw = (Worker*)calloc((size_t)(e.P ? e.P : 1), sizeof(Worker));
  e.dw = (Worker*)calloc((size_t)e.D, sizeof(Worker));
  e.pe = (PrefillExec*)calloc((size_t)(e.P ? e.P : 1), sizeof(PrefillExec));
  e.de = (DecodeExec*)calloc((size_t)e.D, sizeof(DecodeExec));
  int id = 0, k = 0; /* build_workers (src/sim_engine.cpp:175-203) */
  for (int g = 0; g < plan->n_prefill_groups; ++g)
    for (int c = 0; c < plan->prefill_count[g]; ++c, ++k) {
      e.pw[k].id = id++;
      e.pw[k].di = deg_index(pf, plan->prefill_degree[g]);
      e.pw[k].ttft.window = e.pw[k].itl.window = prm->stat_window;
    }
  k = 0;
  for (int g = 0; g < plan->n_decode_groups; ++g)
    for (int c = 0; c < plan->decode_count[g]; ++c, ++k) {
      e.dw[k].id = id++;
      e.dw[k].di = deg_index(pf, plan->decode_degree[g]);
      e.dw[k].kv_cap = (int64_t)plan->decode_degree[g] * pf->gpu_memory_capacity;
      e.dw[k].ttft.window = e.dw[k].itl.window = prm->stat_window;
    }
  const int64_t S = tr->n_sessions;
  e.s = (SessionRt*)calloc((size_t)(S ? S : 1), sizeof(SessionRt));
  e.adm = (int64_t*)calloc((size_t)(S ? S : 1), sizeof(int64_t));
  e.id_sorted_idx = (int64_t*)calloc((size_t)(S ? S : 1), sizeof(int64_t));
  for (int64_t i = 0; i < S; ++i) e.id_sorted_idx[i] = i;
  g_sort_tr = tr;
  qsort(e.id_sorted_idx, (size_t)S, sizeof(int64_t), cmp_idx_by_id);
  for (int64_t i = 0; i < S; ++i) { /* preload arrivals with seq 0..S-1 */
    Event ev = mk_event(tr->arrival_time[i], K_ARRIVAL);
    ev.session = i;
    schedule(&e, ev);
  }
  while (e.ev.n > 0) {
    const Event ev = heap_pop(&e.ev);
    if (ev.time < e.now) out->counters.events_in_order = 0;
    e.now = ev.time;
    switch (ev.kind) {
      case K_ARRIVAL: on_arrival(&e, ev.session); break;
      case K_INTERACTION: on_interaction(&e, ev.session); break;
      case K_KV: on_kv(&e, &ev); break;
      case K_PREFILL_DONE: on_prefill_done(&e, ev.worker); break;
      case K_DECODE_STEP: on_decode_step(&e, ev.worker - e.P); break;
      default: break;
    }
  }
  for (int d = 0; d < e.D; ++d) out->counters.kv_bytes_residual += e.dw[d].kv_used;
  out->n_decisions = e.n_dec;
  out->n_ttft = e.n_ttft;
  out->n_sessions = e.n_sess;
  out->attainment.sessions_total = S;
  out->attainment.sessions_completed = e.n_sess;
  if (out->sessions) qsort(out->sessions, (size_t)e.n_sess, sizeof(pdsim_session_outcome), cmp_outcome);
  for (int p = 0; p < e.P; ++p) {
    free(e.pw[p].queue.v);
    free(e.pw[p].ttft.t);
    free(e.pw[p].ttft.v);
  }
  for (int d = 0; d < e.D; ++d) {
    free(e.dw[d].queue.v);
    free(e.dw[d].batch);
    free(e.dw[d].ttft.t);
    free(e.dw[d].ttft.v);
    free(e.dw[d].itl.t);
    free(e.dw[d].itl.v);
    free(e.de[d].cohort);
  }
  free(e.pw);
  free(e.dw);
  free(e.pe);
  free(e.de);
  free(e.s);
  free(e.adm);
  free(e.id_sorted_idx);
  free(e.ev.v);
  return PDSIM_OK;
}
