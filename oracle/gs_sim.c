/*
 * gs_sim.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference simulator
 * greensim::run (proj/src/simkernel.cpp), the caller of the decision engine. It exists to
 *   (1) record the decode-enqueue stream in the reference's own processing order, and
 *   (2) check the GPU closed-loop decode pool (K5) on arbitrary controller parameters.
 * It is pinned field-by-field against the reference's run() (tests/test_oracle_sim.py).
 * Same conventions as gs_oracle.c: operation order is the specification, -ffp-contract=off.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gs_oracle.h"
#include "gs_oracle_int.h"

/* Event kinds double as tie-break priorities at equal times (simkernel.cpp:21-31). */
enum { EV_ARRIVAL = 0, EV_PREFILL_DONE, EV_STEP_END, EV_ENQUEUE, EV_FREQ, EV_COARSE, EV_ADAPT,
       EV_FINE, EV_OPT };
enum { PH_PREFILL = 0, PH_DECODE = 1, PH_IDLE = 2 }; /* simkernel.cpp:15-17 */

typedef struct { /* Ev, simkernel.cpp:33-42 */
  double t;
  int kind;
  uint64_t seq;
  int worker;
  int64_t req;
  double f;
  uint64_t gen;
  int prefill_pool;
} ev_t;

/* EvLater (simkernel.cpp:44-50) as "a pops before b" */
static int ev_before(const ev_t* a, const ev_t* b) {
  if (a->t != b->t) return a->t < b->t;
  if (a->kind != b->kind) return a->kind < b->kind;
  return a->seq < b->seq;
}

typedef struct {
  ev_t* v;
  int64_t n, cap;
} heap_t;

static void heap_push(heap_t* h, ev_t e) {
  if (h->n == h->cap) {
    h->cap = h->cap ? 2 * h->cap : 1024;
    h->v = (ev_t*)realloc(h->v, sizeof(ev_t) * (size_t)h->cap);
  }
  int64_t i = h->n++;
  while (i > 0) {
    const int64_t p = (i - 1) / 2;
    if (!ev_before(&e, &h->v[p])) break;
    h->v[i] = h->v[p];
    i = p;
  }
  h->v[i] = e;
}

static ev_t heap_pop(heap_t* h) {
  const ev_t top = h->v[0];
  const ev_t last = h->v[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= h->n) break;
    if (c + 1 < h->n && ev_before(&h->v[c + 1], &h->v[c])) ++c;
    if (!ev_before(&h->v[c], &last)) break;
    h->v[i] = h->v[c];
    i = c;
  }
  if (h->n > 0) h->v[i] = last;
  return top;
}

/* growable arrays */
#define VEC(T) struct { T* v; int64_t n, cap; }
#define VPUSH(a, x)                                                              \
  do {                                                                           \
    if ((a).n == (a).cap) {                                                      \
      (a).cap = (a).cap ? 2 * (a).cap : 16;                                      \
      (a).v = realloc((a).v, sizeof(*(a).v) * (size_t)(a).cap);                  \
    }                                                                            \
    (a).v[(a).n++] = (x);                                                        \
  } while (0)

typedef struct { double last_ms, power_w; int phase; } pstate_t;     /* PowerState :53-57 */
typedef struct { double act_prefill, act_decode, idle; int64_t n_int; } ledger_t; /* WorkerLedger */

/* ledger_close / ledger_set, simkernel.cpp:60-79 */
static void ledger_close(ledger_t* l, pstate_t* ps, double now) {
  if (now > ps->last_ms) {
    l->n_int++;
    const double joules = ps->power_w * (now - ps->last_ms) / 1000.0;
    if (ps->phase == PH_PREFILL)
      l->act_prefill += joules;
    else if (ps->phase == PH_DECODE)
      l->act_decode += joules;
    else
      l->idle += joules;
  }
  ps->last_ms = now;
}
static void ledger_set(ledger_t* l, pstate_t* ps, double now, int phase, double power) {
  if (phase == ps->phase && power == ps->power_w) return;
  ledger_close(l, ps, now);
  ps->phase = phase;
  ps->power_w = power;
}

typedef struct { /* PrefillWorkerState :81-93 */
  double freq, target;
  int busy;
  int64_t job;
  double job_t_ref, job_rem, job_upd;
  uint64_t gen;
  pstate_t ps;
} pw_t;

typedef struct { int64_t req; int emitted; double last_emit; } stream_t; /* StreamState :95-99 */

typedef struct { double t; int tokens; } tpsev_t;

typedef struct { /* DecodeWorkerState :101-113 */
  double freq, target;
  int stepping;
  VEC(stream_t) active;
  VEC(int64_t) pending; /* FIFO: [p_head, n) */
  int64_t p_head;
  pstate_t ps;
  VEC(tpsev_t) tps; /* TpsWindow deque: [t_head, n) */
  int64_t t_head;
  ring_t tbt;
  ctl_t ctl;
  gso_decision* log;
  int64_t log_cap;
} dw_t;

typedef struct { double t; int pool, worker; double f; } fc_t;
typedef struct { double tick; int cls, worker; double f, window; int infeasible; } pc_t;

typedef struct {
  /* request records (RequestRecord, simkernel.hpp:107-127) */
  int64_t n;
  int64_t* arrival_i;
  int32_t *prompt, *output, *class_queue, *prefill_worker, *decode_worker;
  int8_t* cls;
  double *arrival, *prefill_start, *prefill_end, *first_token, *finish;
  uint8_t *completed, *rejected;
  VEC(double) * tbt; /* per request */
  /* inputs */
  gso_profile prof;
  gso_policy pol;
  int32_t worker_map[64];
  gso_slo slo;
  gso_sim_cfg cfg;
  int routing_enabled, n_queues;
  /* dispatcher: per queue FIFO */
  VEC(int64_t) * q;
  int64_t* q_head;
  /* pools */
  pw_t* pw;
  dw_t* dw;
  ledger_t *pled, *dled;
  double* f_opt_table;
  double *tps_lo, *tps_hi;
  int n_buckets;
  heap_t heap;
  uint64_t next_seq;
  double now;
  int64_t outstanding;
  int64_t rejected_total, n_steps;
  VEC(fc_t) timeline;
  VEC(pc_t) commands;
  /* optimizer snapshots with the RAW running-job state (simkernel.cpp:470-480), for the
     device-side work_fraction test: per non-empty queue snapshot now, class, job range; per
     job prompt, deadline, running flag, remaining_ref, updated_ms, freq, t_ref, and the wf
     the simulator computed from them */
  VEC(double) sn_now;
  VEC(int32_t) sn_cls;
  VEC(int64_t) sn_off;
  VEC(int32_t) sj_prompt;
  VEC(uint8_t) sj_run;
  VEC(double) sj_dl, sj_rem, sj_upd, sj_freq, sj_tref, sj_wf;
  VEC(double) enq_t;
  VEC(int64_t) enq_req;
  gso_decision* decisions;
  int64_t n_decisions;
  double sim_end, last_arrival, end_floor;
  int pool_only;
  char err[256];
} sim_t;

static void schedule(sim_t* s, double t, int kind, int worker, int64_t req, double f, uint64_t gen,
                     int prefill_pool) {
  ev_t e = {t, kind, s->next_seq++, worker, req, f, gen, prefill_pool};
  heap_push(&s->heap, e);
}

static int dvfs(const sim_t* s) { return s->pol.kind == 2; }
static int routing_on(const sim_t* s) { /* routing_enabled(), simkernel.hpp:33-35 */
  return (s->pol.kind == 2 || s->pol.kind == 3) && s->pol.routing_enabled;
}
static double idle_prefill(const sim_t* s) { return s->prof.p_idle_w * s->cfg.gpus_per_prefill_worker; }
static double active_prefill(const sim_t* s, double f) {
  return gso_active_power_w(&s->prof, f) * s->cfg.gpus_per_prefill_worker;
}
static int queue_of_worker(const sim_t* s, int w) { return s->routing_enabled ? s->worker_map[w] : 0; }
/* request_class(r, 1024), simkernel.cpp:113-116 */
static int8_t req_class(int8_t given, int32_t prompt) {
  if (given == 0 || given == 1) return given;
  return prompt <= 1024 ? 0 : 1;
}
static double ttft_for(const gso_slo* slo, int c) { return c == 0 ? slo->ttft_sm_ms : slo->ttft_l_ms; }

/* GpuProfile::decode_step_ms -> decode_step_raw_ms, gpu_model.cpp:99-111 */
static double decode_step_ms(const gso_profile* p, double batch, double f) {
  return (p->dec_alpha0_ms + p->dec_alpha1_ms * batch) +
         (p->dec_beta0_ms + p->dec_beta1_ms * batch) * p->dec_f_ref_mhz / f;
}
/* GpuProfile::prefill_latency_ms -> prefill_latency_raw_ms, gpu_model.cpp:94-97 */
static double prefill_latency_ms(const gso_profile* p, double prompt, double f) {
  const double t_ref = (p->lat_a * prompt + p->lat_b) * prompt + p->lat_c;
  return t_ref * p->lat_f_ref_mhz / f;
}

/* ---------------------------------------------------------------- prefill pool */
static void start_prefill(sim_t* s, int w, int64_t id) { /* simkernel.cpp:268-283 */
  pw_t* pw = &s->pw[w];
  pw->busy = 1;
  pw->job = id;
  pw->job_t_ref = prefill_latency_ms(&s->prof, (double)s->prompt[id], s->prof.f_ref_mhz);
  pw->job_rem = pw->job_t_ref;
  pw->job_upd = s->now;
  ++pw->gen;
  s->prefill_start[id] = s->now;
  s->prefill_worker[id] = w;
  schedule(s, s->now + pw->job_rem * s->prof.f_ref_mhz / pw->freq, EV_PREFILL_DONE, w, id, 0.0,
           pw->gen, 1);
  ledger_set(&s->pled[w], &pw->ps, s->now, PH_PREFILL, active_prefill(s, pw->freq));
}

static void pull_next_prefill(sim_t* s, int w) { /* :285-292 */
  const int q = queue_of_worker(s, w);
  if (s->q_head[q] < s->q[q].n) {
    const int64_t id = s->q[q].v[s->q_head[q]++];
    start_prefill(s, w, id);
  } else {
    ledger_set(&s->pled[w], &s->pw[w].ps, s->now, PH_IDLE, idle_prefill(s));
  }
}

static void on_arrival(sim_t* s, const ev_t* ev) { /* :294-315 */
  const int64_t id = ev->req;
  const int q = s->routing_enabled ? gso_classify(s->pol.n_thresholds, s->pol.thresholds, s->prompt[id]) : 0;
  s->class_queue[id] = q;
  if (s->q[q].n - s->q_head[q] >= (int64_t)s->cfg.max_queue) {
    s->rejected[id] = 1;
    s->rejected_total++;
    --s->outstanding;
    return;
  }
  VPUSH(s->q[q], id);
  for (int w = 0; w < s->cfg.n_prefill_workers; ++w) {
    if (!s->pw[w].busy && queue_of_worker(s, w) == q) {
      pull_next_prefill(s, w);
      break;
    }
  }
}

static void on_prefill_done(sim_t* s, const ev_t* ev) { /* :317-326 */
  pw_t* pw = &s->pw[ev->worker];
  if (ev->gen != pw->gen || pw->job != ev->req) return;
  s->prefill_end[ev->req] = s->now;
  pw->busy = 0;
  pw->job = -1;
  schedule(s, s->now + s->cfg.handoff_delay_ms, EV_ENQUEUE, -1, ev->req, 0.0, 0, 0);
  pull_next_prefill(s, ev->worker);
}

/* ---------------------------------------------------------------- decode pool */
static void start_decode_step(sim_t* s, int w) { /* :330-345 */
  dw_t* dw = &s->dw[w];
  while ((int)dw->active.n < s->cfg.max_batch && dw->p_head < dw->pending.n) {
    stream_t st = {dw->pending.v[dw->p_head++], 0, s->now};
    VPUSH(dw->active, st);
  }
  if (dw->active.n == 0) {
    ledger_set(&s->dled[w], &dw->ps, s->now, PH_IDLE, s->prof.p_idle_w);
    return;
  }
  dw->stepping = 1;
  const double step = decode_step_ms(&s->prof, (double)dw->active.n, dw->freq);
  schedule(s, s->now + step, EV_STEP_END, w, -1, 0.0, 0, 0);
  ledger_set(&s->dled[w], &dw->ps, s->now, PH_DECODE, gso_active_power_w(&s->prof, dw->freq));
}

static void on_decode_enqueue(sim_t* s, const ev_t* ev) { /* :347-363 */
  VPUSH(s->enq_t, s->now); /* the stream, in processing order */
  VPUSH(s->enq_req, ev->req);
  int best = 0;
  for (int w = 1; w < s->cfg.n_decode_workers; ++w) {
    const int64_t lw = s->dw[w].active.n + (s->dw[w].pending.n - s->dw[w].p_head);
    const int64_t lb = s->dw[best].active.n + (s->dw[best].pending.n - s->dw[best].p_head);
    if (lw < lb) best = w;
  }
  dw_t* dw = &s->dw[best];
  if (dw->active.n + (dw->pending.n - dw->p_head) >= (int64_t)s->cfg.max_queue) {
    s->rejected[ev->req] = 1;
    s->rejected_total++;
    --s->outstanding;
    return;
  }
  s->decode_worker[ev->req] = best;
  VPUSH(dw->pending, ev->req);
  if (!dw->stepping) start_decode_step(s, best);
}

static void on_decode_step_end(sim_t* s, const ev_t* ev) { /* :365-393 */
  dw_t* dw = &s->dw[ev->worker];
  dw->stepping = 0;
  s->n_steps++;
  const int emitted_tokens = (int)dw->active.n;
  int64_t keep = 0;
  for (int64_t i = 0; i < dw->active.n; ++i) {
    stream_t st = dw->active.v[i];
    const int64_t r = st.req;
    if (st.emitted == 0) {
      s->first_token[r] = s->now;
    } else {
      const double gap = s->now - st.last_emit;
      VPUSH(s->tbt[r], gap);
      ring_record(&dw->tbt, gap);
    }
    st.last_emit = s->now;
    ++st.emitted;
    if (st.emitted >= s->output[r]) {
      s->finish[r] = s->now;
      s->completed[r] = 1;
      --s->outstanding;
    } else {
      dw->active.v[keep++] = st;
    }
  }
  dw->active.n = keep;
  tpsev_t te = {s->now, emitted_tokens};
  VPUSH(dw->tps, te);
  start_decode_step(s, ev->worker);
}

/* ---------------------------------------------------------------- actuation */
static void command_freq(sim_t* s, int prefill_pool, int w, double f) { /* :397-404 */
  double* target = prefill_pool ? &s->pw[w].target : &s->dw[w].target;
  if (f == *target) return;
  *target = f;
  schedule(s, s->now + s->cfg.actuation_delay_ms, EV_FREQ, w, -1, f, 0, prefill_pool);
}

static void on_freq_applied(sim_t* s, const ev_t* ev) { /* :406-437 */
  if (ev->prefill_pool) {
    pw_t* pw = &s->pw[ev->worker];
    if (ev->f == pw->freq) return;
    const double f_old = pw->freq;
    pw->freq = ev->f;
    if (pw->busy) {
      const double elapsed = s->now - pw->job_upd;
      pw->job_rem -= elapsed * f_old / s->prof.f_ref_mhz;
      pw->job_rem = std_max(pw->job_rem, 0.0);
      pw->job_upd = s->now;
      ++pw->gen;
      schedule(s, s->now + pw->job_rem * s->prof.f_ref_mhz / pw->freq, EV_PREFILL_DONE, ev->worker,
               pw->job, 0.0, pw->gen, 1);
      ledger_set(&s->pled[ev->worker], &pw->ps, s->now, PH_PREFILL, active_prefill(s, pw->freq));
    }
    fc_t fc = {s->now, 1, ev->worker, ev->f};
    VPUSH(s->timeline, fc);
  } else {
    dw_t* dw = &s->dw[ev->worker];
    if (ev->f == dw->freq) return;
    dw->freq = ev->f;
    if (dw->stepping)
      ledger_set(&s->dled[ev->worker], &dw->ps, s->now, PH_DECODE,
                 gso_active_power_w(&s->prof, dw->freq));
    fc_t fc = {s->now, 0, ev->worker, ev->f};
    VPUSH(s->timeline, fc);
  }
}

/* ---------------------------------------------------------------- control ticks */
static void ctl_reserve(dw_t* dw) {
  if (dw->ctl.n_rec + 2 >= dw->log_cap) {
    dw->log_cap = dw->log_cap ? 2 * dw->log_cap : 4096;
    dw->log = (gso_decision*)realloc(dw->log, sizeof(gso_decision) * (size_t)dw->log_cap);
    dw->ctl.out = dw->log;
    dw->ctl.cap = dw->log_cap;
  }
}

/* TpsWindow::tps, decode_ctl.cpp:113-118 */
static double tps_now(dw_t* dw, double now, double window) {
  while (dw->t_head < dw->tps.n && dw->tps.v[dw->t_head].t < now - window) dw->t_head++;
  int tokens = 0;
  for (int64_t j = dw->t_head; j < dw->tps.n; ++j) tokens += dw->tps.v[j].tokens;
  return tokens * 1000.0 / window;
}

static void on_fine_tick(sim_t* s) { /* :441-451 */
  if (s->outstanding <= 0) return;
  for (int w = 0; w < s->cfg.n_decode_workers; ++w) {
    dw_t* dw = &s->dw[w];
    ctl_reserve(dw);
    const int has = dw->tbt.n > 0;
    ctl_fine(&dw->ctl, s->now, has, has ? ring_p95(&dw->tbt) : 0.0);
    command_freq(s, 0, w, dw->ctl.sp);
  }
  schedule(s, s->now + s->pol.decode_ctl.fine_period_ms, EV_FINE, -1, -1, 0.0, 0, 0);
}

static void on_coarse_tick(sim_t* s) { /* :453-458 */
  if (s->outstanding <= 0) return;
  for (int w = 0; w < s->cfg.n_decode_workers; ++w) {
    dw_t* dw = &s->dw[w];
    ctl_reserve(dw);
    ctl_coarse(&dw->ctl, s->now, tps_now(dw, s->now, s->pol.decode_ctl.coarse_period_ms));
  }
  schedule(s, s->now + s->pol.decode_ctl.coarse_period_ms, EV_COARSE, -1, -1, 0.0, 0, 0);
}

static void on_adapt_tick(sim_t* s) { /* :460-464 */
  if (s->outstanding <= 0) return;
  for (int w = 0; w < s->cfg.n_decode_workers; ++w) {
    ctl_reserve(&s->dw[w]);
    ctl_adapt(&s->dw[w].ctl, s->now);
  }
  schedule(s, s->now + s->pol.decode_ctl.adapt_period_s * 1000.0, EV_ADAPT, -1, -1, 0.0, 0, 0);
}

static double prefill_deadline(const sim_t* s, int64_t id) { /* :499-501 */
  return s->arrival[id] + ttft_for(&s->slo, s->cls[id]) - s->pol.prefill_opt.first_token_allowance_ms;
}

static void on_optimizer_tick(sim_t* s) { /* :466-497 */
  if (s->outstanding <= 0) return;
  VEC(int32_t) prompt = {0};
  VEC(double) dl = {0};
  VEC(double) wf = {0};
  for (int q = 0; q < s->n_queues; ++q) {
    prompt.n = dl.n = wf.n = 0;
    for (int w = 0; w < s->cfg.n_prefill_workers; ++w) {
      const pw_t* pw = &s->pw[w];
      if (!pw->busy || queue_of_worker(s, w) != q) continue;
      const double done = (s->now - pw->job_upd) * pw->freq / s->prof.f_ref_mhz;
      const double remaining = std_max(pw->job_rem - done, 0.0);
      VPUSH(prompt, s->prompt[pw->job]);
      VPUSH(dl, prefill_deadline(s, pw->job));
      VPUSH(wf, remaining / pw->job_t_ref);
      VPUSH(s->sj_run, 1);
      VPUSH(s->sj_rem, pw->job_rem);
      VPUSH(s->sj_upd, pw->job_upd);
      VPUSH(s->sj_freq, pw->freq);
      VPUSH(s->sj_tref, pw->job_t_ref);
    }
    for (int64_t k = s->q_head[q]; k < s->q[q].n; ++k) {
      const int64_t id = s->q[q].v[k];
      VPUSH(prompt, s->prompt[id]);
      VPUSH(dl, prefill_deadline(s, id));
      VPUSH(wf, 1.0);
      VPUSH(s->sj_run, 0);
      VPUSH(s->sj_rem, 0.0);
      VPUSH(s->sj_upd, 0.0);
      VPUSH(s->sj_freq, 0.0);
      VPUSH(s->sj_tref, 0.0);
    }
    if (prompt.n == 0) continue; /* queue_optimizer_tick skips empty queues, prefill_opt.cpp:64 */
    VPUSH(s->sn_now, s->now);
    VPUSH(s->sn_cls, q);
    VPUSH(s->sn_off, s->sj_prompt.n);
    for (int64_t k = 0; k < prompt.n; ++k) {
      VPUSH(s->sj_prompt, prompt.v[k]);
      VPUSH(s->sj_dl, dl.v[k]);
      VPUSH(s->sj_wf, wf.v[k]);
    }
    double f, window, e;
    int infeasible, fidx;
    gso_queue_tick_one(&s->prof, &s->pol.prefill_opt, prompt.n, prompt.v, dl.v, wf.v, s->now, &f,
                       &window, &infeasible, &fidx, &e);
    for (int w = 0; w < s->cfg.n_prefill_workers; ++w) {
      if (queue_of_worker(s, w) != q) continue;
      pc_t pc = {s->now, q, w, f, window, infeasible};
      VPUSH(s->commands, pc);
      command_freq(s, 1, w, f);
    }
  }
  free(prompt.v);
  free(dl.v);
  free(wf.v);
  schedule(s, s->now + s->pol.prefill_opt.resolve_period_ms, EV_OPT, -1, -1, 0.0, 0, 0);
}

/* ---------------------------------------------------------------- setup / teardown */
static int cmp_dec(const void* a, const void* b) { /* stable sort key (tick, worker), :521-525 */
  const gso_decision* x = (const gso_decision*)a;
  const gso_decision* y = (const gso_decision*)b;
  if (x->tick_ms != y->tick_ms) return x->tick_ms < y->tick_ms ? -1 : 1;
  if (x->worker != y->worker) return x->worker < y->worker ? -1 : 1;
  return x->pad_ < y->pad_ ? -1 : (x->pad_ > y->pad_); /* pad_ carries the merge position */
}

static void finalize(sim_t* s) { /* :503-530 */
  double end = 0.0;
  for (int64_t i = 0; i < s->n; ++i) {
    end = std_max(end, s->finish[i]);
    end = std_max(end, s->prefill_end[i]);
    end = std_max(end, s->arrival[i]);
  }
  for (int64_t k = 0; k < s->timeline.n; ++k) end = std_max(end, s->timeline.v[k].t);
  if (s->pool_only) end = std_max(end, s->end_floor);
  s->sim_end = end;
  for (int w = 0; w < s->cfg.n_prefill_workers; ++w) ledger_close(&s->pled[w], &s->pw[w].ps, end);
  for (int w = 0; w < s->cfg.n_decode_workers; ++w) ledger_close(&s->dled[w], &s->dw[w].ps, end);
  int64_t total = 0;
  for (int w = 0; w < s->cfg.n_decode_workers; ++w) total += s->dw[w].ctl.n_rec;
  s->decisions = (gso_decision*)malloc(sizeof(gso_decision) * (size_t)(total ? total : 1));
  s->n_decisions = 0;
  for (int w = 0; w < s->cfg.n_decode_workers; ++w)
    for (int64_t k = 0; k < s->dw[w].ctl.n_rec; ++k) {
      s->decisions[s->n_decisions] = s->dw[w].log[k];
      s->decisions[s->n_decisions].pad_ = (int32_t)s->n_decisions;
      s->n_decisions++;
    }
  qsort(s->decisions, (size_t)s->n_decisions, sizeof(gso_decision), cmp_dec);
  for (int64_t k = 0; k < s->n_decisions; ++k) s->decisions[k].pad_ = 0;
  /* end floor = the prefill side's part of sim_end (for gso_pool_run / K5) */
  double fl = 0.0;
  for (int64_t i = 0; i < s->n; ++i) {
    fl = std_max(fl, s->prefill_end[i]);
    fl = std_max(fl, s->arrival[i]);
  }
  for (int64_t k = 0; k < s->timeline.n; ++k)
    if (s->timeline.v[k].pool) fl = std_max(fl, s->timeline.v[k].t);
  if (!s->pool_only) s->end_floor = fl;
}

void gso_sim_free(void* h);

static sim_t* sim_alloc(const gso_profile* prof, const gso_policy* pol, const gso_slo* slo,
                        const gso_sim_cfg* cfg, int64_t n, const int64_t* arrival_ms,
                        const int32_t* prompt, const int32_t* output, const int8_t* cls,
                        char* err, size_t err_cap) {
  sim_t* s = (sim_t*)calloc(1, sizeof(sim_t));
  s->prof = *prof;
  s->pol = *pol;
  s->slo = *slo;
  s->cfg = *cfg;
  if (cfg->n_prefill_workers <= 0 || cfg->n_prefill_workers > 64 || cfg->n_decode_workers <= 0 ||
      cfg->max_batch <= 0 || cfg->max_queue <= 0 || n <= 0) {
    if (err && err_cap) snprintf(err, err_cap, "sim: bad configuration");
    free(s);
    return NULL;
  }
  for (int w = 0; w < cfg->n_prefill_workers; ++w) s->worker_map[w] = pol->worker_map ? pol->worker_map[w] : 0;
  s->pol.worker_map = s->worker_map;
  s->routing_enabled = routing_on(s);
  s->n_queues = s->routing_enabled ? pol->n_thresholds + 1 : 1;
  s->n = n;
#define A(f, T) s->f = (T*)calloc((size_t)n, sizeof(T))
  A(arrival_i, int64_t); A(prompt, int32_t); A(output, int32_t); A(class_queue, int32_t);
  A(prefill_worker, int32_t); A(decode_worker, int32_t); A(cls, int8_t); A(arrival, double);
  A(prefill_start, double); A(prefill_end, double); A(first_token, double); A(finish, double);
  A(completed, uint8_t); A(rejected, uint8_t);
#undef A
  s->tbt = calloc((size_t)n, sizeof(*s->tbt));
  for (int64_t i = 0; i < n; ++i) {
    s->arrival_i[i] = arrival_ms[i];
    s->arrival[i] = (double)arrival_ms[i];
    s->prompt[i] = prompt ? prompt[i] : 0;
    s->output[i] = output[i];
    s->cls[i] = req_class(cls ? cls[i] : -1, s->prompt[i]);
    s->prefill_worker[i] = s->decode_worker[i] = -1;
    s->prefill_start[i] = s->prefill_end[i] = s->first_token[i] = s->finish[i] = -1.0;
    s->class_queue[i] = 0;
  }
  s->q = calloc((size_t)s->n_queues, sizeof(*s->q));
  s->q_head = (int64_t*)calloc((size_t)s->n_queues, sizeof(int64_t));
  s->pw = (pw_t*)calloc((size_t)cfg->n_prefill_workers, sizeof(pw_t));
  s->dw = (dw_t*)calloc((size_t)cfg->n_decode_workers, sizeof(dw_t));
  s->pled = (ledger_t*)calloc((size_t)cfg->n_prefill_workers, sizeof(ledger_t));
  s->dled = (ledger_t*)calloc((size_t)cfg->n_decode_workers, sizeof(ledger_t));
  s->outstanding = n;
  /* Sim::init, simkernel.cpp:186-250 */
  if (dvfs(s)) {
    double levels[64];
    int nl = 0;
    for (double l = cfg->band_tps_lo; l <= cfg->band_tps_hi + 1e-9 && nl < 64; l += cfg->band_tps_step)
      levels[nl++] = l;
    const double t_slo_eff = pol->decode_ctl.tslo_ms * pol->decode_ctl.margin_decode;
    s->n_buckets = nl;
    s->tps_lo = (double*)malloc(sizeof(double) * (size_t)nl);
    s->tps_hi = (double*)malloc(sizeof(double) * (size_t)nl);
    s->f_opt_table = (double*)malloc(sizeof(double) * (size_t)nl);
    uint8_t feas[64];
    if (gso_build_band_table(prof, nl, levels, t_slo_eff, cfg->n_decode_workers, cfg->max_batch,
                             s->tps_lo, s->tps_hi, s->f_opt_table, feas) != 0) {
      if (err && err_cap) snprintf(err, err_cap, "sim: band table");
      gso_sim_free(s);
      return NULL;
    }
    gso_band_table tb = {nl, s->tps_lo, s->tps_hi, s->f_opt_table};
    for (int w = 0; w < cfg->n_decode_workers; ++w) {
      dw_t* dw = &s->dw[w];
      dw->log_cap = 4096;
      dw->log = (gso_decision*)malloc(sizeof(gso_decision) * (size_t)dw->log_cap);
      if (ctl_setup(&dw->ctl, &pol->decode_ctl, &tb, prof->f_min_mhz, prof->f_max_mhz, w, dw->log,
                    dw->log_cap) != 0) {
        if (err && err_cap) snprintf(err, err_cap, "sim: controller config");
        gso_sim_free(s);
        return NULL;
      }
    }
  }
  const double f0p = pol->kind == 1 ? pol->fixed_freq_mhz : prof->f_max_mhz;
  for (int w = 0; w < cfg->n_prefill_workers; ++w) {
    s->pw[w].freq = s->pw[w].target = f0p;
    s->pw[w].job = -1;
    s->pw[w].ps.power_w = idle_prefill(s);
    s->pw[w].ps.phase = PH_IDLE;
    fc_t fc = {0.0, 1, w, f0p};
    VPUSH(s->timeline, fc);
  }
  /* initial_decode_freq, :171-176 */
  const double f0d = pol->kind == 1 ? pol->fixed_freq_mhz
                     : (dvfs(s) ? s->dw[0].ctl.sp : prof->f_max_mhz);
  for (int w = 0; w < cfg->n_decode_workers; ++w) {
    dw_t* dw = &s->dw[w];
    dw->freq = dw->target = f0d;
    dw->ps.power_w = prof->p_idle_w;
    dw->ps.phase = PH_IDLE;
    const int cap = pol->decode_ctl.tbt_window_tokens > 0 ? pol->decode_ctl.tbt_window_tokens : 256;
    dw->tbt.cap = cap;
    dw->tbt.buf = (double*)malloc(sizeof(double) * (size_t)cap);
    dw->tbt.scratch = (double*)malloc(sizeof(double) * (size_t)cap);
    fc_t fc = {0.0, 0, w, f0d};
    VPUSH(s->timeline, fc);
  }
  return s;
}

static void sim_loop(sim_t* s) { /* Sim::run_loop, simkernel.cpp:150-169 */
  while (s->heap.n > 0) {
    const ev_t ev = heap_pop(&s->heap);
    s->now = ev.t;
    switch (ev.kind) {
      case EV_ARRIVAL: on_arrival(s, &ev); break;
      case EV_PREFILL_DONE: on_prefill_done(s, &ev); break;
      case EV_STEP_END: on_decode_step_end(s, &ev); break;
      case EV_ENQUEUE: on_decode_enqueue(s, &ev); break;
      case EV_FREQ: on_freq_applied(s, &ev); break;
      case EV_COARSE: on_coarse_tick(s); break;
      case EV_ADAPT: on_adapt_tick(s); break;
      case EV_FINE: on_fine_tick(s); break;
      case EV_OPT: on_optimizer_tick(s); break;
    }
  }
  finalize(s);
}

static void schedule_ticks(sim_t* s, int with_optimizer) { /* :243-248 */
  if (!dvfs(s)) return;
  schedule(s, s->pol.decode_ctl.fine_period_ms, EV_FINE, -1, -1, 0.0, 0, 0);
  schedule(s, s->pol.decode_ctl.coarse_period_ms, EV_COARSE, -1, -1, 0.0, 0, 0);
  schedule(s, s->pol.decode_ctl.adapt_period_s * 1000.0, EV_ADAPT, -1, -1, 0.0, 0, 0);
  if (with_optimizer)
    schedule(s, s->pol.prefill_opt.resolve_period_ms, EV_OPT, -1, -1, 0.0, 0, 0);
}

void* gso_sim_run(const gso_profile* prof, const gso_policy* pol, const gso_slo* slo,
                  const gso_sim_cfg* cfg, int64_t n, const int64_t* arrival_ms,
                  const int32_t* prompt, const int32_t* output, const int8_t* cls,
                  int64_t n_scripted, const gso_scripted* scripted, char* err, size_t err_cap) {
  sim_t* s = sim_alloc(prof, pol, slo, cfg, n, arrival_ms, prompt, output, cls, err, err_cap);
  if (!s) return NULL;
  for (int64_t i = 0; i < n; ++i) {
    schedule(s, s->arrival[i], EV_ARRIVAL, -1, i, 0.0, 0, 0);
    s->last_arrival = std_max(s->last_arrival, s->arrival[i]);
  }
  for (int64_t k = 0; k < n_scripted; ++k)
    schedule(s, scripted[k].time_ms + cfg->actuation_delay_ms, EV_FREQ, scripted[k].worker, -1,
             scripted[k].f_mhz, 0, scripted[k].prefill_pool);
  schedule_ticks(s, 1);
  sim_loop(s);
  return s;
}

void* gso_pool_run(const gso_profile* prof, const gso_policy* pol, const gso_slo* slo,
                   const gso_sim_cfg* cfg, int64_t n, const int64_t* arrival_ms,
                   const int32_t* prompt, const int32_t* output, const int8_t* cls,
                   int64_t n_stream, const double* enq_t, const int64_t* enq_req,
                   double end_floor_ms, char* err, size_t err_cap) {
  sim_t* s = sim_alloc(prof, pol, slo, cfg, n, arrival_ms, prompt, output, cls, err, err_cap);
  if (!s) return NULL;
  s->pool_only = 1;
  s->end_floor = end_floor_ms;
  /* Requests not in the stream were rejected by the prefill side before the stream's last
   * enqueue, so outstanding <= 0 exactly when every streamed request is done. */
  s->outstanding = n_stream;
  for (int64_t i = 0; i < n; ++i) s->last_arrival = std_max(s->last_arrival, s->arrival[i]);
  for (int64_t k = 0; k < n_stream; ++k) {
    s->prefill_end[enq_req[k]] = 0.0; /* marker "reached the decode pool"; end_floor covers
                                         the prefill side's part of sim_end */
    schedule(s, enq_t[k], EV_ENQUEUE, -1, enq_req[k], 0.0, 0, 0);
  }
  schedule_ticks(s, 0);
  sim_loop(s);
  return s;
}

void gso_sim_free(void* h) {
  sim_t* s = (sim_t*)h;
  if (!s) return;
  free(s->arrival_i); free(s->prompt); free(s->output); free(s->class_queue);
  free(s->prefill_worker); free(s->decode_worker); free(s->cls); free(s->arrival);
  free(s->prefill_start); free(s->prefill_end); free(s->first_token); free(s->finish);
  free(s->completed); free(s->rejected);
  if (s->tbt)
    for (int64_t i = 0; i < s->n; ++i) free(s->tbt[i].v);
  free(s->tbt);
  for (int q = 0; q < s->n_queues && s->q; ++q) free(s->q[q].v);
  free(s->q); free(s->q_head); free(s->pw);
  for (int w = 0; w < s->cfg.n_decode_workers && s->dw; ++w) {
    free(s->dw[w].active.v); free(s->dw[w].pending.v); free(s->dw[w].tps.v);
    free(s->dw[w].tbt.buf); free(s->dw[w].tbt.scratch); free(s->dw[w].log); free(s->dw[w].ctl.f_opt);
  }
  free(s->dw); free(s->pled); free(s->dled); free(s->f_opt_table); free(s->tps_lo); free(s->tps_hi);
  free(s->heap.v); free(s->timeline.v); free(s->commands.v); free(s->enq_t.v); free(s->enq_req.v);
  free(s->sn_now.v); free(s->sn_cls.v); free(s->sn_off.v); free(s->sj_prompt.v); free(s->sj_run.v);
  free(s->sj_dl.v); free(s->sj_rem.v); free(s->sj_upd.v); free(s->sj_freq.v); free(s->sj_tref.v);
  free(s->sj_wf.v);
  free(s->decisions);
  free(s);
}

void gso_sim_snapshot_sizes(void* h, int64_t* n_snap, int64_t* n_jobs) {
  const sim_t* s = (const sim_t*)h;
  *n_snap = s->sn_now.n;
  *n_jobs = s->sj_prompt.n;
}

void gso_sim_snapshots(void* h, double* now, int32_t* cls, int64_t* off, int32_t* prompt,
                       double* deadline, uint8_t* running, double* rem_ref, double* upd_ms,
                       double* freq, double* t_ref, double* wf) {
  const sim_t* s = (const sim_t*)h;
  for (int64_t i = 0; i < s->sn_now.n; ++i) {
    now[i] = s->sn_now.v[i];
    cls[i] = s->sn_cls.v[i];
    off[i] = s->sn_off.v[i];
  }
  off[s->sn_now.n] = s->sj_prompt.n;
  for (int64_t j = 0; j < s->sj_prompt.n; ++j) {
    prompt[j] = s->sj_prompt.v[j];
    deadline[j] = s->sj_dl.v[j];
    running[j] = s->sj_run.v[j];
    rem_ref[j] = s->sj_rem.v[j];
    upd_ms[j] = s->sj_upd.v[j];
    freq[j] = s->sj_freq.v[j];
    t_ref[j] = s->sj_tref.v[j];
    wf[j] = s->sj_wf.v[j];
  }
}

void gso_sim_sizes(void* h, int64_t* z) {
  const sim_t* s = (const sim_t*)h;
  int64_t nt = 0;
  for (int64_t i = 0; i < s->n; ++i) nt += s->tbt[i].n;
  z[0] = s->n; z[1] = nt; z[2] = s->n_decisions; z[3] = s->timeline.n; z[4] = s->commands.n;
  z[5] = s->enq_t.n; z[6] = s->cfg.n_prefill_workers; z[7] = s->cfg.n_decode_workers;
  z[8] = s->rejected_total; z[9] = s->n_steps;
}

void gso_sim_requests(void* h, int32_t* class_queue, int32_t* prefill_worker,
                      int32_t* decode_worker, double* prefill_start, double* prefill_end,
                      double* first_token, double* finish, uint8_t* completed, uint8_t* rejected,
                      int8_t* cls) {
  const sim_t* s = (const sim_t*)h;
  const size_t n = (size_t)s->n;
  memcpy(class_queue, s->class_queue, 4 * n);
  memcpy(prefill_worker, s->prefill_worker, 4 * n);
  memcpy(decode_worker, s->decode_worker, 4 * n);
  memcpy(prefill_start, s->prefill_start, 8 * n);
  memcpy(prefill_end, s->prefill_end, 8 * n);
  memcpy(first_token, s->first_token, 8 * n);
  memcpy(finish, s->finish, 8 * n);
  memcpy(completed, s->completed, n);
  memcpy(rejected, s->rejected, n);
  memcpy(cls, s->cls, n);
  /* gso_pool_run does not simulate the prefill side: prefill_start stays -1 and
   * prefill_end is 0 for every streamed request (a "reached decode" marker) */
}

void gso_sim_tbt(void* h, int64_t* off, double* samples) {
  const sim_t* s = (const sim_t*)h;
  off[0] = 0;
  for (int64_t i = 0; i < s->n; ++i) {
    memcpy(samples + off[i], s->tbt[i].v, sizeof(double) * (size_t)s->tbt[i].n);
    off[i + 1] = off[i] + s->tbt[i].n;
  }
}

void gso_sim_ledgers(void* h, double* p3, double* d3, int64_t* n_int) {
  const sim_t* s = (const sim_t*)h;
  for (int w = 0; w < s->cfg.n_prefill_workers; ++w) {
    p3[3 * w] = s->pled[w].act_prefill; p3[3 * w + 1] = s->pled[w].act_decode; p3[3 * w + 2] = s->pled[w].idle;
    n_int[w] = s->pled[w].n_int;
  }
  for (int w = 0; w < s->cfg.n_decode_workers; ++w) {
    d3[3 * w] = s->dled[w].act_prefill; d3[3 * w + 1] = s->dled[w].act_decode; d3[3 * w + 2] = s->dled[w].idle;
    n_int[s->cfg.n_prefill_workers + w] = s->dled[w].n_int;
  }
}

void gso_sim_decisions(void* h, gso_decision* out) {
  const sim_t* s = (const sim_t*)h;
  memcpy(out, s->decisions, sizeof(gso_decision) * (size_t)s->n_decisions);
}

void gso_sim_timeline(void* h, double* t, uint8_t* pool, int32_t* worker, double* f) {
  const sim_t* s = (const sim_t*)h;
  for (int64_t k = 0; k < s->timeline.n; ++k) {
    t[k] = s->timeline.v[k].t; pool[k] = (uint8_t)s->timeline.v[k].pool;
    worker[k] = s->timeline.v[k].worker; f[k] = s->timeline.v[k].f;
  }
}

void gso_sim_commands(void* h, double* tick, int32_t* cls, int32_t* worker, double* f,
                      double* window, uint8_t* infeasible) {
  const sim_t* s = (const sim_t*)h;
  for (int64_t k = 0; k < s->commands.n; ++k) {
    const pc_t* c = &s->commands.v[k];
    tick[k] = c->tick; cls[k] = c->cls; worker[k] = c->worker; f[k] = c->f; window[k] = c->window;
    infeasible[k] = (uint8_t)c->infeasible;
  }
}

void gso_sim_enqueue(void* h, double* t, int64_t* req) {
  const sim_t* s = (const sim_t*)h;
  memcpy(t, s->enq_t.v, sizeof(double) * (size_t)s->enq_t.n);
  memcpy(req, s->enq_req.v, sizeof(int64_t) * (size_t)s->enq_req.n);
}

void gso_sim_scalars(void* h, double* d) {
  const sim_t* s = (const sim_t*)h;
  d[0] = s->sim_end; d[1] = s->last_arrival; d[2] = s->end_floor;
}

/* ---------------------------------------------------------------- K5 summary */
static uint64_t fnv(uint64_t h, uint64_t w) { return (h ^ w) * 0x100000001b3ull; }
static uint64_t bits(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
#define FNV0 0xcbf29ce484222325ull

void gso_pool_summary_from(const gso_slo* slo, int64_t n, const double* arrival,
                           const int8_t* cls, const int32_t* decode_worker,
                           const double* prefill_end, const double* first_token,
                           const double* finish, const uint8_t* completed,
                           const uint8_t* rejected, const int64_t* tbt_off, const double* tbt,
                           int n_decode, const double* decode3, int64_t n_dec,
                           const gso_decision* dec, int64_t n_tl, const double* tl_t,
                           const uint8_t* tl_pool, const int32_t* tl_worker, const double* tl_f,
                           double sim_end_ms, int64_t n_steps, gso_pool_summary* o) {
  memset(o, 0, sizeof(*o));
  /* RunResult::decode_pool_j (simkernel.cpp:617-621) with WorkerLedger::total_j */
  double e = 0.0, act = 0.0, idle = 0.0;
  for (int w = 0; w < n_decode; ++w) {
    e += decode3[3 * w] + decode3[3 * w + 1] + decode3[3 * w + 2];
    act += decode3[3 * w + 1];
    idle += decode3[3 * w + 2];
  }
  o->decode_pool_j = e;
  o->active_decode_j = act;
  o->idle_j = idle;
  o->sim_end_ms = sim_end_ms;
  o->n_steps = n_steps;
  uint64_t rd = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (completed[i]) {
      /* slo_pass_rates, metrics.cpp:42-72 */
      o->n_completed++;
      if (first_token[i] - arrival[i] <= ttft_for(slo, cls[i])) o->n_ttft_ok++;
      const int64_t ng = tbt_off[i + 1] - tbt_off[i];
      if (ng == 0 || gso_quantile(ng, tbt + tbt_off[i], 0.95) <= slo->tbt_p95_ms) o->n_tbt_ok++;
      for (int64_t k = tbt_off[i]; k < tbt_off[i + 1]; ++k) {
        o->tbt_samples++;
        if (tbt[k] <= slo->tbt_p95_ms) o->tbt_samples_ok++;
      }
      uint64_t gs = 0; /* sum of the gaps' bit patterns mod 2^64 */
      for (int64_t k = tbt_off[i]; k < tbt_off[i + 1]; ++k) gs += bits(tbt[k]);
      uint64_t h = fnv(FNV0, (uint64_t)i);
      h = fnv(h, bits(first_token[i]));
      h = fnv(h, bits(finish[i]));
      h = fnv(h, (uint64_t)(uint32_t)decode_worker[i]);
      h = fnv(h, (uint64_t)ng);
      h = fnv(h, gs);
      rd += h;
    } else if (rejected[i] && prefill_end[i] >= 0.0) { /* decode-side rejection */
      o->n_rejected++;
      rd += fnv(fnv(FNV0, (uint64_t)i), 0xdeadull);
    }
  }
  o->request_digest = rd;
  /* decisions: per worker chain in log order (stable merge keeps it), then combine */
  uint64_t dd = FNV0;
  for (int w = 0; w < n_decode; ++w) {
    uint64_t h = FNV0;
    for (int64_t k = 0; k < n_dec; ++k) {
      if (dec[k].worker != w) continue;
      h = fnv(h, bits(dec[k].command_mhz));
      const uint64_t w2 = bits(dec[k].band_lo) ^ (bits(dec[k].band_hi) << 13) ^
                          ((uint64_t)(uint32_t)dec[k].bucket << 48) ^
                          ((uint64_t)(uint32_t)dec[k].action << 56);
      h = fnv(h, w2);
    }
    dd = fnv(dd, h);
  }
  o->decision_digest = dd;
  o->n_decisions = n_dec;
  /* decode rows of the freq timeline; the first n_decode decode rows are the t = 0 rows */
  uint64_t fd = FNV0;
  int64_t nf = 0;
  for (int w = 0; w < n_decode; ++w) {
    uint64_t h = FNV0;
    int seen_initial = 0;
    for (int64_t k = 0; k < n_tl; ++k) {
      if (tl_pool[k] || tl_worker[k] != w) continue;
      if (!seen_initial) { seen_initial = 1; continue; }
      h = fnv(fnv(h, bits(tl_t[k])), bits(tl_f[k]));
      nf++;
    }
    fd = fnv(fd, h);
  }
  o->freq_digest = fd;
  o->n_freq_changes = nf;
}

void gso_sim_summary(void* h, const gso_slo* slo, gso_pool_summary* out) {
  sim_t* s = (sim_t*)h;
  int64_t z[10];
  gso_sim_sizes(h, z);
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(s->n + 1));
  double* tb = (double*)malloc(sizeof(double) * (size_t)(z[1] ? z[1] : 1));
  gso_sim_tbt(h, off, tb);
  double* t = (double*)malloc(sizeof(double) * (size_t)z[3]);
  double* f = (double*)malloc(sizeof(double) * (size_t)z[3]);
  uint8_t* pool = (uint8_t*)malloc((size_t)z[3]);
  int32_t* wk = (int32_t*)malloc(sizeof(int32_t) * (size_t)z[3]);
  gso_sim_timeline(h, t, pool, wk, f);
  double* d3 = (double*)malloc(sizeof(double) * 3 * (size_t)s->cfg.n_decode_workers);
  for (int w = 0; w < s->cfg.n_decode_workers; ++w) {
    d3[3 * w] = s->dled[w].act_prefill; d3[3 * w + 1] = s->dled[w].act_decode; d3[3 * w + 2] = s->dled[w].idle;
  }
  gso_pool_summary_from(slo, s->n, s->arrival, s->cls, s->decode_worker, s->prefill_end,
                        s->first_token, s->finish, s->completed, s->rejected, off, tb,
                        s->cfg.n_decode_workers, d3, s->n_decisions, s->decisions, z[3], t, pool,
                        wk, f, s->sim_end, s->n_steps, out);
  free(off); free(tb); free(t); free(f); free(pool); free(wk); free(d3);
}
