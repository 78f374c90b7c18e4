/*
 * gs_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference's
 * decision-engine hot path, used as the parity checker and as a CPU baseline.
 * Every function cites the reference file:line it restates (paths under
 * /root/reference/proj). Compiled with -ffp-contract=off: the operation order below
 * IS the specification; do not "simplify" an expression.
 *
 * std::min(a,b) is (b < a) ? b : a, std::max(a,b) is (a < b) ? b : a and
 * std::clamp(v,lo,hi) is v < lo ? lo : (hi < v ? hi : v); the helpers below keep those
 * exact comparison directions.
 */
#include "gs_oracle.h"
#include "gs_oracle_int.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

GSO_INTERNAL double std_min(double a, double b) { return (b < a) ? b : a; }
GSO_INTERNAL double std_max(double a, double b) { return (a < b) ? b : a; }
GSO_INTERNAL double std_clamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* ---------------- grid and models (gpu_model.cpp, gpu_model.hpp) ---------------- */

/* FrequencyGrid::on_grid, gpu_model.cpp:18-22 */
GSO_INTERNAL int on_grid(const gso_profile* p, double f) {
  if (f < p->f_min_mhz - 1e-9 || f > p->f_max_mhz + 1e-9) return 0;
  const double k = (f - p->f_min_mhz) / p->step_mhz;
  return fabs(k - round(k)) < 1e-9;
}

/* FrequencyGrid::size, gpu_model.cpp:24-26 */
int gso_grid_size(const gso_profile* p) {
  return (int)(size_t)round((p->f_max_mhz - p->f_min_mhz) / p->step_mhz) + 1;
}

/* FrequencyGrid::at, gpu_model.cpp:28 */
double gso_grid_at(const gso_profile* p, int i) { return p->f_min_mhz + p->step_mhz * (double)i; }

/* PowerModel::active_power_w, gpu_model.hpp:64 */
double gso_active_power_w(const gso_profile* p, double f) {
  return ((p->k3 * f + p->k2) * f + p->k1) * f + p->k0;
}

/* prefill_latency_raw_ms t_ref part, gpu_model.cpp:96-99 */
static double lat_t_ref(const gso_profile* p, double L) { return (p->lat_a * L + p->lat_b) * L + p->lat_c; }

/* GpuProfile::validate and the per-model validators, gpu_model.cpp:9-16, 42-87 */
int gso_profile_validate(const gso_profile* p) {
  /* FrequencyGrid::validate :9-16 */
  if (p->f_min_mhz <= 0.0 || p->f_max_mhz <= p->f_min_mhz) return -1;
  if (p->step_mhz <= 0.0) return -1;
  {
    const double steps = (p->f_max_mhz - p->f_min_mhz) / p->step_mhz;
    if (fabs(steps - round(steps)) > 1e-9) return -1;
    if (!on_grid(p, p->f_ref_mhz)) return -1;
  }
  /* LatencyModel::validate :42-56 (raw latency at f_ref is t_ref*f_ref/f_ref) */
  if (p->lat_a < 0.0) return -1;
  if (p->lat_f_ref_mhz <= 0.0) return -1;
  {
    static const double probes[5] = {1.0, 256.0, 1024.0, 8192.0, 65536.0};
    for (int i = 0; i < 5; ++i)
      if (lat_t_ref(p, probes[i]) * p->lat_f_ref_mhz / p->lat_f_ref_mhz <= 0.0) return -1;
    if (p->lat_a > 0.0 && p->lat_b < 0.0) {
      const double vertex = -p->lat_b / (2.0 * p->lat_a);
      if (vertex >= 1.0 && vertex <= 65536.0 &&
          p->lat_a * vertex * vertex + p->lat_b * vertex + p->lat_c <= 0.0)
        return -1;
    }
  }
  /* DecodeStepModel::validate :58-64 */
  if (p->dec_alpha0_ms < 0 || p->dec_alpha1_ms < 0 || p->dec_beta0_ms < 0 || p->dec_beta1_ms < 0)
    return -1;
  if (p->dec_f_ref_mhz <= 0.0) return -1;
  if (p->dec_alpha0_ms + p->dec_alpha1_ms + p->dec_beta0_ms + p->dec_beta1_ms <= 0.0) return -1;
  /* PowerModel::validate :66-78 */
  if (p->p_idle_w <= 0.0) return -1;
  {
    double prev = -1.0;
    const int n = gso_grid_size(p);
    for (int i = 0; i < n; ++i) {
      const double pw = gso_active_power_w(p, gso_grid_at(p, i));
      if (pw <= p->p_idle_w) return -1;
      if (pw <= prev) return -1;
      prev = pw;
    }
  }
  /* GpuProfile::validate :85-86 */
  if (p->lat_f_ref_mhz != p->f_ref_mhz || p->dec_f_ref_mhz != p->f_ref_mhz) return -1;
  return 0;
}

/* ---------------- prefill objective (prefill_opt.cpp) ---------------- */

/* PrefillBatch::t_ref_total_ms, prefill_opt.cpp:9-14 (left-to-right, snapshot order) */
double gso_t_ref_total_ms(const gso_profile* p, int64_t n, const int32_t* prompt, const double* wf) {
  double total = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    const double L = (double)prompt[k];
    total += (wf ? wf[k] : 1.0) * ((p->lat_a * L + p->lat_b) * L + p->lat_c);
  }
  return total;
}

/* energy_total on a precomputed T_ref: busy_time_ms :19, energy_total :24-29 */
static void energy_from_t(const gso_profile* p, double t_ref, double f, double window,
                          double* active, double* idle, double* total, int* feasible) {
  const double busy = t_ref * p->f_ref_mhz / f;
  *feasible = busy <= window;
  *active = gso_active_power_w(p, f) * busy / 1000.0;
  *idle = p->p_idle_w * (window - busy) / 1000.0;
  *total = *active + *idle;
}

/* energy_total, prefill_opt.cpp:22-31 (busy_time_ms :16-20 throws on empty / off-grid) */
int gso_energy_total(const gso_profile* p, int64_t n, const int32_t* prompt, const double* wf,
                     double f, double window_ms, double* active_j, double* idle_j,
                     double* total_j, int* feasible) {
  if (n <= 0 || !on_grid(p, f)) return -1;
  energy_from_t(p, gso_t_ref_total_ms(p, n, prompt, wf), f, window_ms, active_j, idle_j, total_j,
                feasible);
  return 0;
}

/* energy_total_closed_form_j, prefill_opt.cpp:33-43 */
double gso_energy_closed_form(const gso_profile* p, int64_t n, const int32_t* prompt,
                              const double* wf, double f, double window_ms) {
  const double t_ref = gso_t_ref_total_ms(p, n, prompt, wf);
  const double f_ref = p->f_ref_mhz;
  const double active = f_ref * t_ref * (p->k3 * f * f + p->k2 * f + p->k1 + p->k0 / f) / 1000.0;
  const double idle = p->p_idle_w * (window_ms - f_ref * t_ref / f) / 1000.0;
  return active + idle;
}

/* select_frequency, prefill_opt.cpp:45-56 — ascending scan, strict '<' keeps the lowest f */
int gso_select_frequency_t(const gso_profile* p, double t_ref, double window_ms, double* f_out,
                           double* e_out) {
  int best = -1;
  double best_e = 0.0;
  const int G = gso_grid_size(p);
  for (int i = 0; i < G; ++i) {
    const double f = gso_grid_at(p, i);
    double a, idl, tot;
    int feas;
    energy_from_t(p, t_ref, f, window_ms, &a, &idl, &tot, &feas);
    if (!feas) continue;
    if (best < 0 || tot < best_e) {
      best = i;
      best_e = tot;
    }
  }
  if (best >= 0) {
    if (f_out) *f_out = gso_grid_at(p, best);
    if (e_out) *e_out = best_e;
  }
  return best;
}

int gso_select_frequency(const gso_profile* p, int64_t n, const int32_t* prompt, const double* wf,
                         double window_ms, double* f_out, double* e_out) {
  if (n <= 0) return -2; /* busy_time_ms throws ModelError on an empty batch */
  return gso_select_frequency_t(p, gso_t_ref_total_ms(p, n, prompt, wf), window_ms, f_out, e_out);
}

/* queue_optimizer_tick body for one non-empty queue, prefill_opt.cpp:63-80 */
void gso_queue_tick_one(const gso_profile* p, const gso_qopt_cfg* cfg, int64_t n,
                        const int32_t* prompt, const double* deadline, const double* wf,
                        double now_ms, double* f_out, double* window_out, int* infeasible_out,
                        int* f_idx_out, double* e_out) {
  double min_slack = INFINITY;
  for (int64_t k = 0; k < n; ++k) min_slack = std_min(min_slack, deadline[k] - now_ms);
  const double window = std_max(cfg->margin_prefill * min_slack, cfg->min_budget_ms);
  double f = 0.0, e = 0.0;
  const int idx = gso_select_frequency(p, n, prompt, wf, window, &f, &e);
  *window_out = window;
  if (idx >= 0) {
    *f_out = f;
    *infeasible_out = 0;
  } else {
    *f_out = p->f_max_mhz;
    *infeasible_out = 1;
  }
  if (f_idx_out) *f_idx_out = idx;
  if (e_out) *e_out = idx >= 0 ? e : 0.0;
}

/* ---------------- routing (router.cpp, simkernel.cpp) ---------------- */

/* classify, router.cpp:26-31 */
int gso_classify(int n_thr, const int32_t* thresholds, int32_t prompt) {
  int c = 0;
  for (int i = 0; i < n_thr; ++i)
    if (thresholds[i] < prompt) ++c;
  return c;
}

/*
 * Offline window binning (SURVEY.md 8(d) convention). Per request: queue class
 * (router.cpp:26-31) and SLO class SM iff prompt <= 1024 (simkernel.cpp:113-116,258-260).
 * Per cell (window, class): job count, T_ref summed left-to-right in arrival order
 * (prefill_opt.cpp:9-14 with work_fraction = 1), minimum prefill deadline
 * (arrival + TTFT(SM/L)) - allowance (simkernel.cpp:499-501), and the stable FIFO of
 * request indices per cell (Dispatcher::dispatch, router.cpp:37-43).
 */
int gso_route_bin(int64_t n_req, const int64_t* arrival_ms, const int32_t* prompt, int n_thr,
                  const int32_t* thresholds, int64_t window_ms, int64_t w0, int64_t n_windows,
                  int n_profiles, const gso_profile* profiles, double ttft_sm_ms, double ttft_l_ms,
                  double first_token_allowance_ms, uint8_t* cls_out, uint32_t* cell_count,
                  double* cell_t_ref, double* cell_min_deadline, int64_t* fifo_out) {
  const int C = n_thr + 1;
  const int64_t cells = n_windows * C;
  for (int64_t c = 0; c < cells; ++c) {
    cell_count[c] = 0;
    cell_min_deadline[c] = INFINITY;
    for (int p = 0; p < n_profiles; ++p) cell_t_ref[(int64_t)p * cells + c] = 0.0;
  }
  for (int64_t i = 0; i < n_req; ++i) {
    const int cls = gso_classify(n_thr, thresholds, prompt[i]);
    cls_out[i] = (uint8_t)cls;
    const int64_t w = arrival_ms[i] / window_ms - w0;
    if (w < 0 || w >= n_windows) continue;
    const int64_t cell = w * C + cls;
    cell_count[cell] += 1;
    const double L = (double)prompt[i];
    for (int p = 0; p < n_profiles; ++p) {
      const gso_profile* pr = &profiles[p];
      cell_t_ref[(int64_t)p * cells + cell] += 1.0 * ((pr->lat_a * L + pr->lat_b) * L + pr->lat_c);
    }
    const double ttft = prompt[i] <= 1024 ? ttft_sm_ms : ttft_l_ms;
    const double dl = (double)arrival_ms[i] + ttft - first_token_allowance_ms;
    cell_min_deadline[cell] = std_min(cell_min_deadline[cell], dl);
  }
  if (fifo_out) {
    /* exclusive prefix over cells, then a stable pass in arrival order */
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cells + 1));
    if (!pos) return -1;
    int64_t acc = 0;
    for (int64_t c = 0; c < cells; ++c) {
      pos[c] = acc;
      acc += cell_count[c];
    }
    for (int64_t i = 0; i < n_req; ++i) {
      const int64_t w = arrival_ms[i] / window_ms - w0;
      if (w < 0 || w >= n_windows) continue;
      fifo_out[pos[w * C + cls_out[i]]++] = i;
    }
    free(pos);
  }
  return 0;
}

/* ---------------- decode control (decode_ctl.cpp, metrics.cpp) ---------------- */

GSO_INTERNAL int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* quantile, metrics.cpp:11-19 (nearest rank; the sample value is sort-independent) */
double gso_quantile(int64_t n, const double* samples, double q) {
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(s, samples, sizeof(double) * (size_t)n);
  qsort(s, (size_t)n, sizeof(double), cmp_double);
  const size_t rank = (size_t)ceil(q * (double)n);
  const double v = s[rank == 0 ? 0 : rank - 1];
  free(s);
  return v;
}

/* decode_steady_state, decode_ctl.cpp:28-50 */
int gso_decode_steady_state(const gso_profile* p, double tps, double f, int max_batch,
                            double* batch, double* tbt_ms) {
  const double fr = p->dec_f_ref_mhz / f;
  const double s0 = p->dec_alpha0_ms + p->dec_beta0_ms * fr;
  const double s1 = p->dec_alpha1_ms + p->dec_beta1_ms * fr;
  const double cap_tps = 1000.0 * max_batch / (s0 + s1 * max_batch);
  if (tps > cap_tps) {
    *batch = max_batch;
    *tbt_ms = s0 + s1 * max_batch;
    return 0;
  }
  const double denom = 1000.0 - tps * s1;
  double b = denom > 0 ? tps * s0 / denom : (double)max_batch;
  b = std_clamp(b, 1.0, (double)max_batch);
  *batch = b;
  *tbt_ms = s0 + s1 * b;
  return 1;
}

/* build_band_table, decode_ctl.cpp:76-111 (+ FreqBandTable::validate :64-74) */
int gso_build_band_table(const gso_profile* p, int n, const double* levels, double t_slo_ms,
                         int workers, int max_batch, double* tps_lo, double* tps_hi,
                         double* f_opt, uint8_t* feasible) {
  if (n <= 0) return -1;
  for (int i = 0; i + 1 < n; ++i)
    if (levels[i] >= levels[i + 1]) return -1;
  if (workers < 1 || max_batch < 1) return -1;
  const int G = gso_grid_size(p);
  for (int i = 0; i < n; ++i) {
    tps_lo[i] = i == 0 ? 0.0 : 0.5 * (levels[i - 1] + levels[i]);
    tps_hi[i] = i + 1 < n ? 0.5 * (levels[i] + levels[i + 1]) : INFINITY;
    const double tau_w = levels[i] / workers;
    double best_f = 0.0, best_energy = 0.0;
    int found = 0;
    for (int k = 0; k < G; ++k) {
      const double f = gso_grid_at(p, k);
      double b, tbt;
      const int sust = gso_decode_steady_state(p, tau_w, f, max_batch, &b, &tbt);
      if (!sust || tbt > t_slo_ms) continue;
      const double ept = gso_active_power_w(p, f) / levels[i];
      if (!found || ept < best_energy) {
        best_f = f;
        best_energy = ept;
        found = 1;
      }
    }
    feasible[i] = (uint8_t)found;
    f_opt[i] = found ? best_f : p->f_max_mhz;
  }
  /* FreqBandTable::validate */
  if (tps_lo[0] != 0.0) return -1;
  for (int i = 0; i + 1 < n; ++i) {
    if (tps_hi[i] != tps_lo[i + 1]) return -1;
    if (tps_lo[i] >= tps_hi[i]) return -1;
  }
  if (tps_hi[n - 1] != INFINITY) return -1;
  return 0;
}

/* DecodeCtlConfig::validate, decode_ctl.cpp:12-26 */
int gso_ctl_cfg_validate(const gso_ctl_cfg* c) {
  if (c->tslo_ms <= 0) return -1;
  if (c->margin_decode < 0.2 || c->margin_decode > 2.0) return -1;
  if (c->fine_period_ms <= 0 || c->coarse_period_ms <= 0 || c->adapt_period_s <= 0) return -1;
  if (c->step_mhz <= 0 || c->max_step_mhz < c->step_mhz) return -1;
  if (c->hysteresis_count < 1) return -1;
  if (c->bias_threshold <= 0 || c->bias_threshold >= 1) return -1;
  if (c->tbt_window_tokens < 1) return -1;
  if (c->tps_scale <= 0) return -1;
  if (c->lower_margin >= c->upper_margin) return -1;
  return 0;
}

GSO_INTERNAL int table_validate(const gso_band_table* t) {
  if (t->n <= 0) return -1;
  if (t->tps_lo[0] != 0.0) return -1;
  for (int i = 0; i + 1 < t->n; ++i) {
    if (t->tps_hi[i] != t->tps_lo[i + 1]) return -1;
    if (t->tps_lo[i] >= t->tps_hi[i]) return -1;
  }
  if (t->tps_hi[t->n - 1] != INFINITY) return -1;
  return 0;
}

/* TBT ring (TbtWindow, decode_ctl.cpp:120-128) */
GSO_INTERNAL void ring_record(ring_t* r, double x) {
  if (r->n < r->cap) {
    r->buf[(r->head + r->n) % r->cap] = x;
    r->n++;
  } else { /* push_back then pop_front */
    r->buf[r->head] = x;
    r->head = (r->head + 1) % r->cap;
  }
}

GSO_INTERNAL double ring_p95(ring_t* r) {
  for (int i = 0; i < r->n; ++i) r->scratch[i] = r->buf[(r->head + i) % r->cap];
  qsort(r->scratch, (size_t)r->n, sizeof(double), cmp_double);
  const size_t rank = (size_t)ceil(0.95 * (double)r->n);
  return r->scratch[rank == 0 ? 0 : rank - 1];
}

/* TpsWindow (decode_ctl.cpp:113-118): drop events with t < now - window, sum the rest. */
typedef struct {
  double window;
  const gso_telemetry* tel;
  int64_t lo, hi; /* live events are [lo, hi) of tel */
} tpswin_t;

static double tps_now(tpswin_t* w, double now) {
  while (w->lo < w->hi && w->tel->t_ms[w->lo] < now - w->window) w->lo++;
  int tokens = 0;
  for (int64_t j = w->lo; j < w->hi; ++j) tokens += w->tel->tokens[j];
  return tokens * 1000.0 / w->window;
}

int64_t gso_n_ticks(double period_ms, double t_end_ms) {
  int64_t n = 0;
  for (double t = period_ms; t <= t_end_ms; t = t + period_ms) ++n;
  return n;
}

/* Sim's tick composition (simkernel.cpp:441-458): step-end telemetry at t <= tick first
 * (event kind 2 sorts before ticks 5..7, simkernel.cpp:21-31,44-50). */
void gso_window_series(const gso_telemetry* tel, int tbt_capacity, double fine_period_ms,
                       double coarse_period_ms, double t_end_ms, uint8_t* fine_has,
                       double* fine_p95, double* coarse_tps) {
  ring_t ring = {tbt_capacity, 0, 0, (double*)malloc(sizeof(double) * (size_t)tbt_capacity),
                 (double*)malloc(sizeof(double) * (size_t)tbt_capacity)};
  tpswin_t tw = {coarse_period_ms, tel, 0, 0};
  double tf = fine_period_ms, tc = coarse_period_ms;
  int64_t kf = 0, kc = 0, j = 0;
  for (;;) {
    const double t = std_min(tf, tc);
    if (t > t_end_ms) break;
    while (j < tel->n_events && tel->t_ms[j] <= t) {
      for (int64_t g = tel->gap_off[j]; g < tel->gap_off[j + 1]; ++g) ring_record(&ring, tel->gaps[g]);
      ++j;
    }
    tw.hi = j;
    if (tc == t) {
      coarse_tps[kc++] = tps_now(&tw, t);
      tc = t + coarse_period_ms;
    }
    if (tf == t) {
      fine_has[kf] = ring.n > 0;
      fine_p95[kf] = ring.n > 0 ? ring_p95(&ring) : 0.0;
      ++kf;
      tf = t + fine_period_ms;
    }
  }
  free(ring.buf);
  free(ring.scratch);
}

/* DecodeController, decode_ctl.cpp:130-228. The adjustments_ vector is only ever read as
 * three counts (size, clamped-up, clamped-down) and cleared as a whole, so counters
 * restate it exactly. */
GSO_INTERNAL void ctl_log(ctl_t* c, double now, int bucket, int action) {
  if (c->n_rec < c->cap) {
    gso_decision* r = &c->out[c->n_rec];
    r->tick_ms = now;
    r->worker = c->worker;
    r->tps = c->last_tps;
    r->p95_tbt_ms = c->last_p95;
    r->bucket = bucket;
    r->band_lo = c->lo;
    r->band_hi = c->hi;
    r->command_mhz = c->sp;
    r->action = action;
    r->pad_ = 0;
  }
  c->n_rec++;
}

/* FreqBandTable::band :52-57 via DecodeController::load_band :137-142 */
GSO_INTERNAL void ctl_load_band(ctl_t* c, int bucket) {
  const double f = c->f_opt[bucket];
  c->lo = std_max(c->f_min, f - c->cfg.step_mhz);
  c->hi = std_min(c->f_max, f + c->cfg.step_mhz);
}

/* FreqBandTable::bucket_index :47-51 */
GSO_INTERNAL int ctl_bucket_index(const ctl_t* c, double tps) {
  for (int i = 0; i < c->n; ++i)
    if (tps <= c->tps_hi[i]) return i;
  return c->n - 1;
}

GSO_INTERNAL void ctl_init(ctl_t* c) {
  c->current = c->n - 1;
  c->pending = -1;
  c->consecutive = 0;
  ctl_load_band(c, c->current);
  c->sp = c->f_opt[c->current];
  c->last_tps = 0.0;
  c->last_p95 = 0.0;
  c->adj_total = c->adj_up = c->adj_dn = 0;
  c->n_rec = 0;
}

/* on_fine_tick :148-167 */
GSO_INTERNAL void ctl_fine(ctl_t* c, double now, int has, double p95) {
  int dir = 0;
  if (has) {
    c->last_p95 = p95;
    const double margin = p95 / (c->cfg.margin_decode * c->cfg.tslo_ms);
    if (margin > c->cfg.upper_margin)
      dir = +1;
    else if (margin < c->cfg.lower_margin)
      dir = -1;
  }
  const double delta = std_min(c->cfg.step_mhz, c->cfg.max_step_mhz);
  const double raw = c->sp + dir * delta;
  const double clamped = std_clamp(raw, c->lo, c->hi);
  const int hit = dir != 0 && clamped != raw;
  c->sp = clamped;
  c->adj_total++;
  if (hit && dir > 0) c->adj_up++;
  if (hit && dir < 0) c->adj_dn++;
  ctl_log(c, now, c->current, dir > 0 ? GSO_ACT_UP : dir < 0 ? GSO_ACT_DOWN : GSO_ACT_HOLD);
}

/* on_coarse_tick :169-198 */
GSO_INTERNAL void ctl_coarse(ctl_t* c, double now, double worker_tps) {
  c->last_tps = worker_tps * c->cfg.tps_scale;
  const int observed = ctl_bucket_index(c, c->last_tps);
  int action;
  if (observed == c->current) {
    c->pending = -1;
    c->consecutive = 0;
    action = GSO_ACT_COARSE_HOLD;
  } else {
    if (observed == c->pending) {
      ++c->consecutive;
    } else {
      c->pending = observed;
      c->consecutive = 1;
    }
    if (c->consecutive >= c->cfg.hysteresis_count) {
      c->current = observed;
      ctl_load_band(c, c->current);
      c->sp = std_clamp(c->sp, c->lo, c->hi);
      c->pending = -1;
      c->consecutive = 0;
      c->adj_total = c->adj_up = c->adj_dn = 0;
      action = GSO_ACT_COARSE_COMMIT;
    } else {
      action = GSO_ACT_COARSE_PENDING;
    }
  }
  ctl_log(c, now, observed, action);
}

/* on_adapt_tick :200-228 */
GSO_INTERNAL void ctl_adapt(ctl_t* c, double now) {
  const int total = (int)c->adj_total;
  const int up = (int)c->adj_up, dn = (int)c->adj_dn;
  c->adj_total = c->adj_up = c->adj_dn = 0;
  if (total == 0) return;
  int shift = 0;
  if (up > c->cfg.bias_threshold * total)
    shift = +1;
  else if (dn > c->cfg.bias_threshold * total)
    shift = -1;
  if (shift == 0) return;
  c->f_opt[c->current] = std_clamp(c->f_opt[c->current] + shift * c->cfg.step_mhz, c->f_min, c->f_max);
  ctl_load_band(c, c->current);
  c->sp = std_clamp(c->sp, c->lo, c->hi);
  ctl_log(c, now, c->current, shift > 0 ? GSO_ACT_ADAPT_UP : GSO_ACT_ADAPT_DOWN);
}

GSO_INTERNAL int ctl_setup(ctl_t* c, const gso_ctl_cfg* cfg, const gso_band_table* t, double f_min,
                     double f_max, int worker, gso_decision* out, int64_t cap) {
  if (gso_ctl_cfg_validate(cfg) != 0 || table_validate(t) != 0) return -1;
  memset(c, 0, sizeof(*c));
  c->cfg = *cfg;
  c->n = t->n;
  c->tps_hi = t->tps_hi;
  c->f_opt = (double*)malloc(sizeof(double) * (size_t)t->n);
  memcpy(c->f_opt, t->f_opt_mhz, sizeof(double) * (size_t)t->n);
  c->f_min = f_min;
  c->f_max = f_max;
  c->worker = worker;
  c->out = out;
  c->cap = cap;
  ctl_init(c);
  return 0;
}

/* Tick driver shared by both replay forms: simkernel.cpp:243-248 schedules the first
 * ticks at one period and every handler re-schedules at now + period (:450,457,463);
 * at equal times coarse (5) < adapt (6) < fine (7). */
int64_t gso_replay_telemetry(const gso_ctl_cfg* cfg, const gso_band_table* table, double f_min,
                             double f_max, int worker, const gso_telemetry* tel, double t_end_ms,
                             gso_decision* out, int64_t cap) {
  ctl_t c;
  if (ctl_setup(&c, cfg, table, f_min, f_max, worker, out, cap) != 0) return -1;
  ring_t ring = {cfg->tbt_window_tokens, 0, 0,
                 (double*)malloc(sizeof(double) * (size_t)cfg->tbt_window_tokens),
                 (double*)malloc(sizeof(double) * (size_t)cfg->tbt_window_tokens)};
  tpswin_t tw = {cfg->coarse_period_ms, tel, 0, 0};
  double tf = cfg->fine_period_ms, tc = cfg->coarse_period_ms, ta = cfg->adapt_period_s * 1000.0;
  int64_t j = 0;
  for (;;) {
    const double t = std_min(tf, std_min(tc, ta));
    if (t > t_end_ms) break;
    while (j < tel->n_events && tel->t_ms[j] <= t) {
      for (int64_t g = tel->gap_off[j]; g < tel->gap_off[j + 1]; ++g) ring_record(&ring, tel->gaps[g]);
      ++j;
    }
    tw.hi = j;
    if (tc == t) {
      ctl_coarse(&c, t, tps_now(&tw, t));
      tc = t + cfg->coarse_period_ms;
    }
    if (ta == t) {
      ctl_adapt(&c, t);
      ta = t + cfg->adapt_period_s * 1000.0;
    }
    if (tf == t) {
      const int has = ring.n > 0;
      ctl_fine(&c, t, has, has ? ring_p95(&ring) : 0.0);
      tf = t + cfg->fine_period_ms;
    }
  }
  free(ring.buf);
  free(ring.scratch);
  free(c.f_opt);
  return c.n_rec;
}

int64_t gso_replay_series(const gso_ctl_cfg* cfg, const gso_band_table* table, double f_min,
                          double f_max, int worker, const uint8_t* fine_has,
                          const double* fine_p95, const double* coarse_tps, double t_end_ms,
                          gso_decision* out, int64_t cap) {
  ctl_t c;
  if (ctl_setup(&c, cfg, table, f_min, f_max, worker, out, cap) != 0) return -1;
  double tf = cfg->fine_period_ms, tc = cfg->coarse_period_ms, ta = cfg->adapt_period_s * 1000.0;
  int64_t kf = 0, kc = 0;
  for (;;) {
    const double t = std_min(tf, std_min(tc, ta));
    if (t > t_end_ms) break;
    if (tc == t) {
      ctl_coarse(&c, t, coarse_tps[kc++]);
      tc = t + cfg->coarse_period_ms;
    }
    if (ta == t) {
      ctl_adapt(&c, t);
      ta = t + cfg->adapt_period_s * 1000.0;
    }
    if (tf == t) {
      ctl_fine(&c, t, fine_has[kf], fine_p95[kf]);
      ++kf;
      tf = t + cfg->fine_period_ms;
    }
  }
  free(c.f_opt);
  return c.n_rec;
}

/* Word-wise FNV-1a trajectory digest (K3 outputs). */
/* per record: w1 = command bits, w2 = band_lo bits ^ (band_hi bits << 13) ^ (bucket << 48)
 * ^ (action << 56); h = (h ^ w) * FNV64 prime, in log order (same as the GPU K3b). */
uint64_t gso_digest_records(const gso_decision* r, int64_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t cmd, lo, hi;
    memcpy(&cmd, &r[i].command_mhz, 8);
    memcpy(&lo, &r[i].band_lo, 8);
    memcpy(&hi, &r[i].band_hi, 8);
    const uint64_t w2 = lo ^ (hi << 13) ^ ((uint64_t)(uint32_t)r[i].bucket << 48) ^
                        ((uint64_t)(uint32_t)r[i].action << 56);
    h = (h ^ cmd) * 0x100000001b3ull;
    h = (h ^ w2) * 0x100000001b3ull;
  }
  return h;
}

/* ---------------- trace generators (rng.hpp, trace.cpp) ---------------- */

/* std::mt19937_64 as specified by [rand.predef] (the reference wraps it, rng.hpp:12-50) */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64_t;

static void mt64_seed(mt64_t* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64_t* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

static double rng_u01(mt64_t* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; } /* rng.hpp:22-25 */

static int64_t rng_int(mt64_t* g, int64_t lo, int64_t hi) { /* rng.hpp:28-37 */
  const uint64_t span = (uint64_t)(hi - lo) + 1;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % span;
  uint64_t x;
  do {
    x = mt64_next(g);
  } while (x >= limit);
  return lo + (int64_t)(x % span);
}

static double rng_exp(mt64_t* g, double mean) { /* rng.hpp:42-48 */
  double u;
  do {
    u = rng_u01(g);
  } while (u <= 0.0);
  return -mean * log(u);
}

static int sample_length(mt64_t* g, double mean) { /* trace.cpp:47-52 */
  int64_t lo = llround(mean * 0.5);
  if (lo < 1) lo = 1;
  int64_t hi = llround(mean * 1.5);
  if (hi < lo) hi = lo;
  return (int)rng_int(g, lo, hi);
}

/* gen_poisson_trace, trace.cpp:152-175 */
int64_t gso_gen_poisson_trace(double qps, int64_t duration_ms, double prompt_mean_short,
                              double prompt_mean_long, double long_fraction, double output_mean,
                              uint64_t seed, int64_t cap, int64_t* arrival, int32_t* prompt,
                              int32_t* output) {
  mt64_t g;
  mt64_seed(&g, seed);
  double now = 0.0;
  const double mean_gap = 1000.0 / qps;
  int64_t n = 0;
  for (;;) {
    now += rng_exp(&g, mean_gap);
    if (now >= (double)duration_ms) break;
    const int is_long = rng_u01(&g) < long_fraction;
    const int p = sample_length(&g, is_long ? prompt_mean_long : prompt_mean_short);
    const int o = sample_length(&g, output_mean);
    if (n < cap) {
      arrival[n] = (int64_t)now;
      prompt[n] = p;
      output[n] = o;
    }
    ++n;
  }
  return n;
}

/* gen_sinusoid_decode_trace, trace.cpp:239-285 */
typedef struct {
  double mean, amp, period, two_pi;
} sinus_t;

static double sin_cum(const sinus_t* s, double t_ms) {
  return s->mean * t_ms / 1000.0 +
         s->amp / 1000.0 * (s->period / s->two_pi) * (1.0 - cos(s->two_pi * t_ms / s->period));
}

static double sin_invert(const sinus_t* s, double target, double lo) {
  double hi = lo + 1000.0;
  while (sin_cum(s, hi) < target) hi += 1000.0;
  for (int i = 0; i < 60 && hi - lo > 1e-6; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (sin_cum(s, mid) < target)
      lo = mid;
    else
      hi = mid;
  }
  return 0.5 * (lo + hi);
}

int64_t gso_gen_sinusoid_decode_trace(double tps_mean, double tps_amp, double period_ms,
                                      int64_t duration_ms, uint64_t seed, int64_t cap,
                                      int64_t* arrival, int32_t* prompt, int32_t* output) {
  const sinus_t s = {tps_mean, tps_amp, period_ms, 2.0 * 3.14159265358979323846};
  mt64_t g;
  mt64_seed(&g, seed);
  double cum_tokens = 0.0, prev_t = 0.0;
  int64_t n = 0;
  for (;;) {
    const double t_exact = cum_tokens == 0.0 ? 0.0 : sin_invert(&s, cum_tokens, prev_t);
    const int64_t a = (int64_t)llround(t_exact);
    if (a >= duration_ms) break;
    prev_t = t_exact;
    const int o = (int)rng_int(&g, 64, 192);
    if (n < cap) {
      arrival[n] = a;
      prompt[n] = 32;
      output[n] = o;
    }
    ++n;
    cum_tokens += o;
  }
  return n;
}
