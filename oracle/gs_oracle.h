/*
 * gs_oracle.h — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the GreenLLM decision-engine hot path of the
 * reference `greensim` library (/root/reference/proj), plus the plain-data
 * types shared with the reference shim (ref_capi.cpp, compiled into
 * oracle/_ref/). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.
 *
 * Parity of this restatement is pinned two ways (tests/test_oracle_*.py):
 *   1. the reference's own golden values, and
 *   2. element-wise equality against oracle/_ref/libgreensim_ref.so, i.e. the
 *      reference sources compiled unmodified from /root/reference.
 *
 * All arithmetic is IEEE binary64, round-to-nearest, evaluated in the
 * reference's operation order; the library is compiled with
 * -ffp-contract=off so that no FMA contraction can change a bit.
 */
#ifndef GS_ORACLE_H
#define GS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* greensim::GpuProfile minus the name (gpu_model.hpp:16-87). */
typedef struct gso_profile {
  double f_min_mhz, f_max_mhz, step_mhz, f_ref_mhz;                 /* FrequencyGrid   :16-28 */
  double lat_a, lat_b, lat_c, lat_f_ref_mhz;                         /* LatencyModel    :32-39 */
  double dec_alpha0_ms, dec_alpha1_ms, dec_beta0_ms, dec_beta1_ms,   /* DecodeStepModel :45-53 */
      dec_f_ref_mhz;
  double k3, k2, k1, k0, p_idle_w;                                   /* PowerModel      :57-67 */
} gso_profile;

/* greensim::QueueOptimizerConfig (prefill_opt.hpp:61-68). */
typedef struct gso_qopt_cfg {
  double resolve_period_ms, margin_prefill, min_budget_ms, first_token_allowance_ms;
} gso_qopt_cfg;

/* greensim::DecodeCtlConfig (decode_ctl.hpp:13-29). */
typedef struct gso_ctl_cfg {
  double tslo_ms, margin_decode, fine_period_ms, coarse_period_ms, adapt_period_s;
  double step_mhz, max_step_mhz;
  int32_t hysteresis_count, tbt_window_tokens;
  double bias_threshold, tps_scale, upper_margin, lower_margin;
} gso_ctl_cfg;

/* greensim::DecisionRecord (decode_ctl.hpp:95-105) with the action string as an enum. */
enum {
  GSO_ACT_HOLD = 0, GSO_ACT_UP = 1, GSO_ACT_DOWN = 2,
  GSO_ACT_COARSE_HOLD = 3, GSO_ACT_COARSE_PENDING = 4, GSO_ACT_COARSE_COMMIT = 5,
  GSO_ACT_ADAPT_UP = 6, GSO_ACT_ADAPT_DOWN = 7
};
typedef struct gso_decision {
  double tick_ms, tps, p95_tbt_ms, band_lo, band_hi, command_mhz;
  int32_t worker, bucket, action, pad_;
} gso_decision;

/* One TPS-bucketed band table (decode_ctl.hpp:39-64), SoA. */
typedef struct gso_band_table {
  int32_t n;
  const double* tps_lo;
  const double* tps_hi;
  const double* f_opt_mhz;
} gso_band_table;

/*
 * Raw decode telemetry of one decode worker (what Sim feeds the windows,
 * simkernel.cpp:365-393): step-end events sorted by time; event j emitted
 * tokens[j] tokens at t_ms[j] and recorded gaps[gap_off[j] .. gap_off[j+1])
 * into the TBT ring in that order.
 */
typedef struct gso_telemetry {
  int64_t n_events;
  const double* t_ms;
  const int32_t* tokens;
  const int64_t* gap_off; /* n_events + 1 */
  const double* gaps;
} gso_telemetry;

/* ---------------- prefill objective (prefill_opt.cpp) ---------------- */
int gso_profile_validate(const gso_profile* p);                  /* gpu_model.cpp:80-87; 0 ok */
int gso_grid_size(const gso_profile* p);                         /* gpu_model.cpp:24-26 */
double gso_grid_at(const gso_profile* p, int i);                 /* gpu_model.cpp:28 */
double gso_active_power_w(const gso_profile* p, double f);       /* gpu_model.hpp:64 */
double gso_t_ref_total_ms(const gso_profile* p, int64_t n, const int32_t* prompt,
                          const double* wf /* NULL = all 1.0 */); /* prefill_opt.cpp:9-14 */
/* energy_total (prefill_opt.cpp:22-31); returns 0 ok, -1 ModelError. */
int gso_energy_total(const gso_profile* p, int64_t n, const int32_t* prompt, const double* wf,
                     double f, double window_ms, double* active_j, double* idle_j,
                     double* total_j, int* feasible);
double gso_energy_closed_form(const gso_profile* p, int64_t n, const int32_t* prompt,
                              const double* wf, double f, double window_ms); /* :33-43 */
/* select_frequency (prefill_opt.cpp:45-56): returns grid index of the choice or -1 (nullopt). */
int gso_select_frequency(const gso_profile* p, int64_t n, const int32_t* prompt, const double* wf,
                         double window_ms, double* f_out, double* e_out);
/* select on a precomputed T_ref (same bits as the batch form; used for binned cells). */
int gso_select_frequency_t(const gso_profile* p, double t_ref, double window_ms, double* f_out,
                           double* e_out);
/* queue_optimizer_tick for one non-empty class queue (prefill_opt.cpp:63-80). */
void gso_queue_tick_one(const gso_profile* p, const gso_qopt_cfg* cfg, int64_t n,
                        const int32_t* prompt, const double* deadline, const double* wf,
                        double now_ms, double* f_out, double* window_out, int* infeasible_out,
                        int* f_idx_out, double* e_out);

/* ---------------- routing (router.cpp) ---------------- */
int gso_classify(int n_thr, const int32_t* thresholds, int32_t prompt); /* router.cpp:26-31 */
/* Offline binning convention: window k = [k*W, (k+1)*W), class = classify().
 * Per cell (window-major, class-minor): count, T_ref (arrival order), min deadline,
 * and the stable FIFO order of request indices (Dispatcher, router.cpp:37-43). */
int gso_route_bin(int64_t n_req, const int64_t* arrival_ms, const int32_t* prompt, int n_thr,
                  const int32_t* thresholds, int64_t window_ms, int64_t w0, int64_t n_windows,
                  int n_profiles, const gso_profile* profiles, double ttft_sm_ms, double ttft_l_ms,
                  double first_token_allowance_ms, uint8_t* cls_out, uint32_t* cell_count,
                  double* cell_t_ref /* [n_profiles][cells] */, double* cell_min_deadline,
                  int64_t* fifo_out /* n_req or NULL */);

/* ---------------- decode control (decode_ctl.cpp, metrics.cpp) ---------------- */
double gso_quantile(int64_t n, const double* samples, double q);         /* metrics.cpp:11-19 */
int gso_decode_steady_state(const gso_profile* p, double tps, double f, int max_batch,
                            double* batch, double* tbt_ms);               /* decode_ctl.cpp:28-50 */
/* build_band_table (decode_ctl.cpp:76-111); returns 0 ok, -1 ModelError. */
int gso_build_band_table(const gso_profile* p, int n_levels, const double* levels, double t_slo_ms,
                         int workers, int max_batch, double* tps_lo, double* tps_hi,
                         double* f_opt, uint8_t* feasible);
int gso_ctl_cfg_validate(const gso_ctl_cfg* c);                           /* decode_ctl.cpp:12-26 */

/*
 * Window statistics of one telemetry stream as Sim's ticks observe them
 * (simkernel.cpp:441-458; decode_ctl.cpp:113-128): the P95 at every fine tick and
 * the TPS at every coarse tick up to t_end_ms inclusive.
 */
int64_t gso_n_ticks(double period_ms, double t_end_ms);
void gso_window_series(const gso_telemetry* tel, int tbt_capacity, double fine_period_ms,
                       double coarse_period_ms, double t_end_ms, uint8_t* fine_has,
                       double* fine_p95, double* coarse_tps);

/*
 * Open-loop controller replay of one worker: the DecodeController composed with the
 * windows exactly as Sim's fine/coarse/adapt ticks do. Writes up to cap records and
 * returns the record count (or -1 on ModelError). Two drivers: from raw telemetry,
 * and from precomputed window series.
 */
int64_t gso_replay_telemetry(const gso_ctl_cfg* cfg, const gso_band_table* table, double f_min,
                             double f_max, int worker, const gso_telemetry* tel, double t_end_ms,
                             gso_decision* out, int64_t cap);
int64_t gso_replay_series(const gso_ctl_cfg* cfg, const gso_band_table* table, double f_min,
                          double f_max, int worker, const uint8_t* fine_has,
                          const double* fine_p95, const double* coarse_tps, double t_end_ms,
                          gso_decision* out, int64_t cap);

/* 64-bit trajectory digest (FNV-1a over the record fields). */
uint64_t gso_digest_records(const gso_decision* recs, int64_t n);

/* ---------------- trace generators (trace.cpp, rng.hpp) ---------------- */
int64_t gso_gen_poisson_trace(double qps, int64_t duration_ms, double prompt_mean_short,
                              double prompt_mean_long, double long_fraction, double output_mean,
                              uint64_t seed, int64_t cap, int64_t* arrival, int32_t* prompt,
                              int32_t* output);
int64_t gso_gen_sinusoid_decode_trace(double tps_mean, double tps_amp, double period_ms,
                                      int64_t duration_ms, uint64_t seed, int64_t cap,
                                      int64_t* arrival, int32_t* prompt, int32_t* output);

/* ---------------- the reference simulator (simkernel.cpp) ----------------
 * gso_sim_run restates greensim::run (simkernel.cpp:119-560): the two-pool discrete-event
 * simulator that calls the decision engine. It is pinned field-by-field against the
 * reference's own run() (tests/test_oracle_sim.py) and serves two roles: it records the
 * decode-enqueue stream in the reference's processing order (same-time ties follow the
 * event sequence numbers, simkernel.cpp:44-50), and it is the checker for the GPU
 * closed-loop decode pool (K5). gso_pool_run drives the SAME decode-pool code from such a
 * stream alone (prefill never waits on decode, so the stream is a function of the prefill
 * side only). Results are read through an opaque handle (gso_sim_free). */
typedef struct gso_sim_cfg { /* SimConfig, simkernel.hpp:88-104 */
  int32_t n_prefill_workers, n_decode_workers, gpus_per_prefill_worker, max_batch, max_queue;
  int32_t pad_;
  double actuation_delay_ms, handoff_delay_ms, band_tps_lo, band_tps_hi, band_tps_step;
} gso_sim_cfg;

typedef struct gso_slo { double ttft_sm_ms, ttft_l_ms, tbt_p95_ms; } gso_slo; /* SloConfig :53-62 */

typedef struct gso_policy {  /* GovernorPolicy, simkernel.hpp:26-45 */
  int32_t kind;              /* 0 defaultnv, 1 fixed, 2 greenllm, 3 prefillsplit */
  int32_t routing_enabled;   /* RoutingConfig::enabled (router.hpp:19-29) */
  int32_t n_thresholds;
  int32_t thresholds[7];
  const int32_t* worker_map; /* [n_prefill_workers] */
  double fixed_freq_mhz;
  gso_qopt_cfg prefill_opt;
  gso_ctl_cfg decode_ctl;
} gso_policy;

typedef struct gso_scripted { /* ScriptedFreqEvent, simkernel.hpp:76-81 */
  double time_ms;
  int32_t prefill_pool, worker;
  double f_mhz;
} gso_scripted;

/* Decode-side summary of one run (the K5 output). Digests:
 *   decision_digest  per decode worker, the K3 record digest (gso_digest_records) of that
 *                    worker's DecisionRecords in log order; combined h = (h ^ d_w) * P over w
 *   freq_digest      per decode worker, FNV-1a over (applied_ms bits, f bits) of its applied
 *                    changes (t = 0 initial rows excluded); combined the same way
 *   request_digest   sum mod 2^64 over requests that reached the decode pool of
 *                    FNV-1a(id, first_token bits, finish bits, decode_worker, n_gaps,
 *                    sum of the gaps' bit patterns mod 2^64), or FNV-1a(id, 0xdead) for a
 *                    decode-side rejection (a request's gaps are consecutive step lengths
 *                    of its worker, so first/finish/worker plus the sum pin them) */
typedef struct gso_pool_summary {
  double decode_pool_j, active_decode_j, idle_j, sim_end_ms;
  int64_t n_completed, n_rejected, n_ttft_ok, n_tbt_ok, tbt_samples, tbt_samples_ok;
  int64_t n_decisions, n_freq_changes, n_steps;
  uint64_t decision_digest, freq_digest, request_digest;
} gso_pool_summary;

void* gso_sim_run(const gso_profile* prof, const gso_policy* pol, const gso_slo* slo,
                  const gso_sim_cfg* cfg, int64_t n, const int64_t* arrival_ms,
                  const int32_t* prompt, const int32_t* output, const int8_t* cls /* NULL/-1 */,
                  int64_t n_scripted, const gso_scripted* scripted, char* err, size_t err_cap);
/* Decode pool alone, driven by an enqueue stream (t, request) in processing order.
 * end_floor_ms = the prefill side's contribution to sim_end_ms (simkernel.cpp:506-512). */
void* gso_pool_run(const gso_profile* prof, const gso_policy* pol, const gso_slo* slo,
                   const gso_sim_cfg* cfg, int64_t n, const int64_t* arrival_ms,
                   const int32_t* prompt, const int32_t* output, const int8_t* cls,
                   int64_t n_stream,
                   const double* enq_t, const int64_t* enq_req, double end_floor_ms,
                   char* err, size_t err_cap);
void gso_sim_free(void* h);
/* [0] requests, [1] tbt samples, [2] decisions, [3] timeline rows, [4] prefill commands,
 * [5] enqueues, [6] prefill workers, [7] decode workers, [8] rejected, [9] decode steps */
void gso_sim_sizes(void* h, int64_t* s);
void gso_sim_requests(void* h, int32_t* class_queue, int32_t* prefill_worker,
                      int32_t* decode_worker, double* prefill_start, double* prefill_end,
                      double* first_token, double* finish, uint8_t* completed, uint8_t* rejected,
                      int8_t* cls);
void gso_sim_tbt(void* h, int64_t* off /* [n+1] */, double* samples);
/* per worker: active_prefill_j, active_decode_j, idle_j; n_intervals per worker */
void gso_sim_ledgers(void* h, double* prefill3, double* decode3, int64_t* n_intervals);
void gso_sim_decisions(void* h, gso_decision* out);
void gso_sim_timeline(void* h, double* t, uint8_t* pool, int32_t* worker, double* f);
void gso_sim_commands(void* h, double* tick, int32_t* cls, int32_t* worker, double* f,
                      double* window, uint8_t* infeasible);
void gso_sim_enqueue(void* h, double* t, int64_t* req);
/* [0] sim_end_ms, [1] last_arrival_ms, [2] end floor (prefill-side part of sim_end) */
void gso_sim_scalars(void* h, double* d);
void gso_sim_summary(void* h, const gso_slo* slo, gso_pool_summary* out);

/* The K5 summary from plain arrays (shared by the restatement and the reference shim). */
void gso_pool_summary_from(const gso_slo* slo, int64_t n, const double* arrival,
                           const int8_t* cls, const int32_t* decode_worker,
                           const double* prefill_end, const double* first_token,
                           const double* finish, const uint8_t* completed,
                           const uint8_t* rejected, const int64_t* tbt_off,
                           const double* tbt, int n_decode, const double* decode3,
                           int64_t n_dec, const gso_decision* dec, int64_t n_tl,
                           const double* tl_t, const uint8_t* tl_pool, const int32_t* tl_worker,
                           const double* tl_f, double sim_end_ms, int64_t n_steps,
                           gso_pool_summary* out);

/* ---- trace CSV (gs_trace.c): load_trace / save_trace_csv (trace.cpp:56-145) */
enum { /* greensim::TraceError::Kind order (trace.hpp:36-40) */
  GSO_TRACE_EMPTY = 0, GSO_TRACE_NON_MONOTONE = 1, GSO_TRACE_MALFORMED = 2,
  GSO_TRACE_BAD_HEADER = 3, GSO_TRACE_CLASS_MISMATCH = 4
};
typedef struct gso_trace_err {
  int32_t kind, detail; /* detail: 1 columns, 2-4 bad field, 5 range, 6 monotone, 7 class, 8 mismatch */
  int64_t row;          /* 1-based row counter of the failing line, -1 if none */
  char msg[8192];       /* the reference's TraceError message */
} gso_trace_err;
/* rows parsed (the first min(rows, cap) are stored), or -1 with *err */
int64_t gso_trace_parse(const char* bytes, int64_t n, int32_t class_threshold, int64_t cap,
                        int64_t* arrival, int32_t* prompt, int32_t* output, uint8_t* slo_cls,
                        int32_t* has_class, gso_trace_err* err);
/* the CSV text (written when out has room); returns its byte count */
int64_t gso_trace_format(int64_t n, const int64_t* arrival, const int32_t* prompt,
                         const int32_t* output, const uint8_t* slo_cls, char* out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif
