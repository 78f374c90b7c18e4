/*
 * gsb.h — C ABI of the B200-native GreenLLM decision engine (libgsb.so).
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch types.
 * Every compute entry point runs hand-written sm_100a CUDA kernels on caller-owned
 * DEVICE buffers on the caller's stream (`stream` is a cudaStream_t; NULL means the
 * context's own stream). There is no CPU fallback: a call on a host without a usable
 * B200 returns GSB_CUDA_ERROR.
 *
 * Reference interfaces replaced (paths under /root/reference/proj):
 *   include/greensim/gpu_model.hpp:16-87    FrequencyGrid / LatencyModel / DecodeStepModel /
 *                                           PowerModel / GpuProfile (+ validate())
 *   include/greensim/router.hpp:19-56       RoutingConfig, classify(), Dispatcher
 *   include/greensim/prefill_opt.hpp:13-88  PrefillBatch::t_ref_total_ms, busy_time_ms,
 *                                           energy_total, select_frequency,
 *                                           QueueOptimizerConfig, queue_optimizer_tick
 *   include/greensim/decode_ctl.hpp:13-165  DecodeCtlConfig, decode_steady_state,
 *                                           build_band_table, TpsWindow, TbtWindow,
 *                                           DecodeController, DecisionRecord
 *   include/greensim/metrics.hpp:14-16      quantile (nearest rank, the TBT-window P95)
 *
 * Error behaviour mirrors the reference's typed exceptions: ModelError -> GSB_MODEL_ERROR,
 * RouterError -> GSB_ROUTER_ERROR, TraceError -> GSB_TRACE_ERROR; gsb_last_error() holds
 * the message. Infeasibility is a value, not an error (prefill_opt.hpp:55-57,79).
 *
 * Threading: a context is single-owner (one per host thread), like DecodeController
 * (SPEC.md:435). Distinct contexts may run concurrently.
 */
#ifndef GSB_H
#define GSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSB_ABI_VERSION 1
#define GSB_MAX_PROFILES 4   /* profiles evaluated in one prefill pass */
#define GSB_MAX_GRID 256     /* clock grid points per profile (81 for 210..1410/15) */
#define GSB_MAX_CLASSES 8    /* length classes (<= 7 routing thresholds) */
#define GSB_MAX_BUCKETS 32   /* TPS buckets per band table */
#define GSB_MAX_TBT_WINDOW 256

typedef enum gsb_status {
  GSB_OK = 0,
  GSB_MODEL_ERROR = 1,  /* greensim::ModelError  (gpu_model.hpp:11-13) */
  GSB_ROUTER_ERROR = 2, /* greensim::RouterError (router.hpp:13-15) */
  GSB_TRACE_ERROR = 3,  /* greensim::TraceError  (trace.hpp:36-40) */
  GSB_CUDA_ERROR = 4,
  GSB_INVALID_ARGUMENT = 5
} gsb_status;

typedef struct gsb_ctx gsb_ctx;

/* greensim::GpuProfile minus its name; same field order as gpu_model.hpp:16-87. */
typedef struct gsb_profile {
  double f_min_mhz, f_max_mhz, step_mhz, f_ref_mhz;                 /* FrequencyGrid   */
  double lat_a, lat_b, lat_c, lat_f_ref_mhz;                         /* LatencyModel    */
  double dec_alpha0_ms, dec_alpha1_ms, dec_beta0_ms, dec_beta1_ms,   /* DecodeStepModel */
      dec_f_ref_mhz;
  double k3, k2, k1, k0, p_idle_w;                                   /* PowerModel      */
} gsb_profile;

/* greensim::QueueOptimizerConfig (prefill_opt.hpp:61-68). */
typedef struct gsb_qopt_cfg {
  double resolve_period_ms, margin_prefill, min_budget_ms, first_token_allowance_ms;
} gsb_qopt_cfg;

/* greensim::DecodeCtlConfig (decode_ctl.hpp:13-29). */
typedef struct gsb_ctl_cfg {
  double tslo_ms, margin_decode, fine_period_ms, coarse_period_ms, adapt_period_s;
  double step_mhz, max_step_mhz;
  int32_t hysteresis_count, tbt_window_tokens;
  double bias_threshold, tps_scale, upper_margin, lower_margin;
} gsb_ctl_cfg;

/* greensim::DecisionRecord (decode_ctl.hpp:95-105); action is an enum instead of a string:
 * 0 hold, 1 up, 2 down, 3 coarse_hold, 4 coarse_pending, 5 coarse_commit, 6 adapt_up,
 * 7 adapt_down. */
typedef struct gsb_decision {
  double tick_ms, tps, p95_tbt_ms, band_lo, band_hi, command_mhz;
  int32_t worker, bucket, action, pad_;
} gsb_decision;

/* ---------------------------------------------------------------- context */
const char* gsb_version(void);
const char* gsb_status_string(int status);
int gsb_ctx_create(int device, gsb_ctx** out);
void gsb_ctx_destroy(gsb_ctx* ctx);
const char* gsb_last_error(const gsb_ctx* ctx);
void* gsb_ctx_stream(gsb_ctx* ctx); /* the context's own cudaStream_t */
int gsb_synchronize(gsb_ctx* ctx);

/* GpuProfile::validate (gpu_model.cpp:80-87), host-side; GSB_MODEL_ERROR + message. */
int gsb_profile_validate(const gsb_profile* p, char* msg, size_t msg_cap);
/* DecodeCtlConfig::validate (decode_ctl.cpp:12-26). */
int gsb_ctl_cfg_validate(const gsb_ctl_cfg* c, char* msg, size_t msg_cap);

/* Installs the profile set used by the prefill kernels (validated; per-clock tables of
 * f_i, 1/f_i and P(f_i) are built once here, gpu_model.cpp:24-28, gpu_model.hpp:64). */
int gsb_set_profiles(gsb_ctx* ctx, int n_profiles, const gsb_profile* profiles);

/* As gsb_set_profiles; flags & GSB_PROFILES_UNCHECKED skips GpuProfile::validate and keeps only
 * the structural checks the kernels need (finite grid, step > 0, 1..GSB_MAX_GRID clocks). The
 * reference's evaluators never validate their profile argument (prefill_opt.cpp:16-56), and its
 * tests call them with profiles validate() rejects (flat power, test_prefill_opt.cpp:98,135). */
#define GSB_PROFILES_UNCHECKED 1
/* flags & GSB_PROFILES_ASYNC: return without waiting for the (pinned, stream-ordered) table
 * upload; valid when every later launch uses the context's own stream (stream == NULL). */
#define GSB_PROFILES_ASYNC 2
int gsb_set_profiles_ex(gsb_ctx* ctx, int n_profiles, const gsb_profile* profiles, int flags);

/* ---------------------------------------------------------------- device memory */
/* Plumbing for hosts without their own CUDA runtime (cgo, JNI, the C++ drop-in in
 * paper_2508_16449_b200/cpp): device allocation on the context's device and copies on `stream`
 * (NULL = the context's stream). kind: 0 host->device, 1 device->host, 2 device->device.
 * gsb_memcpy returns once the copy is enqueued; call gsb_synchronize before reading a
 * device->host result. */
int gsb_malloc(gsb_ctx* ctx, size_t bytes, void** d_out);
int gsb_free(gsb_ctx* ctx, void* d_ptr);
/* Page-locked host memory (asynchronous DMA for gsb_memcpy). */
int gsb_host_alloc(gsb_ctx* ctx, size_t bytes, void** h_out);
int gsb_host_free(gsb_ctx* ctx, void* h_ptr);
int gsb_memcpy(gsb_ctx* ctx, void* dst, const void* src, size_t bytes, int kind, void* stream);

/* ---------------------------------------------------------------- K1: route + bin */
/* Routing / binning configuration. Offline window convention: window k of
 * the pass covers [(w0+k)*window_ms, (w0+k+1)*window_ms); jobs of a cell are the requests
 * of that class arriving in the window, in arrival order (Dispatcher FIFO, router.cpp:37-43). */
typedef struct gsb_route_cfg {
  int32_t n_thresholds;                 /* RoutingConfig::thresholds (router.hpp:19-29) */
  int32_t thresholds[GSB_MAX_CLASSES - 1];
  int32_t enabled;                      /* RoutingConfig::enabled; 0 -> one queue */
  int32_t slo_boundary_tokens;          /* SM/L boundary, 1024 (simkernel.cpp:258-260) */
  int64_t window_ms, w0, n_windows;
  double ttft_sm_ms, ttft_l_ms;         /* SloConfig (simkernel.hpp:53-62) */
  double first_token_allowance_ms;      /* QueueOptimizerConfig (prefill_opt.hpp:66-67) */
} gsb_route_cfg;

/* RoutingConfig::validate (router.cpp:7-24) for n_prefill_workers / worker_map. */
int gsb_routing_validate(const gsb_route_cfg* cfg, int n_prefill_workers,
                         const int32_t* worker_map, char* msg, size_t msg_cap);

/* classify(cfg, prompt) (router.cpp:26-31) for n prompts: the number of the n_thresholds
 * (host array, 0..GSB_MAX_CLASSES-1 entries, any order) strictly below the prompt. */
int gsb_classify(gsb_ctx* ctx, int n_thresholds, const int32_t* thresholds, int64_t n,
                 const int32_t* d_prompt, int32_t* d_class, void* stream);

/* Window start indices: bounds[k] = first request with arrival >= (w0+k)*window_ms,
 * k = 0..n_windows (arrival must be non-decreasing, trace.cpp:109-111).
 * d_arrival_ms (here and in gsb_route_bin*) may be PINNED HOST memory (cudaHostAlloc /
 * cudaHostRegister): with unified addressing the kernels read it in place over PCIe. From pinned
 * host memory a dense trace (>= 64 requests per window) takes an interpolation search: one
 * arrival per 256 requests plus a 64-byte probe per window edge (more where a probe misses);
 * otherwise the pass reads
 * one 32-byte sector per 32 requests plus the 32-request tiles holding a window start. Either
 * way a host-resident trace needs no arrival upload (K1b reads arrivals only in deadline mode). */
int gsb_window_bounds(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req,
                      const int64_t* d_arrival_ms, int64_t* d_bounds, void* stream);

/* classify() per request (router.cpp:26-31) and, per cell = window*C + class:
 *   d_count[cell]        jobs in the cell
 *   d_t_ref[p*cells+cell] PrefillBatch::t_ref_total_ms over the cell's FIFO for profile p
 *                        (prefill_opt.cpp:9-14, left-to-right, bit-exact)
 *   d_min_deadline[cell] min_j (arrival_j + TTFT(SM/L)) - allowance (simkernel.cpp:499-501);
 *                        optional (NULL)
 * d_bounds from gsb_window_bounds. C = n_thresholds + 1 (or 1 when routing is disabled). */
int gsb_route_bin(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req,
                  const int64_t* d_arrival_ms, const int32_t* d_prompt, const int64_t* d_bounds,
                  uint8_t* d_class, uint32_t* d_count, double* d_t_ref, double* d_min_deadline,
                  void* stream);

/* The non-empty cells of a pass (count > 0) in ascending order, as K1b emits them in the same
 * pass as gsb_route_bin (decoupled look-back across its CTAs): K2 then runs as one wave of fully
 * populated warps over the list (an empty queue gives no command, prefill_opt.cpp:64). The
 * per-cell inputs K2 needs are also written in list order, so K2 reads them coalesced. */
typedef struct gsb_cell_list {
  uint32_t* d_cells;        /* [capacity] ascending non-empty cells (cells < 2^32) */
  int64_t* d_n;             /* [1] entries, written on the device */
  double* d_t_ref;          /* optional [P][capacity]: t_ref of the listed cells, per profile */
  double* d_min_deadline;   /* optional [capacity]: min_deadline of the listed cells */
  int64_t capacity;         /* >= cells of the pass */
} gsb_cell_list;

/* gsb_route_bin plus the cell list. Uses per-context sync words: calls on one context must be
 * stream-ordered. */
int gsb_route_bin_list(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req,
                       const int64_t* d_arrival, const int32_t* d_prompt, const int64_t* d_bounds,
                       uint8_t* d_class, uint32_t* d_count, double* d_t_ref,
                       double* d_min_deadline, const gsb_cell_list* list, void* stream);

/* Dispatcher queue contents: stable per-cell FIFO of request indices (cell-major), i.e.
 * Dispatcher::queue(q) of every window (router.cpp:37-43). d_cell_off[cells+1] receives
 * the exclusive prefix of d_count. */
int gsb_fifo_order(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req,
                   const uint8_t* d_class, const int64_t* d_bounds, const uint32_t* d_count,
                   int64_t* d_cell_off, int64_t* d_fifo, void* stream);

/* ---------------------------------------------------------------- K2: prefill objective */
typedef enum gsb_window_mode {
  GSB_FIXED_WINDOW = 0,    /* D = fixed_window_ms for every cell (select_frequency) */
  GSB_DEADLINE_SLACK = 1,  /* D = max(margin * (min_deadline - now), min_budget), now =
                              window start; queue_optimizer_tick, prefill_opt.cpp:63-67 */
  GSB_PER_CELL_WINDOW = 2  /* D = d_window[cell] */
} gsb_window_mode;

typedef struct gsb_select_cfg {
  int32_t mode;             /* gsb_window_mode */
  int32_t n_classes;        /* C of the cell layout (DEADLINE_SLACK: cell -> window) */
  double fixed_window_ms;   /* GSB_FIXED_WINDOW */
  int64_t w0, window_ms;    /* GSB_DEADLINE_SLACK: now = (w0 + cell / C) * window_ms */
  gsb_qopt_cfg qopt;
} gsb_select_cfg;

/* Exhaustive window-energy argmin for every (cell, profile) over the profile's clock grid:
 * energy_total (prefill_opt.cpp:22-31) at every grid clock, feasible iff busy <= D,
 * ascending scan with strict '<' (lowest clock on ties, prefill_opt.cpp:45-56).
 * Outputs per (p, cell) at index p*n_cells + cell:
 *   d_f_idx   grid index of the choice; -1 = nothing feasible (nullopt; a queue tick pins
 *             f_max with infeasible=true, prefill_opt.cpp:75-78); -2 = empty cell (no command)
 *   d_energy  energy_j of the choice (FrequencyChoice::energy_j), 0 otherwise
 * d_window (optional) receives / supplies the budget D per cell (PrefillFreqCommand::window_ms).
 * d_count may be NULL (all cells non-empty). */
int gsb_prefill_select(gsb_ctx* ctx, const gsb_select_cfg* cfg, int64_t n_cells,
                       const double* d_t_ref, const uint32_t* d_count,
                       const double* d_min_deadline, double* d_window, int16_t* d_f_idx,
                       double* d_energy, void* stream);

/* Ragged explicit batches (the reference's own call shape): batch b has jobs
 * [d_off[b], d_off[b+1]) with prompt tokens, work_fraction (NULL = 1.0) and, for
 * DEADLINE_SLACK, absolute deadlines and a per-batch now. Mode FIXED/PER_CELL uses
 * d_window[b] (PER_CELL) or cfg->fixed_window_ms. T_ref is the left-to-right sum of
 * wf*((a*L+b)*L+c) (prefill_opt.cpp:9-14). One profile (index `profile`). */
int gsb_select_batches(gsb_ctx* ctx, const gsb_select_cfg* cfg, int profile, int64_t n_batches,
                       const int64_t* d_off, const int32_t* d_prompt, const double* d_wf,
                       const double* d_deadline, const double* d_now, double* d_window,
                       int16_t* d_f_idx, double* d_energy, double* d_t_ref_out, void* stream);

/* The raw state of the running prefill job in a snapshot (the fields simkernel.cpp:476-479
 * reads): job j with d_running[j] != 0 gets
 *   work_fraction = max(remaining_ref - ((now - updated) * freq) / f_ref, 0) / t_ref
 * in the reference's operation order (now = the batch's d_now, f_ref = the profile's grid
 * f_ref); every other job 1.0 (or d_wf[j]). */
typedef struct gsb_running_jobs {
  const uint8_t* d_running;          /* [jobs] */
  const double* d_remaining_ref_ms;  /* PrefillWorker::job_remaining_ref */
  const double* d_updated_ms;        /* PrefillWorker::job_updated_ms */
  const double* d_freq_mhz;          /* PrefillWorker::freq (the applied clock) */
  const double* d_t_ref_ms;          /* PrefillWorker::job_t_ref_ms */
} gsb_running_jobs;

/* gsb_select_batches with the running jobs' work_fraction computed on the device from their raw
 * state (queue_optimizer_tick snapshots exactly as Sim::on_optimizer_tick builds them). */
int gsb_select_batches_running(gsb_ctx* ctx, const gsb_select_cfg* cfg, int profile,
                               int64_t n_batches, const int64_t* d_off, const int32_t* d_prompt,
                               const double* d_wf, const gsb_running_jobs* run,
                               const double* d_deadline, const double* d_now, double* d_window,
                               int16_t* d_f_idx, double* d_energy, double* d_t_ref_out,
                               void* stream);

/* busy_time_ms + energy_total at one given clock per batch (prefill_opt.cpp:16-31): full
 * breakdown. d_feasible[b] = 2 marks the reference's ModelError (empty batch or off-grid
 * clock, prefill_opt.cpp:17-18). */
int gsb_energy_batches(gsb_ctx* ctx, int profile, int64_t n_batches, const int64_t* d_off,
                       const int32_t* d_prompt, const double* d_wf, const double* d_f_mhz,
                       const double* d_window, double* d_busy, double* d_active, double* d_idle,
                       double* d_total, uint8_t* d_feasible, void* stream);

/* PrefillBatch::t_ref_total_ms(m) (prefill_opt.cpp:9-14) of n ragged batches under the latency
 * model lat_abc = {a, b, c} alone (the reference takes a LatencyModel, not a profile):
 * d_out[b] = left-to-right sum of wf*((a*L+b)*L+c); 0 for an empty batch. */
int gsb_t_ref_batches(gsb_ctx* ctx, const double lat_abc[3], int64_t n_batches,
                      const int64_t* d_off, const int32_t* d_prompt, const double* d_wf,
                      double* d_out, void* stream);

/* energy_total_closed_form_j (prefill_opt.cpp:33-43, Eq. 13; a cross-check of energy_total)
 * per batch at clock d_f_mhz[b] and window d_window[b]; NaN for an off-grid clock (the
 * reference's ModelError). */
int gsb_energy_closed_form_batches(gsb_ctx* ctx, int profile, int64_t n_batches,
                                   const int64_t* d_off, const int32_t* d_prompt,
                                   const double* d_wf, const double* d_f_mhz,
                                   const double* d_window, double* d_out, void* stream);

/* Per (profile, class) summary of a K2 pass for the end-of-run reductions:
 * n_cmd, n_infeasible, n_empty, sum_energy (fixed-shape tree order, deterministic),
 * and the argmin cell (min energy, then lowest cell index). */
typedef struct gsb_class_summary {
  int64_t n_cmd, n_infeasible, n_empty;
  double sum_energy_j;
  double min_energy_j;
  int64_t argmin_cell;
} gsb_class_summary;
int gsb_prefill_summary(gsb_ctx* ctx, int n_profiles, int n_classes, int64_t n_cells,
                        const int16_t* d_f_idx, const double* d_energy,
                        gsb_class_summary* d_out /* [n_profiles*n_classes] */, void* stream);

/* K2 with the per-class summary fused: gsb_prefill_select's outputs plus the
 * gsb_prefill_summary record of every (profile, class). The per-chunk partials are folded in
 * K2's epilogue and one small kernel combines them. Same fixed-shape tree as
 * gsb_prefill_summary, so the two paths give identical bytes. Needs cfg->n_classes with n_cells = windows x classes.
 * Replaces the reference's end-of-run energy / SLO tallies over queue_optimizer_tick's
 * commands (prefill_opt.cpp:58-82 callers, simkernel.cpp:487). */
int gsb_prefill_select_summary(gsb_ctx* ctx, const gsb_select_cfg* cfg, int64_t n_cells,
                               const double* d_t_ref, const uint32_t* d_count,
                               const double* d_min_deadline, double* d_window, int16_t* d_f_idx,
                               double* d_energy, gsb_class_summary* d_summary, void* stream);

/* gsb_prefill_select_summary over a cell list from gsb_route_bin_list (its d_t_ref /
 * d_min_deadline are used when present, else d_t_ref / d_min_deadline are gathered per cell;
 * list == NULL: the list is built from d_count first). d_summary may be NULL. Results are
 * identical to gsb_prefill_select_summary's. */
int gsb_prefill_select_list(gsb_ctx* ctx, const gsb_select_cfg* cfg, int64_t n_cells,
                            const double* d_t_ref, const uint32_t* d_count,
                            const gsb_cell_list* list, const double* d_min_deadline,
                            double* d_window, int16_t* d_f_idx, double* d_energy,
                            gsb_class_summary* d_summary, void* stream);

/* The whole offline prefill pass in one call: gsb_window_bounds + gsb_route_bin_list +
 * gsb_prefill_select_list (+ the per-class summary when d_summary != NULL), with identical
 * outputs, where K1b and K2 run as ONE persistent kernel (routing tiles first, then K2 chunks
 * of the cell list as soon as their entries are written). scfg->mode: FIXED_WINDOW or
 * DEADLINE_SLACK (the latter needs d_min_deadline and list->d_min_deadline); list->d_t_ref is
 * required. Profiles whose grid is not 81 short-divisor clocks take the two-call path. */
int gsb_prefill_pass(gsb_ctx* ctx, const gsb_route_cfg* rcfg, int64_t n_req,
                     const int64_t* d_arrival, const int32_t* d_prompt, int64_t* d_bounds,
                     uint8_t* d_class, uint32_t* d_count, double* d_t_ref,
                     double* d_min_deadline, const gsb_cell_list* list,
                     const gsb_select_cfg* scfg, double* d_window, int16_t* d_f_idx,
                     double* d_energy, gsb_class_summary* d_summary, void* stream);

/* The same pass from HOST buffers, pipelined: the windows are split into K = n_chunks
 * consecutive ranges of decreasing size (chunk k = windows [a_k, a_k+1), a_k = nW * S_k /
 * (K (K+1) / 2) with S_k = K + (K-1) + ... + (K-k+1), integer division), their requests found
 * by a host lower_bound over h_arrival. K1a' reads the PINNED h_arrival in place once; per
 * chunk the prompt upload (a copy engine, its own stream), K1b, K2 with the finish and the
 * summary (two alternating compute streams) and the read-back of the chunk's rows of h_f_idx /
 * h_energy (another copy engine) overlap the neighbouring chunks' work. h_arrival and h_prompt must be pinned (cudaHostAlloc
 * / cudaHostRegister); h_f_idx [P][cells] and h_energy [P][cells] are host arrays (pinned for an
 * asynchronous read-back: a pageable one blocks the call until its chunk is done) receiving
 * exactly gsb_prefill_pass's d_f_idx / d_energy. h_summary (optional, pinned host
 * [n_chunks][P*C]) receives each chunk's gsb_class_summary records, argmin
 * cells relative to the chunk: combine them with gsb_combine_summaries and cell offsets
 * a_k * C (as ranks). mode FIXED_WINDOW or DEADLINE_SLACK; 1 <= n_chunks <=
 * min(64, n_windows). Stream-ordered: the outputs are valid once `stream` has synchronized. The
 * chunk split reads h_arrival on the host at call time, so the call is not for graph capture. */
int gsb_prefill_pass_host(gsb_ctx* ctx, const gsb_route_cfg* rcfg, int64_t n_req,
                          const int64_t* h_arrival, const int32_t* h_prompt,
                          const gsb_select_cfg* scfg, int n_chunks, int16_t* h_f_idx,
                          double* h_energy, gsb_class_summary* h_summary, void* stream);

/* M/G/1 side output of a pass (BASELINE north_star (2)): per (profile, cell) the utilisation
 * rho = lambda E[s], the Pollaczek-Khinchine mean wait Wq = lambda E[s^2] / (2 (1 - rho)) in ms
 * (+inf when rho >= 1) and the energy per request E / n, with service times s_j = (f_ref / f)
 * t_j at the command's clock (f_max when infeasible) and lambda = jobs / window_ms.
 * PARITY-UNPINNED: the reference has no M/G/1 term; never an input of the
 * bit-exact decisions. Outputs [P][cells]; empty cells 0. d_bounds / d_class from K1,
 * d_f_idx / d_energy from K2. */
int gsb_mg1_side_output(gsb_ctx* ctx, int n_classes, int64_t n_windows, double window_ms,
                        const int32_t* d_prompt, const uint8_t* d_class, const int64_t* d_bounds,
                        const int16_t* d_f_idx, const double* d_energy, double* d_wq_ms,
                        double* d_rho, double* d_energy_per_request, void* stream);

/* ---------------------------------------------------------------- K6: trace CSV ingest */
/* greensim::TraceError::Kind (trace.hpp:36-40), in the reference's enum order */
enum {
  GSB_TRACE_KIND_EMPTY = 0, GSB_TRACE_KIND_NON_MONOTONE = 1, GSB_TRACE_KIND_MALFORMED = 2,
  GSB_TRACE_KIND_BAD_HEADER = 3, GSB_TRACE_KIND_CLASS_MISMATCH = 4, GSB_TRACE_KIND_BAD_SHAPE = 5
};
/* which load_trace check failed, in the reference's order (trace.cpp:80-127) */
enum {
  GSB_TRACE_DETAIL_NONE = 0, GSB_TRACE_DETAIL_COLUMNS = 1, GSB_TRACE_DETAIL_ARRIVAL = 2,
  GSB_TRACE_DETAIL_PROMPT = 3, GSB_TRACE_DETAIL_OUTPUT = 4, GSB_TRACE_DETAIL_RANGE = 5,
  GSB_TRACE_DETAIL_MONOTONE = 6, GSB_TRACE_DETAIL_CLASS = 7, GSB_TRACE_DETAIL_MISMATCH = 8
};
typedef struct gsb_trace_parse_result {
  int32_t status;         /* GSB_OK or GSB_TRACE_ERROR */
  int32_t kind;           /* GSB_TRACE_KIND_* when status == GSB_TRACE_ERROR */
  int32_t detail;         /* GSB_TRACE_DETAIL_* */
  int32_t has_class;      /* the header carried the class column */
  int32_t n_cols;         /* columns of the failing row */
  int32_t line_len;       /* bytes of line[] */
  int32_t line_truncated; /* the failing line was longer than line[] */
  int32_t pad_;
  int64_t row;            /* the reference's 1-based row counter of the failing line (-1: none) */
  int64_t n_rows;         /* requests parsed */
  int64_t max_arrival_ms; /* last (= largest) arrival; Trace::meta.duration_ms = max(0, this) */
  char line[1024];        /* the failing line after the '\r' strip (NUL-terminated) */
} gsb_trace_parse_result;

/* greensim::load_trace (trace.cpp:56-129) over a CSV image already in device memory:
 * "arrival_ms,prompt_tokens,output_tokens[,class]" -> SoA (arrival i64, prompt i32, output i32,
 * SLO class u8: 0 = SM iff prompt <= class_threshold, 1 = L; trace.cpp:32-34). Request ids are
 * the row indices. Synchronous (the row count is returned in *res). Errors mirror TraceError:
 * GSB_TRACE_ERROR with res->kind / res->row and gsb_last_error() = the reference's message;
 * the earliest failing row wins, and within a row the reference's check order. Outputs need
 * cap_rows entries; more rows -> GSB_INVALID_ARGUMENT with res->n_rows = the count needed.
 * n_bytes < 4 GiB. */
int gsb_trace_parse(gsb_ctx* ctx, const char* d_bytes, int64_t n_bytes, int32_t class_threshold,
                    int64_t cap_rows, int64_t* d_arrival, int32_t* d_prompt, int32_t* d_output,
                    uint8_t* d_slo_class, gsb_trace_parse_result* res, void* stream);

/* greensim::save_trace_csv (trace.cpp:131-145) into device memory: header (with ",class" iff
 * d_slo_class != NULL, i.e. every request carries a class) + one row per request, '\n'
 * line ends, integers as ostream prints them. d_out == NULL: size query. *h_bytes = bytes. */
int gsb_trace_format(gsb_ctx* ctx, int64_t n, const int64_t* d_arrival, const int32_t* d_prompt,
                     const int32_t* d_output, const uint8_t* d_slo_class, char* d_out,
                     int64_t cap_bytes, int64_t* h_bytes, void* stream);

/* ---------------------------------------------------------------- simulator wire formats */
/* greensim::freq_timeline_csv / prefill_commands_csv (simkernel.cpp:686-714) rendered on the
 * GPU from device-resident SoA records (FreqChangeRecord / PrefillCommandRecord,
 * simkernel.hpp:131-146): header + one line per record, numbers as snprintf("%.10g") from the
 * exact binary value (simkernel.cpp:679-683), integers as std::to_string. d_out == NULL: size
 * query; *h_bytes = bytes. Synchronous. */
int gsb_freq_timeline_csv(gsb_ctx* ctx, int64_t n, const double* d_applied_ms,
                          const uint8_t* d_prefill_pool, const int32_t* d_worker,
                          const double* d_f_mhz, char* d_out, int64_t cap_bytes, int64_t* h_bytes,
                          void* stream);
int gsb_prefill_commands_csv(gsb_ctx* ctx, int64_t n, const double* d_tick_ms,
                             const int32_t* d_class, const int32_t* d_worker,
                             const double* d_f_mhz, const double* d_window_ms,
                             const uint8_t* d_infeasible, char* d_out, int64_t cap_bytes,
                             int64_t* h_bytes, void* stream);
/* greensim::decision_log_csv (decode_ctl.cpp:231-247) of K3b / K5 decision records: header +
 * one line per record, numbers as snprintf("%.6g"), worker / bucket as std::to_string, the
 * action by name. d_out == NULL: size query; *h_bytes = bytes. Synchronous. */
int gsb_decision_log_csv(gsb_ctx* ctx, int64_t n, const gsb_decision* d_records, char* d_out,
                         int64_t cap_bytes, int64_t* h_bytes, void* stream);
/* snprintf("%.10g") of n values: value i's text at d_out32 + 32*i, its length in d_len[i]. */
int gsb_format_g10(gsb_ctx* ctx, int64_t n, const double* d_values, char* d_out32,
                   int32_t* d_len, void* stream);
/* the same for snprintf("%.<precision>g"), precision 6 or 10 */
int gsb_format_g(gsb_ctx* ctx, int precision, int64_t n, const double* d_values, char* d_out32,
                 int32_t* d_len, void* stream);

/* ---------------------------------------------------------------- K3/K4: decode control */
/* Raw decode telemetry of S streams (one decode worker each), CSR layout:
 * events of stream s are [d_ev_off[s], d_ev_off[s+1]) sorted by time; event j emitted
 * d_tokens[j] tokens at d_t_ms[j] and recorded gaps [d_gap_off[j], d_gap_off[j+1]) into the
 * TBT ring in that order (simkernel.cpp:365-393). */
typedef struct gsb_telemetry {
  int64_t n_streams;
  const int64_t* d_ev_off;  /* [S+1] */
  const double* d_t_ms;     /* [E] */
  const int32_t* d_tokens;  /* [E] */
  const int64_t* d_gap_off; /* [E+1] (global gap indices) */
  const double* d_gaps;     /* [G] */
} gsb_telemetry;

/* Window statistics as Sim's ticks observe them (simkernel.cpp:441-458): the TbtWindow
 * P95 (nearest rank over the last `tbt_capacity` gaps, decode_ctl.cpp:120-128,
 * metrics.cpp:11-19) at every fine tick and the TpsWindow rate (decode_ctl.cpp:113-118,
 * window = coarse period) at every coarse tick, ticks up to t_end_ms inclusive.
 * Outputs [S][n_fine] and [S][n_coarse] where n_* = gsb_n_ticks(period, t_end_ms). */
int64_t gsb_n_ticks(double period_ms, double t_end_ms);
int gsb_window_series(gsb_ctx* ctx, const gsb_telemetry* tel, int tbt_capacity,
                      double fine_period_ms, double coarse_period_ms, double t_end_ms,
                      uint8_t* d_fine_has, double* d_fine_p95, double* d_coarse_tps,
                      void* stream);

/* Band tables for T (profile, t_slo, workers, max_batch) tuples on n_levels ascending
 * TPS levels (build_band_table, decode_ctl.cpp:76-111). Outputs [T][n_levels]. */
int gsb_build_band_tables(gsb_ctx* ctx, int64_t n_tables, const gsb_profile* d_profiles,
                          const int32_t* d_profile_of, const double* d_t_slo_ms,
                          const int32_t* d_workers, const int32_t* d_max_batch, int n_levels,
                          const double* d_levels, double* d_tps_lo, double* d_tps_hi,
                          double* d_f_opt, uint8_t* d_feasible, void* stream);

/* Open-loop DecodeController replay (decode_ctl.cpp:130-228) of N trajectories, one GPU
 * lane each, composed with the window series of stream d_stream_of[n] exactly as Sim's
 * fine/coarse/adapt ticks (simkernel.cpp:243-248,441-464; tie order coarse < adapt < fine).
 * Band table d_table_of[n] of the [T][n_buckets] tables (tps_hi, f_opt), clamped to
 * [f_min, f_max] of the grid. Per trajectory outputs:
 *   d_digest[n]  word-wise FNV-1a over (command, band_lo, band_hi, action|bucket<<32)
 *                of every DecisionRecord in log order
 *   d_n_rec[n]   number of DecisionRecords
 *   d_counts[n*8] per-action counts (optional)
 *   d_mean_cmd[n] mean fine-tick command in MHz, left-to-right sum / count (optional)
 *   d_records / rec_cap: full DecisionRecords, rec_cap per trajectory (optional)
 * The series' fine/coarse periods must equal every cfg's (checked on host). */
typedef struct gsb_replay_args {
  int64_t n_traj;
  const gsb_ctl_cfg* d_cfg;      /* [N] */
  const int32_t* d_table_of;     /* [N] */
  const int32_t* d_stream_of;    /* [N] */
  const int32_t* d_worker;       /* [N] DecisionRecord::worker */
  int32_t n_buckets;             /* per table */
  const double* d_tps_hi;        /* [T][n_buckets] */
  const double* d_f_opt;         /* [T][n_buckets] */
  double f_min_mhz, f_max_mhz;
  double fine_period_ms, coarse_period_ms, t_end_ms;
  const uint8_t* d_fine_has;     /* [S][n_fine] */
  const double* d_fine_p95;      /* [S][n_fine] */
  const double* d_coarse_tps;    /* [S][n_coarse] */
  uint64_t* d_digest;
  int64_t* d_n_rec;
  int32_t* d_counts;             /* optional */
  double* d_mean_cmd;            /* optional */
  gsb_decision* d_records;       /* optional */
  int64_t rec_cap;
} gsb_replay_args;
int gsb_decode_replay(gsb_ctx* ctx, const gsb_replay_args* a, void* stream);

/* Resumable DecodeController state (the private members of decode_ctl.hpp:129-151): band,
 * set point, last observations, coarse-loop streak, the adjustment counts adaptation reads,
 * and the controller's own (adapted) copy of the table's f_opt. initialized == 0 means "not
 * yet constructed": the kernel applies the constructor (decode_ctl.cpp:130-140) first. */
typedef struct gsb_ctl_state {
  double band_lo, band_hi, set_point, last_tps, last_p95;
  int32_t current_bucket, pending_bucket, consecutive;
  int32_t adj_total, adj_up, adj_down;
  int32_t initialized, pad_;
  double f_opt[GSB_MAX_BUCKETS];
} gsb_ctl_state;

/* Scripted DecodeController (decode_ctl.hpp:116-150 call sequences, e.g. the reference's own
 * unit tests): trajectory n executes calls [d_ev_off[n], d_ev_off[n+1]) in order, kind 0 =
 * on_fine_tick(t, has ? value : nullopt), 1 = on_coarse_tick(t, value), 2 = on_adapt_tick(t).
 * Uses a->n_traj, d_cfg, d_table_of, d_worker, n_buckets, d_tps_hi, d_f_opt, f_min/f_max,
 * d_digest, d_n_rec, d_records/rec_cap (records of THIS call, from index 0).
 * d_state [N] (optional, in/out): resumes each controller from its state (constructing it from
 * table d_table_of[n] when initialized == 0) and writes the state after the script back, so a
 * long-lived controller costs O(calls) in total. NULL = construct fresh, discard the state. */
int gsb_decode_script(gsb_ctx* ctx, const gsb_replay_args* a, const int64_t* d_ev_off,
                      const int8_t* d_kind, const double* d_t, const double* d_value,
                      const uint8_t* d_has, gsb_ctl_state* d_state, void* stream);

/* Nearest-rank quantile (metrics.cpp:11-19) of each of n_sets sample sets
 * [d_off[s], d_off[s+1]) of any size (TbtWindow::p95 is q = 0.95 over the ring; sets up to 4096
 * are sorted in shared memory, larger ones take an exact radix select). An empty set yields NaN
 * (the reference throws std::invalid_argument). */
int gsb_quantile_batch(gsb_ctx* ctx, double q, int64_t n_sets, const int64_t* d_off,
                       const double* d_samples, double* d_out, void* stream);

/* TpsWindow::tps(now) (decode_ctl.cpp:113-118) for n windows: events [d_off[w], d_off[w+1])
 * (time-sorted, as recorded) with window span d_window_ms[w], evaluated at d_now[w]. */
int gsb_tps_window_batch(gsb_ctx* ctx, int64_t n, const int64_t* d_off, const double* d_t,
                         const int32_t* d_tokens, const double* d_window_ms, const double* d_now,
                         double* d_out, void* stream);

/* decode_steady_state (decode_ctl.cpp:28-50) for n (tps, f, max_batch) points of one profile. */
int gsb_steady_state_batch(gsb_ctx* ctx, int64_t n, const gsb_profile* d_profile,
                           const double* d_tps, const double* d_f, const int32_t* d_max_batch,
                           uint8_t* d_sustainable, double* d_batch, double* d_tbt, void* stream);

/* Host-side validation of a replay batch (band tables + configs), host pointers. */
int gsb_replay_validate(const gsb_ctl_cfg* cfgs, int64_t n, int32_t n_buckets,
                        const double* tps_lo, const double* tps_hi, int64_t n_tables,
                        char* msg, size_t msg_cap);


/* ---------------------------------------------------------------- K5: closed-loop decode pool */
/* The decode side of the reference simulator (simkernel.cpp:330-464: continuous batching up to
 * max_batch, step time decode_step_raw_ms (gpu_model.cpp:99-103), least-loaded enqueue,
 * actuation delay, identical-target drop, per-worker power ledgers, TbtWindow/TpsWindow and the
 * DecodeController's fine/coarse/adapt ticks, which stop once nothing is outstanding) replayed
 * for N scenarios at once, one warp each. The input is the decode-enqueue stream: the
 * (time, request) pairs of simkernel.cpp:347 in the reference's processing order. The prefill
 * pool never waits on the decode pool, so one stream (recorded by the oracle's restated
 * simulator, or any caller's own) serves every decode parameter set. */
typedef struct gsb_pool_cfg {  /* SimConfig (simkernel.hpp:88-104) decode side + SloConfig */
  int32_t n_decode_workers;    /* 1..30 */
  int32_t max_batch;           /* 1..256 */
  int32_t max_queue;           /* per-worker backlog cap: enqueue at load >= cap is rejected */
  int32_t tbt_cap;             /* >= every scenario's tbt_window_tokens, <= GSB_MAX_TBT_WINDOW */
  int32_t tps_cap;             /* TpsWindow deque capacity (gsb_decode_pool_tps_cap) */
  int32_t pending_cap;         /* per-worker FIFO capacity (>= max_queue is always enough) */
  double actuation_delay_ms;
  double tbt_p95_ms;           /* SloConfig::tbt_p95_ms (pass-rate counts) */
} gsb_pool_cfg;

typedef struct gsb_pool_stream {
  int64_t n_streams;
  const int64_t* d_off;          /* [S+1] enqueues of stream s are [off[s], off[s+1]) */
  const double* d_t_ms;          /* [E] enqueue instants, processing order */
  const int32_t* d_req;          /* [E] request ids */
  const double* d_end_floor_ms;  /* [S] prefill side's part of sim_end_ms (NULL = 0) */
  int64_t n_requests;            /* per-request arrays below, indexed by request id */
  const int32_t* d_output_tokens;
  const double* d_arrival_ms;
  const double* d_ttft_slo_ms;   /* SloConfig::ttft_for(SM/L) of the request */
} gsb_pool_stream;

/* Decode-side outcome of one scenario. Digests (identical definitions in the oracle,
 * gs_oracle.h gso_pool_summary): decision_digest = FNV over workers of each worker's K3
 * record digest; freq_digest = FNV over workers of FNV-1a(applied_ms, f) of its applied
 * changes; request_digest = sum mod 2^64 of FNV-1a(id, first_token, finish, worker, n_gaps,
 * sum of gap bit patterns) per completed request (FNV-1a(id, 0xdead) per decode-side
 * rejection). status != 0 means a
 * capacity was exceeded (1 pending FIFO, 2 TPS deque, 4 pending clock applications, 8 tbt_cap
 * below a scenario's window): the scenario's outputs are then invalid. */
typedef struct gsb_pool_summary {
  double decode_pool_j, active_decode_j, idle_j, sim_end_ms;
  int64_t n_completed, n_rejected, n_ttft_ok, n_tbt_ok, tbt_samples, tbt_samples_ok;
  int64_t n_decisions, n_freq_changes, n_steps;
  uint64_t decision_digest, freq_digest, request_digest;
  int32_t status, pad_;
} gsb_pool_summary;

typedef struct gsb_pool_args {
  int64_t n_scen;
  const gsb_ctl_cfg* d_cfg;      /* [N] DecodeCtlConfig per scenario */
  const double* d_fixed_mhz;     /* [N] optional: > 0 pins every decode clock, no controller
                                    (FixedFreq; DefaultNV / PrefillSplit pass f_max) */
  const int32_t* d_table_of;     /* [N] band table (NULL = 0) */
  const int32_t* d_stream_of;    /* [N] enqueue stream (NULL = 0) */
  int32_t n_buckets;
  const double* d_tps_hi;        /* [T][n_buckets] */
  const double* d_f_opt;         /* [T][n_buckets] */
  gsb_pool_summary* d_out;       /* [N] */
  double* d_ledger;              /* optional [N][W][2]: active_decode_j, idle_j per worker */
  gsb_decision* d_records;       /* optional [N][W][rec_cap]: each worker's log in order */
  int64_t rec_cap;
  double* d_freq;                /* optional [N][W][freq_cap][2]: (applied_ms, f) per worker */
  int64_t freq_cap;
  int32_t* d_req_worker;         /* optional [N][n_requests]: RequestRecord::decode_worker */
  double* d_req_first;           /* optional [N][n_requests]: first_token_ms */
  double* d_req_finish;          /* optional [N][n_requests]: finish_ms */
} gsb_pool_args;

/* Upper bound on the TpsWindow deque length for a profile (2 coarse periods of the shortest
 * possible step + 3); -1 when unbounded or > 4096. */
int gsb_decode_pool_tps_cap(const gsb_profile* prof, int32_t max_batch, double coarse_period_ms);
/* prof is a HOST pointer (passed as a kernel parameter); everything in st / a is device memory. */
int gsb_decode_pool(gsb_ctx* ctx, const gsb_profile* prof, const gsb_pool_cfg* cfg,
                    const gsb_pool_stream* st, const gsb_pool_args* a, void* stream);

/* ---------------------------------------------------------------- multi-GPU reductions */
/* The path shards with no data exchange (windows / scenarios per rank); the
 * only collective is the end-of-run gather of small records, combined on every rank in RANK
 * ORDER, so the global result is bitwise identical everywhere (an fp64 all-reduce would not be).
 * The transport is the caller's: gather(d_send, d_recv, bytes, stream, user) must place every
 * rank's `bytes` from d_send into d_recv in rank order (device memory, on `stream`) and return 0
 * -- e.g. ncclAllGather(d_send, d_recv, bytes, ncclUint8, comm, stream) with comm in user
 * (INTEGRATION.md). This replaces the reference's serial sweep (simkernel.cpp:663-676). */
typedef int (*gsb_allgather_fn)(const void* d_send, void* d_recv, size_t bytes, void* stream,
                                void* user);

/* Rank-order combine of per-rank prefill summaries (host memory, [world][n_records], rank r's
 * cells offset by h_cell_offsets[r]): counts add, energies fold left to right over ranks, the
 * argmin keeps the lowest energy then the lowest global cell. No device needed. */
int gsb_combine_summaries(int world, int n_records, const gsb_class_summary* h_per_rank,
                          const int64_t* h_cell_offsets, gsb_class_summary* h_out);
/* gather (the caller's transport) + gsb_combine_summaries: d_local = this rank's n_records
 * summaries (device), h_out = the global records (host, identical on every rank). */
int gsb_reduce_summaries(gsb_ctx* ctx, int world, int rank, int n_records,
                         const gsb_class_summary* d_local, const int64_t* h_cell_offsets,
                         gsb_allgather_fn gather, void* user, gsb_class_summary* h_out,
                         void* stream);

/* Decode-pool end-of-run tally (the K5 scenario summaries of one rank folded in order). */
typedef struct gsb_decode_tally {
  int64_t n_scenarios;
  double decode_pool_j, min_decode_pool_j;
  int64_t argmin_scenario;
  int64_t n_completed, n_rejected, n_ttft_ok, n_tbt_ok, tbt_samples, tbt_samples_ok;
  int64_t n_decisions, n_freq_changes;
  uint64_t digest;  /* sum mod 2^64 of splitmix64(decision ^ freq ^ request digest ^ scenario) */
} gsb_decode_tally;
/* Fold n scenario summaries (host) of global scenarios [scen0, scen0 + n) in order. */
int gsb_tally_pool(int64_t n, const gsb_pool_summary* h_summary, int64_t scen0,
                   gsb_decode_tally* h_out);
/* Rank-order combine of [world] tallies (host). */
int gsb_combine_tallies(int world, const gsb_decode_tally* h_per_rank, gsb_decode_tally* h_out);
/* gather (caller's transport, device staging in the context) + gsb_combine_tallies. */
int gsb_reduce_tallies(gsb_ctx* ctx, int world, int rank, const gsb_decode_tally* h_local,
                       gsb_allgather_fn gather, void* user, gsb_decode_tally* h_out,
                       void* stream);

/* ---------------------------------------------------------------- microbenchmarks */
/* FP64 pipe peak probe: n_threads lanes each run `iters` independent DFMA chains;
 * returns the DFMA count in *d_out-sized work (used by bench.py for the roofline). */
int gsb_fp64_probe(gsb_ctx* ctx, int64_t n_threads, int iters, double* d_sink, void* stream);

/* Self-test of the correctly-rounded division used by K2/K3:
 * per_divisor random dividends for every clock of profile 0 and for 1000; writes the count
 * of results that differ in any bit from IEEE division to *d_mismatches. */
int gsb_selftest_division(gsb_ctx* ctx, int64_t per_divisor, uint64_t seed,
                          unsigned long long* d_mismatches, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GSB_H */
