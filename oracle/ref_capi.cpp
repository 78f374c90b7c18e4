// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C ABI over the UNMODIFIED reference library (/root/reference/proj/src, compiled
// by oracle/Makefile into oracle/_ref/libgreensim_ref.so). Python tests and the
// bench's CPU-baseline leg load it with ctypes to (a) pin the plain-C restatement
// (gs_oracle.c) and (b) time the reference's own CPU path. Nothing here is
// reference source; it only calls the reference's public API.
//
// Capture hooks: the Makefile links with -Wl,--wrap for queue_optimizer_tick and
// the DecodeController tick methods, so a reference `run()` can record the exact
// optimizer snapshots (simkernel.cpp:466-497) and controller inputs
// (simkernel.cpp:441-464) that the reference's own simulator produced.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <optional>
#include <thread>
#include <vector>

#include "greensim/decode_ctl.hpp"
#include "greensim/trace.hpp"
#include "greensim/gpu_model.hpp"
#include "greensim/metrics.hpp"
#include "greensim/prefill_opt.hpp"
#include "greensim/router.hpp"
#include "greensim/simkernel.hpp"
#include "greensim/trace.hpp"
#include "gs_oracle.h"

using namespace greensim;

namespace {

GpuProfile to_profile(const gso_profile* c) {
  GpuProfile p;
  p.name = "capi";
  p.grid = FrequencyGrid{c->f_min_mhz, c->f_max_mhz, c->step_mhz, c->f_ref_mhz};
  p.prefill = LatencyModel{c->lat_a, c->lat_b, c->lat_c, c->lat_f_ref_mhz};
  p.decode = DecodeStepModel{c->dec_alpha0_ms, c->dec_alpha1_ms, c->dec_beta0_ms, c->dec_beta1_ms,
                             c->dec_f_ref_mhz};
  p.power = PowerModel{c->k3, c->k2, c->k1, c->k0, c->p_idle_w};
  return p;
}

DecodeCtlConfig to_cfg(const gso_ctl_cfg* c) {
  DecodeCtlConfig d;
  d.tslo_ms = c->tslo_ms;
  d.margin_decode = c->margin_decode;
  d.fine_period_ms = c->fine_period_ms;
  d.coarse_period_ms = c->coarse_period_ms;
  d.adapt_period_s = c->adapt_period_s;
  d.step_mhz = c->step_mhz;
  d.max_step_mhz = c->max_step_mhz;
  d.hysteresis_count = c->hysteresis_count;
  d.tbt_window_tokens = c->tbt_window_tokens;
  d.bias_threshold = c->bias_threshold;
  d.tps_scale = c->tps_scale;
  d.upper_margin = c->upper_margin;
  d.lower_margin = c->lower_margin;
  return d;
}

QueueOptimizerConfig to_qcfg(const gso_qopt_cfg* c) {
  QueueOptimizerConfig q;
  q.resolve_period_ms = c->resolve_period_ms;
  q.margin_prefill = c->margin_prefill;
  q.min_budget_ms = c->min_budget_ms;
  q.first_token_allowance_ms = c->first_token_allowance_ms;
  return q;
}

PrefillBatch to_batch(int64_t n, const int32_t* prompt, const double* wf, const double* deadline) {
  PrefillBatch b;
  b.jobs.reserve(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k)
    b.jobs.push_back(PrefillJob{k, prompt[k], deadline ? deadline[k] : 0.0, wf ? wf[k] : 1.0});
  return b;
}

int action_code(const std::string& a) {
  static const char* names[] = {"hold",           "up",           "down",       "coarse_hold",
                                "coarse_pending", "coarse_commit", "adapt_up", "adapt_down"};
  for (int i = 0; i < 8; ++i)
    if (a == names[i]) return i;
  return -1;
}

void to_c_record(const DecisionRecord& r, gso_decision* o) {
  o->tick_ms = r.tick_ms;
  o->tps = r.tps;
  o->p95_tbt_ms = r.p95_tbt_ms;
  o->band_lo = r.band_lo;
  o->band_hi = r.band_hi;
  o->command_mhz = r.command_mhz;
  o->worker = r.worker;
  o->bucket = r.bucket;
  o->action = action_code(r.action);
  o->pad_ = 0;
}

FreqBandTable to_table(const gso_band_table* t) {
  FreqBandTable out;
  for (int i = 0; i < t->n; ++i) out.buckets.push_back({t->tps_lo[i], t->tps_hi[i], t->f_opt_mhz[i], true});
  return out;
}

// ---- capture state for the --wrap hooks -------------------------------------------------
struct Capture {
  bool on = false;
  // optimizer snapshots (one per non-empty or empty class queue at each tick)
  std::vector<double> snap_now;
  std::vector<int32_t> snap_class;
  std::vector<int64_t> snap_off{0};
  std::vector<int64_t> job_id;
  std::vector<int32_t> job_prompt;
  std::vector<double> job_deadline, job_wf;
  // commands returned per tick (class-ordered)
  std::vector<double> cmd_now, cmd_f, cmd_window;
  std::vector<int32_t> cmd_class;
  std::vector<uint8_t> cmd_infeasible;
  // controller inputs
  std::map<const void*, int> ctl_index;
  std::vector<int32_t> fine_worker;
  std::vector<double> fine_t, fine_p95;
  std::vector<uint8_t> fine_has;
  std::vector<int32_t> coarse_worker;
  std::vector<double> coarse_t, coarse_tps;
  std::vector<int32_t> adapt_worker;
  std::vector<double> adapt_t;
  int worker_of(const void* self) {
    auto it = ctl_index.find(self);
    if (it != ctl_index.end()) return it->second;
    const int w = static_cast<int>(ctl_index.size());
    ctl_index.emplace(self, w);
    return w;
  }
};
thread_local Capture g_cap;

}  // namespace

// ---- --wrap hooks (symbols resolved by the linker; see oracle/Makefile) ------------------
#define QOT _ZN8greensim20queue_optimizer_tickERKSt6vectorINS_18ClassQueueSnapshotESaIS1_EEdRKNS_20QueueOptimizerConfigERKNS_10GpuProfileE
#define FINE _ZN8greensim16DecodeController12on_fine_tickEdSt8optionalIdE
#define COARSE _ZN8greensim16DecodeController14on_coarse_tickEdd
#define ADAPT _ZN8greensim16DecodeController13on_adapt_tickEd
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)

extern "C" {
std::vector<PrefillFreqCommand> CAT(__real_, QOT)(const std::vector<ClassQueueSnapshot>&, double,
                                                  const QueueOptimizerConfig&, const GpuProfile&);
std::vector<PrefillFreqCommand> CAT(__wrap_, QOT)(const std::vector<ClassQueueSnapshot>& q,
                                                  double now, const QueueOptimizerConfig& cfg,
                                                  const GpuProfile& p) {
  auto out = CAT(__real_, QOT)(q, now, cfg, p);
  if (g_cap.on) {
    for (const auto& s : q) {
      g_cap.snap_now.push_back(now);
      g_cap.snap_class.push_back(s.class_id);
      for (const auto& j : s.batch.jobs) {
        g_cap.job_id.push_back(j.request_id);
        g_cap.job_prompt.push_back(j.prompt_tokens);
        g_cap.job_deadline.push_back(j.deadline_ms);
        g_cap.job_wf.push_back(j.work_fraction);
      }
      g_cap.snap_off.push_back(static_cast<int64_t>(g_cap.job_id.size()));
    }
    for (const auto& c : out) {
      g_cap.cmd_now.push_back(now);
      g_cap.cmd_class.push_back(c.class_id);
      g_cap.cmd_f.push_back(c.f_mhz);
      g_cap.cmd_window.push_back(c.window_ms);
      g_cap.cmd_infeasible.push_back(c.infeasible ? 1 : 0);
    }
  }
  return out;
}

double CAT(__real_, FINE)(DecodeController*, double, std::optional<double>);
double CAT(__wrap_, FINE)(DecodeController* self, double now, std::optional<double> p95) {
  if (g_cap.on) {
    g_cap.fine_worker.push_back(g_cap.worker_of(self));
    g_cap.fine_t.push_back(now);
    g_cap.fine_has.push_back(p95.has_value() ? 1 : 0);
    g_cap.fine_p95.push_back(p95.value_or(0.0));
  }
  return CAT(__real_, FINE)(self, now, p95);
}
void CAT(__real_, COARSE)(DecodeController*, double, double);
void CAT(__wrap_, COARSE)(DecodeController* self, double now, double tps) {
  if (g_cap.on) {
    g_cap.coarse_worker.push_back(g_cap.worker_of(self));
    g_cap.coarse_t.push_back(now);
    g_cap.coarse_tps.push_back(tps);
  }
  CAT(__real_, COARSE)(self, now, tps);
}
void CAT(__real_, ADAPT)(DecodeController*, double);
void CAT(__wrap_, ADAPT)(DecodeController* self, double now) {
  if (g_cap.on) {
    g_cap.adapt_worker.push_back(g_cap.worker_of(self));
    g_cap.adapt_t.push_back(now);
  }
  CAT(__real_, ADAPT)(self, now);
}
}  // extern "C"

// ---- plain C API ------------------------------------------------------------------------
extern "C" {

int ref_profile_validate(const gso_profile* c) {
  try {
    to_profile(c).validate();
    return 0;
  } catch (const ModelError&) {
    return -1;
  }
}

void ref_default_profile(gso_profile* c) {
  const GpuProfile p = GpuProfile::default_profile();
  *c = gso_profile{p.grid.f_min_mhz,    p.grid.f_max_mhz,    p.grid.step_mhz,     p.grid.f_ref_mhz,
                   p.prefill.a,         p.prefill.b,         p.prefill.c,         p.prefill.f_ref_mhz,
                   p.decode.alpha0_ms,  p.decode.alpha1_ms,  p.decode.beta0_ms,   p.decode.beta1_ms,
                   p.decode.f_ref_mhz,  p.power.k3,          p.power.k2,          p.power.k1,
                   p.power.k0,          p.power.p_idle_w};
}

double ref_active_power_w(const gso_profile* c, double f) { return to_profile(c).active_power_w(f); }

double ref_t_ref_total_ms(const gso_profile* c, int64_t n, const int32_t* prompt, const double* wf) {
  return to_batch(n, prompt, wf, nullptr).t_ref_total_ms(to_profile(c).prefill);
}

int ref_energy_total(const gso_profile* c, int64_t n, const int32_t* prompt, const double* wf,
                     double f, double window, double* active, double* idle, double* total,
                     int* feasible) {
  try {
    const auto e = energy_total(to_batch(n, prompt, wf, nullptr), f, window, to_profile(c));
    *active = e.active_j;
    *idle = e.idle_j;
    *total = e.total_j;
    *feasible = e.feasible ? 1 : 0;
    return 0;
  } catch (const ModelError&) {
    return -1;
  }
}

double ref_energy_closed_form(const gso_profile* c, int64_t n, const int32_t* prompt,
                              const double* wf, double f, double window) {
  return energy_total_closed_form_j(to_batch(n, prompt, wf, nullptr), f, window, to_profile(c));
}

// returns 1 if a feasible clock exists (f/e written), 0 for nullopt
int ref_select_frequency(const gso_profile* c, int64_t n, const int32_t* prompt, const double* wf,
                         double window, double* f_out, double* e_out) {
  const auto r = select_frequency(to_batch(n, prompt, wf, nullptr), window, to_profile(c));
  if (!r) return 0;
  *f_out = r->f_mhz;
  *e_out = r->energy_j;
  return 1;
}

// Batched select_frequency over ragged batches (used as the timed CPU baseline);
// threads > 1 splits batches over std::threads with thread-local profile copies.
void ref_select_frequency_many(const gso_profile* c, int64_t n_batches, const int64_t* off,
                               const int32_t* prompt, const double* wf, const double* windows,
                               int threads, double* f_out, double* e_out, uint8_t* found) {
  auto work = [&](int64_t lo, int64_t hi) {
    const GpuProfile prof = to_profile(c);
    PrefillBatch b;
    for (int64_t i = lo; i < hi; ++i) {
      b.jobs.clear();
      for (int64_t k = off[i]; k < off[i + 1]; ++k)
        b.jobs.push_back(PrefillJob{k, prompt[k], 0.0, wf ? wf[k] : 1.0});
      if (b.jobs.empty()) {
        found[i] = 0;
        continue;
      }
      const auto r = select_frequency(b, windows[i], prof);
      found[i] = r ? 1 : 0;
      f_out[i] = r ? r->f_mhz : 0.0;
      e_out[i] = r ? r->energy_j : 0.0;
    }
  };
  if (threads <= 1) {
    work(0, n_batches);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = n_batches * t / threads, hi = n_batches * (t + 1) / threads;
    pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
}

// The reference's own CPU path for one offline prefill pass over a trace (bench.py's reference
// arm and cpu_baseline; DESIGN.md offline window convention): window k covers arrivals in
// [(w0+k)*window_ms, (w0+k+1)*window_ms). Per window, Dispatcher::dispatch (router.cpp:33-43)
// routes its requests into per-class FIFOs, each non-empty queue is drained with
// Dispatcher::pop into a PrefillBatch in FIFO order, and select_frequency (prefill_opt.cpp:45-56)
// runs for every profile with window D. Windows are split into contiguous ranges, one std::thread
// and one Dispatcher each (request ids are the trace indices, so no id repeats). Outputs per
// (p, cell = k*C + c) at p*cells + cell, optional: grid index of the choice (-1 infeasible, -2
// empty queue) and its energy (0 otherwise). Returns the number of (cell, profile) pairs that
// ran select_frequency (each evaluates every grid clock).
//
// mode 1 (DEADLINE_SLACK) instead calls queue_optimizer_tick (prefill_opt.cpp:58-82) once per
// window and profile at now = window start over the window's class snapshots, each job carrying
// the simulator's prefill deadline arrival + ttft_for(request_class(r, 1024)) - allowance
// (simkernel.cpp:113-116,298,499-501): f_idx -1 marks an infeasible command (pinned at f_max),
// window_out[cell] receives the command's window (profile 0), energy is not produced.
int64_t ref_prefill_pass_ex(int mode, int n_prof, const gso_profile* profs, int enabled, int n_thr,
                            const int32_t* thr, int64_t n_req, const int64_t* arrival,
                            const int32_t* prompt, int64_t window_ms, int64_t w0,
                            int64_t n_windows, double D, const gso_qopt_cfg* qc, double ttft_sm,
                            double ttft_l, int threads, int16_t* f_idx, double* energy,
                            double* window_out) {
  RoutingConfig cfg;
  cfg.enabled = enabled != 0;
  cfg.thresholds.assign(thr, thr + n_thr);
  const int C = cfg.enabled ? n_thr + 1 : 1;
  const int64_t cells = n_windows * C;
  std::vector<GpuProfile> prof;
  for (int p = 0; p < n_prof; ++p) prof.push_back(to_profile(&profs[p]));
  threads = std::max(1, threads);
  std::vector<int64_t> evaluated(static_cast<size_t>(threads), 0);
  auto work = [&](int t) {
    const int64_t k0 = n_windows * t / threads, k1 = n_windows * (t + 1) / threads;
    Dispatcher d(cfg);
    int64_t i = std::lower_bound(arrival, arrival + n_req, (w0 + k0) * window_ms) - arrival;
    PrefillBatch b;
    int64_t ev = 0;
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t end_ms = (w0 + k + 1) * window_ms;
      for (; i < n_req && arrival[i] < end_ms; ++i) {
        Request r;
        r.id = i;
        r.arrival_ms = arrival[i];
        r.prompt_tokens = prompt[i];
        r.output_tokens = 1;
        d.dispatch(r);
      }
      if (mode == 1) {
        QueueOptimizerConfig qcfg;
        qcfg.resolve_period_ms = qc->resolve_period_ms;
        qcfg.margin_prefill = qc->margin_prefill;
        qcfg.min_budget_ms = qc->min_budget_ms;
        qcfg.first_token_allowance_ms = qc->first_token_allowance_ms;
        std::vector<ClassQueueSnapshot> snaps(static_cast<size_t>(C));
        for (int q = 0; q < C; ++q) {
          snaps[static_cast<size_t>(q)].class_id = q;
          for (int p = 0; p < n_prof && f_idx; ++p) f_idx[p * cells + k * C + q] = -2;
          while (!d.empty(q)) {
            const int64_t id = d.pop(q);
            const double arr = static_cast<double>(arrival[id]);
            const double ttft = prompt[id] <= 1024 ? ttft_sm : ttft_l;
            snaps[static_cast<size_t>(q)].batch.jobs.push_back(
                PrefillJob{id, prompt[id], arr + ttft - qcfg.first_token_allowance_ms, 1.0});
          }
        }
        const double now = static_cast<double>((w0 + k) * window_ms);
        for (int p = 0; p < n_prof; ++p) {
          const auto cmds = queue_optimizer_tick(snaps, now, qcfg, prof[static_cast<size_t>(p)]);
          ev += static_cast<int64_t>(cmds.size());
          for (const auto& c : cmds) {
            const int64_t cell = k * C + c.class_id;
            if (f_idx)
              f_idx[p * cells + cell] =
                  c.infeasible ? int16_t{-1}
                               : static_cast<int16_t>(std::llround(
                                     (c.f_mhz - profs[p].f_min_mhz) / profs[p].step_mhz));
            if (window_out && p == 0) window_out[cell] = c.window_ms;
          }
        }
        continue;
      }
      for (int q = 0; q < C; ++q) {
        const int64_t cell = k * C + q;
        if (d.empty(q)) {
          for (int p = 0; p < n_prof; ++p) {
            if (f_idx) f_idx[p * cells + cell] = -2;
            if (energy) energy[p * cells + cell] = 0.0;
          }
          continue;
        }
        b.jobs.clear();
        while (!d.empty(q)) {
          const int64_t id = d.pop(q);
          b.jobs.push_back(PrefillJob{id, prompt[id], 0.0, 1.0});
        }
        for (int p = 0; p < n_prof; ++p) {
          const auto r = select_frequency(b, D, prof[static_cast<size_t>(p)]);
          ++ev;
          if (f_idx)
            f_idx[p * cells + cell] = r ? static_cast<int16_t>(std::llround(
                                              (r->f_mhz - profs[p].f_min_mhz) / profs[p].step_mhz))
                                        : int16_t{-1};
          if (energy) energy[p * cells + cell] = r ? r->energy_j : 0.0;
        }
      }
    }
    evaluated[static_cast<size_t>(t)] = ev;
  };
  if (threads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  int64_t total = 0;
  for (int64_t e : evaluated) total += e;
  return total;
}

int64_t ref_prefill_pass(int n_prof, const gso_profile* profs, int enabled, int n_thr,
                         const int32_t* thr, int64_t n_req, const int64_t* arrival,
                         const int32_t* prompt, int64_t window_ms, int64_t w0, int64_t n_windows,
                         double D, int threads, int16_t* f_idx, double* energy) {
  return ref_prefill_pass_ex(0, n_prof, profs, enabled, n_thr, thr, n_req, arrival, prompt,
                             window_ms, w0, n_windows, D, nullptr, 0.0, 0.0, threads, f_idx,
                             energy, nullptr);
}

// freq_timeline_csv / prefill_commands_csv (simkernel.cpp:686-714) over SoA records; returns
// the byte count, copying at most cap bytes into out.
int64_t ref_freq_timeline_csv(int64_t n, const double* applied, const uint8_t* pool,
                              const int32_t* worker, const double* f, char* out, int64_t cap) {
  std::vector<FreqChangeRecord> r(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i)
    r[static_cast<size_t>(i)] = FreqChangeRecord{applied[i], pool[i] != 0, worker[i], f[i]};
  const std::string s = freq_timeline_csv(r);
  std::memcpy(out, s.data(), static_cast<size_t>(std::min<int64_t>(cap, s.size())));
  return static_cast<int64_t>(s.size());
}

int64_t ref_prefill_commands_csv(int64_t n, const double* tick, const int32_t* cls,
                                 const int32_t* worker, const double* f, const double* window,
                                 const uint8_t* infeasible, char* out, int64_t cap) {
  std::vector<PrefillCommandRecord> r(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i)
    r[static_cast<size_t>(i)] =
        PrefillCommandRecord{tick[i], cls[i], worker[i], f[i], window[i], infeasible[i] != 0};
  const std::string s = prefill_commands_csv(r);
  std::memcpy(out, s.data(), static_cast<size_t>(std::min<int64_t>(cap, s.size())));
  return static_cast<int64_t>(s.size());
}

// decision_log_csv (decode_ctl.cpp:237-247) over records in the gsb_decision layout (6 doubles:
// tick, tps, p95, band_lo, band_hi, command; then worker, bucket, action index, pad). Its
// ostringstream does not survive the Python interpreter's libstdc++ once numpy is loaded: call
// it through oracle/_ref/ref_save_trace --decisions (Reference.decision_log_csv does).
struct RefDecisionIn {
  double tick_ms, tps, p95_tbt_ms, band_lo, band_hi, command_mhz;
  int32_t worker, bucket, action, pad_;
};
int64_t ref_decision_log_csv(int64_t n, const RefDecisionIn* rec, char* out, int64_t cap) {
  static const char* const kNames[8] = {"hold",           "up",            "down",
                                        "coarse_hold",    "coarse_pending", "coarse_commit",
                                        "adapt_up",       "adapt_down"};
  std::vector<DecisionRecord> r(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    const RefDecisionIn& d = rec[i];
    DecisionRecord& x = r[static_cast<size_t>(i)];
    x.tick_ms = d.tick_ms;
    x.worker = d.worker;
    x.tps = d.tps;
    x.p95_tbt_ms = d.p95_tbt_ms;
    x.bucket = d.bucket;
    x.band_lo = d.band_lo;
    x.band_hi = d.band_hi;
    x.command_mhz = d.command_mhz;
    x.action = kNames[d.action & 7];
  }
  const std::string s = decision_log_csv(r);
  if (out) std::memcpy(out, s.data(), static_cast<size_t>(std::min<int64_t>(cap, s.size())));
  return static_cast<int64_t>(s.size());
}

// queue_optimizer_tick over n_queues snapshots at one instant; returns #commands.
int ref_queue_optimizer_tick(const gso_profile* c, const gso_qopt_cfg* qc, int n_queues,
                             const int32_t* class_ids, const int64_t* off, const int32_t* prompt,
                             const double* deadline, const double* wf, double now,
                             int32_t* cmd_class, double* cmd_f, double* cmd_window,
                             uint8_t* cmd_infeasible) {
  std::vector<ClassQueueSnapshot> snaps;
  for (int q = 0; q < n_queues; ++q) {
    ClassQueueSnapshot s;
    s.class_id = class_ids[q];
    for (int64_t k = off[q]; k < off[q + 1]; ++k)
      s.batch.jobs.push_back(PrefillJob{k, prompt[k], deadline[k], wf ? wf[k] : 1.0});
    snaps.push_back(std::move(s));
  }
  const auto cmds = queue_optimizer_tick(snaps, now, to_qcfg(qc), to_profile(c));
  for (size_t i = 0; i < cmds.size(); ++i) {
    cmd_class[i] = cmds[i].class_id;
    cmd_f[i] = cmds[i].f_mhz;
    cmd_window[i] = cmds[i].window_ms;
    cmd_infeasible[i] = cmds[i].infeasible ? 1 : 0;
  }
  return static_cast<int>(cmds.size());
}

int ref_classify(int n_thr, const int32_t* thr, int32_t prompt) {
  RoutingConfig cfg;
  cfg.thresholds.assign(thr, thr + n_thr);
  return classify(cfg, prompt);
}

// Dispatcher over a request list: queue index per request and the per-queue FIFO
// contents concatenated queue-major. Returns 0, or -1 on RouterError.
int ref_dispatch(int enabled, int n_thr, const int32_t* thr, int64_t n, const int64_t* ids,
                 const int32_t* prompt, int32_t* queue_out, int64_t* fifo_out,
                 int64_t* queue_sizes) {
  RoutingConfig cfg;
  cfg.enabled = enabled != 0;
  cfg.thresholds.assign(thr, thr + n_thr);
  try {
    Dispatcher d(cfg);
    for (int64_t i = 0; i < n; ++i) {
      Request r;
      r.id = ids[i];
      r.arrival_ms = i;
      r.prompt_tokens = prompt[i];
      r.output_tokens = 1;
      queue_out[i] = d.dispatch(r);
    }
    int64_t pos = 0;
    for (int q = 0; q < d.n_queues(); ++q) {
      queue_sizes[q] = static_cast<int64_t>(d.size(q));
      for (int64_t id : d.queue(q)) fifo_out[pos++] = id;
    }
    return 0;
  } catch (const RouterError&) {
    return -1;
  }
}

double ref_quantile(int64_t n, const double* s, double q) {
  return quantile(std::span<const double>(s, static_cast<size_t>(n)), q);
}

int ref_decode_steady_state(const gso_profile* c, double tps, double f, int max_batch,
                            double* batch, double* tbt) {
  const auto ss = decode_steady_state(to_profile(c), tps, f, max_batch);
  *batch = ss.batch;
  *tbt = ss.tbt_ms;
  return ss.sustainable ? 1 : 0;
}

int ref_build_band_table(const gso_profile* c, int n, const double* levels, double t_slo,
                         int workers, int max_batch, double* lo, double* hi, double* fopt,
                         uint8_t* feasible) {
  try {
    const auto t = build_band_table(to_profile(c), std::span<const double>(levels, n), t_slo,
                                    workers, max_batch);
    for (int i = 0; i < n; ++i) {
      lo[i] = t.buckets[i].tps_lo;
      hi[i] = t.buckets[i].tps_hi;
      fopt[i] = t.buckets[i].f_opt_mhz;
      feasible[i] = t.buckets[i].feasible ? 1 : 0;
    }
    return 0;
  } catch (const ModelError&) {
    return -1;
  }
}

int ref_ctl_cfg_validate(const gso_ctl_cfg* c) {
  try {
    to_cfg(c).validate();
    return 0;
  } catch (const ModelError&) {
    return -1;
  }
}

// TpsWindow / TbtWindow direct drivers for window-semantics tests.
double ref_tps_window(double window_ms, int64_t n, const double* t, const int32_t* tokens,
                      double now) {
  TpsWindow w(window_ms);
  for (int64_t i = 0; i < n; ++i) w.record(t[i], tokens[i]);
  return w.tps(now);
}

double ref_tbt_window_p95(int capacity, int64_t n, const double* gaps) {
  TbtWindow w(capacity);
  for (int64_t i = 0; i < n; ++i) w.record(gaps[i]);
  return w.p95();
}

// Open-loop replay: DecodeController + TbtWindow + TpsWindow composed in Sim's order
// (simkernel.cpp:441-464 with the (t, kind) tie-break of simkernel.cpp:21-31,44-50).
int64_t ref_replay_telemetry(const gso_ctl_cfg* cc, const gso_band_table* tb, double f_min,
                             double f_max, double step, double f_ref, int worker,
                             const gso_telemetry* tel, double t_end, gso_decision* out,
                             int64_t cap) {
  try {
    const DecodeCtlConfig cfg = to_cfg(cc);
    DecodeController ctl(cfg, to_table(tb), FrequencyGrid{f_min, f_max, step, f_ref}, worker);
    TbtWindow tbt(cfg.tbt_window_tokens);
    TpsWindow tps(cfg.coarse_period_ms);
    double tf = cfg.fine_period_ms, tc = cfg.coarse_period_ms, ta = cfg.adapt_period_s * 1000.0;
    int64_t j = 0;
    for (;;) {
      const double t = std::min(tf, std::min(tc, ta));
      if (t > t_end) break;
      while (j < tel->n_events && tel->t_ms[j] <= t) {
        for (int64_t g = tel->gap_off[j]; g < tel->gap_off[j + 1]; ++g) tbt.record(tel->gaps[g]);
        tps.record(tel->t_ms[j], tel->tokens[j]);
        ++j;
      }
      if (tc == t) {
        ctl.on_coarse_tick(t, tps.tps(t));
        tc = t + cfg.coarse_period_ms;
      }
      if (ta == t) {
        ctl.on_adapt_tick(t);
        ta = t + cfg.adapt_period_s * 1000.0;
      }
      if (tf == t) {
        std::optional<double> p95;
        if (!tbt.empty()) p95 = tbt.p95();
        ctl.on_fine_tick(t, p95);
        tf = t + cfg.fine_period_ms;
      }
    }
    const auto& log = ctl.log();
    const int64_t n = static_cast<int64_t>(log.size());
    for (int64_t i = 0; i < n && i < cap; ++i) to_c_record(log[static_cast<size_t>(i)], out + i);
    return n;
  } catch (const ModelError&) {
    return -1;
  }
}

// DecodeController driven by an explicit call script (kind 0 fine, 1 coarse, 2 adapt), the
// shape of the reference's own unit tests; also returns command(), current_bucket() and the
// (adapted) table f_opt after the script.
int64_t ref_decode_script(const gso_ctl_cfg* cc, const gso_band_table* tb, double f_min,
                          double f_max, double step, double f_ref, int worker, int64_t n_ev,
                          const int8_t* kind, const double* t, const double* value,
                          const uint8_t* has, gso_decision* out, int64_t cap, double* final_cmd,
                          int32_t* final_bucket, double* final_f_opt) {
  try {
    DecodeController ctl(to_cfg(cc), to_table(tb), FrequencyGrid{f_min, f_max, step, f_ref}, worker);
    for (int64_t e = 0; e < n_ev; ++e) {
      if (kind[e] == 1) {
        ctl.on_coarse_tick(t[e], value[e]);
      } else if (kind[e] == 2) {
        ctl.on_adapt_tick(t[e]);
      } else {
        std::optional<double> p;
        if (has[e]) p = value[e];
        ctl.on_fine_tick(t[e], p);
      }
    }
    const auto& log = ctl.log();
    const int64_t n = static_cast<int64_t>(log.size());
    for (int64_t i = 0; i < n && i < cap; ++i) to_c_record(log[static_cast<size_t>(i)], out + i);
    *final_cmd = ctl.command();
    *final_bucket = ctl.current_bucket();
    for (std::size_t b = 0; b < ctl.table().buckets.size(); ++b) final_f_opt[b] = ctl.table().buckets[b].f_opt_mhz;
    return n;
  } catch (const ModelError&) {
    return -1;
  }
}

// Open-loop replay of many scenarios on shared telemetry (timed CPU baseline).
// Scenario s uses cfgs[s], tables[table_of[s]], telemetry tels[tel_of[s]], worker id
// worker_of[s]; emits per-scenario record counts and FNV digests.
void ref_replay_many(int64_t n_scen, const gso_ctl_cfg* cfgs, const gso_band_table* tables,
                     const int32_t* table_of, const gso_telemetry* tels, const int32_t* tel_of,
                     const int32_t* worker_of, double f_min, double f_max, double step,
                     double f_ref, double t_end, int threads, int64_t* n_records,
                     uint64_t* digests);

int64_t ref_gen_poisson_trace(double qps, int64_t duration, double short_mean, double long_mean,
                              double long_fraction, double output_mean, uint64_t seed,
                              int64_t cap, int64_t* arrival, int32_t* prompt, int32_t* output) {
  LoadShape s;
  s.kind = LoadShapeKind::PoissonQps;
  s.rate = qps;
  s.prompt_mean_short = short_mean;
  s.prompt_mean_long = long_mean;
  s.long_fraction = long_fraction;
  s.output_mean = output_mean;
  const Trace t = gen_poisson_trace(qps, duration, s, seed);
  const int64_t n = static_cast<int64_t>(t.requests.size());
  for (int64_t i = 0; i < n && i < cap; ++i) {
    arrival[i] = t.requests[i].arrival_ms;
    prompt[i] = t.requests[i].prompt_tokens;
    output[i] = t.requests[i].output_tokens;
  }
  return n;
}

int64_t ref_gen_sinusoid_decode_trace(double mean, double amp, double period, int64_t duration,
                                      uint64_t seed, int64_t cap, int64_t* arrival,
                                      int32_t* prompt, int32_t* output) {
  const Trace t = gen_sinusoid_decode_trace(mean, amp, period, duration, seed);
  const int64_t n = static_cast<int64_t>(t.requests.size());
  for (int64_t i = 0; i < n && i < cap; ++i) {
    arrival[i] = t.requests[i].arrival_ms;
    prompt[i] = t.requests[i].prompt_tokens;
    output[i] = t.requests[i].output_tokens;
  }
  return n;
}

// ---- captured reference run ---------------------------------------------------------------
struct RefRun {
  RunResult result;
  Capture cap;
  std::vector<gso_decision> decisions;
};

// Runs the reference simulator (policy: 0 defaultnv, 1 fixed, 2 greenllm, 3 prefillsplit)
// with the capture hooks on. Returns an owning handle (ref_run_free).
void* ref_run_capture(int64_t n, const int64_t* arrival, const int32_t* prompt,
                      const int32_t* output, const gso_profile* prof, int policy, double fixed_f,
                      int n_thr, const int32_t* thr, int n_prefill_workers,
                      const int32_t* worker_map, const gso_qopt_cfg* qcfg,
                      const gso_ctl_cfg* ccfg) {
  Trace tr;
  tr.meta.name = "capi";
  for (int64_t i = 0; i < n; ++i) {
    Request r;
    r.id = i;
    r.arrival_ms = arrival[i];
    r.prompt_tokens = prompt[i];
    r.output_tokens = output[i];
    tr.requests.push_back(r);
    tr.meta.duration_ms = std::max(tr.meta.duration_ms, arrival[i]);
  }
  GovernorPolicy pol;
  switch (policy) {
    case 0: pol = GovernorPolicy::default_nv(); break;
    case 1: pol = GovernorPolicy::fixed(fixed_f); break;
    case 2: pol = GovernorPolicy::greenllm(); break;
    default: pol = GovernorPolicy::prefill_split(); break;
  }
  if (policy >= 2) {
    pol.routing.thresholds.assign(thr, thr + n_thr);
    pol.routing.worker_map.assign(worker_map, worker_map + n_prefill_workers);
  }
  if (qcfg) pol.prefill_opt = to_qcfg(qcfg);
  if (ccfg) pol.decode_ctl = to_cfg(ccfg);
  SimConfig sc;
  sc.n_prefill_workers = n_prefill_workers;
  auto* rr = new RefRun;
  g_cap = Capture{};
  g_cap.on = true;
  try {
    rr->result = run(tr, to_profile(prof), pol, 1, SloConfig{}, sc);
  } catch (...) {
    g_cap.on = false;
    delete rr;
    return nullptr;
  }
  g_cap.on = false;
  rr->cap = std::move(g_cap);
  g_cap = Capture{};
  for (const auto& d : rr->result.decode_decisions) {
    gso_decision c;
    to_c_record(d, &c);
    rr->decisions.push_back(c);
  }
  return rr;
}

void ref_run_free(void* h) { delete static_cast<RefRun*>(h); }

// Sizes: [0] snapshots, [1] jobs, [2] commands, [3] fine, [4] coarse, [5] adapt,
// [6] decisions, [7] requests, [8] controllers.
void ref_run_sizes(void* h, int64_t* s) {
  const auto* r = static_cast<RefRun*>(h);
  s[0] = static_cast<int64_t>(r->cap.snap_now.size());
  s[1] = static_cast<int64_t>(r->cap.job_id.size());
  s[2] = static_cast<int64_t>(r->cap.cmd_now.size());
  s[3] = static_cast<int64_t>(r->cap.fine_t.size());
  s[4] = static_cast<int64_t>(r->cap.coarse_t.size());
  s[5] = static_cast<int64_t>(r->cap.adapt_t.size());
  s[6] = static_cast<int64_t>(r->decisions.size());
  s[7] = static_cast<int64_t>(r->result.requests.size());
  s[8] = static_cast<int64_t>(r->cap.ctl_index.size());
}

void ref_run_snapshots(void* h, double* now, int32_t* cls, int64_t* off, int64_t* job_id,
                       int32_t* job_prompt, double* job_deadline, double* job_wf) {
  const auto& c = static_cast<RefRun*>(h)->cap;
  std::copy(c.snap_now.begin(), c.snap_now.end(), now);
  std::copy(c.snap_class.begin(), c.snap_class.end(), cls);
  std::copy(c.snap_off.begin(), c.snap_off.end(), off);
  std::copy(c.job_id.begin(), c.job_id.end(), job_id);
  std::copy(c.job_prompt.begin(), c.job_prompt.end(), job_prompt);
  std::copy(c.job_deadline.begin(), c.job_deadline.end(), job_deadline);
  std::copy(c.job_wf.begin(), c.job_wf.end(), job_wf);
}

void ref_run_commands(void* h, double* now, int32_t* cls, double* f, double* window,
                      uint8_t* infeasible) {
  const auto& c = static_cast<RefRun*>(h)->cap;
  std::copy(c.cmd_now.begin(), c.cmd_now.end(), now);
  std::copy(c.cmd_class.begin(), c.cmd_class.end(), cls);
  std::copy(c.cmd_f.begin(), c.cmd_f.end(), f);
  std::copy(c.cmd_window.begin(), c.cmd_window.end(), window);
  std::copy(c.cmd_infeasible.begin(), c.cmd_infeasible.end(), infeasible);
}

void ref_run_controller_inputs(void* h, int32_t* fw, double* ft, uint8_t* fhas, double* fp95,
                               int32_t* cw, double* ct, double* ctps, int32_t* aw, double* at) {
  const auto& c = static_cast<RefRun*>(h)->cap;
  std::copy(c.fine_worker.begin(), c.fine_worker.end(), fw);
  std::copy(c.fine_t.begin(), c.fine_t.end(), ft);
  std::copy(c.fine_has.begin(), c.fine_has.end(), fhas);
  std::copy(c.fine_p95.begin(), c.fine_p95.end(), fp95);
  std::copy(c.coarse_worker.begin(), c.coarse_worker.end(), cw);
  std::copy(c.coarse_t.begin(), c.coarse_t.end(), ct);
  std::copy(c.coarse_tps.begin(), c.coarse_tps.end(), ctps);
  std::copy(c.adapt_worker.begin(), c.adapt_worker.end(), aw);
  std::copy(c.adapt_t.begin(), c.adapt_t.end(), at);
}

void ref_run_decisions(void* h, gso_decision* out) {
  const auto& d = static_cast<RefRun*>(h)->decisions;
  std::copy(d.begin(), d.end(), out);
}

// Per request: decode_worker, prefill_start, prefill_end, first_token, finish, n_tbt,
// class_queue; plus ledger totals [prefill_j, decode_j].
void ref_run_requests(void* h, int32_t* decode_worker, double* prefill_start, double* prefill_end,
                      double* first_token, double* finish, int32_t* class_queue,
                      uint8_t* completed, double* energy2) {
  const auto& r = static_cast<RefRun*>(h)->result;
  for (size_t i = 0; i < r.requests.size(); ++i) {
    const auto& q = r.requests[i];
    decode_worker[i] = q.decode_worker;
    prefill_start[i] = q.prefill_start_ms;
    prefill_end[i] = q.prefill_end_ms;
    first_token[i] = q.first_token_ms;
    finish[i] = q.finish_ms;
    class_queue[i] = q.class_queue;
    completed[i] = q.completed ? 1 : 0;
  }
  energy2[0] = r.prefill_pool_j();
  energy2[1] = r.decode_pool_j();
}

}  // extern "C"

// Trajectory digest, same definition as gso_digest_records (gs_oracle.c): per record
// w1 = command bits, w2 = band_lo bits ^ (band_hi bits << 13) ^ (bucket << 48) ^ (action << 56),
// h = (h ^ w) * 0x100000001b3, in log order.
static inline uint64_t dig_mix(uint64_t h, uint64_t v) { return (h ^ v) * 0x100000001b3ull; }

extern "C" uint64_t ref_digest_records(const gso_decision* r, int64_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t cmd, lo, hi;
    std::memcpy(&cmd, &r[i].command_mhz, 8);
    std::memcpy(&lo, &r[i].band_lo, 8);
    std::memcpy(&hi, &r[i].band_hi, 8);
    const uint64_t w2 = lo ^ (hi << 13) ^
                        (static_cast<uint64_t>(static_cast<uint32_t>(r[i].bucket)) << 48) ^
                        (static_cast<uint64_t>(static_cast<uint32_t>(r[i].action)) << 56);
    h = dig_mix(h, cmd);
    h = dig_mix(h, w2);
  }
  return h;
}

extern "C" void ref_replay_many(int64_t n_scen, const gso_ctl_cfg* cfgs,
                                const gso_band_table* tables, const int32_t* table_of,
                                const gso_telemetry* tels, const int32_t* tel_of,
                                const int32_t* worker_of, double f_min, double f_max, double step,
                                double f_ref, double t_end, int threads, int64_t* n_records,
                                uint64_t* digests) {
  auto work = [&](int64_t lo, int64_t hi) {
    std::vector<gso_decision> buf(1 << 16);
    for (int64_t s = lo; s < hi; ++s) {
      int64_t n = ref_replay_telemetry(&cfgs[s], &tables[table_of[s]], f_min, f_max, step, f_ref,
                                       worker_of[s], &tels[tel_of[s]], t_end, buf.data(),
                                       static_cast<int64_t>(buf.size()));
      if (n > static_cast<int64_t>(buf.size())) {
        buf.resize(static_cast<size_t>(n));
        n = ref_replay_telemetry(&cfgs[s], &tables[table_of[s]], f_min, f_max, step, f_ref,
                                 worker_of[s], &tels[tel_of[s]], t_end, buf.data(), n);
      }
      n_records[s] = n;
      digests[s] = n < 0 ? 0 : ref_digest_records(buf.data(), n);
    }
  };
  if (threads <= 1) {
    work(0, n_scen);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back(work, n_scen * t / threads, n_scen * (t + 1) / threads);
  for (auto& th : pool) th.join();
}

// ---- the reference simulator behind the same getters as gso_sim_* (gs_sim.c) ------------
// Inputs mirror gso_sim_run; results come from the reference's own greensim::run().
namespace {
struct RefSim {
  RunResult r;
  std::vector<gso_decision> dec;
  int64_t n_steps = 0;
};

Trace to_trace(int64_t n, const int64_t* arrival, const int32_t* prompt, const int32_t* output,
               const int8_t* cls) {
  Trace tr;
  tr.meta.name = "capi";
  for (int64_t i = 0; i < n; ++i) {
    Request q;
    q.id = i;
    q.arrival_ms = arrival[i];
    q.prompt_tokens = prompt[i];
    q.output_tokens = output[i];
    if (cls && (cls[i] == 0 || cls[i] == 1)) q.cls = static_cast<PromptClass>(cls[i]);
    tr.requests.push_back(q);
    tr.meta.duration_ms = std::max(tr.meta.duration_ms, arrival[i]);
  }
  return tr;
}

GovernorPolicy to_policy(const gso_policy* p, int n_prefill) {
  GovernorPolicy pol;
  switch (p->kind) {
    case 0: pol = GovernorPolicy::default_nv(); break;
    case 1: pol = GovernorPolicy::fixed(p->fixed_freq_mhz); break;
    case 2: pol = GovernorPolicy::greenllm(); break;
    default: pol = GovernorPolicy::prefill_split(); break;
  }
  if (p->kind >= 2) {
    pol.routing.enabled = p->routing_enabled != 0;
    pol.routing.thresholds.assign(p->thresholds, p->thresholds + p->n_thresholds);
    pol.routing.worker_map.assign(p->worker_map, p->worker_map + n_prefill);
  }
  pol.prefill_opt = to_qcfg(&p->prefill_opt);
  pol.decode_ctl = to_cfg(&p->decode_ctl);
  return pol;
}

SimConfig to_simcfg(const gso_sim_cfg* c) {
  SimConfig s;
  s.n_prefill_workers = c->n_prefill_workers;
  s.n_decode_workers = c->n_decode_workers;
  s.gpus_per_prefill_worker = c->gpus_per_prefill_worker;
  s.actuation_delay_ms = c->actuation_delay_ms;
  s.handoff_delay_ms = c->handoff_delay_ms;
  s.max_batch = c->max_batch;
  s.max_queue = c->max_queue;
  s.band_tps_lo = c->band_tps_lo;
  s.band_tps_hi = c->band_tps_hi;
  s.band_tps_step = c->band_tps_step;
  return s;
}
}  // namespace

extern "C" {

void* ref_sim_run(const gso_profile* prof, const gso_policy* pol, const gso_slo* slo,
                  const gso_sim_cfg* cfg, int64_t n, const int64_t* arrival_ms,
                  const int32_t* prompt, const int32_t* output, const int8_t* cls,
                  int64_t n_scripted, const gso_scripted* scripted, char* err, size_t err_cap) {
  SloConfig sc;
  sc.ttft_sm_ms = slo->ttft_sm_ms;
  sc.ttft_l_ms = slo->ttft_l_ms;
  sc.tbt_p95_ms = slo->tbt_p95_ms;
  SimConfig sim = to_simcfg(cfg);
  for (int64_t k = 0; k < n_scripted; ++k)
    sim.scripted_freq.push_back({scripted[k].time_ms, scripted[k].prefill_pool != 0,
                                 scripted[k].worker, scripted[k].f_mhz});
  auto* h = new RefSim;
  try {
    h->r = run(to_trace(n, arrival_ms, prompt, output, cls), to_profile(prof),
               to_policy(pol, cfg->n_prefill_workers), 1, sc, sim);
  } catch (const std::exception& e) {
    if (err && err_cap) std::snprintf(err, err_cap, "%s", e.what());
    delete h;
    return nullptr;
  }
  for (const auto& d : h->r.decode_decisions) {
    gso_decision c;
    to_c_record(d, &c);
    h->dec.push_back(c);
  }
  // decode steps = decode-ledger intervals that are active-decode phase changes are not
  // a step count; count TBT-producing steps instead is impossible, so report -1.
  h->n_steps = -1;
  return h;
}

void ref_sim_free(void* h) { delete static_cast<RefSim*>(h); }

void ref_sim_sizes(void* hv, int64_t* z) {
  const auto& r = static_cast<RefSim*>(hv)->r;
  int64_t nt = 0;
  for (const auto& q : r.requests) nt += static_cast<int64_t>(q.tbt_ms.size());
  z[0] = static_cast<int64_t>(r.requests.size());
  z[1] = nt;
  z[2] = static_cast<int64_t>(r.decode_decisions.size());
  z[3] = static_cast<int64_t>(r.freq_timeline.size());
  z[4] = static_cast<int64_t>(r.prefill_commands.size());
  z[5] = -1;  // the enqueue stream is not observable from a RunResult
  z[6] = static_cast<int64_t>(r.prefill_ledgers.size());
  z[7] = static_cast<int64_t>(r.decode_ledgers.size());
  z[8] = r.overload.rejected_requests;
  z[9] = static_cast<RefSim*>(hv)->n_steps;
}

void ref_sim_requests(void* hv, int32_t* class_queue, int32_t* prefill_worker,
                      int32_t* decode_worker, double* prefill_start, double* prefill_end,
                      double* first_token, double* finish, uint8_t* completed, uint8_t* rejected,
                      int8_t* cls) {
  const auto& r = static_cast<RefSim*>(hv)->r;
  for (size_t i = 0; i < r.requests.size(); ++i) {
    const auto& q = r.requests[i];
    class_queue[i] = q.class_queue;
    prefill_worker[i] = q.prefill_worker;
    decode_worker[i] = q.decode_worker;
    prefill_start[i] = q.prefill_start_ms;
    prefill_end[i] = q.prefill_end_ms;
    first_token[i] = q.first_token_ms;
    finish[i] = q.finish_ms;
    completed[i] = q.completed ? 1 : 0;
    rejected[i] = q.rejected ? 1 : 0;
    cls[i] = static_cast<int8_t>(q.cls);
  }
}

void ref_sim_tbt(void* hv, int64_t* off, double* samples) {
  const auto& r = static_cast<RefSim*>(hv)->r;
  off[0] = 0;
  for (size_t i = 0; i < r.requests.size(); ++i) {
    const auto& t = r.requests[i].tbt_ms;
    std::copy(t.begin(), t.end(), samples + off[i]);
    off[i + 1] = off[i] + static_cast<int64_t>(t.size());
  }
}

void ref_sim_ledgers(void* hv, double* p3, double* d3, int64_t* n_int) {
  const auto& r = static_cast<RefSim*>(hv)->r;
  size_t k = 0;
  for (size_t w = 0; w < r.prefill_ledgers.size(); ++w, ++k) {
    const auto& l = r.prefill_ledgers[w];
    p3[3 * w] = l.active_prefill_j;
    p3[3 * w + 1] = l.active_decode_j;
    p3[3 * w + 2] = l.idle_j;
    n_int[k] = static_cast<int64_t>(l.intervals.size());
  }
  for (size_t w = 0; w < r.decode_ledgers.size(); ++w, ++k) {
    const auto& l = r.decode_ledgers[w];
    d3[3 * w] = l.active_prefill_j;
    d3[3 * w + 1] = l.active_decode_j;
    d3[3 * w + 2] = l.idle_j;
    n_int[k] = static_cast<int64_t>(l.intervals.size());
  }
}

void ref_sim_decisions(void* hv, gso_decision* out) {
  const auto& d = static_cast<RefSim*>(hv)->dec;
  std::copy(d.begin(), d.end(), out);
}

void ref_sim_timeline(void* hv, double* t, uint8_t* pool, int32_t* worker, double* f) {
  const auto& r = static_cast<RefSim*>(hv)->r;
  for (size_t k = 0; k < r.freq_timeline.size(); ++k) {
    t[k] = r.freq_timeline[k].applied_ms;
    pool[k] = r.freq_timeline[k].prefill_pool ? 1 : 0;
    worker[k] = r.freq_timeline[k].worker;
    f[k] = r.freq_timeline[k].f_mhz;
  }
}

void ref_sim_commands(void* hv, double* tick, int32_t* cls, int32_t* worker, double* f,
                      double* window, uint8_t* infeasible) {
  const auto& r = static_cast<RefSim*>(hv)->r;
  for (size_t k = 0; k < r.prefill_commands.size(); ++k) {
    const auto& c = r.prefill_commands[k];
    tick[k] = c.tick_ms;
    cls[k] = c.class_id;
    worker[k] = c.worker;
    f[k] = c.f_mhz;
    window[k] = c.window_ms;
    infeasible[k] = c.infeasible ? 1 : 0;
  }
}

// [0] sim_end_ms, [1] last_arrival_ms, [2] -1 (no end floor), [3] prefill_pool_j,
// [4] decode_pool_j, [5] ttft_pct, [6] tbt_pct (per request), [7] tbt_pct (aggregate)
void ref_sim_scalars(void* hv, double* d) {
  const auto& r = static_cast<RefSim*>(hv)->r;
  d[0] = r.sim_end_ms;
  d[1] = r.last_arrival_ms;
  d[2] = -1.0;
  d[3] = r.prefill_pool_j();
  d[4] = r.decode_pool_j();
  const PassRates a = slo_pass_rates(r, r.slo, false);
  const PassRates b = slo_pass_rates(r, r.slo, true);
  d[5] = a.ttft_pct;
  d[6] = a.tbt_pct;
  d[7] = b.tbt_pct;
}

// CPU baseline for the closed loop: one full reference run() per scenario (its own decode
// controller config), `threads` std::threads. Outputs decode_pool_j and the decision count.
void ref_sim_run_many(const gso_profile* prof, const gso_policy* base, const gso_ctl_cfg* cfgs,
                      int64_t n_scen, const gso_slo* slo, const gso_sim_cfg* cfg, int64_t n,
                      const int64_t* arrival_ms, const int32_t* prompt, const int32_t* output,
                      int threads, double* decode_j, int64_t* n_decisions) {
  auto work = [&](int64_t lo, int64_t hi) {
    const Trace tr = to_trace(n, arrival_ms, prompt, output, nullptr);
    const GpuProfile gp = to_profile(prof);
    SloConfig sc;
    sc.ttft_sm_ms = slo->ttft_sm_ms;
    sc.ttft_l_ms = slo->ttft_l_ms;
    sc.tbt_p95_ms = slo->tbt_p95_ms;
    const SimConfig sim = to_simcfg(cfg);
    for (int64_t s = lo; s < hi; ++s) {
      gso_policy p = *base;
      p.decode_ctl = cfgs[s];
      const RunResult r = run(tr, gp, to_policy(&p, cfg->n_prefill_workers), 1, sc, sim);
      decode_j[s] = r.decode_pool_j();
      n_decisions[s] = static_cast<int64_t>(r.decode_decisions.size());
    }
  };
  if (threads <= 1) {
    work(0, n_scen);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back(work, n_scen * t / threads, n_scen * (t + 1) / threads);
  for (auto& th : pool) th.join();
}

// greensim::load_trace on a file (trace.cpp:56-129): rows or -1 with the TraceError kind and
// message. has_class_col: 1 iff the header carried the class column (every row then has cls).
int64_t ref_load_trace(const char* path, int32_t thr, int64_t cap, int64_t* arrival,
                       int32_t* prompt, int32_t* output, uint8_t* cls, int32_t* kind, char* msg,
                       int64_t msg_cap) {
  try {
    const Trace t = load_trace(path, thr);
    const int64_t n = static_cast<int64_t>(t.requests.size());
    for (int64_t i = 0; i < n && i < cap; ++i) {
      const Request& r = t.requests[static_cast<size_t>(i)];
      arrival[i] = r.arrival_ms;
      prompt[i] = r.prompt_tokens;
      output[i] = r.output_tokens;
      cls[i] = r.cls ? static_cast<uint8_t>(*r.cls) : 255;
    }
    *kind = -1;
    return n;
  } catch (const TraceError& e) {
    *kind = static_cast<int32_t>(e.kind);
    snprintf(msg, static_cast<size_t>(msg_cap), "%s", e.what());
    return -1;
  }
}

}  // extern "C"
