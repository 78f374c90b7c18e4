// gsb_decode.cu — decode dual-loop controller path.
//   (K3a, the window statistics, lives in gsb_window.cu)
//   K4  k_band_tables    : build_band_table for many (profile, t_slo, workers, batch) tuples
//   K3b k_decode_replay  : DecodeController state machine, one lane per trajectory,
//                          sequential in time, parallel across scenarios
// The window statistics depend only on the telemetry stream (not on controller
// parameters), so K3a runs once per stream and every trajectory on that stream reads the
// same series: the CPU reference recomputes them per scenario (copy + sort per fine tick).
#include <cmath>

#include "gsb_common.cuh"
#include "gsb_ctl.cuh"

using gsb::std_clamp;
using gsb::std_max;
using gsb::std_min;

namespace {

using namespace gsbctl;

// ---------------------------------------------------------------- K4: band tables
struct BandParams {
  int64_t n_tables;
  const gsb_profile* profiles;
  const int32_t* profile_of;
  const double* t_slo;
  const int32_t* workers;
  const int32_t* max_batch;
  int n_levels;
  const double* levels;
  double *tps_lo, *tps_hi, *f_opt;
  uint8_t* feasible;
};

// decode_steady_state, decode_ctl.cpp:28-50
__device__ bool steady_tbt(const gsb_profile& p, double tps, double f, int max_batch, double* tbt) {
  const double fr = p.dec_f_ref_mhz / f;
  const double s0 = p.dec_alpha0_ms + p.dec_beta0_ms * fr;
  const double s1 = p.dec_alpha1_ms + p.dec_beta1_ms * fr;
  const double cap_tps = 1000.0 * max_batch / (s0 + s1 * max_batch);
  if (tps > cap_tps) {
    *tbt = s0 + s1 * max_batch;
    return false;
  }
  const double denom = 1000.0 - tps * s1;
  double b = denom > 0 ? tps * s0 / denom : static_cast<double>(max_batch);
  b = std_clamp(b, 1.0, static_cast<double>(max_batch));
  *tbt = s0 + s1 * b;
  return true;
}

// decode_steady_state (decode_ctl.cpp:28-50) for a batch of (tps, f, max_batch) points
__global__ void k_steady(int64_t n, const gsb_profile* __restrict__ prof, const double* __restrict__ tps,
                         const double* __restrict__ f, const int32_t* __restrict__ max_batch,
                         uint8_t* __restrict__ sust, double* __restrict__ batch, double* __restrict__ tbt) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const gsb_profile p = *prof;
  const double fr = p.dec_f_ref_mhz / f[i];
  const double s0 = p.dec_alpha0_ms + p.dec_beta0_ms * fr;
  const double s1 = p.dec_alpha1_ms + p.dec_beta1_ms * fr;
  const int mb = max_batch[i];
  const double cap_tps = 1000.0 * mb / (s0 + s1 * mb);
  if (tps[i] > cap_tps) {
    sust[i] = 0;
    batch[i] = mb;
    tbt[i] = s0 + s1 * mb;
    return;
  }
  const double denom = 1000.0 - tps[i] * s1;
  double b = denom > 0 ? tps[i] * s0 / denom : static_cast<double>(mb);
  b = std_clamp(b, 1.0, static_cast<double>(mb));
  sust[i] = 1;
  batch[i] = b;
  tbt[i] = s0 + s1 * b;
}

// build_band_table, decode_ctl.cpp:76-111: one lane per (table, level), clocks ascending,
// strict '<' on energy per token P(f)/level.
__global__ void k_band_tables(const __grid_constant__ BandParams a) {
  const int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (id >= a.n_tables * a.n_levels) return;
  const int64_t t = id / a.n_levels;
  const int i = static_cast<int>(id - t * a.n_levels);
  const gsb_profile p = a.profiles[a.profile_of[t]];
  const int n = a.n_levels;
  const double* L = a.levels;
  const int64_t o = t * n + i;
  a.tps_lo[o] = i == 0 ? 0.0 : 0.5 * (L[i - 1] + L[i]);
  a.tps_hi[o] = i + 1 < n ? 0.5 * (L[i] + L[i + 1]) : INFINITY;
  const int workers = a.workers[t], mb = a.max_batch[t];
  const double tau_w = L[i] / workers;
  const int G = static_cast<int>(rint((p.f_max_mhz - p.f_min_mhz) / p.step_mhz)) + 1;
  double best_f = 0.0, best_e = 0.0;
  bool found = false;
  for (int k = 0; k < G; ++k) {
    const double f = p.f_min_mhz + p.step_mhz * static_cast<double>(k);
    double tbt;
    if (!steady_tbt(p, tau_w, f, mb, &tbt) || tbt > a.t_slo[t]) continue;
    const double pw = ((p.k3 * f + p.k2) * f + p.k1) * f + p.k0;
    const double ept = pw / L[i];
    if (!found || ept < best_e) {
      best_f = f;
      best_e = ept;
      found = true;
    }
  }
  a.feasible[o] = found ? 1 : 0;
  a.f_opt[o] = found ? best_f : p.f_max_mhz;
}

// ---------------------------------------------------------------- K3b: controller replay
struct ReplayParams {
  gsb_replay_args a;
  int64_t n_fine, n_coarse;
};

template <bool COUNTS, bool RECORDS>
__global__ void __launch_bounds__(128, 5) k_decode_replay(const __grid_constant__ ReplayParams rp) {
  const gsb_replay_args& a = rp.a;
  const int64_t n = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (n >= a.n_traj) return;
  const gsb_ctl_cfg cfg = a.d_cfg[n];
  const int NB = a.n_buckets;
  const int64_t tb = a.d_table_of[n];
  const int64_t s = a.d_stream_of[n];
  const int worker = a.d_worker[n];
  double f_opt[GSB_MAX_BUCKETS];  // per-controller copy; adaptation mutates it (decode_ctl.hpp:132)
  for (int b = 0; b < NB; ++b) f_opt[b] = a.d_f_opt[tb * NB + b];
  gsb_decision* rec = RECORDS ? a.d_records + n * a.rec_cap : nullptr;
  const CtlK k = make_k(cfg, NB, a.d_tps_hi + tb * NB, a.f_min_mhz, a.f_max_mhz);
  Ctl<COUNTS> c;
  ctl_init(c, f_opt, k);
  const double adapt_period = cfg.adapt_period_s * 1000.0;
  const uint8_t* __restrict__ fine_has = a.d_fine_has + s * rp.n_fine;
  const double* __restrict__ fine_p95 = a.d_fine_p95 + s * rp.n_fine;
  const double* __restrict__ coarse_tps = a.d_coarse_tps + s * rp.n_coarse;

  // prefetch ring: the series value of fine tick kf+j sits in pr[j] / hr[j], so the shared
  // series' L1/L2 latency is hidden behind four ticks of controller work
  const int64_t nf = rp.n_fine;
  double pr[4];
  uint8_t hr[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    pr[j] = j < nf ? fine_p95[j] : 0.0;
    hr[j] = j < nf ? fine_has[j] : 0;
  }
  auto fine_tick = [&](int64_t kf, double now) {
    const bool has = hr[0] != 0;
    const double p95 = pr[0];
    pr[0] = pr[1];
    pr[1] = pr[2];
    pr[2] = pr[3];
    hr[0] = hr[1];
    hr[1] = hr[2];
    hr[2] = hr[3];
    const int64_t nxt = kf + 4;
    pr[3] = nxt < nf ? fine_p95[nxt] : 0.0;
    hr[3] = nxt < nf ? fine_has[nxt] : 0;
    on_fine<COUNTS, RECORDS>(c, k, has, p95, now, a.rec_cap, rec, worker);
  };

  // Tick driver (simkernel.cpp:243-248,441-464): next instant = min of the three schedules,
  // at equal times coarse (kind 5) < adapt (6) < fine (7). Generic in the tick type: when all
  // periods are whole milliseconds every accumulated instant is an exact integer, so int64
  // ticks reproduce the reference's repeated double additions exactly with ALU compares.
  auto run = [&](auto fine_p, auto coarse_p, auto adapt_p, auto t_end) {
    using TT = decltype(fine_p);
    TT tf = fine_p, tc = coarse_p, ta = adapt_p;
    int64_t kf = 0, kc = 0;
    for (;;) {
      const TT m1 = (tc < tf) ? tc : tf;
      const TT t = (ta < m1) ? ta : m1;
      if (t > t_end) break;
      const double td = static_cast<double>(t);
      if (tc == t) {
        on_coarse<COUNTS, RECORDS>(c, f_opt, k, coarse_tps[kc++], td, a.rec_cap, rec, worker);
        tc = t + coarse_p;
      }
      if (ta == t) {
        on_adapt<COUNTS, RECORDS>(c, f_opt, k, td, a.rec_cap, rec, worker);
        ta = t + adapt_p;
      }
      if (tf == t) {
        fine_tick(kf++, td);
        tf = t + fine_p;
      }
    }
  };
  // Aligned schedule: coarse and adapt periods are whole multiples of a whole-ms fine period,
  // so every coarse/adapt instant IS a fine instant (k * fine) and the merge reduces to the
  // fine ticks k = 1..nf with two down-counters; same event order (coarse, adapt, fine).
  auto run_aligned = [&](int64_t fine_p, int64_t rc, int64_t ra, int64_t nticks) {
    int64_t cc = rc, ca = ra, kc = 0;
    for (int64_t q = 1; q <= nticks; ++q) {
      const double td = RECORDS ? static_cast<double>(q * fine_p) : 0.0;
      if (--cc == 0) {
        cc = rc;
        on_coarse<COUNTS, RECORDS>(c, f_opt, k, coarse_tps[kc++], td, a.rec_cap, rec, worker);
      }
      if (--ca == 0) {
        ca = ra;
        on_adapt<COUNTS, RECORDS>(c, f_opt, k, td, a.rec_cap, rec, worker);
      }
      fine_tick(q - 1, td);
    }
  };
  auto whole_ms = [](double x) { return x >= 1.0 && x < 2147483648.0 && x == rint(x); };
  const bool int_sched = whole_ms(cfg.fine_period_ms) && whole_ms(cfg.coarse_period_ms) &&
                         whole_ms(adapt_period) && a.t_end_ms >= 0.0 &&
                         a.t_end_ms < 4503599627370496.0;
  const int64_t fi = static_cast<int64_t>(cfg.fine_period_ms);
  const int64_t ci = static_cast<int64_t>(cfg.coarse_period_ms);
  const int64_t ai = static_cast<int64_t>(adapt_period);
  if (int_sched && ci % fi == 0 && ai % fi == 0) {
    run_aligned(fi, ci / fi, ai / fi, static_cast<int64_t>(floor(a.t_end_ms)) / fi);
  } else if (int_sched) {
    run(fi, ci, ai, static_cast<int64_t>(floor(a.t_end_ms)));
  } else {
    run(cfg.fine_period_ms, cfg.coarse_period_ms, adapt_period, a.t_end_ms);
  }
  a.d_digest[n] = c.digest;
  a.d_n_rec[n] = c.n_rec;
  if (COUNTS) {
#pragma unroll
    for (int q = 0; q < 8; ++q) a.d_counts[n * 8 + q] = c.cnt[q];
  }
  if (a.d_mean_cmd) a.d_mean_cmd[n] = c.n_fine ? c.sum_cmd / static_cast<double>(c.n_fine) : 0.0;
}

// ---------------------------------------------------------------- K3s: scripted controller
// The reference's DecodeController API takes arbitrary call sequences (tests drive it with
// explicit times and values, proj/tests/test_decode_ctl.cpp). One lane per controller walks
// its script of (kind, t, value, has) calls through the same handlers as K3b.
struct ScriptParams {
  gsb_replay_args a;  // n_traj, d_cfg, d_table_of, d_worker, n_buckets, d_tps_hi, d_f_opt,
                      // f_min/f_max, d_digest, d_n_rec, d_records, rec_cap
  const int64_t* ev_off;
  const int8_t* kind;  // 0 fine, 1 coarse, 2 adapt
  const double* t;
  const double* value;
  const uint8_t* has;
  gsb_ctl_state* state;  // optional, in/out
};

__global__ void __launch_bounds__(128) k_decode_script(const __grid_constant__ ScriptParams sp) {
  const gsb_replay_args& a = sp.a;
  const int64_t n = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (n >= a.n_traj) return;
  const gsb_ctl_cfg cfg = a.d_cfg[n];
  const int NB = a.n_buckets;
  const int64_t tb = a.d_table_of[n];
  const int worker = a.d_worker[n];
  gsb_ctl_state* st = sp.state ? sp.state + n : nullptr;
  const bool resume = st && st->initialized;
  double f_opt[GSB_MAX_BUCKETS];
  for (int b = 0; b < NB; ++b) f_opt[b] = resume ? st->f_opt[b] : a.d_f_opt[tb * NB + b];
  gsb_decision* rec = a.d_records ? a.d_records + n * a.rec_cap : nullptr;
  const CtlK k = make_k(cfg, NB, a.d_tps_hi + tb * NB, a.f_min_mhz, a.f_max_mhz);
  Ctl<false> c;
  ctl_init(c, f_opt, k);
  if (resume) {
    c.lo = st->band_lo;
    c.hi = st->band_hi;
    c.sp = st->set_point;
    c.last_tps = st->last_tps;
    c.last_p95 = st->last_p95;
    c.current = st->current_bucket;
    c.pending = st->pending_bucket;
    c.consecutive = st->consecutive;
    c.adj_total = st->adj_total;
    c.adj_up = st->adj_up;
    c.adj_dn = st->adj_down;
  }
  for (int64_t e = sp.ev_off[n]; e < sp.ev_off[n + 1]; ++e) {
    const double now = sp.t[e];
    if (sp.kind[e] == 1)
      on_coarse<false, true>(c, f_opt, k, sp.value[e], now, a.rec_cap, rec, worker);
    else if (sp.kind[e] == 2)
      on_adapt<false, true>(c, f_opt, k, now, a.rec_cap, rec, worker);
    else
      on_fine<false, true>(c, k, sp.has[e] != 0, sp.value[e], now, a.rec_cap, rec, worker);
  }
  a.d_digest[n] = c.digest;
  a.d_n_rec[n] = c.n_rec;
  if (st) {
    st->band_lo = c.lo;
    st->band_hi = c.hi;
    st->set_point = c.sp;
    st->last_tps = c.last_tps;
    st->last_p95 = c.last_p95;
    st->current_bucket = c.current;
    st->pending_bucket = c.pending;
    st->consecutive = c.consecutive;
    st->adj_total = c.adj_total;
    st->adj_up = c.adj_up;
    st->adj_down = c.adj_dn;
    st->initialized = 1;
    st->pad_ = 0;
    for (int b = 0; b < NB; ++b) st->f_opt[b] = f_opt[b];
  }
}

}  // namespace

extern "C" {

int gsb_build_band_tables(gsb_ctx* ctx, int64_t n_tables, const gsb_profile* d_profiles,
                          const int32_t* d_profile_of, const double* d_t_slo_ms,
                          const int32_t* d_workers, const int32_t* d_max_batch, int n_levels,
                          const double* d_levels, double* d_tps_lo, double* d_tps_hi,
                          double* d_f_opt, uint8_t* d_feasible, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  if (n_levels < 1 || n_levels > GSB_MAX_BUCKETS)
    return gsb_set_error(ctx, GSB_MODEL_ERROR, "band table: need 1..32 TPS levels");
  if (n_tables <= 0) return GSB_OK;
  BandParams bp{n_tables, d_profiles, d_profile_of, d_t_slo_ms, d_workers, d_max_batch, n_levels,
                d_levels, d_tps_lo, d_tps_hi, d_f_opt, d_feasible};
  const int64_t n = n_tables * n_levels;
  k_band_tables<<<static_cast<unsigned>((n + 127) / 128), 128, 0, gsb_pick_stream(ctx, stream)>>>(bp);
  return gsb_check_launch(ctx, "band_tables");
}

int gsb_steady_state_batch(gsb_ctx* ctx, int64_t n, const gsb_profile* d_profile,
                           const double* d_tps, const double* d_f, const int32_t* d_max_batch,
                           uint8_t* d_sustainable, double* d_batch, double* d_tbt, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  if (n <= 0) return GSB_OK;
  k_steady<<<static_cast<unsigned>((n + 127) / 128), 128, 0, gsb_pick_stream(ctx, stream)>>>(
      n, d_profile, d_tps, d_f, d_max_batch, d_sustainable, d_batch, d_tbt);
  return gsb_check_launch(ctx, "steady_state");
}

int gsb_decode_script(gsb_ctx* ctx, const gsb_replay_args* a, const int64_t* d_ev_off,
                      const int8_t* d_kind, const double* d_t, const double* d_value,
                      const uint8_t* d_has, gsb_ctl_state* d_state, void* stream) {
  if (!ctx || !a) return GSB_INVALID_ARGUMENT;
  if (a->n_buckets < 1 || a->n_buckets > GSB_MAX_BUCKETS)
    return gsb_set_error(ctx, GSB_MODEL_ERROR, "band table: need 1..32 buckets");
  if (a->n_traj <= 0) return GSB_OK;
  ScriptParams sp{*a, d_ev_off, d_kind, d_t, d_value, d_has, d_state};
  k_decode_script<<<static_cast<unsigned>((a->n_traj + 127) / 128), 128, 0,
                    gsb_pick_stream(ctx, stream)>>>(sp);
  return gsb_check_launch(ctx, "decode_script");
}

int gsb_decode_replay(gsb_ctx* ctx, const gsb_replay_args* a, void* stream) {
  if (!ctx || !a) return GSB_INVALID_ARGUMENT;
  if (a->n_buckets < 1 || a->n_buckets > GSB_MAX_BUCKETS)
    return gsb_set_error(ctx, GSB_MODEL_ERROR, "band table: need 1..32 buckets");
  if (a->n_traj <= 0) return GSB_OK;
  ReplayParams rp{*a, gsb_n_ticks(a->fine_period_ms, a->t_end_ms),
                  gsb_n_ticks(a->coarse_period_ms, a->t_end_ms)};
  const unsigned blocks = static_cast<unsigned>((a->n_traj + 127) / 128);
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  const bool counts = a->d_counts != nullptr, records = a->d_records != nullptr && a->rec_cap > 0;
  if (counts && records)
    k_decode_replay<true, true><<<blocks, 128, 0, s>>>(rp);
  else if (counts)
    k_decode_replay<true, false><<<blocks, 128, 0, s>>>(rp);
  else if (records)
    k_decode_replay<false, true><<<blocks, 128, 0, s>>>(rp);
  else
    k_decode_replay<false, false><<<blocks, 128, 0, s>>>(rp);
  return gsb_check_launch(ctx, "decode_replay");
}

}  // extern "C"

