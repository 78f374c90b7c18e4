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

using gsb::std_clamp;
using gsb::std_max;
using gsb::std_min;

namespace {

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
enum : int { A_HOLD = 0, A_UP, A_DOWN, A_CHOLD, A_CPEND, A_CCOMMIT, A_AUP, A_ADOWN };

struct Ctl {
  double lo, hi, sp, last_tps, last_p95;
  int current, pending, consecutive;
  int adj_total, adj_up, adj_dn;
  uint64_t digest;
  int64_t n_rec;
  int cnt[8];
  double sum_cmd;
  int64_t n_fine;
};

__device__ __forceinline__ uint64_t mix(uint64_t h, uint64_t v) { return (h ^ v) * 0x100000001b3ull; }

struct ReplayCtx {
  const gsb_replay_args* a;
  int64_t n;
  int worker;
  gsb_decision* rec;  // this trajectory's record slab or nullptr
};

__device__ __forceinline__ void emit(Ctl& c, const ReplayCtx& rc, double now, int bucket, int action) {
  c.digest = mix(c.digest, static_cast<uint64_t>(__double_as_longlong(c.sp)));
  c.digest = mix(c.digest, static_cast<uint64_t>(__double_as_longlong(c.lo)));
  c.digest = mix(c.digest, static_cast<uint64_t>(__double_as_longlong(c.hi)));
  c.digest = mix(c.digest, static_cast<uint64_t>(static_cast<uint32_t>(action)) |
                               (static_cast<uint64_t>(static_cast<uint32_t>(bucket)) << 32));
#pragma unroll
  for (int k = 0; k < 8; ++k) c.cnt[k] += action == k ? 1 : 0;
  if (rc.rec && c.n_rec < rc.a->rec_cap) {
    gsb_decision& r = rc.rec[c.n_rec];
    r.tick_ms = now;
    r.tps = c.last_tps;
    r.p95_tbt_ms = c.last_p95;
    r.band_lo = c.lo;
    r.band_hi = c.hi;
    r.command_mhz = c.sp;
    r.worker = rc.worker;
    r.bucket = bucket;
    r.action = action;
    r.pad_ = 0;
  }
  ++c.n_rec;
}

struct ReplayParams {
  gsb_replay_args a;
  int64_t n_fine, n_coarse;
};

// FreqBandTable::band via DecodeController::load_band (decode_ctl.cpp:52-57, 137-142)
__device__ __forceinline__ void load_band(Ctl& c, const double* f_opt, int bucket, double step,
                                          double f_min, double f_max) {
  const double f = f_opt[bucket];
  c.lo = std_max(f_min, f - step);
  c.hi = std_min(f_max, f + step);
}

__global__ void __launch_bounds__(128) k_decode_replay(const __grid_constant__ ReplayParams rp) {
  const gsb_replay_args& a = rp.a;
  const int64_t n = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (n >= a.n_traj) return;
  const gsb_ctl_cfg cfg = a.d_cfg[n];
  const int NB = a.n_buckets;
  const int64_t tb = a.d_table_of[n];
  const int64_t s = a.d_stream_of[n];
  const double* tps_hi = a.d_tps_hi + tb * NB;
  double f_opt[GSB_MAX_BUCKETS];  // per-controller copy; adaptation mutates it (decode_ctl.hpp:132)
  for (int b = 0; b < NB; ++b) f_opt[b] = a.d_f_opt[tb * NB + b];
  const ReplayCtx rc{&a, n, a.d_worker[n], a.d_records ? a.d_records + n * a.rec_cap : nullptr};
  const double f_min = a.f_min_mhz, f_max = a.f_max_mhz, step = cfg.step_mhz;

  // DecodeController ctor (decode_ctl.cpp:130-140): start in the top bucket at its f_opt
  Ctl c;
  c.current = NB - 1;
  c.pending = -1;
  c.consecutive = 0;
  load_band(c, f_opt, c.current, step, f_min, f_max);
  c.sp = f_opt[c.current];
  c.last_tps = 0.0;
  c.last_p95 = 0.0;
  c.adj_total = c.adj_up = c.adj_dn = 0;
  c.digest = 0xcbf29ce484222325ull;
  c.n_rec = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) c.cnt[k] = 0;
  c.sum_cmd = 0.0;
  c.n_fine = 0;

  const double den = cfg.margin_decode * cfg.tslo_ms;
  const double rden = gsb::short_divisor_dev(den) ? 1.0 / den : 0.0;
  const double delta = std_min(cfg.step_mhz, cfg.max_step_mhz);
  const double adapt_period = cfg.adapt_period_s * 1000.0;
  const uint8_t* __restrict__ fine_has = a.d_fine_has + s * rp.n_fine;
  const double* __restrict__ fine_p95 = a.d_fine_p95 + s * rp.n_fine;
  const double* __restrict__ coarse_tps = a.d_coarse_tps + s * rp.n_coarse;

  double tf = cfg.fine_period_ms, tc = cfg.coarse_period_ms, ta = adapt_period;
  int64_t kf = 0, kc = 0;
  for (;;) {
    const double t = std_min(tf, std_min(tc, ta));
    if (t > a.t_end_ms) break;
    if (tc == t) {
      // on_coarse_tick, decode_ctl.cpp:169-198
      c.last_tps = coarse_tps[kc++] * cfg.tps_scale;
      int observed = NB - 1;
      for (int b = NB - 1; b >= 0; --b)
        if (c.last_tps <= tps_hi[b]) observed = b;  // first bucket with tps <= tps_hi
      int action;
      if (observed == c.current) {
        c.pending = -1;
        c.consecutive = 0;
        action = A_CHOLD;
      } else {
        if (observed == c.pending) {
          ++c.consecutive;
        } else {
          c.pending = observed;
          c.consecutive = 1;
        }
        if (c.consecutive >= cfg.hysteresis_count) {
          c.current = observed;
          load_band(c, f_opt, c.current, step, f_min, f_max);
          c.sp = std_clamp(c.sp, c.lo, c.hi);
          c.pending = -1;
          c.consecutive = 0;
          c.adj_total = c.adj_up = c.adj_dn = 0;  // adjustments_.clear()
          action = A_CCOMMIT;
        } else {
          action = A_CPEND;
        }
      }
      emit(c, rc, t, observed, action);
      tc = t + cfg.coarse_period_ms;
    }
    if (ta == t) {
      // on_adapt_tick, decode_ctl.cpp:200-228
      const int total = c.adj_total, up = c.adj_up, dn = c.adj_dn;
      c.adj_total = c.adj_up = c.adj_dn = 0;
      if (total != 0) {
        int shift = 0;
        if (up > cfg.bias_threshold * total)
          shift = +1;
        else if (dn > cfg.bias_threshold * total)
          shift = -1;
        if (shift != 0) {
          f_opt[c.current] = std_clamp(f_opt[c.current] + shift * step, f_min, f_max);
          load_band(c, f_opt, c.current, step, f_min, f_max);
          c.sp = std_clamp(c.sp, c.lo, c.hi);
          emit(c, rc, t, c.current, shift > 0 ? A_AUP : A_ADOWN);
        }
      }
      ta = t + adapt_period;
    }
    if (tf == t) {
      // on_fine_tick, decode_ctl.cpp:148-167
      int dir = 0;
      if (fine_has[kf]) {
        const double p95 = fine_p95[kf];
        c.last_p95 = p95;
        const double margin = rden != 0.0 ? gsb::div_pre_fast(p95, den, rden) : __ddiv_rn(p95, den);
        if (margin > cfg.upper_margin)
          dir = +1;
        else if (margin < cfg.lower_margin)
          dir = -1;
      }
      ++kf;
      const double raw = c.sp + dir * delta;
      const double clamped = std_clamp(raw, c.lo, c.hi);
      const bool hit = dir != 0 && clamped != raw;
      c.sp = clamped;
      c.adj_total += 1;
      c.adj_up += (hit && dir > 0) ? 1 : 0;
      c.adj_dn += (hit && dir < 0) ? 1 : 0;
      c.sum_cmd = c.sum_cmd + c.sp;
      c.n_fine += 1;
      emit(c, rc, t, c.current, dir > 0 ? A_UP : (dir < 0 ? A_DOWN : A_HOLD));
      tf = t + cfg.fine_period_ms;
    }
  }
  a.d_digest[n] = c.digest;
  a.d_n_rec[n] = c.n_rec;
  if (a.d_counts) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a.d_counts[n * 8 + k] = c.cnt[k];
  }
  if (a.d_mean_cmd) a.d_mean_cmd[n] = c.n_fine ? c.sum_cmd / static_cast<double>(c.n_fine) : 0.0;
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

int gsb_decode_replay(gsb_ctx* ctx, const gsb_replay_args* a, void* stream) {
  if (!ctx || !a) return GSB_INVALID_ARGUMENT;
  if (a->n_buckets < 1 || a->n_buckets > GSB_MAX_BUCKETS)
    return gsb_set_error(ctx, GSB_MODEL_ERROR, "band table: need 1..32 buckets");
  if (a->n_traj <= 0) return GSB_OK;
  ReplayParams rp{*a, gsb_n_ticks(a->fine_period_ms, a->t_end_ms),
                  gsb_n_ticks(a->coarse_period_ms, a->t_end_ms)};
  k_decode_replay<<<static_cast<unsigned>((a->n_traj + 127) / 128), 128, 0, gsb_pick_stream(ctx, stream)>>>(rp);
  return gsb_check_launch(ctx, "decode_replay");
}

}  // extern "C"

