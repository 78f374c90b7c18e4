// gsb_ctl.cuh — the DecodeController state machine (decode_ctl.cpp:130-228) as device
// handlers shared by the open-loop replay (K3b, gsb_decode.cu) and the closed-loop decode
// pool (K5, gsb_pool.cu). One lane owns one controller.
#pragma once

#include "gsb_common.cuh"

namespace gsbctl {

using gsb::std_clamp;
using gsb::std_max;
using gsb::std_min;

// ---------------------------------------------------------------- K3b: controller replay
enum : int { A_HOLD = 0, A_UP, A_DOWN, A_CHOLD, A_CPEND, A_CCOMMIT, A_AUP, A_ADOWN };

template <bool COUNTS>
struct Ctl {
  double lo, hi, sp, last_tps, last_p95;
  int current, pending, consecutive;
  int adj_total, adj_up, adj_dn;
  uint64_t digest;
  int64_t n_rec;
  int cnt[COUNTS ? 8 : 1];
  double sum_cmd;
  int64_t n_fine;
};

__device__ __forceinline__ uint64_t mix(uint64_t h, uint64_t v) { return (h ^ v) * 0x100000001b3ull; }

// One DecisionRecord: digest (w1 = command bits, w2 = band_lo ^ band_hi << 13 ^ bucket << 48 ^
// action << 56; same definition as gso_digest_records), optional per-action counts and the
// optional full record.
template <bool COUNTS, bool RECORDS>
__device__ __forceinline__ void emit(Ctl<COUNTS>& c, int64_t rec_cap, gsb_decision* rec,
                                     int worker, double now, int bucket, int action) {
  const uint64_t w1 = static_cast<uint64_t>(__double_as_longlong(c.sp));
  const uint64_t w2 = static_cast<uint64_t>(__double_as_longlong(c.lo)) ^
                      (static_cast<uint64_t>(__double_as_longlong(c.hi)) << 13) ^
                      (static_cast<uint64_t>(static_cast<uint32_t>(bucket)) << 48) ^
                      (static_cast<uint64_t>(static_cast<uint32_t>(action)) << 56);
  c.digest = mix(mix(c.digest, w1), w2);
  if (COUNTS) {
#pragma unroll
    for (int k = 0; k < 8; ++k) c.cnt[k] += action == k ? 1 : 0;
  }
  if (RECORDS && rec && c.n_rec < rec_cap) {
    gsb_decision& r = rec[c.n_rec];
    r.tick_ms = now;
    r.tps = c.last_tps;
    r.p95_tbt_ms = c.last_p95;
    r.band_lo = c.lo;
    r.band_hi = c.hi;
    r.command_mhz = c.sp;
    r.worker = worker;
    r.bucket = bucket;
    r.action = action;
    r.pad_ = 0;
  }
  ++c.n_rec;
}

// FreqBandTable::band via DecodeController::load_band (decode_ctl.cpp:52-57, 137-142)
template <bool COUNTS>
__device__ __forceinline__ void load_band(Ctl<COUNTS>& c, const double* f_opt, int bucket,
                                          double step, double f_min, double f_max) {
  const double f = f_opt[bucket];
  c.lo = std_max(f_min, f - step);
  c.hi = std_min(f_max, f + step);
}

// smallest double > x (x finite)
__device__ __forceinline__ double next_up(double x) {
  if (x == 0.0) return 4.9406564584124654e-324;
  const long long b = __double_as_longlong(x);
  return __longlong_as_double(x > 0.0 ? b + 1 : b - 1);
}

// Fine-loop direction (decode_ctl.cpp:150-157): margin = RN(p95 / den), dir = +1 if margin > U,
// -1 if margin < L. No full division: q1 = fma(r, fma(-den, q, p95), q) with q = RN(p95 * r),
// r = RN(1/den), is always within one ulp of RN(p95/den), so the decision
// is exact unless q1 falls in [U, succ(U)] or [pred(L), L]; only then the IEEE quotient is formed.
__device__ __forceinline__ int fine_dir(double p95, double den, double r, double U, double succU,
                                        double L, double predL) {
  if (gsb::dividend_in_fast_range(p95)) {
    const double q = __dmul_rn(p95, r);
    const double e = __fma_rn(-den, q, p95);
    const double q1 = __fma_rn(r, e, q);
    if (q1 > succU) return +1;
    if (!(q1 >= U)) {
      if (q1 < predL) return -1;
      if (q1 > L) return 0;
    }
  }
  const double m = __ddiv_rn(p95, den);
  return m > U ? +1 : (m < L ? -1 : 0);
}

// Per-trajectory constants of the controller (decode_ctl.hpp:13-29 plus derived values).
struct CtlK {
  double den, rden, U, succU, L, predL, delta, step, f_min, f_max, tps_scale, bias;
  int hysteresis, NB;
  const double* tps_hi;
};

__device__ __forceinline__ CtlK make_k(const gsb_ctl_cfg& cfg, int NB, const double* tps_hi,
                                       double f_min, double f_max) {
  CtlK k;
  k.den = cfg.margin_decode * cfg.tslo_ms;
  k.rden = 1.0 / k.den;
  k.U = cfg.upper_margin;
  k.L = cfg.lower_margin;
  k.succU = next_up(k.U);
  k.predL = -next_up(-k.L);
  // dir * delta of decode_ctl.cpp:159-160 as a select: (+1)*d = d, (-1)*d = -d, 0*d = +0
  k.delta = std_min(cfg.step_mhz, cfg.max_step_mhz);
  k.step = cfg.step_mhz;
  k.f_min = f_min;
  k.f_max = f_max;
  k.tps_scale = cfg.tps_scale;
  k.bias = cfg.bias_threshold;
  k.hysteresis = cfg.hysteresis_count;
  k.NB = NB;
  k.tps_hi = tps_hi;
  return k;
}

// DecodeController ctor (decode_ctl.cpp:130-140): start in the top bucket at its f_opt
template <bool COUNTS>
__device__ __forceinline__ void ctl_init(Ctl<COUNTS>& c, const double* f_opt, const CtlK& k) {
  c.current = k.NB - 1;
  c.pending = -1;
  c.consecutive = 0;
  load_band(c, f_opt, c.current, k.step, k.f_min, k.f_max);
  c.sp = f_opt[c.current];
  c.last_tps = 0.0;
  c.last_p95 = 0.0;
  c.adj_total = c.adj_up = c.adj_dn = 0;
  c.digest = 0xcbf29ce484222325ull;
  c.n_rec = 0;
  if (COUNTS) {
#pragma unroll
    for (int q = 0; q < 8; ++q) c.cnt[q] = 0;
  }
  c.sum_cmd = 0.0;
  c.n_fine = 0;
}

// on_coarse_tick, decode_ctl.cpp:169-198
template <bool COUNTS, bool RECORDS>
__device__ __forceinline__ void on_coarse(Ctl<COUNTS>& c, double* f_opt, const CtlK& k,
                                          double worker_tps, double now,
                                          int64_t rec_cap, gsb_decision* rec, int worker) {
  c.last_tps = worker_tps * k.tps_scale;
  int observed = k.NB - 1;
  for (int b = k.NB - 1; b >= 0; --b)
    if (c.last_tps <= k.tps_hi[b]) observed = b;  // first bucket with tps <= tps_hi
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
    if (c.consecutive >= k.hysteresis) {
      c.current = observed;
      load_band(c, f_opt, c.current, k.step, k.f_min, k.f_max);
      c.sp = std_clamp(c.sp, c.lo, c.hi);
      c.pending = -1;
      c.consecutive = 0;
      c.adj_total = c.adj_up = c.adj_dn = 0;  // adjustments_.clear()
      action = A_CCOMMIT;
    } else {
      action = A_CPEND;
    }
  }
  emit<COUNTS, RECORDS>(c, rec_cap, rec, worker, now, observed, action);
}

// on_adapt_tick, decode_ctl.cpp:200-228 (adjustments_ is only read as three counts)
template <bool COUNTS, bool RECORDS>
__device__ __forceinline__ void on_adapt(Ctl<COUNTS>& c, double* f_opt, const CtlK& k, double now,
                                         int64_t rec_cap, gsb_decision* rec, int worker) {
  const int total = c.adj_total, up = c.adj_up, dn = c.adj_dn;
  c.adj_total = c.adj_up = c.adj_dn = 0;
  if (total == 0) return;
  int shift = 0;
  if (up > k.bias * total)
    shift = +1;
  else if (dn > k.bias * total)
    shift = -1;
  if (shift == 0) return;
  f_opt[c.current] = std_clamp(f_opt[c.current] + shift * k.step, k.f_min, k.f_max);
  load_band(c, f_opt, c.current, k.step, k.f_min, k.f_max);
  c.sp = std_clamp(c.sp, c.lo, c.hi);
  emit<COUNTS, RECORDS>(c, rec_cap, rec, worker, now, c.current, shift > 0 ? A_AUP : A_ADOWN);
}

// on_fine_tick, decode_ctl.cpp:148-167
template <bool COUNTS, bool RECORDS>
__device__ __forceinline__ void on_fine(Ctl<COUNTS>& c, const CtlK& k, bool has, double p95,
                                        double now, int64_t rec_cap, gsb_decision* rec,
                                        int worker) {
  int dir = 0;
  if (has) {
    c.last_p95 = p95;
    dir = fine_dir(p95, k.den, k.rden, k.U, k.succU, k.L, k.predL);
  }
  const double raw = c.sp + (dir > 0 ? k.delta : (dir < 0 ? -k.delta : 0.0));
  const double clamped = std_clamp(raw, c.lo, c.hi);
  const bool hit = dir != 0 && clamped != raw;
  c.sp = clamped;
  c.adj_total += 1;
  c.adj_up += (hit && dir > 0) ? 1 : 0;
  c.adj_dn += (hit && dir < 0) ? 1 : 0;
  c.sum_cmd = c.sum_cmd + c.sp;
  c.n_fine += 1;
  emit<COUNTS, RECORDS>(c, rec_cap, rec, worker, now, c.current, dir > 0 ? A_UP : (dir < 0 ? A_DOWN : A_HOLD));
}

}  // namespace gsbctl
