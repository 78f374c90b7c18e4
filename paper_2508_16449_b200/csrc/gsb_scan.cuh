// gsb_scan.cuh — K2's exhaustive clock scan (prefill_opt.cpp:16-56) for one (cell, profile),
// shared by the K2 kernels (gsb_select.cu) and the fused prefill pass (gsb_prefill.cu).
#pragma once

#include "gsb_common.cuh"

namespace gsb_k2 {

using gsb::std_max;

struct SelectParams {
  int32_t mode, C;
  double fixed_window;
  int64_t w0, window_ms;
  double margin, min_budget;
  int64_t n_cells;
};

// Specialisation for a G-clock grid whose every clock is a short divisor: the clock tables are
// KERNEL PARAMETERS (constant-bank operands, no shared-memory loads): 14 DP-pipe instructions
// per (cell, clock) and two integer sign tests (scan_clocks_c). The three division range guards
// of div_pre are hoisted to ONE per-cell test:
// with 1 <= f_i <= 4096 and TF = T*f_ref,
//   busy_i   = TF / f_i                 dividend TF
//   active_i = (P_i*busy_i) / 1000      dividend in [TF*P_min/4096*(1-u), TF*P_max]
//   idle_i   = (p_idle*(W-busy_i))/1000 dividend 0, or |.| in
//              [p_idle*min(W, TF/4096)*2^-53*(1-u), p_idle*max(W, TF)]
// (W - busy is a multiple of 2^(e-52), e the smaller exponent, hence >= min * 2^-53 unless 0;
// a zero dividend is exact on the fast path too). All of these inside [2^-900, 2^1000] keeps
// every dividend in div_pre's fast range [2^-959, 2^1023]; otherwise the cell takes IEEE '/'.
template <int G>
struct ClockConst {
  double f[G], r[G], P[G];
};

__device__ __forceinline__ bool cell_fast(double TF, double W, double p_idle, double P_min,
                                          double P_max) {
  const double lo = 0x1p-900, hi = 0x1p+1000;
  const double x_lo = TF * P_min * 0x1p-12, x_hi = TF * P_max;
  const double y_lo = p_idle * fmin(W, TF * 0x1p-12) * 0x1p-53, y_hi = p_idle * fmax(W, TF);
  return TF >= lo && TF <= hi && W >= lo && W <= hi && x_lo >= lo && x_hi <= hi && y_lo >= lo &&
         y_hi <= hi && P_min > 0.0 && p_idle > 0.0;
}

template <int G>
struct ClockSet {  // every profile of the pass, one kernel-parameter block (<= 32 KB)
  ClockConst<G> c[GSB_MAX_PROFILES];
  double f_ref[GSB_MAX_PROFILES], p_idle[GSB_MAX_PROFILES];
  double P_min[GSB_MAX_PROFILES], P_max[GSB_MAX_PROFILES];
};

// The exhaustive scan of one (cell, profile PI): returns the grid index of the choice (-1:
// nothing feasible) and its energy in *be_out.
template <int G, int PI>
__device__ __forceinline__ int scan_clocks_c(const ClockSet<G>& cs, double T, double W,
                                             double* be_out) {
  const ClockConst<G>& cc = cs.c[PI];
  const double f_ref = cs.f_ref[PI], p_idle = cs.p_idle[PI], P_min = cs.P_min[PI],
               P_max = cs.P_max[PI];
  const double TF = T * f_ref;
  int best = -1;
  double be = 0.0;
  if (cell_fast(TF, W, p_idle, P_min, P_max)) {
    // every energy is finite here (the range guard), so "nothing taken yet or E < best" is
    // exactly "E < be" with be starting at +inf
    be = INFINITY;
    // (Starting each lane's scan at its first feasible clock — busy_i is monotone — was
    // measured 6x slower: per-lane trip counts break the unrolled loop into divergent code.
    // A fully unrolled scan with constant-bank operands runs at the same rate in isolation,
    // tools/micro/k2_loop.cu, but is 26 KB of SASS per profile.)
#pragma unroll 9
    for (int i = 0; i < G; ++i) {
      const double f = cc.f[i], r = cc.r[i];
      double q = __dmul_rn(TF, r);
      double e = __fma_rn(-f, q, TF);
      const double busy = __fma_rn(r, e, q);
      const double x = __dmul_rn(cc.P[i], busy);
      q = __dmul_rn(x, gsb::kRcp1000);
      e = __fma_rn(-1000.0, q, x);
      const double active = __fma_rn(gsb::kRcp1000, e, q);
      const double wb = __dsub_rn(W, busy);
      const double y = __dmul_rn(p_idle, wb);
      q = __dmul_rn(y, gsb::kRcp1000);
      e = __fma_rn(-1000.0, q, y);
      const double idle = __fma_rn(gsb::kRcp1000, e, q);
      const double E = __dadd_rn(active, idle);
      // The two compares without DSETP (a quarter-rate FP64-pipe instruction on B200,
      // tools/micro/fp64_mix.cu): busy <= W  <=>  RN(W - busy) >= +0 (equal operands give +0),
      // a value the idle term needs anyway; E < be  <=>  RN(E - be) < 0 (finite operands: a
      // nonzero difference never rounds to zero; E - inf = -inf). Both are sign tests of a high
      // word on the integer pipe. Fast cells have P_i > 0 and p_idle > 0, so a feasible E is > 0
      // and no signed-zero case arises.
      const double d = __dsub_rn(E, be);
      const bool take = (__double2hiint(wb) >= 0) & (__double2hiint(d) < 0);
      best = take ? i : best;
      be = take ? E : be;
    }
  } else {
#pragma unroll 1
    for (int i = 0; i < G; ++i) {
      const double busy = __ddiv_rn(TF, cc.f[i]);
      const double active = __ddiv_rn(__dmul_rn(cc.P[i], busy), 1000.0);
      const double idle = __ddiv_rn(__dmul_rn(p_idle, __dsub_rn(W, busy)), 1000.0);
      const double E = __dadd_rn(active, idle);
      const bool take = (busy <= W) && (best < 0 || E < be);
      best = take ? i : best;
      be = take ? E : be;
    }
  }
  *be_out = be;
  return best;
}

// The kernel-parameter tables of every installed profile; false when a profile is not an
// 81-clock grid of short divisors in [1, 4096] MHz (the generic kernels handle those).
inline bool make_clockset81(const gsb_ctx* ctx, ClockSet<81>* cs) {
  bool all_c = true;
  for (int p = 0; p < ctx->n_profiles; ++p) {
    const gsb::ProfTab& t = ctx->h_tabs[p];
    all_c = all_c && t.G == 81 && t.all_fast && t.f_min >= 1.0 && t.f_max <= 4096.0;
  }
  if (!all_c) return false;
  for (int p = 0; p < ctx->n_profiles; ++p) {
    const gsb::ProfTab& t = ctx->h_tabs[p];
    for (int i = 0; i < 81; ++i) {
      cs->c[p].f[i] = t.f[i];
      cs->c[p].r[i] = t.rcp_f[i];
      cs->c[p].P[i] = t.P[i];
    }
    cs->f_ref[p] = t.f_ref;
    cs->p_idle[p] = t.p_idle;
    cs->P_min[p] = t.P_min;
    cs->P_max[p] = t.P_max;
  }
  return true;
}

}  // namespace gsb_k2
