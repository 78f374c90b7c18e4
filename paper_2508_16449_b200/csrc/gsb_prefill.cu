// gsb_prefill.cu — K1 (length-class routing + window binning) and K2 (prefill window-energy
// objective over every (window x class x clock) triple + deterministic argmin).
//
// Layouts: requests are SoA in HBM (arrival i64, prompt i32),
// sorted by arrival; cells are window-major/class-minor (cell = w*C + c); per-profile cell
// arrays are [P][cells]. Every per-cell T_ref is ONE left-to-right fp64 chain in arrival
// order, exactly prefill_opt.cpp:9-14; parallelism is across cells, never inside a chain.
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cmath>

#include "gsb_common.cuh"

using gsb::ProfTab;
using gsb::std_max;
using gsb::std_min;

namespace {

struct U32ToI64 {
  __host__ __device__ int64_t operator()(uint32_t x) const { return static_cast<int64_t>(x); }
};

constexpr int kRouteThreads = 256;
constexpr int kRouteChunk = 1024;  // requests staged in shared memory per round

struct RouteParams {
  int32_t n_thr;
  int32_t thr[GSB_MAX_CLASSES - 1];
  int32_t C;
  int32_t slo_boundary;
  int32_t want_deadline;
  int64_t window_ms, w0, n_windows;
  double ttft_sm, ttft_l, allowance;
  double lat_a[GSB_MAX_PROFILES], lat_b[GSB_MAX_PROFILES], lat_c[GSB_MAX_PROFILES];
};

// ---------------------------------------------------------------- K1a: window bounds
__global__ void k_window_bounds(const int64_t* __restrict__ arrival, int64_t n, int64_t window_ms,
                                int64_t w0, int64_t n_windows, int64_t* __restrict__ bounds) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k > n_windows) return;
  const int64_t key = (w0 + k) * window_ms;
  int64_t lo = 0, hi = n;  // first index with arrival >= key
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(arrival + mid) < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  bounds[k] = lo;
}

// classify(), router.cpp:26-31: number of thresholds strictly below the prompt.
__device__ __forceinline__ int classify_dev(const RouteParams& rp, int32_t L) {
  int c = 0;
#pragma unroll
  for (int k = 0; k < GSB_MAX_CLASSES - 1; ++k) c += (k < rp.n_thr && rp.thr[k] < L) ? 1 : 0;
  return c;
}

// ---------------------------------------------------------------- K1b: route + bin
// One CTA owns WPB = 256 / C consecutive windows; thread t owns cell (window t / C, class t % C).
// The CTA streams its request range through shared memory in 1 KiB chunks: a coalesced,
// lane-parallel pass classifies each request once and computes its per-profile reference
// latency term once; then every cell thread folds its window's slice in arrival order into
// its own fp64 chain (registers), so each chain sees exactly the reference's summation order.
template <int P>
__global__ void __launch_bounds__(kRouteThreads)
k_route_bin(const __grid_constant__ RouteParams rp, const int64_t* __restrict__ arrival,
            const int32_t* __restrict__ prompt, const int64_t* __restrict__ bounds,
            uint8_t* __restrict__ cls_out, uint32_t* __restrict__ count,
            double* __restrict__ t_ref, double* __restrict__ min_deadline) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_term = reinterpret_cast<double*>(smem);            // [P][chunk]
  double* s_dl = s_term + P * kRouteChunk;                      // [chunk] (deadline mode)
  uint8_t* s_cls = reinterpret_cast<uint8_t*>(s_dl + kRouteChunk);

  const int C = rp.C;
  const int WPB = kRouteThreads / C;
  const int t = threadIdx.x;
  const int64_t wb = static_cast<int64_t>(blockIdx.x) * WPB;
  const int wl = t / C, c = t - (t / C) * C;
  const int64_t w = wb + wl;
  const bool owner = wl < WPB && w < rp.n_windows;
  const int64_t wend = min(wb + WPB, rp.n_windows);
  const int64_t rs = bounds[wb], re = bounds[wend];
  const int64_t my_s = owner ? bounds[w] : 0, my_e = owner ? bounds[w + 1] : 0;

  double acc[P];
#pragma unroll
  for (int p = 0; p < P; ++p) acc[p] = 0.0;
  uint32_t cnt = 0;
  double mdl = INFINITY;

  for (int64_t cs = rs; cs < re; cs += kRouteChunk) {
    const int64_t ce = min(cs + kRouteChunk, re);
    for (int64_t i = cs + t; i < ce; i += kRouteThreads) {
      const int32_t L = prompt[i];
      const int cl = C > 1 ? classify_dev(rp, L) : 0;
      cls_out[i] = static_cast<uint8_t>(cl);
      const int k = static_cast<int>(i - cs);
      s_cls[k] = static_cast<uint8_t>(cl);
      const double Ld = static_cast<double>(L);
#pragma unroll
      for (int p = 0; p < P; ++p) s_term[p * kRouteChunk + k] = (rp.lat_a[p] * Ld + rp.lat_b[p]) * Ld + rp.lat_c[p];
      if (rp.want_deadline) {
        // (arrival + TTFT(SM/L)) - first_token_allowance, simkernel.cpp:499-501
        const double ttft = L <= rp.slo_boundary ? rp.ttft_sm : rp.ttft_l;
        s_dl[k] = static_cast<double>(arrival[i]) + ttft - rp.allowance;
      }
    }
    __syncthreads();
    if (owner) {
      const int64_t a0 = max(my_s, cs), a1 = min(my_e, ce);
      for (int64_t i = a0; i < a1; ++i) {
        const int k = static_cast<int>(i - cs);
        if (s_cls[k] == c) {
#pragma unroll
          for (int p = 0; p < P; ++p) acc[p] = acc[p] + 1.0 * s_term[p * kRouteChunk + k];
          ++cnt;
          if (rp.want_deadline) mdl = std_min(mdl, s_dl[k]);
        }
      }
    }
    __syncthreads();
  }
  if (owner) {
    const int64_t cells = rp.n_windows * C;
    const int64_t cell = w * C + c;
    count[cell] = cnt;
#pragma unroll
    for (int p = 0; p < P; ++p) t_ref[p * cells + cell] = acc[p];
    if (rp.want_deadline && min_deadline) min_deadline[cell] = mdl;
  }
}

// ---------------------------------------------------------------- K1c: Dispatcher FIFO
__global__ void k_fifo(int32_t C, int64_t n_windows, const uint8_t* __restrict__ cls,
                       const int64_t* __restrict__ bounds, const int64_t* __restrict__ cell_off,
                       int64_t* __restrict__ fifo) {
  const int64_t cell = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (cell >= n_windows * C) return;
  const int64_t w = cell / C;
  const int c = static_cast<int>(cell - w * C);
  int64_t pos = cell_off[cell];
  for (int64_t i = bounds[w]; i < bounds[w + 1]; ++i)
    if (cls[i] == c) fifo[pos++] = i;
}

// ---------------------------------------------------------------- K2: objective + argmin
struct SelectParams {
  int32_t mode, C;
  double fixed_window;
  int64_t w0, window_ms;
  double margin, min_budget;
  int64_t n_cells;
};

// energy_total at every grid clock (prefill_opt.cpp:16-31) and the ascending strict-'<'
// argmin over feasible clocks (prefill_opt.cpp:45-56). One lane per (cell, profile); the
// clock loop runs over the profile's tables staged in shared memory (uniform broadcast
// reads). Per clock: busy = (T*f_ref)/f_i, feasible = busy <= W,
// active = (P_i*busy)/1000, idle = (p_idle*(W-busy))/1000, E = active + idle.
template <bool FAST>
__device__ __forceinline__ int argmin_clock(const double* s_f, const double* s_r, const double* s_P,
                                            int G, double TF, double W, double p_idle,
                                            double* best_e) {
  int best = -1;
  double be = 0.0;
  for (int i = 0; i < G; ++i) {
    const double f = s_f[i];
    const double busy = FAST ? gsb::div_pre_fast(TF, f, s_r[i]) : __ddiv_rn(TF, f);
    const double active = gsb::div_pre_fast(__dmul_rn(s_P[i], busy), 1000.0, gsb::kRcp1000);
    const double idle = gsb::div_pre_fast(__dmul_rn(p_idle, __dsub_rn(W, busy)), 1000.0, gsb::kRcp1000);
    const double e = __dadd_rn(active, idle);
    const bool take = (busy <= W) && (best < 0 || e < be);
#ifdef GSB_DEBUG_ARGMIN
    printf("i=%d f=%.1f busy=%a act=%a idle=%a e=%a be=%a take=%d\n", i, f, busy, active, idle, e,
           be, (int)take);
#endif
    best = take ? i : best;
    be = take ? e : be;
  }
  *best_e = be;
  return best;
}

__global__ void __launch_bounds__(256)
k_prefill_select(const __grid_constant__ SelectParams sp, const ProfTab* __restrict__ tabs,
                 const double* __restrict__ t_ref, const uint32_t* __restrict__ count,
                 const double* __restrict__ min_deadline, double* __restrict__ window,
                 int16_t* __restrict__ f_idx, double* __restrict__ energy) {
  __shared__ double s_f[GSB_MAX_GRID], s_r[GSB_MAX_GRID], s_P[GSB_MAX_GRID];
  __shared__ int s_fast;
  const int p = blockIdx.y;
  const ProfTab* tab = tabs + p;
  const int G = tab->G;
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    s_f[i] = tab->f[i];
    s_r[i] = tab->rcp_f[i];
    s_P[i] = tab->P[i];
  }
  if (threadIdx.x == 0) {
    int fast = 1;
    for (int i = 0; i < G; ++i) fast &= tab->rcp_f[i] != 0.0;
    s_fast = fast;
  }
  __syncthreads();
  const bool fast = s_fast != 0;
  const double f_ref = tab->f_ref, p_idle = tab->p_idle;
  const int64_t n = sp.n_cells;
  for (int64_t cell = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; cell < n;
       cell += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t o = p * n + cell;
    if (count && count[cell] == 0) {  // empty queue: no command (prefill_opt.cpp:64)
      f_idx[o] = -2;
      energy[o] = 0.0;
      continue;
    }
    double W;
    if (sp.mode == GSB_FIXED_WINDOW) {
      W = sp.fixed_window;
    } else if (sp.mode == GSB_DEADLINE_SLACK) {
      // min_j(deadline_j - now) == min_deadline - now (subtraction is monotone), then
      // window = std::max(margin * min_slack, min_budget), prefill_opt.cpp:65-67.
      const double now = static_cast<double>((sp.w0 + cell / sp.C) * sp.window_ms);
      W = std_max(sp.margin * (min_deadline[cell] - now), sp.min_budget);
    } else {
      W = window[cell];
    }
    if (p == 0 && window && sp.mode != GSB_PER_CELL_WINDOW) window[cell] = W;
    const double TF = t_ref[o] * f_ref;
    double be;
    const int best = fast ? argmin_clock<true>(s_f, s_r, s_P, G, TF, W, p_idle, &be)
                          : argmin_clock<false>(s_f, s_r, s_P, G, TF, W, p_idle, &be);
    f_idx[o] = static_cast<int16_t>(best);
    energy[o] = best >= 0 ? be : 0.0;
  }
}

// ---------------------------------------------------------------- ragged batches
__global__ void __launch_bounds__(256)
k_select_batches(const __grid_constant__ SelectParams sp, const ProfTab* __restrict__ tab,
                 int64_t n_batches, const int64_t* __restrict__ off,
                 const int32_t* __restrict__ prompt, const double* __restrict__ wf,
                 const double* __restrict__ deadline, const double* __restrict__ now_ms,
                 double* __restrict__ window, int16_t* __restrict__ f_idx,
                 double* __restrict__ energy, double* __restrict__ t_out) {
  __shared__ double s_f[GSB_MAX_GRID], s_r[GSB_MAX_GRID], s_P[GSB_MAX_GRID];
  __shared__ int s_fast;
  const int G = tab->G;
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    s_f[i] = tab->f[i];
    s_r[i] = tab->rcp_f[i];
    s_P[i] = tab->P[i];
  }
  if (threadIdx.x == 0) {
    int fast = 1;
    for (int i = 0; i < G; ++i) fast &= tab->rcp_f[i] != 0.0;
    s_fast = fast;
  }
  __syncthreads();
  const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (b >= n_batches) return;
  const int64_t j0 = off[b], j1 = off[b + 1];
  if (j1 <= j0) {
    f_idx[b] = -2;
    energy[b] = 0.0;
    if (t_out) t_out[b] = 0.0;
    return;
  }
  // PrefillBatch::t_ref_total_ms, prefill_opt.cpp:9-14
  double T = 0.0;
  double min_slack = INFINITY;
  const double now = (sp.mode == GSB_DEADLINE_SLACK) ? now_ms[b] : 0.0;
  for (int64_t j = j0; j < j1; ++j) {
    const double L = static_cast<double>(prompt[j]);
    const double w = wf ? wf[j] : 1.0;
    T = T + w * ((tab->lat_a * L + tab->lat_b) * L + tab->lat_c);
    if (sp.mode == GSB_DEADLINE_SLACK) min_slack = std_min(min_slack, deadline[j] - now);
  }
  double W;
  if (sp.mode == GSB_FIXED_WINDOW)
    W = sp.fixed_window;
  else if (sp.mode == GSB_DEADLINE_SLACK)
    W = std_max(sp.margin * min_slack, sp.min_budget);
  else
    W = window[b];
  if (window && sp.mode != GSB_PER_CELL_WINDOW) window[b] = W;
  if (t_out) t_out[b] = T;
  const double TF = T * tab->f_ref;
  double be;
  const int best = s_fast ? argmin_clock<true>(s_f, s_r, s_P, G, TF, W, tab->p_idle, &be)
                          : argmin_clock<false>(s_f, s_r, s_P, G, TF, W, tab->p_idle, &be);
  f_idx[b] = static_cast<int16_t>(best);
  energy[b] = best >= 0 ? be : 0.0;
}

// energy_total(batch, f, window) breakdown, prefill_opt.cpp:16-31; feasible = 2 flags the
// reference's ModelError (empty batch or off-grid clock, prefill_opt.cpp:17-18).
__global__ void k_energy_batches(const ProfTab* __restrict__ tab, int64_t n_batches,
                                 const int64_t* __restrict__ off, const int32_t* __restrict__ prompt,
                                 const double* __restrict__ wf, const double* __restrict__ f_mhz,
                                 const double* __restrict__ window, double* __restrict__ busy_out,
                                 double* __restrict__ active,
                                 double* __restrict__ idle, double* __restrict__ total,
                                 uint8_t* __restrict__ feasible) {
  const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (b >= n_batches) return;
  const double f = f_mhz[b];
  const double k = (f - tab->f_min) / tab->step;
  const bool on_grid = !(f < tab->f_min - 1e-9 || f > tab->f_max + 1e-9) && fabs(k - rint(k)) < 1e-9;
  if (off[b + 1] <= off[b] || !on_grid) {
    feasible[b] = 2;
    busy_out[b] = active[b] = idle[b] = total[b] = 0.0;
    return;
  }
  double T = 0.0;
  for (int64_t j = off[b]; j < off[b + 1]; ++j) {
    const double L = static_cast<double>(prompt[j]);
    T = T + (wf ? wf[j] : 1.0) * ((tab->lat_a * L + tab->lat_b) * L + tab->lat_c);
  }
  const double busy = T * tab->f_ref / f;                            // busy_time_ms :19
  const double W = window[b];
  busy_out[b] = busy;
  const double P = ((tab->k3 * f + tab->k2) * f + tab->k1) * f + tab->k0;  // gpu_model.hpp:64
  feasible[b] = busy <= W ? 1 : 0;
  const double a = P * busy / 1000.0;
  const double d = tab->p_idle * (W - busy) / 1000.0;
  active[b] = a;
  idle[b] = d;
  total[b] = a + d;
}

// ---------------------------------------------------------------- per-class summary
// One CTA per (profile, class): each thread folds cells w = t, t+256, ... sequentially, then a
// fixed-shape shared-memory tree combines them -> bitwise identical on every run/rank.
__global__ void __launch_bounds__(256)
k_summary(int C, int64_t n_cells, const int16_t* __restrict__ f_idx, const double* __restrict__ energy,
          gsb_class_summary* __restrict__ out) {
  __shared__ double s_sum[256], s_min[256];
  __shared__ long long s_cmd[256], s_inf[256], s_emp[256], s_arg[256];
  const int pc = blockIdx.x;
  const int p = pc / C, c = pc - (pc / C) * C;
  const int64_t n_w = n_cells / C;
  double sum = 0.0, mn = INFINITY;
  long long cmd = 0, inf = 0, emp = 0, arg = -1;
  for (int64_t w = threadIdx.x; w < n_w; w += blockDim.x) {
    const int64_t cell = w * C + c;
    const int64_t o = p * n_cells + cell;
    const int fi = f_idx[o];
    if (fi == -2) {
      ++emp;
      continue;
    }
    ++cmd;
    if (fi < 0) {
      ++inf;
      continue;
    }
    const double e = energy[o];
    sum = sum + e;
    if (e < mn) {
      mn = e;
      arg = cell;
    }
  }
  const int t = threadIdx.x;
  s_sum[t] = sum;
  s_min[t] = mn;
  s_cmd[t] = cmd;
  s_inf[t] = inf;
  s_emp[t] = emp;
  s_arg[t] = arg;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (t < s) {
      s_sum[t] = s_sum[t] + s_sum[t + s];
      s_cmd[t] += s_cmd[t + s];
      s_inf[t] += s_inf[t + s];
      s_emp[t] += s_emp[t + s];
      const double m2 = s_min[t + s];
      const long long a2 = s_arg[t + s];
      if (a2 >= 0 && (s_arg[t] < 0 || m2 < s_min[t] || (m2 == s_min[t] && a2 < s_arg[t]))) {
        s_min[t] = m2;
        s_arg[t] = a2;
      }
    }
    __syncthreads();
  }
  if (t == 0) {
    gsb_class_summary r;
    r.n_cmd = s_cmd[0];
    r.n_infeasible = s_inf[0];
    r.n_empty = s_emp[0];
    r.sum_energy_j = s_sum[0];
    r.min_energy_j = s_min[0];
    r.argmin_cell = s_arg[0];
    out[pc] = r;
  }
}

// ---------------------------------------------------------------- FP64 pipe probe
__global__ void k_fp64_probe(int iters, double* sink) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1.0, a2 = a0 + 2.0, a3 = a0 + 3.0;
  double a4 = a0 + 4.0, a5 = a0 + 5.0, a6 = a0 + 6.0, a7 = a0 + 7.0;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = __fma_rn(a0, m, c); a1 = __fma_rn(a1, m, c); a2 = __fma_rn(a2, m, c); a3 = __fma_rn(a3, m, c);
    a4 = __fma_rn(a4, m, c); a5 = __fma_rn(a5, m, c); a6 = __fma_rn(a6, m, c); a7 = __fma_rn(a7, m, c);
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) sink[0] = s;  // never true; keeps the chains alive
}

// ---------------------------------------------------------------- division self-test
__device__ __forceinline__ uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// For divisor d = (profile-0 grid clock | 1000) and random dividends (wide exponent range,
// near-midpoint quotients, tiny/zero values that exercise the guard), count results of
// div_pre that differ in any bit from IEEE __ddiv_rn.
__global__ void k_selftest_div(const ProfTab* __restrict__ tab, int64_t per_div, uint64_t seed,
                               unsigned long long* __restrict__ bad) {
  const int G = tab->G;
  const int di = blockIdx.y;  // 0..G (G == 1000.0)
  const double b = di < G ? tab->f[di] : 1000.0;
  const double r = di < G ? tab->rcp_f[di] : gsb::kRcp1000;
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < per_div;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t s = seed ^ (static_cast<uint64_t>(i) * 0x2545f4914f6cdd1dull) ^ (static_cast<uint64_t>(di) << 48);
    const uint64_t m = splitmix(s);
    const uint64_t k = splitmix(s);
    double a;
    const int kind = static_cast<int>(k & 7);
    if (kind < 4) {  // wide exponent range, random mantissa and sign
      const uint64_t e = 64 + (k >> 8) % (0x7fe - 64);
      a = __longlong_as_double(static_cast<long long>((m & ((1ull << 52) - 1)) | (e << 52) |
                                                      ((k & 8) ? (1ull << 63) : 0)));
    } else if (kind < 7) {  // a ~= b * (q + ulp(q)/2): quotient next to a rounding midpoint
      const uint64_t e = 1023 - 40 + (k >> 8) % 80;
      const double q = __longlong_as_double(static_cast<long long>((m & ((1ull << 52) - 1)) | (e << 52)));
      const double half = __longlong_as_double(static_cast<long long>((e - 53) << 52));
      a = __fma_rn(b, half, __dmul_rn(b, q));
      if (kind == 6) a = __longlong_as_double(__double_as_longlong(a) + ((k >> 20) & 3) - 1);
    } else {  // tiny, subnormal and zero dividends (guard path)
      const uint64_t e = (k >> 8) % 80;
      a = __longlong_as_double(static_cast<long long>((m & ((1ull << 52) - 1)) | (e << 52)));
    }
    const double x = gsb::div_pre(a, b, r);
    const double y = __ddiv_rn(a, b);
    local += __double_as_longlong(x) != __double_as_longlong(y) ? 1ull : 0ull;
  }
  if (local) atomicAdd(bad, local);
}

RouteParams make_route_params(gsb_ctx* ctx, const gsb_route_cfg* cfg) {
  RouteParams rp{};
  rp.n_thr = cfg->enabled ? cfg->n_thresholds : 0;
  for (int i = 0; i < GSB_MAX_CLASSES - 1; ++i) rp.thr[i] = i < cfg->n_thresholds ? cfg->thresholds[i] : 0;
  rp.C = cfg->enabled ? cfg->n_thresholds + 1 : 1;
  rp.slo_boundary = cfg->slo_boundary_tokens;
  rp.window_ms = cfg->window_ms;
  rp.w0 = cfg->w0;
  rp.n_windows = cfg->n_windows;
  rp.ttft_sm = cfg->ttft_sm_ms;
  rp.ttft_l = cfg->ttft_l_ms;
  rp.allowance = cfg->first_token_allowance_ms;
  for (int p = 0; p < ctx->n_profiles; ++p) {
    rp.lat_a[p] = ctx->profiles[p].lat_a;
    rp.lat_b[p] = ctx->profiles[p].lat_b;
    rp.lat_c[p] = ctx->profiles[p].lat_c;
  }
  return rp;
}

int check_route_cfg(gsb_ctx* ctx, const gsb_route_cfg* cfg) {
  if (!cfg || cfg->window_ms <= 0 || cfg->n_windows <= 0 || cfg->w0 < 0)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "route: bad window configuration");
  if (cfg->enabled) {
    char msg[256];
    const int rc = gsb_routing_validate(cfg, -1, nullptr, msg, sizeof msg);
    if (rc != GSB_OK) return gsb_set_error(ctx, rc, msg);
  }
  return GSB_OK;
}

}  // namespace

extern "C" {

int gsb_window_bounds(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req,
                      const int64_t* d_arrival, int64_t* d_bounds, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  int rc = check_route_cfg(ctx, cfg);
  if (rc) return rc;
  const int64_t n = cfg->n_windows + 1;
  k_window_bounds<<<static_cast<unsigned>((n + 255) / 256), 256, 0, gsb_pick_stream(ctx, stream)>>>(
      d_arrival, n_req, cfg->window_ms, cfg->w0, cfg->n_windows, d_bounds);
  return gsb_check_launch(ctx, "window_bounds");
}

int gsb_route_bin(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req, const int64_t* d_arrival,
                  const int32_t* d_prompt, const int64_t* d_bounds, uint8_t* d_class,
                  uint32_t* d_count, double* d_t_ref, double* d_min_deadline, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  int rc = check_route_cfg(ctx, cfg);
  if (rc) return rc;
  if (ctx->n_profiles < 1) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "route: no profiles set");
  (void)n_req;
  RouteParams rp = make_route_params(ctx, cfg);
  rp.want_deadline = d_min_deadline != nullptr;
  const int WPB = kRouteThreads / rp.C;
  const int64_t blocks = (cfg->n_windows + WPB - 1) / WPB;
  const size_t smem = static_cast<size_t>(ctx->n_profiles + 1) * kRouteChunk * sizeof(double) + kRouteChunk;
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  switch (ctx->n_profiles) {
#define GSB_ROUTE_CASE(P)                                                                          \
  case P:                                                                                          \
    cudaFuncSetAttribute(k_route_bin<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                         static_cast<int>(smem));                                                   \
    k_route_bin<P><<<static_cast<unsigned>(blocks), kRouteThreads, smem, s>>>(                     \
        rp, d_arrival, d_prompt, d_bounds, d_class, d_count, d_t_ref, d_min_deadline);             \
    break;
    GSB_ROUTE_CASE(1)
    GSB_ROUTE_CASE(2)
    GSB_ROUTE_CASE(3)
    GSB_ROUTE_CASE(4)
#undef GSB_ROUTE_CASE
  }
  return gsb_check_launch(ctx, "route_bin");
}

int gsb_fifo_order(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req, const uint8_t* d_class,
                   const int64_t* d_bounds, const uint32_t* d_count, int64_t* d_cell_off,
                   int64_t* d_fifo, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  int rc = check_route_cfg(ctx, cfg);
  if (rc) return rc;
  (void)n_req;
  const int C = cfg->enabled ? cfg->n_thresholds + 1 : 1;
  const int64_t cells = cfg->n_windows * C;
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  // exclusive prefix of the cell counts (u32 -> i64) with CUB
  cudaMemsetAsync(d_cell_off, 0, sizeof(int64_t), s);
  size_t tmp = 0;
  thrust::transform_iterator<U32ToI64, const uint32_t*, int64_t> in(d_count, U32ToI64{});
  cub::DeviceScan::InclusiveSum(nullptr, tmp, in, d_cell_off + 1, static_cast<int>(cells), s);
  void* d_tmp = gsb_scratch(ctx, tmp);
  if (!d_tmp) return gsb_set_error(ctx, GSB_CUDA_ERROR, "fifo: scratch allocation failed");
  cub::DeviceScan::InclusiveSum(d_tmp, tmp, in, d_cell_off + 1, static_cast<int>(cells), s);
  k_fifo<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, s>>>(C, cfg->n_windows, d_class, d_bounds,
                                                                    d_cell_off, d_fifo);
  return gsb_check_launch(ctx, "fifo_order");
}

int gsb_prefill_select(gsb_ctx* ctx, const gsb_select_cfg* cfg, int64_t n_cells,
                       const double* d_t_ref, const uint32_t* d_count, const double* d_min_deadline,
                       double* d_window, int16_t* d_f_idx, double* d_energy, void* stream) {
  if (!ctx || !cfg) return GSB_INVALID_ARGUMENT;
  if (ctx->n_profiles < 1) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select: no profiles set");
  if (cfg->mode == GSB_DEADLINE_SLACK && (!d_min_deadline || cfg->n_classes < 1 || cfg->window_ms <= 0))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select: deadline mode needs min_deadline and layout");
  if (cfg->mode == GSB_PER_CELL_WINDOW && !d_window)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select: per-cell mode needs d_window");
  if (n_cells <= 0) return GSB_OK;
  SelectParams sp{};
  sp.mode = cfg->mode;
  sp.C = cfg->n_classes;
  sp.fixed_window = cfg->fixed_window_ms;
  sp.w0 = cfg->w0;
  sp.window_ms = cfg->window_ms;
  sp.margin = cfg->qopt.margin_prefill;
  sp.min_budget = cfg->qopt.min_budget_ms;
  sp.n_cells = n_cells;
  const int64_t want = (n_cells + 255) / 256;
  const unsigned gx = static_cast<unsigned>(std::min<int64_t>(want, 65535LL * 16));
  dim3 grid(gx, static_cast<unsigned>(ctx->n_profiles));
  k_prefill_select<<<grid, 256, 0, gsb_pick_stream(ctx, stream)>>>(
      sp, static_cast<const ProfTab*>(ctx->d_tabs), d_t_ref, d_count, d_min_deadline, d_window,
      d_f_idx, d_energy);
  return gsb_check_launch(ctx, "prefill_select");
}

int gsb_select_batches(gsb_ctx* ctx, const gsb_select_cfg* cfg, int profile, int64_t n_batches,
                       const int64_t* d_off, const int32_t* d_prompt, const double* d_wf,
                       const double* d_deadline, const double* d_now, double* d_window,
                       int16_t* d_f_idx, double* d_energy, double* d_t_ref_out, void* stream) {
  if (!ctx || !cfg) return GSB_INVALID_ARGUMENT;
  if (profile < 0 || profile >= ctx->n_profiles)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select_batches: bad profile index");
  if (cfg->mode == GSB_DEADLINE_SLACK && (!d_deadline || !d_now))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select_batches: deadline mode needs deadlines and now");
  if (cfg->mode == GSB_PER_CELL_WINDOW && !d_window)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select_batches: per-batch mode needs d_window");
  if (n_batches <= 0) return GSB_OK;
  SelectParams sp{};
  sp.mode = cfg->mode;
  sp.fixed_window = cfg->fixed_window_ms;
  sp.margin = cfg->qopt.margin_prefill;
  sp.min_budget = cfg->qopt.min_budget_ms;
  sp.n_cells = n_batches;
  k_select_batches<<<static_cast<unsigned>((n_batches + 255) / 256), 256, 0, gsb_pick_stream(ctx, stream)>>>(
      sp, static_cast<const ProfTab*>(ctx->d_tabs) + profile, n_batches, d_off, d_prompt, d_wf,
      d_deadline, d_now, d_window, d_f_idx, d_energy, d_t_ref_out);
  return gsb_check_launch(ctx, "select_batches");
}

int gsb_energy_batches(gsb_ctx* ctx, int profile, int64_t n_batches, const int64_t* d_off,
                       const int32_t* d_prompt, const double* d_wf, const double* d_f_mhz,
                       const double* d_window, double* d_busy, double* d_active, double* d_idle,
                       double* d_total, uint8_t* d_feasible, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  if (profile < 0 || profile >= ctx->n_profiles)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "energy_batches: bad profile index");
  if (n_batches <= 0) return GSB_OK;
  k_energy_batches<<<static_cast<unsigned>((n_batches + 255) / 256), 256, 0, gsb_pick_stream(ctx, stream)>>>(
      static_cast<const ProfTab*>(ctx->d_tabs) + profile, n_batches, d_off, d_prompt, d_wf, d_f_mhz,
      d_window, d_busy, d_active, d_idle, d_total, d_feasible);
  return gsb_check_launch(ctx, "energy_batches");
}

int gsb_prefill_summary(gsb_ctx* ctx, int n_profiles, int n_classes, int64_t n_cells,
                        const int16_t* d_f_idx, const double* d_energy, gsb_class_summary* d_out,
                        void* stream) {
  if (!ctx || n_profiles < 1 || n_classes < 1 || n_cells % n_classes)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "summary: bad shape");
  k_summary<<<static_cast<unsigned>(n_profiles * n_classes), 256, 0, gsb_pick_stream(ctx, stream)>>>(
      n_classes, n_cells, d_f_idx, d_energy, d_out);
  return gsb_check_launch(ctx, "prefill_summary");
}

int gsb_selftest_division(gsb_ctx* ctx, int64_t per_divisor, uint64_t seed,
                          unsigned long long* d_mismatches, void* stream) {
  if (!ctx || ctx->n_profiles < 1) return GSB_INVALID_ARGUMENT;
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  cudaMemsetAsync(d_mismatches, 0, sizeof(unsigned long long), s);
  const ProfTab* tab = static_cast<const ProfTab*>(ctx->d_tabs);
  const gsb_profile& p0 = ctx->profiles[0];
  const int G = static_cast<int>(std::round((p0.f_max_mhz - p0.f_min_mhz) / p0.step_mhz)) + 1;
  const dim3 grid(static_cast<unsigned>(std::min<int64_t>((per_divisor + 255) / 256, 1024)),
                  static_cast<unsigned>(G + 1));
  k_selftest_div<<<grid, 256, 0, s>>>(tab, per_divisor, seed, d_mismatches);
  return gsb_check_launch(ctx, "selftest_division");
}

int gsb_fp64_probe(gsb_ctx* ctx, int64_t n_threads, int iters, double* d_sink, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  k_fp64_probe<<<static_cast<unsigned>((n_threads + 255) / 256), 256, 0, gsb_pick_stream(ctx, stream)>>>(iters, d_sink);
  return gsb_check_launch(ctx, "fp64_probe");
}

}  // extern "C"
