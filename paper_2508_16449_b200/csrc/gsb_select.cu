// gsb_select.cu — K2 (prefill window-energy objective over every (window x class x clock)
// triple + deterministic argmin), the per-class summary reductions, the ragged-batch entry
// points (select_frequency / queue_optimizer_tick / energy_total call shapes), the FP64 probe
// and the division self-test. K1 (routing and binning) lives in gsb_prefill.cu.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "gsb_common.cuh"

using gsb::ProfTab;
using gsb::std_max;
using gsb::std_min;

namespace {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- per-class summary
// Per (profile, class) reduction of a K2 pass (n_cmd, n_infeasible, n_empty, sum E, argmin
// cell). Fixed-shape tree, so bitwise identical on every run and every rank:
//   CTA (x, p) owns cells [256x, 256x+256) of profile p: slot t = cell - 256x;
//   level 1: thread (segment s < 8, class c) folds the class-c slots of [32s, 32s+32) in slot
//            order; level 2: thread c folds its 8 segments in order -> parts[p][c][x];
//   final:   k_summary_final, one warp per (p, c): lane l folds x = l, l+32, ... in order,
//            then a fixed 5-level shuffle tree.
// K2 runs levels 1-2 in its own epilogue (gsb_prefill_select_summary: the objective, argmin
// and partial reduction are one launch); gsb_prefill_summary runs the same tree from the
// stored f_idx / energy, so both give identical bytes.
constexpr int kSumCta = 256;  // (128-cell tiles measured slower: 30-32 vs 28 us, 2x partials)

struct Part {
  double sum, mn;
  long long cmd, inf, emp, arg;
};

__device__ __forceinline__ Part part_identity() { return Part{0.0, INFINITY, 0, 0, 0, -1}; }

// one cell's contribution: f_idx -2 empty, -1 infeasible (a command pinned at f_max), else a
// choice with energy e (the argmin skips non-finite energies, as a '<' scan from +inf does)
__device__ __forceinline__ Part part_of_cell(int fi, double e, long long cell) {
  Part v = part_identity();
  if (fi == -2) {
    v.emp = 1;
    return v;
  }
  v.cmd = 1;
  if (fi < 0) {
    v.inf = 1;
    return v;
  }
  v.sum = e;
  if (e < INFINITY) {
    v.mn = e;
    v.arg = cell;
  }
  return v;
}

__device__ __forceinline__ void part_combine(Part& x, const Part& y) {
  x.sum = x.sum + y.sum;
  x.cmd += y.cmd;
  x.inf += y.inf;
  x.emp += y.emp;
  if (y.arg >= 0 && (x.arg < 0 || y.mn < x.mn || (y.mn == x.mn && y.arg < x.arg))) {
    x.mn = y.mn;
    x.arg = y.arg;
  }
}

struct SumArgs {
  Part* parts;  // [P][C][gridDim.x]
};

struct SumSmem {
  Part s1[kSumCta];  // slot t's contribution
  Part s2[8 * GSB_MAX_CLASSES];
};

// Levels 1-2 of the tree for tile (x, p) once sm.s1 holds every slot's contribution (the
// caller synchronises before and after).
__device__ __forceinline__ void summary_tile(SumSmem& sm, int C, const SumArgs& sa, int x, int p,
                                             int nx) {
  const int t = threadIdx.x;
  const long long cell0 = static_cast<long long>(x) * kSumCta;
  if (t < 8 * C) {
    const int c = t % C, seg = t / C;
    const int r0 = static_cast<int>((cell0 + seg * 32) % C);
    Part a = part_identity();
    for (int j = seg * 32 + (c - r0 + C) % C; j < seg * 32 + 32; j += C) part_combine(a, sm.s1[j]);
    sm.s2[seg * C + c] = a;
  }
  __syncthreads();
  if (t < C) {
    Part a = sm.s2[t];
    for (int seg = 1; seg < 8; ++seg) part_combine(a, sm.s2[seg * C + t]);
    sa.parts[(static_cast<long long>(p) * C + t) * nx + x] = a;
  }
}

__device__ __forceinline__ Part part_shfl_down(const Part& v, int o) {
  Part r;
  r.sum = __shfl_down_sync(kFull, v.sum, o);
  r.mn = __shfl_down_sync(kFull, v.mn, o);
  r.cmd = __shfl_down_sync(kFull, v.cmd, o);
  r.inf = __shfl_down_sync(kFull, v.inf, o);
  r.emp = __shfl_down_sync(kFull, v.emp, o);
  r.arg = __shfl_down_sync(kFull, v.arg, o);
  return r;
}

// one warp per (profile, class) pc: lane l folds the partials x = l, l+32, ... in x order,
// then a fixed 5-level shuffle tree
__global__ void __launch_bounds__(32)
k_summary_final(const Part* __restrict__ parts, int nx, gsb_class_summary* __restrict__ out) {
  const int pc = blockIdx.x, lane = threadIdx.x;
  gsb::grid_dep_wait();  // the tile partials (programmatic dependent launch)
  Part a = part_identity();
  const Part* src = parts + static_cast<long long>(pc) * nx;
#pragma unroll 4
  for (int x = lane; x < nx; x += 32) part_combine(a, src[x]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Part y = part_shfl_down(a, o);
    if (lane < o) part_combine(a, y);
  }
  if (lane == 0) {
    gsb_class_summary o;
    o.n_cmd = a.cmd;
    o.n_infeasible = a.inf;
    o.n_empty = a.emp;
    o.sum_energy_j = a.sum;
    o.min_energy_j = a.mn;
    o.argmin_cell = a.arg;
    out[pc] = o;
  }
}

// gsb_prefill_summary: the same tree from stored f_idx / energy
__global__ void __launch_bounds__(kSumCta)
k_summary(int C, int64_t n_cells, const int16_t* __restrict__ f_idx,
          const double* __restrict__ energy, SumArgs sa) {
  __shared__ SumSmem sm;
  const int64_t cell = static_cast<int64_t>(blockIdx.x) * kSumCta + threadIdx.x;
  Part v = part_identity();
  if (cell < n_cells) {
    const int64_t o = static_cast<int64_t>(blockIdx.y) * n_cells + cell;
    v = part_of_cell(f_idx[o], energy[o], cell);
  }
  sm.s1[threadIdx.x] = v;
  __syncthreads();
  summary_tile(sm, C, sa, static_cast<int>(blockIdx.x), static_cast<int>(blockIdx.y),
               static_cast<int>(gridDim.x));
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

// The same ascending strict-'<' scan spread over a warp (latency path for single batches): lane
// l evaluates clocks l, l+32, ... The sequential scan's result is (a) the first feasible clock if
// its energy is NaN (nothing compares below NaN, so it sticks), else (b) the lowest-index minimum
// over the feasible non-NaN energies (later NaNs never win). Each lane tracks its first feasible
// clock and its own (b); the warp reduces both with index tie-breaks, so the outcome is the
// sequential one bit for bit. Returns the clock index (-1: none feasible) in every lane.
template <bool FAST>
__device__ __forceinline__ int argmin_clock_warp(const double* s_f, const double* s_r,
                                                 const double* s_P, int G, double TF, double W,
                                                 double p_idle, double* best_e) {
  const int lane = threadIdx.x & 31;
  int first = INT_MAX;
  double first_e = 0.0;
  int best = -1;
  double be = 0.0;
  for (int i = lane; i < G; i += 32) {
    const double f = s_f[i];
    const double busy = FAST ? gsb::div_pre_fast(TF, f, s_r[i]) : __ddiv_rn(TF, f);
    const double active = gsb::div_pre_fast(__dmul_rn(s_P[i], busy), 1000.0, gsb::kRcp1000);
    const double idle = gsb::div_pre_fast(__dmul_rn(p_idle, __dsub_rn(W, busy)), 1000.0, gsb::kRcp1000);
    const double e = __dadd_rn(active, idle);
    if (busy <= W) {
      if (first == INT_MAX) {
        first = i;
        first_e = e;
      }
      if (e == e && (best < 0 || e < be)) {
        best = i;
        be = e;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int of = __shfl_xor_sync(0xffffffffu, first, o);
    const double ofe = __shfl_xor_sync(0xffffffffu, first_e, o);
    if (of < first) {
      first = of;
      first_e = ofe;
    }
    const int ob = __shfl_xor_sync(0xffffffffu, best, o);
    const double obe = __shfl_xor_sync(0xffffffffu, be, o);
    if (ob >= 0 && (best < 0 || obe < be || (obe == be && ob < best))) {
      best = ob;
      be = obe;
    }
  }
  if (first != INT_MAX && first_e != first_e) {
    *best_e = first_e;
    return first;
  }
  *best_e = be;
  return best;
}

// W of a cell per the window mode (prefill_opt.cpp:63-67 for DEADLINE_SLACK):
// min_j(deadline_j - now) == min_deadline - now because subtraction is monotone.
__device__ __forceinline__ double cell_window(const SelectParams& sp, int64_t cell,
                                              const double* __restrict__ min_deadline,
                                              const double* __restrict__ window) {
  if (sp.mode == GSB_FIXED_WINDOW) return sp.fixed_window;
  if (sp.mode == GSB_DEADLINE_SLACK) {
    const double now = static_cast<double>((sp.w0 + cell / sp.C) * sp.window_ms);
    return std_max(sp.margin * (min_deadline[cell] - now), sp.min_budget);
  }
  return window[cell];
}

// Specialisation for a G-clock grid whose every clock is a short divisor: the clock tables are
// KERNEL PARAMETERS (constant-bank operands of the DFMA/DMUL themselves, no shared-memory loads)
// and the clock loop is fully unrolled: 15 DP-pipe instructions per (cell, clock), nothing else
// but two selects. The three division range guards of div_pre are hoisted to ONE per-cell test:
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
         y_hi <= hi;
}

template <int G>
struct ClockSet {  // every profile of the pass, one kernel-parameter block (<= 32 KB)
  ClockConst<G> c[GSB_MAX_PROFILES];
  double f_ref[GSB_MAX_PROFILES], p_idle[GSB_MAX_PROFILES];
  double P_min[GSB_MAX_PROFILES], P_max[GSB_MAX_PROFILES];
};

// cells first, first + stride, ... of profile PI; SUM: one cell (stride = n) and its summary
// contribution in *part
template <int G, int PI, bool SUM>
__device__ __forceinline__ void select_cells_c(const SelectParams& sp, const ClockSet<G>& cs,
                                               const double* __restrict__ t_ref,
                                               const uint32_t* __restrict__ count,
                                               const double* __restrict__ min_deadline,
                                               double* __restrict__ window,
                                               int16_t* __restrict__ f_idx,
                                               double* __restrict__ energy, Part* part,
                                               int64_t first, int64_t stride) {
  const ClockConst<G>& cc = cs.c[PI];
  const int p = PI;
  const double f_ref = cs.f_ref[PI], p_idle = cs.p_idle[PI], P_min = cs.P_min[PI],
               P_max = cs.P_max[PI];
  const int64_t n = sp.n_cells;
  for (int64_t cell = first; cell < n; cell += stride) {
    const int64_t o = p * n + cell;
    if (count && count[cell] == 0) {  // empty queue: no command (prefill_opt.cpp:64)
      f_idx[o] = -2;
      energy[o] = 0.0;
      if (SUM) *part = part_of_cell(-2, 0.0, cell);
      continue;
    }
    const double W = cell_window(sp, cell, min_deadline, window);
    if (p == 0 && window && sp.mode != GSB_PER_CELL_WINDOW) window[cell] = W;
    const double TF = t_ref[o] * f_ref;
    int best = -1;
    double be = 0.0;
    if (cell_fast(TF, W, p_idle, P_min, P_max)) {
      // every energy is finite here (the range guard), so "nothing taken yet or E < best"
      // is exactly "E < be" with be starting at +inf: one compare per clock
      be = INFINITY;
      // (Starting each lane's scan at its first feasible clock — busy_i is monotone — was
      // measured 6x slower: per-lane trip counts break the unrolled loop into divergent code.)
      // unrolled 9x, not 81x: the table operands become uniform constant loads, and the four
      // profile variants stay small enough for the instruction cache (a fully unrolled 81-clock
      // scan is ~26 KB of SASS per profile: 2x slower on B200 from instruction-fetch stalls,
      // even with every profile of a cell in one thread walking the variants in order)
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
        const double y = __dmul_rn(p_idle, __dsub_rn(W, busy));
        q = __dmul_rn(y, gsb::kRcp1000);
        e = __fma_rn(-1000.0, q, y);
        const double idle = __fma_rn(gsb::kRcp1000, e, q);
        const double E = __dadd_rn(active, idle);
        // (integer-pipe compares of the bit patterns were measured slower: the kernel is
        // issue-bound as much as FP64-bound, and they add instructions)
        const bool take = (busy <= W) && (E < be);
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
    f_idx[o] = static_cast<int16_t>(best);
    energy[o] = best >= 0 ? be : 0.0;
    if (SUM) *part = part_of_cell(best, be, cell);
  }
}

// blockIdx.y = profile; the switch picks an instantiation whose table offsets are constants
template <int G>
__global__ void __launch_bounds__(256)
k_prefill_select_c(const __grid_constant__ SelectParams sp, const __grid_constant__ ClockSet<G> cs,
                   const double* __restrict__ t_ref, const uint32_t* __restrict__ count,
                   const double* __restrict__ min_deadline, double* __restrict__ window,
                   int16_t* __restrict__ f_idx, double* __restrict__ energy) {
  const int64_t first = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
#define GSB_SEL(PI)                                                                             \
  select_cells_c<G, PI, false>(sp, cs, t_ref, count, min_deadline, window, f_idx, energy, nullptr, \
                               first, stride)
  switch (blockIdx.y) {
    case 0: GSB_SEL(0); break;
    case 1: GSB_SEL(1); break;
    case 2: GSB_SEL(2); break;
    default: GSB_SEL(3); break;
  }
#undef GSB_SEL
}

// (Measured and rejected: two cells per thread sharing the per-clock table loads — 47 vs 28 us,
// more code and half the busy warps; 6 CTAs/SM at 40 registers — no change.)
// K2 with the per-class summary fused: CTA (x, p) owns the 256-cell tile x of profile p. It
// compacts the tile's NON-EMPTY cells onto its first threads (ballot + warp-offset scan), so
// the 81-clock loop runs with every lane busy; warps with nothing to evaluate (and not needed
// by the summary tree) exit at once and free their slots for the next CTAs. Empty queues give
// no command (prefill_opt.cpp:64) and cost no FP64 issue slots. Each cell's result goes to its
// own slot, so the summary tree (summary_tile) is the one gsb_prefill_summary runs, bit for bit.
template <int G>
__global__ void __launch_bounds__(kSumCta, 5)
k_prefill_select_sum(const __grid_constant__ SelectParams sp, const __grid_constant__ ClockSet<G> cs,
                     const double* __restrict__ t_ref, const uint32_t* __restrict__ count,
                     const double* __restrict__ min_deadline, double* __restrict__ window,
                     int16_t* __restrict__ f_idx, double* __restrict__ energy, SumArgs sa) {
  __shared__ SumSmem sm;
  __shared__ int s_slot[kSumCta];
  __shared__ int s_wcnt[kSumCta / 32 + 1];
  const int t = threadIdx.x, lane = t & 31, wib = t >> 5;
  const int64_t n = sp.n_cells;
  const int p = static_cast<int>(blockIdx.y), x = static_cast<int>(blockIdx.x);
  const int64_t cell = static_cast<int64_t>(x) * kSumCta + t;
  gsb::grid_dep_wait();  // K1's cells (programmatic dependent launch)
  gsb::grid_dep_launch();
  const bool live = cell < n;
  const bool busy = live && (!count || count[cell] != 0);
  if (live && !busy) {  // empty queue: no command
    const int64_t o = p * n + cell;
    f_idx[o] = -2;
    energy[o] = 0.0;
  }
  sm.s1[t] = live ? part_of_cell(-2, 0.0, cell) : part_identity();
  const unsigned b = __ballot_sync(kFull, busy);
  if (lane == 0) s_wcnt[wib] = __popc(b);
  __syncthreads();
  if (t == 0) {
    int run = 0;
    for (int w = 0; w < kSumCta / 32; ++w) {
      const int c = s_wcnt[w];
      s_wcnt[w] = run;
      run += c;
    }
    s_wcnt[kSumCta / 32] = run;
  }
  __syncthreads();
  if (busy) s_slot[s_wcnt[wib] + __popc(b & ((1u << lane) - 1u))] = t;
  __syncthreads();
  const int n_busy = s_wcnt[kSumCta / 32];
  // warps past the compacted work and the summary tree's 8 x C threads leave now
  if ((wib << 5) >= max(n_busy, 8 * sp.C)) return;
  if (t < n_busy) {
    const int slot = s_slot[t];
    Part v;
#define GSB_SEL(PI)                                                                            \
  select_cells_c<G, PI, true>(sp, cs, t_ref, nullptr, min_deadline, window, f_idx, energy, &v, \
                              static_cast<int64_t>(x) * kSumCta + slot, n)
    switch (p) {
      case 0: GSB_SEL(0); break;
      case 1: GSB_SEL(1); break;
      case 2: GSB_SEL(2); break;
      default: GSB_SEL(3); break;
    }
#undef GSB_SEL
    sm.s1[slot] = v;
  }
  __syncthreads();
  summary_tile(sm, sp.C, sa, x, p, static_cast<int>(gridDim.x));
}

__global__ void __launch_bounds__(256)
k_prefill_select(const __grid_constant__ SelectParams sp, const ProfTab* __restrict__ tabs,
                 int p_base, const double* __restrict__ t_ref, const uint32_t* __restrict__ count,
                 const double* __restrict__ min_deadline, double* __restrict__ window,
                 int16_t* __restrict__ f_idx, double* __restrict__ energy) {
  __shared__ double s_f[GSB_MAX_GRID], s_r[GSB_MAX_GRID], s_P[GSB_MAX_GRID];
  __shared__ int s_fast;
  const int p = p_base + static_cast<int>(blockIdx.y);
  const ProfTab* tab = tabs + p;
  const int G = tab->G;
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    s_f[i] = tab->f[i];
    s_r[i] = tab->rcp_f[i];
    s_P[i] = tab->P[i];
  }
  if (threadIdx.x == 0) s_fast = tab->all_fast;  // every rcp_f[i] != 0, set by gsb_set_profiles
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
  if (threadIdx.x == 0) s_fast = tab->all_fast;  // every rcp_f[i] != 0, set by gsb_set_profiles
  __syncthreads();
  // one warp per batch: the queue tick and select_frequency calls are a handful of batches, so
  // latency (the 81-clock chain) matters more than lanes per batch
  const int64_t b = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const bool lead = (threadIdx.x & 31) == 0;
  if (b >= n_batches) return;  // warp-uniform
  const int64_t j0 = off[b], j1 = off[b + 1];
  if (j1 <= j0) {
    if (lead) {
      f_idx[b] = -2;
      energy[b] = 0.0;
      if (t_out) t_out[b] = 0.0;
    }
    return;
  }
  // PrefillBatch::t_ref_total_ms, prefill_opt.cpp:9-14 (every lane folds the same jobs in the
  // same order: broadcast loads, identical bits)
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
  const double TF = T * tab->f_ref;
  double be;
  const int best = s_fast ? argmin_clock_warp<true>(s_f, s_r, s_P, G, TF, W, tab->p_idle, &be)
                          : argmin_clock_warp<false>(s_f, s_r, s_P, G, TF, W, tab->p_idle, &be);
  if (lead) {
    if (window && sp.mode != GSB_PER_CELL_WINDOW) window[b] = W;
    if (t_out) t_out[b] = T;
    f_idx[b] = static_cast<int16_t>(best);
    energy[b] = best >= 0 ? be : 0.0;
  }
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

__global__ void k_energy_closed_form(const ProfTab* __restrict__ tab, int64_t n_batches,
                                     const int64_t* __restrict__ off,
                                     const int32_t* __restrict__ prompt,
                                     const double* __restrict__ wf, const double* __restrict__ f_mhz,
                                     const double* __restrict__ window, double* __restrict__ out) {
  const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (b >= n_batches) return;
  const double f = f_mhz[b];
  const double k = (f - tab->f_min) / tab->step;
  if (f < tab->f_min - 1e-9 || f > tab->f_max + 1e-9 || !(fabs(k - rint(k)) < 1e-9)) {
    out[b] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  double T = 0.0;
  for (int64_t j = off[b]; j < off[b + 1]; ++j) {
    const double L = static_cast<double>(prompt[j]);
    T = T + (wf ? wf[j] : 1.0) * ((tab->lat_a * L + tab->lat_b) * L + tab->lat_c);
  }
  const double fT = tab->f_ref * T;
  const double poly = tab->k3 * f * f + tab->k2 * f + tab->k1 + tab->k0 / f;
  const double active = fT * poly / 1000.0;
  const double idle = tab->p_idle * (window[b] - fT / f) / 1000.0;
  out[b] = active + idle;
}

}  // namespace

extern "C" {

int gsb_energy_closed_form_batches(gsb_ctx* ctx, int profile, int64_t n_batches,
                                   const int64_t* d_off, const int32_t* d_prompt,
                                   const double* d_wf, const double* d_f_mhz,
                                   const double* d_window, double* d_out, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  if (profile < 0 || profile >= ctx->n_profiles)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "energy_closed_form: bad profile index");
  if (n_batches <= 0) return GSB_OK;
  k_energy_closed_form<<<static_cast<unsigned>((n_batches + 255) / 256), 256, 0,
                         gsb_pick_stream(ctx, stream)>>>(
      static_cast<const ProfTab*>(ctx->d_tabs) + profile, n_batches, d_off, d_prompt, d_wf,
      d_f_mhz, d_window, d_out);
  return gsb_check_launch(ctx, "energy_closed_form");
}

int gsb_prefill_select_summary(gsb_ctx* ctx, const gsb_select_cfg* cfg, int64_t n_cells,
                               const double* d_t_ref, const uint32_t* d_count,
                               const double* d_min_deadline, double* d_window, int16_t* d_f_idx,
                               double* d_energy, gsb_class_summary* d_summary, void* stream) {
  if (!ctx || !cfg) return GSB_INVALID_ARGUMENT;
  if (ctx->n_profiles < 1) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select: no profiles set");
  if (cfg->mode == GSB_DEADLINE_SLACK && (!d_min_deadline || cfg->n_classes < 1 || cfg->window_ms <= 0))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select: deadline mode needs min_deadline and layout");
  if (cfg->mode == GSB_PER_CELL_WINDOW && !d_window)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select: per-cell mode needs d_window");
  if (d_summary && (cfg->n_classes < 1 || cfg->n_classes > GSB_MAX_CLASSES || n_cells % cfg->n_classes))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select: summary needs n_cells = windows x n_classes");
  if (n_cells <= 0) {
    if (d_summary)
      return gsb_prefill_summary(ctx, ctx->n_profiles, cfg->n_classes, 0, d_f_idx, d_energy,
                                 d_summary, stream);
    return GSB_OK;
  }
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
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  bool all_c = true;
  for (int p = 0; p < ctx->n_profiles; ++p) {
    const ProfTab& t = ctx->h_tabs[p];
    all_c = all_c && t.G == 81 && t.all_fast && t.f_min >= 1.0 && t.f_max <= 4096.0;
  }
  if (all_c) {
    ClockSet<81> cs{};  // filled per call (host), passed by value as the kernel parameter
    for (int p = 0; p < ctx->n_profiles; ++p) {
      const ProfTab& t = ctx->h_tabs[p];
      for (int i = 0; i < 81; ++i) {
        cs.c[p].f[i] = t.f[i];
        cs.c[p].r[i] = t.rcp_f[i];
        cs.c[p].P[i] = t.P[i];
      }
      cs.f_ref[p] = t.f_ref;
      cs.p_idle[p] = t.p_idle;
      cs.P_min[p] = t.P_min;
      cs.P_max[p] = t.P_max;
    }
    const dim3 grid(gx, static_cast<unsigned>(ctx->n_profiles));
    const int64_t tiles = want * ctx->n_profiles;
    if (d_summary && want == static_cast<int64_t>(gx)) {  // one CTA per 256-cell tile
      SumArgs sa{static_cast<Part*>(gsb_scratch(ctx, sizeof(Part) * static_cast<size_t>(tiles) *
                                                         static_cast<size_t>(cfg->n_classes)))};
      if (!sa.parts) return gsb_set_error(ctx, GSB_CUDA_ERROR, "select: scratch allocation failed");
      gsb::launch_pdl(k_prefill_select_sum<81>, grid, dim3(kSumCta), 0, s, sp, cs, d_t_ref,
                      d_count, d_min_deadline, d_window, d_f_idx, d_energy, sa);
      gsb::launch_pdl(k_summary_final, dim3(static_cast<unsigned>(ctx->n_profiles * cfg->n_classes)),
                      dim3(32), 0, s, static_cast<const Part*>(sa.parts), static_cast<int>(want),
                      d_summary);
      return gsb_check_launch(ctx, "prefill_select");
    }
    k_prefill_select_c<81><<<grid, 256, 0, s>>>(sp, cs, d_t_ref, d_count, d_min_deadline,
                                                d_window, d_f_idx, d_energy);
    const int rc = gsb_check_launch(ctx, "prefill_select");
    if (rc || !d_summary) return rc;
    return gsb_prefill_summary(ctx, ctx->n_profiles, cfg->n_classes, n_cells, d_f_idx, d_energy,
                               d_summary, stream);
  }
  for (int p = 0; p < ctx->n_profiles; ++p) {
    {
      k_prefill_select<<<dim3(gx, 1), 256, 0, s>>>(sp, static_cast<const ProfTab*>(ctx->d_tabs), p,
                                                   d_t_ref, d_count, d_min_deadline, d_window,
                                                   d_f_idx, d_energy);
    }
    const int rc = gsb_check_launch(ctx, "prefill_select");
    if (rc) return rc;
  }
  if (!d_summary) return GSB_OK;
  return gsb_prefill_summary(ctx, ctx->n_profiles, cfg->n_classes, n_cells, d_f_idx, d_energy,
                             d_summary, stream);
}

int gsb_prefill_select(gsb_ctx* ctx, const gsb_select_cfg* cfg, int64_t n_cells,
                       const double* d_t_ref, const uint32_t* d_count, const double* d_min_deadline,
                       double* d_window, int16_t* d_f_idx, double* d_energy, void* stream) {
  return gsb_prefill_select_summary(ctx, cfg, n_cells, d_t_ref, d_count, d_min_deadline, d_window,
                                    d_f_idx, d_energy, nullptr, stream);
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
  k_select_batches<<<static_cast<unsigned>((n_batches + 7) / 8), 256, 0, gsb_pick_stream(ctx, stream)>>>(
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
  if (!ctx || n_profiles < 1 || n_profiles > GSB_MAX_PROFILES || n_classes < 1 ||
      n_classes > GSB_MAX_CLASSES || n_cells < 0 || n_cells % n_classes)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "summary: bad shape");
  const int64_t gx = std::max<int64_t>(1, (n_cells + kSumCta - 1) / kSumCta);
  if (gx > 65535LL * 16) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "summary: too many cells");
  SumArgs sa{static_cast<Part*>(gsb_scratch(ctx, sizeof(Part) * static_cast<size_t>(gx) *
                                                     n_profiles * n_classes))};
  if (!sa.parts) return gsb_set_error(ctx, GSB_CUDA_ERROR, "summary: scratch allocation failed");
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  k_summary<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(n_profiles)), kSumCta, 0, s>>>(
      n_classes, n_cells, d_f_idx, d_energy, sa);
  k_summary_final<<<static_cast<unsigned>(n_profiles * n_classes), 32, 0, s>>>(
      sa.parts, static_cast<int>(gx), d_out);
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
