// gsb_select.cu — K2 (prefill window-energy objective over every (window x class x clock)
// triple + deterministic argmin), the per-class summary reductions, the ragged-batch entry
// points (select_frequency / queue_optimizer_tick / energy_total call shapes), the FP64 probe
// and the division self-test. K1 (routing and binning) lives in gsb_prefill.cu.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "gsb_common.cuh"
#include "gsb_scan.cuh"

using gsb::ProfTab;
using gsb::std_max;
using gsb::std_min;

namespace {

using gsb_k2::SelectParams;
using gsb_k2::ClockConst;
using gsb_k2::ClockSet;
using gsb_k2::cell_fast;
using gsb_k2::scan_clocks_c;

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- per-class summary
// Per (profile, class) reduction of a K2 pass (n_cmd, n_infeasible, n_empty, sum E, argmin
// cell); the fixed-shape tree is described at k_cells_finish.
// The argmin travels as an order-preserving 64-bit key of the energy (negative: all bits
// flipped, else the sign bit set), so combining two parts compares integers on the ALU pipe
// instead of issuing quarter-rate DSETPs on the FP64 pipe K2 is bound by.
__device__ __forceinline__ unsigned long long e_key(double x) {
  unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
  if ((u << 1) == 0) u = 0;  // -0 == +0, as the double compare has it
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double e_unkey(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(u));
}
constexpr unsigned long long kKeyInf = 0xfff0000000000000ull;  // e_key(+inf)

struct alignas(16) Part {  // 32 bytes: two 16-byte loads
  double sum;
  unsigned long long mnk;  // e_key of the minimum energy (kKeyInf: none)
  long long arg;           // its cell (lowest on ties), -1: none
  int cmd, inf;
};

__device__ __forceinline__ Part part_identity() { return Part{0.0, kKeyInf, -1, 0, 0}; }

// one non-empty cell's contribution: f_idx -1 infeasible (a command pinned at f_max), else a
// choice with energy e (the argmin skips non-finite energies, as a '<' scan from +inf does);
// empty cells are not listed (n_empty = windows - commands)
__device__ __forceinline__ Part part_of_cell(int fi, double e, long long cell) {
  Part v = part_identity();
  if (fi == -2) return v;
  v.cmd = 1;
  if (fi < 0) {
    v.inf = 1;
    return v;
  }
  v.sum = e;
  if (e < INFINITY) {
    v.mnk = e_key(e);
    v.arg = cell;
  }
  return v;
}

__device__ __forceinline__ void part_combine(Part& x, const Part& y) {
  x.sum = x.sum + y.sum;
  x.cmd += y.cmd;
  x.inf += y.inf;
  if (y.arg >= 0 && (x.arg < 0 || y.mnk < x.mnk || (y.mnk == x.mnk && y.arg < x.arg))) {
    x.mnk = y.mnk;
    x.arg = y.arg;
  }
}

// ---------------------------------------------------------------- K2: objective + argmin
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

// cells first, first + stride, ... of profile PI
template <int G, int PI>
__device__ __forceinline__ void select_cells_c(const SelectParams& sp, const ClockSet<G>& cs,
                                               const double* __restrict__ t_ref,
                                               const uint32_t* __restrict__ count,
                                               const double* __restrict__ min_deadline,
                                               double* __restrict__ window,
                                               int16_t* __restrict__ f_idx,
                                               double* __restrict__ energy, int64_t first,
                                               int64_t stride) {
  const int p = PI;
  const int64_t n = sp.n_cells;
  for (int64_t cell = first; cell < n; cell += stride) {
    const int64_t o = p * n + cell;
    if (count && count[cell] == 0) {  // empty queue: no command (prefill_opt.cpp:64)
      f_idx[o] = -2;
      energy[o] = 0.0;
      continue;
    }
    const double W = cell_window(sp, cell, min_deadline, window);
    if (p == 0 && window && sp.mode != GSB_PER_CELL_WINDOW) window[cell] = W;
    double be;
    const int best = scan_clocks_c<G, PI>(cs, t_ref[o], W, &be);
    f_idx[o] = static_cast<int16_t>(best);
    energy[o] = best >= 0 ? be : 0.0;
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
  select_cells_c<G, PI>(sp, cs, t_ref, count, min_deadline, window, f_idx, energy, first, stride)
  switch (blockIdx.y) {
    case 0: GSB_SEL(0); break;
    case 1: GSB_SEL(1); break;
    case 2: GSB_SEL(2); break;
    default: GSB_SEL(3); break;
  }
#undef GSB_SEL
}

// (Measured and rejected: two cells per thread sharing the per-clock table loads — 47 vs 28 us,
// more code and half the busy warps; 6 CTAs/SM at 40 registers — no change; round 1's per-tile
// compaction of 256-cell tiles: 1.7 waves of ragged warps, replaced by the global list below.)

// ---------------------------------------------------------------- non-empty cell lists
// K2 evaluates only non-empty (cell, profile) pairs (an empty queue gives no command,
// prefill_opt.cpp:64). Compacting the non-empty cells into ONE ascending list lets K2 run as a
// single wave of fully populated warps (one lane per (listed cell, profile)) instead of
// per-tile compaction with ragged warps and a 1.7-wave tail.
//
// k_compact: one pass with decoupled look-back. A CTA takes the next 2048-item tile by ticket
// (so every tile it waits on belongs to a CTA that is already running), publishes its count,
// and its first warp sums its predecessors' published counts 32 tiles at a time until it
// reaches a published inclusive prefix. Status word: launch epoch (24 bits) | flag (2 bits:
// 1 = tile count, 2 = inclusive prefix) | value (38 bits). The epoch advances once per launch
// (the last CTA to finish bumps it and rewinds the ticket counters), so no reset pass is
// needed and a captured graph can replay the kernel.
constexpr int kCompactThreads = 256, kCompactItems = 8;
constexpr int kCompactTile = kCompactThreads * kCompactItems;

using gsb::CompactHdr;

struct NonEmptyCount {  // K1's queue sizes: non-empty iff count != 0
  const uint32_t* p;
  __device__ __forceinline__ unsigned mask8(int64_t i0, int64_t n) const {
    unsigned m = 0;
    if (i0 + 8 <= n && (reinterpret_cast<uintptr_t>(p + i0) & 15) == 0) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(p + i0));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(p + i0) + 1);
      m = (a.x != 0) | (a.y != 0) << 1 | (a.z != 0) << 2 | (a.w != 0) << 3 | (b.x != 0) << 4 |
          (b.y != 0) << 5 | (b.z != 0) << 6 | (b.w != 0) << 7;
    } else {
      for (int j = 0; j < 8; ++j)
        if (i0 + j < n && p[i0 + j] != 0) m |= 1u << j;
    }
    return m;
  }
};

template <class Src>
__global__ void __launch_bounds__(kCompactThreads)
k_compact(Src src, int64_t n, CompactHdr* __restrict__ hdr,
          unsigned long long* __restrict__ status, uint32_t* __restrict__ list,
          int64_t* __restrict__ n_list) {
  __shared__ unsigned s_tile, s_epoch;
  __shared__ int s_warp[kCompactThreads / 32];
  __shared__ long long s_excl;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  gsb::grid_dep_wait();  // the producer of src (K1) has finished
  gsb::grid_dep_launch();
  if (t == 0) {
    s_epoch = *reinterpret_cast<volatile unsigned*>(&hdr->epoch);
    s_tile = atomicAdd(&hdr->ticket, 1u);
  }
  __syncthreads();
  const unsigned tile = s_tile, ep = s_epoch & 0xffffffu;
  const unsigned n_tiles = static_cast<unsigned>((n + kCompactTile - 1) / kCompactTile);
  const int64_t i0 = static_cast<int64_t>(tile) * kCompactTile + t * kCompactItems;
  const unsigned m = src.mask8(i0, n);
  const int c = __popc(m);
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  int wbase = 0, agg = 0;
#pragma unroll
  for (int k = 0; k < kCompactThreads / 32; ++k) {
    wbase += k < w ? s_warp[k] : 0;
    agg += s_warp[k];
  }
  if (w == 0) {
    const long long excl = gsb::lookback_prefix(status, tile, ep, agg);
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  int64_t pos = s_excl + wbase + incl - c;
  for (unsigned mm = m; mm; mm &= mm - 1) list[pos++] = static_cast<uint32_t>(i0 + __ffs(mm) - 1);
  if (t == 0 && tile == n_tiles - 1) {
    *n_list = s_excl + agg;
    gsb::lookback_finish(hdr, s_epoch);
  }
}

// ---------------------------------------------------------------- per-class summary tree
// The per-(profile, class) summary of a pass, over the DENSE cell array (cell = w*C + c, so the
// class-c cells are every C-th cell: no list, no per-class routing). Fixed shape, hence bitwise
// identical on every run and rank, whichever entry point runs it:
//   level 1  CTA (x, p) owns cells [x*T*K, (x+1)*T*K) with T = 32*C threads: thread t folds
//            cells base + t + k*T, k = 0..K-1 (class t % C, windows in order); the same kernel
//            writes the empty cells' "no command" outputs (-2, 0) when it is given the counts
//   level 2  class c: slot j = t / C (0..31); (c, s) folds slots [8s, 8s+8) in order, then
//            (s0 + s1) + (s2 + s3)                                          -> block part
//   final    k_summary_final (one CTA per (profile, class)): thread q folds block parts q,
//            q + 256, ... in order, then a fixed 256-wide tree
// Empty cells only count (n_empty = windows - commands). Round 1's per-tile tree (and a list-
// ordered one measured this round: ~15 extra instructions per cell inside the FP64-bound K2,
// 4 us) are replaced by this memory-bound pass over 10 B per (cell, profile).
constexpr int kSumK = 4;        // cells per thread in level 1
constexpr int kFinalCta = 256;

__device__ __forceinline__ Part part_shfl_down_w(const Part& v, int o, int width) {
  Part r;
  r.sum = __shfl_down_sync(kFull, v.sum, o, width);
  r.mnk = __shfl_down_sync(kFull, v.mnk, o, width);
  r.cmd = __shfl_down_sync(kFull, v.cmd, o, width);
  r.inf = __shfl_down_sync(kFull, v.inf, o, width);
  r.arg = __shfl_down_sync(kFull, v.arg, o, width);
  return r;
}

__device__ __forceinline__ Part ld_part_cg(const Part* p) {  // L2 (written by other CTAs)
  const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
  const longlong2 b = __ldcg(reinterpret_cast<const longlong2*>(p) + 1);
  Part r;
  r.sum = a.x;
  r.mnk = static_cast<unsigned long long>(__double_as_longlong(a.y));
  r.arg = b.x;
  r.cmd = static_cast<int>(b.y & 0xffffffffll);
  r.inf = static_cast<int>(b.y >> 32);
  return r;
}

// Level 1 + 2 (and the empty-cell fill): grid (X, P), 32*C threads. count != NULL: cells with
// count 0 get f_idx -2 / energy 0 (K2 evaluates only the listed, non-empty cells); else the
// emptiness is read from f_idx (gsb_prefill_summary over stored results). parts == NULL: fill only.
template <int C>
__global__ void __launch_bounds__(32 * C)
k_cells_finish(int64_t n_cells, const uint32_t* __restrict__ count, int16_t* __restrict__ f_idx,
               double* __restrict__ energy, Part* __restrict__ parts, int64_t n_blocks,
               int early_fill) {
  constexpr int T = 32 * C;
  __shared__ Part sl[32][C];
  __shared__ Part s2[4][C];
  const int t = threadIdx.x, p = blockIdx.y;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * T * kSumK;
  int16_t* fi = f_idx + p * n_cells;
  double* en = energy + p * n_cells;
  // The empty cells' outputs need only K1's counts. early_fill: those were complete before K2
  // started (K2 waits on K1 before it lets this grid launch), so they are written BEFORE the
  // dependency wait and a programmatic launch overlaps them with K2's tail (K2 writes only the
  // listed cells). The fused pass produces the counts in the primary kernel itself: no early fill.
  if (!early_fill) gsb::grid_dep_wait();
  uint32_t cnt[kSumK];
#pragma unroll
  for (int k = 0; k < kSumK; ++k) {
    const int64_t cell = base + t + k * T;
    cnt[k] = (count && cell < n_cells) ? __ldg(count + cell) : 1u;
  }
#pragma unroll
  for (int k = 0; k < kSumK; ++k) {
    const int64_t cell = base + t + k * T;
    if (cell < n_cells && cnt[k] == 0) {  // empty queue: no command (prefill_opt.cpp:64)
      fi[cell] = -2;
      en[cell] = 0.0;
    }
  }
  gsb::grid_dep_launch();
  gsb::grid_dep_wait();  // K2's results (also keeps this grid ordered after K2 when fill-only)
  if (!parts) return;
  Part a = part_identity();
  int16_t f[kSumK];
  double e[kSumK];
#pragma unroll
  for (int k = 0; k < kSumK; ++k) {  // every load first, then the fold in cell order
    const int64_t cell = base + t + k * T;
    const bool live = cell < n_cells && cnt[k] != 0;
    f[k] = live ? fi[cell] : int16_t{-2};
    e[k] = live ? en[cell] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < kSumK; ++k) part_combine(a, part_of_cell(f[k], e[k], base + t + k * T));
  const int c = t % C, j = t / C;
  sl[j][c] = a;
  __syncthreads();
  if (t < 4 * C) {  // (c, s): slots [8s, 8s+8) of class c
    const int cc = t % C, ss = t / C;
    Part b = sl[8 * ss][cc];
#pragma unroll
    for (int i = 1; i < 8; ++i) part_combine(b, sl[8 * ss + i][cc]);
    s2[ss][cc] = b;
  }
  __syncthreads();
  if (t < C) {
    Part b0 = s2[0][t], b2 = s2[2][t];
    part_combine(b0, s2[1][t]);
    part_combine(b2, s2[3][t]);
    part_combine(b0, b2);
    parts[(static_cast<int64_t>(p) * C + t) * n_blocks + blockIdx.x] = b0;
  }
}

// final level: CTA (p, c) over the n_blocks block parts of (p, c)
__global__ void __launch_bounds__(kFinalCta)
k_summary_final(const Part* __restrict__ parts, int C, int64_t n_blocks, int64_t n_windows,
                gsb_class_summary* __restrict__ out) {
  __shared__ Part red[kFinalCta / 32];
  const int pc = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  gsb::grid_dep_wait();  // the block parts
  const Part* src = parts + static_cast<int64_t>(pc) * n_blocks;
  Part a = part_identity();
  int64_t x = t;
  for (; x + kFinalCta < n_blocks; x += 2 * kFinalCta) {  // two loads in flight, in order
    const Part p0 = ld_part_cg(src + x), p1 = ld_part_cg(src + x + kFinalCta);
    part_combine(a, p0);
    part_combine(a, p1);
  }
  for (; x < n_blocks; x += kFinalCta) part_combine(a, ld_part_cg(src + x));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Part y = part_shfl_down_w(a, o, 32);
    if (lane < o) part_combine(a, y);
  }
  if (lane == 0) red[w] = a;
  __syncthreads();
  if (w == 0) {
    a = lane < kFinalCta / 32 ? red[lane] : part_identity();
#pragma unroll
    for (int o = kFinalCta / 64; o > 0; o >>= 1) {
      const Part y = part_shfl_down_w(a, o, 32);
      if (lane < o) part_combine(a, y);
    }
    if (lane == 0) {
      gsb_class_summary o;
      o.n_cmd = a.cmd;
      o.n_infeasible = a.inf;
      o.n_empty = n_windows - a.cmd;
      o.sum_energy_j = a.sum;
      o.min_energy_j = a.arg >= 0 ? e_unkey(a.mnk) : INFINITY;
      o.argmin_cell = a.arg;
      out[pc] = o;
    }
  }
}

// K2 over the non-empty list: CTA unit (profile p, chunk ch) evaluates list positions
// [128 ch, 128 ch + 128) of profile p, one lane each (the profile is uniform per CTA, so the
// per-profile constant-operand instantiation runs with no divergence). Persistent grid: units
// b = blockIdx.x, + gridDim.x, ... (one wave at C4). Inputs in list order when K1b wrote them
// (T_ref / min_deadline: coalesced, no dependent gather). Empty cells are finished by
// k_cells_finish (their "no command" outputs and the summary), not here.
struct ListIn {
  const uint32_t* list;
  const int64_t* n_list;
  const double* t_ref;         // [P][cap] in list order, or NULL (gather t_ref[p][cell])
  const double* min_deadline;  // [cap] in list order, or NULL (gather)
  int64_t cap;
};

#ifndef GSB_K2_CTA
#define GSB_K2_CTA 64
#endif
// 2-warp CTAs: a one-wave K2 is FP64-pipe bound per SM, and its warps of work split over the
// SMs in CTA-sized lumps, so 2-warp CTAs (up to 20 per SM) leave at most 2 warps of imbalance
// per SM where 4-warp CTAs left 4 (36 vs 40 warps at C4)
constexpr int kListCta = GSB_K2_CTA;

template <int G>
__global__ void __launch_bounds__(kListCta, 1280 / kListCta)
k_prefill_select_list(const __grid_constant__ SelectParams sp, const __grid_constant__ ClockSet<G> cs,
                      int P, ListIn li, const double* __restrict__ t_ref,
                      const double* __restrict__ min_deadline, double* __restrict__ window,
                      int16_t* __restrict__ f_idx, double* __restrict__ energy) {
  const int t = threadIdx.x;
  gsb::grid_dep_wait();  // the list and K1's cells
  gsb::grid_dep_launch();
  const int64_t n = sp.n_cells;
  const int64_t nl = *li.n_list;  // one list for every profile (emptiness is per cell); < 2^32
  const unsigned nch = static_cast<unsigned>((nl + kListCta - 1) / kListCta);
  const unsigned units = nch * static_cast<unsigned>(P);
  for (unsigned b = blockIdx.x; b < units; b += gridDim.x) {
    const int p = static_cast<int>(b / nch);
    const int64_t k = static_cast<int64_t>(b - static_cast<unsigned>(p) * nch) * kListCta + t;
    if (k >= nl) continue;
    const int64_t cell = li.list[k];
    const double T = li.t_ref ? li.t_ref[p * li.cap + k] : t_ref[p * n + cell];
    double W;
    if (sp.mode == GSB_FIXED_WINDOW) {
      W = sp.fixed_window;
    } else if (sp.mode == GSB_DEADLINE_SLACK) {
      const double mdl = li.min_deadline ? li.min_deadline[k] : min_deadline[cell];
      const double now = static_cast<double>((sp.w0 + cell / sp.C) * sp.window_ms);
      W = std_max(sp.margin * (mdl - now), sp.min_budget);
    } else {
      W = window[cell];
    }
    if (p == 0 && window && sp.mode != GSB_PER_CELL_WINDOW) window[cell] = W;
    double be;
    int best;
    switch (p) {
      case 0: best = scan_clocks_c<G, 0>(cs, T, W, &be); break;
      case 1: best = scan_clocks_c<G, 1>(cs, T, W, &be); break;
      case 2: best = scan_clocks_c<G, 2>(cs, T, W, &be); break;
      default: best = scan_clocks_c<G, 3>(cs, T, W, &be); break;
    }
    const int64_t o = p * n + cell;
    f_idx[o] = static_cast<int16_t>(best);
    energy[o] = best >= 0 ? be : 0.0;
  }
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
                 double* __restrict__ energy, double* __restrict__ t_out, gsb_running_jobs run) {
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
    double w = wf ? wf[j] : 1.0;
    if (run.d_running && run.d_running[j]) {
      // the running job's outstanding share at the snapshot (simkernel.cpp:476-479): work done
      // since its last update at the applied clock, in reference time, off its remaining work
      const double done = (now_ms[b] - run.d_updated_ms[j]) * run.d_freq_mhz[j] / tab->f_ref;
      const double remaining = std_max(run.d_remaining_ref_ms[j] - done, 0.0);
      w = remaining / run.d_t_ref_ms[j];
    }
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

// ---------------------------------------------------------------- M/G/1 side output
// BASELINE north_star (2) asks for an M/G/1-style waiting time and the energy per request beside
// each decision. The reference has no such term (SPEC.md:294 lists it as a non-goal), so this is
// a labelled, parity-UNPINNED side output, never an input of the bit-exact argmin: for cell
// (window w, class c) of profile p with n jobs, service times s_j = (f_ref / f) t_j at the
// command's clock f (f_max when infeasible), t_j = (a L_j + b) L_j + c, arrival rate
// lambda = n / window_ms, Pollaczek-Khinchine: rho = lambda E[s], Wq = lambda E[s^2] /
// (2 (1 - rho)) (+inf when rho >= 1), and E / n. One thread per (cell, profile) walks the window's
// requests of its class in arrival order (deterministic sums).
__global__ void k_mg1(int P, int C, int64_t n_windows, double window_ms,
                      const ProfTab* __restrict__ tabs, const int32_t* __restrict__ prompt,
                      const uint8_t* __restrict__ cls, const int64_t* __restrict__ bounds,
                      const int16_t* __restrict__ f_idx, const double* __restrict__ energy,
                      double* __restrict__ wq, double* __restrict__ rho,
                      double* __restrict__ e_req) {
  const int64_t cells = n_windows * C;
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= cells * P) return;
  const int p = static_cast<int>(i / cells);
  const int64_t cell = i - p * cells, w = cell / C;
  const int c = static_cast<int>(cell - w * C);
  const ProfTab& t = tabs[p];
  const int fi = f_idx[i];
  if (fi == -2) {  // empty queue: no command
    wq[i] = rho[i] = e_req[i] = 0.0;
    return;
  }
  double s1 = 0.0, s2 = 0.0;
  int64_t n = 0;
  for (int64_t j = bounds[w]; j < bounds[w + 1]; ++j) {
    if (cls[j] != c) continue;
    const double L = static_cast<double>(prompt[j]);
    const double tj = (t.lat_a * L + t.lat_b) * L + t.lat_c;
    s1 += tj;
    s2 += tj * tj;
    ++n;
  }
  const double f = fi >= 0 ? t.f[fi] : t.f_max;
  const double k = t.f_ref / f;
  const double lambda = static_cast<double>(n) / window_ms;
  const double es = k * s1 / static_cast<double>(n), es2 = k * k * s2 / static_cast<double>(n);
  const double r = lambda * es;
  rho[i] = r;
  wq[i] = r < 1.0 ? lambda * es2 / (2.0 * (1.0 - r)) : INFINITY;
  e_req[i] = fi >= 0 ? energy[i] / static_cast<double>(n) : 0.0;
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

// The non-empty list of a pass built by k_compact (when K1b did not emit one): the list and its
// count in the context scratch, the look-back statuses in the context's zeroed sync words.
struct ListPass {
  uint32_t* list;
  int64_t* n_list;
  CompactHdr* hdr;
  unsigned long long* status;
  int64_t n_tiles;
};

size_t align_up(size_t x) { return (x + 255) & ~size_t{255}; }

bool list_pass_buffers(gsb_ctx* ctx, int64_t n_cells, size_t scratch_offset, ListPass* lp) {
  lp->n_tiles = (n_cells + kCompactTile - 1) / kCompactTile;
  char* sc = static_cast<char*>(gsb_scratch(
      ctx, scratch_offset + align_up(sizeof(uint32_t) * n_cells) + sizeof(int64_t)));
  char* sy = static_cast<char*>(gsb_sync_words(
      ctx, 256 + align_up(sizeof(unsigned long long) * std::max<int64_t>(1, lp->n_tiles))));
  if (!sc || !sy) return false;
  lp->list = reinterpret_cast<uint32_t*>(sc + scratch_offset);
  lp->n_list = reinterpret_cast<int64_t*>(sc + scratch_offset + align_up(sizeof(uint32_t) * n_cells));
  lp->hdr = reinterpret_cast<CompactHdr*>(sy);
  lp->status = reinterpret_cast<unsigned long long*>(sy + 256);
  return true;
}

template <class Src>
cudaError_t launch_compact(const ListPass& lp, Src src, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaMemsetAsync(lp.n_list, 0, sizeof(int64_t), s);
  return gsb::launch_pdl(k_compact<Src>, dim3(static_cast<unsigned>(lp.n_tiles)),
                         dim3(kCompactThreads), 0, s, src, n, lp.hdr, lp.status, lp.list,
                         lp.n_list);
}

// Block parts of the summary tree (placed at the start of the context scratch).
int64_t finish_blocks(int C, int64_t n_cells) {
  const int64_t per = static_cast<int64_t>(32) * C * kSumK;
  return std::max<int64_t>(1, (n_cells + per - 1) / per);
}

size_t finish_scratch_bytes(int P, int C, int64_t n_cells) {
  return align_up(sizeof(Part) * static_cast<size_t>(P) * C * finish_blocks(C, n_cells));
}

// k_cells_finish (+ k_summary_final when out != NULL) for a [P][n_cells] result.
cudaError_t launch_finish(gsb_ctx* ctx, int P, int C, int64_t n_cells, const uint32_t* count,
                          int16_t* f_idx, double* energy, gsb_class_summary* out, Part* parts,
                          cudaStream_t s, bool early_fill = true) {
  (void)ctx;
  const int64_t nb = finish_blocks(C, n_cells);
  if (nb > 65535LL * 1024) return cudaErrorInvalidValue;
  Part* pp = out ? parts : nullptr;
  const dim3 grid(static_cast<unsigned>(nb), static_cast<unsigned>(P));
  cudaError_t e = cudaSuccess;
  if (n_cells > 0) {
    switch (C) {
#define GSB_FIN(CC)                                                                             \
  case CC:                                                                                    \
    e = gsb::launch_pdl(k_cells_finish<CC>, grid, dim3(32 * CC), 0, s, n_cells, count, f_idx,  \
                        energy, pp, nb, early_fill ? 1 : 0);                                  \
    break;
      GSB_FIN(1) GSB_FIN(2) GSB_FIN(3) GSB_FIN(4) GSB_FIN(5) GSB_FIN(6) GSB_FIN(7) GSB_FIN(8)
#undef GSB_FIN
      default: return cudaErrorInvalidValue;
    }
  }
  if (e != cudaSuccess || !out) return e;
  return gsb::launch_pdl(k_summary_final, dim3(static_cast<unsigned>(P * C)), dim3(kFinalCta), 0,
                         s, static_cast<const Part*>(parts), C, n_cells > 0 ? nb : int64_t{0},
                         n_cells / C, out);
}

template <class K>
int resident_ctas(gsb_ctx* ctx, K kernel, int threads) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, 0) != cudaSuccess || nb < 1)
    nb = 1;
  return nb * ctx->n_sms;
}

}  // namespace

size_t gsb_finish_scratch_bytes(int P, int C, int64_t n_cells) {
  return finish_scratch_bytes(P, C, n_cells);
}

// for the fused pass (gsb_prefill.cu): the empty cells' outputs and the summary
int gsb_internal_finish(gsb_ctx* ctx, int P, int C, int64_t n_cells, const uint32_t* count,
                        int16_t* f_idx, double* energy, gsb_class_summary* out, cudaStream_t s) {
  void* parts = out ? gsb_scratch(ctx, finish_scratch_bytes(P, C, n_cells)) : nullptr;
  if (out && !parts) return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass: scratch allocation failed");
  if (launch_finish(ctx, P, C, n_cells, count, f_idx, energy, out, static_cast<Part*>(parts), s,
                    /*early_fill=*/false) != cudaSuccess)
    return gsb_check_launch(ctx, "prefill_pass (finish)");
  return GSB_OK;
}

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
  return gsb_prefill_select_list(ctx, cfg, n_cells, d_t_ref, d_count, nullptr, d_min_deadline,
                                 d_window, d_f_idx, d_energy, d_summary, stream);
}

int gsb_prefill_select_list(gsb_ctx* ctx, const gsb_select_cfg* cfg, int64_t n_cells,
                            const double* d_t_ref, const uint32_t* d_count,
                            const gsb_cell_list* list, const double* d_min_deadline,
                            double* d_window, int16_t* d_f_idx, double* d_energy,
                            gsb_class_summary* d_summary, void* stream) {
  const uint32_t* d_list = list ? list->d_cells : nullptr;
  if (d_list && (!list->d_n || list->capacity < n_cells))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "select: bad cell list");
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
  ClockSet<81> cs{};  // filled per call (host), passed by value as the kernel parameter
  const bool all_c = gsb_k2::make_clockset81(ctx, &cs);
  if (all_c) {
    if (d_count && n_cells < (int64_t{1} << 32)) {
      // non-empty list (K1b's, or k_compact's) + one wave of K2 over it, then the empty cells'
      // outputs and the summary in one memory-bound pass
      const int P = ctx->n_profiles, Cn = std::max(1, cfg->n_classes);
      const size_t fin_bytes = d_summary ? finish_scratch_bytes(P, Cn, n_cells) : 0;
      ListPass lp{};
      ListIn li{};
      if (d_list) {  // K1b's list (gsb_route_bin_list) and its list-order inputs
        li = ListIn{d_list, list->d_n, list->d_t_ref, list->d_min_deadline, list->capacity};
        if (fin_bytes && !gsb_scratch(ctx, fin_bytes))
          return gsb_set_error(ctx, GSB_CUDA_ERROR, "select: scratch allocation failed");
      } else {
        if (!list_pass_buffers(ctx, n_cells, fin_bytes, &lp))
          return gsb_set_error(ctx, GSB_CUDA_ERROR, "select: scratch allocation failed");
        if (launch_compact(lp, NonEmptyCount{d_count}, n_cells, s) != cudaSuccess)
          return gsb_check_launch(ctx, "prefill_select (compact)");
        li = ListIn{lp.list, lp.n_list, nullptr, nullptr, n_cells};
      }
      static int grid_k2 = 0;
      if (!grid_k2) grid_k2 = resident_ctas(ctx, k_prefill_select_list<81>, kListCta);
      gsb::launch_pdl(k_prefill_select_list<81>, dim3(static_cast<unsigned>(grid_k2)),
                      dim3(kListCta), 0, s, sp, cs, P, li, d_t_ref, d_min_deadline, d_window,
                      d_f_idx, d_energy);
      if (launch_finish(ctx, P, Cn, n_cells, d_count, d_f_idx, d_energy, d_summary,
                        static_cast<Part*>(ctx->d_scratch), s) != cudaSuccess)
        return gsb_check_launch(ctx, "prefill_select (finish)");
      return gsb_check_launch(ctx, "prefill_select");
    }
    const dim3 grid(gx, static_cast<unsigned>(ctx->n_profiles));
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
  return gsb_select_batches_running(ctx, cfg, profile, n_batches, d_off, d_prompt, d_wf, nullptr,
                                    d_deadline, d_now, d_window, d_f_idx, d_energy, d_t_ref_out,
                                    stream);
}

int gsb_select_batches_running(gsb_ctx* ctx, const gsb_select_cfg* cfg, int profile,
                               int64_t n_batches, const int64_t* d_off, const int32_t* d_prompt,
                               const double* d_wf, const gsb_running_jobs* run,
                               const double* d_deadline, const double* d_now, double* d_window,
                               int16_t* d_f_idx, double* d_energy, double* d_t_ref_out,
                               void* stream) {
  if (!ctx || !cfg) return GSB_INVALID_ARGUMENT;
  gsb_running_jobs rj{};
  if (run && run->d_running) {
    if (!run->d_remaining_ref_ms || !run->d_updated_ms || !run->d_freq_mhz || !run->d_t_ref_ms ||
        !d_now)
      return gsb_set_error(ctx, GSB_INVALID_ARGUMENT,
                           "select_batches: running jobs need their state and the snapshot now");
    rj = *run;
  }
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
      d_deadline, d_now, d_window, d_f_idx, d_energy, d_t_ref_out, rj);
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
  if (n_cells >= (int64_t{1} << 32))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "summary: too many cells");
  // the same tree as the K2 path (k_cells_finish, emptiness read from f_idx), identical bytes
  void* parts = gsb_scratch(ctx, finish_scratch_bytes(n_profiles, n_classes, n_cells));
  if (!parts) return gsb_set_error(ctx, GSB_CUDA_ERROR, "summary: scratch allocation failed");
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  if (launch_finish(ctx, n_profiles, n_classes, n_cells, nullptr, const_cast<int16_t*>(d_f_idx),
                    const_cast<double*>(d_energy), d_out, static_cast<Part*>(parts), s) !=
      cudaSuccess)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "summary: too many cells");
  return gsb_check_launch(ctx, "prefill_summary");
}

int gsb_mg1_side_output(gsb_ctx* ctx, int n_classes, int64_t n_windows, double window_ms,
                        const int32_t* d_prompt, const uint8_t* d_class, const int64_t* d_bounds,
                        const int16_t* d_f_idx, const double* d_energy, double* d_wq_ms,
                        double* d_rho, double* d_energy_per_request, void* stream) {
  if (!ctx || n_classes < 1 || n_windows < 0 || !(window_ms > 0.0))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "mg1: bad shape");
  const int64_t total = n_windows * n_classes * ctx->n_profiles;
  if (total == 0) return GSB_OK;
  k_mg1<<<static_cast<unsigned>((total + 127) / 128), 128, 0, gsb_pick_stream(ctx, stream)>>>(
      ctx->n_profiles, n_classes, n_windows, window_ms, static_cast<const ProfTab*>(ctx->d_tabs),
      d_prompt, d_class, d_bounds, d_f_idx, d_energy, d_wq_ms, d_rho, d_energy_per_request);
  return gsb_check_launch(ctx, "mg1_side_output");
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
