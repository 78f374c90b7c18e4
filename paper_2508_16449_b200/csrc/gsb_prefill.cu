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
#include <type_traits>
#include <cmath>

#include "gsb_common.cuh"

using gsb::ProfTab;
using gsb::std_max;
using gsb::std_min;

namespace {

struct U32ToI64 {
  __host__ __device__ int64_t operator()(uint32_t x) const { return static_cast<int64_t>(x); }
};

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
// floor(a / d) for a >= 0, d > 0 without a 64-bit integer divide: a double estimate, then an
// exact integer correction (the estimate is off by at most one for a < 2^62).
__device__ __forceinline__ int64_t div_floor(int64_t a, int64_t d, double rd) {
  int64_t q = static_cast<int64_t>(static_cast<double>(a) * rd);
  if (q * d > a) --q;
  if ((q + 1) * d <= a) ++q;
  return q;
}

// bounds[k] = #requests whose window index (arrival / W - w0) is < k, k = 0..n_windows, i.e. the
// first request of window k (arrivals are non-decreasing, trace.cpp:109-111). Request i owns
// the entries k in (w(i-1), w(i)] (request 0 covers k <= w(0), a virtual request n the tail),
// so every entry is written exactly once.
// Lane l of a warp owns tile l of 32 requests. It reads only the LAST arrival of its tile (one
// 32-byte sector per 32 requests) and takes the previous tile's from its neighbour: with sorted
// arrivals a tile holds a window edge iff its two ends differ. The warp then resolves its edge
// tiles cooperatively, up to four at a time: lane l loads element l of each of them (four
// independent coalesced loads in flight), so a warp pays two dependent DRAM latencies in the
// common case and the pass reads ~1/8 of the arrivals plus the edge tiles.
constexpr int kBoundsTile = 32;
constexpr int kBoundsBatch = 4;
constexpr unsigned kFull = 0xffffffffu;

__global__ void __launch_bounds__(256)
k_window_bounds(const int64_t* __restrict__ arrival, int64_t n, int64_t window_ms, int64_t w0,
                int64_t n_windows, int64_t* __restrict__ bounds) {
  gsb::grid_dep_wait();    // the arrivals may come from the previous launch (e.g. a copy)
  gsb::grid_dep_launch();  // K1b may be scheduled now; it waits for this grid's bounds
  const double rd = 1.0 / static_cast<double>(window_ms);
  const int lane = threadIdx.x & 31;
  const int64_t span = ((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5) *
                       (32 * kBoundsTile);
  if (span > n) return;  // warp-uniform
  auto win = [&](int64_t i) -> int64_t {
    if (i < 0) return -1;
    if (i >= n) return n_windows;
    return div_floor(__ldg(arrival + i), window_ms, rd) - w0;
  };
  const int64_t t0 = span + static_cast<int64_t>(lane) * kBoundsTile;
  const bool live = t0 <= n;
  const int64_t wlast = live ? win(min(t0 + kBoundsTile - 1, n)) : 0;
  int64_t wprev = __shfl_up_sync(kFull, wlast, 1);
  if (lane == 0) wprev = win(t0 - 1);
  unsigned edges = __ballot_sync(kFull, live && wlast != wprev);
  while (edges) {
    int src[kBoundsBatch];
    int64_t a[kBoundsBatch];
#pragma unroll
    for (int k = 0; k < kBoundsBatch; ++k) {  // issue the batch's loads together
      src[k] = edges ? __ffs(static_cast<int>(edges)) - 1 : -1;
      edges &= edges - 1;
      const int64_t i = span + static_cast<int64_t>(src[k]) * kBoundsTile + lane;
      a[k] = (src[k] >= 0 && i < n) ? __ldg(arrival + i) : 0;
    }
#pragma unroll
    for (int k = 0; k < kBoundsBatch; ++k) {
      if (src[k] < 0) break;  // warp-uniform
      const int64_t wp0 = __shfl_sync(kFull, wprev, src[k]);
      const int64_t i = span + static_cast<int64_t>(src[k]) * kBoundsTile + lane;
      const int64_t wi = i < n ? div_floor(a[k], window_ms, rd) - w0 : n_windows;
      int64_t wp = __shfl_up_sync(kFull, wi, 1);
      if (lane == 0) wp = wp0;
      if (i <= n && wi != wp) {
        const int64_t hi = min(wi, n_windows);
        for (int64_t k2 = max(wp + 1, int64_t{0}); k2 <= hi; ++k2) bounds[k2] = i;
      }
    }
  }
}

// classify(), router.cpp:26-31: number of thresholds strictly below the prompt. The thresholds
// are ascending and distinct (RoutingConfig::validate, router.cpp:7-11, checked host-side) and
// padded with INT_MAX, so the count is a branch-free binary search: ceil(log2 C) compares on
// thresholds held in registers.
template <int C>
__device__ __forceinline__ int classify_c(const int32_t (&t)[GSB_MAX_CLASSES - 1], int32_t L) {
  if (C == 1) return 0;
  if (C == 2) return t[0] < L ? 1 : 0;
  if (C <= 4) {
    const bool hi = t[1] < L;
    return (hi ? 2 : 0) + ((hi ? t[2] : t[0]) < L ? 1 : 0);
  }
  const bool hi = t[3] < L;
  const bool mid = (hi ? t[5] : t[1]) < L;
  const int32_t lo = mid ? (hi ? t[6] : t[2]) : (hi ? t[4] : t[0]);
  return (hi ? 4 : 0) + (mid ? 2 : 0) + (lo < L ? 1 : 0);
}

// ---------------------------------------------------------------- K1b: route + bin
// One CTA of kRouteWarps warps owns G = 32 / P consecutive windows. Per chunk of
// <= kRouteCap requests of its range (normally one chunk: C4 windows hold ~300 requests, G = 8):
//   0. one TMA bulk copy (cp.async.bulk, mbarrier completion) stages the chunk's prompts in
//      shared memory: the only HBM read of the prompts;
//   A. each warp takes a contiguous quarter of the chunk: classify() (router.cpp:26-31), write
//      the class, key = (window g, class c), per-warp key histogram (match.any + leader add),
//      min of prefill deadlines (simkernel.cpp:499-501) per key (order-free: min is exact);
//      phase A also records each request's rank among its warp's requests of the same key
//      (the running per-warp count + its lane rank in the round);
//   B. stable counting sort of the chunk by key: request j goes to cursor off[key] + (counts
//      of warps < w) + its rank, so every (g, c) run is in ARRIVAL order (no second match);
//   C. fold: lane (g, p) of warp w walks window g's runs of the classes c = w (mod warps) and
//      extends T[g][c][p] += (a_p L + b_p) L + c_p left to right, exactly prefill_opt.cpp:9-14.
//      The P lanes of a window read the same entry (broadcast); run lengths of a class are
//      similar across windows, so lanes stay busy, and the warps fold different classes.
// Shared memory is 8 B per chunk slot (prompt, key|rank, sorted index), so nine CTAs share an SM and
// the C4 grid (1,250 CTAs) is one wave (P = 1 holds 32 windows x C keys per CTA: fewer CTAs).
constexpr int kRouteWarps = 4;
constexpr int kRouteCap = 2544;  // requests per chunk
constexpr int kRouteMinBlocks = 9;

__device__ __forceinline__ unsigned long long ord_f64(double x) {  // order-preserving key
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord_f64(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(u));
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <int K, bool DL>
struct RouteSmem {  // one CTA
  // key (window g, class c) in the low kKeyBits, the request's rank among its warp's requests
  // of that key above them
  static constexpr int kKeyBits = K <= 64 ? 6 : 8;
  using KR = typename std::conditional<K <= 64, uint16_t, uint32_t>::type;
  alignas(16) int32_t stage[kRouteCap + 4];  // prompts of [c0 & ~3, c1)
  uint16_t srt[kRouteCap];                   // stage index of the chunk's requests, by key (stable)
  KR kr[kRouteCap];
  uint64_t bar;
  int64_t bnd[33];
  int32_t lb[33];  // chunk-local window starts, lb[G] = "never"
  int32_t off[K + 1];
  int32_t hist[kRouteWarps][K];  // per-warp key counts, then per-warp scatter cursors
  uint32_t cnt[K];
  unsigned long long mdl[DL ? K : 1];
};

template <int C, int P, bool DL, int GW>
__global__ void __launch_bounds__(kRouteWarps * 32, GW * C > 64 ? 6 : kRouteMinBlocks)
k_route_bin(const __grid_constant__ RouteParams rp, const int64_t* __restrict__ arrival,
            const int32_t* __restrict__ prompt, const int64_t* __restrict__ bounds,
            uint8_t* __restrict__ cls_out, uint32_t* __restrict__ count,
            double* __restrict__ t_ref, double* __restrict__ min_deadline) {
  constexpr int G = GW, K = G * C, E = (K + 31) / 32, NW = kRouteWarps;
  constexpr int kNever = 0x3fffffff;
  using S = RouteSmem<K, DL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& s = *reinterpret_cast<S*>(smem_raw);
  const int tid = threadIdx.x, wib = tid >> 5, lane = tid & 31;
  const unsigned lt = lanemask_lt();
  int32_t th[GSB_MAX_CLASSES - 1];
#pragma unroll
  for (int k = 0; k < GSB_MAX_CLASSES - 1; ++k) th[k] = rp.thr[k];
  const int64_t w_first = static_cast<int64_t>(blockIdx.x) * G;
  gsb::grid_dep_wait();  // K1a's bounds (programmatic dependent launch)
  gsb::grid_dep_launch();
  for (int k = tid; k <= G; k += NW * 32) s.bnd[k] = bounds[min(w_first + k, rp.n_windows)];
  for (int k = tid; k < K; k += NW * 32) {
    s.cnt[k] = 0;
    if (DL) s.mdl[k] = ~0ull;
  }
  if (tid == 0) gsb::mbar_init(&s.bar, 1);
  __syncthreads();
  const int64_t b0 = s.bnd[0], bG = s.bnd[G];
  const bool tma = (reinterpret_cast<uintptr_t>(prompt) & 15) == 0;
  uint32_t parity = 0;
  // fold role: lane (fg, fp) = (window, profile)
  const int fg = lane / P, fp = lane - (lane / P) * P;
  const bool folder = lane < G * P;
  const double la = rp.lat_a[fp], lb = rp.lat_b[fp], lc = rp.lat_c[fp];
  constexpr int CPW = (C + NW - 1) / NW;  // classes per warp in the fold: c = wib + k * NW
  double acc[CPW];
#pragma unroll
  for (int k = 0; k < CPW; ++k) acc[k] = 0.0;

  for (int64_t c0 = b0; c0 < bG; c0 += kRouteCap) {
    const int64_t c1 = min(c0 + static_cast<int64_t>(kRouteCap), bG);
    const int nc = static_cast<int>(c1 - c0);
    const int64_t a0 = c0 & ~int64_t{3};  // stage[i - a0] = prompt[i]
    // ---- 0: stage the chunk (TMA for the 16-byte-aligned body, threads for the <= 3 tail)
    const int64_t a1 = tma ? (c1 & ~int64_t{3}) : a0;
    if (tid == 0 && a1 > a0) {
      gsb::fence_proxy_async_smem();
      const uint32_t bytes = static_cast<uint32_t>((a1 - a0) * 4);
      gsb::mbar_expect_tx(&s.bar, bytes);
      gsb::bulk_g2s(s.stage, prompt + a0, bytes, &s.bar);
    }
    for (int64_t i = max(a1, c0) + tid; i < c1; i += NW * 32) s.stage[i - a0] = __ldg(prompt + i);
    for (int k = tid; k < NW * K; k += NW * 32) (&s.hist[0][0])[k] = 0;
    if (tid <= G)
      s.lb[tid] = tid == G ? kNever : static_cast<int>(min(max(s.bnd[tid] - c0, int64_t{0}),
                                                           static_cast<int64_t>(kNever)));
    if (a1 > a0) {  // one thread polls the barrier; the others wait in bar.sync
      if (tid == 0) gsb::mbar_wait(&s.bar, parity);
      parity ^= 1;
    }
    __syncthreads();
    const int sb = static_cast<int>(c0 - a0);  // stage index of chunk position 0
    const int32_t* st = s.stage + sb;
    // this warp's contiguous part [j0, j1) of the chunk
    const int q = ((nc + NW * 32 - 1) / (NW * 32)) * 32;
    const int j0 = min(wib * q, nc), j1 = min(j0 + q, nc);
    int32_t* hist_w = s.hist[wib];
    // ---- A: classify, key, histogram, deadlines
    {
      int g_lo = 0;  // window of the round's first request (warp-uniform)
      while (s.lb[g_lo + 1] <= j0) ++g_lo;
      int nb = s.lb[g_lo + 1];
      uint8_t* cls_p = cls_out + c0 + j0 + lane;
#pragma unroll 4
      for (int r = j0; r < j1; r += 32, cls_p += 32) {
        const int j = r + lane;
        const bool valid = j < j1;
        const int32_t L = st[valid ? j : j0];
        const int cl = classify_c<C>(th, L);
        int g = g_lo;
        if (nb <= r + 32) {  // a window starts inside this round (or right after it)
          int k = g_lo + 1;
          for (; s.lb[k] <= r + 32; ++k) g += j >= s.lb[k] ? 1 : 0;
          g_lo = k - 1;
          nb = s.lb[k];
        }
        const int key = g * C + cl;
        const unsigned m = __match_any_sync(kFull, valid ? key : 0x10000);
        const unsigned below = m & lt;
        const int base = hist_w[valid ? key : 0];
        __syncwarp();
        if (valid) {
          *cls_p = static_cast<uint8_t>(cl);
          s.kr[j] = static_cast<typename S::KR>(key | ((base + __popc(below)) << S::kKeyBits));
          if (below == 0) hist_w[key] = base + __popc(m);
          if (DL) {
            const double ttft = L <= rp.slo_boundary ? rp.ttft_sm : rp.ttft_l;
            const double dl = static_cast<double>(__ldg(arrival + c0 + j)) + ttft - rp.allowance;
            if (dl == dl) atomicMin(&s.mdl[key], ord_f64(dl));
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // ---- exclusive scan of the key totals (warp 0, lane l owns keys [l*E, l*E+E)); the
    //      per-warp counts become the warps' scatter cursors
    if (wib == 0) {
      int loc[E];
      int sum = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int k = lane * E + e;
        int t = 0;
        if (k < K) {
#pragma unroll
          for (int w = 0; w < NW; ++w) t += s.hist[w][k];
        }
        loc[e] = t;
        sum += t;
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += v;
      }
      int run = incl - sum;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int k = lane * E + e;
        if (k < K) {
          s.off[k] = run;
          int cur = run;
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const int h = s.hist[w][k];
            s.hist[w][k] = cur;
            cur += h;
          }
          s.cnt[k] += static_cast<uint32_t>(loc[e]);
          run += loc[e];
        }
      }
      if (lane == 31) s.off[K] = incl;
    }
    __syncthreads();
    // ---- B: stable scatter of the stage indices by key (arrival order inside each key): the
    //      warp's cursor for the key plus the rank phase A recorded
#pragma unroll 4
    for (int j = j0 + lane; j < j1; j += 32) {
      const unsigned v = s.kr[j];
      const int key = static_cast<int>(v & ((1u << S::kKeyBits) - 1u));
      s.srt[hist_w[key] + static_cast<int>(v >> S::kKeyBits)] = static_cast<uint16_t>(sb + j);
    }
    __syncthreads();
    // ---- C: ordered fold, lane (window fg, profile fp) of warp w, classes c = w (mod NW)
    if (folder) {
#pragma unroll
      for (int k = 0; k < CPW; ++k) {
        const int c = wib + k * NW;
        if (c >= C) break;
        const int o = s.off[fg * C + c], n = s.off[fg * C + c + 1] - o;
        const uint16_t* run = s.srt + o;
        double a = acc[k];
        // arithmetic, not a table: a per-profile (a L + b) L + c lookup table gathered from
        // L1/L2 measured 2x slower (latency-bound at 31% issue) than these 5 DP operations
#pragma unroll 8
        for (int j = 0; j < n; ++j) {
          const double Ld = static_cast<double>(s.stage[run[j]]);
          a = a + 1.0 * ((la * Ld + lb) * Ld + lc);
        }
        acc[k] = a;
      }
    }
    __syncthreads();
  }
  const int64_t cells = rp.n_windows * C;
  if (folder && w_first + fg < rp.n_windows) {
    const int64_t cell0 = (w_first + fg) * C;
#pragma unroll
    for (int k = 0; k < CPW; ++k) {
      const int c = wib + k * NW;
      if (c < C) t_ref[fp * cells + cell0 + c] = acc[k];
    }
  }
  for (int k = tid; k < K; k += NW * 32) {
    const int64_t w = w_first + k / C;
    if (w >= rp.n_windows) continue;
    const int64_t cell = w * C + k % C;
    count[cell] = s.cnt[k];
    if (DL && min_deadline) {
      const unsigned long long v = s.mdl[DL ? k : 0];
      min_deadline[cell] = v == ~0ull ? INFINITY : unord_f64(v);
    }
  }
}

template <int C, int P, bool DL, int G>
int launch_route_bin_g(const RouteParams& rp, const int64_t* d_arrival, const int32_t* d_prompt,
                       const int64_t* d_bounds, uint8_t* d_class, uint32_t* d_count,
                       double* d_t_ref, double* d_min_deadline, cudaStream_t s) {
  const size_t smem = sizeof(RouteSmem<G * C, DL>);
  if (cudaFuncSetAttribute(k_route_bin<C, P, DL, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return -1;
  const unsigned blocks = static_cast<unsigned>((rp.n_windows + G - 1) / G);
  if (gsb::launch_pdl(k_route_bin<C, P, DL, G>, dim3(blocks), dim3(kRouteWarps * 32), smem, s, rp,
                      d_arrival, d_prompt, d_bounds, d_class, d_count, d_t_ref,
                      d_min_deadline) != cudaSuccess)
    return -1;
  return 0;
}

// G = 32 / P windows per CTA (lanes (window, profile) fill the fold warp). With one profile and
// dense windows (32 windows would not fit one chunk) G = 8: four times the CTAs, one chunk each,
// for small traces that would otherwise run a few long CTAs (fold lanes are cheap at P = 1).
template <int C, int P, bool DL>
int launch_route_bin(const RouteParams& rp, int64_t n_req, const int64_t* d_arrival,
                     const int32_t* d_prompt, const int64_t* d_bounds, uint8_t* d_class,
                     uint32_t* d_count, double* d_t_ref, double* d_min_deadline, cudaStream_t s) {
  if constexpr (P == 1) {
    if (n_req > rp.n_windows * (kRouteCap / 32))
      return launch_route_bin_g<C, P, DL, 8>(rp, d_arrival, d_prompt, d_bounds, d_class, d_count,
                                             d_t_ref, d_min_deadline, s);
  }
  return launch_route_bin_g<C, P, DL, 32 / P>(rp, d_arrival, d_prompt, d_bounds, d_class, d_count,
                                              d_t_ref, d_min_deadline, s);
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

RouteParams make_route_params(gsb_ctx* ctx, const gsb_route_cfg* cfg) {
  RouteParams rp{};
  rp.n_thr = cfg->enabled ? cfg->n_thresholds : 0;
  for (int i = 0; i < GSB_MAX_CLASSES - 1; ++i)
    rp.thr[i] = i < rp.n_thr ? cfg->thresholds[i] : 2147483647;  // never below a prompt
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

// ---------------------------------------------------------------- single-call entry kernels
// classify() for a flat prompt array (router.cpp:26-31); thresholds by value, unused = INT_MAX.
struct Thr {
  int32_t t[GSB_MAX_CLASSES - 1];
};

__global__ void k_classify(Thr th, int64_t n, const int32_t* __restrict__ prompt,
                           int32_t* __restrict__ cls) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t L = prompt[i];
    int c = 0;
#pragma unroll
    for (int k = 0; k < GSB_MAX_CLASSES - 1; ++k) c += th.t[k] < L ? 1 : 0;
    cls[i] = c;
  }
}

// PrefillBatch::t_ref_total_ms under a bare LatencyModel (prefill_opt.cpp:9-14)
__global__ void k_t_ref_batches(double la, double lb, double lc, int64_t n_batches,
                                const int64_t* __restrict__ off, const int32_t* __restrict__ prompt,
                                const double* __restrict__ wf, double* __restrict__ out) {
  const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (b >= n_batches) return;
  double T = 0.0;
  for (int64_t j = off[b]; j < off[b + 1]; ++j) {
    const double L = static_cast<double>(prompt[j]);
    T = T + (wf ? wf[j] : 1.0) * ((la * L + lb) * L + lc);
  }
  out[b] = T;
}

// energy_total_closed_form_j (prefill_opt.cpp:33-43), same operation order
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

int gsb_classify(gsb_ctx* ctx, int n_thresholds, const int32_t* thresholds, int64_t n,
                 const int32_t* d_prompt, int32_t* d_class, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  if (n_thresholds < 0 || n_thresholds > GSB_MAX_CLASSES - 1 || (n_thresholds && !thresholds))
    return gsb_set_error(ctx, GSB_ROUTER_ERROR, "routing: more than 7 thresholds");
  if (n <= 0) return GSB_OK;
  Thr th;
  for (int k = 0; k < GSB_MAX_CLASSES - 1; ++k) th.t[k] = k < n_thresholds ? thresholds[k] : INT_MAX;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  k_classify<<<blocks, 256, 0, gsb_pick_stream(ctx, stream)>>>(th, n, d_prompt, d_class);
  return gsb_check_launch(ctx, "classify");
}

int gsb_t_ref_batches(gsb_ctx* ctx, const double lat_abc[3], int64_t n_batches,
                      const int64_t* d_off, const int32_t* d_prompt, const double* d_wf,
                      double* d_out, void* stream) {
  if (!ctx || !lat_abc) return GSB_INVALID_ARGUMENT;
  if (n_batches <= 0) return GSB_OK;
  k_t_ref_batches<<<static_cast<unsigned>((n_batches + 255) / 256), 256, 0,
                    gsb_pick_stream(ctx, stream)>>>(lat_abc[0], lat_abc[1], lat_abc[2], n_batches,
                                                   d_off, d_prompt, d_wf, d_out);
  return gsb_check_launch(ctx, "t_ref_batches");
}

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

int gsb_window_bounds(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req,
                      const int64_t* d_arrival, int64_t* d_bounds, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  int rc = check_route_cfg(ctx, cfg);
  if (rc) return rc;
  const int64_t warps = n_req / (32 * kBoundsTile) + 1;
  const int64_t blocks = (warps + 7) / 8;
  k_window_bounds<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), 256, 0,
                    gsb_pick_stream(ctx, stream)>>>(d_arrival, n_req, cfg->window_ms, cfg->w0,
                                                    cfg->n_windows, d_bounds);
  return gsb_check_launch(ctx, "window_bounds");
}

int gsb_route_bin(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req, const int64_t* d_arrival,
                  const int32_t* d_prompt, const int64_t* d_bounds, uint8_t* d_class,
                  uint32_t* d_count, double* d_t_ref, double* d_min_deadline, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  int rc = check_route_cfg(ctx, cfg);
  if (rc) return rc;
  if (ctx->n_profiles < 1) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "route: no profiles set");
  RouteParams rp = make_route_params(ctx, cfg);
  rp.want_deadline = d_min_deadline != nullptr;
  const int P = ctx->n_profiles;
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  const bool dl = rp.want_deadline != 0;
  const int key = (rp.C - 1) * 8 + (P - 1) * 2 + (dl ? 1 : 0);
  int lrc = 0;
  switch (key) {
#define GSB_RB(CC, PP)                                                                          \
  case ((CC)-1) * 8 + ((PP)-1) * 2:                                                            \
    lrc = launch_route_bin<CC, PP, false>(rp, n_req, d_arrival, d_prompt, d_bounds, d_class,   \
                                          d_count, d_t_ref, d_min_deadline, s);                \
    break;                                                                                      \
  case ((CC)-1) * 8 + ((PP)-1) * 2 + 1:                                                        \
    lrc = launch_route_bin<CC, PP, true>(rp, n_req, d_arrival, d_prompt, d_bounds, d_class,    \
                                         d_count, d_t_ref, d_min_deadline, s);                 \
    break;
#define GSB_RB_P(CC) GSB_RB(CC, 1) GSB_RB(CC, 2) GSB_RB(CC, 3) GSB_RB(CC, 4)
    GSB_RB_P(1) GSB_RB_P(2) GSB_RB_P(3) GSB_RB_P(4) GSB_RB_P(5) GSB_RB_P(6) GSB_RB_P(7) GSB_RB_P(8)
#undef GSB_RB_P
#undef GSB_RB
    default:
      return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "route: need 1..8 classes, 1..4 profiles");
  }
  if (lrc) return gsb_set_error(ctx, GSB_CUDA_ERROR, "route: shared-memory attribute refused");
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
