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
#include <cstdlib>
#include <cstdio>
#include <string>
#include <chrono>

#include "gsb_common.cuh"
#include "gsb_scan.cuh"

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
  int32_t prompt_host;  // prompts in pinned host memory: plain loads instead of the TMA stage
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
                int64_t n_windows, int64_t* __restrict__ bounds, unsigned* __restrict__ zero_words,
                int64_t n_zero) {
  gsb::grid_dep_wait();    // the arrivals may come from the previous launch (e.g. a copy)
  gsb::grid_dep_launch();  // K1b may be scheduled now; it waits for this grid's bounds
  // the fused pass's counters (tickets, per-chunk readiness) start every pass at zero
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_zero;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    zero_words[i] = 0;
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

// K1a for dense traces (>= kSearchDense requests per window on average): an interpolation
// search that touches ~1 sector per 256 requests plus one 64-byte half line per probe
// (round 2: 13.3 MB of DRAM traffic at C4 from the sampled pass above, whose one sector per 32
// requests the L2 fetches as whole lines, and 198 us when the arrivals are pinned host memory
// read over PCIe as 32-byte requests).
// bounds[k] = #{i : arrival[i] < T_k}, T_k = (w0 + k) * W, because win(a) < k <=> a < T_k for
// integer a and W > 0 (the same values the sampled pass writes). Block j = requests
// [jS, e_j], e_j = min((j + 1)S, n) - 1; it owns the edges k in (win(e_{j-1}), win(e_j)]
// (win(e_{-1}) = -1), whose answers lie in [jS, e_j]: arrival[e_{j-1}] < T_k <= arrival[e_j].
// One warp per block: the CTA's 8 warps share the 9 bracket samples (one load each), then each
// warp probes kProbe consecutive arrivals (an aligned 64-byte half line) around the interpolated
// position until the probe holds the edge; each probe that misses shrinks the bracket past
// it, so the loop terminates. All edges k..win(arrival[q]) share the answer q (empty windows)
// and are written at once. The warp after the last block writes n for the tail edges.
#ifndef GSB_SEARCH_S
#define GSB_SEARCH_S 256
#endif
constexpr int kSearchS = GSB_SEARCH_S;  // requests per block
constexpr int kSearchWarps = 8;    // blocks per CTA
#ifndef GSB_SEARCH_PROBE
#define GSB_SEARCH_PROBE 8
#endif
// arrivals per probe: 8 = an aligned 64-byte half line. Over PCIe at C4, K1a' and the
// host-buffer pass measured 73-75 us / 0.364 ms (8), 75-77 us / 0.37 ms (16) and 88 us / 0.385 ms
// (32): the misses' extra round trips cost less than the bytes saved on the shared H2D link.
// 4 (one sector) measured 82 us alone and the same e2e as 8.
constexpr int kProbe = GSB_SEARCH_PROBE;
static_assert(kProbe == 4 || kProbe == 8 || kProbe == 16 || kProbe == 32, "probe of 4-32 arrivals");
constexpr int64_t kProbeAlign = kProbe >= 16 ? 16 : kProbe;
constexpr int kSearchDense = 64;   // launch rule: n >= kSearchDense * (n_windows + 1)

__global__ void __launch_bounds__(kSearchWarps * 32)
k_window_bounds_search(const int64_t* __restrict__ arrival, int64_t n, int64_t window_ms,
                       int64_t w0, int64_t n_windows, int64_t* __restrict__ bounds,
                       unsigned* __restrict__ zero_words, int64_t n_zero) {
  gsb::grid_dep_wait();
  gsb::grid_dep_launch();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_zero;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    zero_words[i] = 0;
  __shared__ int64_t s_a[kSearchWarps + 1];  // arrival[e_{j-1}] for the CTA's blocks and the last
  const double rd = 1.0 / static_cast<double>(window_ms);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t m = (n + kSearchS - 1) / kSearchS;  // blocks; block m = the tail
  const int64_t jb = static_cast<int64_t>(blockIdx.x) * kSearchWarps;
  auto last_of = [&](int64_t j) -> int64_t { return min((j + 1) * kSearchS, n) - 1; };
  if (threadIdx.x <= kSearchWarps) {
    const int64_t j = jb + threadIdx.x - 1;  // the sample ending block j
    s_a[threadIdx.x] = (j >= 0 && j < m) ? __ldg(arrival + last_of(j)) : 0;
  }
  __syncthreads();
  const int64_t j = jb + wib;
  if (j > m) return;  // warp-uniform
  auto win = [&](int64_t a) -> int64_t { return div_floor(a, window_ms, rd) - w0; };
  const int64_t w_lo = j == 0 ? -1 : win(s_a[wib]);
  if (j == m) {  // tail: edges past the last request's window
    for (int64_t k = max(w_lo + 1, int64_t{0}) + lane; k <= n_windows; k += 32) bounds[k] = n;
    return;
  }
  const int64_t e = last_of(j), a_e = s_a[wib + 1];
  const int64_t ke = min(win(a_e), n_windows);
  int64_t lo = j * kSearchS - 1, a_lo = j == 0 ? 0 : s_a[wib];
  for (int64_t k = max(w_lo + 1, int64_t{0}); k <= ke;) {
    const int64_t T = (w0 + k) * window_ms;
    int64_t hi = e, a_hi = a_e;  // answer in (lo, hi]
    int64_t q, v;                // answer and arrival[q]
    for (;;) {     // arrival[lo] < T <= arrival[hi] (lo may be -1)
      if (hi - lo == 1) {
        q = hi;
        v = a_hi;
        break;
      }
      int64_t g = lo + 1;
      if (lo >= 0) {
        const double frac = static_cast<double>(T - a_lo) / static_cast<double>(a_hi - a_lo);
        g = lo + static_cast<int64_t>(ceil(frac * static_cast<double>(hi - lo)));
        g = min(max(g, lo + 1), hi);
      }
      const int64_t p0 =
          max(min(g - kProbe / 2, hi - (kProbe - 1)), lo + 1) & ~(kProbeAlign - 1);
      const int64_t i = p0 + lane;
      const int64_t x = (lane < kProbe && i < n) ? __ldg(arrival + i) : INT64_MAX;
      const unsigned below = __ballot_sync(kFull, x < T);  // a prefix of the lanes (sorted)
      const int c = __popc(below);
      if (c == 0) {
        hi = min(hi, p0);
        a_hi = __shfl_sync(kFull, x, 0);
      } else if (c == kProbe) {
        lo = max(lo, p0 + kProbe - 1);
        a_lo = __shfl_sync(kFull, x, kProbe - 1);
      } else {
        q = p0 + c;
        v = __shfl_sync(kFull, x, c);
        break;
      }
    }
    const int64_t kend = min(win(v), ke);  // T_k' <= v for every k' in [k, kend]
    for (int64_t k2 = k + lane; k2 <= kend; k2 += 32) bounds[k2] = q;
    k = kend + 1;  // T_k > v: the next answer is past q
    lo = q;
    a_lo = v;
  }
}

// Pinned host memory (cudaHostAlloc / cudaHostRegister), which the kernels read in place over
// PCIe. (cudaPointerGetAttributes enqueues nothing, so it is legal inside a graph capture.)
bool is_host_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// K1a launch: the interpolation search when the arrivals are pinned HOST memory read over PCIe
// (dense traces whose thresholds (w0 + k) * W fit in int64): 3x fewer bytes than the sampled
// pass (C4 e2e: 0.51 -> 0.42 ms per step with two-line probes, then 0.41 with 64-byte ones). From
// device memory the sampled pass stays: two dependent DRAM round trips instead of the search's
// two or three (6.7 vs 8.7 us at C4, graph-timed).
void launch_window_bounds(const int64_t* d_arrival, int64_t n, int64_t window_ms, int64_t w0,
                          int64_t n_windows, int64_t* d_bounds, unsigned* zero_words,
                          int64_t n_zero, cudaStream_t s) {
  const int64_t lim = INT64_MAX / window_ms - 1;
  const bool fits = w0 > -lim && w0 < lim - n_windows - 1;
  // GSB_BOUNDS=sampled / search forces one kernel (tests compare both with a host search)
  const char* force = std::getenv("GSB_BOUNDS");
  const bool host = !force && is_host_ptr(d_arrival);
  const bool search = force && force[0] == 's' && force[1] == 'e'
                          ? fits
                          : (force && force[0] == 's'
                                 ? false
                                 : host && fits && n >= kSearchDense * (n_windows + 1));
  if (search) {
    const int64_t blocks = ((n + kSearchS - 1) / kSearchS + 1 + kSearchWarps - 1) / kSearchWarps;
    k_window_bounds_search<<<static_cast<unsigned>(blocks), kSearchWarps * 32, 0, s>>>(
        d_arrival, n, window_ms, w0, n_windows, d_bounds, zero_words, n_zero);
    return;
  }
  const int64_t warps = n / (32 * kBoundsTile) + 1;
  const int64_t blocks = (warps + 7) / 8;
  k_window_bounds<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), 256, 0, s>>>(
      d_arrival, n, window_ms, w0, n_windows, d_bounds, zero_words, n_zero);
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
  int32_t lwarp[kRouteWarps];  // non-empty list: per-warp counts, the CTA's prefix, the epoch
  long long lexcl;
  unsigned lepoch;
  int32_t lpos[K];             // list position of cell k relative to lexcl (-1: empty)
};

// Optional output of K1b: the ascending list of non-empty cells (count > 0) for K2, built in
// the same pass by the decoupled look-back (gsb::lookback_prefix) over the CTAs in launch
// order (CTA b owns cells [b*G*C, (b+1)*G*C), so CTA order is cell order).
constexpr long long kChunk = 128;  // list positions per K2 chunk (the fused pass's readiness unit)

struct ListOut {
  uint32_t* list;            // [cells] (NULL: no list)
  int64_t* n_list;
  double* t_ref;             // optional [P][cap]: t_ref in list order
  double* min_deadline;      // optional [cap]
  int64_t cap;
  gsb::CompactHdr* hdr;
  unsigned long long* status;  // [tiles]
  unsigned* ready;           // fused pass only: entries written per chunk of kChunk positions
  unsigned* nl_known;        // fused pass only: set once *n_list is final
};

// One K1b tile (windows [tile*G, tile*G + G)), run by all threads of a CTA whose s.bar was
// initialised (parity: the barrier's phase, carried across the tiles of a persistent CTA).
template <int C, int P, bool DL, int GW>
__device__ __forceinline__ void route_bin_tile(
    const RouteParams& rp, const int64_t* __restrict__ arrival, const int32_t* __restrict__ prompt,
    const int64_t* __restrict__ bounds, uint8_t* __restrict__ cls_out,
    uint32_t* __restrict__ count, double* __restrict__ t_ref, double* __restrict__ min_deadline,
    const ListOut& lo, RouteSmem<GW * C, DL>& s, unsigned tile, unsigned n_tiles,
    uint32_t& parity) {
  constexpr int G = GW, K = G * C, E = (K + 31) / 32, NW = kRouteWarps;
  constexpr int kNever = 0x3fffffff;
  using S = RouteSmem<K, DL>;
  const int tid = threadIdx.x, wib = tid >> 5, lane = tid & 31;
  const unsigned lt = lanemask_lt();
  int32_t th[GSB_MAX_CLASSES - 1];
#pragma unroll
  for (int k = 0; k < GSB_MAX_CLASSES - 1; ++k) th[k] = rp.thr[k];
  const int64_t w_first = static_cast<int64_t>(tile) * G;
  for (int k = tid; k <= G; k += NW * 32) s.bnd[k] = bounds[min(w_first + k, rp.n_windows)];
  for (int k = tid; k < K; k += NW * 32) {
    s.cnt[k] = 0;
    if (DL) s.mdl[k] = ~0ull;
  }
  unsigned epoch = 0;  // read now, used in the epilogue (the load's latency hides behind the pass)
  if (tid == 0 && lo.list) epoch = __ldcg(&lo.hdr->epoch);
  __syncthreads();
  const int64_t b0 = s.bnd[0], bG = s.bnd[G];
  const bool tma = !rp.prompt_host && (reinterpret_cast<uintptr_t>(prompt) & 15) == 0;
  // fold role: lane (fg, fp) = (window, profile)
  const int fg = lane / P, fp = lane - (lane / P) * P;
  const bool folder = lane < G * P;
  const double la = rp.lat_a[fp], lb = rp.lat_b[fp], lc = rp.lat_c[fp];
  constexpr int CPW = (C + NW - 1) / NW;  // classes per warp in the fold: c = wib + k * NW
  // (a class -> warp map rotated by tile, to spread a skewed mix's populated classes over the
  // SM sub-partitions, measured 4 us slower at C4: 33.3 vs 29.3 us)
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
#pragma unroll 8
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
        // the key group's leader takes the group's slots with one shared-memory atomic and
        // hands the base to the group (no read-modify-write of the histogram across the warp)
        const int leader = __ffs(static_cast<int>(m)) - 1;
        int base = 0;
        if (valid && below == 0) base = atomicAdd(&hist_w[key], __popc(m));
        base = __shfl_sync(kFull, base, leader);
        if (valid) {
          *cls_p = static_cast<uint8_t>(cl);
          s.kr[j] = static_cast<typename S::KR>(key | ((base + __popc(below)) << S::kKeyBits));
          if (DL) {
            const double ttft = L <= rp.slo_boundary ? rp.ttft_sm : rp.ttft_l;
            const double dl = static_cast<double>(__ldg(arrival + c0 + j)) + ttft - rp.allowance;
            if (dl == dl) atomicMin(&s.mdl[key], ord_f64(dl));
          }
        }
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
      if (lo.list && c1 == bG) {
        // the counts are final after the last chunk's scan: publish this tile's non-empty cell
        // count NOW, before the fold, so that successors' look-backs rarely wait on this tile
        int ne = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int k = lane * E + e;
          ne += (k < K && w_first + k / C < rp.n_windows && s.cnt[k] != 0) ? 1 : 0;
        }
        ne = __reduce_add_sync(kFull, static_cast<unsigned>(ne));
        if (lane == 0) gsb::lookback_publish(lo.status, tile, epoch, ne);  // lane 0 = tid 0
      }
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
  if (lo.list) {  // this CTA's non-empty cells, in cell order, at their global list positions
    constexpr int KT = (K + NW * 32 - 1) / (NW * 32);  // consecutive cells per thread
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      const int k = tid * KT + j;
      if (k < K && w_first + k / C < rp.n_windows && s.cnt[k] != 0) m |= 1u << j;
    }
    const int c = __popc(m);
    int incl = c;  // (this thread's cells' positions: below, once the warp prefix is known)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s.lwarp[wib] = incl;
    if (tid == 0) s.lepoch = epoch;
    __syncthreads();
    int wbase = 0, agg = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      wbase += k < wib ? s.lwarp[k] : 0;
      agg += s.lwarp[k];
    }
    if (wib == 0) {  // (the tile count was published after the last chunk's scan)
      const long long excl = gsb::lookback_prefix(lo.status, tile, s.lepoch, agg,
                                                  /*published=*/b0 < bG);
      if (lane == 0) s.lexcl = excl;
    }
    __syncthreads();
    int rel = wbase + incl - c;
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      const int k = tid * KT + j;
      if (k >= K) break;
      const bool ne = (m >> j) & 1u;
      s.lpos[k] = ne ? rel : -1;
      if (ne) {
        lo.list[s.lexcl + rel] = static_cast<uint32_t>(w_first * C + k);
        if (DL && lo.min_deadline) {
          const unsigned long long v = s.mdl[DL ? k : 0];
          lo.min_deadline[s.lexcl + rel] = v == ~0ull ? INFINITY : unord_f64(v);
        }
        ++rel;
      }
    }
    if (lo.t_ref) {  // the fold lanes' T_ref, in list order
      __syncthreads();
      if (folder && w_first + fg < rp.n_windows) {
#pragma unroll
        for (int k = 0; k < CPW; ++k) {
          const int c = wib + k * NW;
          if (c >= C) continue;
          const int r = s.lpos[fg * C + c];
          if (r >= 0) lo.t_ref[fp * lo.cap + s.lexcl + r] = acc[k];
        }
      }
    }
    if (lo.ready) __threadfence();  // this thread's list entries before the chunk counters
    __syncthreads();
    if (tid == 0) {
      if (lo.ready && agg > 0) {  // the fused pass: count this tile's entries into their chunks
        const long long e0 = s.lexcl, e1 = s.lexcl + agg;
        for (long long ch = e0 / kChunk; ch * kChunk < e1; ++ch) {
          const long long lo_ = max(e0, ch * kChunk), hi_ = min(e1, (ch + 1) * kChunk);
          atomicAdd(lo.ready + ch, static_cast<unsigned>(hi_ - lo_));
        }
      }
      if (tile == n_tiles - 1) {
        *lo.n_list = s.lexcl + agg;
        if (lo.ready) {
          __threadfence();
          atomicExch(lo.nl_known, 1u);
        }
        gsb::lookback_finish(lo.hdr, s.lepoch);
      }
    }
  }
  __syncthreads();  // the next tile of a persistent CTA reuses the shared memory
}

template <int C, int P, bool DL, int GW>
__global__ void __launch_bounds__(kRouteWarps * 32, GW * C > 64 ? 6 : kRouteMinBlocks)
k_route_bin(const __grid_constant__ RouteParams rp, const int64_t* __restrict__ arrival,
            const int32_t* __restrict__ prompt, const int64_t* __restrict__ bounds,
            uint8_t* __restrict__ cls_out, uint32_t* __restrict__ count,
            double* __restrict__ t_ref, double* __restrict__ min_deadline, ListOut lo) {
  using S = RouteSmem<GW * C, DL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& s = *reinterpret_cast<S*>(smem_raw);
  gsb::grid_dep_wait();  // K1a's bounds (programmatic dependent launch)
  gsb::grid_dep_launch();
  if (threadIdx.x == 0) gsb::mbar_init(&s.bar, 1);
  __syncthreads();
  uint32_t parity = 0;
  route_bin_tile<C, P, DL, GW>(rp, arrival, prompt, bounds, cls_out, count, t_ref, min_deadline,
                               lo, s, blockIdx.x, gridDim.x, parity);
}

// ---------------------------------------------------------------- the fused prefill pass
// K1b and K2 in ONE persistent kernel (gsb_prefill_pass): every CTA first takes K1b tiles by
// ticket (route, bin, ordered T_ref fold, list entries by look-back) and, once no tile is left,
// K2 chunks (128 listed cells x one profile) in list order, each as soon as the tiles that
// write its entries have counted them in (per-chunk readiness counters). The FP64-bound scan of
// the early chunks so runs beside the issue-bound routing of the late tiles on the same SMs, and
// neither kernel boundary nor one-wave ramp/tail separates the two halves. Forward progress:
// every tile is taken by a running CTA before any CTA waits on a chunk, and a tile waits only on
// lower tiles (look-back).
struct PassHdr {
  unsigned tile_ticket, chunk_ticket, pad0, pad1;
};

struct PassK2 {
  gsb_k2::SelectParams sp;
  double* window;
  int16_t* f_idx;
  double* energy;
  PassHdr* ph;
};

template <int C, int P, bool DL, int GW>
__global__ void __launch_bounds__(kRouteWarps * 32, GW * C > 64 ? 6 : kRouteMinBlocks)
k_prefill_pass(const __grid_constant__ RouteParams rp, const __grid_constant__ gsb_k2::ClockSet<81> cs,
               const int64_t* __restrict__ arrival, const int32_t* __restrict__ prompt,
               const int64_t* __restrict__ bounds, uint8_t* __restrict__ cls_out,
               uint32_t* __restrict__ count, double* __restrict__ t_ref,
               double* __restrict__ min_deadline, ListOut lo, PassK2 pk) {
  using S = RouteSmem<GW * C, DL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& s = *reinterpret_cast<S*>(smem_raw);
  __shared__ unsigned s_work;
  __shared__ int s_avail;
  const int tid = threadIdx.x;
  gsb::grid_dep_wait();  // K1a's bounds and zeroed counters
  gsb::grid_dep_launch();
  if (tid == 0) gsb::mbar_init(&s.bar, 1);
  __syncthreads();
  uint32_t parity = 0;
  const unsigned n_tiles = static_cast<unsigned>((rp.n_windows + GW - 1) / GW);
  for (;;) {  // ---- K1b tiles
    if (tid == 0) s_work = atomicAdd(&pk.ph->tile_ticket, 1u);
    __syncthreads();
    const unsigned t = s_work;
    __syncthreads();
    if (t >= n_tiles) break;
    route_bin_tile<C, P, DL, GW>(rp, arrival, prompt, bounds, cls_out, count, t_ref,
                                 min_deadline, lo, s, t, n_tiles, parity);
  }
  const gsb_k2::SelectParams& sp = pk.sp;
  const int64_t n = sp.n_cells;
  for (;;) {  // ---- K2 chunks, list order (chunk-major, profile-minor)
    if (tid == 0) {
      const unsigned c = atomicAdd(&pk.ph->chunk_ticket, 1u);
      const long long ch = c / P;
      int avail = -1;
      if (ch * kChunk < n) {
        const volatile unsigned* rd = lo.ready + ch;
        for (;;) {
          const unsigned r = *rd;
          if (r == kChunk) {
            avail = static_cast<int>(kChunk);
            break;
          }
          if (*reinterpret_cast<volatile unsigned*>(lo.nl_known)) {
            const long long nl = *reinterpret_cast<volatile long long*>(lo.n_list);
            if (ch * kChunk >= nl) break;  // past the end of the list
            if (r == static_cast<unsigned>(nl - ch * kChunk)) {
              avail = static_cast<int>(r);
              break;
            }
          }
          __nanosleep(64);
        }
        __threadfence();  // acquire: the entries the counter covers
      }
      s_work = c;
      s_avail = avail;
    }
    __syncthreads();
    const unsigned c = s_work;
    const int avail = s_avail;
    __syncthreads();
    if (avail < 0) break;
    if (tid >= avail) continue;
    const int p = static_cast<int>(c % P);
    const long long k = static_cast<long long>(c / P) * kChunk + tid;
    const int64_t cell = __ldcg(lo.list + k);
    const double T = __ldcg(lo.t_ref + p * lo.cap + k);
    double W;
    if (sp.mode == GSB_FIXED_WINDOW) {
      W = sp.fixed_window;
    } else {  // GSB_DEADLINE_SLACK (the pass takes FIXED or DEADLINE_SLACK)
      const double mdl = __ldcg(lo.min_deadline + k);
      const double now = static_cast<double>((sp.w0 + cell / sp.C) * sp.window_ms);
      W = gsb::std_max(sp.margin * (mdl - now), sp.min_budget);
    }
    if (p == 0 && pk.window) pk.window[cell] = W;
    double be;
    int best;
    switch (p) {
      case 0: best = gsb_k2::scan_clocks_c<81, 0>(cs, T, W, &be); break;
      case 1: best = gsb_k2::scan_clocks_c<81, 1>(cs, T, W, &be); break;
      case 2: best = gsb_k2::scan_clocks_c<81, 2>(cs, T, W, &be); break;
      default: best = gsb_k2::scan_clocks_c<81, 3>(cs, T, W, &be); break;
    }
    const int64_t o = p * n + cell;
    pk.f_idx[o] = static_cast<int16_t>(best);
    pk.energy[o] = best >= 0 ? be : 0.0;
  }
}

template <int C, int P, bool DL, int G>
int launch_pass_g(gsb_ctx* ctx, const RouteParams& rp, const gsb_k2::ClockSet<81>& cs,
                  const int64_t* d_arrival, const int32_t* d_prompt, const int64_t* d_bounds,
                  uint8_t* d_class, uint32_t* d_count, double* d_t_ref, double* d_min_deadline,
                  const ListOut& lo, const PassK2& pk, cudaStream_t s) {
  const size_t smem = sizeof(RouteSmem<G * C, DL>);
  auto kern = k_prefill_pass<C, P, DL, G>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRouteWarps * 32, smem) !=
          cudaSuccess || per_sm < 1)
    return -1;
  // persistent: every CTA resident (the chunk waits rely on it)
  const unsigned blocks = static_cast<unsigned>(per_sm * ctx->n_sms);
  if (gsb::launch_pdl(kern, dim3(blocks), dim3(kRouteWarps * 32), smem, s, rp, cs, d_arrival,
                      d_prompt, d_bounds, d_class, d_count, d_t_ref, d_min_deadline, lo,
                      pk) != cudaSuccess)
    return -1;
  return 0;
}

template <int C, int P, bool DL>
int launch_pass(gsb_ctx* ctx, const RouteParams& rp, int64_t n_req,
                const gsb_k2::ClockSet<81>& cs, const int64_t* d_arrival, const int32_t* d_prompt,
                const int64_t* d_bounds, uint8_t* d_class, uint32_t* d_count, double* d_t_ref,
                double* d_min_deadline, const ListOut& lo, const PassK2& pk, cudaStream_t s) {
  if constexpr (P == 1) {
    if (n_req > rp.n_windows * (kRouteCap / 32))
      return launch_pass_g<C, P, DL, 8>(ctx, rp, cs, d_arrival, d_prompt, d_bounds, d_class,
                                        d_count, d_t_ref, d_min_deadline, lo, pk, s);
  }
  return launch_pass_g<C, P, DL, 32 / P>(ctx, rp, cs, d_arrival, d_prompt, d_bounds, d_class,
                                         d_count, d_t_ref, d_min_deadline, lo, pk, s);
}

template <int C, int P, bool DL, int G>
int launch_route_bin_g(const RouteParams& rp, const int64_t* d_arrival, const int32_t* d_prompt,
                       const int64_t* d_bounds, uint8_t* d_class, uint32_t* d_count,
                       double* d_t_ref, double* d_min_deadline, const ListOut& lo, cudaStream_t s) {
  const size_t smem = sizeof(RouteSmem<G * C, DL>);
  if (cudaFuncSetAttribute(k_route_bin<C, P, DL, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return -1;
  const unsigned blocks = static_cast<unsigned>((rp.n_windows + G - 1) / G);
  if (gsb::launch_pdl(k_route_bin<C, P, DL, G>, dim3(blocks), dim3(kRouteWarps * 32), smem, s, rp,
                      d_arrival, d_prompt, d_bounds, d_class, d_count, d_t_ref,
                      d_min_deadline, lo) != cudaSuccess)
    return -1;
  return 0;
}

// G = 32 / P windows per CTA (lanes (window, profile) fill the fold warp). With one profile and
// dense windows (32 windows would not fit one chunk) G = 8: four times the CTAs, one chunk each,
// for small traces that would otherwise run a few long CTAs (fold lanes are cheap at P = 1).
template <int C, int P, bool DL>
int launch_route_bin(const RouteParams& rp, int64_t n_req, const int64_t* d_arrival,
                     const int32_t* d_prompt, const int64_t* d_bounds, uint8_t* d_class,
                     uint32_t* d_count, double* d_t_ref, double* d_min_deadline,
                     const ListOut& lo, cudaStream_t s) {
  if constexpr (P == 1) {
    if (n_req > rp.n_windows * (kRouteCap / 32))
      return launch_route_bin_g<C, P, DL, 8>(rp, d_arrival, d_prompt, d_bounds, d_class, d_count,
                                             d_t_ref, d_min_deadline, lo, s);
  }
  return launch_route_bin_g<C, P, DL, 32 / P>(rp, d_arrival, d_prompt, d_bounds, d_class, d_count,
                                              d_t_ref, d_min_deadline, lo, s);
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

int gsb_window_bounds(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req,
                      const int64_t* d_arrival, int64_t* d_bounds, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  int rc = check_route_cfg(ctx, cfg);
  if (rc) return rc;
  launch_window_bounds(d_arrival, n_req, cfg->window_ms, cfg->w0, cfg->n_windows, d_bounds,
                       nullptr, 0, gsb_pick_stream(ctx, stream));
  return gsb_check_launch(ctx, "window_bounds");
}

int gsb_route_bin(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req, const int64_t* d_arrival,
                  const int32_t* d_prompt, const int64_t* d_bounds, uint8_t* d_class,
                  uint32_t* d_count, double* d_t_ref, double* d_min_deadline, void* stream) {
  return gsb_route_bin_list(ctx, cfg, n_req, d_arrival, d_prompt, d_bounds, d_class, d_count,
                            d_t_ref, d_min_deadline, nullptr, stream);
}

int gsb_route_bin_list(gsb_ctx* ctx, const gsb_route_cfg* cfg, int64_t n_req,
                       const int64_t* d_arrival, const int32_t* d_prompt, const int64_t* d_bounds,
                       uint8_t* d_class, uint32_t* d_count, double* d_t_ref,
                       double* d_min_deadline, const gsb_cell_list* list, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  int rc = check_route_cfg(ctx, cfg);
  if (rc) return rc;
  if (ctx->n_profiles < 1) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "route: no profiles set");
  ListOut lo{};
  if (list && list->d_cells) {
    const int C = cfg->enabled ? cfg->n_thresholds + 1 : 1;
    const int64_t cells = cfg->n_windows * C;
    if (!list->d_n || cells >= (int64_t{1} << 32) || list->capacity < cells)
      return gsb_set_error(ctx, GSB_INVALID_ARGUMENT,
                           "route: list needs d_n, capacity >= cells and < 2^32 cells");
    // K1b CTAs own >= 8 windows each: one look-back status per CTA after the 256-byte header
    char* sy = static_cast<char*>(gsb_sync_words(
        ctx, 256 + sizeof(unsigned long long) * static_cast<size_t>(cfg->n_windows / 8 + 2)));
    if (!sy) return gsb_set_error(ctx, GSB_CUDA_ERROR, "route: sync allocation failed");
    lo = ListOut{list->d_cells, list->d_n, list->d_t_ref,
                 d_min_deadline ? list->d_min_deadline : nullptr, list->capacity,
                 reinterpret_cast<gsb::CompactHdr*>(sy),
                 reinterpret_cast<unsigned long long*>(sy + 256), nullptr, nullptr};
  }
  RouteParams rp = make_route_params(ctx, cfg);
  rp.prompt_host = is_host_ptr(d_prompt) ? 1 : 0;
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
                                          d_count, d_t_ref, d_min_deadline, lo, s);            \
    break;                                                                                      \
  case ((CC)-1) * 8 + ((PP)-1) * 2 + 1:                                                        \
    lrc = launch_route_bin<CC, PP, true>(rp, n_req, d_arrival, d_prompt, d_bounds, d_class,    \
                                         d_count, d_t_ref, d_min_deadline, lo, s);             \
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

int gsb_prefill_pass(gsb_ctx* ctx, const gsb_route_cfg* rcfg, int64_t n_req,
                     const int64_t* d_arrival, const int32_t* d_prompt, int64_t* d_bounds,
                     uint8_t* d_class, uint32_t* d_count, double* d_t_ref,
                     double* d_min_deadline, const gsb_cell_list* list,
                     const gsb_select_cfg* scfg, double* d_window, int16_t* d_f_idx,
                     double* d_energy, gsb_class_summary* d_summary, void* stream) {
  if (!ctx || !scfg || !list) return GSB_INVALID_ARGUMENT;
  int rc = check_route_cfg(ctx, rcfg);
  if (rc) return rc;
  if (ctx->n_profiles < 1) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "pass: no profiles set");
  const int C = rcfg->enabled ? rcfg->n_thresholds + 1 : 1;
  const int64_t cells = rcfg->n_windows * C;
  const bool dl = scfg->mode == GSB_DEADLINE_SLACK;
  if (scfg->mode != GSB_FIXED_WINDOW && !dl)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "pass: FIXED_WINDOW or DEADLINE_SLACK only");
  if (!list->d_cells || !list->d_n || !list->d_t_ref || list->capacity < cells ||
      cells >= (int64_t{1} << 32) || (dl && (!d_min_deadline || !list->d_min_deadline)))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT,
                         "pass: needs a full cell list (cells, n, t_ref, min_deadline when "
                         "DEADLINE_SLACK) and < 2^32 cells");
  if (d_summary && scfg->n_classes != C)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "pass: summary needs n_classes = C");
  gsb_k2::ClockSet<81> cs{};
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  if (!gsb_k2::make_clockset81(ctx, &cs)) {  // generic grids: the two-call path
    rc = gsb_window_bounds(ctx, rcfg, n_req, d_arrival, d_bounds, stream);
    if (!rc)
      rc = gsb_route_bin_list(ctx, rcfg, n_req, d_arrival, d_prompt, d_bounds, d_class, d_count,
                              d_t_ref, dl ? d_min_deadline : nullptr, list, stream);
    if (!rc)
      rc = gsb_prefill_select_list(ctx, scfg, cells, d_t_ref, d_count, list,
                                   dl ? d_min_deadline : nullptr, d_window, d_f_idx, d_energy,
                                   d_summary, stream);
    return rc;
  }
  // sync words: [0,256) look-back header, [256,512) pass header, the per-chunk readiness
  // counters, then the look-back statuses (one per K1b tile, tiles own >= 8 windows)
  const int64_t max_chunks = (cells + kChunk - 1) / kChunk;
  const size_t o_rd = 512, o_st = (o_rd + sizeof(unsigned) * max_chunks + 255) & ~size_t{255};
  char* sy = static_cast<char*>(gsb_sync_words(
      ctx, o_st + sizeof(unsigned long long) * static_cast<size_t>(rcfg->n_windows / 8 + 2)));
  if (!sy) return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass: sync allocation failed");
  PassHdr* ph = reinterpret_cast<PassHdr*>(sy + 256);
  unsigned* ready = reinterpret_cast<unsigned*>(sy + o_rd);
  // K1a (window bounds), which also zeroes the pass header and the readiness counters
  launch_window_bounds(d_arrival, n_req, rcfg->window_ms, rcfg->w0, rcfg->n_windows, d_bounds,
                       reinterpret_cast<unsigned*>(ph),
                       static_cast<int64_t>((o_st - 256) / sizeof(unsigned)), s);
  RouteParams rp = make_route_params(ctx, rcfg);
  rp.prompt_host = is_host_ptr(d_prompt) ? 1 : 0;
  rp.want_deadline = dl ? 1 : 0;
  const ListOut lo{list->d_cells, list->d_n, list->d_t_ref, dl ? list->d_min_deadline : nullptr,
                   list->capacity, reinterpret_cast<gsb::CompactHdr*>(sy),
                   reinterpret_cast<unsigned long long*>(sy + o_st), ready, &ph->pad0};
  PassK2 pk{};
  pk.sp.mode = scfg->mode;
  pk.sp.C = C;
  pk.sp.fixed_window = scfg->fixed_window_ms;
  pk.sp.w0 = rcfg->w0;
  pk.sp.window_ms = rcfg->window_ms;
  pk.sp.margin = scfg->qopt.margin_prefill;
  pk.sp.min_budget = scfg->qopt.min_budget_ms;
  pk.sp.n_cells = cells;
  pk.window = d_window;
  pk.f_idx = d_f_idx;
  pk.energy = d_energy;
  pk.ph = ph;
  const int P = ctx->n_profiles;
  const int key = (C - 1) * 8 + (P - 1) * 2 + (dl ? 1 : 0);
  int lrc = 0;
  double* mdl = dl ? d_min_deadline : nullptr;
  switch (key) {
#define GSB_PS(CC, PP)                                                                           \
  case ((CC)-1) * 8 + ((PP)-1) * 2:                                                             \
    lrc = launch_pass<CC, PP, false>(ctx, rp, n_req, cs, d_arrival, d_prompt, d_bounds, d_class, \
                                     d_count, d_t_ref, mdl, lo, pk, s);                         \
    break;                                                                                       \
  case ((CC)-1) * 8 + ((PP)-1) * 2 + 1:                                                         \
    lrc = launch_pass<CC, PP, true>(ctx, rp, n_req, cs, d_arrival, d_prompt, d_bounds, d_class,  \
                                    d_count, d_t_ref, mdl, lo, pk, s);                          \
    break;
#define GSB_PS_P(CC) GSB_PS(CC, 1) GSB_PS(CC, 2) GSB_PS(CC, 3) GSB_PS(CC, 4)
    GSB_PS_P(1) GSB_PS_P(2) GSB_PS_P(3) GSB_PS_P(4) GSB_PS_P(5) GSB_PS_P(6) GSB_PS_P(7) GSB_PS_P(8)
#undef GSB_PS_P
#undef GSB_PS
    default:
      return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "pass: need 1..8 classes, 1..4 profiles");
  }
  if (lrc) return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass: launch configuration refused");
  rc = gsb_check_launch(ctx, "prefill_pass");
  if (rc) return rc;
  return gsb_internal_finish(ctx, P, C, cells, d_count, d_f_idx, d_energy, d_summary, s);
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


// The offline pass from HOST buffers, pipelined over window chunks (include/gsb.h). PCIe is
// full duplex and the copy engines are separate from the SMs, so chunk k's prompt upload (up
// stream), its K1b / K2 / finish / summary (a compute stream) and its read-back (down stream)
// overlap the neighbouring chunks' work. K1a' (latency-bound probes of the pinned arrivals over
// PCIe) runs once, up front, on a fourth stream beside the first uploads. A chunk's small K1b / K2 grids are
// latency-bound and fill a fraction of the GPU, so consecutive chunks run on two alternating
// compute streams, each chunk with its own look-back sync words and summary scratch (swapped
// into the context while its kernels are enqueued; the context's own are untouched). Every chunk is an independent pass over
// windows [a_k, a_k+1) and their requests [r_k, r_k+1) (found by a host lower_bound over the
// pinned arrivals, the same values as the device bounds), with its own device buffers.
int gsb_prefill_pass_host(gsb_ctx* ctx, const gsb_route_cfg* rcfg, int64_t n_req,
                          const int64_t* h_arrival, const int32_t* h_prompt,
                          const gsb_select_cfg* scfg, int n_chunks, int16_t* h_f_idx,
                          double* h_energy, gsb_class_summary* h_summary, void* stream) {
  if (!ctx || !scfg || !h_f_idx || !h_energy || n_req < 0 || (n_req > 0 && (!h_arrival || !h_prompt)))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "pass_host: null or negative argument");
  int rc = check_route_cfg(ctx, rcfg);
  if (rc) return rc;
  if (scfg->mode != GSB_FIXED_WINDOW && scfg->mode != GSB_DEADLINE_SLACK)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "pass_host: mode must be FIXED_WINDOW or DEADLINE_SLACK");
  if (n_chunks < 1 || n_chunks > 64 || n_chunks > rcfg->n_windows)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT,
                         "pass_host: n_chunks must be in [1, min(64, n_windows)]");
  if (ctx->n_profiles < 1) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "pass_host: no profiles set");
  const int64_t nW = rcfg->n_windows, W = rcfg->window_ms;
  const int C = rcfg->enabled ? rcfg->n_thresholds + 1 : 1, P = ctx->n_profiles;
  const int64_t cells = nW * C;
  const int K = n_chunks;
  if (scfg->n_classes != C)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "pass_host: scfg->n_classes != classes of rcfg");
  const bool dl = scfg->mode == GSB_DEADLINE_SLACK;
  // chunk k: windows [a[k], a[k+1]), requests [r[k], r[k+1]) = those with arrival in
  // [(w0 + a[k]) W, (w0 + a[k+1]) W): lower_bound over the sorted host arrivals
  std::vector<int64_t> a(K + 1), r(K + 1);
  // decreasing chunk sizes (weights K, K-1, ..., 1): the last chunk's kernels and read-back,
  // which nothing overlaps, are the smallest
  const int64_t wsum = static_cast<int64_t>(K) * (K + 1) / 2;
  int64_t acc = 0;
  for (int k = 0; k <= K; ++k) {
    a[k] = nW * acc / wsum;
    if (k < K) acc += K - k;
    const int64_t T = (rcfg->w0 + a[k]) * W;
    r[k] = std::lower_bound(h_arrival, h_arrival + n_req, T) - h_arrival;
  }
  // device layout: the per-chunk sync words (zeroed once, at allocation), the prompts, then
  // per chunk its own buffers (256-byte aligned)
  auto al = [](size_t b) { return (b + 255) & ~size_t{255}; };
  std::vector<size_t> off(K + 1), sync_off(K), scr_off(K);
  std::vector<size_t> sync_b(K), scr_b(K);
  size_t bytes = 0;
  for (int k = 0; k < K; ++k) {
    const int64_t wk = a[k + 1] - a[k];
    sync_b[k] = al(256 + sizeof(unsigned long long) * static_cast<size_t>(wk / 8 + 2));
    sync_off[k] = bytes;
    bytes += sync_b[k];
  }
  const size_t sync_total = bytes;
  bytes += al(sizeof(int32_t) * std::max<int64_t>(n_req, 1));
  const size_t bounds_off = bytes;
  bytes += al(sizeof(int64_t) * (nW + 1));
  const size_t class_off = bytes;
  bytes += al(std::max<int64_t>(n_req, 1));
  const size_t summ_b = sizeof(gsb_class_summary) * P * C;
  for (int k = 0; k < K; ++k) {
    off[k] = bytes;
    const int64_t nk = r[k + 1] - r[k], wk = a[k + 1] - a[k], ck = wk * C;
    (void)nk;
    bytes += al(4 * ck) + 2 * al(8 * P * ck) + al(4 * ck) + al(8) + al(2 * P * ck) +
             al(8 * P * ck) + al(summ_b) + (dl ? 2 * al(8 * ck) : 0);
    scr_b[k] = al(gsb_finish_scratch_bytes(P, C, std::max<int64_t>(ck, 1)));
    scr_off[k] = bytes;
    bytes += scr_b[k];
  }
  // the sync words' layout depends on the chunk split: a call with another split re-zeroes
  const bool new_split = ctx->hostpass_bytes < bytes || ctx->hp_sync_total != sync_total ||
                         ctx->hp_chunks != K;
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  if (bytes > ctx->hostpass_bytes) {  // grow: nothing of an earlier call may still use the old one
    if (ctx->d_hostpass) {
      cudaStreamSynchronize(s);
      if (ctx->up_stream) cudaStreamSynchronize(ctx->up_stream);
      if (ctx->down_stream) cudaStreamSynchronize(ctx->down_stream);
      cudaFree(ctx->d_hostpass);
      ctx->d_hostpass = nullptr;
      ctx->hostpass_bytes = 0;
    }
    if (cudaMalloc(&ctx->d_hostpass, bytes) != cudaSuccess) {
      cudaGetLastError();
      ctx->d_hostpass = nullptr;
      return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: device allocation failed");
    }
    ctx->hostpass_bytes = bytes;
  }
  if (new_split) {  // zero state for every chunk's look-back words (then stream-ordered reuse)
    if (cudaMemsetAsync(ctx->d_hostpass, 0, sync_total, s) != cudaSuccess)
      return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: sync-word reset failed");
    ctx->hp_sync_total = sync_total;
    ctx->hp_chunks = K;
  }
  if ((!ctx->up_stream && cudaStreamCreateWithFlags(&ctx->up_stream, cudaStreamNonBlocking) != cudaSuccess) ||
      (!ctx->down_stream && cudaStreamCreateWithFlags(&ctx->down_stream, cudaStreamNonBlocking) != cudaSuccess) ||
      (!ctx->search_stream && cudaStreamCreateWithFlags(&ctx->search_stream, cudaStreamNonBlocking) != cudaSuccess) ||
      (!ctx->compute2 && cudaStreamCreateWithFlags(&ctx->compute2, cudaStreamNonBlocking) != cudaSuccess))
    return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: stream creation failed");
  const size_t n_ev = 3 + 2 * static_cast<size_t>(K);
  while (ctx->hp_events.size() < n_ev) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: event creation failed");
    ctx->hp_events.push_back(e);
  }
  cudaEvent_t ev_start = ctx->hp_events[0], ev_end = ctx->hp_events[1];
  char* base = static_cast<char*>(ctx->d_hostpass);
  int32_t* d_prompt = reinterpret_cast<int32_t*>(base + sync_total);
  // the copies start after everything queued before this call on the caller's stream (an
  // earlier call's kernels may still read the same device buffers)
  if (cudaEventRecord(ev_start, s) != cudaSuccess ||
      cudaStreamWaitEvent(ctx->up_stream, ev_start, 0) != cudaSuccess ||
      cudaStreamWaitEvent(ctx->down_stream, ev_start, 0) != cudaSuccess ||
      cudaStreamWaitEvent(ctx->search_stream, ev_start, 0) != cudaSuccess ||
      cudaStreamWaitEvent(ctx->compute2, ev_start, 0) != cudaSuccess)
    return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: event ordering failed");
  // diagnostics (GSB_HP_TRACE=1): timing events per stage, printed after a synchronize
  const bool trace = std::getenv("GSB_HP_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> tev;
  auto mark = [&](const std::string& name, cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.emplace_back(name, e);
  };
  mark("start", s);
  // host-side cost of each call group (diagnostics: the host issues ~35 us of calls per chunk)
  using hclock = std::chrono::steady_clock;
  std::vector<std::pair<std::string, double>> hts;
  auto hmark = [&, t0 = hclock::now()](const std::string& name) {
    if (trace)
      hts.emplace_back(name, std::chrono::duration<double, std::micro>(hclock::now() - t0).count());
  };
  // K1a' once over the whole window range (the chunks use slices of one bounds array): a
  // search per chunk would keep its PCIe-latency-bound CTAs resident across the whole upload,
  // and K2's one-wave grid of a chunk cannot become resident beside them
  int64_t* d_bounds_all = reinterpret_cast<int64_t*>(base + bounds_off);
  uint8_t* d_class_all = reinterpret_cast<uint8_t*>(base + class_off);
  rc = gsb_window_bounds(ctx, rcfg, n_req, h_arrival, d_bounds_all, ctx->search_stream);
  if (rc) return rc;
  cudaEvent_t ev_search = ctx->hp_events[2 + 2 * K];
  if (cudaEventRecord(ev_search, ctx->search_stream) != cudaSuccess)
    return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: event record failed");
  mark("search", ctx->search_stream);
  hmark("search issued");
  for (int k = 0; k < K; ++k) {
    const int64_t nk = r[k + 1] - r[k], wk = a[k + 1] - a[k], ck = wk * C;
    cudaEvent_t ev_up = ctx->hp_events[2 + 2 * k], ev_done = ctx->hp_events[3 + 2 * k];
    if (nk > 0 && cudaMemcpyAsync(d_prompt + r[k], h_prompt + r[k], sizeof(int32_t) * nk,
                                  cudaMemcpyHostToDevice, ctx->up_stream) != cudaSuccess)
      return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: prompt upload failed");
    if (cudaEventRecord(ev_up, ctx->up_stream) != cudaSuccess)
      return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: event record failed");
    mark("upload" + std::to_string(k), ctx->up_stream);
    hmark("upload" + std::to_string(k) + " issued");
    char* q = base + off[k];
    auto take = [&](size_t b) { char* p0 = q; q += al(b); return p0; };
    uint32_t* d_count = reinterpret_cast<uint32_t*>(take(4 * ck));
    double* d_t_ref = reinterpret_cast<double*>(take(8 * P * ck));
    double* d_t_list = reinterpret_cast<double*>(take(8 * P * ck));
    uint32_t* d_list = reinterpret_cast<uint32_t*>(take(4 * ck));
    int64_t* d_nl = reinterpret_cast<int64_t*>(take(8));
    int16_t* d_fi = reinterpret_cast<int16_t*>(take(2 * P * ck));
    double* d_en = reinterpret_cast<double*>(take(8 * P * ck));
    gsb_class_summary* d_sm = reinterpret_cast<gsb_class_summary*>(take(summ_b));
    double* d_mdl = dl ? reinterpret_cast<double*>(take(8 * ck)) : nullptr;
    double* d_mdl_list = dl ? reinterpret_cast<double*>(take(8 * ck)) : nullptr;
    gsb_route_cfg cfg_k = *rcfg;
    cfg_k.w0 = rcfg->w0 + a[k];
    cfg_k.n_windows = wk;
    gsb_select_cfg sc_k = *scfg;
    sc_k.w0 = scfg->w0 + a[k];
    const gsb_cell_list list{d_list, d_nl, d_t_list, d_mdl_list, ck};
    cudaStream_t cs = (k & 1) ? ctx->compute2 : s;
    if (cudaStreamWaitEvent(cs, ev_search, 0) != cudaSuccess ||
        cudaStreamWaitEvent(cs, ev_up, 0) != cudaSuccess)
      rc = gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: event wait failed");
    mark("compute_begin" + std::to_string(k), cs);
    // the chunk's own look-back words and summary scratch, in place of the context's
    void* const sv_sync = ctx->d_sync;
    void* const sv_scr = ctx->d_scratch;
    const size_t sv_sync_b = ctx->sync_bytes, sv_scr_b = ctx->scratch_bytes;
    ctx->d_sync = base + sync_off[k];
    ctx->sync_bytes = sync_b[k];
    ctx->d_scratch = base + scr_off[k];
    ctx->scratch_bytes = scr_b[k];
    if (!rc)
      // absolute request indices: the full arrays and the chunk's slice of the bounds
      rc = gsb_route_bin_list(ctx, &cfg_k, n_req, h_arrival, d_prompt, d_bounds_all + a[k],
                              d_class_all, d_count, d_t_ref, d_mdl, &list, cs);
    hmark("route" + std::to_string(k) + " issued");
    if (!rc)
      rc = gsb_prefill_select_list(ctx, &sc_k, ck, d_t_ref, d_count, &list, d_mdl, nullptr, d_fi,
                                   d_en, h_summary ? d_sm : nullptr, cs);
    hmark("select" + std::to_string(k) + " issued");
    const bool swapped_ok = ctx->d_sync == base + sync_off[k] && ctx->d_scratch == base + scr_off[k];
    if (!swapped_ok) {  // a callee grew a buffer: keep the new one for gsb_ctx_destroy to free,
                        // and drop the chunk regions it retired (they belong to d_hostpass)
      auto& rs = ctx->retired_scratch;
      rs.erase(std::remove_if(rs.begin(), rs.end(), [&](void* v) {
                 return static_cast<char*>(v) >= base && static_cast<char*>(v) < base + bytes;
               }), rs.end());
      if (ctx->d_sync != base + sync_off[k]) rs.push_back(ctx->d_sync);
      if (ctx->d_scratch != base + scr_off[k]) rs.push_back(ctx->d_scratch);
    }
    ctx->d_sync = sv_sync;
    ctx->sync_bytes = sv_sync_b;
    ctx->d_scratch = sv_scr;
    ctx->scratch_bytes = sv_scr_b;
    if (!rc && !swapped_ok)  // a callee outgrew the chunk's workspace (sizing bug): fail loudly
      rc = gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: chunk workspace outgrown");
    if (rc) return rc;
    // the read-back of chunk k (its P rows into the [P][cells] host arrays) runs beside the
    // next chunk's upload and kernels
    mark("compute_end" + std::to_string(k), cs);
    if (cudaEventRecord(ev_done, cs) != cudaSuccess ||
        cudaStreamWaitEvent(ctx->down_stream, ev_done, 0) != cudaSuccess ||
        cudaMemcpy2DAsync(h_f_idx + a[k] * C, sizeof(int16_t) * cells, d_fi, sizeof(int16_t) * ck,
                          sizeof(int16_t) * ck, P, cudaMemcpyDeviceToHost, ctx->down_stream) != cudaSuccess ||
        cudaMemcpy2DAsync(h_energy + a[k] * C, sizeof(double) * cells, d_en, sizeof(double) * ck,
                          sizeof(double) * ck, P, cudaMemcpyDeviceToHost, ctx->down_stream) != cudaSuccess ||
        (h_summary && cudaMemcpyAsync(h_summary + static_cast<size_t>(k) * P * C, d_sm, summ_b,
                                      cudaMemcpyDeviceToHost, ctx->down_stream) != cudaSuccess))
      return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: read-back failed");
  }
  // the caller's stream covers the read-backs (the host outputs are valid after it syncs)
  mark("readback_end", ctx->down_stream);
  if (cudaEventRecord(ev_end, ctx->down_stream) != cudaSuccess ||
      cudaStreamWaitEvent(s, ev_end, 0) != cudaSuccess)
    return gsb_set_error(ctx, GSB_CUDA_ERROR, "pass_host: final join failed");
  if (trace) {
    cudaStreamSynchronize(s);
    for (auto& [name, e] : tev) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0].second, e);
      std::fprintf(stderr, "gsb_hp %-16s %8.1f us\n", name.c_str(), ms * 1e3);
    }
    for (auto& te : tev) cudaEventDestroy(te.second);
    for (auto& [name, us] : hts) std::fprintf(stderr, "gsb_hp host %-18s %8.1f us\n", name.c_str(), us);
  }
  return GSB_OK;
}

}  // extern "C"
