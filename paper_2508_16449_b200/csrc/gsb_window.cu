// gsb_window.cu — K3a: the decode controller's window statistics, as Sim's ticks see them.
//
//   TbtWindow (decode_ctl.cpp:120-128): ring of the last `cap` inter-token gaps, P95 by
//     nearest rank = sorted[ceil(0.95 n) - 1] (metrics.cpp:11-19), read at every fine tick.
//   TpsWindow (decode_ctl.cpp:113-118): token sum of step-end events with
//     t >= now - window, times 1000 / window, read at every coarse tick.
//
// Step-end telemetry at t <= tick time is recorded before the tick (event kind 2 sorts
// before ticks 5..7, simkernel.cpp:21-31,44-50). Both statistics at tick k are therefore a
// pure function of the telemetry prefix recorded before tick k: the window is the last
// min(cap, #gaps) gaps before the tick, and the TPS set is a time range of events. So the
// series is computed in PARALLEL ACROSS TICKS (no sequential ring walk): one warp per
// (stream, fine tick) selects the k-th largest of <= 256 gaps with an in-register tournament;
// one thread per (stream, coarse tick) sums its event range.
#include <cmath>
#include <vector>

#include "gsb_common.cuh"

namespace {

struct WinParams {
  int64_t n_streams;
  const int64_t* ev_off;
  const double* t_ms;
  const int32_t* tokens;
  const int64_t* gap_off;
  const double* gaps;
  int cap;
  double window_ms;  // TpsWindow span = coarse period (simkernel.cpp:229)
  const double* fine_t;
  int64_t n_fine;
  const double* coarse_t;
  int64_t n_coarse;
  uint8_t* fine_has;
  double* fine_p95;
  double* coarse_tps;
};

// first event index in [lo, hi) whose time is > tau (all events at <= tau are recorded)
__device__ __forceinline__ int64_t upper_event(const double* __restrict__ t, int64_t lo, int64_t hi,
                                               double tau) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (t[mid] <= tau)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// first event index in [lo, hi) whose time is NOT < thr (TpsWindow keeps t >= now - window)
__device__ __forceinline__ int64_t first_not_less(const double* __restrict__ t, int64_t lo,
                                                  int64_t hi, double thr) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (t[mid] < thr)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// order-preserving map double -> u64 (0 is reserved for "no element")
__device__ __forceinline__ uint64_t key_of(double x) {
  const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double val_of(uint64_t k) {
  const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(u));
}

__device__ __forceinline__ void cswap_desc(uint64_t& a, uint64_t& b) {
  const uint64_t hi = a > b ? a : b, lo = a > b ? b : a;
  a = hi;
  b = lo;
}

// 8-input sorting network (19 compare-exchanges), descending
__device__ __forceinline__ void sort8_desc(uint64_t (&k)[8]) {
  cswap_desc(k[0], k[2]); cswap_desc(k[1], k[3]); cswap_desc(k[4], k[6]); cswap_desc(k[5], k[7]);
  cswap_desc(k[0], k[4]); cswap_desc(k[1], k[5]); cswap_desc(k[2], k[6]); cswap_desc(k[3], k[7]);
  cswap_desc(k[0], k[1]); cswap_desc(k[2], k[3]); cswap_desc(k[4], k[5]); cswap_desc(k[6], k[7]);
  cswap_desc(k[2], k[4]); cswap_desc(k[3], k[5]);
  cswap_desc(k[1], k[4]); cswap_desc(k[3], k[6]);
  cswap_desc(k[1], k[2]); cswap_desc(k[3], k[4]); cswap_desc(k[5], k[6]);
}

// One warp per (stream, fine tick). The window is gaps [cnt - n, cnt) of the stream, n <=
// 256: lane l holds elements l, l+32, ..., sorts its 8 keys, then kth = n - rank + 1 rounds
// of "warp max of the lane heads, the lowest winning lane pops" return the rank-th smallest
// (k <= 13 for n <= 256), the same value std::sort + index gives.
__global__ void __launch_bounds__(256) k_tbt_p95(const __grid_constant__ WinParams a) {
  const int64_t wid = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= a.n_streams * a.n_fine) return;
  const int64_t s = wid / a.n_fine, k = wid - s * a.n_fine;
  const int64_t e0 = a.ev_off[s], e1 = a.ev_off[s + 1];
  const double tau = a.fine_t[k];
  int64_t e = 0;
  if (lane == 0) e = upper_event(a.t_ms, e0, e1, tau);
  e = __shfl_sync(0xffffffffu, e, 0);
  const int64_t cnt = a.gap_off[e], g0 = a.gap_off[e0];
  const int64_t total = cnt - g0;
  const int n = static_cast<int>(total < a.cap ? total : a.cap);
  const int64_t o = s * a.n_fine + k;
  if (n == 0) {
    if (lane == 0) {
      a.fine_has[o] = 0;
      a.fine_p95[o] = 0.0;
    }
    return;
  }
  const double* win = a.gaps + (cnt - n);
  uint64_t key[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int idx = lane + 32 * j;
    key[j] = idx < n ? key_of(win[idx]) : 0ull;
  }
  sort8_desc(key);
  const int rank = static_cast<int>(ceil(0.95 * static_cast<double>(n)));  // >= 1 for n >= 1
  const int kth = n - rank + 1;
  int head = 0;
  uint64_t best = 0;
  for (int r = 0; r < kth; ++r) {
    uint64_t cur = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) cur = head == j ? key[j] : cur;
    const unsigned hi = static_cast<unsigned>(cur >> 32), lo = static_cast<unsigned>(cur);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    const unsigned who = __ballot_sync(0xffffffffu, hi == mhi && lo == mlo);
    if (lane == __ffs(static_cast<int>(who)) - 1) ++head;
    best = (static_cast<uint64_t>(mhi) << 32) | mlo;
  }
  if (lane == 0) {
    a.fine_has[o] = 1;
    a.fine_p95[o] = val_of(best);
  }
}

// One thread per (stream, coarse tick): TpsWindow::tps, decode_ctl.cpp:113-118.
__global__ void k_tps(const __grid_constant__ WinParams a) {
  const int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (id >= a.n_streams * a.n_coarse) return;
  const int64_t s = id / a.n_coarse, k = id - s * a.n_coarse;
  const int64_t e0 = a.ev_off[s], e1 = a.ev_off[s + 1];
  const double now = a.coarse_t[k];
  const int64_t hi = upper_event(a.t_ms, e0, e1, now);
  const int64_t lo = first_not_less(a.t_ms, e0, hi, now - a.window_ms);
  int tokens = 0;
  for (int64_t j = lo; j < hi; ++j) tokens += a.tokens[j];
  a.coarse_tps[s * a.n_coarse + k] = tokens * 1000.0 / a.window_ms;
}

}  // namespace

extern "C" int gsb_window_series(gsb_ctx* ctx, const gsb_telemetry* tel, int tbt_capacity,
                                 double fine_period_ms, double coarse_period_ms, double t_end_ms,
                                 uint8_t* d_fine_has, double* d_fine_p95, double* d_coarse_tps,
                                 void* stream) {
  if (!ctx || !tel) return GSB_INVALID_ARGUMENT;
  if (tbt_capacity < 1 || tbt_capacity > GSB_MAX_TBT_WINDOW)
    return gsb_set_error(ctx, GSB_MODEL_ERROR, "decode ctl: tbt window must hold 1..256 samples");
  if (fine_period_ms <= 0 || coarse_period_ms <= 0)
    return gsb_set_error(ctx, GSB_MODEL_ERROR, "decode ctl: periods must be > 0");
  if (tel->n_streams <= 0) return GSB_OK;
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  // tick instants exactly as Sim re-schedules them: t_1 = period, t_{k+1} = t_k + period
  // (simkernel.cpp:243-248,450,457); cached on the device per (periods, horizon)
  if (!ctx->d_ticks || ctx->tick_key[0] != fine_period_ms || ctx->tick_key[1] != coarse_period_ms ||
      ctx->tick_key[2] != t_end_ms) {
    std::vector<double> h;
    for (double t = fine_period_ms; t <= t_end_ms; t = t + fine_period_ms) h.push_back(t);
    const int64_t nf = static_cast<int64_t>(h.size());
    for (double t = coarse_period_ms; t <= t_end_ms; t = t + coarse_period_ms) h.push_back(t);
    cudaStreamSynchronize(s);
    if (ctx->d_ticks) cudaFree(ctx->d_ticks);
    ctx->d_ticks = nullptr;
    if (cudaMalloc(&ctx->d_ticks, sizeof(double) * (h.size() + 1)) != cudaSuccess)
      return gsb_set_error(ctx, GSB_CUDA_ERROR, "window_series: tick buffer allocation failed");
    cudaMemcpy(ctx->d_ticks, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
    ctx->tick_key[0] = fine_period_ms;
    ctx->tick_key[1] = coarse_period_ms;
    ctx->tick_key[2] = t_end_ms;
    ctx->n_fine_ticks = nf;
    ctx->n_coarse_ticks = static_cast<int64_t>(h.size()) - nf;
  }
  WinParams wp{};
  wp.n_streams = tel->n_streams;
  wp.ev_off = tel->d_ev_off;
  wp.t_ms = tel->d_t_ms;
  wp.tokens = tel->d_tokens;
  wp.gap_off = tel->d_gap_off;
  wp.gaps = tel->d_gaps;
  wp.cap = tbt_capacity;
  wp.window_ms = coarse_period_ms;
  wp.fine_t = static_cast<const double*>(ctx->d_ticks);
  wp.n_fine = ctx->n_fine_ticks;
  wp.coarse_t = wp.fine_t + ctx->n_fine_ticks;
  wp.n_coarse = ctx->n_coarse_ticks;
  wp.fine_has = d_fine_has;
  wp.fine_p95 = d_fine_p95;
  wp.coarse_tps = d_coarse_tps;
  const int64_t warps = wp.n_streams * wp.n_fine;
  if (warps > 0) {
    k_tbt_p95<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, s>>>(wp);
    int rc = gsb_check_launch(ctx, "tbt_p95");
    if (rc) return rc;
  }
  const int64_t threads = wp.n_streams * wp.n_coarse;
  if (threads > 0) {
    k_tps<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(wp);
    return gsb_check_launch(ctx, "tps");
  }
  return GSB_OK;
}

// ---------------------------------------------------------------- batched quantile / TPS
namespace {

constexpr int kQMax = 4096;

// Sets larger than kQMax (the reference takes any size, metrics.cpp:11-19): the element of
// 0-based rank r = max(ceil(q n), 1) - 1 in ascending order, found by an 8-pass radix select
// (8-bit digits, most significant first) over order-preserving 64-bit keys of the doubles
// (negative: all bits flipped, else the sign bit set), each pass one read of the set. Ties
// (equal keys) are the same double, so the result is the value std::sort would put there.
__device__ __forceinline__ uint64_t q_key(double v) {
  const uint64_t u = static_cast<uint64_t>(__double_as_longlong(v));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ void quantile_radix_select(double q, const double* __restrict__ x, int64_t n,
                                      double* __restrict__ out) {
  __shared__ unsigned long long hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ long long s_k;
  const int64_t rank = static_cast<int64_t>(ceil(q * static_cast<double>(n)));
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_k = rank == 0 ? 0 : rank - 1;
  }
  uint64_t mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t k = q_key(x[i]);
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1ull);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long k = s_k;
      int b = 0;
      for (; b < 255; ++b) {
        const long long h = static_cast<long long>(hist[b]);
        if (k < h) break;
        k -= h;
      }
      s_k = k;
      s_prefix = prefix | (static_cast<uint64_t>(b) << shift);
    }
    mask |= 0xffull << shift;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint64_t k = s_prefix;
    const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    *out = __longlong_as_double(static_cast<long long>(u));
  }
}

// One CTA per set: stage <= 4096 samples in shared memory (padded with +inf to a power of two),
// bitonic sort, read sorted[ceil(q n) - 1] (rank 0 -> minimum), metrics.cpp:14-18.
__global__ void __launch_bounds__(256) k_quantile(double q, int64_t n_sets,
                                                  const int64_t* __restrict__ off,
                                                  const double* __restrict__ x,
                                                  double* __restrict__ out) {
  __shared__ double s[kQMax];
  const int64_t set = blockIdx.x;
  if (set >= n_sets) return;
  const int64_t b0 = off[set], n64 = off[set + 1] - b0;
  if (n64 <= 0) {
    if (threadIdx.x == 0) out[set] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  if (n64 > kQMax) {  // any larger set: exact radix select of the same rank
    quantile_radix_select(q, x + b0, n64, out + set);
    return;
  }
  const int n = static_cast<int>(n64);
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = threadIdx.x; i < m; i += blockDim.x) s[i] = i < n ? x[b0 + i] : INFINITY;
  __syncthreads();
  for (int kk = 2; kk <= m; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const bool up = (i & kk) == 0;
          const double a = s[i], b = s[p];
          if ((a > b) == up) {
            s[i] = b;
            s[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    const int64_t rank = static_cast<int64_t>(ceil(q * static_cast<double>(n)));
    out[set] = s[rank == 0 ? 0 : rank - 1];
  }
}

__global__ void k_tps_window(int64_t n, const int64_t* __restrict__ off, const double* __restrict__ t,
                             const int32_t* __restrict__ tokens, const double* __restrict__ window,
                             const double* __restrict__ now, double* __restrict__ out) {
  const int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (w >= n) return;
  const double thr = now[w] - window[w];
  int64_t j = off[w];
  const int64_t e = off[w + 1];
  while (j < e && t[j] < thr) ++j;  // front pops (events are time-sorted)
  int sum = 0;
  for (; j < e; ++j) sum += tokens[j];
  out[w] = sum * 1000.0 / window[w];
}

}  // namespace

extern "C" int gsb_quantile_batch(gsb_ctx* ctx, double q, int64_t n_sets, const int64_t* d_off,
                                  const double* d_samples, double* d_out, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  if (!(q >= 0.0 && q <= 1.0)) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "quantile: q outside [0, 1]");
  if (n_sets <= 0) return GSB_OK;
  k_quantile<<<static_cast<unsigned>(n_sets), 256, 0, gsb_pick_stream(ctx, stream)>>>(q, n_sets, d_off,
                                                                                     d_samples, d_out);
  return gsb_check_launch(ctx, "quantile");
}

extern "C" int gsb_tps_window_batch(gsb_ctx* ctx, int64_t n, const int64_t* d_off, const double* d_t,
                                    const int32_t* d_tokens, const double* d_window_ms,
                                    const double* d_now, double* d_out, void* stream) {
  if (!ctx) return GSB_INVALID_ARGUMENT;
  if (n <= 0) return GSB_OK;
  k_tps_window<<<static_cast<unsigned>((n + 127) / 128), 128, 0, gsb_pick_stream(ctx, stream)>>>(
      n, d_off, d_t, d_tokens, d_window_ms, d_now, d_out);
  return gsb_check_launch(ctx, "tps_window");
}
