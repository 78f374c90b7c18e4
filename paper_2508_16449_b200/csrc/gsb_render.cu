// gsb_render.cu — the simulator's CSV wire formats rendered on the GPU from device-resident
// records: freq_timeline_csv and prefill_commands_csv (simkernel.cpp:686-714) and the
// controllers' decision_log_csv (decode_ctl.cpp:231-247, '%.6g'), byte for byte.
//
// Numbers go through the reference's fmt_g = snprintf("%.10g") (simkernel.cpp:679-683): ten
// significant digits, correctly rounded from the double's EXACT binary value (ties to even, as
// glibc does), %f form for decimal exponents -4..9 and %e form (two-digit minimum exponent)
// otherwise, trailing zeros and a bare point removed. fmt_g10 finds the digits D and exponent X
// with a double estimate, then settles them EXACTLY by comparing the value with D and D + 1/2 at
// that scale as big integers (m * 2^e * 10^s against K/2: 2 m 5^max(s,0) 2^max(a,0) vs
// K 5^max(-s,0) 2^max(-a,0), a = e + s), so every double, subnormals included, prints as glibc
// prints it. Integers (class, worker) print as std::to_string.
//
// Passes per call: per-record line lengths, a CUB exclusive scan, then every record writes its
// line at its offset (the header is copied first); like gsb_trace_format, synchronous.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <string>

#include "gsb_common.cuh"

namespace {

// ---------------------------------------------------------------- exact %.10g
constexpr int kLimbs = 40;  // 1280 bits: 2 m 5^333 2^a and (2D+1) 5^324 2^a all fit

struct Big {
  uint32_t w[kLimbs];
  int n;  // limbs in use (w[n..) are not read)
};

__device__ __forceinline__ void big_set(Big& a, unsigned long long v) {
  a.w[0] = static_cast<uint32_t>(v);
  a.w[1] = static_cast<uint32_t>(v >> 32);
  a.n = a.w[1] ? 2 : 1;
}

__device__ __forceinline__ void big_mul_small(Big& a, uint32_t m) {
  unsigned long long c = 0;
  for (int i = 0; i < a.n; ++i) {
    const unsigned long long t = static_cast<unsigned long long>(a.w[i]) * m + c;
    a.w[i] = static_cast<uint32_t>(t);
    c = t >> 32;
  }
  if (c && a.n < kLimbs) a.w[a.n++] = static_cast<uint32_t>(c);
}

__device__ __forceinline__ void big_mul_pow5(Big& a, int s) {
  constexpr uint32_t k5_13 = 1220703125u;  // 5^13 < 2^32
  uint32_t p5[13] = {1, 5, 25, 125, 625, 3125, 15625, 78125, 390625, 1953125, 9765625,
                     48828125, 244140625};
  while (s >= 13) {
    big_mul_small(a, k5_13);
    s -= 13;
  }
  if (s) big_mul_small(a, p5[s]);
}

__device__ __forceinline__ void big_shl(Big& a, int k) {
  const int limbs = k >> 5, bits = k & 31;
  if (bits) {
    uint32_t carry = 0;
    for (int i = 0; i < a.n; ++i) {
      const uint32_t v = a.w[i];
      a.w[i] = (v << bits) | carry;
      carry = v >> (32 - bits);
    }
    if (carry && a.n < kLimbs) a.w[a.n++] = carry;
  }
  if (limbs) {
    const int n = min(a.n + limbs, kLimbs);
    for (int i = n - 1; i >= limbs; --i) a.w[i] = a.w[i - limbs];
    for (int i = 0; i < limbs; ++i) a.w[i] = 0;
    a.n = n;
  }
}

__device__ __forceinline__ int big_cmp(const Big& a, const Big& b) {
  int na = a.n, nb = b.n;
  while (na > 1 && a.w[na - 1] == 0) --na;
  while (nb > 1 && b.w[nb - 1] == 0) --nb;
  if (na != nb) return na < nb ? -1 : 1;
  for (int i = na - 1; i >= 0; --i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}

// sign of (m 2^e 10^s - K/2): the value at scale 10^s against the half-integer K/2
__device__ int cmp_scaled(unsigned long long m, int e, int s, unsigned long long K) {
  Big L, R;
  big_set(L, m);
  big_shl(L, 1);
  big_set(R, K);
  if (s >= 0)
    big_mul_pow5(L, s);
  else
    big_mul_pow5(R, -s);
  const int a = e + s;
  if (a >= 0)
    big_shl(L, a);
  else
    big_shl(R, -a);
  return big_cmp(L, R);
}

__device__ __forceinline__ double pow10_d(int s) {  // 10^s: exact for |s| <= 22 (estimates only)
  const double t[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                        1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
  if (s >= 0 && s <= 22) return t[s];
  if (s < 0 && s >= -22) return 1.0 / t[-s];
  return exp10(static_cast<double>(s));
}

__host__ __device__ constexpr unsigned long long pow10_u(int k) {
  return k == 0 ? 1ull : 10ull * pow10_u(k - 1);
}

// snprintf(buf, 40, "%.<PR>g", v) for PR = 10 (fmt_g, simkernel.cpp:679-683) or 6 (fmt_num,
// decode_ctl.cpp:231-235); returns the length (<= PR + 7)
template <int PR>
__device__ int fmt_g(double v, char* out) {
  constexpr unsigned long long kLo = pow10_u(PR - 1), kHi = pow10_u(PR);
  constexpr double kHiD = static_cast<double>(kHi), kLoD = static_cast<double>(kLo);
  int n = 0;
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
  const bool neg = bits >> 63;
  const int be = static_cast<int>((bits >> 52) & 0x7ff);
  unsigned long long mant = bits & ((1ull << 52) - 1);
  if (be == 0x7ff) {  // glibc: "inf" / "nan" with the sign
    if (neg) out[n++] = '-';
    const char* t = mant ? "nan" : "inf";
    for (int i = 0; i < 3; ++i) out[n++] = t[i];
    return n;
  }
  if (neg) out[n++] = '-';
  if (be == 0 && mant == 0) {
    out[n++] = '0';
    return n;
  }
  int e;
  if (be == 0) {
    e = -1074;
  } else {
    mant |= 1ull << 52;
    e = be - 1075;
  }
  const double av = fabs(v);
  int X = static_cast<int>(floor(log10(av)));
  unsigned long long D = 0;
  for (int iter = 0; iter < 8; ++iter) {
    const int s = (PR - 1) - X;
    // estimate (relative error ~1e-15), in two factors so neither overflows at the range ends
    const double x = (av * pow10_d(s / 2)) * pow10_d(s - s / 2);
    // the estimate only moves X when clearly off; the exact floor below settles the boundary
    if (x >= 1.01 * kHiD) {
      ++X;
      continue;
    }
    if (x < 0.99 * kLoD) {
      --X;
      continue;
    }
    D = static_cast<unsigned long long>(x);
    // exact floor: D <= value * 10^s < D + 1
    for (int k = 0; k < 8 && D > 0 && cmp_scaled(mant, e, s, 2 * D) < 0; ++k) --D;
    for (int k = 0; k < 8 && cmp_scaled(mant, e, s, 2 * D + 2) >= 0; ++k) ++D;
    if (D < kLo) {  // exactly below the decade: one digit too few
      --X;
      continue;
    }
    if (D >= kHi) {  // exactly at or above the next decade
      ++X;
      continue;
    }
    // round half to even on the exact value
    const int c = cmp_scaled(mant, e, s, 2 * D + 1);
    if (c > 0 || (c == 0 && (D & 1))) ++D;
    if (D == kHi) {  // 99..9.5.. rounds up to the next decade: exactly 10^(PR-1) there
      D = kLo;
      ++X;
    }
    break;
  }
  char dg[PR];
  for (int i = PR - 1; i >= 0; --i) {
    dg[i] = static_cast<char>('0' + D % 10);
    D /= 10;
  }
  int last = PR - 1;  // last significant digit after stripping trailing zeros
  while (last > 0 && dg[last] == '0') --last;
  if (X < -4 || X >= PR) {
    out[n++] = dg[0];
    if (last > 0) {
      out[n++] = '.';
      for (int i = 1; i <= last; ++i) out[n++] = dg[i];
    }
    out[n++] = 'e';
    out[n++] = X < 0 ? '-' : '+';
    const int ax = X < 0 ? -X : X;
    if (ax >= 100) out[n++] = static_cast<char>('0' + ax / 100);
    out[n++] = static_cast<char>('0' + (ax / 10) % 10);
    out[n++] = static_cast<char>('0' + ax % 10);
  } else if (X >= 0) {
    for (int i = 0; i <= X; ++i) out[n++] = dg[i];
    if (last > X) {
      out[n++] = '.';
      for (int i = X + 1; i <= last; ++i) out[n++] = dg[i];
    }
  } else {
    out[n++] = '0';
    out[n++] = '.';
    for (int i = 0; i < -X - 1; ++i) out[n++] = '0';
    for (int i = 0; i <= last; ++i) out[n++] = dg[i];
  }
  return n;
}

__device__ __forceinline__ int fmt_g10(double v, char* out) { return fmt_g<10>(v, out); }

__device__ __forceinline__ int fmt_int(long long v, char* out) {  // std::to_string
  int n = 0;
  unsigned long long u = v < 0 ? 0ull - static_cast<unsigned long long>(v)
                               : static_cast<unsigned long long>(v);
  if (v < 0) out[n++] = '-';
  char t[20];
  int k = 0;
  do {
    t[k++] = static_cast<char>('0' + u % 10);
    u /= 10;
  } while (u);
  while (k) out[n++] = t[--k];
  return n;
}

// ---------------------------------------------------------------- record lines
struct FreqRecords {  // FreqChangeRecord (simkernel.hpp:131-136), SoA
  const double* applied_ms;
  const uint8_t* prefill_pool;
  const int32_t* worker;
  const double* f_mhz;
};

struct CommandRecords {  // PrefillCommandRecord (simkernel.hpp:139-146), SoA
  const double* tick_ms;
  const int32_t* class_id;
  const int32_t* worker;
  const double* f_mhz;
  const double* window_ms;
  const uint8_t* infeasible;
};

// freq_timeline_csv's line for record i (simkernel.cpp:688-695); returns its length
__device__ int line_of(const FreqRecords& r, int64_t i, char* b) {
  int n = fmt_g10(r.applied_ms[i], b);
  const char* pool = r.prefill_pool[i] ? ",prefill," : ",decode,";
  for (const char* p = pool; *p; ++p) b[n++] = *p;
  n += fmt_int(r.worker[i], b + n);
  b[n++] = ',';
  n += fmt_g10(r.f_mhz[i], b + n);
  b[n++] = '\n';
  return n;
}

// prefill_commands_csv's line for record i (simkernel.cpp:701-712)
__device__ int line_of(const CommandRecords& r, int64_t i, char* b) {
  int n = fmt_g10(r.tick_ms[i], b);
  b[n++] = ',';
  n += fmt_int(r.class_id[i], b + n);
  b[n++] = ',';
  n += fmt_int(r.worker[i], b + n);
  b[n++] = ',';
  n += fmt_g10(r.f_mhz[i], b + n);
  b[n++] = ',';
  n += fmt_g10(r.window_ms[i], b + n);
  b[n++] = ',';
  b[n++] = r.infeasible[i] ? '1' : '0';
  b[n++] = '\n';
  return n;
}

struct DecisionRecords {  // gsb_decision (K3b / K5 decision logs) = DecisionRecord
  const gsb_decision* r;   // (decode_ctl.hpp:95-105) with the action as its index
};

__constant__ char c_actions[8][16] = {"hold",           "up",          "down",
                                      "coarse_hold",    "coarse_pending", "coarse_commit",
                                      "adapt_up",       "adapt_down"};

// decision_log_csv's line for record i (decode_ctl.cpp:237-246), '%.6g' numbers
__device__ int line_of(const DecisionRecords& d, int64_t i, char* b) {
  const gsb_decision r = d.r[i];
  int n = fmt_g<6>(r.tick_ms, b);
  b[n++] = ',';
  n += fmt_int(r.worker, b + n);
  b[n++] = ',';
  n += fmt_g<6>(r.tps, b + n);
  b[n++] = ',';
  n += fmt_g<6>(r.p95_tbt_ms, b + n);
  b[n++] = ',';
  n += fmt_int(r.bucket, b + n);
  b[n++] = ',';
  n += fmt_g<6>(r.band_lo, b + n);
  b[n++] = ',';
  n += fmt_g<6>(r.band_hi, b + n);
  b[n++] = ',';
  n += fmt_g<6>(r.command_mhz, b + n);
  b[n++] = ',';
  const char* a = c_actions[static_cast<unsigned>(r.action) & 7u];
  for (int k = 0; a[k]; ++k) b[n++] = a[k];
  b[n++] = '\n';
  return n;
}

// longest line: decisions, 6 x 13 (%.6g) + 2 x 11 (int) + 14 (action) + separators
constexpr int kLineMax = 128;

template <class R>
__global__ void k_render_len(R r, int64_t n, unsigned long long* __restrict__ len) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  char b[kLineMax];
  len[i] = static_cast<unsigned long long>(line_of(r, i, b));
}

template <class R>
__global__ void k_render_write(R r, int64_t n, int64_t base,
                               const unsigned long long* __restrict__ off, char* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  char b[kLineMax];
  const int k = line_of(r, i, b);
  char* d = out + base + off[i];
  for (int j = 0; j < k; ++j) d[j] = b[j];
}

template <class R>
int render(gsb_ctx* ctx, const char* what, const char* header, R r, int64_t n, char* d_out,
           int64_t cap, int64_t* h_bytes, void* stream) {
  if (!ctx || !h_bytes || n < 0) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, what);
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  const int64_t hl = static_cast<int64_t>(strlen(header));
  unsigned long long body = 0;
  unsigned long long* off = nullptr;
  const unsigned g = static_cast<unsigned>((n + 127) / 128);
  if (n > 0) {
    size_t cub_tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_tmp, static_cast<unsigned long long*>(nullptr),
                                  static_cast<unsigned long long*>(nullptr),
                                  static_cast<int>(n + 1), s);
    const size_t lens = static_cast<size_t>(n + 1) * sizeof(unsigned long long);
    char* scr = static_cast<char*>(gsb_scratch(ctx, 2 * lens + cub_tmp + 256));
    if (!scr) return gsb_set_error(ctx, GSB_CUDA_ERROR, "render: scratch allocation failed");
    auto* len = reinterpret_cast<unsigned long long*>(scr);
    off = len + (n + 1);
    void* d_cub = scr + ((2 * lens + 255) / 256) * 256;
    cudaMemsetAsync(len + n, 0, sizeof(unsigned long long), s);
    k_render_len<R><<<g, 128, 0, s>>>(r, n, len);
    cub::DeviceScan::ExclusiveSum(d_cub, cub_tmp, len, off, static_cast<int>(n + 1), s);
    cudaMemcpyAsync(&body, off + n, sizeof(body), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return gsb_check_launch(ctx, what);
  }
  *h_bytes = hl + static_cast<int64_t>(body);
  if (!d_out) return GSB_OK;  // size query
  if (cap < *h_bytes) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "render: cap_bytes too small");
  cudaMemcpyAsync(d_out, header, static_cast<size_t>(hl), cudaMemcpyHostToDevice, s);
  if (n > 0) k_render_write<R><<<g, 128, 0, s>>>(r, n, hl, off, d_out);
  cudaStreamSynchronize(s);
  return gsb_check_launch(ctx, what);
}

// single values (tests, and any host that wants the reference's fmt_g on the device)
template <int PR>
__global__ void k_fmt_g(int64_t n, const double* __restrict__ v, char* __restrict__ out,
                        int32_t* __restrict__ len) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  char b[32];
  const int k = fmt_g<PR>(v[i], b);
  for (int j = 0; j < k; ++j) out[i * 32 + j] = b[j];
  len[i] = k;
}

}  // namespace

extern "C" {

int gsb_freq_timeline_csv(gsb_ctx* ctx, int64_t n, const double* d_applied_ms,
                          const uint8_t* d_prefill_pool, const int32_t* d_worker,
                          const double* d_f_mhz, char* d_out, int64_t cap_bytes, int64_t* h_bytes,
                          void* stream) {
  return render(ctx, "freq_timeline_csv", "applied_ms,pool,worker,f_mhz\n",
                FreqRecords{d_applied_ms, d_prefill_pool, d_worker, d_f_mhz}, n, d_out, cap_bytes,
                h_bytes, stream);
}

int gsb_prefill_commands_csv(gsb_ctx* ctx, int64_t n, const double* d_tick_ms,
                             const int32_t* d_class, const int32_t* d_worker,
                             const double* d_f_mhz, const double* d_window_ms,
                             const uint8_t* d_infeasible, char* d_out, int64_t cap_bytes,
                             int64_t* h_bytes, void* stream) {
  return render(ctx, "prefill_commands_csv", "tick_ms,class,worker,f_mhz,window_ms,infeasible\n",
                CommandRecords{d_tick_ms, d_class, d_worker, d_f_mhz, d_window_ms, d_infeasible},
                n, d_out, cap_bytes, h_bytes, stream);
}

int gsb_decision_log_csv(gsb_ctx* ctx, int64_t n, const gsb_decision* d_records, char* d_out,
                         int64_t cap_bytes, int64_t* h_bytes, void* stream) {
  return render(ctx, "decision_log_csv",
                "tick_ms,worker,tps,p95_tbt_ms,bucket,band_lo,band_hi,command_mhz,action\n",
                DecisionRecords{d_records}, n, d_out, cap_bytes, h_bytes, stream);
}

int gsb_format_g(gsb_ctx* ctx, int precision, int64_t n, const double* d_values, char* d_out32,
                 int32_t* d_len, void* stream) {
  if (!ctx || n < 0 || (precision != 6 && precision != 10)) return GSB_INVALID_ARGUMENT;
  if (n == 0) return GSB_OK;
  const unsigned g = static_cast<unsigned>((n + 127) / 128);
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  if (precision == 6)
    k_fmt_g<6><<<g, 128, 0, s>>>(n, d_values, d_out32, d_len);
  else
    k_fmt_g<10><<<g, 128, 0, s>>>(n, d_values, d_out32, d_len);
  return gsb_check_launch(ctx, "format_g");
}

int gsb_format_g10(gsb_ctx* ctx, int64_t n, const double* d_values, char* d_out32,
                   int32_t* d_len, void* stream) {
  return gsb_format_g(ctx, 10, n, d_values, d_out32, d_len, stream);
}

}  // extern "C"
