// gsb_trace.cu — K6: trace CSV ingest and output.
//
// gsb_trace_parse replaces greensim::load_trace (trace.cpp:56-129): the request CSV
// "arrival_ms,prompt_tokens,output_tokens[,class]" becomes the SoA the router/binner (K1)
// reads, with the reference's row semantics and its first-error-wins TraceError behaviour.
// gsb_trace_format replaces save_trace_csv (trace.cpp:131-145).
//
// Line model (std::getline on an ifstream, trace.cpp:60-78): a line ends at each '\n' and,
// when the file does not end with '\n', at the end of the file; one trailing '\r' is
// stripped; line 0 is the header; later empty lines are skipped but still counted by the
// reference's row counter (row = line index + 1).
//
// Passes (HBM-resident bytes, 4 KB tiles of 256 threads x 16 bytes):
//   1. k_csv_count:  per tile, line ends and non-empty lines (a line is attributed to the tile
//      holding its end), and the first end (the header's);
//   2. CUB exclusive scan of the packed (ends << 32 | non-empty) tile counts;
//   3. k_csv_parse:  per tile, the block-wide rank of each line end gives its line index and
//      output row; one thread parses one line (field split, from_chars restatement, range and
//      class checks) and writes arrival/prompt/output/SLO class at its row; errors are folded
//      into one 64-bit atomicMin key (row << 4 | check), so the earliest row wins and, within
//      a row, the reference's check order;
//   4. k_csv_monotone: arrival[r] < arrival[r-1] (trace.cpp:108-111) keyed by r's row.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <string>

#include "gsb_common.cuh"

namespace {

constexpr int kTrThreads = 256;
constexpr int kPerThread = 64;  // parse: bytes per thread (four 16-byte groups)
constexpr int kTile = kTrThreads * kPerThread;  // 8 KB
constexpr int kPre = 256;        // bytes staged before the tile (line starts)
constexpr int kMaxLines = 1024;  // listed lines per tile (a denser tile parses in place)
constexpr unsigned long long kNoErr = ~0ull;

struct TraceParams {
  const unsigned char* bytes;
  int64_t n;
  int64_t n_tiles;
  int64_t header_end;  // position of line 0's end (host-side uses; kernels read ParseState)
  int32_t has_class;
  int32_t threshold;
  int64_t cap_rows;    // rows >= cap_rows are not written (the host reports the overflow)
};

// Written on the device by k_csv_header and read back ONCE at the end of gsb_trace_parse (the
// header check, the row count and the first error all come back in one copy).
struct ParseState {
  int64_t header_end;  // line 0's end
  int64_t n_rows;      // non-empty lines after the header
  int64_t last_arrival;
  unsigned long long err;  // (row << 4 | check), ~0: none
  int32_t hdr;         // 3 / 4: a recognised header with that many columns; 0: unrecognised
  int32_t pad;
};

__device__ __forceinline__ unsigned char byte_at(const unsigned char* __restrict__ b, int64_t n,
                                                 int64_t i) {
  return (i >= 0 && i < n) ? __ldg(b + i) : static_cast<unsigned char>(0);
}

// stage [t*kTile - kPre, (t+1)*kTile) (bytes outside the file read as 0)
__device__ __forceinline__ void stage_tile(const TraceParams& tp, int64_t t, unsigned char* sm) {
  const int64_t s0 = t * kTile - kPre;
  for (int i = threadIdx.x; i < (kTile + kPre) / 16; i += kTrThreads) {
    const int64_t g = s0 + 16 * static_cast<int64_t>(i);
    uint4 v;
    if (g >= 0 && g + 16 <= tp.n && (reinterpret_cast<uintptr_t>(tp.bytes + g) & 15) == 0) {
      v = __ldg(reinterpret_cast<const uint4*>(tp.bytes + g));
    } else {
      unsigned char q[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) q[k] = byte_at(tp.bytes, tp.n, g + k);
      memcpy(&v, q, 16);
    }
    *reinterpret_cast<uint4*>(sm + 16 * i) = v;
  }
}

// bit k of the result: byte k of the 16 bytes q equals c (SIMD byte compare + MSB gather)
__device__ __forceinline__ unsigned eq_mask16(const uint4& q, unsigned c4) {
  unsigned m = 0;
  const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned e = __vcmpeq4(w[i], c4) & 0x80808080u;  // 0x80 per matching byte
    m |= ((e * 0x00204081u) >> 28) << (4 * i);              // gather the 4 MSBs
  }
  return m;
}

// Line ends and non-empty line ends among the 16 bytes [b0, b0 + 16) of a staged tile:
// bit k <-> byte b0 + k. A line ends at each '\n' and at n when the file does not end with
// '\n'; the line ending at b is empty iff byte b-1 is '\n' (or b is the file start) or byte
// b-1 is '\r' preceded by '\n' or the file start (one '\r' is stripped).
__device__ __forceinline__ void line_ends16_q(const uint4& q, unsigned char p1, unsigned char p2,
                                              int64_t n, int64_t b0, bool last_is_nl,
                                              unsigned* ends, unsigned* nonempty) {
  unsigned nl = eq_mask16(q, 0x0a0a0a0au), cr = eq_mask16(q, 0x0d0d0d0du);
  const int64_t live = n - b0;  // bytes of this chunk inside the file
  const unsigned in = live >= 16 ? 0xffffu : (live <= 0 ? 0u : (1u << live) - 1u);
  nl &= in;
  cr &= in;
  // 18-bit windows, bit j <-> byte b0 - 2 + j; the byte before the file start acts as '\n'
  unsigned nlx = (nl << 2) | (p1 == '\n' ? 2u : 0u) | (p2 == '\n' ? 1u : 0u);
  const unsigned crx = (cr << 2) | (p1 == '\r' ? 2u : 0u) | (p2 == '\r' ? 1u : 0u);
  if (b0 == 0) nlx |= 2u;
  unsigned e = nl;
  if (!last_is_nl && n > 0 && live >= 0 && live < 16) e |= 1u << live;  // the virtual end at n
  const unsigned empty = ((nlx >> 1) | ((crx >> 1) & nlx)) & 0xffffu;
  *ends = e;
  *nonempty = e & ~empty;
}

__device__ __forceinline__ void line_ends16(const unsigned char* sm, int64_t s0, int64_t n,
                                            int64_t b0, bool last_is_nl, unsigned* ends,
                                            unsigned* nonempty) {
  const uint4 q = *reinterpret_cast<const uint4*>(sm + (b0 - s0));
  line_ends16_q(q, sm[b0 - 1 - s0], sm[b0 - 2 - s0], n, b0, last_is_nl, ends, nonempty);
}

struct MaxI64 {
  __device__ __forceinline__ long long operator()(long long a, long long b) const {
    return a > b ? a : b;
  }
};


// line ends and empty lines among the 16 bytes q = [b0, b0 + 16), counts only: exact per-byte
// match masks (0x80 in each matching byte of a 64-bit word), one-byte shifts across the two
// words for the "previous byte" tests, popcounts. p1, p2: bytes b0-1, b0-2.
__device__ __forceinline__ void count16(const TraceParams& tp, const uint4& q, unsigned char p1,
                                        unsigned char p2, int64_t b0, bool last_is_nl,
                                        unsigned& n_end, unsigned& n_emp) {
  const unsigned long long w0 = (static_cast<unsigned long long>(q.y) << 32) | q.x;
  const unsigned long long w1 = (static_cast<unsigned long long>(q.w) << 32) | q.z;
  auto match = [](unsigned long long w, unsigned long long c8) {
    const unsigned long long x = w ^ c8;
    return ~(((x & 0x7f7f7f7f7f7f7f7full) + 0x7f7f7f7f7f7f7f7full) | x | 0x7f7f7f7f7f7f7f7full);
  };
  const int64_t live = tp.n - b0;  // bytes of this chunk inside the file
  unsigned long long in0 = ~0ull, in1 = ~0ull;
  if (live < 16) {
    in0 = live >= 8 ? ~0ull : (live <= 0 ? 0ull : (1ull << (8 * live)) - 1ull);
    in1 = live <= 8 ? 0ull : (1ull << (8 * (live - 8))) - 1ull;
  }
  const unsigned long long nl0 = match(w0, 0x0a0a0a0a0a0a0a0aull) & in0,
                           nl1 = match(w1, 0x0a0a0a0a0a0a0a0aull) & in1;
  const unsigned long long cr0 = match(w0, 0x0d0d0d0d0d0d0d0dull) & in0,
                           cr1 = match(w1, 0x0d0d0d0d0d0d0d0dull) & in1;
  // previous-byte masks (byte j <-> byte j-1 of the chunk); the byte before the file start
  // acts as '\n'
  const unsigned long long p1nl = (p1 == '\n' || b0 == 0) ? 0x80ull : 0ull;
  const unsigned long long p1cr = p1 == '\r' ? 0x80ull : 0ull;
  const unsigned long long p2nl = p2 == '\n' ? 0x80ull : 0ull;
  const unsigned long long nlm1_0 = (nl0 << 8) | p1nl, nlm1_1 = (nl1 << 8) | (nl0 >> 56);
  const unsigned long long crm1_0 = (cr0 << 8) | p1cr, crm1_1 = (cr1 << 8) | (cr0 >> 56);
  const unsigned long long nlm2_0 = (nl0 << 16) | (p1nl << 8) | p2nl,
                           nlm2_1 = (nl1 << 16) | (nl0 >> 48);
  const unsigned long long emp0 = nl0 & (nlm1_0 | (crm1_0 & nlm2_0));
  const unsigned long long emp1 = nl1 & (nlm1_1 | (crm1_1 & nlm2_1));
  n_end = __popcll(nl0) + __popcll(nl1);
  n_emp = __popcll(emp0) + __popcll(emp1);
  if (!last_is_nl && tp.n > 0 && live >= 0 && live < 16) {  // the virtual end at n
    ++n_end;
    // the last line is empty iff its only content is one '\r' after a line start
    const int64_t b = tp.n;
    const unsigned char c1 = byte_at(tp.bytes, tp.n, b - 1), c2 = byte_at(tp.bytes, tp.n, b - 2);
    if (c1 == '\r' && (b - 1 == 0 || c2 == '\n')) ++n_emp;
  }
}

// Count pass: no staging and no block barrier. Thread g reads the 64 bytes [64g, 64g + 64)
// with four independent 16-byte vector loads, takes the two bytes before them from its left
// neighbour (a shuffle), and the warp's packed (line ends << 32 | non-empty lines) sum goes to
// its tile with one atomic add (integer, so the per-tile totals are exact and order-free).
constexpr int kCountChunks = 4;
__global__ void __launch_bounds__(kTrThreads)
k_csv_count(const TraceParams tp, unsigned long long* __restrict__ tile_cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t b0 =
      (static_cast<int64_t>(blockIdx.x) * kTrThreads + threadIdx.x) * (16 * kCountChunks);
  uint4 q[kCountChunks];
  const bool fast = b0 + 16 * kCountChunks <= tp.n &&
                    (reinterpret_cast<uintptr_t>(tp.bytes + b0) & 15) == 0;
#pragma unroll
  for (int k = 0; k < kCountChunks; ++k) {
    if (fast) {
      q[k] = __ldg(reinterpret_cast<const uint4*>(tp.bytes + b0) + k);
    } else {
      unsigned char c[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) c[j] = byte_at(tp.bytes, tp.n, b0 + 16 * k + j);
      memcpy(&q[k], c, 16);
    }
  }
  const unsigned left = __shfl_up_sync(0xffffffffu, q[kCountChunks - 1].w, 1);
  unsigned char p1 = static_cast<unsigned char>(left >> 24), p2 = static_cast<unsigned char>(left >> 16);
  if (lane == 0) {
    p1 = byte_at(tp.bytes, tp.n, b0 - 1);
    p2 = byte_at(tp.bytes, tp.n, b0 - 2);
  }
  const bool last_is_nl = tp.n > 0 && __ldg(tp.bytes + tp.n - 1) == '\n';
  unsigned tot_end = 0, tot_emp = 0;
#pragma unroll
  for (int k = 0; k < kCountChunks; ++k) {
    unsigned e, m;
    count16(tp, q[k], p1, p2, b0 + 16 * k, last_is_nl, e, m);
    tot_end += e;
    tot_emp += m;
    p1 = static_cast<unsigned char>(q[k].w >> 24);
    p2 = static_cast<unsigned char>(q[k].w >> 16);
  }
  unsigned long long v = (static_cast<unsigned long long>(tot_end) << 32) | (tot_end - tot_emp);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0 && v) atomicAdd(tile_cnt + b0 / kTile, v);
}

__device__ __forceinline__ unsigned long long err_key(int64_t line, int detail) {
  return (static_cast<unsigned long long>(line + 1) << 4) | static_cast<unsigned long long>(detail);
}

__global__ void __launch_bounds__(kTrThreads)
k_csv_parse(TraceParams tp, const unsigned long long* __restrict__ tile_pref,
            int64_t* __restrict__ arrival, int32_t* __restrict__ prompt,
            int32_t* __restrict__ output, uint8_t* __restrict__ slo_cls,
            uint32_t* __restrict__ line_of_row, ParseState* __restrict__ ps) {
  const int hdr = ps->hdr;
  if (hdr == 0) return;  // unrecognised header: nothing is parsed (the host reports it)
  tp.has_class = hdr == 4 ? 1 : 0;
  tp.header_end = ps->header_end;
  unsigned long long* err = &ps->err;
  __shared__ __align__(16) unsigned char sm[kTile + kPre + 16];
  using BS = cub::BlockScan<unsigned long long, kTrThreads>;
  using BS2 = cub::BlockScan<long long, kTrThreads>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ typename BS2::TempStorage tmp2;
  __shared__ int64_t s_st[kMaxLines];  // the tile's non-empty lines: start, end (tile-relative),
  __shared__ int32_t s_b[kMaxLines];   // line index (tile-relative)
  __shared__ int32_t s_ln[kMaxLines];
  __shared__ unsigned long long s_cm[(kTile + kPre) / 64 + 1];  // comma bitmap of the stage
  const int64_t t = blockIdx.x;
  stage_tile(tp, t, sm);
  __syncthreads();
  const int64_t s0 = t * kTile - kPre;
  const bool last_is_nl = tp.n > 0 && __ldg(tp.bytes + tp.n - 1) == '\n';
  const int64_t b0 = t * kTile + kPerThread * threadIdx.x;
  unsigned long long ends = 0, nonempty = 0;  // bit k: byte b0 + k ends a (non-empty) line
#pragma unroll
  for (int h = 0; h < kPerThread / 16; ++h) {
    unsigned e, ne16;
    line_ends16(sm, s0, tp.n, b0 + 16 * h, last_is_nl, &e, &ne16);
    ends |= static_cast<unsigned long long>(e) << (16 * h);
    nonempty |= static_cast<unsigned long long>(ne16) << (16 * h);
  }
  // the comma bitmap of the staged bytes (bit i <-> byte s0 + i), for the line fast path
  {
    const unsigned char* mine = sm + kPre + kPerThread * threadIdx.x;
    unsigned long long cw = 0;
#pragma unroll
    for (int h = 0; h < kPerThread / 16; ++h)
      cw |= static_cast<unsigned long long>(
                eq_mask16(*reinterpret_cast<const uint4*>(mine + 16 * h), 0x2c2c2c2cu))
            << (16 * h);
    s_cm[kPre / 64 + threadIdx.x] = cw;
    if (threadIdx.x < kPre / 64) {
      const unsigned char* pre_b = sm + 64 * threadIdx.x;
      unsigned long long cp = 0;
#pragma unroll
      for (int h = 0; h < 4; ++h)
        cp |= static_cast<unsigned long long>(
                  eq_mask16(*reinterpret_cast<const uint4*>(pre_b + 16 * h), 0x2c2c2c2cu))
              << (16 * h);
      s_cm[threadIdx.x] = cp;
    }
    if (threadIdx.x == 0) s_cm[(kTile + kPre) / 64] = 0;
  }
  const unsigned nl = __popcll(ends), ne = __popcll(nonempty);
  unsigned long long pre, agg;
  BS(tmp).ExclusiveSum((static_cast<unsigned long long>(nl) << 32) | ne, pre, agg);
  __syncthreads();
  // the previous line end before this thread's bytes: exclusive max-scan of the threads' last
  // ends; the tile's first line looks back into the previous tile (one thread per tile)
  long long prev;
  BS2(tmp2).ExclusiveScan(ends ? static_cast<long long>(b0 + 63 - __clzll(ends)) : -1LL, prev,
                          -1LL, MaxI64{});
  if (threadIdx.x == 0) prev = -1;
  const unsigned long long tp0 = tile_pref[t];
  int64_t line = static_cast<int64_t>(tp0 >> 32) + static_cast<int64_t>(pre >> 32);
  int64_t nonempty_before = static_cast<int64_t>(tp0 & 0xffffffffull) +
                            static_cast<int64_t>(pre & 0xffffffffull);
  const int expect = tp.has_class ? 4 : 3;
  if (ends && prev < 0) {  // this thread holds the tile's first line end
    int64_t st = b0 + __ffsll(static_cast<long long>(ends)) - 2;
    while (st >= 0) {
      const unsigned char c = st >= s0 ? sm[st - s0] : __ldg(tp.bytes + st);
      if (c == '\n') break;
      --st;
    }
    prev = st;  // -1 at the file start
  }
  // one non-empty line [st, b) (st may precede the staged bytes): fields, checks, outputs
  auto parse_one = [&](const int64_t st, const int64_t b, const int64_t my_line,
                       const int64_t ne_idx) {
    if (b <= tp.header_end) return;  // the header
    const int64_t row = ne_idx - 1;  // the header is the first non-empty line
    const bool in_sm = st >= s0;
    auto at = [&](int64_t i) -> unsigned char { return in_sm ? sm[i - s0] : __ldg(tp.bytes + i); };
    int64_t en = b;
    if (en > st && at(en - 1) == '\r') --en;
    // one pass over the line: columns split on ',' (a trailing ',' adds no column,
    // std::getline(ss, col, ',')), from_chars<int64> on columns 0-2 (optional '-', >= 1
    // digit, the whole column, no overflow), the class column's bytes
    unsigned long long v0 = 0, v1 = 0, v2 = 0;
    bool ok0 = false, ok1 = false, ok2 = false;
    unsigned char c0 = 0, c1 = 0;
    int clen = 0, ncols;
    const int len = static_cast<int>(min(en - st, static_cast<int64_t>(INT32_MAX)));
    bool general = !(in_sm && len <= 64 && st - s0 >= 16);
    if (!general) {
      // fast path: the line's comma mask from the tile's comma bitmap (s_cm), then each
      // numeric column as at most two 8-digit SWAR words (unaligned 8-byte smem reads)
      const int qo = static_cast<int>(st - s0);
      const unsigned char* q = sm + qo;
      const int cw = qo >> 6, cb = qo & 63;
      unsigned long long cm = s_cm[cw] >> cb;
      if (cb) cm |= s_cm[cw + 1] << (64 - cb);
      if (len < 64) cm &= (1ull << len) - 1ull;
      const bool trailing = (cm >> (len - 1)) & 1ull;
      ncols = __popcll(cm) + (trailing ? 0 : 1);  // a final ',' adds no column
      int fs[4], fe[4];
      unsigned long long m = cm;
      int f0 = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = m ? __ffsll(static_cast<long long>(m)) - 1 : len;
        m &= m - 1ull;
        fs[k] = f0;
        fe[k] = e;
        f0 = min(e + 1, len);
      }
      // the 8 bytes q[end-8, end) as a little-endian word (qo >= 16 keeps them staged)
      auto ld8 = [&](int end) -> unsigned long long {
        const int off = qo + end - 8;
        const int sh = (off & 7) * 8;
        const unsigned long long* w = reinterpret_cast<const unsigned long long*>(sm + (off & ~7));
        return sh ? (w[0] >> sh) | (w[1] << (64 - sh)) : w[0];
      };
      // n (1..8) digits in the top n bytes of x: their value, and whether all are '0'..'9'
      auto parse8 = [](unsigned long long x, int n, bool& dig) -> unsigned long long {
        const unsigned long long keep = ~0ull << (8 * (8 - n));
        x = (x & keep) | (0x3030303030303030ull & ~keep);  // leading '0's
        dig = ((x & 0xF0F0F0F0F0F0F0F0ull) == 0x3030303030303030ull) &&
              (((x + 0x0606060606060606ull) & 0xF0F0F0F0F0F0F0F0ull) == 0x3030303030303030ull);
        x -= 0x3030303030303030ull;
        x = x * 10 + (x >> 8);
        return (((x & 0x000000FF000000FFull) * (100 + (1000000ull << 32))) +
                (((x >> 16) & 0x000000FF000000FFull) * (1 + (10000ull << 32)))) >> 32;
      };
      // from_chars<int64> on the whole column: >= 1 digit; a sign or more than 16 digits
      // (possible overflow) goes to the general path
      auto num = [&](int a0, int a1, unsigned long long& v, bool& ok) {
        const int n = a1 - a0;
        if (n > 16 || (n > 0 && q[a0] == '-')) {
          general = true;
          return;
        }
        ok = false;
        v = 0;
        if (n == 0) return;
        bool d_lo;
        const unsigned long long lo = parse8(ld8(a1), n > 8 ? 8 : n, d_lo);
        if (n > 8) {
          bool d_hi;
          const unsigned long long hi = parse8(ld8(a1 - 8), n - 8, d_hi);
          v = hi * 100000000ull + lo;
          ok = d_lo && d_hi;
        } else {
          v = lo;
          ok = d_lo;
        }
      };
      if (ncols == expect) {
        num(fs[0], fe[0], v0, ok0);
        num(fs[1], fe[1], v1, ok1);
        num(fs[2], fe[2], v2, ok2);
        if (expect == 4) {
          clen = fe[3] - fs[3];
          c0 = clen > 0 ? q[fs[3]] : 0;
          c1 = clen > 1 ? q[fs[3] + 1] : 0;
        }
      }
    }
    if (general) {
    // general path (long lines or columns, lines starting before the staged bytes): one
    // scalar pass
    c0 = c1 = 0;
    clen = 0;
    unsigned long long cur = 0;
    int col = 0, flen = 0, sig = 0;
    bool neg = false, bad = false;
    auto close_field = [&]() {
      if (col < 3) {
        const unsigned long long lim = neg ? 0x8000000000000000ull : 0x7fffffffffffffffull;
        const bool ok = !bad && flen > (neg ? 1 : 0) && cur <= lim;
        const unsigned long long val = neg ? 0ull - cur : cur;
        if (col == 0) { v0 = val; ok0 = ok; }
        if (col == 1) { v1 = val; ok1 = ok; }
        if (col == 2) { v2 = val; ok2 = ok; }
      } else if (col == 3) {
        clen = flen;
      }
      ++col;
      cur = 0;
      flen = sig = 0;
      neg = bad = false;
    };
    bool last_comma = false;
    for (int64_t i = st; i < en; ++i) {
      const unsigned char c = at(i);
      last_comma = c == ',';
      if (c == ',') {
        close_field();
        continue;
      }
      if (col < 3) {
        if (flen == 0 && c == '-') {
          neg = true;
        } else {
          const unsigned d = static_cast<unsigned>(c) - '0';
          if (d > 9) {
            bad = true;
          } else if (cur != 0 || d != 0) {  // leading zeros are free
            if (++sig > 19) bad = true;     // > 19 significant digits overflows int64
            else cur = cur * 10 + d;
          }
        }
      } else if (col == 3) {
        if (flen == 0) c0 = c;
        if (flen == 1) c1 = c;
      }
      ++flen;
    }
    if (last_comma) {
      ncols = col;  // the empty text after the final ',' is not a column
    } else {
      close_field();
      ncols = col;
    }
    }
    int detail = 0;
    if (ncols != expect) detail = GSB_TRACE_DETAIL_COLUMNS;
    else if (!ok0) detail = GSB_TRACE_DETAIL_ARRIVAL;
    else if (!ok1) detail = GSB_TRACE_DETAIL_PROMPT;
    else if (!ok2) detail = GSB_TRACE_DETAIL_OUTPUT;
    const int64_t a = static_cast<int64_t>(v0);
    // static_cast<int>(int64) (trace.cpp:98-99): two's-complement truncation
    const int32_t pi = static_cast<int32_t>(static_cast<uint32_t>(v1));
    const int32_t oi = static_cast<int32_t>(static_cast<uint32_t>(v2));
    if (!detail && (a < 0 || pi < 1 || oi < 1)) detail = GSB_TRACE_DETAIL_RANGE;
    const uint8_t cls = pi <= tp.threshold ? 0 : 1;  // classify_by_threshold, trace.cpp:32-34
    if (!detail && tp.has_class) {
      int fc = -1;
      if (clen == 2 && c0 == 'S' && c1 == 'M') fc = 0;
      if (clen == 1 && c0 == 'L') fc = 1;
      if (fc < 0)
        detail = GSB_TRACE_DETAIL_CLASS;
      else if (fc != cls)
        detail = GSB_TRACE_DETAIL_MISMATCH;
    }
    if (row >= tp.cap_rows) return;  // more rows than the caller's buffers: reported
    arrival[row] = a;
    prompt[row] = pi;
    output[row] = oi;
    slo_cls[row] = cls;
    line_of_row[row] = static_cast<uint32_t>(my_line);
    if (detail) atomicMin(err, err_key(my_line, detail));
  };
  const int64_t line0 = static_cast<int64_t>(tp0 >> 32);
  const int64_t ne0 = static_cast<int64_t>(tp0 & 0xffffffffull);
  const int n_ne = static_cast<int>(agg & 0xffffffffull);
  if (n_ne <= kMaxLines) {
    // the tile's non-empty lines listed in order, then parsed round-robin: every thread gets
    // the same number of lines (+-1) instead of the lines ending in its own 64 bytes
    int idx = static_cast<int>(pre & 0xffffffffull);
    while (ends) {
      const int k = __ffsll(static_cast<long long>(ends)) - 1;
      ends &= ends - 1ull;
      const int64_t b = b0 + k;
      const int64_t st = prev + 1;
      prev = b;
      const int64_t my_line = line++;
      if (!((nonempty >> k) & 1ull)) continue;  // empty line: skipped (still counted)
      s_st[idx] = st;
      s_b[idx] = static_cast<int32_t>(b - s0);
      s_ln[idx] = static_cast<int32_t>(my_line - line0);
      ++idx;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_ne; i += kTrThreads)
      parse_one(s_st[i], s0 + s_b[i], line0 + s_ln[i], ne0 + i);
  } else {
    while (ends) {
      const int k = __ffsll(static_cast<long long>(ends)) - 1;
      ends &= ends - 1ull;
      const int64_t b = b0 + k;
      const int64_t st = prev + 1;
      prev = b;
      const int64_t my_line = line++;
      if (!((nonempty >> k) & 1ull)) continue;  // empty line: skipped (still counted)
      parse_one(st, b, my_line, nonempty_before++);
    }
  }
}

// trace.cpp:108-111: arrivals non-decreasing (checked after the range checks of the same row)
__global__ void k_csv_monotone(const int64_t* __restrict__ arrival,
                               const uint32_t* __restrict__ line_of_row, int64_t cap_rows,
                               ParseState* __restrict__ ps) {
  if (ps->hdr == 0) return;
  const int64_t n_rows = ps->n_rows;
  if (n_rows <= 0 || n_rows > cap_rows) return;  // reported by the host before any row error
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = 1 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_rows;
       r += stride)
    if (arrival[r] < arrival[r - 1])
      atomicMin(&ps->err, err_key(line_of_row[r], GSB_TRACE_DETAIL_MONOTONE));
  if (blockIdx.x == 0 && threadIdx.x == 0) ps->last_arrival = arrival[n_rows - 1];
}

// the header's end (line 0): one warp walks the file from byte 0, 32 bytes per step (ballot of
// the line-end bytes), so the usual short header costs one coalesced load
__constant__ char c_hdr4[] = "arrival_ms,prompt_tokens,output_tokens,class";

// ...then (trace.cpp:63-74) line 0 after one '\r' strip against the two accepted headers, the
// row count from the line scan, and the error key's reset: ParseState for the parse kernels
__global__ void k_csv_header(const TraceParams tp, const unsigned long long* __restrict__ tile_pref,
                             int64_t nt, ParseState* __restrict__ ps) {
  const int lane = threadIdx.x;
  const bool last_is_nl = tp.n > 0 && tp.bytes[tp.n - 1] == '\n';
  int64_t he = tp.n;
  for (int64_t b0 = 0;; b0 += 32) {
    const int64_t b = b0 + lane;
    const bool e = b < tp.n ? tp.bytes[b] == '\n' : (b == tp.n && tp.n > 0 && !last_is_nl);
    const unsigned m = __ballot_sync(0xffffffffu, e);
    if (m) {
      he = b0 + __ffs(static_cast<int>(m)) - 1;
      break;
    }
    if (b0 + 32 > tp.n) break;  // no end at all (n == 0)
  }
  int64_t hlen = he;
  if (hlen > 0 && tp.bytes[hlen - 1] == '\r') --hlen;
  constexpr int64_t k4 = sizeof(c_hdr4) - 1, k3 = k4 - 6;  // "...,class" / without ",class"
  bool ok = true;
  if (hlen == k4 || hlen == k3) {
    for (int64_t i = lane; i < hlen; i += 32) ok = ok && tp.bytes[i] == c_hdr4[i];
    ok = __all_sync(0xffffffffu, ok);
  }
  if (lane == 0) {
    ps->header_end = he;
    ps->hdr = (hlen == k4 && ok) ? 4 : ((hlen == k3 && ok) ? 3 : 0);
    ps->n_rows = static_cast<int64_t>(tile_pref[nt - 1] & 0xffffffffull) - 1;  // minus the header
    ps->last_arrival = 0;
    ps->err = kNoErr;
  }
}

// the byte range of line L (error reporting): one thread, binary search of the tile prefix
__global__ void k_csv_locate(const TraceParams tp, const unsigned long long* __restrict__ tile_pref,
                             int64_t L, int64_t* __restrict__ out /* [2]: start, end */) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t lo = 0, hi = tp.n_tiles - 1;  // last tile with pref.nl <= L
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (static_cast<int64_t>(tile_pref[mid] >> 32) <= L) lo = mid; else hi = mid - 1;
  }
  int64_t line = static_cast<int64_t>(tile_pref[lo] >> 32);
  const bool last_is_nl = tp.n > 0 && tp.bytes[tp.n - 1] == '\n';
  int64_t b = lo * kTile;
  for (;; ++b) {
    const bool e = b < tp.n ? tp.bytes[b] == '\n' : (b == tp.n && tp.n > 0 && !last_is_nl);
    if (e) {
      if (line == L) break;
      ++line;
    }
    if (b >= tp.n) break;
  }
  int64_t st = b - 1;
  while (st >= 0 && tp.bytes[st] != '\n') --st;
  out[0] = st + 1;
  out[1] = b;
}

// ---------------------------------------------------------------- save_trace_csv
__device__ __forceinline__ int n_digits(int64_t v) {  // ostream << int64: '-' + digits
  unsigned long long u = v < 0 ? 0ull - static_cast<unsigned long long>(v) : static_cast<unsigned long long>(v);
  int d = 1;
  while (u >= 10) {
    u /= 10;
    ++d;
  }
  return d + (v < 0 ? 1 : 0);
}

__device__ __forceinline__ void put_int(char* dst, int64_t v, int len) {
  unsigned long long u = v < 0 ? 0ull - static_cast<unsigned long long>(v) : static_cast<unsigned long long>(v);
  for (int i = len - 1; i >= (v < 0 ? 1 : 0); --i) {
    dst[i] = static_cast<char>('0' + u % 10);
    u /= 10;
  }
  if (v < 0) dst[0] = '-';
}

__device__ __forceinline__ int row_len(int64_t a, int32_t p, int32_t o, int cls) {
  return n_digits(a) + n_digits(p) + n_digits(o) + 2 + (cls < 0 ? 0 : (cls == 0 ? 3 : 2)) + 1;
}

__global__ void k_csv_row_len(int64_t n, const int64_t* __restrict__ a, const int32_t* __restrict__ p,
                              const int32_t* __restrict__ o, const uint8_t* __restrict__ cls,
                              unsigned long long* __restrict__ len) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  len[r] = static_cast<unsigned long long>(row_len(a[r], p[r], o[r], cls ? cls[r] : -1));
}

__global__ void k_csv_write(int64_t n, int64_t base, const int64_t* __restrict__ a,
                            const int32_t* __restrict__ p, const int32_t* __restrict__ o,
                            const uint8_t* __restrict__ cls, const unsigned long long* __restrict__ off,
                            char* __restrict__ out) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  char* d = out + base + off[r];
  const int la = n_digits(a[r]), lp = n_digits(p[r]), lo = n_digits(o[r]);
  put_int(d, a[r], la);
  d += la;
  *d++ = ',';
  put_int(d, p[r], lp);
  d += lp;
  *d++ = ',';
  put_int(d, o[r], lo);
  d += lo;
  if (cls) {
    *d++ = ',';
    if (cls[r] == 0) {
      *d++ = 'S';
      *d++ = 'M';
    } else {
      *d++ = 'L';
    }
  }
  *d = '\n';
}

const char kHdr3[] = "arrival_ms,prompt_tokens,output_tokens";
const char kHdr4[] = "arrival_ms,prompt_tokens,output_tokens,class";

void set_result_line(gsb_trace_parse_result* r, const char* p, int64_t len) {
  const int64_t k = std::min<int64_t>(len, static_cast<int64_t>(sizeof(r->line) - 1));
  memcpy(r->line, p, static_cast<size_t>(k));
  r->line[k] = 0;
  r->line_len = static_cast<int32_t>(k);
  r->line_truncated = len > k ? 1 : 0;
}

}  // namespace

extern "C" {

int gsb_trace_parse(gsb_ctx* ctx, const char* d_bytes, int64_t n_bytes, int32_t class_threshold,
                    int64_t cap_rows, int64_t* d_arrival, int32_t* d_prompt, int32_t* d_output,
                    uint8_t* d_slo_class, gsb_trace_parse_result* res, void* stream) {
  if (!ctx || !res || n_bytes < 0 || (n_bytes > 0 && !d_bytes))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "trace_parse: bad arguments");
  if (n_bytes >= (int64_t{1} << 32))
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "trace_parse: input must be < 4 GiB");
  memset(res, 0, sizeof(*res));
  res->row = -1;
  auto fail = [&](int kind, int detail, int64_t row, const std::string& msg) {
    res->status = GSB_TRACE_ERROR;
    res->kind = kind;
    res->detail = detail;
    res->row = row;
    return gsb_set_error(ctx, GSB_TRACE_ERROR, msg);
  };
  if (n_bytes == 0) return fail(GSB_TRACE_KIND_EMPTY, 0, -1, "empty trace file");
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  TraceParams tp{};
  tp.bytes = reinterpret_cast<const unsigned char*>(d_bytes);
  tp.n = n_bytes;
  tp.n_tiles = n_bytes / kTile + 1;  // the virtual end at n may open a tile
  tp.threshold = class_threshold;
  tp.cap_rows = cap_rows;
  // scratch: [tile counts + 1][prefix + 1][ParseState][locate 2][line_of_row (cap)][cub tmp]
  const size_t nt = static_cast<size_t>(tp.n_tiles) + 1;
  size_t cub_tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_tmp, static_cast<unsigned long long*>(nullptr),
                                static_cast<unsigned long long*>(nullptr), static_cast<int>(nt), s);
  const size_t head = 2 * nt * sizeof(unsigned long long) + sizeof(ParseState) + 32;
  const size_t lor = static_cast<size_t>(std::max<int64_t>(cap_rows, 1)) * sizeof(uint32_t);
  char* scr = static_cast<char*>(gsb_scratch(ctx, head + lor + cub_tmp + 256));
  if (!scr) return gsb_set_error(ctx, GSB_CUDA_ERROR, "trace_parse: scratch allocation failed");
  auto* cnt = reinterpret_cast<unsigned long long*>(scr);
  auto* pref = cnt + nt;
  auto* ps = reinterpret_cast<ParseState*>(pref + nt);
  auto* loc = reinterpret_cast<int64_t*>(ps + 1);
  auto* line_of_row = reinterpret_cast<uint32_t*>(scr + head);
  void* d_cub = scr + ((head + lor + 255) / 256) * 256;
  // everything on the stream, ONE read-back at the end: the header check (line 0 against the
  // two accepted headers), the row count and the first failing row come back together
  cudaMemsetAsync(cnt, 0, nt * sizeof(unsigned long long), s);
  k_csv_count<<<static_cast<unsigned>((n_bytes / (16 * kCountChunks) + 1 + kTrThreads - 1) /
                                      kTrThreads),
                kTrThreads, 0, s>>>(tp, cnt);
  cub::DeviceScan::ExclusiveSum(d_cub, cub_tmp, cnt, pref, static_cast<int>(nt), s);
  k_csv_header<<<1, 32, 0, s>>>(tp, pref, static_cast<int64_t>(nt), ps);
  k_csv_parse<<<static_cast<unsigned>(tp.n_tiles), kTrThreads, 0, s>>>(
      tp, pref, d_arrival, d_prompt, d_output, d_slo_class, line_of_row, ps);
  k_csv_monotone<<<static_cast<unsigned>(ctx->n_sms * 8), 256, 0, s>>>(d_arrival, line_of_row,
                                                                       cap_rows, ps);
  ParseState st{};
  cudaMemcpyAsync(&st, ps, sizeof(st), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return gsb_check_launch(ctx, "trace_parse");
  const int rc = gsb_check_launch(ctx, "trace_parse");
  if (rc) return rc;
  const int64_t header_end = st.header_end;
  if (st.hdr == 0) {  // trace.cpp:63-74: the whole header line in the message
    std::string full(static_cast<size_t>(header_end), '\0');
    if (!full.empty()) cudaMemcpy(&full[0], d_bytes, full.size(), cudaMemcpyDeviceToHost);
    if (!full.empty() && full.back() == '\r') full.pop_back();
    set_result_line(res, full.data(), static_cast<int64_t>(full.size()));
    return fail(GSB_TRACE_KIND_BAD_HEADER, 0, 1, "unrecognized trace header: " + full);
  }
  tp.has_class = st.hdr == 4 ? 1 : 0;
  res->has_class = tp.has_class;
  tp.header_end = header_end;
  const int64_t n_rows = st.n_rows;
  if (n_rows <= 0) return fail(GSB_TRACE_KIND_EMPTY, 0, -1, "trace has no rows");
  if (n_rows > cap_rows) {
    res->n_rows = n_rows;
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "trace_parse: more rows than cap_rows");
  }
  const unsigned long long ek = st.err;
  if (ek == kNoErr) {
    res->n_rows = n_rows;
    res->max_arrival_ms = st.last_arrival;  // arrivals are non-decreasing: the last is the max
    return GSB_OK;
  }
  // the earliest failing row: fetch its bytes, the host formats the reference's message
  const int64_t row = static_cast<int64_t>(ek >> 4);
  const int detail = static_cast<int>(ek & 15);
  k_csv_locate<<<1, 32, 0, s>>>(tp, pref, row - 1, loc);
  int64_t se[2];
  cudaMemcpyAsync(se, loc, sizeof(se), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  std::string line(static_cast<size_t>(se[1] - se[0]), '\0');
  if (!line.empty())
    cudaMemcpy(&line[0], d_bytes + se[0], line.size(), cudaMemcpyDeviceToHost);
  if (!line.empty() && line.back() == '\r') line.pop_back();
  set_result_line(res, line.data(), static_cast<int64_t>(line.size()));
  const std::string r = "row " + std::to_string(row) + ": ";
  // column split for the message (same rule as the kernel)
  std::string cols[4];
  int ncols = 0;
  size_t f0 = 0;
  for (size_t i = 0; i <= line.size(); ++i) {
    if (i == line.size() || line[i] == ',') {
      if (i == line.size() && i == f0 && ncols > 0) break;
      if (ncols < 4) cols[ncols] = line.substr(f0, i - f0);
      ++ncols;
      f0 = i + 1;
    }
  }
  res->n_cols = ncols;
  const int expect = tp.has_class ? 4 : 3;
  switch (detail) {
    case GSB_TRACE_DETAIL_COLUMNS:
      return fail(GSB_TRACE_KIND_MALFORMED, detail, row,
                  r + "expected " + std::to_string(expect) + " columns, got " + std::to_string(ncols));
    case GSB_TRACE_DETAIL_ARRIVAL:
      return fail(GSB_TRACE_KIND_MALFORMED, detail, row, r + "bad arrival_ms '" + cols[0] + "'");
    case GSB_TRACE_DETAIL_PROMPT:
      return fail(GSB_TRACE_KIND_MALFORMED, detail, row, r + "bad prompt_tokens '" + cols[1] + "'");
    case GSB_TRACE_DETAIL_OUTPUT:
      return fail(GSB_TRACE_KIND_MALFORMED, detail, row, r + "bad output_tokens '" + cols[2] + "'");
    case GSB_TRACE_DETAIL_RANGE:
      return fail(GSB_TRACE_KIND_MALFORMED, detail, row, r + "out-of-range field");
    case GSB_TRACE_DETAIL_MONOTONE:
      return fail(GSB_TRACE_KIND_NON_MONOTONE, detail, row, r + "arrivals must be non-decreasing");
    case GSB_TRACE_DETAIL_CLASS:
      return fail(GSB_TRACE_KIND_MALFORMED, detail, row, r + "class must be SM or L");
    default:
      return fail(GSB_TRACE_KIND_CLASS_MISMATCH, detail, row,
                  r + "class column disagrees with threshold " + std::to_string(class_threshold));
  }
}

int gsb_trace_format(gsb_ctx* ctx, int64_t n, const int64_t* d_arrival, const int32_t* d_prompt,
                     const int32_t* d_output, const uint8_t* d_slo_class, char* d_out,
                     int64_t cap_bytes, int64_t* h_bytes, void* stream) {
  if (!ctx || !h_bytes || n < 0) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "trace_format: bad arguments");
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  // has_class = all_of(requests, has cls): vacuously true for an empty trace (trace.cpp:134-137)
  const char* hdr = (d_slo_class || n == 0) ? kHdr4 : kHdr3;
  const int64_t hl = static_cast<int64_t>(strlen(hdr)) + 1;
  if (n == 0) {
    *h_bytes = hl;
    if (!d_out) return GSB_OK;
    if (cap_bytes < hl) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "trace_format: cap_bytes too small");
    std::string h = std::string(hdr) + "\n";
    cudaMemcpyAsync(d_out, h.data(), static_cast<size_t>(hl), cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    return gsb_check_launch(ctx, "trace_format");
  }
  size_t cub_tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_tmp, static_cast<unsigned long long*>(nullptr),
                                static_cast<unsigned long long*>(nullptr), static_cast<int>(n + 1), s);
  const size_t lens = static_cast<size_t>(n + 1) * sizeof(unsigned long long);
  char* scr = static_cast<char*>(gsb_scratch(ctx, 2 * lens + cub_tmp + 256));
  if (!scr) return gsb_set_error(ctx, GSB_CUDA_ERROR, "trace_format: scratch allocation failed");
  auto* len = reinterpret_cast<unsigned long long*>(scr);
  auto* off = len + (n + 1);
  void* d_cub = scr + ((2 * lens + 255) / 256) * 256;
  cudaMemsetAsync(len + n, 0, sizeof(unsigned long long), s);
  const unsigned g = static_cast<unsigned>((n + 255) / 256);
  k_csv_row_len<<<g, 256, 0, s>>>(n, d_arrival, d_prompt, d_output, d_slo_class, len);
  cub::DeviceScan::ExclusiveSum(d_cub, cub_tmp, len, off, static_cast<int>(n + 1), s);
  unsigned long long body = 0;
  cudaMemcpyAsync(&body, off + n, sizeof(body), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return gsb_check_launch(ctx, "trace_format");
  *h_bytes = hl + static_cast<int64_t>(body);
  if (!d_out) return GSB_OK;  // size query
  if (cap_bytes < *h_bytes) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "trace_format: cap_bytes too small");
  std::string h = std::string(hdr) + "\n";
  cudaMemcpyAsync(d_out, h.data(), static_cast<size_t>(hl), cudaMemcpyHostToDevice, s);
  k_csv_write<<<g, 256, 0, s>>>(n, hl, d_arrival, d_prompt, d_output, d_slo_class, off, d_out);
  cudaStreamSynchronize(s);
  return gsb_check_launch(ctx, "trace_format");
}

}  // extern "C"
