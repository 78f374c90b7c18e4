/*
 * gs_trace.c — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference's trace CSV reader and writer, sequential like the
 * reference (std::getline over the file):
 *   greensim::load_trace      proj/src/trace.cpp:56-129
 *   greensim::save_trace_csv  proj/src/trace.cpp:131-145
 *   classify_by_threshold     proj/src/trace.cpp:32-34
 * Pinned against the reference (oracle/_ref: ref_load_trace, and the ref_save_trace tool) on
 * valid and malformed fixtures by tests/test_oracle_trace.py.
 */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "gs_oracle.h"

static const char kH3[] = "arrival_ms,prompt_tokens,output_tokens";
static const char kH4[] = "arrival_ms,prompt_tokens,output_tokens,class";

static void set_err(gso_trace_err* e, int kind, int detail, int64_t row, const char* msg) {
  e->kind = kind;
  e->detail = detail;
  e->row = row;
  snprintf(e->msg, sizeof(e->msg), "%s", msg);
}

/* std::from_chars<int64_t> over the whole field (trace.cpp:84-91) */
static int parse_i64(const char* p, int64_t len, int64_t* out) {
  int64_t i = 0;
  int neg = 0;
  if (len > 0 && p[0] == '-') {
    neg = 1;
    i = 1;
  }
  if (i >= len) return 0;
  unsigned long long v = 0;
  for (; i < len; ++i) {
    const unsigned d = (unsigned)(unsigned char)p[i] - '0';
    if (d > 9) return 0;
    const unsigned long long lim = neg ? 0x8000000000000000ull : 0x7fffffffffffffffull;
    if (v > (lim - d) / 10) return 0; /* v*10 + d > lim: result_out_of_range */
    v = v * 10 + d;
  }
  *out = neg ? (int64_t)(0ull - v) : (int64_t)v;
  return 1;
}

/* std::getline(ss, col, ','): a trailing ',' yields no empty last column */
static int split_cols(const char* s, int64_t len, int64_t* fs, int64_t* fl) {
  int n = 0;
  int64_t f0 = 0;
  for (int64_t i = 0; i <= len; ++i) {
    if (i == len || s[i] == ',') {
      if (i == len && i == f0 && n > 0) break;
      if (n < 4) {
        fs[n] = f0;
        fl[n] = i - f0;
      }
      ++n;
      f0 = i + 1;
    }
  }
  return n;
}

int64_t gso_trace_parse(const char* b, int64_t n, int32_t thr, int64_t cap, int64_t* arrival,
                        int32_t* prompt, int32_t* output, uint8_t* cls, int32_t* has_class,
                        gso_trace_err* err) {
  memset(err, 0, sizeof(*err));
  err->row = -1;
  if (n <= 0) { /* the first getline fails */
    set_err(err, GSO_TRACE_EMPTY, 0, -1, "empty trace file");
    return -1;
  }
  int64_t pos = 0, row = 0, nr = 0, prev = -1;
  int hc = -1;
  char msg[8192];
  while (pos < n) { /* one std::getline per iteration */
    int64_t e = pos;
    while (e < n && b[e] != '\n') ++e;
    const int64_t st = pos;
    int64_t len = e - st;
    pos = e + 1; /* past the '\n' (or past the end) */
    ++row;
    if (len > 0 && b[st + len - 1] == '\r') --len;
    const char* s = b + st;
    if (row == 1) { /* header, trace.cpp:63-74 */
      if (len == (int64_t)sizeof(kH3) - 1 && memcmp(s, kH3, (size_t)len) == 0) {
        hc = 0;
      } else if (len == (int64_t)sizeof(kH4) - 1 && memcmp(s, kH4, (size_t)len) == 0) {
        hc = 1;
      } else {
        int k = snprintf(msg, sizeof(msg), "unrecognized trace header: ");
        int64_t c = len < (int64_t)sizeof(msg) - k - 1 ? len : (int64_t)sizeof(msg) - k - 1;
        memcpy(msg + k, s, (size_t)c);
        msg[k + c] = 0;
        set_err(err, GSO_TRACE_BAD_HEADER, 0, 1, msg);
        return -1;
      }
      *has_class = hc;
      continue;
    }
    if (len == 0) continue; /* empty line: skipped, row counted */
    int64_t fs[4], fl[4];
    const int ncols = split_cols(s, len, fs, fl);
    const int expect = hc ? 4 : 3;
    if (ncols != expect) {
      snprintf(msg, sizeof(msg), "row %lld: expected %d columns, got %d", (long long)row, expect,
               ncols);
      set_err(err, GSO_TRACE_MALFORMED, 1, row, msg);
      return -1;
    }
    int64_t v[3];
    static const char* what[3] = {"arrival_ms", "prompt_tokens", "output_tokens"};
    for (int k = 0; k < 3; ++k) {
      if (!parse_i64(s + fs[k], fl[k], &v[k])) {
        int w = snprintf(msg, sizeof(msg), "row %lld: bad %s '", (long long)row, what[k]);
        int64_t c = fl[k] < (int64_t)sizeof(msg) - w - 2 ? fl[k] : (int64_t)sizeof(msg) - w - 2;
        memcpy(msg + w, s + fs[k], (size_t)c);
        msg[w + c] = '\'';
        msg[w + c + 1] = 0;
        set_err(err, GSO_TRACE_MALFORMED, 2 + k, row, msg);
        return -1;
      }
    }
    const int32_t pi = (int32_t)(uint32_t)(uint64_t)v[1]; /* static_cast<int>, trace.cpp:98 */
    const int32_t oi = (int32_t)(uint32_t)(uint64_t)v[2];
    if (v[0] < 0 || pi < 1 || oi < 1) {
      snprintf(msg, sizeof(msg), "row %lld: out-of-range field", (long long)row);
      set_err(err, GSO_TRACE_MALFORMED, 5, row, msg);
      return -1;
    }
    if (v[0] < prev) {
      snprintf(msg, sizeof(msg), "row %lld: arrivals must be non-decreasing", (long long)row);
      set_err(err, GSO_TRACE_NON_MONOTONE, 6, row, msg);
      return -1;
    }
    prev = v[0];
    const uint8_t c = pi <= thr ? 0 : 1; /* classify_by_threshold */
    if (hc) {
      const char* q = s + fs[3];
      int fc = -1;
      if (fl[3] == 2 && q[0] == 'S' && q[1] == 'M') fc = 0;
      if (fl[3] == 1 && q[0] == 'L') fc = 1;
      if (fc < 0) {
        snprintf(msg, sizeof(msg), "row %lld: class must be SM or L", (long long)row);
        set_err(err, GSO_TRACE_MALFORMED, 7, row, msg);
        return -1;
      }
      if (fc != c) {
        snprintf(msg, sizeof(msg), "row %lld: class column disagrees with threshold %d",
                 (long long)row, thr);
        set_err(err, GSO_TRACE_CLASS_MISMATCH, 8, row, msg);
        return -1;
      }
    }
    if (nr < cap) {
      arrival[nr] = v[0];
      prompt[nr] = pi;
      output[nr] = oi;
      cls[nr] = c;
    }
    ++nr;
  }
  if (nr == 0) {
    set_err(err, GSO_TRACE_EMPTY, 0, -1, "trace has no rows");
    return -1;
  }
  return nr;
}

int64_t gso_trace_format(int64_t n, const int64_t* a, const int32_t* p, const int32_t* o,
                         const uint8_t* cls, char* out, int64_t cap) {
  int64_t w = 0;
  char line[96];
  /* all_of over the requests' classes: vacuously true for an empty trace (trace.cpp:134-137) */
  int k = snprintf(line, sizeof(line), "%s\n", (cls || n == 0) ? kH4 : kH3);
  if (out && w + k <= cap) memcpy(out + w, line, (size_t)k);
  w += k;
  for (int64_t r = 0; r < n; ++r) {
    if (cls)
      k = snprintf(line, sizeof(line), "%lld,%d,%d,%s\n", (long long)a[r], p[r], o[r],
                   cls[r] == 0 ? "SM" : "L");
    else
      k = snprintf(line, sizeof(line), "%lld,%d,%d\n", (long long)a[r], p[r], o[r]);
    if (out && w + k <= cap) memcpy(out + w, line, (size_t)k);
    w += k;
  }
  return w;
}
