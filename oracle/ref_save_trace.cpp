// TEST INFRASTRUCTURE ONLY: runs the reference's greensim::save_trace_csv (trace.cpp:131-145)
// in its own process (the reference's ofstream path does not survive being dlopen'ed into the
// Python interpreter). Input: a raw file of  n (i64) | arrival i64[n] | prompt i32[n] |
// output i32[n] | has_cls (u8) | cls u8[n];  output: the CSV written by the reference.
// `--decisions IN OUT`: IN = n (i64) | n decision records in the gsb_decision layout (64 B);
// OUT = the reference's decision_log_csv of them (its ostringstream path, same reason).
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "greensim/trace.hpp"

extern "C" int64_t ref_decision_log_csv(int64_t n, const void* rec, char* out, int64_t cap);

static int decisions(const char* in, const char* out) {
  FILE* f = std::fopen(in, "rb");
  if (!f) return 3;
  int64_t n = 0;
  if (std::fread(&n, 8, 1, f) != 1) return 4;
  std::vector<unsigned char> rec(static_cast<size_t>(n) * 64);
  if (std::fread(rec.data(), 1, rec.size(), f) != rec.size()) return 5;
  std::fclose(f);
  const int64_t k = ref_decision_log_csv(n, rec.data(), nullptr, 0);
  std::vector<char> buf(static_cast<size_t>(k));
  ref_decision_log_csv(n, rec.data(), buf.data(), k);
  FILE* o = std::fopen(out, "wb");
  if (!o) return 6;
  std::fwrite(buf.data(), 1, buf.size(), o);
  std::fclose(o);
  return 0;
}

int main(int argc, char** argv) {
  if (argc == 4 && std::string(argv[1]) == "--decisions") return decisions(argv[2], argv[3]);
  if (argc != 3) return 2;
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 3;
  int64_t n = 0;
  if (std::fread(&n, 8, 1, f) != 1) return 4;
  std::vector<int64_t> a(static_cast<size_t>(n));
  std::vector<int32_t> p(static_cast<size_t>(n)), o(static_cast<size_t>(n));
  std::vector<uint8_t> c(static_cast<size_t>(n));
  uint8_t has = 0;
  const size_t un = static_cast<size_t>(n);
  if (std::fread(a.data(), 8, un, f) != un || std::fread(p.data(), 4, un, f) != un ||
      std::fread(o.data(), 4, un, f) != un || std::fread(&has, 1, 1, f) != 1 ||
      std::fread(c.data(), 1, un, f) != un)
    return 5;
  std::fclose(f);
  greensim::Trace t;
  t.requests.resize(un);
  for (size_t i = 0; i < un; ++i) {
    auto& r = t.requests[i];
    r.id = static_cast<int64_t>(i);
    r.arrival_ms = a[i];
    r.prompt_tokens = p[i];
    r.output_tokens = o[i];
    if (has) r.cls = static_cast<greensim::PromptClass>(c[i]);
  }
  greensim::save_trace_csv(t, argv[2]);
  return 0;
}
