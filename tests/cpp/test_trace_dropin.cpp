// Trace CSV checks of the C++ drop-in (greensim::load_trace / save_trace_csv over K6): the
// reference's proj/tests/test_trace.cpp cases 1-2 restated (its generator cases exercise code
// that is not on the decision-engine path), plus the reference's messages, row counter and
// meta fields.
#include <doctest.h>

#include <cstdio>
#include <filesystem>
#include <fstream>
#include <random>
#include <string>

#include "greensim/trace.hpp"

using namespace greensim;
namespace fs = std::filesystem;

namespace {
fs::path put(const std::string& name, const std::string& body) {
  const fs::path p = fs::temp_directory_path() / name;
  std::ofstream(p, std::ios::binary) << body;
  return p;
}

std::string load_error(const fs::path& p, TraceError::Kind* kind = nullptr, int thr = 1024) {
  try {
    (void)load_trace(p, thr);
  } catch (const TraceError& e) {
    if (kind) *kind = e.kind;
    return e.what();
  }
  return "";
}
}  // namespace

TEST_CASE("load_trace on the GPU: classes, order, errors (test_trace.cpp case 1)") {
  const Trace t = load_trace(put("gsb_t_good.csv",
                                 "arrival_ms,prompt_tokens,output_tokens\n0,512,128\n100,2048,256\n"));
  REQUIRE(t.requests.size() == 2);
  CHECK(t.requests[0].cls == PromptClass::ShortMedium);
  CHECK(t.requests[1].cls == PromptClass::Long);
  CHECK(t.requests[1].arrival_ms == 100);
  CHECK(t.requests[1].id == 1);
  CHECK(t.meta.name == "gsb_t_good");
  CHECK(t.meta.duration_ms == 100);
  CHECK(t.meta.nominal_qps == doctest::Approx(20.0));

  TraceError::Kind k{};
  CHECK(load_error(put("gsb_t_empty.csv", "arrival_ms,prompt_tokens,output_tokens\n"), &k) ==
        "trace has no rows");
  CHECK(k == TraceError::Kind::EmptyTrace);
  CHECK(load_error(put("gsb_t_void.csv", ""), &k) == "empty trace file");
  CHECK(load_error(put("gsb_t_unordered.csv",
                       "arrival_ms,prompt_tokens,output_tokens\n100,512,128\n50,512,128\n"),
                   &k) == "row 3: arrivals must be non-decreasing");
  CHECK(k == TraceError::Kind::NonMonotoneArrivals);
  CHECK(load_error(put("gsb_t_malformed.csv", "arrival_ms,prompt_tokens,output_tokens\n0,512\n"),
                   &k) == "row 2: expected 3 columns, got 2");
  CHECK(k == TraceError::Kind::MalformedRow);
  CHECK(load_error(put("gsb_t_header.csv", "time,prompt,output\n0,512,128\n"), &k) ==
        "unrecognized trace header: time,prompt,output");
  CHECK(k == TraceError::Kind::BadHeader);
  CHECK(load_error(put("gsb_t_class.csv",
                       "arrival_ms,prompt_tokens,output_tokens,class\n0,2048,128,SM\n"),
                   &k) == "row 2: class column disagrees with threshold 1024");
  CHECK(k == TraceError::Kind::ClassMismatch);
  CHECK(load_error(put("gsb_t_field.csv",
                       "arrival_ms,prompt_tokens,output_tokens\r\n\r\n0,1,1\r\n1,x2,1\r\n")) ==
        "row 4: bad prompt_tokens 'x2'");
  CHECK(load_error(fs::temp_directory_path() / "gsb_t_missing_file.csv", &k) ==
        "cannot open trace file: " + (fs::temp_directory_path() / "gsb_t_missing_file.csv").string());
}

TEST_CASE("trace CSV round trip on the GPU (test_trace.cpp case 2)") {
  std::mt19937_64 rng(11);
  Trace t;
  int64_t now = 0;
  for (int i = 0; i < 20000; ++i) {
    Request r;
    r.id = i;
    now += static_cast<int64_t>(rng() % 400);
    r.arrival_ms = now;
    r.prompt_tokens = 1 + static_cast<int>(rng() % 6000);
    r.output_tokens = 1 + static_cast<int>(rng() % 512);
    r.cls = r.prompt_tokens <= 1024 ? PromptClass::ShortMedium : PromptClass::Long;
    t.requests.push_back(r);
  }
  const fs::path p = fs::temp_directory_path() / "gsb_t_roundtrip.csv";
  save_trace_csv(t, p);
  const Trace back = load_trace(p);
  REQUIRE(back.requests.size() == t.requests.size());
  for (std::size_t i = 0; i < t.requests.size(); ++i) {
    CHECK(back.requests[i].arrival_ms == t.requests[i].arrival_ms);
    CHECK(back.requests[i].prompt_tokens == t.requests[i].prompt_tokens);
    CHECK(back.requests[i].output_tokens == t.requests[i].output_tokens);
    CHECK(back.requests[i].cls == t.requests[i].cls);
  }
  // without classes: no class column, and the loader classifies by the threshold
  for (auto& r : t.requests) r.cls.reset();
  save_trace_csv(t, p);
  std::ifstream in(p);
  std::string header;
  std::getline(in, header);
  CHECK(header == "arrival_ms,prompt_tokens,output_tokens");
  const Trace back2 = load_trace(p, 2000);
  CHECK(back2.requests[5].cls == (t.requests[5].prompt_tokens <= 2000 ? PromptClass::ShortMedium
                                                                       : PromptClass::Long));
}
