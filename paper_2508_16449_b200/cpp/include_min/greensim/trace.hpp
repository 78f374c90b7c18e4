// Minimal greensim/trace.hpp for the standalone drop-in: the request record the router reads and
// the trace CSV reader/writer (reference proj/include/greensim/trace.hpp:12-40, 54-58). The
// generators are not on the decision-engine path. A build that links the reference's own simulator puts the
// reference's full trace.hpp on the include path instead of this directory.
#pragma once

#include <cstdint>
#include <filesystem>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace greensim {

enum class PromptClass { ShortMedium = 0, Long = 1 };

struct Request {
  std::int64_t id = 0;
  std::int64_t arrival_ms = 0;
  int prompt_tokens = 0;
  int output_tokens = 0;
  std::optional<PromptClass> cls;
};

const char* prompt_class_name(PromptClass c);

struct TraceMeta {  // trace.hpp:24-28
  std::string name;
  std::int64_t duration_ms = 0;  // >= last arrival
  double nominal_qps = 0.0;
};

struct Trace {  // trace.hpp:30-33
  std::vector<Request> requests;
  TraceMeta meta;
};

struct TraceError : std::runtime_error {
  enum class Kind { EmptyTrace, NonMonotoneArrivals, MalformedRow, BadHeader, ClassMismatch, BadShape };
  TraceError(Kind k, const std::string& msg) : std::runtime_error(msg), kind(k) {}
  Kind kind;
};

// trace.hpp:54-58; on the B200 both are K6 kernels (gsb_trace_parse / gsb_trace_format).
Trace load_trace(const std::filesystem::path& path, int class_threshold = 1024);
void save_trace_csv(const Trace& trace, const std::filesystem::path& path);

}  // namespace greensim
