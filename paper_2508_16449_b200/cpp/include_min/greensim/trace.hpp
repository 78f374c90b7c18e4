// Minimal greensim/trace.hpp for the standalone drop-in: the request record the router reads
// (reference proj/include/greensim/trace.hpp:12-22, 36-40). Trace I/O and the generators are not
// on the decision-engine path. A build that links the reference's own simulator puts the
// reference's full trace.hpp on the include path instead of this directory.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>

namespace greensim {

enum class PromptClass { ShortMedium = 0, Long = 1 };

struct Request {
  std::int64_t id = 0;
  std::int64_t arrival_ms = 0;
  int prompt_tokens = 0;
  int output_tokens = 0;
  std::optional<PromptClass> cls;
};

struct TraceError : std::runtime_error {
  enum class Kind { EmptyTrace, NonMonotoneArrivals, MalformedRow, BadHeader, ClassMismatch, BadShape };
  TraceError(Kind k, const std::string& msg) : std::runtime_error(msg), kind(k) {}
  Kind kind;
};

}  // namespace greensim
