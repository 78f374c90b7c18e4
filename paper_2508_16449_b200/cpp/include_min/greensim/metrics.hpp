// Minimal greensim/metrics.hpp for the standalone drop-in: the nearest-rank quantile behind the
// TBT-window P95 (reference proj/include/greensim/metrics.hpp:14-16), computed on the GPU by
// gsb_quantile_batch. Run summaries are not on the decision-engine path.
#pragma once

#include <span>
#include <stdexcept>

namespace greensim {

double quantile(std::span<const double> samples, double q);

}  // namespace greensim
