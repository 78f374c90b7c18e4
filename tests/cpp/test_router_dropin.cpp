// Router checks of the C++ drop-in (the reference's proj/tests/test_router.cpp cases 1-4 restated;
// its case 5 runs the full simulator, which is outside the decision-engine path), plus batch-form
// consistency checks of the B200 entry points against their single-call forms.
#include <doctest.h>

#include <random>

#include "greensim/decode_ctl.hpp"
#include "greensim/prefill_opt.hpp"
#include "greensim/router.hpp"

using namespace greensim;

namespace {
Request make_req(std::int64_t id, std::int64_t t, int prompt) {
  Request r;
  r.id = id;
  r.arrival_ms = t;
  r.prompt_tokens = prompt;
  r.output_tokens = 8;
  return r;
}
}  // namespace

TEST_CASE("router: thresholds are inclusive on the lower class") {
  RoutingConfig two;
  CHECK(classify(two, 1) == 0);
  CHECK(classify(two, 1024) == 0);
  CHECK(classify(two, 1025) == 1);
  CHECK(classify(two, 1 << 20) == 1);
  RoutingConfig four;
  four.thresholds = {256, 1024, 4096};
  four.worker_map = {0, 1, 2, 3};
  CHECK(classify(four, 256) == 0);
  CHECK(classify(four, 257) == 1);
  CHECK(classify(four, 4096) == 2);
  CHECK(classify(four, 4097) == 3);
}

TEST_CASE("router: per-class FIFO, single dispatch per id") {
  Dispatcher d{RoutingConfig{}};
  REQUIRE(d.n_queues() == 2);
  CHECK(d.dispatch(make_req(10, 0, 64)) == 0);
  CHECK(d.dispatch(make_req(11, 1, 5000)) == 1);
  CHECK(d.dispatch(make_req(12, 2, 1024)) == 0);
  CHECK(d.size(0) == 2);
  CHECK(d.front(0) == 10);
  CHECK(d.pop(0) == 10);
  CHECK(d.front(0) == 12);
  CHECK_FALSE(d.empty(1));
  CHECK_THROWS_AS(d.dispatch(make_req(11, 3, 64)), RouterError);
  Dispatcher e{RoutingConfig{}};
  const int prompts[] = {3000, 10, 20, 4000, 30};
  for (int i = 0; i < 5; ++i) e.dispatch(make_req(i, i, prompts[i]));
  CHECK(e.queue(0) == std::deque<std::int64_t>{1, 2, 4});
  CHECK(e.queue(1) == std::deque<std::int64_t>{0, 3});
}

TEST_CASE("router: disabled routing is one queue") {
  RoutingConfig off;
  off.enabled = false;
  Dispatcher d(off);
  CHECK(d.n_queues() == 1);
  CHECK(d.dispatch(make_req(0, 0, 9000)) == 0);
  CHECK(d.dispatch(make_req(1, 0, 9)) == 0);
}

TEST_CASE("router: validation") {
  RoutingConfig c;
  c.thresholds = {512, 512};
  CHECK_THROWS_AS(c.validate(2), RouterError);
  c.thresholds = {900, 100};
  CHECK_THROWS_AS(c.validate(2), RouterError);
  c.thresholds = {0};
  CHECK_THROWS_AS(c.validate(2), RouterError);
  c = RoutingConfig{};
  c.worker_map = {1, 1};
  CHECK_THROWS_AS(c.validate(2), RouterError);
  c.worker_map = {0, 1, 0};
  CHECK_THROWS_AS(c.validate(2), RouterError);
  c.worker_map = {0, 2};
  CHECK_THROWS_AS(c.validate(2), RouterError);
  c = RoutingConfig{};
  CHECK_NOTHROW(c.validate(2));
  c.enabled = false;
  c.worker_map = {};
  CHECK_NOTHROW(c.validate(5));
}

TEST_CASE("batch forms equal the single-call forms") {
  RoutingConfig cfg;
  cfg.thresholds = {128, 1024, 8192};
  cfg.worker_map = {0, 1, 2, 3};
  std::mt19937 rng(7);
  std::uniform_int_distribution<int> Ld(1, 20000);
  std::vector<int> prompts(3000);
  for (int& p : prompts) p = Ld(rng);
  const std::vector<int> cls = classify_batch(cfg, prompts);
  int mismatches = 0;
  for (std::size_t i = 0; i < prompts.size(); i += 97) mismatches += cls[i] != classify(cfg, prompts[i]);
  CHECK(mismatches == 0);

  const GpuProfile p = GpuProfile::default_profile();
  std::vector<PrefillBatch> batches;
  std::vector<double> windows;
  std::uniform_int_distribution<int> nd(1, 6);
  std::uniform_real_distribution<double> Wd(20.0, 5000.0);
  for (int b = 0; b < 200; ++b) {
    PrefillBatch pb;
    for (int k = 0, n = nd(rng); k < n; ++k) pb.jobs.push_back(PrefillJob{k, Ld(rng) % 8192 + 1, 0.0, 1.0});
    batches.push_back(pb);
    windows.push_back(Wd(rng));
  }
  const auto all = select_frequency_batch(batches, windows, p);
  for (std::size_t b = 0; b < batches.size(); b += 13) {
    const auto one = select_frequency(batches[b], windows[b], p);
    REQUIRE(one.has_value() == all[b].has_value());
    if (one) {
      CHECK(one->f_mhz == all[b]->f_mhz);
      CHECK(one->energy_j == all[b]->energy_j);
    }
  }
  CHECK_THROWS_AS(select_frequency(PrefillBatch{}, 100.0, p), ModelError);
  CHECK_THROWS_AS(busy_time_ms(batches[0], 211.0, p), ModelError);
}

TEST_CASE("decode controller: quantile and window helpers") {
  std::vector<double> v;
  for (int i = 100; i >= 1; --i) v.push_back(i);
  CHECK(quantile(v, 0.0) == 1.0);
  CHECK(quantile(v, 0.95) == 95.0);
  CHECK(quantile(v, 1.0) == 100.0);
  CHECK_THROWS_AS(quantile(std::vector<double>{}, 0.5), std::invalid_argument);
  CHECK_THROWS_AS(quantile(v, 1.5), std::invalid_argument);
  // any set size, as metrics.cpp:11-19 (io.cpp's tbt_digest passes a request's whole TBT list)
  std::vector<double> big;
  for (int i = 0; i < 50000; ++i) big.push_back(static_cast<double>((i * 7919) % 50000) * 0.5 - 3.0);
  CHECK(quantile(big, 0.0) == -3.0);
  CHECK(quantile(big, 0.95) == 47500.0 * 0.5 - 3.0 - 0.5);
  CHECK(quantile(big, 1.0) == 49999.0 * 0.5 - 3.0);
}
