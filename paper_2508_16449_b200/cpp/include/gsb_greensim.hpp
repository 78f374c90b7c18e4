// gsb_greensim.hpp — the reference's C++ decision-engine API (namespace greensim), served by the
// sm_100a kernels of libgsb.so. Drop-in for the hot path of SURVEY.md §8(b): a program written
// against the reference headers
//   greensim/gpu_model.hpp   (types, gpu_model.hpp:11-91, minus fits / FLOPs)
//   greensim/router.hpp      (router.hpp:13-56)
//   greensim/prefill_opt.hpp (prefill_opt.hpp:13-88)
//   greensim/decode_ctl.hpp  (decode_ctl.hpp:13-165)
//   greensim/metrics.hpp     (quantile only, metrics.hpp:14-16)
//   greensim/trace.hpp       (Request / PromptClass, trace.hpp:12-22)
// compiles unchanged against paper_2508_16449_b200/cpp/include and links libgreensim_b200.so.
//
// Value semantics, argument meaning and the typed exceptions (ModelError, RouterError,
// std::invalid_argument) are the reference's. Every evaluation — routing, T_ref sums, window
// energies, the clock argmin, steady states, band tables, window statistics, and each
// DecodeController transition — is a libgsb kernel launch on the process's B200 (device 0, or
// $GSB_DEVICE); without a usable GPU every such call throws greensim::GpuError. Only argument
// validation, queue bookkeeping, the CSV renderer and the log auditor are host code.
#pragma once

#include <cstdint>
#include <deque>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

// Request / PromptClass / TraceError and quantile() come from greensim/trace.hpp and
// greensim/metrics.hpp: the minimal ones in ../include_min for the standalone drop-in, or the
// reference's own when its simulator is compiled over this library (paper_2508_16449_b200/cpp/
// Makefile, target sim).
#include "greensim/metrics.hpp"
#include "greensim/trace.hpp"

namespace greensim {

// ------------------------------------------------------------------ errors
struct ModelError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RouterError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// No B200 / libgsb failure (not in the reference: it has no device).
struct GpuError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ device models
struct FrequencyGrid {
  double f_min_mhz = 210.0;
  double f_max_mhz = 1410.0;
  double step_mhz = 15.0;
  double f_ref_mhz = 1410.0;

  void validate() const;
  bool on_grid(double f) const;
  std::size_t size() const;
  double at(std::size_t i) const;
  std::vector<double> frequencies() const;
  double clamp_to_grid(double f) const;
};

struct LatencyModel {
  double a = 0.0, b = 0.0, c = 0.0;
  double f_ref_mhz = 1410.0;
  void validate() const;
};

struct DecodeStepModel {
  double alpha0_ms = 0.0, alpha1_ms = 0.0, beta0_ms = 0.0, beta1_ms = 0.0;
  double f_ref_mhz = 1410.0;
  void validate() const;
};

struct PowerModel {
  double k3 = 0.0, k2 = 0.0, k1 = 0.0, k0 = 0.0;
  double p_idle_w = 0.0;
  double active_power_w(double f) const { return ((k3 * f + k2) * f + k1) * f + k0; }
  void validate(const FrequencyGrid& grid) const;
};

struct GpuProfile {
  std::string name = "default";
  FrequencyGrid grid;
  LatencyModel prefill;
  DecodeStepModel decode;
  PowerModel power;

  void validate() const;
  double prefill_latency_ms(double prompt_tokens, double f) const;
  double decode_step_ms(double batch, double f) const;
  double active_power_w(double f) const;
  double idle_power_w() const { return power.p_idle_w; }
  static GpuProfile default_profile();
};

double prefill_latency_raw_ms(const LatencyModel& m, double prompt_tokens, double f);
double decode_step_raw_ms(const DecodeStepModel& m, double batch, double f);

// ------------------------------------------------------------------ routing
struct RoutingConfig {
  bool enabled = true;
  std::vector<int> thresholds{1024};
  std::vector<int> worker_map{0, 1};
  int n_classes() const { return static_cast<int>(thresholds.size()) + 1; }
  void validate(int n_prefill_workers) const;
};

int classify(const RoutingConfig& cfg, int prompt_tokens);
// B200 batch form: one launch for a whole arrival batch.
std::vector<int> classify_batch(const RoutingConfig& cfg, std::span<const int> prompt_tokens);

class Dispatcher {
 public:
  explicit Dispatcher(const RoutingConfig& cfg);
  int dispatch(const Request& r);
  int n_queues() const { return static_cast<int>(lanes_.size()); }
  bool empty(int queue) const { return lanes_[static_cast<std::size_t>(queue)].empty(); }
  std::size_t size(int queue) const { return lanes_[static_cast<std::size_t>(queue)].size(); }
  std::int64_t front(int queue) const { return lanes_[static_cast<std::size_t>(queue)].front(); }
  std::int64_t pop(int queue);
  const std::deque<std::int64_t>& queue(int q) const { return lanes_[static_cast<std::size_t>(q)]; }

 private:
  RoutingConfig config_;
  std::vector<std::deque<std::int64_t>> lanes_;
  std::unordered_set<std::int64_t> dispatched_;
};

// ------------------------------------------------------------------ prefill objective
struct PrefillJob {
  std::int64_t request_id = 0;
  int prompt_tokens = 0;
  double deadline_ms = 0.0;
  double work_fraction = 1.0;
};

struct PrefillBatch {
  std::vector<PrefillJob> jobs;
  double t_ref_total_ms(const LatencyModel& m) const;
};

struct EnergyBreakdown {
  double active_j = 0.0, idle_j = 0.0, total_j = 0.0;
  bool feasible = true;
};

struct FrequencyChoice {
  double f_mhz = 0.0;
  double energy_j = 0.0;
};

double busy_time_ms(const PrefillBatch& batch, double f, const GpuProfile& profile);
EnergyBreakdown energy_total(const PrefillBatch& batch, double f, double window_ms,
                             const GpuProfile& profile);
double energy_total_closed_form_j(const PrefillBatch& batch, double f, double window_ms,
                                  const GpuProfile& profile);
std::optional<FrequencyChoice> select_frequency(const PrefillBatch& batch, double window_ms,
                                                const GpuProfile& profile);
// B200 batch form: every (batch, window) pair in one K2 launch.
std::vector<std::optional<FrequencyChoice>> select_frequency_batch(
    std::span<const PrefillBatch> batches, std::span<const double> windows_ms,
    const GpuProfile& profile);

struct QueueOptimizerConfig {
  double resolve_period_ms = 100.0;
  double margin_prefill = 0.95;
  double min_budget_ms = 100.0;
  double first_token_allowance_ms = 100.0;
};

struct ClassQueueSnapshot {
  int class_id = 0;
  PrefillBatch batch;
};

struct PrefillFreqCommand {
  int class_id = 0;
  double f_mhz = 0.0;
  double window_ms = 0.0;
  bool infeasible = false;
};

std::vector<PrefillFreqCommand> queue_optimizer_tick(const std::vector<ClassQueueSnapshot>& queues,
                                                     double now_ms, const QueueOptimizerConfig& cfg,
                                                     const GpuProfile& profile);

// ------------------------------------------------------------------ decode control
struct DecodeCtlConfig {
  double tslo_ms = 100.0;
  double margin_decode = 0.95;
  double fine_period_ms = 20.0;
  double coarse_period_ms = 200.0;
  double adapt_period_s = 6.0;
  double step_mhz = 15.0;
  double max_step_mhz = 30.0;
  int hysteresis_count = 3;
  double bias_threshold = 0.8;
  int tbt_window_tokens = 256;
  double tps_scale = 4.0;
  double upper_margin = 1.0;
  double lower_margin = 0.65;
  void validate() const;
};

struct DecodeSteadyState {
  bool sustainable = false;
  double batch = 0.0;
  double tbt_ms = 0.0;
};
DecodeSteadyState decode_steady_state(const GpuProfile& profile, double per_worker_tps, double f,
                                      int max_batch);

struct BandBucket {
  double tps_lo = 0.0;
  double tps_hi = 0.0;
  double f_opt_mhz = 0.0;
  bool feasible = true;
};

struct FreqBandTable {
  std::vector<BandBucket> buckets;
  int bucket_index(double tps) const;
  std::pair<double, double> band(int bucket, const FrequencyGrid& grid, double step_mhz) const;
  void validate() const;
};

FreqBandTable build_band_table(const GpuProfile& profile, std::span<const double> tps_levels,
                               double t_slo_ms, int decode_workers, int max_batch);

class TpsWindow {
 public:
  explicit TpsWindow(double window_ms = 200.0) : span_ms_(window_ms) {}
  void record(double t_ms, int tokens) { events_.emplace_back(t_ms, tokens); }
  double tps(double now_ms);

 private:
  double span_ms_;
  std::deque<std::pair<double, int>> events_;
};

class TbtWindow {
 public:
  explicit TbtWindow(int capacity = 256) : cap_(capacity) {}
  void record(double interval_ms);
  bool empty() const { return ring_.empty(); }
  double p95() const;

 private:
  int cap_;
  std::deque<double> ring_;
};

struct DecisionRecord {
  double tick_ms = 0.0;
  int worker = 0;
  double tps = 0.0;
  double p95_tbt_ms = 0.0;
  int bucket = 0;
  double band_lo = 0.0;
  double band_hi = 0.0;
  double command_mhz = 0.0;
  std::string action;
};

// Each call is one launch of the scripted controller kernel, resumed from the controller's
// device-format state (gsb_ctl_state) — the same transition code as the batched replay (K3b).
class DecodeController {
 public:
  DecodeController(const DecodeCtlConfig& cfg, FreqBandTable table, const FrequencyGrid& grid,
                   int worker_id);
  double on_fine_tick(double now_ms, std::optional<double> p95_tbt_ms);
  void on_coarse_tick(double now_ms, double worker_tps);
  void on_adapt_tick(double now_ms);
  double command() const { return command_; }
  const std::vector<DecisionRecord>& log() const { return log_; }
  const FreqBandTable& table() const { return table_; }
  int current_bucket() const { return bucket_; }

 private:
  void step(int kind, double now_ms, double value, bool has);

  DecodeCtlConfig cfg_;
  FreqBandTable table_;  // the controller's own copy; adaptation rewrites f_opt
  FrequencyGrid grid_;
  int worker_;
  std::vector<unsigned char> state_;  // opaque gsb_ctl_state
  std::vector<DecisionRecord> log_;
  double command_ = 0.0;
  int bucket_ = 0;
};

std::string decision_log_csv(std::span<const DecisionRecord> records);

struct AuditResult {
  int violations = 0;
  std::vector<std::string> messages;
};
AuditResult audit_decision_log(std::span<const DecisionRecord> records, const DecodeCtlConfig& cfg);

}  // namespace greensim
