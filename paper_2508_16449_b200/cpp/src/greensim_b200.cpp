// greensim_b200.cpp — the reference's C++ decision-engine API over libgsb.so (include/gsb.h).
//
// Every evaluation is a libgsb kernel launch: one call = one packed host->device copy of its
// inputs, the launch(es), one device->host copy of its outputs. Host code here is limited to
// argument validation (the reference's exception rules), queue / ring bookkeeping, grid and
// table accessors, the CSV renderer and the log auditor. Reference semantics cited per function
// (paths under /root/reference/proj).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <limits>
#include <map>
#include <mutex>
#include <set>
#include <sstream>

#include "gsb.h"
#include "gsb_greensim.hpp"

namespace greensim {
namespace {

// ------------------------------------------------------------------ device runtime
// One libgsb context per process (device 0 or $GSB_DEVICE), guarded by a mutex, plus a
// grow-only device staging buffer. Deliberately never torn down: CUDA's own static teardown
// may already have run when static destructors execute.
struct Runtime {
  std::mutex mu;
  gsb_ctx* ctx = nullptr;
  void* d_buf = nullptr;
  size_t d_cap = 0;
  unsigned char* h_pin = nullptr;  // page-locked mirror of d_buf (async DMA both ways)
  size_t h_cap = 0;
  gsb_profile installed{};
  bool has_installed = false;
};

Runtime& runtime() {
  static Runtime* r = new Runtime;
  return *r;
}

[[noreturn]] void raise(int status, const std::string& msg) {
  switch (status) {
    case GSB_MODEL_ERROR: throw ModelError(msg);
    case GSB_ROUTER_ERROR: throw RouterError(msg);
    case GSB_TRACE_ERROR: throw TraceError(TraceError::Kind::BadShape, msg);
    case GSB_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw GpuError("libgsb: " + msg);
  }
}

void check(gsb_ctx* ctx, int rc) {
  if (rc != GSB_OK) raise(rc, ctx ? gsb_last_error(ctx) : gsb_status_string(rc));
}

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// One API call's device traffic. Segments are laid out in one buffer: pure inputs first, then
// in/out and output segments. commit() uploads the whole image in ONE copy; fetch() brings the
// output tail back in ONE copy and synchronizes.
class Call {
 public:
  Call() : rt_(runtime()), lock_(rt_.mu) {
    if (!rt_.ctx) {
      const char* env = std::getenv("GSB_DEVICE");
      const int dev = env ? std::atoi(env) : 0;
      const int rc = gsb_ctx_create(dev, &rt_.ctx);
      if (rc != GSB_OK) {
        rt_.ctx = nullptr;
        throw GpuError("libgsb: no usable sm_100 device (gsb_ctx_create failed); the B200 "
                       "drop-in has no CPU path");
      }
    }
  }
  gsb_ctx* ctx() const { return rt_.ctx; }

  size_t in(const void* host, size_t bytes) {
    const size_t off = reserve(bytes);
    if (bytes) std::memcpy(image_.data() + off, host, bytes);
    return off;
  }
  template <class T>
  size_t in_vec(const std::vector<T>& v) { return in(v.data(), v.size() * sizeof(T)); }
  size_t out(size_t bytes) {
    if (first_out_ == npos) first_out_ = image_.size();
    return reserve(bytes);
  }
  size_t inout(const void* host, size_t bytes) {
    if (first_out_ == npos) first_out_ = image_.size();
    return in(host, bytes);
  }

  void commit() {
    const size_t total = std::max<size_t>(image_.size(), kAlign);
    if (total > rt_.d_cap) {  // every earlier call has synchronized: the buffers are idle
      gsb_free(rt_.ctx, rt_.d_buf);
      gsb_host_free(rt_.ctx, rt_.h_pin);
      rt_.d_buf = nullptr;
      rt_.h_pin = nullptr;
      rt_.d_cap = rt_.h_cap = 0;
      const size_t cap = std::max<size_t>(total * 2, size_t{1} << 20);
      check(rt_.ctx, gsb_malloc(rt_.ctx, cap, &rt_.d_buf));
      void* h = nullptr;
      check(rt_.ctx, gsb_host_alloc(rt_.ctx, cap, &h));
      rt_.h_pin = static_cast<unsigned char*>(h);
      rt_.d_cap = rt_.h_cap = cap;
    }
    std::memcpy(rt_.h_pin, image_.data(), image_.size());
    check(rt_.ctx, gsb_memcpy(rt_.ctx, rt_.d_buf, rt_.h_pin, image_.size(), 0, nullptr));
  }
  template <class T>
  T* dev(size_t off) const { return reinterpret_cast<T*>(static_cast<unsigned char*>(rt_.d_buf) + off); }

  void fetch() {
    const bool tail = first_out_ != npos && first_out_ < image_.size();
    if (tail)
      check(rt_.ctx, gsb_memcpy(rt_.ctx, rt_.h_pin + first_out_, dev<unsigned char>(first_out_),
                                image_.size() - first_out_, 1, nullptr));
    check(rt_.ctx, gsb_synchronize(rt_.ctx));
    if (tail) std::memcpy(image_.data() + first_out_, rt_.h_pin + first_out_, image_.size() - first_out_);
  }
  template <class T>
  const T* host(size_t off) const { return reinterpret_cast<const T*>(image_.data() + off); }

  // Profile tables for the prefill kernels; re-installed only when the profile changes.
  // Unchecked: the reference's evaluators never call GpuProfile::validate.
  void install(const gsb_profile& p) {
    if (rt_.has_installed && std::memcmp(&rt_.installed, &p, sizeof p) == 0) return;
    // ASYNC: every launch of this library goes to the context's stream, behind the upload
    check(rt_.ctx, gsb_set_profiles_ex(rt_.ctx, 1, &p, GSB_PROFILES_UNCHECKED | GSB_PROFILES_ASYNC));
    rt_.installed = p;
    rt_.has_installed = true;
  }

 private:
  static constexpr size_t npos = static_cast<size_t>(-1);
  size_t reserve(size_t bytes) {
    const size_t off = image_.size();
    image_.resize(off + align_up(std::max<size_t>(bytes, 1)));
    return off;
  }
  Runtime& rt_;
  std::lock_guard<std::mutex> lock_;
  std::vector<unsigned char> image_;
  size_t first_out_ = npos;
};

gsb_profile to_c(const GpuProfile& p) {
  gsb_profile c;
  std::memset(&c, 0, sizeof c);
  c.f_min_mhz = p.grid.f_min_mhz;
  c.f_max_mhz = p.grid.f_max_mhz;
  c.step_mhz = p.grid.step_mhz;
  c.f_ref_mhz = p.grid.f_ref_mhz;
  c.lat_a = p.prefill.a;
  c.lat_b = p.prefill.b;
  c.lat_c = p.prefill.c;
  c.lat_f_ref_mhz = p.prefill.f_ref_mhz;
  c.dec_alpha0_ms = p.decode.alpha0_ms;
  c.dec_alpha1_ms = p.decode.alpha1_ms;
  c.dec_beta0_ms = p.decode.beta0_ms;
  c.dec_beta1_ms = p.decode.beta1_ms;
  c.dec_f_ref_mhz = p.decode.f_ref_mhz;
  c.k3 = p.power.k3;
  c.k2 = p.power.k2;
  c.k1 = p.power.k1;
  c.k0 = p.power.k0;
  c.p_idle_w = p.power.p_idle_w;
  return c;
}

gsb_ctl_cfg to_c(const DecodeCtlConfig& d) {
  gsb_ctl_cfg c;
  std::memset(&c, 0, sizeof c);
  c.tslo_ms = d.tslo_ms;
  c.margin_decode = d.margin_decode;
  c.fine_period_ms = d.fine_period_ms;
  c.coarse_period_ms = d.coarse_period_ms;
  c.adapt_period_s = d.adapt_period_s;
  c.step_mhz = d.step_mhz;
  c.max_step_mhz = d.max_step_mhz;
  c.hysteresis_count = d.hysteresis_count;
  c.tbt_window_tokens = d.tbt_window_tokens;
  c.bias_threshold = d.bias_threshold;
  c.tps_scale = d.tps_scale;
  c.upper_margin = d.upper_margin;
  c.lower_margin = d.lower_margin;
  return c;
}

// Ragged job arrays (CSR) of a set of batches, as the batch kernels take them.
struct Jobs {
  std::vector<int64_t> off{0};
  std::vector<int32_t> prompt;
  std::vector<double> wf, deadline;
  void add(const PrefillBatch& b, bool deadlines) {
    for (const PrefillJob& j : b.jobs) {
      prompt.push_back(j.prompt_tokens);
      wf.push_back(j.work_fraction);
      if (deadlines) deadline.push_back(j.deadline_ms);
    }
    off.push_back(static_cast<int64_t>(prompt.size()));
  }
};

std::string fmt_fixed(double v) {  // std::to_string(double)
  char b[64];
  std::snprintf(b, sizeof b, "%f", v);
  return b;
}

void need(bool ok, const char* msg) {
  if (!ok) throw ModelError(msg);
}

}  // namespace

// ================================================================== gpu_model.hpp
// FrequencyGrid (gpu_model.cpp:9-40): the grid is the index set the kernels scan.
void FrequencyGrid::validate() const {
  need(f_min_mhz > 0.0 && f_max_mhz > f_min_mhz, "grid: need 0 < f_min < f_max");
  need(step_mhz > 0.0, "grid: step must be > 0");
  const double span = (f_max_mhz - f_min_mhz) / step_mhz;
  need(std::abs(span - std::round(span)) <= 1e-9, "grid: span must be an integer number of steps");
  need(on_grid(f_ref_mhz), "grid: f_ref must lie on the grid");
}

bool FrequencyGrid::on_grid(double f) const {
  if (f < f_min_mhz - 1e-9 || f > f_max_mhz + 1e-9) return false;
  const double k = (f - f_min_mhz) / step_mhz;
  return std::abs(k - std::round(k)) < 1e-9;
}

std::size_t FrequencyGrid::size() const {
  return static_cast<std::size_t>(std::round((f_max_mhz - f_min_mhz) / step_mhz)) + 1;
}

double FrequencyGrid::at(std::size_t i) const { return f_min_mhz + step_mhz * static_cast<double>(i); }

std::vector<double> FrequencyGrid::frequencies() const {
  std::vector<double> v;
  v.reserve(size());
  for (std::size_t i = 0, n = size(); i < n; ++i) v.push_back(at(i));
  return v;
}

double FrequencyGrid::clamp_to_grid(double f) const {
  const double x = std::clamp(f, f_min_mhz, f_max_mhz);
  return f_min_mhz + std::round((x - f_min_mhz) / step_mhz) * step_mhz;
}

// Model validators: the same rules libgsb applies in gsb_profile_validate (gpu_model.cpp:42-78).
void LatencyModel::validate() const {
  need(a >= 0.0, "latency model: a must be >= 0");
  need(f_ref_mhz > 0.0, "latency model: f_ref must be > 0");
  for (double L : {1.0, 256.0, 1024.0, 8192.0, 65536.0})
    if (!(prefill_latency_raw_ms(*this, L, f_ref_mhz) > 0.0))
      throw ModelError("latency model: nonpositive latency at L=" + fmt_fixed(L));
  if (a > 0.0 && b < 0.0) {
    const double v = -b / (2.0 * a);
    if (v >= 1.0 && v <= 65536.0 && a * v * v + b * v + c <= 0.0)
      throw ModelError("latency model: nonpositive latency at vertex");
  }
}

void DecodeStepModel::validate() const {
  need(alpha0_ms >= 0 && alpha1_ms >= 0 && beta0_ms >= 0 && beta1_ms >= 0,
       "decode model: coefficients must be >= 0");
  need(f_ref_mhz > 0.0, "decode model: f_ref must be > 0");
  need(alpha0_ms + alpha1_ms + beta0_ms + beta1_ms > 0.0, "decode model: step time must be positive");
}

void PowerModel::validate(const FrequencyGrid& grid) const {
  need(p_idle_w > 0.0, "power model: p_idle must be > 0");
  double last = -1.0;
  for (double f : grid.frequencies()) {
    const double p = active_power_w(f);
    if (p <= p_idle_w) throw ModelError("power model: active power must exceed p_idle at f=" + fmt_fixed(f));
    need(p > last, "power model: active power must be strictly increasing on the grid");
    last = p;
  }
}

void GpuProfile::validate() const {
  const gsb_profile c = to_c(*this);
  char msg[256];
  const int rc = gsb_profile_validate(&c, msg, sizeof msg);
  if (rc != GSB_OK) raise(rc, msg);
}

double prefill_latency_raw_ms(const LatencyModel& m, double L, double f) {
  return ((m.a * L + m.b) * L + m.c) * m.f_ref_mhz / f;
}

double decode_step_raw_ms(const DecodeStepModel& m, double B, double f) {
  return (m.alpha0_ms + m.alpha1_ms * B) + (m.beta0_ms + m.beta1_ms * B) * m.f_ref_mhz / f;
}

namespace {
void require_on_grid(const FrequencyGrid& g, double f) {
  if (!g.on_grid(f)) throw ModelError("frequency " + fmt_fixed(f) + " MHz is not on the grid");
}
}  // namespace

double GpuProfile::prefill_latency_ms(double L, double f) const {
  require_on_grid(grid, f);
  return prefill_latency_raw_ms(prefill, L, f);
}

double GpuProfile::decode_step_ms(double B, double f) const {
  require_on_grid(grid, f);
  need(B >= 1.0, "decode step: batch must be >= 1");
  return decode_step_raw_ms(decode, B, f);
}

double GpuProfile::active_power_w(double f) const {
  require_on_grid(grid, f);
  return power.active_power_w(f);
}

// The calibrated synthetic device (gpu_model.cpp:121-130, profiles/default.json).
GpuProfile GpuProfile::default_profile() {
  GpuProfile p;
  p.name = "synth-a100-40g";
  p.grid = FrequencyGrid{210.0, 1410.0, 15.0, 1410.0};
  p.prefill = LatencyModel{2.0e-5, 0.12, 8.0, 1410.0};
  p.decode = DecodeStepModel{14.5, 0.1, 9.0, 0.135, 1410.0};
  p.power = PowerModel{1.6e-7, -1.0e-4, 0.05, 216.5, 15.0};
  p.validate();
  return p;
}

// ================================================================== router.hpp
// RoutingConfig::validate (router.cpp:7-24) through gsb_routing_validate; worker_map's length
// is the host-side part of the rule.
void RoutingConfig::validate(int n_prefill_workers) const {
  if (thresholds.size() > GSB_MAX_CLASSES - 1) {
    // the ordering / positivity messages take precedence, as in the reference
    for (std::size_t i = 0; i + 1 < thresholds.size(); ++i)
      if (thresholds[i] >= thresholds[i + 1]) throw RouterError("routing: thresholds must be ascending and distinct");
    throw RouterError("routing: more than 7 thresholds (GSB_MAX_CLASSES)");
  }
  gsb_route_cfg c;
  std::memset(&c, 0, sizeof c);
  c.n_thresholds = static_cast<int32_t>(thresholds.size());
  for (std::size_t i = 0; i < thresholds.size(); ++i) c.thresholds[i] = thresholds[i];
  char msg[256];
  c.enabled = 0;
  int rc = gsb_routing_validate(&c, n_prefill_workers, nullptr, msg, sizeof msg);
  if (rc != GSB_OK) raise(rc, msg);
  if (!enabled) return;
  if (static_cast<int>(worker_map.size()) != n_prefill_workers)
    throw RouterError("routing: worker_map must name a class per prefill worker");
  c.enabled = 1;
  const std::vector<int32_t> wm(worker_map.begin(), worker_map.end());
  rc = gsb_routing_validate(&c, n_prefill_workers, wm.data(), msg, sizeof msg);
  if (rc != GSB_OK) raise(rc, msg);
}

std::vector<int> classify_batch(const RoutingConfig& cfg, std::span<const int> prompts) {
  if (cfg.thresholds.size() > GSB_MAX_CLASSES - 1)
    throw RouterError("routing: more than 7 thresholds (GSB_MAX_CLASSES)");
  std::vector<int> out(prompts.size());
  if (prompts.empty()) return out;
  const std::vector<int32_t> thr(cfg.thresholds.begin(), cfg.thresholds.end());
  const std::vector<int32_t> L(prompts.begin(), prompts.end());
  Call call;
  const size_t o_in = call.in_vec(L);
  const size_t o_out = call.out(L.size() * sizeof(int32_t));
  call.commit();
  check(call.ctx(), gsb_classify(call.ctx(), static_cast<int>(thr.size()), thr.data(),
                                 static_cast<int64_t>(L.size()), call.dev<int32_t>(o_in),
                                 call.dev<int32_t>(o_out), nullptr));
  call.fetch();
  const int32_t* cls = call.host<int32_t>(o_out);
  std::copy(cls, cls + L.size(), out.begin());
  return out;
}

int classify(const RoutingConfig& cfg, int prompt_tokens) {
  const int one[1] = {prompt_tokens};
  return classify_batch(cfg, one)[0];
}

// Dispatcher (router.cpp:33-50): per-class FIFO of request ids; double dispatch is an error.
Dispatcher::Dispatcher(const RoutingConfig& cfg)
    : config_(cfg), lanes_(cfg.enabled ? static_cast<std::size_t>(cfg.n_classes()) : 1) {}

int Dispatcher::dispatch(const Request& r) {
  if (dispatched_.count(r.id)) throw RouterError("request " + std::to_string(r.id) + " dispatched twice");
  const int lane = config_.enabled ? classify(config_, r.prompt_tokens) : 0;
  dispatched_.insert(r.id);
  lanes_[static_cast<std::size_t>(lane)].push_back(r.id);
  return lane;
}

std::int64_t Dispatcher::pop(int queue) {
  auto& lane = lanes_[static_cast<std::size_t>(queue)];
  const std::int64_t id = lane.front();
  lane.pop_front();
  return id;
}

// ================================================================== prefill_opt.hpp
double PrefillBatch::t_ref_total_ms(const LatencyModel& m) const {
  Jobs J;
  J.add(*this, false);
  if (J.prompt.empty()) return 0.0;
  const double abc[3] = {m.a, m.b, m.c};
  Call call;
  const size_t o_off = call.in_vec(J.off), o_L = call.in_vec(J.prompt), o_wf = call.in_vec(J.wf);
  const size_t o_out = call.out(sizeof(double));
  call.commit();
  check(call.ctx(), gsb_t_ref_batches(call.ctx(), abc, 1, call.dev<int64_t>(o_off),
                                      call.dev<int32_t>(o_L), call.dev<double>(o_wf),
                                      call.dev<double>(o_out), nullptr));
  call.fetch();
  return *call.host<double>(o_out);
}

namespace {
// busy_time_ms + energy_total (prefill_opt.cpp:16-31) of one batch at one clock (K2 pointwise).
EnergyBreakdown energy_point(const PrefillBatch& batch, double f, double window_ms,
                             const GpuProfile& profile, double* busy_out) {
  Jobs J;
  J.add(batch, false);
  Call call;
  call.install(to_c(profile));
  const size_t o_off = call.in_vec(J.off), o_L = call.in_vec(J.prompt), o_wf = call.in_vec(J.wf);
  const size_t o_f = call.in(&f, sizeof f), o_w = call.in(&window_ms, sizeof window_ms);
  const size_t o_busy = call.out(8), o_a = call.out(8), o_i = call.out(8), o_t = call.out(8),
               o_fe = call.out(1);
  call.commit();
  check(call.ctx(), gsb_energy_batches(call.ctx(), 0, 1, call.dev<int64_t>(o_off), call.dev<int32_t>(o_L),
                                       call.dev<double>(o_wf), call.dev<double>(o_f),
                                       call.dev<double>(o_w), call.dev<double>(o_busy),
                                       call.dev<double>(o_a), call.dev<double>(o_i),
                                       call.dev<double>(o_t), call.dev<uint8_t>(o_fe), nullptr));
  call.fetch();
  const uint8_t fe = *call.host<uint8_t>(o_fe);
  if (fe == 2) {  // the reference's ModelError cases, in its check order (prefill_opt.cpp:17-18)
    if (batch.jobs.empty()) throw ModelError("busy_time: empty batch");
    throw ModelError("busy_time: frequency off grid");
  }
  EnergyBreakdown e;
  e.feasible = fe == 1;
  e.active_j = *call.host<double>(o_a);
  e.idle_j = *call.host<double>(o_i);
  e.total_j = *call.host<double>(o_t);
  if (busy_out) *busy_out = *call.host<double>(o_busy);
  return e;
}
}  // namespace

double busy_time_ms(const PrefillBatch& batch, double f, const GpuProfile& profile) {
  double busy = 0.0;
  energy_point(batch, f, 0.0, profile, &busy);
  return busy;
}

EnergyBreakdown energy_total(const PrefillBatch& batch, double f, double window_ms,
                             const GpuProfile& profile) {
  return energy_point(batch, f, window_ms, profile, nullptr);
}

double energy_total_closed_form_j(const PrefillBatch& batch, double f, double window_ms,
                                  const GpuProfile& profile) {
  if (!profile.grid.on_grid(f)) throw ModelError("energy closed form: frequency off grid");
  Jobs J;
  J.add(batch, false);
  Call call;
  call.install(to_c(profile));
  const size_t o_off = call.in_vec(J.off), o_L = call.in_vec(J.prompt), o_wf = call.in_vec(J.wf);
  const size_t o_f = call.in(&f, sizeof f), o_w = call.in(&window_ms, sizeof window_ms);
  const size_t o_out = call.out(8);
  call.commit();
  check(call.ctx(), gsb_energy_closed_form_batches(call.ctx(), 0, 1, call.dev<int64_t>(o_off),
                                                   call.dev<int32_t>(o_L), call.dev<double>(o_wf),
                                                   call.dev<double>(o_f), call.dev<double>(o_w),
                                                   call.dev<double>(o_out), nullptr));
  call.fetch();
  return *call.host<double>(o_out);
}

std::vector<std::optional<FrequencyChoice>> select_frequency_batch(
    std::span<const PrefillBatch> batches, std::span<const double> windows_ms,
    const GpuProfile& profile) {
  if (batches.size() != windows_ms.size())
    throw std::invalid_argument("select_frequency_batch: one window per batch");
  std::vector<std::optional<FrequencyChoice>> out(batches.size());
  if (batches.empty()) return out;
  Jobs J;
  for (const PrefillBatch& b : batches) J.add(b, false);
  const std::vector<double> W(windows_ms.begin(), windows_ms.end());
  const int64_t n = static_cast<int64_t>(batches.size());
  Call call;
  call.install(to_c(profile));
  const size_t o_off = call.in_vec(J.off), o_L = call.in_vec(J.prompt), o_wf = call.in_vec(J.wf);
  const size_t o_w = call.in_vec(W);
  const size_t o_idx = call.out(sizeof(int16_t) * n), o_e = call.out(sizeof(double) * n);
  call.commit();
  gsb_select_cfg sc;
  std::memset(&sc, 0, sizeof sc);
  sc.mode = GSB_PER_CELL_WINDOW;
  sc.n_classes = 1;
  check(call.ctx(), gsb_select_batches(call.ctx(), &sc, 0, n, call.dev<int64_t>(o_off),
                                       call.dev<int32_t>(o_L), call.dev<double>(o_wf), nullptr,
                                       nullptr, call.dev<double>(o_w), call.dev<int16_t>(o_idx),
                                       call.dev<double>(o_e), nullptr, nullptr));
  call.fetch();
  const int16_t* idx = call.host<int16_t>(o_idx);
  const double* en = call.host<double>(o_e);
  for (int64_t b = 0; b < n; ++b) {
    // an empty batch reaches busy_time_ms in the reference's scan (prefill_opt.cpp:50)
    if (idx[b] == -2) throw ModelError("busy_time: empty batch");
    if (idx[b] >= 0) out[b] = FrequencyChoice{profile.grid.at(static_cast<std::size_t>(idx[b])), en[b]};
  }
  return out;
}

std::optional<FrequencyChoice> select_frequency(const PrefillBatch& batch, double window_ms,
                                                const GpuProfile& profile) {
  return select_frequency_batch(std::span<const PrefillBatch>(&batch, 1),
                                std::span<const double>(&window_ms, 1), profile)[0];
}

// queue_optimizer_tick (prefill_opt.cpp:58-82): one K2 launch in deadline-slack mode over the
// non-empty snapshots; empty queues produce no command.
std::vector<PrefillFreqCommand> queue_optimizer_tick(const std::vector<ClassQueueSnapshot>& queues,
                                                     double now_ms, const QueueOptimizerConfig& cfg,
                                                     const GpuProfile& profile) {
  std::vector<const ClassQueueSnapshot*> live;
  for (const ClassQueueSnapshot& q : queues)
    if (!q.batch.jobs.empty()) live.push_back(&q);
  std::vector<PrefillFreqCommand> out;
  if (live.empty()) return out;
  Jobs J;
  for (const ClassQueueSnapshot* q : live) J.add(q->batch, true);
  const int64_t n = static_cast<int64_t>(live.size());
  const std::vector<double> now(static_cast<std::size_t>(n), now_ms);
  Call call;
  call.install(to_c(profile));
  const size_t o_off = call.in_vec(J.off), o_L = call.in_vec(J.prompt), o_wf = call.in_vec(J.wf);
  const size_t o_dl = call.in_vec(J.deadline), o_now = call.in_vec(now);
  const size_t o_w = call.out(sizeof(double) * n), o_idx = call.out(sizeof(int16_t) * n),
               o_e = call.out(sizeof(double) * n);
  call.commit();
  gsb_select_cfg sc;
  std::memset(&sc, 0, sizeof sc);
  sc.mode = GSB_DEADLINE_SLACK;
  sc.n_classes = 1;
  sc.qopt = gsb_qopt_cfg{cfg.resolve_period_ms, cfg.margin_prefill, cfg.min_budget_ms,
                         cfg.first_token_allowance_ms};
  check(call.ctx(), gsb_select_batches(call.ctx(), &sc, 0, n, call.dev<int64_t>(o_off),
                                       call.dev<int32_t>(o_L), call.dev<double>(o_wf),
                                       call.dev<double>(o_dl), call.dev<double>(o_now),
                                       call.dev<double>(o_w), call.dev<int16_t>(o_idx),
                                       call.dev<double>(o_e), nullptr, nullptr));
  call.fetch();
  const double* W = call.host<double>(o_w);
  const int16_t* idx = call.host<int16_t>(o_idx);
  for (int64_t b = 0; b < n; ++b) {
    PrefillFreqCommand c;
    c.class_id = live[static_cast<std::size_t>(b)]->class_id;
    c.window_ms = W[b];
    c.infeasible = idx[b] < 0;
    c.f_mhz = c.infeasible ? profile.grid.f_max_mhz : profile.grid.at(static_cast<std::size_t>(idx[b]));
    out.push_back(c);
  }
  return out;
}

// ================================================================== metrics.hpp
// Nearest-rank quantile (metrics.cpp:11-19) through gsb_quantile_batch (any set size: sets up
// to 4096 samples are sorted in shared memory, larger ones take an exact radix select).
double quantile(std::span<const double> samples, double q) {
  if (samples.empty()) throw std::invalid_argument("quantile: empty sample set");
  if (q < 0.0 || q > 1.0) throw std::invalid_argument("quantile: q outside [0, 1]");
  const int64_t off[2] = {0, static_cast<int64_t>(samples.size())};
  Call call;
  const size_t o_off = call.in(off, sizeof off);
  const size_t o_s = call.in(samples.data(), samples.size() * sizeof(double));
  const size_t o_out = call.out(sizeof(double));
  call.commit();
  check(call.ctx(), gsb_quantile_batch(call.ctx(), q, 1, call.dev<int64_t>(o_off), call.dev<double>(o_s),
                                       call.dev<double>(o_out), nullptr));
  call.fetch();
  return *call.host<double>(o_out);
}

// ================================================================== decode_ctl.hpp
void DecodeCtlConfig::validate() const {
  const gsb_ctl_cfg c = to_c(*this);
  char msg[256];
  const int rc = gsb_ctl_cfg_validate(&c, msg, sizeof msg);
  if (rc != GSB_OK) raise(rc, msg);
}

DecodeSteadyState decode_steady_state(const GpuProfile& profile, double tps, double f, int max_batch) {
  const gsb_profile p = to_c(profile);
  const int32_t mb = max_batch;
  Call call;
  const size_t o_p = call.in(&p, sizeof p), o_tps = call.in(&tps, 8), o_f = call.in(&f, 8),
               o_mb = call.in(&mb, 4);
  const size_t o_s = call.out(1), o_b = call.out(8), o_t = call.out(8);
  call.commit();
  check(call.ctx(), gsb_steady_state_batch(call.ctx(), 1, call.dev<gsb_profile>(o_p), call.dev<double>(o_tps),
                                           call.dev<double>(o_f), call.dev<int32_t>(o_mb),
                                           call.dev<uint8_t>(o_s), call.dev<double>(o_b),
                                           call.dev<double>(o_t), nullptr));
  call.fetch();
  DecodeSteadyState s;
  s.sustainable = *call.host<uint8_t>(o_s) != 0;
  s.batch = *call.host<double>(o_b);
  s.tbt_ms = *call.host<double>(o_t);
  return s;
}

// FreqBandTable accessors (decode_ctl.cpp:52-74)
int FreqBandTable::bucket_index(double tps) const {
  const auto it = std::find_if(buckets.begin(), buckets.end(),
                               [tps](const BandBucket& b) { return tps <= b.tps_hi; });
  return it == buckets.end() ? static_cast<int>(buckets.size()) - 1
                             : static_cast<int>(it - buckets.begin());
}

std::pair<double, double> FreqBandTable::band(int bucket, const FrequencyGrid& grid, double step) const {
  const double f = buckets[static_cast<std::size_t>(bucket)].f_opt_mhz;
  return {std::max(grid.f_min_mhz, f - step), std::min(grid.f_max_mhz, f + step)};
}

void FreqBandTable::validate() const {
  need(!buckets.empty(), "band table: empty");
  std::vector<double> lo, hi;
  for (const BandBucket& b : buckets) {
    lo.push_back(b.tps_lo);
    hi.push_back(b.tps_hi);
  }
  if (buckets.size() > GSB_MAX_BUCKETS) {
    need(lo[0] == 0.0, "band table: must start at 0 TPS");
    throw ModelError("band table: more than 32 buckets (GSB_MAX_BUCKETS)");
  }
  const gsb_ctl_cfg none{};
  char msg[256];
  const int rc = gsb_replay_validate(&none, 0, static_cast<int32_t>(buckets.size()), lo.data(),
                                     hi.data(), 1, msg, sizeof msg);
  if (rc != GSB_OK) raise(rc, msg);
}

// build_band_table (decode_ctl.cpp:76-111): argument rules here, the (level x clock) scan in K4.
FreqBandTable build_band_table(const GpuProfile& profile, std::span<const double> levels,
                               double t_slo_ms, int decode_workers, int max_batch) {
  need(!levels.empty(), "band table: need at least one TPS level");
  for (std::size_t i = 0; i + 1 < levels.size(); ++i)
    need(levels[i] < levels[i + 1], "band table: levels must be ascending");
  need(decode_workers >= 1 && max_batch >= 1, "band table: bad pool shape");
  const int nl = static_cast<int>(levels.size());
  const gsb_profile p = to_c(profile);
  const int32_t zero = 0, workers = decode_workers, mb = max_batch;
  const std::vector<double> lv(levels.begin(), levels.end());
  Call call;
  const size_t o_p = call.in(&p, sizeof p), o_po = call.in(&zero, 4), o_slo = call.in(&t_slo_ms, 8),
               o_w = call.in(&workers, 4), o_mb = call.in(&mb, 4), o_lv = call.in_vec(lv);
  const size_t o_lo = call.out(8 * nl), o_hi = call.out(8 * nl), o_f = call.out(8 * nl),
               o_fe = call.out(nl);
  call.commit();
  check(call.ctx(), gsb_build_band_tables(call.ctx(), 1, call.dev<gsb_profile>(o_p), call.dev<int32_t>(o_po),
                                          call.dev<double>(o_slo), call.dev<int32_t>(o_w),
                                          call.dev<int32_t>(o_mb), nl, call.dev<double>(o_lv),
                                          call.dev<double>(o_lo), call.dev<double>(o_hi),
                                          call.dev<double>(o_f), call.dev<uint8_t>(o_fe), nullptr));
  call.fetch();
  FreqBandTable t;
  for (int i = 0; i < nl; ++i)
    t.buckets.push_back(BandBucket{call.host<double>(o_lo)[i], call.host<double>(o_hi)[i],
                                   call.host<double>(o_f)[i], call.host<uint8_t>(o_fe)[i] != 0});
  t.validate();
  return t;
}

// TpsWindow::tps (decode_ctl.cpp:113-118): aging out is deque bookkeeping; the rate over the
// remaining events is gsb_tps_window_batch.
double TpsWindow::tps(double now_ms) {
  while (!events_.empty() && events_.front().first < now_ms - span_ms_) events_.pop_front();
  std::vector<double> t;
  std::vector<int32_t> tok;
  for (const auto& [ti, n] : events_) {
    t.push_back(ti);
    tok.push_back(n);
  }
  const int64_t off[2] = {0, static_cast<int64_t>(t.size())};
  Call call;
  const size_t o_off = call.in(off, sizeof off), o_t = call.in_vec(t), o_k = call.in_vec(tok),
               o_w = call.in(&span_ms_, 8), o_now = call.in(&now_ms, 8);
  const size_t o_out = call.out(8);
  call.commit();
  check(call.ctx(), gsb_tps_window_batch(call.ctx(), 1, call.dev<int64_t>(o_off), call.dev<double>(o_t),
                                         call.dev<int32_t>(o_k), call.dev<double>(o_w),
                                         call.dev<double>(o_now), call.dev<double>(o_out), nullptr));
  call.fetch();
  return *call.host<double>(o_out);
}

// TbtWindow (decode_ctl.cpp:120-128): ring bookkeeping here, P95 in gsb_quantile_batch.
void TbtWindow::record(double interval_ms) {
  ring_.push_back(interval_ms);
  while (static_cast<int>(ring_.size()) > cap_) ring_.pop_front();
}

double TbtWindow::p95() const {
  const std::vector<double> v(ring_.begin(), ring_.end());
  return quantile(v, 0.95);
}

// ------------------------------------------------------------------ DecodeController
namespace {
const char* const kActionNames[8] = {"hold", "up", "down", "coarse_hold", "coarse_pending",
                                     "coarse_commit", "adapt_up", "adapt_down"};
}

DecodeController::DecodeController(const DecodeCtlConfig& cfg, FreqBandTable table,
                                   const FrequencyGrid& grid, int worker_id)
    : cfg_(cfg), table_(std::move(table)), grid_(grid), worker_(worker_id) {
  cfg_.validate();
  table_.validate();
  gsb_ctl_state st;
  std::memset(&st, 0, sizeof st);  // initialized = 0: the kernel runs the constructor
  state_.assign(reinterpret_cast<unsigned char*>(&st), reinterpret_cast<unsigned char*>(&st) + sizeof st);
  step(-1, 0.0, 0.0, false);
}

// One transition (or, for kind < 0, only the constructor) on the GPU: K3s resumed from state_.
void DecodeController::step(int kind, double now_ms, double value, bool has) {
  const int NB = static_cast<int>(table_.buckets.size());
  std::vector<double> tps_hi, f_opt;
  for (const BandBucket& b : table_.buckets) {
    tps_hi.push_back(b.tps_hi);
    f_opt.push_back(b.f_opt_mhz);
  }
  const gsb_ctl_cfg c = to_c(cfg_);
  const int32_t zero = 0, worker = worker_;
  const int n_ev = kind < 0 ? 0 : 1;
  const int64_t ev_off[2] = {0, n_ev};
  const int8_t k8 = static_cast<int8_t>(kind < 0 ? 0 : kind);
  const uint8_t h8 = has ? 1 : 0;
  Call call;
  const size_t o_cfg = call.in(&c, sizeof c), o_tb = call.in(&zero, 4), o_wk = call.in(&worker, 4),
               o_hi = call.in_vec(tps_hi), o_f = call.in_vec(f_opt), o_ev = call.in(ev_off, sizeof ev_off),
               o_k = call.in(&k8, 1), o_t = call.in(&now_ms, 8), o_v = call.in(&value, 8),
               o_h = call.in(&h8, 1);
  const size_t o_st = call.inout(state_.data(), state_.size());
  const size_t o_dg = call.out(8), o_nr = call.out(8), o_rec = call.out(sizeof(gsb_decision) * 1);
  call.commit();
  gsb_replay_args a;
  std::memset(&a, 0, sizeof a);
  a.n_traj = 1;
  a.d_cfg = call.dev<gsb_ctl_cfg>(o_cfg);
  a.d_table_of = call.dev<int32_t>(o_tb);
  a.d_worker = call.dev<int32_t>(o_wk);
  a.n_buckets = NB;
  a.d_tps_hi = call.dev<double>(o_hi);
  a.d_f_opt = call.dev<double>(o_f);
  a.f_min_mhz = grid_.f_min_mhz;
  a.f_max_mhz = grid_.f_max_mhz;
  a.d_digest = call.dev<uint64_t>(o_dg);
  a.d_n_rec = call.dev<int64_t>(o_nr);
  a.d_records = call.dev<gsb_decision>(o_rec);
  a.rec_cap = 1;
  check(call.ctx(), gsb_decode_script(call.ctx(), &a, call.dev<int64_t>(o_ev), call.dev<int8_t>(o_k),
                                      call.dev<double>(o_t), call.dev<double>(o_v),
                                      call.dev<uint8_t>(o_h), call.dev<gsb_ctl_state>(o_st), nullptr));
  call.fetch();
  std::memcpy(state_.data(), call.host<unsigned char>(o_st), state_.size());
  const auto* st = reinterpret_cast<const gsb_ctl_state*>(state_.data());
  command_ = st->set_point;
  bucket_ = st->current_bucket;
  for (int b = 0; b < NB; ++b) table_.buckets[static_cast<std::size_t>(b)].f_opt_mhz = st->f_opt[b];
  if (*call.host<int64_t>(o_nr) > 0) {
    const gsb_decision& r = *call.host<gsb_decision>(o_rec);
    log_.push_back(DecisionRecord{r.tick_ms, r.worker, r.tps, r.p95_tbt_ms, r.bucket, r.band_lo,
                                  r.band_hi, r.command_mhz, kActionNames[r.action & 7]});
  }
}

double DecodeController::on_fine_tick(double now_ms, std::optional<double> p95) {
  step(0, now_ms, p95.value_or(0.0), p95.has_value());
  return command_;
}

void DecodeController::on_coarse_tick(double now_ms, double worker_tps) { step(1, now_ms, worker_tps, true); }

void DecodeController::on_adapt_tick(double now_ms) { step(2, now_ms, 0.0, false); }

// ------------------------------------------------------------------ log rendering and audit
// decision_log_csv (decode_ctl.cpp:231-247): '%.6g' numbers, fixed header.
std::string decision_log_csv(std::span<const DecisionRecord> records) {
  auto g6 = [](double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.6g", v);
    return std::string(b);
  };
  std::string s = "tick_ms,worker,tps,p95_tbt_ms,bucket,band_lo,band_hi,command_mhz,action\n";
  for (const DecisionRecord& r : records) {
    s += g6(r.tick_ms) + ',' + std::to_string(r.worker) + ',' + g6(r.tps) + ',' + g6(r.p95_tbt_ms) +
         ',' + std::to_string(r.bucket) + ',' + g6(r.band_lo) + ',' + g6(r.band_hi) + ',' +
         g6(r.command_mhz) + ',' + r.action + '\n';
  }
  return s;
}

// audit_decision_log (decode_ctl.cpp:249-313): per worker (ascending id), in log order —
// containment of every command in its band, the fine-tick rate limit inside an unchanged band,
// a full hysteresis streak behind every commit, adaptation moving the band by one step at most.
namespace {
struct WorkerAudit {
  explicit WorkerAudit(const DecodeCtlConfig& c) : cfg(c) {}
  const DecodeCtlConfig& cfg;
  const DecisionRecord* last_fine = nullptr;
  int streak = 0;
  int streak_bucket = -1;
  std::vector<std::string> found;

  void observe(const DecisionRecord& r) {
    const std::string& a = r.action;
    const bool fine = a == "up" || a == "down" || a == "hold";
    const bool coarse = a.compare(0, 7, "coarse_") == 0;
    const bool adapt = a.compare(0, 6, "adapt_") == 0;
    if (!fine && !coarse && !adapt) {
      found.push_back("unknown action " + a);
      return;
    }
    if (r.command_mhz < r.band_lo - 1e-9 || r.command_mhz > r.band_hi + 1e-9)
      found.push_back("command outside band");
    if (coarse) {
      if (a == "coarse_pending") {
        streak = r.bucket == streak_bucket ? streak + 1 : 1;
        streak_bucket = r.bucket;
      } else {
        if (a != "coarse_hold") {  // commit closes the streak it ends
          const int len = r.bucket == streak_bucket ? streak + 1 : 1;
          if (len < cfg.hysteresis_count) found.push_back("band commit without full hysteresis streak");
        }
        streak = 0;
        streak_bucket = -1;
      }
    }
    if (fine) {
      if (last_fine && last_fine->band_lo == r.band_lo && last_fine->band_hi == r.band_hi &&
          std::abs(r.command_mhz - last_fine->command_mhz) > cfg.max_step_mhz + 1e-9)
        found.push_back("fine-tick step exceeds rate limit");
      last_fine = &r;
    }
    if (adapt && last_fine && std::abs(r.band_lo - last_fine->band_lo) > cfg.step_mhz + 1e-9)
      found.push_back("adaptation moved band by more than one step");
  }
};
}  // namespace

AuditResult audit_decision_log(std::span<const DecisionRecord> records, const DecodeCtlConfig& cfg) {
  std::map<int, WorkerAudit> per;  // ordered by worker id
  std::map<int, std::vector<double>> ticks;
  for (const DecisionRecord& r : records) {
    auto it = per.try_emplace(r.worker, cfg).first;
    const std::size_t before = it->second.found.size();
    it->second.observe(r);
    for (std::size_t k = before; k < it->second.found.size(); ++k) ticks[r.worker].push_back(r.tick_ms);
  }
  AuditResult res;
  for (auto& [w, au] : per) {
    const std::vector<double>& t = ticks[w];
    for (std::size_t k = 0; k < au.found.size(); ++k) {
      ++res.violations;
      if (res.messages.size() < 32)
        res.messages.push_back("worker " + std::to_string(w) + " t=" + std::to_string(t[k]) + ": " +
                               au.found[k]);
    }
  }
  return res;
}

// ------------------------------------------------------------------ trace CSV (K6)
const char* prompt_class_name(PromptClass c) {  // trace.cpp:14-16
  return c == PromptClass::ShortMedium ? "SM" : "L";
}

// load_trace (trace.cpp:56-129): the file's bytes go to the device in one copy; K6 parses them
// (rows, checks, SLO classes) and the SoA comes back in one copy.
Trace load_trace(const std::filesystem::path& path, int class_threshold) {
  std::ifstream in(path, std::ios::binary);
  if (!in)
    throw TraceError(TraceError::Kind::MalformedRow, "cannot open trace file: " + path.string());
  const std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  size_t cap = bytes.size() / 6 + 1;  // a valid row holds >= 6 bytes; retried if malformed
  for (int attempt = 0;; ++attempt) {
    Call call;
    const size_t ob = call.in(bytes.data(), bytes.size());
    const size_t oa = call.out(cap * 8), op = call.out(cap * 4), oo = call.out(cap * 4),
                 oc = call.out(cap);
    call.commit();
    gsb_trace_parse_result res;
    const int rc = gsb_trace_parse(call.ctx(), call.dev<char>(ob), static_cast<int64_t>(bytes.size()),
                                   class_threshold, static_cast<int64_t>(cap), call.dev<int64_t>(oa),
                                   call.dev<int32_t>(op), call.dev<int32_t>(oo),
                                   call.dev<uint8_t>(oc), &res, nullptr);
    if (rc == GSB_TRACE_ERROR)
      throw TraceError(static_cast<TraceError::Kind>(res.kind), gsb_last_error(call.ctx()));
    if (rc == GSB_INVALID_ARGUMENT && res.n_rows > static_cast<int64_t>(cap) && attempt == 0) {
      cap = static_cast<size_t>(res.n_rows);
      continue;
    }
    check(call.ctx(), rc);
    call.fetch();
    Trace t;
    const size_t n = static_cast<size_t>(res.n_rows);
    t.requests.resize(n);
    const int64_t* a = call.host<int64_t>(oa);
    const int32_t* p = call.host<int32_t>(op);
    const int32_t* o = call.host<int32_t>(oo);
    const uint8_t* c = call.host<uint8_t>(oc);
    for (size_t i = 0; i < n; ++i) {
      Request& r = t.requests[i];
      r.id = static_cast<int64_t>(i);
      r.arrival_ms = a[i];
      r.prompt_tokens = p[i];
      r.output_tokens = o[i];
      r.cls = static_cast<PromptClass>(c[i]);
    }
    // finalize_meta (trace.cpp:36-45) with duration 0: the largest arrival
    t.meta.name = path.stem().string();
    t.meta.duration_ms = std::max<int64_t>(0, res.max_arrival_ms);
    t.meta.nominal_qps = t.meta.duration_ms > 0 ? 1000.0 * static_cast<double>(n) /
                                                      static_cast<double>(t.meta.duration_ms)
                                                : 0.0;
    return t;
  }
}

// save_trace_csv (trace.cpp:131-145): the SoA goes up in one copy, K6 renders the text, one
// copy brings it back.
void save_trace_csv(const Trace& trace, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write trace file: " + path.string());
  const size_t n = trace.requests.size();
  const bool has_class = std::all_of(trace.requests.begin(), trace.requests.end(),
                                     [](const Request& r) { return r.cls.has_value(); });
  std::vector<int64_t> a(n);
  std::vector<int32_t> p(n), o(n);
  std::vector<uint8_t> c(n);
  for (size_t i = 0; i < n; ++i) {
    const Request& r = trace.requests[i];
    a[i] = r.arrival_ms;
    p[i] = r.prompt_tokens;
    o[i] = r.output_tokens;
    c[i] = r.cls ? static_cast<uint8_t>(*r.cls) : 0;
  }
  // upper bound of the text: 20 + 11 + 11 digits/signs, 3 commas, "SM", '\n' per row
  const size_t cap = 64 + n * 48;
  Call call;
  const size_t oa = call.in_vec(a), op = call.in_vec(p), oo = call.in_vec(o), oc = call.in_vec(c);
  const size_t ot = call.out(cap);
  call.commit();
  int64_t bytes = 0;
  check(call.ctx(), gsb_trace_format(call.ctx(), static_cast<int64_t>(n), call.dev<int64_t>(oa),
                                     call.dev<int32_t>(op), call.dev<int32_t>(oo),
                                     has_class ? call.dev<uint8_t>(oc) : nullptr, call.dev<char>(ot),
                                     static_cast<int64_t>(cap), &bytes, nullptr));
  call.fetch();
  out.write(call.host<char>(ot), bytes);
}

}  // namespace greensim
