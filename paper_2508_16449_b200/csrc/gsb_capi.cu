// gsb_capi.cu — context management, host-side validation (the reference's typed-exception
// rules mapped to status codes) and profile table construction for libgsb.so.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gsb_common.cuh"

namespace {

void put_msg(char* msg, size_t cap, const std::string& s) {
  if (msg && cap) {
    std::snprintf(msg, cap, "%s", s.c_str());
  }
}

std::string fmt_f(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%f", v);  // std::to_string(double) formatting
  return b;
}

// FrequencyGrid::on_grid (gpu_model.cpp:18-22)
bool on_grid(const gsb_profile& p, double f) {
  if (f < p.f_min_mhz - 1e-9 || f > p.f_max_mhz + 1e-9) return false;
  const double k = (f - p.f_min_mhz) / p.step_mhz;
  return std::fabs(k - std::round(k)) < 1e-9;
}

size_t grid_size(const gsb_profile& p) {  // gpu_model.cpp:24-26
  return static_cast<size_t>(std::round((p.f_max_mhz - p.f_min_mhz) / p.step_mhz)) + 1;
}

double grid_at(const gsb_profile& p, size_t i) {  // gpu_model.cpp:28
  return p.f_min_mhz + p.step_mhz * static_cast<double>(i);
}

double power_at(const gsb_profile& p, double f) {  // gpu_model.hpp:64
  return ((p.k3 * f + p.k2) * f + p.k1) * f + p.k0;
}

// GpuProfile::validate (gpu_model.cpp:80-87) with the per-model validators (:9-78).
std::string validate_profile(const gsb_profile& p) {
  if (p.f_min_mhz <= 0.0 || p.f_max_mhz <= p.f_min_mhz) return "grid: need 0 < f_min < f_max";
  if (p.step_mhz <= 0.0) return "grid: step must be > 0";
  const double steps = (p.f_max_mhz - p.f_min_mhz) / p.step_mhz;
  if (std::fabs(steps - std::round(steps)) > 1e-9)
    return "grid: span must be an integer number of steps";
  if (!on_grid(p, p.f_ref_mhz)) return "grid: f_ref must lie on the grid";
  if (p.lat_a < 0.0) return "latency model: a must be >= 0";
  if (p.lat_f_ref_mhz <= 0.0) return "latency model: f_ref must be > 0";
  for (double L : {1.0, 256.0, 1024.0, 8192.0, 65536.0}) {
    const double t = ((p.lat_a * L + p.lat_b) * L + p.lat_c) * p.lat_f_ref_mhz / p.lat_f_ref_mhz;
    if (t <= 0.0) return "latency model: nonpositive latency at L=" + fmt_f(L);
  }
  if (p.lat_a > 0.0 && p.lat_b < 0.0) {
    const double vertex = -p.lat_b / (2.0 * p.lat_a);
    if (vertex >= 1.0 && vertex <= 65536.0 &&
        p.lat_a * vertex * vertex + p.lat_b * vertex + p.lat_c <= 0.0)
      return "latency model: nonpositive latency at vertex";
  }
  if (p.dec_alpha0_ms < 0 || p.dec_alpha1_ms < 0 || p.dec_beta0_ms < 0 || p.dec_beta1_ms < 0)
    return "decode model: coefficients must be >= 0";
  if (p.dec_f_ref_mhz <= 0.0) return "decode model: f_ref must be > 0";
  if (p.dec_alpha0_ms + p.dec_alpha1_ms + p.dec_beta0_ms + p.dec_beta1_ms <= 0.0)
    return "decode model: step time must be positive";
  if (p.p_idle_w <= 0.0) return "power model: p_idle must be > 0";
  double prev = -1.0;
  for (size_t i = 0; i < grid_size(p); ++i) {
    const double f = grid_at(p, i);
    const double pw = power_at(p, f);
    if (pw <= p.p_idle_w) return "power model: active power must exceed p_idle at f=" + fmt_f(f);
    if (pw <= prev) return "power model: active power must be strictly increasing on the grid";
    prev = pw;
  }
  if (p.lat_f_ref_mhz != p.f_ref_mhz || p.dec_f_ref_mhz != p.f_ref_mhz)
    return "profile: latency/decode f_ref must match grid f_ref";
  if (grid_size(p) > GSB_MAX_GRID) return "profile: grid larger than GSB_MAX_GRID";
  return "";
}

// What the clock tables need to be well formed when GpuProfile::validate is skipped.
std::string structural_check(const gsb_profile& p) {
  const double v[] = {p.f_min_mhz, p.f_max_mhz, p.step_mhz, p.f_ref_mhz, p.lat_a, p.lat_b, p.lat_c,
                      p.k3, p.k2, p.k1, p.k0, p.p_idle_w};
  for (double x : v)
    if (!std::isfinite(x)) return "profile: non-finite coefficient";
  if (p.f_min_mhz <= 0.0 || p.f_max_mhz < p.f_min_mhz || p.step_mhz <= 0.0)
    return "grid: need 0 < f_min <= f_max and step > 0";
  if ((p.f_max_mhz - p.f_min_mhz) / p.step_mhz > GSB_MAX_GRID - 1)
    return "profile: grid larger than GSB_MAX_GRID";
  return "";
}

}  // namespace

int gsb_set_error(gsb_ctx* ctx, int status, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return status;
}

int gsb_check_launch(gsb_ctx* ctx, const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return gsb_set_error(ctx, GSB_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
  return GSB_OK;
}

cudaStream_t gsb_pick_stream(gsb_ctx* ctx, void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
}

// Grow-only scratch. An outgrown buffer is retired, not freed: a CUDA graph captured with it
// (or work still in flight on any stream) keeps a valid address; retired buffers are freed
// in gsb_ctx_destroy. Growth is geometric, so the retired total stays below the live size.
void* gsb_scratch(gsb_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->scratch_bytes) return ctx->d_scratch;
  const size_t want = std::max(bytes, ctx->scratch_bytes * 2);
  void* p = nullptr;
  if (cudaMalloc(&p, want) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (ctx->d_scratch) ctx->retired_scratch.push_back(ctx->d_scratch);
  ctx->d_scratch = p;
  ctx->scratch_bytes = want;
  return ctx->d_scratch;
}

void* gsb_sync_words(gsb_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->sync_bytes) return ctx->d_sync;
  const size_t want = std::max(bytes, ctx->sync_bytes * 2);
  void* p = nullptr;
  if (cudaMalloc(&p, want) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  // zeroed before any kernel of the context's stream can use it; the old words (epochs,
  // statuses) are not carried over: a fresh zero state is a valid state
  if (cudaMemsetAsync(p, 0, want, ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    cudaFree(p);
    return nullptr;
  }
  if (ctx->d_sync) ctx->retired_scratch.push_back(ctx->d_sync);
  ctx->d_sync = p;
  ctx->sync_bytes = want;
  return ctx->d_sync;
}

extern "C" {

const char* gsb_version(void) { return "gsb 0.1 (sm_100a, abi 1)"; }

const char* gsb_status_string(int s) {
  switch (s) {
    case GSB_OK: return "ok";
    case GSB_MODEL_ERROR: return "ModelError";
    case GSB_ROUTER_ERROR: return "RouterError";
    case GSB_TRACE_ERROR: return "TraceError";
    case GSB_CUDA_ERROR: return "CudaError";
    case GSB_INVALID_ARGUMENT: return "InvalidArgument";
  }
  return "unknown";
}

int gsb_ctx_create(int device, gsb_ctx** out) {
  if (!out) return GSB_INVALID_ARGUMENT;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) {
    cudaGetLastError();
    return GSB_CUDA_ERROR;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return GSB_CUDA_ERROR;
  if (prop.major != 10) {
    // The kernels are built for sm_100a only; refuse anything else instead of
    // silently failing at the first launch.
    return GSB_CUDA_ERROR;
  }
  auto* c = new gsb_ctx;
  c->device = device;
  c->n_sms = prop.multiProcessorCount;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&c->d_tabs, sizeof(gsb::ProfTab) * GSB_MAX_PROFILES) != cudaSuccess ||
      cudaMallocHost(reinterpret_cast<void**>(&c->h_stage), sizeof(gsb::ProfTab) * GSB_MAX_PROFILES) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->stage_free, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return GSB_CUDA_ERROR;
  }
  *out = c;
  return GSB_OK;
}

void gsb_ctx_destroy(gsb_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaFree(c->d_tabs);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->stage_free) cudaEventDestroy(c->stage_free);
  cudaFree(c->d_scratch);
  cudaFree(c->d_sync);
  for (void* p : c->retired_scratch) cudaFree(p);
  cudaFree(c->d_ticks);
  if (c->up_stream) cudaStreamSynchronize(c->up_stream);
  if (c->down_stream) cudaStreamSynchronize(c->down_stream);
  if (c->search_stream) cudaStreamSynchronize(c->search_stream);
  if (c->compute2) cudaStreamSynchronize(c->compute2);
  cudaFree(c->d_hostpass);
  for (cudaEvent_t e : c->hp_events) cudaEventDestroy(e);
  if (c->up_stream) cudaStreamDestroy(c->up_stream);
  if (c->down_stream) cudaStreamDestroy(c->down_stream);
  if (c->search_stream) cudaStreamDestroy(c->search_stream);
  if (c->compute2) cudaStreamDestroy(c->compute2);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* gsb_last_error(const gsb_ctx* c) { return c ? c->err.c_str() : ""; }

void* gsb_ctx_stream(gsb_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int gsb_synchronize(gsb_ctx* c) {
  const cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return gsb_set_error(c, GSB_CUDA_ERROR, cudaGetErrorString(e));
  return GSB_OK;
}

int gsb_malloc(gsb_ctx* c, size_t bytes, void** d_out) {
  if (!c || !d_out) return GSB_INVALID_ARGUMENT;
  *d_out = nullptr;
  if (bytes == 0) return GSB_OK;
  cudaSetDevice(c->device);
  const cudaError_t e = cudaMalloc(d_out, bytes);
  if (e != cudaSuccess) return gsb_set_error(c, GSB_CUDA_ERROR, std::string("malloc: ") + cudaGetErrorString(e));
  return GSB_OK;
}

int gsb_free(gsb_ctx* c, void* d_ptr) {
  if (!c) return GSB_INVALID_ARGUMENT;
  if (!d_ptr) return GSB_OK;
  cudaSetDevice(c->device);
  const cudaError_t e = cudaFree(d_ptr);
  if (e != cudaSuccess) return gsb_set_error(c, GSB_CUDA_ERROR, std::string("free: ") + cudaGetErrorString(e));
  return GSB_OK;
}

int gsb_host_alloc(gsb_ctx* c, size_t bytes, void** h_out) {
  if (!c || !h_out) return GSB_INVALID_ARGUMENT;
  *h_out = nullptr;
  if (bytes == 0) return GSB_OK;
  cudaSetDevice(c->device);
  const cudaError_t e = cudaMallocHost(h_out, bytes);
  if (e != cudaSuccess) return gsb_set_error(c, GSB_CUDA_ERROR, std::string("host_alloc: ") + cudaGetErrorString(e));
  return GSB_OK;
}

int gsb_host_free(gsb_ctx* c, void* h_ptr) {
  if (!c) return GSB_INVALID_ARGUMENT;
  if (h_ptr && cudaFreeHost(h_ptr) != cudaSuccess) return gsb_set_error(c, GSB_CUDA_ERROR, "host_free failed");
  return GSB_OK;
}

int gsb_memcpy(gsb_ctx* c, void* dst, const void* src, size_t bytes, int kind, void* stream) {
  if (!c || kind < 0 || kind > 2) return GSB_INVALID_ARGUMENT;
  if (bytes == 0) return GSB_OK;
  static const cudaMemcpyKind kinds[3] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost,
                                          cudaMemcpyDeviceToDevice};
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kinds[kind], gsb_pick_stream(c, stream));
  if (e != cudaSuccess) return gsb_set_error(c, GSB_CUDA_ERROR, std::string("memcpy: ") + cudaGetErrorString(e));
  return GSB_OK;
}

int gsb_profile_validate(const gsb_profile* p, char* msg, size_t cap) {
  if (!p) return GSB_INVALID_ARGUMENT;
  const std::string m = validate_profile(*p);
  put_msg(msg, cap, m);
  return m.empty() ? GSB_OK : GSB_MODEL_ERROR;
}

// DecodeCtlConfig::validate (decode_ctl.cpp:12-26)
int gsb_ctl_cfg_validate(const gsb_ctl_cfg* c, char* msg, size_t cap) {
  if (!c) return GSB_INVALID_ARGUMENT;
  std::string m;
  if (c->tslo_ms <= 0) m = "decode ctl: tslo must be > 0";
  else if (c->margin_decode < 0.2 || c->margin_decode > 2.0) m = "decode ctl: margin outside [0.2, 2.0]";
  else if (c->fine_period_ms <= 0 || c->coarse_period_ms <= 0 || c->adapt_period_s <= 0)
    m = "decode ctl: periods must be > 0";
  else if (c->step_mhz <= 0 || c->max_step_mhz < c->step_mhz) m = "decode ctl: need max_step >= step > 0";
  else if (c->hysteresis_count < 1) m = "decode ctl: hysteresis_count must be >= 1";
  else if (c->bias_threshold <= 0 || c->bias_threshold >= 1) m = "decode ctl: bias_threshold must be in (0,1)";
  else if (c->tbt_window_tokens < 1) m = "decode ctl: tbt window must hold >= 1 sample";
  else if (c->tps_scale <= 0) m = "decode ctl: tps_scale must be > 0";
  else if (c->lower_margin >= c->upper_margin) m = "decode ctl: need lower < upper margin";
  put_msg(msg, cap, m);
  return m.empty() ? GSB_OK : GSB_MODEL_ERROR;
}

// RoutingConfig::validate (router.cpp:7-24)
int gsb_routing_validate(const gsb_route_cfg* cfg, int n_prefill_workers,
                         const int32_t* worker_map, char* msg, size_t cap) {
  std::string m;
  const int nt = cfg->n_thresholds;
  // thresholds[] holds GSB_MAX_CLASSES - 1 entries: read no further, reject longer lists after
  // the order / positivity checks (the reference's check order, router.cpp:8-13)
  const int nt_seen = std::min(nt, GSB_MAX_CLASSES - 1);
  if (nt < 1) m = "routing: need at least one threshold";
  for (int i = 0; m.empty() && i + 1 < nt_seen; ++i)
    if (cfg->thresholds[i] >= cfg->thresholds[i + 1])
      m = "routing: thresholds must be ascending and distinct";
  for (int i = 0; m.empty() && i < nt_seen; ++i)
    if (cfg->thresholds[i] < 1) m = "routing: thresholds must be >= 1";
  if (m.empty() && nt > GSB_MAX_CLASSES - 1) m = "routing: more than 7 thresholds";
  if (m.empty() && cfg->enabled) {
    const int C = nt + 1;
    if (!worker_map && n_prefill_workers > 0) m = "routing: worker_map must name a class per prefill worker";
    std::vector<bool> covered(static_cast<size_t>(C), false);
    for (int w = 0; m.empty() && w < n_prefill_workers; ++w) {
      const int c = worker_map[w];
      if (c < 0 || c >= C) m = "routing: worker_map class out of range";
      else covered[static_cast<size_t>(c)] = true;
    }
    if (m.empty() && n_prefill_workers >= 0) {
      for (bool b : covered)
        if (!b) m = "routing: every class needs at least one worker";
    }
  }
  put_msg(msg, cap, m);
  return m.empty() ? GSB_OK : GSB_ROUTER_ERROR;
}

int gsb_set_profiles(gsb_ctx* ctx, int n, const gsb_profile* profiles) {
  return gsb_set_profiles_ex(ctx, n, profiles, 0);
}

int gsb_set_profiles_ex(gsb_ctx* ctx, int n, const gsb_profile* profiles, int flags) {
  if (!ctx || n < 1 || n > GSB_MAX_PROFILES || !profiles)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "set_profiles: need 1..4 profiles");
  for (int p = 0; p < n; ++p) {  // all-or-nothing: check every profile before touching state
    const std::string m = (flags & GSB_PROFILES_UNCHECKED) ? structural_check(profiles[p])
                                                           : validate_profile(profiles[p]);
    if (!m.empty()) return gsb_set_error(ctx, GSB_MODEL_ERROR, m);
  }
  cudaSetDevice(ctx->device);
  // the pinned staging area is reused: wait until the previous upload has read it
  if (cudaEventSynchronize(ctx->stage_free) != cudaSuccess)
    return gsb_set_error(ctx, GSB_CUDA_ERROR, "set_profiles: staging wait failed");
  // d_tabs is read by kernels launched on ANY stream (k_select_batches, k_energy_batches, ...):
  // without GSB_PROFILES_ASYNC (whose contract is "every launch on the context's stream", where
  // stream order already serialises the upload behind them) the new tables may only land once
  // every kernel already issued on the device has finished reading the old ones
  if (!(flags & GSB_PROFILES_ASYNC) && cudaDeviceSynchronize() != cudaSuccess)
    return gsb_set_error(ctx, GSB_CUDA_ERROR, "set_profiles: device sync failed");
  for (int p = 0; p < n; ++p) {
    const gsb_profile& pr = profiles[p];
    gsb::ProfTab& t = ctx->h_stage[p];
    std::memset(&t, 0, sizeof t);
    t.G = static_cast<int32_t>(grid_size(pr));
    t.f_min = pr.f_min_mhz;
    t.f_max = pr.f_max_mhz;
    t.step = pr.step_mhz;
    t.f_ref = pr.f_ref_mhz;
    t.lat_a = pr.lat_a;
    t.lat_b = pr.lat_b;
    t.lat_c = pr.lat_c;
    t.p_idle = pr.p_idle_w;
    t.k3 = pr.k3;
    t.k2 = pr.k2;
    t.k1 = pr.k1;
    t.k0 = pr.k0;
    t.all_fast = 1;
    t.P_min = INFINITY;
    t.P_max = -INFINITY;
    for (int i = 0; i < t.G; ++i) {
      const double f = grid_at(pr, static_cast<size_t>(i));
      t.f[i] = f;
      t.P[i] = power_at(pr, f);
      t.rcp_f[i] = gsb::short_divisor(f) ? 1.0 / f : 0.0;
      t.all_fast &= t.rcp_f[i] != 0.0 ? 1 : 0;
      t.P_min = std::min(t.P_min, t.P[i]);
      t.P_max = std::max(t.P_max, t.P[i]);
    }
    ctx->profiles[p] = pr;
    ctx->h_tabs[p] = t;
  }
  ctx->n_profiles = n;
  const cudaError_t e = cudaMemcpyAsync(ctx->d_tabs, ctx->h_stage, sizeof(gsb::ProfTab) * n,
                                        cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) return gsb_set_error(ctx, GSB_CUDA_ERROR, cudaGetErrorString(e));
  cudaEventRecord(ctx->stage_free, ctx->stream);
  // GSB_PROFILES_ASYNC: the upload is ordered on the context's own stream only (callers that
  // launch with stream == NULL); otherwise wait so launches on any stream see the tables
  if (!(flags & GSB_PROFILES_ASYNC) && cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    return gsb_set_error(ctx, GSB_CUDA_ERROR, "set_profiles: sync failed");
  return GSB_OK;
}

// ---------------------------------------------------------------- multi-GPU reductions
int gsb_combine_summaries(int world, int n, const gsb_class_summary* per_rank,
                          const int64_t* cell_off, gsb_class_summary* out) {
  if (world < 1 || n < 0 || (n && (!per_rank || !out || !cell_off))) return GSB_INVALID_ARGUMENT;
  for (int i = 0; i < n; ++i) {
    gsb_class_summary o{};
    o.min_energy_j = INFINITY;
    o.argmin_cell = -1;
    double e = 0.0;
    for (int r = 0; r < world; ++r) {
      const gsb_class_summary& x = per_rank[static_cast<size_t>(r) * n + i];
      o.n_cmd += x.n_cmd;
      o.n_infeasible += x.n_infeasible;
      o.n_empty += x.n_empty;
      e = e + x.sum_energy_j;
      if (x.argmin_cell >= 0) {
        const int64_t g = x.argmin_cell + cell_off[r];
        if (o.argmin_cell < 0 || x.min_energy_j < o.min_energy_j ||
            (x.min_energy_j == o.min_energy_j && g < o.argmin_cell)) {
          o.min_energy_j = x.min_energy_j;
          o.argmin_cell = g;
        }
      }
    }
    o.sum_energy_j = e;
    out[i] = o;
  }
  return GSB_OK;
}

namespace {
int gather_to_host(gsb_ctx* ctx, int world, const void* d_send, size_t bytes,
                   gsb_allgather_fn gather, void* user, void* h_out, void* stream) {
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  char* d = static_cast<char*>(gsb_scratch(ctx, bytes * (static_cast<size_t>(world) + 1)));
  if (!d) return gsb_set_error(ctx, GSB_CUDA_ERROR, "reduce: scratch allocation failed");
  char* d_send_copy = d + bytes * static_cast<size_t>(world);
  cudaMemcpyAsync(d_send_copy, d_send, bytes, cudaMemcpyDefault, s);
  if (gather(d_send_copy, d, bytes, s, user) != 0)
    return gsb_set_error(ctx, GSB_CUDA_ERROR, "reduce: the all-gather callback failed");
  cudaMemcpyAsync(h_out, d, bytes * static_cast<size_t>(world), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return gsb_check_launch(ctx, "reduce");
  return GSB_OK;
}
inline uint64_t mix64(uint64_t x) {  // splitmix64 finaliser (distributed.py _mix64)
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
}  // namespace

int gsb_reduce_summaries(gsb_ctx* ctx, int world, int rank, int n, const gsb_class_summary* d_local,
                         const int64_t* cell_off, gsb_allgather_fn gather, void* user,
                         gsb_class_summary* h_out, void* stream) {
  if (!ctx || !gather || world < 1 || rank < 0 || rank >= world || n < 0)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "reduce_summaries: bad arguments");
  std::vector<gsb_class_summary> all(static_cast<size_t>(world) * n);
  const int rc = gather_to_host(ctx, world, d_local, sizeof(gsb_class_summary) * n, gather, user,
                                all.data(), stream);
  if (rc) return rc;
  return gsb_combine_summaries(world, n, all.data(), cell_off, h_out);
}

int gsb_tally_pool(int64_t n, const gsb_pool_summary* sm, int64_t scen0, gsb_decode_tally* out) {
  if (n < 0 || !out || (n && !sm)) return GSB_INVALID_ARGUMENT;
  gsb_decode_tally t{};
  t.n_scenarios = n;
  t.min_decode_pool_j = INFINITY;
  t.argmin_scenario = -1;
  double e = 0.0;
  uint64_t dig = 0;
  for (int64_t i = 0; i < n; ++i) {
    const gsb_pool_summary& s = sm[i];
    const double x = s.decode_pool_j;
    e = e + x;
    if (x < t.min_decode_pool_j) {
      t.min_decode_pool_j = x;
      t.argmin_scenario = scen0 + i;
    }
    const uint64_t d = s.decision_digest ^ s.freq_digest ^ s.request_digest;
    dig += mix64(d ^ static_cast<uint64_t>(scen0 + i));
    t.n_completed += s.n_completed;
    t.n_rejected += s.n_rejected;
    t.n_ttft_ok += s.n_ttft_ok;
    t.n_tbt_ok += s.n_tbt_ok;
    t.tbt_samples += s.tbt_samples;
    t.tbt_samples_ok += s.tbt_samples_ok;
    t.n_decisions += s.n_decisions;
    t.n_freq_changes += s.n_freq_changes;
  }
  t.decode_pool_j = e;
  t.digest = dig;
  *out = t;
  return GSB_OK;
}

int gsb_combine_tallies(int world, const gsb_decode_tally* pr, gsb_decode_tally* out) {
  if (world < 1 || !pr || !out) return GSB_INVALID_ARGUMENT;
  gsb_decode_tally t{};
  t.min_decode_pool_j = INFINITY;
  t.argmin_scenario = -1;
  double e = 0.0;
  for (int r = 0; r < world; ++r) {
    const gsb_decode_tally& s = pr[r];
    t.n_scenarios += s.n_scenarios;
    e = e + s.decode_pool_j;
    if (s.argmin_scenario >= 0 &&
        (t.argmin_scenario < 0 || s.min_decode_pool_j < t.min_decode_pool_j)) {
      t.min_decode_pool_j = s.min_decode_pool_j;
      t.argmin_scenario = s.argmin_scenario;
    }
    t.digest += s.digest;
    t.n_completed += s.n_completed;
    t.n_rejected += s.n_rejected;
    t.n_ttft_ok += s.n_ttft_ok;
    t.n_tbt_ok += s.n_tbt_ok;
    t.tbt_samples += s.tbt_samples;
    t.tbt_samples_ok += s.tbt_samples_ok;
    t.n_decisions += s.n_decisions;
    t.n_freq_changes += s.n_freq_changes;
  }
  t.decode_pool_j = e;
  *out = t;
  return GSB_OK;
}

int gsb_reduce_tallies(gsb_ctx* ctx, int world, int rank, const gsb_decode_tally* h_local,
                       gsb_allgather_fn gather, void* user, gsb_decode_tally* h_out,
                       void* stream) {
  if (!ctx || !gather || !h_local || world < 1 || rank < 0 || rank >= world)
    return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "reduce_tallies: bad arguments");
  std::vector<gsb_decode_tally> all(static_cast<size_t>(world));
  const int rc = gather_to_host(ctx, world, h_local, sizeof(gsb_decode_tally), gather, user,
                                all.data(), stream);
  if (rc) return rc;
  return gsb_combine_tallies(world, all.data(), h_out);
}

int64_t gsb_n_ticks(double period_ms, double t_end_ms) {
  int64_t n = 0;
  for (double t = period_ms; t <= t_end_ms; t = t + period_ms) ++n;
  return n;
}

// FreqBandTable::validate (decode_ctl.cpp:64-74) for every table + DecodeCtlConfig::validate.
int gsb_replay_validate(const gsb_ctl_cfg* cfgs, int64_t n, int32_t nb, const double* tps_lo,
                        const double* tps_hi, int64_t n_tables, char* msg, size_t cap) {
  if (nb < 1 || nb > GSB_MAX_BUCKETS) {
    put_msg(msg, cap, "band table: empty or more than GSB_MAX_BUCKETS buckets");
    return GSB_MODEL_ERROR;
  }
  for (int64_t t = 0; t < n_tables; ++t) {
    const double* lo = tps_lo + t * nb;
    const double* hi = tps_hi + t * nb;
    std::string m;
    if (lo[0] != 0.0) m = "band table: must start at 0 TPS";
    for (int i = 0; m.empty() && i + 1 < nb; ++i) {
      if (hi[i] != lo[i + 1]) m = "band table: buckets must tile contiguously";
      else if (lo[i] >= hi[i]) m = "band table: empty bucket";
    }
    if (m.empty() && hi[nb - 1] != INFINITY) m = "band table: last bucket must extend to +inf";
    if (!m.empty()) {
      put_msg(msg, cap, m);
      return GSB_MODEL_ERROR;
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    const int rc = gsb_ctl_cfg_validate(&cfgs[i], msg, cap);
    if (rc != GSB_OK) return rc;
    if (cfgs[i].tbt_window_tokens > GSB_MAX_TBT_WINDOW) {
      put_msg(msg, cap, "decode ctl: tbt window larger than GSB_MAX_TBT_WINDOW");
      return GSB_MODEL_ERROR;
    }
  }
  put_msg(msg, cap, "");
  return GSB_OK;
}

}  // extern "C"
