// gsb_pool.cu — K5: the closed-loop decode pool.
//
// Replays the decode side of the reference simulator (simkernel.cpp:330-464: batching,
// step times, least-loaded enqueue, actuation delay, ledgers, TBT/TPS windows and the
// DecodeController ticks) for thousands of controller parameter sets at once, all driven by
// one decode-enqueue stream (the prefill pool never waits on the decode pool, so the stream
// is independent of decode parameters; the oracle records it, oracle/gs_sim.c).
//
// One WARP per scenario, sequential in simulated time. Every iteration selects the next event
// exactly as the reference's priority queue would (time, then kind: step end 2 < enqueue 3 <
// freq applied 4 < coarse 5 < adapt 6 < fine 7, simkernel.cpp:21-31,44-50) with three warp
// min-reductions, then runs it:
//   * a step end costs O(1 + admissions + completions), not O(batch): every stream active in
//     a step emits exactly once and every gap it records is that step's length, so a
//     stream's whole future is fixed when it joins (it completes at worker step
//     join + output_tokens - 1), and its TBT statistics are differences of per-worker prefix
//     sums over steps (count of gaps <= SLO, sum of gap bit patterns). The warp scans the
//     batch's completion indices with one compare per slot and compacts only on completion;
//   * ticks run one controller per lane (lane w = decode worker w);
//   * for the same reason the 256-sample TBT ring is a short deque of (value, count) runs, and
//     its nearest-rank P95 is found by warp-wide descending max extraction over the runs
//     (usually one round: the longest gap's run already covers the top 5%), exact without
//     sorting.
// Events that the reference orders only by insertion sequence (two workers' step ends, or
// freq applications, at the same instant) touch disjoint worker state and commute.
// Per-worker state lives in shared memory; the FIFO of waiting requests in a global
// workspace slot owned by the warp (persistent grid, scenarios claimed by atomic counter).
#include <cmath>
#include <cstdlib>

#include "gsb_common.cuh"
#include "gsb_ctl.cuh"

using gsb::std_clamp;
using gsb::std_max;
using gsb::std_min;
using namespace gsbctl;

namespace {

constexpr int kWarpsPerBlock = 4;
constexpr int kFQ = 4;  // pending clock applications per worker (delay / fine period + 1)
constexpr uint64_t kFnv0 = 0xcbf29ce484222325ull;
constexpr unsigned kFull = 0xffffffffu;

enum : int { K_STEP = 2, K_ENQ = 3, K_FREQ = 4, K_COARSE = 5, K_ADAPT = 6, K_FINE = 7, K_NONE = 15 };
enum : int { PH_DECODE = 1, PH_IDLE = 2 };
enum : int { ST_PENDING = 1, ST_TPS = 2, ST_FREQ = 4, ST_TBT = 8 };

struct PoolParams {
  gsb_profile prof;
  gsb_pool_cfg cfg;
  gsb_pool_stream st;
  gsb_pool_args a;
  int W, MB, RC, TC;
  int RC_full;          // TBT run capacity the configuration needs (max tbt_window_tokens)
  int64_t warp_bytes;
  int32_t* ws_pending;  // [n_warps][W][pending_cap]
  unsigned* counter;
  unsigned* rerun_n;         // scenarios whose TBT runs outgrew RC < RC_full ...
  uint32_t* rerun_list;      // ... replayed again by a second launch with RC = RC_full
  const uint32_t* list_in;   // second launch: the scenarios to replay (count *list_n)
  const unsigned* list_n;
};

// Worker state touched only at step starts and clock applications: shared memory, one row per
// decode worker (lanes >= W share row W), so the event loop's registers stay for the hot state.
struct WorkerCold {
  double ps_last, ps_power;      // PowerState (simkernel.cpp:53-57)
  double act_j, idle_j;          // WorkerLedger sums
  double last_applied;
  uint64_t fdig;                 // applied-clock digest
  int64_t n_freq;
  int ps_phase;
  int pad_;
};

// shared-memory carve-up of one warp's region
struct Smem {
  uint64_t* bp;    // [W][MB] worker's gap-bits prefix sum at the stream's first token
  double* first;   // [W][MB] first-token instant
  double* rv;      // [W][RC] TBT run values
  double* tt;      // [W][TC] TPS event times
  double* fq_t;    // [W][kFQ]
  double* fq_f;    // [W][kFQ]
  int32_t* fin;    // [W][MB] worker step index at which the stream completes
  int32_t* req;    // [W][MB]
  int32_t* bc;     // [W][MB] worker's (gap <= SLO) prefix count at the first token; bit 31: TTFT met
  int32_t* ttok;   // [W][TC]
  uint16_t* rc;    // [W][RC] TBT run counts
  // the controllers (cold: touched on ticks only), out of registers: lanes >= W share row W
  CtlK* k;         // [1]
  Ctl<false>* ctl; // [W + 1]
  double* fo;      // [W + 1][NB] each controller's f_opt table
  WorkerCold* wc;  // [W + 1]
};

__host__ __device__ inline int64_t ctl_bytes(int W, int NB) {
  return ((static_cast<int64_t>(sizeof(CtlK)) + 15) & ~15ll) +
         ((static_cast<int64_t>(sizeof(Ctl<false>)) * (W + 1) + 15) & ~15ll) + 8ll * (W + 1) * NB +
         static_cast<int64_t>(sizeof(WorkerCold)) * (W + 1);
}

__host__ __device__ inline int64_t smem_bytes(int W, int MB, int RC, int TC, int NB) {
  int64_t b = ctl_bytes(W, NB) + 16ll * W * MB + 8ll * W * RC + 8ll * W * TC + 16ll * W * kFQ +
              12ll * W * MB + 4ll * W * TC + 2ll * W * RC;
  return (b + 15) & ~15ll;
}

__device__ __forceinline__ Smem carve(char* base, int W, int MB, int RC, int TC, int NB) {
  Smem s;
  char* p = base;
  s.k = reinterpret_cast<CtlK*>(p); p += (sizeof(CtlK) + 15) & ~size_t{15};
  s.ctl = reinterpret_cast<Ctl<false>*>(p); p += (sizeof(Ctl<false>) * (W + 1) + 15) & ~size_t{15};
  s.fo = reinterpret_cast<double*>(p); p += 8ll * (W + 1) * NB;
  s.wc = reinterpret_cast<WorkerCold*>(p); p += sizeof(WorkerCold) * (W + 1);
  s.bp = reinterpret_cast<uint64_t*>(p); p += 8ll * W * MB;
  s.first = reinterpret_cast<double*>(p); p += 8ll * W * MB;
  s.rv = reinterpret_cast<double*>(p); p += 8ll * W * RC;
  s.tt = reinterpret_cast<double*>(p); p += 8ll * W * TC;
  s.fq_t = reinterpret_cast<double*>(p); p += 8ll * W * kFQ;
  s.fq_f = reinterpret_cast<double*>(p); p += 8ll * W * kFQ;
  s.fin = reinterpret_cast<int32_t*>(p); p += 4ll * W * MB;
  s.req = reinterpret_cast<int32_t*>(p); p += 4ll * W * MB;
  s.bc = reinterpret_cast<int32_t*>(p); p += 4ll * W * MB;
  s.ttok = reinterpret_cast<int32_t*>(p); p += 4ll * W * TC;
  s.rc = reinterpret_cast<uint16_t*>(p);
  return s;
}

__device__ __forceinline__ uint64_t dbits(double x) {
  return static_cast<uint64_t>(__double_as_longlong(x));
}

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(kFull, v, src); }

// Per-lane state of decode worker w = lane (lanes >= W carry inert copies).
struct Worker {
  double freq, target, P;        // applied clock, last command, P(freq)
  double t_end, t_start;         // step end (+inf when idle), step start
  int n_active, n_new;           // batch size; streams admitted at this step's start
  int step_idx;                  // step ends so far
  int c_le;                      // prefix count of steps with gap <= SLO
  uint64_t p_bits;               // prefix sum of gap bit patterns
  int64_t p_head, p_tail;        // FIFO [head, tail) in the workspace ring
  int fq_head, fq_n;             // pending clock applications
  int r_head, r_n, r_total;      // TBT runs ring
  bool p95_valid;
  double p95;
  int t_head, t_n;               // TPS ring
};

// ledger_close / ledger_set (simkernel.cpp:60-79)
__device__ __forceinline__ void ledger_close(WorkerCold& wk, double now) {
  if (now > wk.ps_last) {
    const double joules = wk.ps_power * (now - wk.ps_last) / 1000.0;
    if (wk.ps_phase == PH_DECODE)
      wk.act_j += joules;
    else
      wk.idle_j += joules;
  }
  wk.ps_last = now;
}
__device__ __forceinline__ void ledger_set(WorkerCold& wk, double now, int phase, double power) {
  if (phase == wk.ps_phase && power == wk.ps_power) return;
  ledger_close(wk, now);
  wk.ps_phase = phase;
  wk.ps_power = power;
}

__device__ __forceinline__ double power_at(const gsb_profile& p, double f) {
  return ((p.k3 * f + p.k2) * f + p.k1) * f + p.k0;  // gpu_model.hpp:64
}

// Nearest-rank P95 of worker w's TBT window (metrics.cpp:11-19): sorted[ceil(0.95 n) - 1], i.e.
// the k-th largest with k = n - ceil(0.95 n) + 1. Descending max extraction over the runs
// (gaps are positive doubles, so their bit patterns order like their values): each round takes
// the largest value below the previous one and all runs equal to it; all lanes get the result.
__device__ double window_p95(const Smem& s, int RC, int w, int r_head, int r_n, int total, int lane) {
  const double* rv = s.rv + w * RC;
  const uint16_t* rc = s.rc + w * RC;
  const int k = total - (static_cast<int>(ceil(0.95 * static_cast<double>(total))) - 1);
  uint64_t prev = ~0ull;
  int acc = 0;
  for (;;) {
    uint64_t m = 0;
    for (int i = lane; i < r_n; i += 32) {
      int pos = r_head + i;
      if (pos >= RC) pos -= RC;
      const uint64_t b = dbits(rv[pos]);
      m = (b < prev && b > m) ? b : m;
    }
    const unsigned mh = __reduce_max_sync(kFull, static_cast<unsigned>(m >> 32));
    const unsigned ml = __reduce_max_sync(kFull, static_cast<unsigned>(m >> 32) == mh
                                                     ? static_cast<unsigned>(m) : 0u);
    const uint64_t mx = (static_cast<uint64_t>(mh) << 32) | ml;
    int c = 0;
    for (int i = lane; i < r_n; i += 32) {
      int pos = r_head + i;
      if (pos >= RC) pos -= RC;
      c += dbits(rv[pos]) == mx ? rc[pos] : 0;
    }
    acc += static_cast<int>(__reduce_add_sync(kFull, static_cast<unsigned>(c)));
    if (acc >= k || mx == 0) return __longlong_as_double(static_cast<long long>(mx));
    prev = mx;
  }
}

template <bool REQ_OUT>
__device__ void run_scenario(const PoolParams& P, const Smem& s, int32_t* pend, int64_t n, int lane) {
  const gsb_profile& prof = P.prof;
  const gsb_pool_cfg& cfg = P.cfg;
  const gsb_pool_args& a = P.a;
  const gsb_pool_stream& st = P.st;
  const int W = P.W, MB = P.MB, RC = P.RC, TC = P.TC;
  const int64_t PC = cfg.pending_cap;
  const bool is_w = lane < W;
  const int w = lane;

  const gsb_ctl_cfg ccfg = a.d_cfg[n];
  const double fixed = a.d_fixed_mhz ? a.d_fixed_mhz[n] : 0.0;
  const bool ctl_on = !(fixed > 0.0);
  const int NB = a.n_buckets;
  const int64_t tb = a.d_table_of ? a.d_table_of[n] : 0;
  const int64_t sid = a.d_stream_of ? a.d_stream_of[n] : 0;
  const int64_t e_begin = st.d_off[sid], e_end = st.d_off[sid + 1];
  const int64_t n_stream = e_end - e_begin;
  const double end_floor = st.d_end_floor_ms ? st.d_end_floor_ms[sid] : 0.0;
  const double tbt_thr = cfg.tbt_p95_ms;
  int status = 0;
  if (ccfg.tbt_window_tokens > P.RC_full) status |= ST_TBT;
  bool runs_full = false;  // lane ww: the run ring (RC < RC_full) could not take a new run

  // controller (lane w), DecodeController ctor (decode_ctl.cpp:130-140)
  // controller state in shared memory (ticks only); lanes >= W work on the shared row W
  double* f_opt = s.fo + (is_w ? w : W) * NB;
  if (lane == 0) *s.k = make_k(ccfg, NB, a.d_tps_hi + tb * NB, prof.f_min_mhz, prof.f_max_mhz);
  __syncwarp();
  const CtlK& k = *s.k;
  Ctl<false>& c = s.ctl[is_w ? w : W];
  if (ctl_on) {
    if (is_w || lane == W) {
      for (int b = 0; b < NB; ++b) f_opt[b] = a.d_f_opt[tb * NB + b];
      ctl_init(c, f_opt, k);
    }
  } else if (is_w || lane == W) {
    c.n_rec = 0;
    c.digest = kFnv0;
  }
  __syncwarp();
  gsb_decision* rec = (a.d_records && a.rec_cap > 0 && is_w)
                          ? a.d_records + (n * W + w) * a.rec_cap : nullptr;
  double* fout = (a.d_freq && a.freq_cap > 0 && is_w) ? a.d_freq + (n * W + w) * a.freq_cap * 2
                                                      : nullptr;
  const int tbt_cap = ccfg.tbt_window_tokens;
  const double tps_window = ccfg.coarse_period_ms;

  // Sim::init (simkernel.cpp:195-233): decode clocks start at controllers_[0].command()
  const double f0 = ctl_on ? shfl_d(c.sp, 0) : fixed;
  Worker wk;
  WorkerCold& wc = s.wc[is_w ? w : W];
  wk.freq = wk.target = f0;
  wk.P = power_at(prof, f0);
  wk.t_end = INFINITY;
  wk.t_start = 0.0;
  wk.n_active = wk.n_new = 0;
  wk.step_idx = 0;
  wk.c_le = 0;
  wk.p_bits = 0;
  wk.p_head = wk.p_tail = 0;
  wk.fq_head = wk.fq_n = 0;
  wc.ps_last = 0.0;
  wc.ps_power = prof.p_idle_w;
  wc.ps_phase = PH_IDLE;
  wc.act_j = wc.idle_j = 0.0;
  wk.r_head = wk.r_n = wk.r_total = 0;
  wk.p95_valid = false;
  wk.p95 = 0.0;
  wk.t_head = wk.t_n = 0;
  wc.fdig = kFnv0;
  wc.n_freq = 0;
  wc.last_applied = 0.0;

  // uniform state
  double tf = ccfg.fine_period_ms, tc = ccfg.coarse_period_ms, ta = ccfg.adapt_period_s * 1000.0;
  bool fine_on = ctl_on, coarse_on = ctl_on, adapt_on = ctl_on;
  int64_t e = e_begin;
  double t_enq = e < e_end ? st.d_t_ms[e] : INFINITY;
  int64_t n_done = 0;
  // lane-local accumulators (warp-reduced at the end)
  int64_t n_completed = 0, n_rejected = 0, n_ttft_ok = 0, n_tbt_ok = 0, samples = 0, samples_ok = 0;
  int64_t n_steps = 0;
  uint64_t rdig = 0;
  double max_finish = 0.0;
  double* req_first = REQ_OUT ? a.d_req_first + n * st.n_requests : nullptr;
  double* req_finish = REQ_OUT ? a.d_req_finish + n * st.n_requests : nullptr;
  int32_t* req_worker = REQ_OUT ? a.d_req_worker + n * st.n_requests : nullptr;

  int32_t* S_req = s.req;
  int32_t* S_fin = s.fin;
  int32_t* S_bc = s.bc;
  uint64_t* S_bp = s.bp;
  double* S_first = s.first;

  // start_decode_step (simkernel.cpp:330-345) of worker ww, whole warp
  auto start_step = [&](int ww, double now) {
    const int na = __shfl_sync(kFull, wk.n_active, ww);
    const int64_t ph = __shfl_sync(kFull, wk.p_head, ww);
    const int64_t pt = __shfl_sync(kFull, wk.p_tail, ww);
    const int take = static_cast<int>(min(static_cast<int64_t>(MB - na), pt - ph));
    const int32_t* ring = pend + static_cast<int64_t>(ww) * PC;
    for (int j = lane; j < take; j += 32) {
      const int slot = ww * MB + na + j;
      S_req[slot] = ring[(ph + j) % PC];
      S_fin[slot] = 0x7fffffff;  // known at its first token (the end of this step)
    }
    __syncwarp();
    if (lane == ww) {
      wk.p_head = ph + take;
      wk.n_active = na + take;
      wk.n_new = take;
      if (wk.n_active == 0) {
        ledger_set(wc, now, PH_IDLE, prof.p_idle_w);
      } else {
        const double B = static_cast<double>(wk.n_active);
        // decode_step_raw_ms, gpu_model.cpp:99-103
        const double step = (prof.dec_alpha0_ms + prof.dec_alpha1_ms * B) +
                            (prof.dec_beta0_ms + prof.dec_beta1_ms * B) * prof.dec_f_ref_mhz / wk.freq;
        wk.t_start = now;
        wk.t_end = now + step;
        ledger_set(wc, now, PH_DECODE, wk.P);
      }
    }
  };

  for (;;) {
    // ---- next event: lexicographic min of (t, kind, lane) over the candidates
    double ct = INFINITY;
    int ck = K_NONE;
    if (is_w) {
      const double tq = wk.fq_n ? s.fq_t[w * kFQ + wk.fq_head] : INFINITY;
      if (wk.t_end <= tq) {
        ct = wk.t_end;
        ck = K_STEP;
      } else {
        ct = tq;
        ck = K_FREQ;
      }
      if (ct == INFINITY) ck = K_NONE;
    } else if (lane == W) {
      ct = t_enq;
      ck = ct == INFINITY ? K_NONE : K_ENQ;
    } else if (lane == W + 1) {
      // ticks: coarse (5) < adapt (6) < fine (7) at equal times
      double t = INFINITY;
      int kk = K_NONE;
      if (coarse_on) { t = tc; kk = K_COARSE; }
      if (adapt_on && ta < t) { t = ta; kk = K_ADAPT; }
      if (fine_on && tf < t) { t = tf; kk = K_FINE; }
      ct = t;
      ck = kk;
    }
    const uint64_t tb_ = dbits(ct);  // non-negative doubles order as their bit patterns
    const unsigned hi = __reduce_min_sync(kFull, static_cast<unsigned>(tb_ >> 32));
    const unsigned lo = __reduce_min_sync(kFull, static_cast<unsigned>(tb_ >> 32) == hi
                                                     ? static_cast<unsigned>(tb_) : 0xffffffffu);
    const bool at_min = (static_cast<unsigned>(tb_ >> 32) == hi) && (static_cast<unsigned>(tb_) == lo);
    const unsigned code = __reduce_min_sync(kFull, at_min ? static_cast<unsigned>(ck * 32 + lane) : 0xffffffffu);
    const int kind = static_cast<int>(code >> 5);
    if (kind >= K_NONE) break;
    const int src = static_cast<int>(code & 31);
    const double now = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(hi) << 32) | lo));

    if (kind == K_STEP) {
      // ---- on_decode_step_end (simkernel.cpp:365-393), worker src
      const int ww = src;
      const int na = __shfl_sync(kFull, wk.n_active, ww);
      const int nn = __shfl_sync(kFull, wk.n_new, ww);
      const double gap = now - shfl_d(wk.t_start, ww);
      const bool le = gap <= tbt_thr;
      // per-worker prefix sums over steps, identical on every lane
      const int sidx = __shfl_sync(kFull, wk.step_idx, ww) + 1;
      const int cle = __shfl_sync(kFull, wk.c_le, ww) + (le ? 1 : 0);
      const int g_total = na - nn;  // continuing streams record this step's gap
      const uint64_t pb = (static_cast<uint64_t>(__shfl_sync(kFull, static_cast<long long>(wk.p_bits), ww))) +
                          (g_total > 0 ? dbits(gap) : 0ull);
      // first tokens of the streams admitted at this step's start (the last nn slots)
      for (int j = na - nn + lane; j < na; j += 32) {
        const int slot = ww * MB + j;
        const int32_t r = S_req[slot];
        const int32_t ou = st.d_output_tokens[r];
        // TTFT = first_token - arrival (simkernel.hpp:125) against SloConfig::ttft_for
        const bool ttft_ok = now - st.d_arrival_ms[r] <= st.d_ttft_slo_ms[r];
        S_fin[slot] = sidx + (ou > 1 ? ou - 1 : 0);
        S_bc[slot] = cle | (ttft_ok ? static_cast<int32_t>(0x80000000u) : 0);
        S_bp[slot] = pb;
        S_first[slot] = now;
        if (REQ_OUT) req_first[r] = now;
      }
      __syncwarp();
      // completions: streams whose last token is this step's (emitted >= output_tokens)
      int kept = 0;
      for (int base = 0; base < na; base += 32) {
        const int j = base + lane;
        const bool done = j < na && S_fin[ww * MB + j] == sidx;
        const unsigned dm = __ballot_sync(kFull, done);
        const unsigned live = base + 32 <= na ? kFull : ((1u << (na - base)) - 1u);
        if (dm == 0) {
          if (kept != base) {  // shift this chunk down over earlier completions
            int32_t r = 0, f = 0, c = 0;
            uint64_t p = 0;
            double fs = 0.0;
            if (j < na) {
              const int slot = ww * MB + j;
              r = S_req[slot]; f = S_fin[slot]; c = S_bc[slot]; p = S_bp[slot]; fs = S_first[slot];
            }
            __syncwarp();
            if (j < na) {
              const int dst = ww * MB + kept + lane;
              S_req[dst] = r; S_fin[dst] = f; S_bc[dst] = c; S_bp[dst] = p; S_first[dst] = fs;
            }
            __syncwarp();
          }
          kept += __popc(live);
          continue;
        }
        int32_t r = 0, f = 0, c = 0;
        uint64_t p = 0;
        double fs = 0.0;
        if (j < na) {
          const int slot = ww * MB + j;
          r = S_req[slot]; f = S_fin[slot]; c = S_bc[slot]; p = S_bp[slot]; fs = S_first[slot];
        }
        if (done) {
          // completion: slo_pass_rates terms (metrics.cpp:42-72) and the request digest
          const int32_t ou = st.d_output_tokens[r];
          const int ng = ou > 1 ? ou - 1 : 0;
          const int nle = cle - (c & 0x7fffffff);
          if (c < 0) ++n_ttft_ok;
          const int rank = static_cast<int>(ceil(0.95 * static_cast<double>(ng)));
          if (ng == 0 || nle >= rank) ++n_tbt_ok;
          samples += ng;
          samples_ok += nle;
          uint64_t h = mix(kFnv0, static_cast<uint64_t>(r));
          h = mix(h, dbits(fs));
          h = mix(h, dbits(now));
          h = mix(h, static_cast<uint64_t>(static_cast<uint32_t>(ww)));
          h = mix(h, static_cast<uint64_t>(ng));
          h = mix(h, pb - p);
          rdig += h;
          ++n_completed;
          max_finish = std_max(max_finish, now);
          if (REQ_OUT) req_finish[r] = now;
        }
        const bool keep = j < na && !done;
        const unsigned km = __ballot_sync(kFull, keep);
        __syncwarp();
        if (keep) {
          const int dst = ww * MB + kept + __popc(km & ((1u << lane) - 1u));
          S_req[dst] = r; S_fin[dst] = f; S_bc[dst] = c; S_bp[dst] = p; S_first[dst] = fs;
        }
        kept += __popc(km);
        __syncwarp();
      }
      const int n_fin = na - kept;
      if (lane == ww) {
        wk.n_active = kept;
        wk.n_new = 0;
        wk.t_end = INFINITY;
        wk.step_idx = sidx;
        wk.c_le = cle;
        wk.p_bits = pb;
        ++n_steps;
        // TbtWindow::record x g_total equal gaps (decode_ctl.cpp:120-123) as one run
        if (g_total > 0) {
          int drop = wk.r_total + g_total - tbt_cap;
          if (g_total >= tbt_cap) {
            wk.r_n = 0;
            wk.r_total = 0;
            drop = 0;
          }
          while (drop > 0) {
            const int pos = w * RC + wk.r_head;
            const int cnt = s.rc[pos];
            if (cnt <= drop) {
              drop -= cnt;
              wk.r_total -= cnt;
              if (++wk.r_head == RC) wk.r_head = 0;
              --wk.r_n;
            } else {
              s.rc[pos] = static_cast<uint16_t>(cnt - drop);
              wk.r_total -= drop;
              drop = 0;
            }
          }
          const int g = min(g_total, tbt_cap);
          int last = wk.r_head + wk.r_n - 1;
          if (last >= RC) last -= RC;
          if (wk.r_n > 0 && s.rv[w * RC + last] == gap) {
            // the same gap as the newest run (same batch and clock): one run (the P95 only
            // sees the multiset of gaps)
            s.rc[w * RC + last] = static_cast<uint16_t>(s.rc[w * RC + last] + g);
            wk.r_total += g;
            wk.p95_valid = false;
          } else if (wk.r_n >= RC) {
            runs_full = true;  // only when RC < tbt_cap: the scenario is replayed with RC_full
          } else {
            int pos = wk.r_head + wk.r_n;
            if (pos >= RC) pos -= RC;
            s.rv[w * RC + pos] = gap;
            s.rc[w * RC + pos] = static_cast<uint16_t>(g);
            ++wk.r_n;
            wk.r_total += g;
            wk.p95_valid = false;
          }
        }
        // TpsWindow::record (decode_ctl.hpp:73); unobservable once no coarse tick is left
        if (!coarse_on) {
        } else if (wk.t_n >= TC) {
          status |= ST_TPS;
        } else {
          int pos = wk.t_head + wk.t_n;
          if (pos >= TC) pos -= TC;
          s.tt[w * TC + pos] = now;
          s.ttok[w * TC + pos] = na;
          ++wk.t_n;
        }
      }
      n_done += n_fin;
      if (__shfl_sync(kFull, static_cast<int>(runs_full), ww)) break;
      __syncwarp();
      start_step(ww, now);
    } else if (kind == K_ENQ) {
      // ---- on_decode_enqueue (simkernel.cpp:347-363): least-loaded, lowest index on ties
      const int32_t r = st.d_req[e];
      const unsigned load = is_w ? static_cast<unsigned>(wk.n_active + (wk.p_tail - wk.p_head)) : 0x7ffffffu;
      const unsigned best_code = __reduce_min_sync(kFull, is_w ? (load << 5) | lane : 0xffffffffu);
      const int best = static_cast<int>(best_code & 31);
      const int64_t best_load = best_code >> 5;
      if (best_load >= cfg.max_queue) {
        if (lane == 0) rdig += mix(mix(kFnv0, static_cast<uint64_t>(r)), 0xdeadull);
        n_rejected += lane == 0 ? 1 : 0;
        ++n_done;
      } else {
        bool stepping = false;
        if (lane == best) {
          if (wk.p_tail - wk.p_head >= PC) {
            status |= ST_PENDING;
          } else {
            pend[static_cast<int64_t>(best) * PC + (wk.p_tail % PC)] = r;
            ++wk.p_tail;
          }
          stepping = wk.t_end != INFINITY;
        }
        if (REQ_OUT && lane == 0) req_worker[r] = best;
        stepping = __shfl_sync(kFull, stepping, best);
        __syncwarp();
        if (!stepping) start_step(best, now);
      }
      ++e;
      t_enq = e < e_end ? st.d_t_ms[e] : INFINITY;
    } else if (kind == K_FREQ) {
      // ---- on_freq_applied, decode branch (simkernel.cpp:428-436)
      if (lane == src) {
        const double f = s.fq_f[w * kFQ + wk.fq_head];
        if (++wk.fq_head == kFQ) wk.fq_head = 0;
        --wk.fq_n;
        if (f != wk.freq) {
          wk.freq = f;
          wk.P = power_at(prof, f);
          if (wk.t_end != INFINITY) ledger_set(wc, now, PH_DECODE, wk.P);
          wc.fdig = mix(mix(wc.fdig, dbits(now)), dbits(f));
          if (fout && wc.n_freq < a.freq_cap) {
            fout[2 * wc.n_freq] = now;
            fout[2 * wc.n_freq + 1] = f;
          }
          ++wc.n_freq;
          wc.last_applied = now;
        }
      }
    } else {
      // ---- control ticks (simkernel.cpp:441-464); stop once nothing is outstanding
      const bool live = n_done < n_stream;
      if (kind == K_COARSE) {
        if (!live) {
          coarse_on = false;
        } else {
          if (is_w) {
            // TpsWindow::tps (decode_ctl.cpp:113-118)
            const double lim = now - tps_window;
            while (wk.t_n > 0 && s.tt[w * TC + wk.t_head] < lim) {
              if (++wk.t_head == TC) wk.t_head = 0;
              --wk.t_n;
            }
            int tokens = 0;
            int q = wk.t_head;
            for (int j = 0; j < wk.t_n; ++j) {
              tokens += s.ttok[w * TC + q];
              if (++q == TC) q = 0;
            }
            on_coarse<false, true>(c, f_opt, k, tokens * 1000.0 / tps_window, now, a.rec_cap, rec, w);
          }
          tc = now + ccfg.coarse_period_ms;
        }
      } else if (kind == K_ADAPT) {
        if (!live) {
          adapt_on = false;
        } else {
          if (is_w) on_adapt<false, true>(c, f_opt, k, now, a.rec_cap, rec, w);
          ta = now + ccfg.adapt_period_s * 1000.0;
        }
      } else {
        if (!live) {
          fine_on = false;
        } else {
          // refresh stale P95s, one worker at a time, whole warp
          unsigned stale = __ballot_sync(kFull, is_w && !wk.p95_valid && wk.r_n > 0);
          while (stale) {
            const int ww = __ffs(stale) - 1;
            stale &= stale - 1;
            const int rh = __shfl_sync(kFull, wk.r_head, ww);
            const int rn = __shfl_sync(kFull, wk.r_n, ww);
            const int rt = __shfl_sync(kFull, wk.r_total, ww);
            const double v = window_p95(s, RC, ww, rh, rn, rt, lane);
            if (lane == ww) {
              wk.p95 = v;
              wk.p95_valid = true;
            }
          }
          if (is_w) {
            on_fine<false, true>(c, k, wk.r_n > 0, wk.p95, now, a.rec_cap, rec, w);
            // command_freq (simkernel.cpp:397-404): identical targets are dropped
            const double cmd = c.sp;
            if (cmd != wk.target) {
              wk.target = cmd;
              if (wk.fq_n >= kFQ) {
                status |= ST_FREQ;
              } else {
                int pos = wk.fq_head + wk.fq_n;
                if (pos >= kFQ) pos -= kFQ;
                s.fq_t[w * kFQ + pos] = now + cfg.actuation_delay_ms;
                s.fq_f[w * kFQ + pos] = cmd;
                ++wk.fq_n;
              }
            }
          }
          tf = now + ccfg.fine_period_ms;
        }
      }
    }
    __syncwarp();
  }

  if (__any_sync(kFull, runs_full)) {  // hand the scenario to the full-capacity launch
    if (lane == 0) P.rerun_list[atomicAdd(P.rerun_n, 1u)] = static_cast<uint32_t>(n);
    return;
  }
  // ---- finalize (simkernel.cpp:503-520) and the summary
  double end = std_max(end_floor, max_finish);
  end = std_max(end, is_w ? wc.last_applied : 0.0);
  for (int off = 16; off > 0; off >>= 1) end = std_max(end, __shfl_xor_sync(kFull, end, off));
  if (is_w) ledger_close(wc, end);
  if (a.d_ledger && is_w) {
    a.d_ledger[(n * W + w) * 2] = wc.act_j;
    a.d_ledger[(n * W + w) * 2 + 1] = wc.idle_j;
  }
  auto sum64 = [&](int64_t v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
  };
  auto sumu64 = [&](uint64_t v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
  };
  n_completed = sum64(n_completed);
  n_rejected = sum64(n_rejected);
  n_ttft_ok = sum64(n_ttft_ok);
  n_tbt_ok = sum64(n_tbt_ok);
  samples = sum64(samples);
  samples_ok = sum64(samples_ok);
  rdig = sumu64(rdig);
  const int64_t n_dec = sum64(is_w ? c.n_rec : 0);
  const int64_t n_fc = sum64(is_w ? wc.n_freq : 0);
  n_steps = sum64(is_w ? n_steps : 0);
  status = static_cast<int>(__reduce_or_sync(kFull, static_cast<unsigned>(status)));
  // RunResult::decode_pool_j (simkernel.cpp:617-621), worker order
  double e_sum = 0.0, act = 0.0, idle = 0.0;
  uint64_t dd = kFnv0, fd = kFnv0;
  for (int ww = 0; ww < W; ++ww) {
    const double aj = shfl_d(wc.act_j, ww);
    const double ij = shfl_d(wc.idle_j, ww);
    e_sum += 0.0 + aj + ij;
    act += aj;
    idle += ij;
    dd = mix(dd, __shfl_sync(kFull, c.digest, ww));
    fd = mix(fd, __shfl_sync(kFull, wc.fdig, ww));
  }
  if (lane == 0) {
    gsb_pool_summary o;
    o.decode_pool_j = e_sum;
    o.active_decode_j = act;
    o.idle_j = idle;
    o.sim_end_ms = end;
    o.n_completed = n_completed;
    o.n_rejected = n_rejected;
    o.n_ttft_ok = n_ttft_ok;
    o.n_tbt_ok = n_tbt_ok;
    o.tbt_samples = samples;
    o.tbt_samples_ok = samples_ok;
    o.n_decisions = n_dec;
    o.n_freq_changes = n_fc;
    o.n_steps = n_steps;
    o.decision_digest = dd;
    o.freq_digest = fd;
    o.request_digest = rdig;
    o.status = status;
    o.pad_ = 0;
    a.d_out[n] = o;
  }
}

template <bool REQ_OUT>
#ifndef GSB_POOL_MINB
#define GSB_POOL_MINB 5
#endif
__global__ void __launch_bounds__(kWarpsPerBlock * 32, GSB_POOL_MINB) k_decode_pool(const __grid_constant__ PoolParams P) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const Smem s = carve(smem + wib * P.warp_bytes, P.W, P.MB, P.RC, P.TC, P.a.n_buckets);
  const int64_t slot = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + wib;
  int32_t* pend = P.ws_pending + slot * P.W * P.cfg.pending_cap;
  for (;;) {
    unsigned n = 0;
    if (lane == 0) {
      n = atomicAdd(P.counter, 1u);
      if (P.list_in) n = n < *P.list_n ? P.list_in[n] : 0xffffffffu;
    }
    n = __shfl_sync(kFull, n, 0);
    if (n >= P.a.n_scen) break;
    run_scenario<REQ_OUT>(P, s, pend, static_cast<int64_t>(n), lane);
    __syncwarp();
  }
}

}  // namespace

extern "C" {

int gsb_decode_pool_tps_cap(const gsb_profile* prof, int32_t max_batch, double coarse_period_ms) {
  // the TPS deque holds the step ends of at most two coarse periods (trimmed at each coarse
  // tick, simkernel.cpp:453-458): 2 * period / shortest step + 3
  if (!prof || !(coarse_period_ms > 0.0)) return -1;
  double best = INFINITY;
  for (int b = 1; b <= max_batch; ++b) {
    const double B = b;
    const double s = (prof->dec_alpha0_ms + prof->dec_alpha1_ms * B) +
                     (prof->dec_beta0_ms + prof->dec_beta1_ms * B) * prof->dec_f_ref_mhz / prof->f_max_mhz;
    best = s < best ? s : best;
  }
  if (!(best > 0.0)) return -1;
  const double n = 2.0 * coarse_period_ms / best + 3.0;
  return n > 4096.0 ? -1 : static_cast<int>(n);
}

int gsb_decode_pool(gsb_ctx* ctx, const gsb_profile* prof, const gsb_pool_cfg* cfg,
                    const gsb_pool_stream* st, const gsb_pool_args* a, void* stream) {
  if (!ctx || !prof || !cfg || !st || !a) return GSB_INVALID_ARGUMENT;
  const int W = cfg->n_decode_workers, MB = cfg->max_batch;
  if (W < 1 || W > 30) return gsb_set_error(ctx, GSB_MODEL_ERROR, "decode pool: 1..30 decode workers");
  if (MB < 1 || MB > 256) return gsb_set_error(ctx, GSB_MODEL_ERROR, "decode pool: max_batch 1..256");
  if (cfg->max_queue < 1) return gsb_set_error(ctx, GSB_MODEL_ERROR, "decode pool: max_queue >= 1");
  if (cfg->tbt_cap < 1 || cfg->tbt_cap > GSB_MAX_TBT_WINDOW)
    return gsb_set_error(ctx, GSB_MODEL_ERROR, "decode pool: tbt_cap 1..256");
  if (cfg->tps_cap < 1 || cfg->pending_cap < 1)
    return gsb_set_error(ctx, GSB_MODEL_ERROR, "decode pool: capacities must be positive");
  if (a->n_buckets < 1 || a->n_buckets > GSB_MAX_BUCKETS)
    return gsb_set_error(ctx, GSB_MODEL_ERROR, "band table: need 1..32 buckets");
  if (a->n_scen <= 0) return GSB_OK;
  if (a->n_scen > 0xffffffffll) return gsb_set_error(ctx, GSB_INVALID_ARGUMENT, "decode pool: too many scenarios");
  const bool req_out = a->d_req_first && a->d_req_finish && a->d_req_worker;
  PoolParams P;
  P.prof = *prof;
  P.cfg = *cfg;
  P.st = *st;
  P.a = *a;
  P.W = W;
  P.MB = MB;
  P.RC_full = cfg->tbt_cap;
  P.TC = cfg->tps_cap;
  auto kern = req_out ? k_decode_pool<true> : k_decode_pool<false>;
  // First launch: a TBT run ring of at most 32 runs per worker (a run is the equal gaps of
  // consecutive steps with the same gap, so a 256-token window rarely holds more than a few),
  // which keeps five 4-scenario CTAs resident per SM (44 KB each; 102 registers since the
  // controllers and the cold worker fields live in shared memory) with the smallest carve-out; the
  // scenarios whose ring fills are replayed by a second launch with the full capacity
  // (runs <= tokens <= tbt_cap). Both launches are always enqueued (graph-capturable); the
  // second exits at once when nothing overflowed. Pool rate by first-launch ring (runs merged):
  // 256: 6.5e4/s (3 CTAs/SM), 128: 7.8e4, 96-32: 8.1-8.2e4 (tools/k5_runcap_sweep.sh).
  int fast_runs = 32;
  if (const char* e = std::getenv("GSB_POOL_RUN_CAP")) fast_runs = std::atoi(e);  // tests
  if (fast_runs < 1) fast_runs = 1;
  const int RC1 = fast_runs < P.RC_full ? fast_runs : P.RC_full;
  const int RC2 = P.RC_full;
  int per_sm[2] = {0, 0};
  int64_t warp_bytes[2];
  warp_bytes[0] = smem_bytes(W, MB, RC1, P.TC, a->n_buckets);
  warp_bytes[1] = smem_bytes(W, MB, RC2, P.TC, a->n_buckets);
  if (warp_bytes[1] * kWarpsPerBlock > 227 * 1024)
    return gsb_set_error(ctx, GSB_MODEL_ERROR, "decode pool: per-scenario state exceeds shared memory");
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(warp_bytes[1] * kWarpsPerBlock)) != cudaSuccess)
    return gsb_check_launch(ctx, "decode_pool attr");
  for (int i = 0; i < 2; ++i) {
    const int64_t block_smem = warp_bytes[i] * kWarpsPerBlock;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[i], kern, kWarpsPerBlock * 32,
                                                  static_cast<size_t>(block_smem));
    if (per_sm[i] < 1) per_sm[i] = 1;
  }
  const int64_t need = (a->n_scen + kWarpsPerBlock - 1) / kWarpsPerBlock;
  int64_t blocks = static_cast<int64_t>(ctx->n_sms) * per_sm[0];
  if (blocks > need) blocks = need;
  int64_t blocks2 = static_cast<int64_t>(ctx->n_sms) * per_sm[1];
  if (blocks2 > blocks) blocks2 = blocks;
  const int64_t ws_ints = blocks * kWarpsPerBlock * W * static_cast<int64_t>(cfg->pending_cap);
  const size_t bytes = 256 + static_cast<size_t>(ws_ints) * 4 + static_cast<size_t>(a->n_scen) * 4;
  char* scratch = static_cast<char*>(gsb_scratch(ctx, bytes));
  if (!scratch) return gsb_set_error(ctx, GSB_CUDA_ERROR, "decode pool: workspace allocation failed");
  unsigned* hdr = reinterpret_cast<unsigned*>(scratch);  // [0] claims, [1] replay claims, [2] replays
  P.ws_pending = reinterpret_cast<int32_t*>(scratch + 256);
  uint32_t* list = reinterpret_cast<uint32_t*>(scratch + 256 + ws_ints * 4);
  cudaStream_t s = gsb_pick_stream(ctx, stream);
  cudaMemsetAsync(hdr, 0, 4 * sizeof(unsigned), s);
  P.rerun_n = hdr + 2;
  P.rerun_list = list;
  P.RC = RC1;
  P.warp_bytes = warp_bytes[0];
  P.counter = hdr;
  P.list_in = nullptr;
  P.list_n = nullptr;
  kern<<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32,
         static_cast<size_t>(warp_bytes[0] * kWarpsPerBlock), s>>>(P);
  if (RC1 == RC2) return gsb_check_launch(ctx, "decode_pool");
  P.RC = RC2;
  P.warp_bytes = warp_bytes[1];
  P.counter = hdr + 1;
  P.list_in = list;
  P.list_n = hdr + 2;
  kern<<<static_cast<unsigned>(blocks2), kWarpsPerBlock * 32,
         static_cast<size_t>(warp_bytes[1] * kWarpsPerBlock), s>>>(P);
  return gsb_check_launch(ctx, "decode_pool");
}

}  // extern "C"
