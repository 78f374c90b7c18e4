"""Synthetic inputs for the decision engine (host-side input production; not the hot path).

Trace shapes are the documented harness conventions of SURVEY.md 8(d): the reference has
no Alibaba/Azure generators, only gen_poisson_trace with a bimodal LoadShape
(proj/src/trace.cpp:152-175), so "Alibaba-shaped" / "Azure-shaped" are LoadShape
parameterisations. These numpy generators draw from the same distributions (exponential
inter-arrival gaps, Bernoulli long mode, lengths uniform on [mean/2, 3*mean/2]) with a
PCG64 stream; the parity tests use the reference's own mt19937_64 generator instead.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import api

# LoadShape parameterisations; alibaba_chat = the reference's chat defaults
# (proj/tools/greensim_cli.cpp:73-80, acceptance_main.cpp:287-292)
LOAD_SHAPES = {
    "alibaba_chat": dict(short=512.0, long=4096.0, long_fraction=0.10, output=128.0),
    "azure_code": dict(short=1024.0, long=6144.0, long_fraction=0.35, output=32.0),
    "azure_conv": dict(short=768.0, long=3072.0, long_fraction=0.15, output=256.0),
}

# routing thresholds for 3 / 5 / 8 length classes
THRESHOLDS = {
    3: [512, 1024],
    5: [256, 512, 1024, 2048],
    8: [128, 256, 512, 768, 1024, 2048, 4096],
}

TPS_LEVELS = np.arange(200.0, 3000.0 + 1e-9, 200.0)  # SimConfig band levels (simkernel.hpp:83-85)


def synth_profiles(n: int = 4) -> list:
    """default.json plus synthetic variants with scaled latency / power coefficients
    (named synth-*, never a real model; each passes GpuProfile::validate)."""
    base = api.GpuProfile.default_profile()
    out = [base]
    for i, (ls, ps) in enumerate([(1.6, 1.25), (0.7, 0.8), (2.5, 1.6)][: n - 1]):
        p = api.GpuProfile(f"synth-{i}", base.grid,
                           api.LatencyModel(base.prefill.a * ls, base.prefill.b * ls,
                                            base.prefill.c * ls, 1410.0),
                           base.decode,
                           api.PowerModel(base.power.k3 * ps, base.power.k2 * ps,
                                          base.power.k1 * ps, base.power.k0 * ps,
                                          base.power.p_idle_w * ps))
        p.validate()
        out.append(p)
    return out


def _lengths(rng, mean, n):
    lo = max(1, int(round(mean * 0.5)))
    hi = max(lo, int(round(mean * 1.5)))
    return rng.integers(lo, hi + 1, n, dtype=np.int64).astype(np.int32)


def poisson_trace(qps: float, duration_ms: int, shape: str, seed: int, t0_ms: int = 0):
    """Poisson arrivals over [t0, t0 + duration) with a bimodal length mix.
    Returns (arrival_ms i64, prompt i32, output i32), arrivals non-decreasing."""
    s = LOAD_SHAPES[shape]
    rng = np.random.default_rng(seed)
    n_est = int(qps * duration_ms / 1000.0 * 1.05 + 10 * np.sqrt(qps * duration_ms / 1000.0) + 100)
    gaps = rng.exponential(1000.0 / qps, n_est)
    t = np.cumsum(gaps)
    t = t[t < duration_ms]
    n = len(t)
    arrival = (t0_ms + np.floor(t)).astype(np.int64)
    is_long = rng.random(n) < s["long_fraction"]
    prompt = np.where(is_long, _lengths(rng, s["long"], n), _lengths(rng, s["short"], n)).astype(np.int32)
    output = _lengths(rng, s["output"], n)
    return arrival, prompt, output


def mixed_trace(qps: float, duration_ms: int, seed: int, segment_ms: int = 6 * 3_600_000,
                t0_ms: int = 0):
    """Multi-day Alibaba + Azure mix: alternating segments of the three shapes (C5)."""
    shapes = ["alibaba_chat", "azure_conv", "azure_code"]
    parts = []
    t = 0
    i = 0
    while t < duration_ms:
        d = min(segment_ms, duration_ms - t)
        parts.append(poisson_trace(qps, d, shapes[i % 3], seed + i, t0_ms + t))
        t += d
        i += 1
    return tuple(np.concatenate([p[k] for p in parts]) for k in range(3))


def decode_telemetry(n_streams: int, t_end_ms: float, seed: int,
                     profile: api.GpuProfile | None = None, tps_mean: float = 1500.0,
                     tps_amp: float = 1000.0, period_ms: float = 120_000.0,
                     n_workers: int = 4, f_mhz: float = 1410.0) -> api.Telemetry:
    """Per-worker step-end telemetry of a sinusoidally loaded decode pool at a fixed clock
    (the offered rate of gen_sinusoid_decode_trace, proj/src/trace.cpp:239-285, spread over
    n_workers). Each step: batch B from the fluid steady state of the offered rate
    (decode_ctl.cpp:28-50) with Poisson jitter, step time decode_step_raw_ms(B, f)
    (gpu_model.cpp:101-103), B tokens emitted, one gap per continuing stream."""
    prof = profile or api.GpuProfile.default_profile()
    d = prof.decode
    rng = np.random.default_rng(seed)
    ev_off, t_all, tok_all, goff, gaps_all = [0], [], [], [0], []
    fr = d.f_ref_mhz / f_mhz
    s0 = d.alpha0_ms + d.beta0_ms * fr
    s1 = d.alpha1_ms + d.beta1_ms * fr
    for s in range(n_streams):
        phase = rng.uniform(0, period_ms)
        t = rng.uniform(0.0, 30.0)
        ts, toks, gs = [], [], []
        prev_b = 1
        while t <= t_end_ms:
            tau = (tps_mean + tps_amp * np.sin(2 * np.pi * (t + phase) / period_ms)) / n_workers
            denom = 1000.0 - tau * s1
            b = tau * s0 / denom if denom > 0 else 64.0
            b = int(np.clip(rng.poisson(max(b, 0.5)), 1, 64))
            step = (d.alpha0_ms + d.alpha1_ms * b) + (d.beta0_ms + d.beta1_ms * b) * fr
            step *= 1.0 + 0.05 * rng.standard_normal()
            t = t + max(step, 1.0)
            cont = min(b, prev_b)
            ts.append(t)
            toks.append(b)
            gs.append(np.full(cont, max(step, 1.0)) * (1.0 + 0.02 * rng.standard_normal(cont)))
            prev_b = b
        t_all.append(np.array(ts))
        tok_all.append(np.array(toks, np.int32))
        for g in gs:
            goff.append(goff[-1] + len(g))
        gaps_all.extend(gs)
        ev_off.append(ev_off[-1] + len(ts))
    return api.Telemetry(np.array(ev_off, np.int64), np.concatenate(t_all),
                         np.concatenate(tok_all), np.array(goff, np.int64),
                         np.concatenate(gaps_all) if gaps_all else np.zeros(0))


@dataclass
class DecodeSweep:
    """A controller parameter sweep: hysteresis x step x TBT target x margin x profile x
    bias (C3 / C4). One scenario = one parameter setting replayed on a 4-worker pool."""
    cfgs: np.ndarray          # CTL_DTYPE [N*W]
    table_of: np.ndarray      # i32 [N*W]
    stream_of: np.ndarray     # i32 [N*W]
    worker: np.ndarray        # i32 [N*W]
    table_profile: np.ndarray  # i32 [T]
    table_tslo: np.ndarray    # f64 [T] (tslo * margin_decode, simkernel.cpp:203-205)
    n_scenarios: int
    n_workers: int


def decode_sweep(n_scenarios: int, n_profiles: int = 4, n_workers: int = 4,
                 streams_per_profile: int = 4, seed: int = 0) -> DecodeSweep:
    hyst = np.array([1, 2, 3, 4, 5])
    steps = np.array([15.0, 30.0, 45.0, 60.0])
    margins = np.array([0.6, 0.8, 0.95, 1.2, 1.5])
    bias = np.array([0.7, 0.8])
    per = len(hyst) * len(steps) * len(margins) * len(bias) * n_profiles
    n_tslo = max(1, -(-n_scenarios // per))
    tslos = np.linspace(50.0, 150.0, n_tslo)
    grid = np.stack(np.meshgrid(np.arange(n_profiles), np.arange(n_tslo), np.arange(len(margins)),
                                np.arange(len(hyst)), np.arange(len(steps)), np.arange(len(bias)),
                                indexing="ij"), -1).reshape(-1, 6)[:n_scenarios]
    # band table per (profile, tslo, margin)
    t_key = (grid[:, 0] * n_tslo + grid[:, 1]) * len(margins) + grid[:, 2]
    uniq, table_idx = np.unique(t_key, return_inverse=True)
    tp = (uniq // (n_tslo * len(margins))).astype(np.int32)
    tt = ((uniq // len(margins)) % n_tslo)
    tm = uniq % len(margins)
    table_tslo = tslos[tt] * margins[tm]
    N = len(grid)
    cfg = np.zeros(N, api.CTL_DTYPE)
    cfg["tslo_ms"] = tslos[grid[:, 1]]
    cfg["margin_decode"] = margins[grid[:, 2]]
    cfg["fine_period_ms"] = 20.0
    cfg["coarse_period_ms"] = 200.0
    cfg["adapt_period_s"] = 6.0
    cfg["step_mhz"] = steps[grid[:, 4]]
    cfg["max_step_mhz"] = np.maximum(30.0, steps[grid[:, 4]])
    cfg["hysteresis_count"] = hyst[grid[:, 3]]
    cfg["tbt_window_tokens"] = 256
    cfg["bias_threshold"] = bias[grid[:, 5]]
    cfg["tps_scale"] = float(n_workers)
    cfg["upper_margin"] = 1.0
    cfg["lower_margin"] = 0.65
    rep = np.repeat
    cfgs = rep(cfg, n_workers)
    table_of = rep(table_idx.astype(np.int32), n_workers)
    worker = np.tile(np.arange(n_workers, dtype=np.int32), N)
    # worker w of a scenario on profile p replays telemetry stream p*streams_per_profile + w
    stream_of = (rep(grid[:, 0] * streams_per_profile, n_workers)
                 + worker % streams_per_profile).astype(np.int32)
    return DecodeSweep(cfgs, table_of, stream_of, worker, tp, table_tslo, N, n_workers)


# ------------------------------------------------------------------ closed-loop decode pool (K5)
def sinusoid_decode_trace(tps_mean: float, tps_amp: float, period_ms: float, duration_ms: int,
                          seed: int):
    """Sinusoidal decode workload with the distributions of gen_sinusoid_decode_trace
    (proj/src/trace.cpp:239-285): request k arrives when the cumulative offered tokens
    L(t) = mean*t/1000 + amp/1000 * P/2pi * (1 - cos(2pi t/P)) reach the tokens of the
    requests before it; prompt 32, output uniform on [64, 192]. PCG64 instead of mt19937_64,
    and a vectorised bisection. Returns (arrival_ms i64, prompt i32, output i32)."""
    rng = np.random.default_rng(seed)
    n_max = int(duration_ms / 1000.0 * (tps_mean + tps_amp) / 64.0) + 16
    out = rng.integers(64, 193, n_max).astype(np.int32)
    target = np.concatenate([[0.0], np.cumsum(out[:-1], dtype=np.float64)])
    two_pi = 2.0 * np.pi

    def cum(t):
        return tps_mean * t / 1000.0 + tps_amp / 1000.0 * (period_ms / two_pi) * (
            1.0 - np.cos(two_pi * t / period_ms))

    lo = np.zeros(n_max)
    hi = np.full(n_max, 1000.0)
    while np.any(cum(hi) < target):
        hi = np.where(cum(hi) < target, hi + 1000.0, hi)
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        below = cum(mid) < target
        lo = np.where(below, mid, lo)
        hi = np.where(below, hi, mid)
    arrival = np.rint(0.5 * (lo + hi)).astype(np.int64)
    keep = arrival < duration_ms
    n = int(np.argmin(keep)) if not keep.all() else n_max
    return arrival[:n], np.full(n, 32, np.int32), out[:n]


def decode_stream(arrival, prompt, output, profile: api.GpuProfile | None = None,
                  routing: api.RoutingConfig | None = None, slo: api.SloConfig = api.SloConfig(),
                  handoff_ms: float = 0.0, prefill_f_mhz: float | None = None) -> api.DecodeStream:
    """Decode-enqueue stream of a prefill pool at a pinned clock (synthetic input for K5):
    per routing class a FIFO served by that class's workers in arrival order, service time
    prefill_latency_ms(prompt, f) (gpu_model.cpp:94-97); the request reaches the decode pool
    handoff_ms after its prefill ends (simkernel.cpp:317-326). The reference's own stream
    (GreenLLM prefill clocks) is recorded by the oracle for the parity tests instead."""
    prof = profile or api.GpuProfile.default_profile()
    rc = routing or api.RoutingConfig()
    f = prefill_f_mhz or prof.grid.f_max_mhz
    lat = prof.prefill
    n = len(arrival)
    thr = np.asarray(rc.thresholds if rc.enabled else [], np.int64)
    cls = (np.asarray(prompt, np.int64)[:, None] > thr[None, :]).sum(1) if len(thr) else np.zeros(n, np.int64)
    workers = {}
    for w, c in enumerate(rc.worker_map if rc.enabled else [0] * 2):
        workers.setdefault(int(c), []).append(0.0)
    L = np.asarray(prompt, np.float64)
    svc = ((lat.a * L + lat.b) * L + lat.c) * lat.f_ref_mhz / f
    end = np.zeros(n)
    arr = np.asarray(arrival, np.float64)
    for i in range(n):
        free = workers[int(cls[i])]
        k = int(np.argmin(free))
        start = max(arr[i], free[k])
        free[k] = end[i] = start + svc[i]
    t = end + handoff_ms
    order = np.argsort(t, kind="stable")
    big = np.asarray(prompt) > 1024  # SLO class SM/L (simkernel.cpp:258-260)
    ttft = np.where(big, slo.ttft_l_ms, slo.ttft_sm_ms).astype(np.float64)
    return api.DecodeStream(t[order], order.astype(np.int32), np.ascontiguousarray(output, np.int32),
                            arr, ttft, float(max(end.max(), arr.max())))


def pool_sweep(n_scenarios: int, seed: int = 0) -> np.ndarray:
    """C3: dual-loop controller sweep hysteresis x step size x TBT target (x margin x bias),
    one DecodeCtlConfig per scenario (CTL_DTYPE [N])."""
    hyst = np.array([1, 2, 3, 4, 5])
    steps = np.array([15.0, 30.0, 45.0, 60.0])
    margins = np.array([0.6, 0.8, 0.95, 1.2, 1.5])
    bias = np.array([0.7, 0.8])
    per = len(hyst) * len(steps) * len(margins) * len(bias)
    n_tslo = max(1, -(-n_scenarios // per))
    tslos = np.linspace(50.0, 150.0, n_tslo)
    g = np.stack(np.meshgrid(np.arange(n_tslo), np.arange(len(margins)), np.arange(len(hyst)),
                             np.arange(len(steps)), np.arange(len(bias)), indexing="ij"),
                 -1).reshape(-1, 5)[:n_scenarios]
    cfg = np.zeros(len(g), api.CTL_DTYPE)
    cfg["tslo_ms"] = tslos[g[:, 0]]
    cfg["margin_decode"] = margins[g[:, 1]]
    cfg["fine_period_ms"] = 20.0
    cfg["coarse_period_ms"] = 200.0
    cfg["adapt_period_s"] = 6.0
    cfg["step_mhz"] = steps[g[:, 3]]
    cfg["max_step_mhz"] = np.maximum(30.0, steps[g[:, 3]])
    cfg["hysteresis_count"] = hyst[g[:, 2]]
    cfg["tbt_window_tokens"] = 256
    cfg["bias_threshold"] = bias[g[:, 4]]
    cfg["tps_scale"] = 4.0
    cfg["upper_margin"] = 1.0
    cfg["lower_margin"] = 0.65
    return cfg
