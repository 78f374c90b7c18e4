"""Python host mirror of the reference's decision-engine interface over libgsb.so.

Names, argument meaning and error behaviour follow /root/reference/proj/include/greensim:
  gpu_model.hpp   FrequencyGrid, LatencyModel, DecodeStepModel, PowerModel, GpuProfile
  prefill_opt.hpp PrefillJob, PrefillBatch, EnergyBreakdown, FrequencyChoice,
                  QueueOptimizerConfig, ClassQueueSnapshot, PrefillFreqCommand,
                  busy_time_ms, energy_total, select_frequency, queue_optimizer_tick
  router.hpp      RoutingConfig, classify, Dispatcher
  decode_ctl.hpp  DecodeCtlConfig, BandBucket, FreqBandTable, build_band_table,
                  DecisionRecord
Every computation runs in the sm_100a kernels behind include/gsb.h on the chosen CUDA
device; this module only marshals arguments (torch is used for device memory and
streams). ModelError / RouterError are raised from the C status codes exactly where the
reference throws.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np
import torch

from . import _lib as L


class ModelError(RuntimeError):
    """greensim::ModelError (gpu_model.hpp:11-13)."""


class RouterError(RuntimeError):
    """greensim::RouterError (router.hpp:13-15)."""


class TraceError(RuntimeError):
    """greensim::TraceError (trace.hpp:36-40); `kind` is the TraceError::Kind name and `row`
    the reference's 1-based row counter of the failing line (None when not row-bound)."""

    def __init__(self, msg: str, kind: Optional[str] = None, row: Optional[int] = None):
        super().__init__(msg)
        self.kind = kind
        self.row = row


class CudaError(RuntimeError):
    pass


_ERRORS = {L.MODEL_ERROR: ModelError, L.ROUTER_ERROR: RouterError, L.TRACE_ERROR: TraceError,
           L.CUDA_ERROR: CudaError, L.INVALID_ARGUMENT: ValueError}


# ------------------------------------------------------------------ gpu_model.hpp
@dataclass
class FrequencyGrid:
    f_min_mhz: float = 210.0
    f_max_mhz: float = 1410.0
    step_mhz: float = 15.0
    f_ref_mhz: float = 1410.0

    def size(self) -> int:  # gpu_model.cpp:24-26
        return int(round((self.f_max_mhz - self.f_min_mhz) / self.step_mhz)) + 1

    def at(self, i: int) -> float:  # gpu_model.cpp:28
        return self.f_min_mhz + self.step_mhz * float(i)

    def frequencies(self) -> list:
        return [self.at(i) for i in range(self.size())]

    def on_grid(self, f: float) -> bool:  # gpu_model.cpp:18-22
        if f < self.f_min_mhz - 1e-9 or f > self.f_max_mhz + 1e-9:
            return False
        k = (f - self.f_min_mhz) / self.step_mhz
        return abs(k - round(k)) < 1e-9


@dataclass
class LatencyModel:
    a: float = 0.0
    b: float = 0.0
    c: float = 0.0
    f_ref_mhz: float = 1410.0


@dataclass
class DecodeStepModel:
    alpha0_ms: float = 0.0
    alpha1_ms: float = 0.0
    beta0_ms: float = 0.0
    beta1_ms: float = 0.0
    f_ref_mhz: float = 1410.0


@dataclass
class PowerModel:
    k3: float = 0.0
    k2: float = 0.0
    k1: float = 0.0
    k0: float = 0.0
    p_idle_w: float = 0.0


@dataclass
class GpuProfile:
    name: str = "default"
    grid: FrequencyGrid = field(default_factory=FrequencyGrid)
    prefill: LatencyModel = field(default_factory=LatencyModel)
    decode: DecodeStepModel = field(default_factory=DecodeStepModel)
    power: PowerModel = field(default_factory=PowerModel)

    @staticmethod
    def default_profile() -> "GpuProfile":
        """GpuProfile::default_profile (gpu_model.cpp:121-130): synth-a100-40g."""
        p = GpuProfile("synth-a100-40g", FrequencyGrid(210.0, 1410.0, 15.0, 1410.0),
                       LatencyModel(2.0e-5, 0.12, 8.0, 1410.0),
                       DecodeStepModel(14.5, 0.1, 9.0, 0.135, 1410.0),
                       PowerModel(1.6e-7, -1.0e-4, 0.05, 216.5, 15.0))
        p.validate()
        return p

    def to_c(self) -> L.CProfile:
        g, a, d, w = self.grid, self.prefill, self.decode, self.power
        return L.CProfile(g.f_min_mhz, g.f_max_mhz, g.step_mhz, g.f_ref_mhz, a.a, a.b, a.c,
                          a.f_ref_mhz, d.alpha0_ms, d.alpha1_ms, d.beta0_ms, d.beta1_ms,
                          d.f_ref_mhz, w.k3, w.k2, w.k1, w.k0, w.p_idle_w)

    def key(self) -> tuple:
        c = self.to_c()
        return tuple(getattr(c, n) for n, _ in c._fields_)

    def validate(self) -> None:
        """GpuProfile::validate (gpu_model.cpp:80-87); raises ModelError."""
        msg = C.create_string_buffer(256)
        rc = L.load().gsb_profile_validate(C.byref(self.to_c()), msg, 256)
        if rc != L.OK:
            raise ModelError(msg.value.decode())

    @staticmethod
    def from_json(path: str) -> "GpuProfile":
        """Profile JSON schema of proj/profiles/*.json (io.hpp:14-19)."""
        with open(path) as fh:
            j = json.load(fh)
        p = GpuProfile(j.get("name", "default"),
                       FrequencyGrid(**{k: float(v) for k, v in j["grid"].items()}),
                       LatencyModel(**{k: float(v) for k, v in j["prefill_latency"].items()}),
                       DecodeStepModel(**{k: float(v) for k, v in j["decode_step"].items()}),
                       PowerModel(**{k: float(v) for k, v in j["power"].items()}))
        p.validate()
        return p

    def to_json(self) -> dict:
        g, a, d, w = self.grid, self.prefill, self.decode, self.power
        return {"name": self.name,
                "grid": {"f_min_mhz": g.f_min_mhz, "f_max_mhz": g.f_max_mhz,
                         "step_mhz": g.step_mhz, "f_ref_mhz": g.f_ref_mhz},
                "prefill_latency": {"a": a.a, "b": a.b, "c": a.c, "f_ref_mhz": a.f_ref_mhz},
                "decode_step": {"alpha0_ms": d.alpha0_ms, "alpha1_ms": d.alpha1_ms,
                                "beta0_ms": d.beta0_ms, "beta1_ms": d.beta1_ms,
                                "f_ref_mhz": d.f_ref_mhz},
                "power": {"k3": w.k3, "k2": w.k2, "k1": w.k1, "k0": w.k0,
                          "p_idle_w": w.p_idle_w}}


# ------------------------------------------------------------------ prefill_opt.hpp
@dataclass
class PrefillJob:
    request_id: int = 0
    prompt_tokens: int = 0
    deadline_ms: float = 0.0
    work_fraction: float = 1.0


@dataclass
class PrefillBatch:
    jobs: list = field(default_factory=list)


@dataclass
class EnergyBreakdown:
    active_j: float = 0.0
    idle_j: float = 0.0
    total_j: float = 0.0
    feasible: bool = True


@dataclass
class FrequencyChoice:
    f_mhz: float = 0.0
    energy_j: float = 0.0


@dataclass
class QueueOptimizerConfig:
    resolve_period_ms: float = 100.0
    margin_prefill: float = 0.95
    min_budget_ms: float = 100.0
    first_token_allowance_ms: float = 100.0

    def to_c(self) -> L.CQoptCfg:
        return L.CQoptCfg(self.resolve_period_ms, self.margin_prefill, self.min_budget_ms,
                          self.first_token_allowance_ms)


@dataclass
class ClassQueueSnapshot:
    class_id: int = 0
    batch: PrefillBatch = field(default_factory=PrefillBatch)


@dataclass
class PrefillFreqCommand:
    class_id: int = 0
    f_mhz: float = 0.0
    window_ms: float = 0.0
    infeasible: bool = False


# ------------------------------------------------------------------ router.hpp
@dataclass
class RoutingConfig:
    enabled: bool = True
    thresholds: list = field(default_factory=lambda: [1024])
    worker_map: list = field(default_factory=lambda: [0, 1])

    def n_classes(self) -> int:
        return len(self.thresholds) + 1

    def validate(self, n_prefill_workers: int) -> None:
        """RoutingConfig::validate (router.cpp:7-24); raises RouterError."""
        wm = np.ascontiguousarray(self.worker_map[:n_prefill_workers] if len(self.worker_map)
                                  >= n_prefill_workers else self.worker_map, np.int32)
        msg = C.create_string_buffer(256)
        cfg = _route_cfg(self, 1, 0, 1)
        thr = [int(t) for t in self.thresholds]
        # the reference's order (router.cpp:8-13) over the WHOLE list, then this ABI's cap
        if not thr:
            raise RouterError("routing: need at least one threshold")
        if any(a >= b for a, b in zip(thr, thr[1:])):
            raise RouterError("routing: thresholds must be ascending and distinct")
        if any(t < 1 for t in thr):
            raise RouterError("routing: thresholds must be >= 1")
        if len(thr) > L.GSB_MAX_CLASSES - 1:
            raise RouterError("routing: more than 7 thresholds")
        if self.enabled and len(self.worker_map) != n_prefill_workers:
            raise RouterError("routing: worker_map must name a class per prefill worker")
        rc = L.load().gsb_routing_validate(C.byref(cfg), n_prefill_workers,
                                           wm.ctypes.data_as(C.c_void_p), msg, 256)
        if rc != L.OK:
            raise RouterError(msg.value.decode())


@dataclass
class SloConfig:
    """greensim::SloConfig (simkernel.hpp:53-62)."""
    ttft_sm_ms: float = 400.0
    ttft_l_ms: float = 2000.0
    tbt_p95_ms: float = 100.0


def _route_cfg(rc: RoutingConfig, window_ms: int, w0: int, n_windows: int,
               slo: SloConfig = SloConfig(), allowance: float = 100.0) -> L.CRouteCfg:
    c = L.CRouteCfg()
    thr = list(rc.thresholds)
    c.n_thresholds = len(thr)
    for i, t in enumerate(thr[:L.GSB_MAX_CLASSES - 1]):
        c.thresholds[i] = int(t)
    c.enabled = 1 if rc.enabled else 0
    c.slo_boundary_tokens = 1024
    c.window_ms, c.w0, c.n_windows = int(window_ms), int(w0), int(n_windows)
    c.ttft_sm_ms, c.ttft_l_ms = slo.ttft_sm_ms, slo.ttft_l_ms
    c.first_token_allowance_ms = allowance
    return c


# ------------------------------------------------------------------ decode_ctl.hpp
@dataclass
class DecodeCtlConfig:
    tslo_ms: float = 100.0
    margin_decode: float = 0.95
    fine_period_ms: float = 20.0
    coarse_period_ms: float = 200.0
    adapt_period_s: float = 6.0
    step_mhz: float = 15.0
    max_step_mhz: float = 30.0
    hysteresis_count: int = 3
    bias_threshold: float = 0.8
    tbt_window_tokens: int = 256
    tps_scale: float = 4.0
    upper_margin: float = 1.0
    lower_margin: float = 0.65

    def to_c(self) -> L.CCtlCfg:
        return L.CCtlCfg(self.tslo_ms, self.margin_decode, self.fine_period_ms,
                         self.coarse_period_ms, self.adapt_period_s, self.step_mhz,
                         self.max_step_mhz, int(self.hysteresis_count),
                         int(self.tbt_window_tokens), self.bias_threshold, self.tps_scale,
                         self.upper_margin, self.lower_margin)

    def validate(self) -> None:
        """DecodeCtlConfig::validate (decode_ctl.cpp:12-26); raises ModelError."""
        msg = C.create_string_buffer(256)
        if L.load().gsb_ctl_cfg_validate(C.byref(self.to_c()), msg, 256) != L.OK:
            raise ModelError(msg.value.decode())


@dataclass
class BandBucket:
    tps_lo: float = 0.0
    tps_hi: float = 0.0
    f_opt_mhz: float = 0.0
    feasible: bool = True


@dataclass
class FreqBandTable:
    buckets: list = field(default_factory=list)

    def bucket_index(self, tps: float) -> int:  # decode_ctl.cpp:47-51
        for i, b in enumerate(self.buckets):
            if tps <= b.tps_hi:
                return i
        return len(self.buckets) - 1

    def band(self, bucket: int, grid: FrequencyGrid, step_mhz: float):  # :52-57
        f = self.buckets[bucket].f_opt_mhz
        lo, hi = f - step_mhz, f + step_mhz
        return (lo if grid.f_min_mhz < lo else grid.f_min_mhz,
                grid.f_max_mhz if grid.f_max_mhz < hi else hi)


ACTIONS = ("hold", "up", "down", "coarse_hold", "coarse_pending", "coarse_commit", "adapt_up",
           "adapt_down")

DECISION_DTYPE = np.dtype([("tick_ms", "<f8"), ("tps", "<f8"), ("p95_tbt_ms", "<f8"),
                           ("band_lo", "<f8"), ("band_hi", "<f8"), ("command_mhz", "<f8"),
                           ("worker", "<i4"), ("bucket", "<i4"), ("action", "<i4"),
                           ("pad_", "<i4")])

CTL_DTYPE = np.dtype([("tslo_ms", "<f8"), ("margin_decode", "<f8"), ("fine_period_ms", "<f8"),
                      ("coarse_period_ms", "<f8"), ("adapt_period_s", "<f8"),
                      ("step_mhz", "<f8"), ("max_step_mhz", "<f8"),
                      ("hysteresis_count", "<i4"), ("tbt_window_tokens", "<i4"),
                      ("bias_threshold", "<f8"), ("tps_scale", "<f8"),
                      ("upper_margin", "<f8"), ("lower_margin", "<f8")])
assert CTL_DTYPE.itemsize == C.sizeof(L.CCtlCfg)


def ctl_cfg_array(cfgs: Sequence[DecodeCtlConfig]) -> np.ndarray:
    a = np.zeros(len(cfgs), CTL_DTYPE)
    for i, c in enumerate(cfgs):
        a[i] = (c.tslo_ms, c.margin_decode, c.fine_period_ms, c.coarse_period_ms,
                c.adapt_period_s, c.step_mhz, c.max_step_mhz, c.hysteresis_count,
                c.tbt_window_tokens, c.bias_threshold, c.tps_scale, c.upper_margin,
                c.lower_margin)
    return a


# ------------------------------------------------------------------ simkernel.hpp (decode pool)
@dataclass
class SimConfig:
    """greensim::SimConfig (simkernel.hpp:88-104), the fields the decode pool reads."""
    n_prefill_workers: int = 2
    n_decode_workers: int = 4
    gpus_per_prefill_worker: int = 2
    actuation_delay_ms: float = 5.0
    handoff_delay_ms: float = 0.0
    max_batch: int = 64
    max_queue: int = 10000
    band_tps_lo: float = 200.0
    band_tps_hi: float = 3000.0
    band_tps_step: float = 200.0

    def band_levels(self) -> np.ndarray:
        """The coarse band-table TPS levels, lo..hi inclusive (simkernel.cpp:200-203)."""
        lv, l = [], self.band_tps_lo
        while l <= self.band_tps_hi + 1e-9:
            lv.append(l)
            l += self.band_tps_step
        return np.array(lv, np.float64)


@dataclass
class DecodeStream:
    """A decode-enqueue stream (simkernel.cpp:347): (instant, request id) in the reference's
    processing order, plus the per-request fields the decode pool reads. One stream drives
    every decode parameter set (the prefill pool never waits on decode)."""
    t_ms: np.ndarray           # f64 [E]
    req: np.ndarray            # i32 [E]
    output_tokens: np.ndarray  # i32 [R] by request id
    arrival_ms: np.ndarray     # f64 [R]
    ttft_slo_ms: np.ndarray    # f64 [R] SloConfig::ttft_for(SM/L)
    end_floor_ms: float = 0.0  # prefill side's part of sim_end_ms


POOL_SUMMARY_DTYPE = np.dtype([
    ("decode_pool_j", "<f8"), ("active_decode_j", "<f8"), ("idle_j", "<f8"),
    ("sim_end_ms", "<f8"), ("n_completed", "<i8"), ("n_rejected", "<i8"), ("n_ttft_ok", "<i8"),
    ("n_tbt_ok", "<i8"), ("tbt_samples", "<i8"), ("tbt_samples_ok", "<i8"),
    ("n_decisions", "<i8"), ("n_freq_changes", "<i8"), ("n_steps", "<i8"),
    ("decision_digest", "<u8"), ("freq_digest", "<u8"), ("request_digest", "<u8"),
    ("status", "<i4"), ("pad_", "<i4")])
assert POOL_SUMMARY_DTYPE.itemsize == C.sizeof(L.CPoolSummary)


# ------------------------------------------------------------------ results
@dataclass
class RouteResult:
    """K1 output (device tensors). cells are window-major, class-minor."""
    n_classes: int
    n_windows: int
    window_ms: int
    w0: int
    bounds: torch.Tensor          # i64 [n_windows+1]
    cls: torch.Tensor             # u8  [n_req]   queue assignment per request
    count: torch.Tensor           # i32 (u32 bits) [cells]
    t_ref: torch.Tensor           # f64 [P, cells]
    min_deadline: Optional[torch.Tensor]   # f64 [cells]
    cell_off: Optional[torch.Tensor] = None  # i64 [cells+1]
    fifo: Optional[torch.Tensor] = None      # i64 [n_req] cell-major FIFO order
    profile_gen: int = -1                    # Engine.profile_gen its t_ref rows were built under
    nonempty: Optional[torch.Tensor] = None  # u32 (as i32) [cells]: non-empty cells, ascending
    n_nonempty: Optional[torch.Tensor] = None  # i64 [1]: entries of nonempty (device)
    t_ref_list: Optional[torch.Tensor] = None  # f64 [P, cells]: t_ref of the listed cells
    min_deadline_list: Optional[torch.Tensor] = None  # f64 [cells]: min_deadline, list order

    def cell_list(self) -> Optional["L.CCellList"]:
        """The gsb_cell_list K1b wrote (None: no list)."""
        if self.nonempty is None:
            return None
        return L.CCellList(_ptr(self.nonempty), _ptr(self.n_nonempty), _ptr(self.t_ref_list),
                           _ptr(self.min_deadline_list), self.nonempty.numel())

    @property
    def n_cells(self) -> int:
        return self.n_windows * self.n_classes


@dataclass
class SelectResult:
    """K2 output (device tensors) per (profile, cell)."""
    f_idx: torch.Tensor           # i16 [P, cells]; -1 infeasible, -2 empty
    energy_j: torch.Tensor        # f64 [P, cells]
    window_ms: torch.Tensor       # f64 [cells]


@dataclass
class HostPassResult:
    """prefill_pass_host output: host f_idx / energy [P, cells] and the per-chunk summary
    records (pinned bytes [chunks, P*C*48]; argmin cells relative to the chunk)."""
    f_idx: torch.Tensor
    energy_j: torch.Tensor
    chunk_summaries: Optional[torch.Tensor]
    chunks: int
    n_windows: int
    n_classes: int

    def chunk_records(self) -> np.ndarray:
        """[chunks, P*C] gsb_class_summary records"""
        from .distributed import SUMMARY_DTYPE
        return self.chunk_summaries.numpy().view(SUMMARY_DTYPE).reshape(self.chunks, -1)

    def summary(self) -> np.ndarray:
        """the chunks' summaries combined in window order (gsb_combine_summaries)"""
        from .distributed import combine_summaries_c
        return combine_summaries_c(self.chunk_records(),
                                   [a * self.n_classes for a in self.chunk_windows()[:-1]])

    def chunk_windows(self) -> list:
        """chunk k = windows [a_k, a_k+1): decreasing sizes, weights K, K-1, ..., 1
        (gsb_prefill_pass_host)"""
        K = self.chunks
        wsum, acc, out = K * (K + 1) // 2, 0, []
        for k in range(K + 1):
            out.append(self.n_windows * acc // wsum)
            if k < K:
                acc += K - k
        return out


@dataclass
class Telemetry:
    """Raw decode telemetry of S streams, CSR (include/gsb.h gsb_telemetry)."""
    ev_off: np.ndarray   # i64 [S+1]
    t_ms: np.ndarray     # f64 [E]
    tokens: np.ndarray   # i32 [E]
    gap_off: np.ndarray  # i64 [E+1]
    gaps: np.ndarray     # f64 [G]

    @property
    def n_streams(self) -> int:
        return len(self.ev_off) - 1


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    raise TypeError(type(t))


@dataclass
class TraceArrays:
    """A request trace on the device (greensim::Trace, trace.hpp:16-33) as SoA; request ids are
    the row indices; slo_class 0 = SM, 1 = L (classify_by_threshold, trace.cpp:32-34)."""
    arrival_ms: torch.Tensor
    prompt_tokens: torch.Tensor
    output_tokens: torch.Tensor
    slo_class: torch.Tensor
    has_class_column: bool
    name: str
    duration_ms: int
    nominal_qps: float


def _pinned(t, dtype) -> bool:
    """a contiguous pinned host tensor of dtype (read in place by the kernels)"""
    return (isinstance(t, torch.Tensor) and t.device.type == "cpu" and t.is_pinned()
            and t.dtype == dtype and t.is_contiguous())


class Engine:
    """One libgsb context on one CUDA device (single owner, like the reference's objects)."""

    def __init__(self, device: int = 0, profiles: Optional[Sequence[GpuProfile]] = None):
        self.lib = L.load()
        self.device = torch.device("cuda", device)
        torch.cuda.init()
        h = C.c_void_p()
        rc = self.lib.gsb_ctx_create(device, C.byref(h))
        if rc != L.OK:
            raise CudaError(f"gsb_ctx_create({device}) failed: "
                            f"{self.lib.gsb_status_string(rc).decode()} (needs an sm_100 GPU)")
        self.ctx = h
        self.profiles: list = []
        self.set_profiles(profiles or [GpuProfile.default_profile()])

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.gsb_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- plumbing
    def _check(self, rc: int):
        if rc != L.OK:
            msg = self.lib.gsb_last_error(self.ctx).decode()
            raise _ERRORS.get(rc, RuntimeError)(msg)

    def stream(self) -> int:
        """The caller's current torch stream as a cudaStream_t. torch's legacy default stream
        has handle 0, which the C ABI reads as "the context's own stream"; pass
        cudaStreamLegacy (1) instead so the kernels stay ordered after torch's copies."""
        s = torch.cuda.current_stream(self.device).cuda_stream
        return s if s else 1

    def _dev(self, a, dtype) -> torch.Tensor:
        if isinstance(a, torch.Tensor):
            return a.to(self.device, dtype).contiguous()
        a = np.ascontiguousarray(a)
        if not a.flags.writeable:
            a = a.copy()
        return torch.as_tensor(a, device=self.device).to(dtype).contiguous()

    def _empty(self, shape, dtype) -> torch.Tensor:
        return torch.empty(shape, dtype=dtype, device=self.device)

    def set_profiles(self, profiles: Sequence[GpuProfile]) -> None:
        arr = (L.CProfile * len(profiles))(*[p.to_c() for p in profiles])
        # (gsb_set_profiles orders the upload after every kernel already issued on the device)
        self._check(self.lib.gsb_set_profiles(self.ctx, len(profiles), C.cast(arr, C.c_void_p)))
        self.profiles = list(profiles)
        self.profile_gen = getattr(self, "profile_gen", 0) + 1

    def _profile_index(self, profile: GpuProfile) -> int:
        """Index of `profile` in the installed set. The reference's free functions take the
        profile as an argument (prefill_opt.hpp:40-57), so a profile outside the set is
        installed (a new generation); RouteResults built under the previous set are then
        rejected by prefill_select instead of being read against the wrong tables."""
        for i, p in enumerate(self.profiles):
            if p.key() == profile.key():
                return i
        self.set_profiles([profile])
        return 0

    def _check_gen(self, rr: "RouteResult") -> None:
        if rr.profile_gen != self.profile_gen:
            raise ModelError("RouteResult was built under another profile set (set_profiles was "
                             "called since); re-run route_bin")

    # ---------------------------------------------------------------- K1
    def window_bounds(self, arrival: torch.Tensor, rc: RoutingConfig, window_ms: int, w0: int,
                      n_windows: int) -> torch.Tensor:
        cfg = _route_cfg(rc, window_ms, w0, n_windows)
        bounds = self._empty(n_windows + 1, torch.int64)
        self._check(self.lib.gsb_window_bounds(self.ctx, C.byref(cfg), arrival.numel(),
                                               _ptr(arrival), _ptr(bounds), self.stream()))
        return bounds

    def route_bin(self, arrival, prompt, routing: RoutingConfig, window_ms: int, w0: int = 0,
                  n_windows: Optional[int] = None, want_deadline: bool = False,
                  want_fifo: bool = False, slo: SloConfig = SloConfig(),
                  allowance_ms: float = 100.0, out: Optional[RouteResult] = None,
                  prompt_ready: Optional[torch.cuda.Event] = None) -> RouteResult:
        """K1: classify every request (router.cpp:26-31) and bin the trace into
        (window, class) cells with the reference-order T_ref per profile.

        prompt_ready: an event after which `prompt` is complete (e.g. its upload on another
        stream); only K1b waits for it, so the window-bounds pass (arrivals only) overlaps it.

        A PINNED host int64 `arrival` tensor is read in place (zero copy): with unified
        addressing the kernels dereference pinned host memory directly, and K1a reads only one
        arrival per 256 requests plus a 64-byte probe per window edge (dense traces; else one
        arrival per 32 requests plus the 32-request tiles that hold a window start; the deadline
        mode reads every arrival once). A pinned int32 `prompt` tensor is read in place by K1b
        (plain loads instead of its TMA stage)."""
        if not _pinned(arrival, torch.int64):
            arrival = self._dev(arrival, torch.int64)
        if not _pinned(prompt, torch.int32):
            prompt = self._dev(prompt, torch.int32)
        n = arrival.numel()
        if n_windows is None:
            last = int(arrival[-1].item()) if n else 0
            n_windows = max(1, last // window_ms - w0 + 1)
        Cn = routing.n_classes() if routing.enabled else 1
        cells = n_windows * Cn
        cfg = _route_cfg(routing, window_ms, w0, n_windows, slo, allowance_ms)
        P = len(self.profiles)
        if out is None:
            out = RouteResult(Cn, n_windows, window_ms, w0, self._empty(n_windows + 1, torch.int64),
                              self._empty(n, torch.uint8), self._empty(cells, torch.int32),
                              self._empty((P, cells), torch.float64),
                              self._empty(cells, torch.float64) if want_deadline else None)
            if cells < 2 ** 32:  # K1b also emits the non-empty cell list K2 runs over
                out.nonempty = self._empty(cells, torch.int32)
                out.n_nonempty = self._empty(1, torch.int64)
                out.t_ref_list = self._empty((P, cells), torch.float64)
                if want_deadline:
                    out.min_deadline_list = self._empty(cells, torch.float64)
        s = self.stream()
        self._check(self.lib.gsb_window_bounds(self.ctx, C.byref(cfg), n, _ptr(arrival),
                                               _ptr(out.bounds), s))
        if prompt_ready is not None:
            torch.cuda.current_stream(self.device).wait_event(prompt_ready)
        cl = out.cell_list()
        self._check(self.lib.gsb_route_bin_list(self.ctx, C.byref(cfg), n, _ptr(arrival),
                                                _ptr(prompt), _ptr(out.bounds), _ptr(out.cls),
                                                _ptr(out.count), _ptr(out.t_ref),
                                                _ptr(out.min_deadline),
                                                C.byref(cl) if cl is not None else None, s))
        out.profile_gen = self.profile_gen
        if want_fifo:
            out.cell_off = self._empty(cells + 1, torch.int64)
            out.fifo = self._empty(n, torch.int64)
            self._check(self.lib.gsb_fifo_order(self.ctx, C.byref(cfg), n, _ptr(out.cls),
                                                _ptr(out.bounds), _ptr(out.count),
                                                _ptr(out.cell_off), _ptr(out.fifo), s))
        return out

    def prefill_pass(self, arrival, prompt, routing: RoutingConfig, window_ms: int, w0: int,
                     n_windows: int, mode: int = L.FIXED_WINDOW, fixed_window_ms: float = 0.0,
                     qopt: QueueOptimizerConfig = QueueOptimizerConfig(),
                     slo: SloConfig = SloConfig(), allowance_ms: float = 100.0,
                     rr: Optional[RouteResult] = None, sel: Optional["SelectResult"] = None,
                     summary_out: Optional[torch.Tensor] = None):
        """route_bin + prefill_select (+ the per-class summary) as ONE fused pass
        (gsb_prefill_pass: K1b and K2 in one persistent kernel). Returns (RouteResult,
        SelectResult), identical to the two-call path's."""
        arrival = self._dev(arrival, torch.int64)
        prompt = self._dev(prompt, torch.int32)
        n = arrival.numel()
        Cn = routing.n_classes() if routing.enabled else 1
        cells = n_windows * Cn
        P = len(self.profiles)
        dl = mode == L.DEADLINE_SLACK
        if rr is None:
            rr = RouteResult(Cn, n_windows, window_ms, w0, self._empty(n_windows + 1, torch.int64),
                             self._empty(n, torch.uint8), self._empty(cells, torch.int32),
                             self._empty((P, cells), torch.float64),
                             self._empty(cells, torch.float64) if dl else None)
            rr.nonempty = self._empty(cells, torch.int32)
            rr.n_nonempty = self._empty(1, torch.int64)
            rr.t_ref_list = self._empty((P, cells), torch.float64)
            if dl:
                rr.min_deadline_list = self._empty(cells, torch.float64)
        if sel is None:
            sel = SelectResult(self._empty((P, cells), torch.int16),
                               self._empty((P, cells), torch.float64),
                               self._empty(cells, torch.float64))
        rcfg = _route_cfg(routing, window_ms, w0, n_windows, slo, allowance_ms)
        scfg = L.CSelectCfg(mode, Cn, fixed_window_ms, w0, window_ms, qopt.to_c())
        cl = rr.cell_list()
        self._check(self.lib.gsb_prefill_pass(
            self.ctx, C.byref(rcfg), n, _ptr(arrival), _ptr(prompt), _ptr(rr.bounds), _ptr(rr.cls),
            _ptr(rr.count), _ptr(rr.t_ref), _ptr(rr.min_deadline), C.byref(cl), C.byref(scfg),
            _ptr(sel.window_ms), _ptr(sel.f_idx), _ptr(sel.energy_j), _ptr(summary_out),
            self.stream()))
        rr.profile_gen = self.profile_gen
        return rr, sel

    def prefill_pass_host(self, arrival: torch.Tensor, prompt: torch.Tensor,
                          routing: RoutingConfig, window_ms: int, w0: int, n_windows: int,
                          mode: int = L.FIXED_WINDOW, fixed_window_ms: float = 0.0,
                          qopt: QueueOptimizerConfig = QueueOptimizerConfig(),
                          slo: SloConfig = SloConfig(), allowance_ms: float = 100.0,
                          chunks: int = 4, out: Optional["HostPassResult"] = None,
                          want_summary: bool = True) -> "HostPassResult":
        """The whole pass from PINNED host arrays to host arrays (gsb_prefill_pass_host): the
        windows split into `chunks` ranges whose prompt upload, kernels and read-back overlap
        each other's (PCIe is full duplex). f_idx / energy equal prefill_pass's bit for bit;
        the per-chunk summaries combine like ranks (HostPassResult.summary()). Stream-ordered:
        synchronize the engine's stream before reading the result."""
        if not (_pinned(arrival, torch.int64) and _pinned(prompt, torch.int32)):
            raise ValueError("prefill_pass_host: arrival (int64) and prompt (int32) must be "
                             "contiguous pinned host tensors")
        Cn = routing.n_classes() if routing.enabled else 1
        cells = n_windows * Cn
        P = len(self.profiles)
        chunks = max(1, min(int(chunks), 64, int(n_windows)))
        if out is None:
            # every host output pinned: a read-back into pageable memory would block the host
            # until its chunk is done, serializing the pipeline
            summ = None
            if want_summary:
                summ = torch.zeros((chunks, P * Cn * self.SUMMARY_DTYPE.itemsize),
                                   dtype=torch.uint8).pin_memory()
            out = HostPassResult(torch.empty((P, cells), dtype=torch.int16).pin_memory(),
                                 torch.empty((P, cells), dtype=torch.float64).pin_memory(),
                                 summ, chunks, n_windows, Cn)
        rcfg = _route_cfg(routing, window_ms, w0, n_windows, slo, allowance_ms)
        scfg = L.CSelectCfg(mode, Cn, fixed_window_ms, w0, window_ms, qopt.to_c())
        self._check(self.lib.gsb_prefill_pass_host(
            self.ctx, C.byref(rcfg), arrival.numel(), _ptr(arrival), _ptr(prompt), C.byref(scfg),
            out.chunks, _ptr(out.f_idx), _ptr(out.energy_j),
            _ptr(out.chunk_summaries) if out.chunk_summaries is not None else None,
            self.stream()))
        return out

    def mg1_side_output(self, rr: RouteResult, sel: "SelectResult", prompt):
        """M/G/1 side output beside the decisions (gsb_mg1_side_output): dict of [P, cells]
        device tensors rho, wq_ms, energy_per_request_j. PARITY-UNPINNED (the reference has no
        M/G/1 term); never an input of the bit-exact argmin."""
        prompt = self._dev(prompt, torch.int32)
        P, cells = sel.f_idx.shape
        out = {k: self._empty((P, cells), torch.float64)
               for k in ("wq_ms", "rho", "energy_per_request_j")}
        self._check(self.lib.gsb_mg1_side_output(
            self.ctx, rr.n_classes, rr.n_windows, float(rr.window_ms), _ptr(prompt), _ptr(rr.cls),
            _ptr(rr.bounds), _ptr(sel.f_idx), _ptr(sel.energy_j), _ptr(out["wq_ms"]),
            _ptr(out["rho"]), _ptr(out["energy_per_request_j"]), self.stream()))
        return out

    # ---------------------------------------------------------------- simulator wire formats
    def _render(self, fn, n, arrays) -> bytes:
        nb = C.c_int64(0)
        self._check(fn(self.ctx, n, *[_ptr(a) for a in arrays], None, 0, C.byref(nb),
                       self.stream()))
        buf = self._empty(max(int(nb.value), 1), torch.uint8)
        self._check(fn(self.ctx, n, *[_ptr(a) for a in arrays], _ptr(buf), int(nb.value),
                       C.byref(nb), self.stream()))
        return bytes(buf[:int(nb.value)].cpu().numpy().tobytes())

    def freq_timeline_csv(self, applied_ms, prefill_pool, worker, f_mhz) -> bytes:
        """freq_timeline_csv (simkernel.cpp:686-697) of FreqChangeRecords given as arrays
        (host or device), rendered on the GPU: '%.10g' numbers, byte-identical."""
        a = [self._dev(applied_ms, torch.float64), self._dev(prefill_pool, torch.uint8),
             self._dev(worker, torch.int32), self._dev(f_mhz, torch.float64)]
        return self._render(self.lib.gsb_freq_timeline_csv, a[0].numel(), a)

    def prefill_commands_csv(self, tick_ms, class_id, worker, f_mhz, window_ms,
                             infeasible) -> bytes:
        """prefill_commands_csv (simkernel.cpp:699-714) of PrefillCommandRecords, on the GPU."""
        a = [self._dev(tick_ms, torch.float64), self._dev(class_id, torch.int32),
             self._dev(worker, torch.int32), self._dev(f_mhz, torch.float64),
             self._dev(window_ms, torch.float64), self._dev(infeasible, torch.uint8)]
        return self._render(self.lib.gsb_prefill_commands_csv, a[0].numel(), a)

    def decision_log_csv(self, records) -> bytes:
        """decision_log_csv (decode_ctl.cpp:231-247) of decision records in the gsb_decision
        layout (DECISION_DTYPE, host or device; e.g. a K3b / K5 records slice), rendered on the
        GPU: '%.6g' numbers, byte-identical."""
        if isinstance(records, torch.Tensor):
            r = records.to(self.device).contiguous().view(torch.uint8).reshape(-1)
        else:
            raw = np.ascontiguousarray(records).view(np.uint8).reshape(-1)
            r = torch.from_numpy(raw.copy()).to(self.device)
        return self._render(self.lib.gsb_decision_log_csv, r.numel() // 64, [r])

    def format_g10(self, values) -> list:
        """snprintf("%.10g") of every value, on the GPU (the reference's fmt_g)."""
        return self.format_g(values, 10)

    def format_g(self, values, precision: int = 10) -> list:
        """snprintf("%.<precision>g") (6 or 10) of every value, on the GPU."""
        v = self._dev(values, torch.float64)
        n = v.numel()
        out = self._empty((max(n, 1), 32), torch.uint8)
        ln = self._empty(max(n, 1), torch.int32)
        self._check(self.lib.gsb_format_g(self.ctx, int(precision), n, _ptr(v), _ptr(out),
                                          _ptr(ln), self.stream()))
        o, l = out.cpu().numpy(), ln.cpu().numpy()
        return [bytes(o[i, :l[i]]).decode() for i in range(n)]

    # ---------------------------------------------------------------- K6: trace CSV
    def parse_trace(self, data, class_threshold: int = 1024, name: str = "trace") -> "TraceArrays":
        """greensim::load_trace (trace.cpp:56-129) of a CSV image (bytes, a uint8 numpy array
        or a uint8 tensor, host or device) on the GPU. Raises TraceError(kind, row) with the
        reference's message."""
        if isinstance(data, (bytes, bytearray, memoryview)):
            host = torch.frombuffer(bytearray(data), dtype=torch.uint8) if len(data) else \
                torch.empty(0, dtype=torch.uint8)
            dev = host.pin_memory().to(self.device, non_blocking=True) if host.numel() else \
                self._empty(0, torch.uint8)
        else:
            dev = self._dev(data, torch.uint8)
        n = int(dev.numel())
        # a valid row holds >= 6 bytes ("0,1,1\n"); a malformed file may need more rows: the
        # call then reports the count and is repeated with room for it
        cap = max(1, n // 6 + 1)
        for _ in range(2):
            arr = self._empty(cap, torch.int64)
            prm = self._empty(cap, torch.int32)
            out = self._empty(cap, torch.int32)
            cls = self._empty(cap, torch.uint8)
            res = L.CTraceResult()
            rc = self.lib.gsb_trace_parse(self.ctx, _ptr(dev) if n else None, n,
                                          int(class_threshold), cap, _ptr(arr), _ptr(prm),
                                          _ptr(out), _ptr(cls), C.byref(res), self.stream())
            if rc == L.INVALID_ARGUMENT and res.n_rows > cap:
                cap = int(res.n_rows)
                continue
            break
        if rc == L.TRACE_ERROR:
            raise TraceError(self.lib.gsb_last_error(self.ctx).decode(errors="replace"),
                             L.TRACE_KINDS[res.kind], res.row if res.row > 0 else None)
        self._check(rc)
        k = int(res.n_rows)
        dur = max(0, int(res.max_arrival_ms))  # finalize_meta (trace.cpp:36-45)
        return TraceArrays(arr[:k], prm[:k], out[:k], cls[:k], bool(res.has_class), name, dur,
                           1000.0 * k / dur if dur > 0 else 0.0)

    def load_trace(self, path, class_threshold: int = 1024) -> "TraceArrays":
        """load_trace(path, class_threshold): file bytes -> GPU parse (meta.name = the stem)."""
        try:
            with open(path, "rb") as f:
                data = f.read()
        except OSError:
            raise TraceError(f"cannot open trace file: {path}", "MalformedRow") from None
        return self.parse_trace(data, class_threshold, os.path.splitext(os.path.basename(path))[0])

    def format_trace(self, arrival, prompt, output, slo_class=None) -> bytes:
        """save_trace_csv's text (trace.cpp:131-145) rendered on the GPU; the class column is
        written iff slo_class is given (every request carries a class)."""
        a = self._dev(arrival, torch.int64)
        p = self._dev(prompt, torch.int32)
        o = self._dev(output, torch.int32)
        c = None if slo_class is None else self._dev(slo_class, torch.uint8)
        n = int(a.numel())
        nb = C.c_int64(0)
        self._check(self.lib.gsb_trace_format(self.ctx, n, _ptr(a), _ptr(p), _ptr(o), _ptr(c),
                                              None, 0, C.byref(nb), self.stream()))
        buf = self._empty(int(nb.value), torch.uint8)
        self._check(self.lib.gsb_trace_format(self.ctx, n, _ptr(a), _ptr(p), _ptr(o), _ptr(c),
                                              _ptr(buf), int(nb.value), C.byref(nb), self.stream()))
        return bytes(buf.cpu().numpy().tobytes())

    def save_trace_csv(self, tr: "TraceArrays", path) -> None:
        with open(path, "wb") as f:
            f.write(self.format_trace(tr.arrival_ms, tr.prompt_tokens, tr.output_tokens,
                                      tr.slo_class))

    # ---------------------------------------------------------------- K2
    def prefill_select(self, rr: RouteResult, mode: int = L.FIXED_WINDOW,
                       fixed_window_ms: float = 0.0,
                       qopt: QueueOptimizerConfig = QueueOptimizerConfig(),
                       window: Optional[torch.Tensor] = None,
                       out: Optional[SelectResult] = None,
                       summary_out: Optional[torch.Tensor] = None) -> SelectResult:
        """K2: energy_total at every (cell, profile, clock) + deterministic argmin. With
        summary_out (a [P*C, 48] byte tensor, see prefill_summary_dev) the per-(profile,
        class) summary is folded into the same launch (gsb_prefill_select_summary)."""
        self._check_gen(rr)
        cfg = L.CSelectCfg(mode, rr.n_classes, fixed_window_ms, rr.w0, rr.window_ms, qopt.to_c())
        P, cells = len(self.profiles), rr.n_cells
        if out is None:
            out = SelectResult(self._empty((P, cells), torch.int16),
                               self._empty((P, cells), torch.float64),
                               window if window is not None else self._empty(cells, torch.float64))
        if summary_out is not None or rr.nonempty is not None:
            cl = rr.cell_list()
            self._check(self.lib.gsb_prefill_select_list(
                self.ctx, C.byref(cfg), cells, _ptr(rr.t_ref), _ptr(rr.count),
                C.byref(cl) if cl is not None else None, _ptr(rr.min_deadline),
                _ptr(out.window_ms), _ptr(out.f_idx), _ptr(out.energy_j), _ptr(summary_out),
                self.stream()))
            return out
        self._check(self.lib.gsb_prefill_select(self.ctx, C.byref(cfg), cells, _ptr(rr.t_ref),
                                                _ptr(rr.count), _ptr(rr.min_deadline),
                                                _ptr(out.window_ms), _ptr(out.f_idx),
                                                _ptr(out.energy_j), self.stream()))
        return out

    def summary_buffer(self, n_classes: int) -> torch.Tensor:
        """Device bytes for P*C gsb_class_summary records (prefill_select(summary_out=...))."""
        return self._empty((len(self.profiles) * n_classes, C.sizeof(L.CClassSummary)),
                           torch.uint8)

    SUMMARY_DTYPE = np.dtype([("n_cmd", "<i8"), ("n_infeasible", "<i8"), ("n_empty", "<i8"),
                              ("sum_energy_j", "<f8"), ("min_energy_j", "<f8"),
                              ("argmin_cell", "<i8")])

    def prefill_summary_dev(self, sel: SelectResult, n_classes: int,
                            out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Per (profile, class) summary into a device byte tensor [P*C, 48] (no host sync)."""
        P, cells = sel.f_idx.shape
        if out is None:
            out = self._empty((P * n_classes, C.sizeof(L.CClassSummary)), torch.uint8)
        self._check(self.lib.gsb_prefill_summary(self.ctx, P, n_classes, cells, _ptr(sel.f_idx),
                                                 _ptr(sel.energy_j), _ptr(out), self.stream()))
        return out

    def prefill_summary(self, sel: SelectResult, n_classes: int) -> np.ndarray:
        P = sel.f_idx.shape[0]
        host = self.prefill_summary_dev(sel, n_classes).cpu().numpy()
        return host.view(self.SUMMARY_DTYPE).reshape(P, n_classes)

    # ---------------------------------------------------------------- ragged batches
    def select_batches(self, off, prompt, windows=None, profile: Optional[GpuProfile] = None,
                       wf=None, mode: int = L.PER_CELL_WINDOW, fixed_window_ms: float = 0.0,
                       deadline=None, now=None,
                       qopt: QueueOptimizerConfig = QueueOptimizerConfig(), running=None):
        """select_frequency / queue_optimizer_tick over CSR batches. Returns device tensors
        (f_idx i16, energy f64, window f64, t_ref f64). running: optional dict of per-job
        arrays (running u8, remaining_ref_ms, updated_ms, freq_mhz, t_ref_ms): the running jobs'
        work_fraction is then computed on the device (simkernel.cpp:476-479; needs now)."""
        pi = 0 if profile is None else self._profile_index(profile)
        off = self._dev(off, torch.int64)
        nb = off.numel() - 1
        prompt = self._dev(prompt, torch.int32)
        wf_t = None if wf is None else self._dev(wf, torch.float64)
        dl = None if deadline is None else self._dev(deadline, torch.float64)
        nw = None if now is None else self._dev(now, torch.float64)
        win = self._dev(windows, torch.float64) if windows is not None else self._empty(nb, torch.float64)
        f_idx = self._empty(nb, torch.int16)
        energy = self._empty(nb, torch.float64)
        t_ref = self._empty(nb, torch.float64)
        cfg = L.CSelectCfg(mode, 1, fixed_window_ms, 0, 1, qopt.to_c())
        rj, keep = None, None
        if running is not None:
            keep = [self._dev(running["running"], torch.uint8)] + [
                self._dev(running[k], torch.float64)
                for k in ("remaining_ref_ms", "updated_ms", "freq_mhz", "t_ref_ms")]
            rj = L.CRunningJobs(*[_ptr(t) for t in keep])
        self._check(self.lib.gsb_select_batches_running(
            self.ctx, C.byref(cfg), pi, nb, _ptr(off), _ptr(prompt), _ptr(wf_t),
            C.byref(rj) if rj is not None else None, _ptr(dl), _ptr(nw), _ptr(win), _ptr(f_idx),
            _ptr(energy), _ptr(t_ref), self.stream()))
        return f_idx, energy, win, t_ref

    def energy_batches(self, off, prompt, f_mhz, windows, profile: Optional[GpuProfile] = None,
                       wf=None):
        pi = 0 if profile is None else self._profile_index(profile)
        off = self._dev(off, torch.int64)
        nb = off.numel() - 1
        prompt = self._dev(prompt, torch.int32)
        wf_t = None if wf is None else self._dev(wf, torch.float64)
        f = self._dev(f_mhz, torch.float64)
        w = self._dev(windows, torch.float64)
        outs = [self._empty(nb, torch.float64) for _ in range(4)]
        feas = self._empty(nb, torch.uint8)
        self._check(self.lib.gsb_energy_batches(self.ctx, pi, nb, _ptr(off), _ptr(prompt),
                                                _ptr(wf_t), _ptr(f), _ptr(w), *[_ptr(o) for o in outs],
                                                _ptr(feas), self.stream()))
        return (*outs, feas)

    # ---------------------------------------------------------------- reference-named calls
    @staticmethod
    def _batch_arrays(batch: PrefillBatch):
        p = np.array([j.prompt_tokens for j in batch.jobs], np.int32)
        wf = np.array([j.work_fraction for j in batch.jobs], np.float64)
        dl = np.array([j.deadline_ms for j in batch.jobs], np.float64)
        return p, wf, dl

    def select_frequency(self, batch: PrefillBatch, window_ms: float,
                         profile: GpuProfile) -> Optional[FrequencyChoice]:
        """select_frequency (prefill_opt.cpp:45-56) on the GPU."""
        if not batch.jobs:
            raise ModelError("busy_time: empty batch")
        p, wf, _ = self._batch_arrays(batch)
        f_idx, e, _, _ = self.select_batches([0, len(p)], p, [window_ms], profile, wf)
        i = int(f_idx[0].item())
        if i < 0:
            return None
        return FrequencyChoice(profile.grid.at(i), float(e[0].item()))

    def energy_total(self, batch: PrefillBatch, f: float, window_ms: float,
                     profile: GpuProfile) -> EnergyBreakdown:
        """energy_total (prefill_opt.cpp:22-31) on the GPU; ModelError as the reference."""
        if not batch.jobs:
            raise ModelError("busy_time: empty batch")
        if not profile.grid.on_grid(f):
            raise ModelError("busy_time: frequency off grid")
        p, wf, _ = self._batch_arrays(batch)
        busy, a, i, t, feas = self.energy_batches([0, len(p)], p, [f], [window_ms], profile, wf)
        if int(feas[0].item()) >= 2:
            raise ModelError("busy_time: frequency off grid")
        return EnergyBreakdown(float(a[0].item()), float(i[0].item()), float(t[0].item()),
                               bool(feas[0].item()))

    def busy_time_ms(self, batch: PrefillBatch, f: float, profile: GpuProfile) -> float:
        """busy_time_ms (prefill_opt.cpp:16-20)."""
        if not batch.jobs:
            raise ModelError("busy_time: empty batch")
        if not profile.grid.on_grid(f):
            raise ModelError("busy_time: frequency off grid")
        p, wf, _ = self._batch_arrays(batch)
        busy, *_ = self.energy_batches([0, len(p)], p, [f], [math.inf], profile, wf)
        return float(busy[0].item())

    def t_ref_total_ms(self, batch: PrefillBatch, profile: GpuProfile) -> float:
        p, wf, _ = self._batch_arrays(batch)
        *_, t = self.select_batches([0, len(p)], p, [0.0], profile, wf)
        return float(t[0].item())

    def queue_optimizer_tick(self, queues: Sequence[ClassQueueSnapshot], now_ms: float,
                             cfg: QueueOptimizerConfig, profile: GpuProfile) -> list:
        """queue_optimizer_tick (prefill_opt.cpp:58-82): one GPU batch per non-empty queue."""
        live = [q for q in queues if q.batch.jobs]
        if not live:
            return []
        off = np.zeros(len(live) + 1, np.int64)
        ps, wfs, dls = [], [], []
        for i, q in enumerate(live):
            p, wf, dl = self._batch_arrays(q.batch)
            ps.append(p), wfs.append(wf), dls.append(dl)
            off[i + 1] = off[i] + len(p)
        f_idx, _, win, _ = self.select_batches(
            off, np.concatenate(ps), None, profile, np.concatenate(wfs), L.DEADLINE_SLACK, 0.0,
            np.concatenate(dls), np.full(len(live), now_ms), cfg)
        f_idx = f_idx.cpu().numpy()
        win = win.cpu().numpy()
        out = []
        for i, q in enumerate(live):
            fi = int(f_idx[i])
            out.append(PrefillFreqCommand(q.class_id,
                                          profile.grid.at(fi) if fi >= 0 else profile.grid.f_max_mhz,
                                          float(win[i]), fi < 0))
        return out

    def classify_many(self, routing: RoutingConfig, prompts) -> np.ndarray:
        """classify (router.cpp:26-31) for a vector of prompts, on the GPU (gsb_classify)."""
        thr = np.ascontiguousarray(routing.thresholds, np.int32)
        if len(thr) > L.GSB_MAX_CLASSES - 1:
            raise RouterError("routing: more than 7 thresholds (GSB_MAX_CLASSES)")
        p = self._dev(np.ascontiguousarray(prompts, np.int32), torch.int32)
        out = self._empty(p.numel(), torch.int32)
        self._check(self.lib.gsb_classify(self.ctx, len(thr), thr.ctypes.data_as(C.c_void_p),
                                          p.numel(), _ptr(p), _ptr(out), self.stream()))
        return out.cpu().numpy().astype(np.int64)

    def t_ref_batches(self, lat: LatencyModel, off, prompt, wf=None) -> torch.Tensor:
        """PrefillBatch::t_ref_total_ms(m) (prefill_opt.cpp:9-14) per CSR batch, under a bare
        LatencyModel (gsb_t_ref_batches)."""
        off = self._dev(off, torch.int64)
        prompt = self._dev(prompt, torch.int32)
        wf_t = None if wf is None else self._dev(wf, torch.float64)
        out = self._empty(off.numel() - 1, torch.float64)
        abc = (C.c_double * 3)(lat.a, lat.b, lat.c)
        self._check(self.lib.gsb_t_ref_batches(self.ctx, abc, off.numel() - 1, _ptr(off),
                                               _ptr(prompt), _ptr(wf_t), _ptr(out), self.stream()))
        return out

    def energy_closed_form_batches(self, off, prompt, f_mhz, windows,
                                   profile: Optional[GpuProfile] = None, wf=None) -> torch.Tensor:
        """energy_total_closed_form_j (prefill_opt.cpp:33-43) per CSR batch; NaN off-grid."""
        pi = 0 if profile is None else self._profile_index(profile)
        ins = [self._dev(off, torch.int64), self._dev(prompt, torch.int32),
               None if wf is None else self._dev(wf, torch.float64),
               self._dev(f_mhz, torch.float64), self._dev(windows, torch.float64)]
        nb = ins[0].numel() - 1
        out = self._empty(nb, torch.float64)
        self._check(self.lib.gsb_energy_closed_form_batches(self.ctx, pi, nb, *[_ptr(x) for x in ins],
                                                            _ptr(out), self.stream()))
        return out

    # ---------------------------------------------------------------- window statistics
    def quantile_batch(self, off, samples, q: float) -> torch.Tensor:
        """Nearest-rank quantile (metrics.cpp:11-19) of every CSR sample set (any size)."""
        off = self._dev(off, torch.int64)
        s = self._dev(samples, torch.float64)
        out = self._empty(off.numel() - 1, torch.float64)
        self._check(self.lib.gsb_quantile_batch(self.ctx, q, off.numel() - 1, _ptr(off), _ptr(s),
                                                _ptr(out), self.stream()))
        return out

    def tps_window_batch(self, off, t_ms, tokens, window_ms, now_ms) -> torch.Tensor:
        """TpsWindow::tps(now) (decode_ctl.cpp:113-118) for every CSR event window."""
        ins = [self._dev(off, torch.int64), self._dev(t_ms, torch.float64),
               self._dev(tokens, torch.int32), self._dev(window_ms, torch.float64),
               self._dev(now_ms, torch.float64)]
        n = ins[0].numel() - 1
        out = self._empty(n, torch.float64)
        self._check(self.lib.gsb_tps_window_batch(self.ctx, n, *[_ptr(x) for x in ins], _ptr(out),
                                                  self.stream()))
        return out

    def steady_state_batch(self, profile: GpuProfile, tps, f, max_batch):
        """decode_steady_state (decode_ctl.cpp:28-50) at many points: (sustainable u8, batch,
        tbt_ms) device tensors."""
        dp = self._dev(np.frombuffer(bytes(profile.to_c()), np.uint8), torch.uint8)
        ins = [self._dev(tps, torch.float64), self._dev(f, torch.float64),
               self._dev(max_batch, torch.int32)]
        n = ins[0].numel()
        sus, b, t = self._empty(n, torch.uint8), self._empty(n, torch.float64), self._empty(n, torch.float64)
        self._check(self.lib.gsb_steady_state_batch(self.ctx, n, _ptr(dp), *[_ptr(x) for x in ins],
                                                    _ptr(sus), _ptr(b), _ptr(t), self.stream()))
        return sus, b, t

    def decode_script(self, cfgs, table_of, worker, tps_hi, f_opt, grid: FrequencyGrid, ev_off,
                      kind, t_ms, value, has, state: Optional[torch.Tensor] = None,
                      rec_cap: int = 0):
        """K3s: DecodeController driven by explicit call scripts (decode_ctl.hpp:116-150), one
        lane per controller; `state` (uint8 [N, sizeof gsb_ctl_state], zero = fresh) resumes
        and receives each controller's state. Returns dict of device tensors."""
        cfg_arr = cfgs if isinstance(cfgs, np.ndarray) else ctl_cfg_array(cfgs)
        N = len(cfg_arr)
        tps_hi_h = np.ascontiguousarray(tps_hi.cpu().numpy() if isinstance(tps_hi, torch.Tensor)
                                        else tps_hi, np.float64)
        NB = tps_hi_h.reshape(-1, tps_hi_h.shape[-1]).shape[1]
        keep = [self._dev(cfg_arr.view(np.uint8), torch.uint8), self._dev(table_of, torch.int32),
                self._dev(worker, torch.int32), self._dev(tps_hi_h, torch.float64),
                self._dev(f_opt, torch.float64), self._dev(ev_off, torch.int64),
                self._dev(kind, torch.int8), self._dev(t_ms, torch.float64),
                self._dev(value, torch.float64), self._dev(has, torch.uint8)]
        out = {"digest": self._empty(N, torch.int64), "n_rec": self._empty(N, torch.int64),
               "records": (self._empty((N, rec_cap, DECISION_DTYPE.itemsize), torch.uint8)
                           if rec_cap else None),
               "state": state if state is not None else torch.zeros(
                   (N, C.sizeof(L.CCtlState)), dtype=torch.uint8, device=self.device)}
        a = L.CReplayArgs(N, _ptr(keep[0]), _ptr(keep[1]), None, _ptr(keep[2]), NB, _ptr(keep[3]),
                          _ptr(keep[4]), grid.f_min_mhz, grid.f_max_mhz, 0.0, 0.0, 0.0, None, None,
                          None, _ptr(out["digest"]), _ptr(out["n_rec"]), None, None,
                          _ptr(out["records"]), rec_cap)
        self._check(self.lib.gsb_decode_script(self.ctx, C.byref(a), *[_ptr(x) for x in keep[5:]],
                                               _ptr(out["state"]), self.stream()))
        torch.cuda.current_stream(self.device).synchronize()
        return out

    def classify(self, routing: RoutingConfig, prompt_tokens: int) -> int:
        return int(self.classify_many(routing, [prompt_tokens])[0])

    # ---------------------------------------------------------------- decode (K3/K4)
    def telemetry_to_device(self, tel: Telemetry):
        d = [self._dev(tel.ev_off, torch.int64), self._dev(tel.t_ms, torch.float64),
             self._dev(tel.tokens, torch.int32), self._dev(tel.gap_off, torch.int64),
             self._dev(tel.gaps, torch.float64)]
        c = L.CTelemetry(tel.n_streams, *[_ptr(x) for x in d])
        return c, d

    def window_series(self, tel: Telemetry, capacity: int, fine_ms: float, coarse_ms: float,
                      t_end_ms: float, dev=None, out=None):
        """K3a: P95 per fine tick, TPS per coarse tick, per stream (device tensors)."""
        c, keep = dev if dev is not None else self.telemetry_to_device(tel)
        nf = self.lib.gsb_n_ticks(fine_ms, t_end_ms)
        nc = self.lib.gsb_n_ticks(coarse_ms, t_end_ms)
        S = tel.n_streams
        if out is not None:
            has, p95, tps = out
        else:
            has = self._empty((S, nf), torch.uint8)
            p95 = self._empty((S, nf), torch.float64)
            tps = self._empty((S, nc), torch.float64)
        self._check(self.lib.gsb_window_series(self.ctx, C.byref(c), capacity, fine_ms, coarse_ms,
                                               t_end_ms, _ptr(has), _ptr(p95), _ptr(tps),
                                               self.stream()))
        return has, p95, tps

    def build_band_tables(self, profiles: Sequence[GpuProfile], profile_of, t_slo_ms, workers,
                          max_batch, levels):
        """K4: build_band_table (decode_ctl.cpp:76-111) for many tuples; raises ModelError
        on invalid levels like the reference."""
        lv = np.ascontiguousarray(levels, np.float64)
        if len(lv) == 0:
            raise ModelError("band table: need at least one TPS level")
        if np.any(lv[:-1] >= lv[1:]):
            raise ModelError("band table: levels must be ascending")
        wk = np.ascontiguousarray(workers, np.int32)
        mb = np.ascontiguousarray(max_batch, np.int32)
        if np.any(wk < 1) or np.any(mb < 1):
            raise ModelError("band table: bad pool shape")
        T = len(profile_of)
        parr = np.frombuffer(b"".join(bytes(p.to_c()) for p in profiles), np.uint8)
        dp = self._dev(parr, torch.uint8)
        outs = [self._empty((T, len(lv)), torch.float64) for _ in range(3)]
        feas = self._empty((T, len(lv)), torch.uint8)
        # inputs must stay referenced until the launch is enqueued: a freed temporary's
        # block can be handed to the next _dev() copy before the kernel reads it
        ins = [self._dev(profile_of, torch.int32), self._dev(t_slo_ms, torch.float64),
               self._dev(wk, torch.int32), self._dev(mb, torch.int32),
               self._dev(lv, torch.float64)]
        self._check(self.lib.gsb_build_band_tables(
            self.ctx, T, _ptr(dp), _ptr(ins[0]), _ptr(ins[1]), _ptr(ins[2]), _ptr(ins[3]),
            len(lv), _ptr(ins[4]), *[_ptr(o) for o in outs], _ptr(feas), self.stream()))
        torch.cuda.current_stream(self.device).synchronize()
        return (*outs, feas)

    def build_band_table(self, profile: GpuProfile, tps_levels, t_slo_ms: float,
                         decode_workers: int, max_batch: int = 64) -> FreqBandTable:
        lo, hi, fo, fe = self.build_band_tables([profile], [0], [t_slo_ms], [decode_workers],
                                                [max_batch], tps_levels)
        lo, hi, fo, fe = (x.cpu().numpy()[0] for x in (lo, hi, fo, fe))
        return FreqBandTable([BandBucket(float(a), float(b), float(c), bool(d))
                              for a, b, c, d in zip(lo, hi, fo, fe)])

    def decode_replay(self, cfgs: Sequence[DecodeCtlConfig] | np.ndarray, table_of, stream_of,
                      worker, tps_lo, tps_hi, f_opt, grid: FrequencyGrid, fine_has, fine_p95,
                      coarse_tps, t_end_ms: float, rec_cap: int = 0, want_counts: bool = True,
                      validate: bool = True):
        """K3b: DecodeController replay, one lane per trajectory. Returns dict of device
        tensors: digest (i64 bits of u64), n_rec, counts [N,8], mean_cmd, records."""
        cfg_arr = cfgs if isinstance(cfgs, np.ndarray) else ctl_cfg_array(cfgs)
        N = len(cfg_arr)
        tps_lo_h = np.ascontiguousarray(tps_lo.cpu().numpy() if isinstance(tps_lo, torch.Tensor)
                                        else tps_lo, np.float64)
        tps_hi_h = np.ascontiguousarray(tps_hi.cpu().numpy() if isinstance(tps_hi, torch.Tensor)
                                        else tps_hi, np.float64)
        T, NB = tps_hi_h.reshape(-1, tps_hi_h.shape[-1]).shape
        fine_ms = float(cfg_arr["fine_period_ms"][0])
        coarse_ms = float(cfg_arr["coarse_period_ms"][0])
        if validate:
            msg = C.create_string_buffer(256)
            rc = self.lib.gsb_replay_validate(cfg_arr.ctypes.data_as(C.c_void_p), N, NB,
                                              tps_lo_h.ctypes.data_as(C.c_void_p),
                                              tps_hi_h.ctypes.data_as(C.c_void_p), T, msg, 256)
            if rc != L.OK:
                raise ModelError(msg.value.decode())
            if np.any(cfg_arr["fine_period_ms"] != fine_ms) or np.any(
                    cfg_arr["coarse_period_ms"] != coarse_ms):
                raise ValueError("decode_replay: all trajectories must share the series periods")
        dcfg = self._dev(cfg_arr.view(np.uint8), torch.uint8)
        keep = [dcfg, self._dev(table_of, torch.int32), self._dev(stream_of, torch.int32),
                self._dev(worker, torch.int32), self._dev(tps_hi_h, torch.float64),
                self._dev(f_opt, torch.float64)]
        out = {"digest": self._empty(N, torch.int64), "n_rec": self._empty(N, torch.int64),
               "counts": self._empty((N, 8), torch.int32) if want_counts else None,
               "mean_cmd": self._empty(N, torch.float64),
               "records": (self._empty((N, rec_cap, DECISION_DTYPE.itemsize), torch.uint8)
                           if rec_cap else None)}
        a = L.CReplayArgs(N, *[_ptr(x) for x in keep[:4]], NB, _ptr(keep[4]), _ptr(keep[5]),
                          grid.f_min_mhz, grid.f_max_mhz, fine_ms, coarse_ms, t_end_ms,
                          _ptr(fine_has), _ptr(fine_p95), _ptr(coarse_tps), _ptr(out["digest"]),
                          _ptr(out["n_rec"]), _ptr(out["counts"]), _ptr(out["mean_cmd"]),
                          _ptr(out["records"]), rec_cap)
        out["_keep"] = keep
        out["_args"] = a
        self.run_replay(out)
        return out

    def run_replay(self, plan: dict) -> None:
        """Re-launch a prepared replay (all inputs/outputs already on the device): the
        timed / graph-captured decode step is this single K3b launch."""
        self._check(self.lib.gsb_decode_replay(self.ctx, C.byref(plan["_args"]), self.stream()))

    # ---------------------------------------------------------------- K5: decode pool
    def decode_pool(self, cfgs, stream: DecodeStream, profile: GpuProfile,
                    sim: SimConfig = SimConfig(), slo: SloConfig = SloConfig(),
                    fixed_mhz=None, details: bool = False, rec_cap: int = 0,
                    freq_cap: int = 0, launch: bool = True) -> dict:
        """K5: the closed-loop decode pool (simkernel.cpp:330-464) for N scenarios, one warp
        each, all on one enqueue stream. cfgs: N DecodeCtlConfigs (or a CTL_DTYPE array);
        fixed_mhz: optional [N] pinned clocks (> 0: FixedFreq-like, no controller). Band
        tables are built on the GPU (K4) per distinct t_slo*margin (simkernel.cpp:200-205).
        Returns a plan dict with device tensors; summary() reads it back."""
        cfg_arr = cfgs if isinstance(cfgs, np.ndarray) else ctl_cfg_array(cfgs)
        N = len(cfg_arr)
        fx = (np.zeros(N) if fixed_mhz is None
              else np.ascontiguousarray(np.broadcast_to(fixed_mhz, (N,)), np.float64))
        levels = sim.band_levels()
        t_eff = cfg_arr["tslo_ms"] * cfg_arr["margin_decode"]
        uniq, table_of = np.unique(t_eff, return_inverse=True)
        T, NB = len(uniq), len(levels)
        lo, hi, fo, _ = self.build_band_tables([profile], [0] * T, uniq,
                                               [sim.n_decode_workers] * T,
                                               [sim.max_batch] * T, levels)
        ctl = fx <= 0.0
        if ctl.any():
            msg = C.create_string_buffer(256)
            sub = np.ascontiguousarray(cfg_arr[ctl])
            rc = self.lib.gsb_replay_validate(sub.ctypes.data_as(C.c_void_p), len(sub), NB,
                                              np.ascontiguousarray(lo.cpu().numpy()).ctypes.data_as(C.c_void_p),
                                              np.ascontiguousarray(hi.cpu().numpy()).ctypes.data_as(C.c_void_p),
                                              T, msg, 256)
            if rc != L.OK:
                raise ModelError(msg.value.decode())
        if np.any(~ctl & ~np.array([profile.grid.on_grid(float(f)) for f in fx])):
            raise ModelError("decode pool: fixed frequency is off-grid")
        tps_cap = max(self.lib.gsb_decode_pool_tps_cap(C.byref(profile.to_c()), sim.max_batch,
                                                       float(c)) for c in np.unique(cfg_arr["coarse_period_ms"]))
        if tps_cap < 1:
            raise ModelError("decode pool: TPS window unbounded for this profile")
        min_fine = float(np.min(cfg_arr["fine_period_ms"][ctl])) if ctl.any() else 1.0
        if ctl.any() and sim.actuation_delay_ms / min_fine + 1 > 4:
            raise ModelError("decode pool: actuation delay above 3 fine periods is not supported")
        n_req = len(stream.output_tokens)
        pc = L.CPoolCfg(sim.n_decode_workers, sim.max_batch, sim.max_queue,
                              int(max(1, cfg_arr["tbt_window_tokens"].max())), int(tps_cap),
                              int(min(sim.max_queue, max(1, len(stream.t_ms)))),
                              sim.actuation_delay_ms, slo.tbt_p95_ms)
        keep = {
            "off": self._dev(np.array([0, len(stream.t_ms)], np.int64), torch.int64),
            "t": self._dev(np.ascontiguousarray(stream.t_ms, np.float64), torch.float64),
            "req": self._dev(np.ascontiguousarray(stream.req, np.int32), torch.int32),
            "floor": self._dev(np.array([stream.end_floor_ms], np.float64), torch.float64),
            "out": self._dev(np.ascontiguousarray(stream.output_tokens, np.int32), torch.int32),
            "arr": self._dev(np.ascontiguousarray(stream.arrival_ms, np.float64), torch.float64),
            "ttft": self._dev(np.ascontiguousarray(stream.ttft_slo_ms, np.float64), torch.float64),
            "cfg": self._dev(cfg_arr.view(np.uint8), torch.uint8),
            "fixed": self._dev(fx, torch.float64),
            "table_of": self._dev(table_of.astype(np.int32), torch.int32),
            "tps_hi": hi.contiguous(), "f_opt": fo.contiguous(),
        }
        st = L.CPoolStream(1, _ptr(keep["off"]), _ptr(keep["t"]), _ptr(keep["req"]),
                           _ptr(keep["floor"]), n_req, _ptr(keep["out"]), _ptr(keep["arr"]),
                           _ptr(keep["ttft"]))
        W = sim.n_decode_workers
        out = {"summary": self._empty(N * POOL_SUMMARY_DTYPE.itemsize, torch.uint8),
               "ledger": self._empty((N, W, 2), torch.float64) if details else None,
               "records": (self._empty((N, W, rec_cap, DECISION_DTYPE.itemsize), torch.uint8)
                           if rec_cap else None),
               "freq": self._empty((N, W, freq_cap, 2), torch.float64) if freq_cap else None,
               "req_worker": self._empty((N, n_req), torch.int32) if details else None,
               "req_first": self._empty((N, n_req), torch.float64) if details else None,
               "req_finish": self._empty((N, n_req), torch.float64) if details else None}
        if details:
            out["req_worker"].fill_(-1)
            out["req_first"].fill_(-1.0)
            out["req_finish"].fill_(-1.0)
        a = L.CPoolArgs(N, _ptr(keep["cfg"]), _ptr(keep["fixed"]), _ptr(keep["table_of"]), None,
                        NB, _ptr(keep["tps_hi"]), _ptr(keep["f_opt"]), _ptr(out["summary"]),
                        _ptr(out["ledger"]), _ptr(out["records"]), rec_cap, _ptr(out["freq"]),
                        freq_cap, _ptr(out["req_worker"]), _ptr(out["req_first"]),
                        _ptr(out["req_finish"]))
        plan = {"out": out, "_keep": keep, "_args": a, "_cfg": pc, "_stream": st,
                "_prof": profile.to_c(), "n": N, "W": W}
        if launch:
            self.run_pool(plan)
        return plan

    def run_pool(self, plan: dict) -> None:
        """(Re-)launch a prepared decode-pool plan: one K5 launch."""
        self._check(self.lib.gsb_decode_pool(self.ctx, C.byref(plan["_prof"]), C.byref(plan["_cfg"]),
                                             C.byref(plan["_stream"]), C.byref(plan["_args"]),
                                             self.stream()))

    @staticmethod
    def pool_summary(plan: dict) -> np.ndarray:
        """The [N] gsb_pool_summary records (POOL_SUMMARY_DTYPE); raises ModelError when a
        scenario exceeded a capacity (its outputs are invalid)."""
        sm = plan["out"]["summary"].cpu().numpy().view(POOL_SUMMARY_DTYPE)
        bad = np.nonzero(sm["status"])[0]
        if len(bad):
            raise ModelError(f"decode pool: capacity exceeded in {len(bad)} scenarios "
                             f"(status {int(sm['status'][bad[0]])})")
        return sm

    def selftest_division(self, per_divisor: int, seed: int = 12345) -> int:
        bad = self._empty(1, torch.int64)
        self._check(self.lib.gsb_selftest_division(self.ctx, per_divisor, seed, _ptr(bad),
                                                   self.stream()))
        return int(bad.item())

    def fp64_probe(self, n_threads: int, iters: int):
        sink = self._empty(1, torch.float64)
        self._check(self.lib.gsb_fp64_probe(self.ctx, n_threads, iters, _ptr(sink), self.stream()))
        return sink


def records_from_bytes(t: torch.Tensor, n: int) -> np.ndarray:
    """Decode one trajectory's record slab (uint8 [cap, 64]) into DecisionRecord rows."""
    return t[:n].cpu().numpy().reshape(-1).view(DECISION_DTYPE)
