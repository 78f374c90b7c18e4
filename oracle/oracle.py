"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU oracles.

* ``Restatement`` loads ``oracle/build/libgs_oracle.so`` (gs_oracle.c, the plain-C
  restatement of the reference hot path).
* ``Reference`` loads ``oracle/_ref/libgreensim_ref.so`` (the unmodified reference
  sources from /root/reference/proj/src behind ref_capi.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference
legs may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATE_SO = os.path.join(HERE, "build", "libgs_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgreensim_ref.so")

_d = C.c_double
_i32 = C.c_int32
_i64 = C.c_int64
_u64 = C.c_uint64
_p = C.c_void_p


class Profile(C.Structure):
    """gso_profile == greensim::GpuProfile minus the name (gpu_model.hpp:16-87)."""

    _fields_ = [(n, _d) for n in (
        "f_min_mhz", "f_max_mhz", "step_mhz", "f_ref_mhz",
        "lat_a", "lat_b", "lat_c", "lat_f_ref_mhz",
        "dec_alpha0_ms", "dec_alpha1_ms", "dec_beta0_ms", "dec_beta1_ms", "dec_f_ref_mhz",
        "k3", "k2", "k1", "k0", "p_idle_w")]

    def tuple(self):
        return tuple(getattr(self, n) for n, _ in self._fields_)


class QoptCfg(C.Structure):
    _fields_ = [("resolve_period_ms", _d), ("margin_prefill", _d), ("min_budget_ms", _d),
                ("first_token_allowance_ms", _d)]


class CtlCfg(C.Structure):
    _fields_ = [("tslo_ms", _d), ("margin_decode", _d), ("fine_period_ms", _d),
                ("coarse_period_ms", _d), ("adapt_period_s", _d), ("step_mhz", _d),
                ("max_step_mhz", _d), ("hysteresis_count", _i32), ("tbt_window_tokens", _i32),
                ("bias_threshold", _d), ("tps_scale", _d), ("upper_margin", _d),
                ("lower_margin", _d)]


class Decision(C.Structure):
    _fields_ = [("tick_ms", _d), ("tps", _d), ("p95_tbt_ms", _d), ("band_lo", _d),
                ("band_hi", _d), ("command_mhz", _d), ("worker", _i32), ("bucket", _i32),
                ("action", _i32), ("pad_", _i32)]


class BandTable(C.Structure):
    _fields_ = [("n", _i32), ("tps_lo", _p), ("tps_hi", _p), ("f_opt_mhz", _p)]


class Telemetry(C.Structure):
    _fields_ = [("n_events", _i64), ("t_ms", _p), ("tokens", _p), ("gap_off", _p), ("gaps", _p)]


class SimCfg(C.Structure):
    """gso_sim_cfg == greensim::SimConfig (simkernel.hpp:88-104) minus scripted_freq."""

    _fields_ = [("n_prefill_workers", _i32), ("n_decode_workers", _i32),
                ("gpus_per_prefill_worker", _i32), ("max_batch", _i32), ("max_queue", _i32),
                ("pad_", _i32), ("actuation_delay_ms", _d), ("handoff_delay_ms", _d),
                ("band_tps_lo", _d), ("band_tps_hi", _d), ("band_tps_step", _d)]


class Slo(C.Structure):
    """gso_slo == greensim::SloConfig (simkernel.hpp:53-62)."""

    _fields_ = [("ttft_sm_ms", _d), ("ttft_l_ms", _d), ("tbt_p95_ms", _d)]


TRACE_KINDS = ("EmptyTrace", "NonMonotoneArrivals", "MalformedRow", "BadHeader",
               "ClassMismatch", "BadShape")  # greensim::TraceError::Kind order


class TraceErr(C.Structure):
    _fields_ = [("kind", _i32), ("detail", _i32), ("row", _i64), ("msg", C.c_char * 8192)]


class Policy(C.Structure):
    """gso_policy == greensim::GovernorPolicy (simkernel.hpp:26-45)."""

    _fields_ = [("kind", _i32), ("routing_enabled", _i32), ("n_thresholds", _i32),
                ("thresholds", _i32 * 7), ("worker_map", _p), ("fixed_freq_mhz", _d),
                ("prefill_opt", QoptCfg), ("decode_ctl", CtlCfg)]


class Scripted(C.Structure):
    _fields_ = [("time_ms", _d), ("prefill_pool", _i32), ("worker", _i32), ("f_mhz", _d)]


class PoolSummary(C.Structure):
    """gso_pool_summary: the decode-side (K5) summary of one run (gs_oracle.h)."""

    _fields_ = [("decode_pool_j", _d), ("active_decode_j", _d), ("idle_j", _d),
                ("sim_end_ms", _d), ("n_completed", _i64), ("n_rejected", _i64),
                ("n_ttft_ok", _i64), ("n_tbt_ok", _i64), ("tbt_samples", _i64),
                ("tbt_samples_ok", _i64), ("n_decisions", _i64), ("n_freq_changes", _i64),
                ("n_steps", _i64), ("decision_digest", _u64), ("freq_digest", _u64),
                ("request_digest", _u64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


POLICY_KINDS = {"defaultnv": 0, "fixed": 1, "greenllm": 2, "prefillsplit": 3}


def default_sim_cfg(**kw) -> SimCfg:
    """SimConfig defaults (simkernel.hpp:88-104)."""
    c = SimCfg(2, 4, 2, 64, 10000, 0, 5.0, 0.0, 200.0, 3000.0, 200.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def default_slo(**kw) -> Slo:
    c = Slo(400.0, 2000.0, 100.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class PolicyHolder:
    """A Policy plus the worker_map array it points to."""

    def __init__(self, kind="greenllm", thresholds=(1024,), worker_map=(0, 1), routing=True,
                 fixed_f=0.0, qcfg=None, ccfg=None):
        self.wm = np.ascontiguousarray(worker_map, np.int32)
        thr = (_i32 * 7)(*thresholds)
        self.c = Policy(POLICY_KINDS[kind], 1 if routing else 0, len(thresholds), thr,
                        ptr(self.wm), fixed_f, qcfg or default_qopt_cfg(),
                        ccfg or default_ctl_cfg())


def _read_sim(lib, pre: str, h) -> dict:
    """Pulls every output of a gso_sim_* / ref_sim_* handle into numpy arrays."""
    z = np.zeros(10, np.int64)
    getattr(lib, pre + "sizes")(h, ptr(z))
    n, nt, nd, ntl, nc, ne, npw, ndw = (int(x) for x in z[:8])
    o = {"n_rejected_total": int(z[8]), "n_steps": int(z[9])}
    for k, dt in (("class_queue", np.int32), ("prefill_worker", np.int32),
                  ("decode_worker", np.int32), ("prefill_start", np.float64),
                  ("prefill_end", np.float64), ("first_token", np.float64),
                  ("finish", np.float64), ("completed", np.uint8), ("rejected", np.uint8),
                  ("cls", np.int8)):
        o[k] = np.zeros(n, dt)
    getattr(lib, pre + "requests")(h, *(ptr(o[k]) for k in (
        "class_queue", "prefill_worker", "decode_worker", "prefill_start", "prefill_end",
        "first_token", "finish", "completed", "rejected", "cls")))
    o["tbt_off"] = np.zeros(n + 1, np.int64)
    o["tbt"] = np.zeros(max(nt, 1))
    getattr(lib, pre + "tbt")(h, ptr(o["tbt_off"]), ptr(o["tbt"]))
    o["tbt"] = o["tbt"][:nt]
    o["prefill3"] = np.zeros((npw, 3))
    o["decode3"] = np.zeros((ndw, 3))
    o["n_intervals"] = np.zeros(npw + ndw, np.int64)
    getattr(lib, pre + "ledgers")(h, ptr(o["prefill3"]), ptr(o["decode3"]), ptr(o["n_intervals"]))
    o["decisions"] = np.zeros(nd, DECISION_DTYPE)
    getattr(lib, pre + "decisions")(h, ptr(o["decisions"]))
    o["tl_t"] = np.zeros(ntl)
    o["tl_pool"] = np.zeros(ntl, np.uint8)
    o["tl_worker"] = np.zeros(ntl, np.int32)
    o["tl_f"] = np.zeros(ntl)
    getattr(lib, pre + "timeline")(h, *(ptr(o[k]) for k in ("tl_t", "tl_pool", "tl_worker", "tl_f")))
    o["cmd_tick"] = np.zeros(nc)
    o["cmd_class"] = np.zeros(nc, np.int32)
    o["cmd_worker"] = np.zeros(nc, np.int32)
    o["cmd_f"] = np.zeros(nc)
    o["cmd_window"] = np.zeros(nc)
    o["cmd_infeasible"] = np.zeros(nc, np.uint8)
    getattr(lib, pre + "commands")(h, *(ptr(o[k]) for k in (
        "cmd_tick", "cmd_class", "cmd_worker", "cmd_f", "cmd_window", "cmd_infeasible")))
    sc = np.zeros(8)
    getattr(lib, pre + "scalars")(h, ptr(sc))
    o["scalars"] = sc
    o["sim_end_ms"] = float(sc[0])
    if ne >= 0:
        o["enq_t"] = np.zeros(ne)
        o["enq_req"] = np.zeros(ne, np.int64)
        getattr(lib, pre + "enqueue")(h, ptr(o["enq_t"]), ptr(o["enq_req"]))
    return o


DECISION_DTYPE = np.dtype([("tick_ms", "<f8"), ("tps", "<f8"), ("p95_tbt_ms", "<f8"),
                           ("band_lo", "<f8"), ("band_hi", "<f8"), ("command_mhz", "<f8"),
                           ("worker", "<i4"), ("bucket", "<i4"), ("action", "<i4"),
                           ("pad_", "<i4")])
assert DECISION_DTYPE.itemsize == C.sizeof(Decision)

ACTIONS = ("hold", "up", "down", "coarse_hold", "coarse_pending", "coarse_commit", "adapt_up",
           "adapt_down")


def default_profile() -> Profile:
    """GpuProfile::default_profile (gpu_model.cpp:121-130), synth-a100-40g."""
    return Profile(210.0, 1410.0, 15.0, 1410.0, 2.0e-5, 0.12, 8.0, 1410.0,
                   14.5, 0.1, 9.0, 0.135, 1410.0, 1.6e-7, -1.0e-4, 0.05, 216.5, 15.0)


def default_ctl_cfg(**kw) -> CtlCfg:
    """DecodeCtlConfig defaults (decode_ctl.hpp:13-29)."""
    c = CtlCfg(100.0, 0.95, 20.0, 200.0, 6.0, 15.0, 30.0, 3, 256, 0.8, 4.0, 1.0, 0.65)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def default_qopt_cfg(**kw) -> QoptCfg:
    c = QoptCfg(100.0, 0.95, 100.0, 100.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_p)


@dataclass
class TelemetryArrays:
    t_ms: np.ndarray      # f64 [E]
    tokens: np.ndarray    # i32 [E]
    gap_off: np.ndarray   # i64 [E+1]
    gaps: np.ndarray      # f64 [G]

    def c(self) -> Telemetry:
        return Telemetry(len(self.t_ms), ptr(self.t_ms), ptr(self.tokens), ptr(self.gap_off),
                         ptr(self.gaps))


class _TableHolder:
    def __init__(self, lo, hi, f):
        self.lo = np.ascontiguousarray(lo, np.float64)
        self.hi = np.ascontiguousarray(hi, np.float64)
        self.f = np.ascontiguousarray(f, np.float64)
        self.c = BandTable(len(self.lo), ptr(self.lo), ptr(self.hi), ptr(self.f))


def band_table(lo, hi, f) -> _TableHolder:
    return _TableHolder(lo, hi, f)


class Restatement:
    """gs_oracle.c — the plain-C restatement."""

    def __init__(self, path: str = RESTATE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle restate`")
        L = self.lib = C.CDLL(path)
        P = C.POINTER(Profile)
        L.gso_profile_validate.argtypes = [P]
        L.gso_grid_size.argtypes = [P]
        L.gso_grid_at.argtypes = [P, C.c_int]
        L.gso_grid_at.restype = _d
        L.gso_active_power_w.argtypes = [P, _d]
        L.gso_active_power_w.restype = _d
        L.gso_t_ref_total_ms.argtypes = [P, _i64, _p, _p]
        L.gso_t_ref_total_ms.restype = _d
        L.gso_energy_total.argtypes = [P, _i64, _p, _p, _d, _d, _p, _p, _p, _p]
        L.gso_energy_closed_form.argtypes = [P, _i64, _p, _p, _d, _d]
        L.gso_energy_closed_form.restype = _d
        L.gso_select_frequency.argtypes = [P, _i64, _p, _p, _d, _p, _p]
        L.gso_select_frequency_t.argtypes = [P, _d, _d, _p, _p]
        L.gso_queue_tick_one.argtypes = [P, C.POINTER(QoptCfg), _i64, _p, _p, _p, _d, _p, _p, _p,
                                         _p, _p]
        L.gso_classify.argtypes = [C.c_int, _p, _i32]
        L.gso_route_bin.argtypes = [_i64, _p, _p, C.c_int, _p, _i64, _i64, _i64, C.c_int, P, _d,
                                    _d, _d, _p, _p, _p, _p, _p]
        L.gso_quantile.argtypes = [_i64, _p, _d]
        L.gso_quantile.restype = _d
        L.gso_decode_steady_state.argtypes = [P, _d, _d, C.c_int, _p, _p]
        L.gso_build_band_table.argtypes = [P, C.c_int, _p, _d, C.c_int, C.c_int, _p, _p, _p, _p]
        L.gso_ctl_cfg_validate.argtypes = [C.POINTER(CtlCfg)]
        L.gso_n_ticks.argtypes = [_d, _d]
        L.gso_n_ticks.restype = _i64
        L.gso_window_series.argtypes = [C.POINTER(Telemetry), C.c_int, _d, _d, _d, _p, _p, _p]
        L.gso_replay_telemetry.argtypes = [C.POINTER(CtlCfg), C.POINTER(BandTable), _d, _d,
                                           C.c_int, C.POINTER(Telemetry), _d, _p, _i64]
        L.gso_replay_telemetry.restype = _i64
        L.gso_replay_series.argtypes = [C.POINTER(CtlCfg), C.POINTER(BandTable), _d, _d, C.c_int,
                                        _p, _p, _p, _d, _p, _i64]
        L.gso_replay_series.restype = _i64
        L.gso_digest_records.argtypes = [_p, _i64]
        L.gso_digest_records.restype = _u64
        L.gso_gen_poisson_trace.argtypes = [_d, _i64, _d, _d, _d, _d, _u64, _i64, _p, _p, _p]
        L.gso_gen_poisson_trace.restype = _i64
        L.gso_gen_sinusoid_decode_trace.argtypes = [_d, _d, _d, _i64, _u64, _i64, _p, _p, _p]
        L.gso_gen_sinusoid_decode_trace.restype = _i64
        SP = [C.POINTER(Profile), C.POINTER(Policy), C.POINTER(Slo), C.POINTER(SimCfg)]
        L.gso_sim_run.argtypes = SP + [_i64, _p, _p, _p, _p, _i64, _p, C.c_char_p, C.c_size_t]
        L.gso_sim_run.restype = _p
        L.gso_pool_run.argtypes = SP + [_i64, _p, _p, _p, _p, _i64, _p, _p, _d, C.c_char_p,
                                        C.c_size_t]
        L.gso_pool_run.restype = _p
        L.gso_sim_free.argtypes = [_p]
        L.gso_sim_snapshot_sizes.argtypes = [_p, _p, _p]
        L.gso_sim_snapshots.argtypes = [_p] + [_p] * 11
        for f, k in (("sizes", 1), ("requests", 10), ("tbt", 2), ("ledgers", 3), ("decisions", 1),
                     ("timeline", 4), ("commands", 6), ("enqueue", 2), ("scalars", 1)):
            getattr(L, "gso_sim_" + f).argtypes = [_p] + [_p] * k
        L.gso_sim_summary.argtypes = [_p, C.POINTER(Slo), C.POINTER(PoolSummary)]
        L.gso_trace_parse.argtypes = [C.c_char_p, _i64, _i32, _i64, _p, _p, _p, _p, _p,
                                      C.POINTER(TraceErr)]
        L.gso_trace_parse.restype = _i64
        L.gso_trace_format.argtypes = [_i64, _p, _p, _p, _p, _p, _i64]
        L.gso_trace_format.restype = _i64
        L.gso_pool_summary_from.argtypes = ([C.POINTER(Slo), _i64] + [_p] * 10 + [C.c_int, _p, _i64,
                                            _p, _i64, _p, _p, _p, _p, _d, _i64,
                                            C.POINTER(PoolSummary)])

    # ---- trace CSV (load_trace / save_trace_csv, trace.cpp:56-145) ----
    def trace_parse(self, data: bytes, class_threshold: int = 1024):
        """(arrival, prompt, output, slo_class, has_class) or a TRACE_ERROR tuple
        ("error", kind name, row, message)."""
        cap = max(1, len(data) // 2 + 2)
        a = np.zeros(cap, np.int64)
        p = np.zeros(cap, np.int32)
        o = np.zeros(cap, np.int32)
        c = np.zeros(cap, np.uint8)
        hc = np.zeros(1, np.int32)
        err = TraceErr()
        n = self.lib.gso_trace_parse(data, len(data), class_threshold, cap, ptr(a), ptr(p), ptr(o),
                                     ptr(c), ptr(hc), C.byref(err))
        if n < 0:
            return ("error", TRACE_KINDS[err.kind], err.row if err.row > 0 else None,
                    err.msg.decode(errors="replace"))
        return a[:n], p[:n], o[:n], c[:n], bool(hc[0])

    def trace_format(self, a, p, o, cls=None) -> bytes:
        a = np.ascontiguousarray(a, np.int64)
        p = np.ascontiguousarray(p, np.int32)
        o = np.ascontiguousarray(o, np.int32)
        c = None if cls is None else np.ascontiguousarray(cls, np.uint8)
        nb = self.lib.gso_trace_format(len(a), ptr(a), ptr(p), ptr(o), ptr(c), None, 0)
        buf = C.create_string_buffer(nb)
        self.lib.gso_trace_format(len(a), ptr(a), ptr(p), ptr(o), ptr(c), C.cast(buf, _p), nb)
        return buf.raw[:nb]

    # ---- prefill ----
    def grid(self, prof: Profile) -> np.ndarray:
        n = self.lib.gso_grid_size(C.byref(prof))
        return np.array([self.lib.gso_grid_at(C.byref(prof), i) for i in range(n)])

    def validate(self, prof: Profile) -> bool:
        return self.lib.gso_profile_validate(C.byref(prof)) == 0

    def active_power(self, prof, f):
        return self.lib.gso_active_power_w(C.byref(prof), f)

    def t_ref(self, prof, prompts, wf=None):
        p = np.ascontiguousarray(prompts, np.int32)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        return self.lib.gso_t_ref_total_ms(C.byref(prof), len(p), ptr(p), ptr(w))

    def energy_total(self, prof, prompts, f, window, wf=None):
        p = np.ascontiguousarray(prompts, np.int32)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        a, i, t, fe = _d(), _d(), _d(), C.c_int()
        rc = self.lib.gso_energy_total(C.byref(prof), len(p), ptr(p), ptr(w), f, window,
                                       C.byref(a), C.byref(i), C.byref(t), C.byref(fe))
        if rc != 0:
            raise ValueError("ModelError")
        return a.value, i.value, t.value, bool(fe.value)

    def closed_form(self, prof, prompts, f, window, wf=None):
        p = np.ascontiguousarray(prompts, np.int32)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        return self.lib.gso_energy_closed_form(C.byref(prof), len(p), ptr(p), ptr(w), f, window)

    def select_frequency(self, prof, prompts, window, wf=None):
        """-> (f_idx, f_mhz, energy_j) or None (nullopt)."""
        p = np.ascontiguousarray(prompts, np.int32)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        f, e = _d(), _d()
        idx = self.lib.gso_select_frequency(C.byref(prof), len(p), ptr(p), ptr(w), window,
                                            C.byref(f), C.byref(e))
        if idx == -2:
            raise ValueError("ModelError: empty batch")
        return None if idx < 0 else (idx, f.value, e.value)

    def select_t(self, prof, t_ref, window):
        f, e = _d(), _d()
        idx = self.lib.gso_select_frequency_t(C.byref(prof), t_ref, window, C.byref(f), C.byref(e))
        return None if idx < 0 else (idx, f.value, e.value)

    def queue_tick_one(self, prof, cfg, prompts, deadlines, now, wf=None):
        p = np.ascontiguousarray(prompts, np.int32)
        d = np.ascontiguousarray(deadlines, np.float64)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        f, win, inf, idx, e = _d(), _d(), C.c_int(), C.c_int(), _d()
        self.lib.gso_queue_tick_one(C.byref(prof), C.byref(cfg), len(p), ptr(p), ptr(d), ptr(w),
                                    now, C.byref(f), C.byref(win), C.byref(inf), C.byref(idx),
                                    C.byref(e))
        return f.value, win.value, bool(inf.value), idx.value, e.value

    def classify(self, thresholds, prompt):
        t = np.ascontiguousarray(thresholds, np.int32)
        return self.lib.gso_classify(len(t), ptr(t), int(prompt))

    def route_bin(self, arrival, prompt, thresholds, window_ms, w0, n_windows, profiles,
                  ttft_sm=400.0, ttft_l=2000.0, allowance=100.0, fifo=True):
        arrival = np.ascontiguousarray(arrival, np.int64)
        prompt = np.ascontiguousarray(prompt, np.int32)
        thr = np.ascontiguousarray(thresholds, np.int32)
        C_ = len(thr) + 1
        cells = n_windows * C_
        P = len(profiles)
        parr = (Profile * P)(*profiles)
        cls = np.zeros(len(arrival), np.uint8)
        cnt = np.zeros(cells, np.uint32)
        tref = np.zeros((P, cells), np.float64)
        mdl = np.zeros(cells, np.float64)
        ff = np.zeros(len(arrival), np.int64) if fifo else None
        rc = self.lib.gso_route_bin(len(arrival), ptr(arrival), ptr(prompt), len(thr), ptr(thr),
                                    window_ms, w0, n_windows, P, parr, ttft_sm, ttft_l, allowance,
                                    ptr(cls), ptr(cnt), ptr(tref), ptr(mdl), ptr(ff))
        assert rc == 0
        return cls, cnt, tref, mdl, ff

    # ---- decode ----
    def quantile(self, xs, q):
        x = np.ascontiguousarray(xs, np.float64)
        return self.lib.gso_quantile(len(x), ptr(x), q)

    def steady_state(self, prof, tps, f, max_batch=64):
        b, t = _d(), _d()
        s = self.lib.gso_decode_steady_state(C.byref(prof), tps, f, max_batch, C.byref(b), C.byref(t))
        return bool(s), b.value, t.value

    def band_table(self, prof, levels, t_slo, workers=4, max_batch=64):
        lv = np.ascontiguousarray(levels, np.float64)
        n = len(lv)
        lo, hi, fo = np.zeros(n), np.zeros(n), np.zeros(n)
        fe = np.zeros(n, np.uint8)
        rc = self.lib.gso_build_band_table(C.byref(prof), n, ptr(lv), t_slo, workers, max_batch,
                                           ptr(lo), ptr(hi), ptr(fo), ptr(fe))
        if rc != 0:
            raise ValueError("ModelError")
        return lo, hi, fo, fe.astype(bool)

    def n_ticks(self, period, t_end):
        return self.lib.gso_n_ticks(period, t_end)

    def window_series(self, tel: TelemetryArrays, capacity, fine_period, coarse_period, t_end):
        nf, nc = self.n_ticks(fine_period, t_end), self.n_ticks(coarse_period, t_end)
        has = np.zeros(nf, np.uint8)
        p95 = np.zeros(nf)
        tps = np.zeros(nc)
        ct = tel.c()
        self.lib.gso_window_series(C.byref(ct), capacity, fine_period, coarse_period, t_end,
                                   ptr(has), ptr(p95), ptr(tps))
        return has, p95, tps

    def replay_telemetry(self, cfg, table: _TableHolder, f_min, f_max, worker, tel, t_end):
        ct = tel.c()
        cap = 1 << 14
        while True:
            out = np.zeros(cap, DECISION_DTYPE)
            n = self.lib.gso_replay_telemetry(C.byref(cfg), C.byref(table.c), f_min, f_max, worker,
                                              C.byref(ct), t_end, ptr(out), cap)
            if n < 0:
                raise ValueError("ModelError")
            if n <= cap:
                return out[:n]
            cap = n

    def replay_series(self, cfg, table: _TableHolder, f_min, f_max, worker, has, p95, tps, t_end):
        has = np.ascontiguousarray(has, np.uint8)
        p95 = np.ascontiguousarray(p95, np.float64)
        tps = np.ascontiguousarray(tps, np.float64)
        cap = 1 << 14
        while True:
            out = np.zeros(cap, DECISION_DTYPE)
            n = self.lib.gso_replay_series(C.byref(cfg), C.byref(table.c), f_min, f_max, worker,
                                           ptr(has), ptr(p95), ptr(tps), t_end, ptr(out), cap)
            if n < 0:
                raise ValueError("ModelError")
            if n <= cap:
                return out[:n]
            cap = n

    def digest(self, recs: np.ndarray) -> int:
        recs = np.ascontiguousarray(recs, DECISION_DTYPE)
        return int(self.lib.gso_digest_records(ptr(recs), len(recs)))

    def gen_poisson_trace(self, qps, duration_ms, short=512.0, long=4096.0, long_fraction=0.1,
                          output=128.0, seed=7):
        cap = int(qps * duration_ms / 1000.0 * 1.2 + 1000)
        while True:
            a = np.zeros(cap, np.int64)
            p = np.zeros(cap, np.int32)
            o = np.zeros(cap, np.int32)
            n = self.lib.gso_gen_poisson_trace(qps, duration_ms, short, long, long_fraction, output,
                                               seed, cap, ptr(a), ptr(p), ptr(o))
            if n <= cap:
                return a[:n], p[:n], o[:n]
            cap = n

    def gen_sinusoid_decode_trace(self, mean, amp, period, duration_ms, seed):
        cap = int(duration_ms / 1000.0 * mean / 64 * 1.5 + 100)
        while True:
            a = np.zeros(cap, np.int64)
            p = np.zeros(cap, np.int32)
            o = np.zeros(cap, np.int32)
            n = self.lib.gso_gen_sinusoid_decode_trace(mean, amp, period, duration_ms, seed, cap,
                                                       ptr(a), ptr(p), ptr(o))
            if n <= cap:
                return a[:n], p[:n], o[:n]
            cap = n


    # ---- the reference simulator restated (gs_sim.c) ----
    def sim_run(self, prof, policy: "PolicyHolder", slo, cfg, arrival, prompt, output, cls=None,
                scripted=None) -> dict:
        """gso_sim_run: the whole two-pool simulator (simkernel.cpp); dict of arrays."""
        arrival = np.ascontiguousarray(arrival, np.int64)
        prompt = np.ascontiguousarray(prompt, np.int32)
        output = np.ascontiguousarray(output, np.int32)
        cls = None if cls is None else np.ascontiguousarray(cls, np.int8)
        sc = None
        if scripted:
            sc = (Scripted * len(scripted))(*[Scripted(*x) for x in scripted])
        err = C.create_string_buffer(256)
        h = self.lib.gso_sim_run(C.byref(prof), C.byref(policy.c), C.byref(slo), C.byref(cfg),
                                 len(arrival), ptr(arrival), ptr(prompt), ptr(output), ptr(cls),
                                 len(scripted or ()), sc, err, 256)
        if not h:
            raise RuntimeError(err.value.decode())
        try:
            out = _read_sim(self.lib, "gso_sim_", h)
            sm = PoolSummary()
            self.lib.gso_sim_summary(h, C.byref(slo), C.byref(sm))
            out["summary"] = sm.as_dict()
            out["snapshots"] = self._snapshots(h)
            return out
        finally:
            self.lib.gso_sim_free(h)

    def _snapshots(self, h) -> dict:
        """The optimizer snapshots with the raw running-job state (gs_sim.c on_optimizer_tick)."""
        ns, nj = np.zeros(1, np.int64), np.zeros(1, np.int64)
        self.lib.gso_sim_snapshot_sizes(h, ptr(ns), ptr(nj))
        ns, nj = int(ns[0]), int(nj[0])
        o = {"now": np.zeros(ns), "cls": np.zeros(ns, np.int32), "off": np.zeros(ns + 1, np.int64),
             "prompt": np.zeros(nj, np.int32), "deadline": np.zeros(nj),
             "running": np.zeros(nj, np.uint8), "rem_ref": np.zeros(nj), "upd_ms": np.zeros(nj),
             "freq": np.zeros(nj), "t_ref": np.zeros(nj), "wf": np.zeros(nj)}
        self.lib.gso_sim_snapshots(h, *(ptr(o[k]) for k in (
            "now", "cls", "off", "prompt", "deadline", "running", "rem_ref", "upd_ms", "freq",
            "t_ref", "wf")))
        return o

    def pool_run(self, prof, policy: "PolicyHolder", slo, cfg, arrival, prompt, output, enq_t,
                 enq_req, end_floor, cls=None) -> dict:
        """gso_pool_run: the decode pool alone, driven by a recorded enqueue stream."""
        arrival = np.ascontiguousarray(arrival, np.int64)
        prompt = np.ascontiguousarray(prompt, np.int32)
        output = np.ascontiguousarray(output, np.int32)
        cls = None if cls is None else np.ascontiguousarray(cls, np.int8)
        enq_t = np.ascontiguousarray(enq_t, np.float64)
        enq_req = np.ascontiguousarray(enq_req, np.int64)
        err = C.create_string_buffer(256)
        h = self.lib.gso_pool_run(C.byref(prof), C.byref(policy.c), C.byref(slo), C.byref(cfg),
                                  len(arrival), ptr(arrival), ptr(prompt), ptr(output), ptr(cls),
                                  len(enq_t), ptr(enq_t), ptr(enq_req), float(end_floor), err, 256)
        if not h:
            raise RuntimeError(err.value.decode())
        try:
            out = _read_sim(self.lib, "gso_sim_", h)
            sm = PoolSummary()
            self.lib.gso_sim_summary(h, C.byref(slo), C.byref(sm))
            out["summary"] = sm.as_dict()
            return out
        finally:
            self.lib.gso_sim_free(h)

    def pool_summary_from(self, slo, arrival, o: dict) -> dict:
        """The K5 summary of any simulator output dict (e.g. the reference's run())."""
        arrival = np.ascontiguousarray(arrival, np.float64)
        sm = PoolSummary()
        d3 = np.ascontiguousarray(o["decode3"])
        self.lib.gso_pool_summary_from(
            C.byref(slo), len(arrival), ptr(arrival), ptr(o["cls"]), ptr(o["decode_worker"]),
            ptr(o["prefill_end"]), ptr(o["first_token"]), ptr(o["finish"]), ptr(o["completed"]),
            ptr(o["rejected"]), ptr(o["tbt_off"]), ptr(o["tbt"] if len(o["tbt"]) else np.zeros(1)),
            d3.shape[0], ptr(d3), len(o["decisions"]), ptr(o["decisions"]), len(o["tl_t"]),
            ptr(o["tl_t"]), ptr(o["tl_pool"]), ptr(o["tl_worker"]), ptr(o["tl_f"]),
            float(o["sim_end_ms"]), int(o.get("n_steps", -1)), C.byref(sm))
        return sm.as_dict()


class Reference:
    """The unmodified reference library behind ref_capi.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` (needs /root/reference)")
        L = self.lib = C.CDLL(path)
        P = C.POINTER(Profile)
        L.ref_profile_validate.argtypes = [P]
        L.ref_default_profile.argtypes = [P]
        L.ref_active_power_w.argtypes = [P, _d]
        L.ref_active_power_w.restype = _d
        L.ref_t_ref_total_ms.argtypes = [P, _i64, _p, _p]
        L.ref_t_ref_total_ms.restype = _d
        L.ref_energy_total.argtypes = [P, _i64, _p, _p, _d, _d, _p, _p, _p, _p]
        L.ref_energy_closed_form.argtypes = [P, _i64, _p, _p, _d, _d]
        L.ref_energy_closed_form.restype = _d
        L.ref_select_frequency.argtypes = [P, _i64, _p, _p, _d, _p, _p]
        L.ref_select_frequency_many.argtypes = [P, _i64, _p, _p, _p, _p, C.c_int, _p, _p, _p]
        L.ref_prefill_pass.argtypes = [C.c_int, _p, C.c_int, C.c_int, _p, _i64, _p, _p, _i64,
                                       _i64, _i64, _d, C.c_int, _p, _p]
        L.ref_prefill_pass.restype = _i64
        L.ref_freq_timeline_csv.argtypes = [_i64, _p, _p, _p, _p, _p, _i64]
        L.ref_freq_timeline_csv.restype = _i64
        L.ref_prefill_commands_csv.argtypes = [_i64, _p, _p, _p, _p, _p, _p, _p, _i64]
        L.ref_prefill_commands_csv.restype = _i64
        L.ref_decision_log_csv.argtypes = [_i64, _p, _p, _i64]
        L.ref_decision_log_csv.restype = _i64
        L.ref_prefill_pass_ex.argtypes = [C.c_int, C.c_int, _p, C.c_int, C.c_int, _p, _i64, _p,
                                          _p, _i64, _i64, _i64, _d, C.POINTER(QoptCfg), _d, _d,
                                          C.c_int, _p, _p, _p]
        L.ref_prefill_pass_ex.restype = _i64
        L.ref_queue_optimizer_tick.argtypes = [P, C.POINTER(QoptCfg), C.c_int, _p, _p, _p, _p, _p,
                                               _d, _p, _p, _p, _p]
        L.ref_classify.argtypes = [C.c_int, _p, _i32]
        L.ref_dispatch.argtypes = [C.c_int, C.c_int, _p, _i64, _p, _p, _p, _p, _p]
        L.ref_quantile.argtypes = [_i64, _p, _d]
        L.ref_quantile.restype = _d
        L.ref_decode_steady_state.argtypes = [P, _d, _d, C.c_int, _p, _p]
        L.ref_build_band_table.argtypes = [P, C.c_int, _p, _d, C.c_int, C.c_int, _p, _p, _p, _p]
        L.ref_ctl_cfg_validate.argtypes = [C.POINTER(CtlCfg)]
        L.ref_tps_window.argtypes = [_d, _i64, _p, _p, _d]
        L.ref_tps_window.restype = _d
        L.ref_tbt_window_p95.argtypes = [C.c_int, _i64, _p]
        L.ref_tbt_window_p95.restype = _d
        L.ref_replay_telemetry.argtypes = [C.POINTER(CtlCfg), C.POINTER(BandTable), _d, _d, _d, _d,
                                           C.c_int, C.POINTER(Telemetry), _d, _p, _i64]
        L.ref_replay_telemetry.restype = _i64
        L.ref_decode_script.argtypes = [C.POINTER(CtlCfg), C.POINTER(BandTable), _d, _d, _d, _d,
                                        C.c_int, _i64, _p, _p, _p, _p, _p, _i64, _p, _p, _p]
        L.ref_decode_script.restype = _i64
        L.ref_replay_many.argtypes = [_i64, _p, _p, _p, _p, _p, _p, _d, _d, _d, _d, _d, C.c_int,
                                      _p, _p]
        L.ref_digest_records.argtypes = [_p, _i64]
        L.ref_digest_records.restype = _u64
        L.ref_gen_poisson_trace.argtypes = [_d, _i64, _d, _d, _d, _d, _u64, _i64, _p, _p, _p]
        L.ref_gen_poisson_trace.restype = _i64
        L.ref_gen_sinusoid_decode_trace.argtypes = [_d, _d, _d, _i64, _u64, _i64, _p, _p, _p]
        L.ref_gen_sinusoid_decode_trace.restype = _i64
        L.ref_run_capture.argtypes = [_i64, _p, _p, _p, P, C.c_int, _d, C.c_int, _p, C.c_int, _p,
                                      C.POINTER(QoptCfg), C.POINTER(CtlCfg)]
        L.ref_run_capture.restype = _p
        L.ref_run_free.argtypes = [_p]
        L.ref_run_sizes.argtypes = [_p, _p]
        L.ref_run_snapshots.argtypes = [_p] + [_p] * 7
        L.ref_run_commands.argtypes = [_p] + [_p] * 5
        L.ref_run_controller_inputs.argtypes = [_p] + [_p] * 9
        L.ref_run_decisions.argtypes = [_p, _p]
        L.ref_run_requests.argtypes = [_p] + [_p] * 8
        SP = [C.POINTER(Profile), C.POINTER(Policy), C.POINTER(Slo), C.POINTER(SimCfg)]
        L.ref_sim_run.argtypes = SP + [_i64, _p, _p, _p, _p, _i64, _p, C.c_char_p, C.c_size_t]
        L.ref_sim_run.restype = _p
        L.ref_sim_free.argtypes = [_p]
        for f, k in (("sizes", 1), ("requests", 10), ("tbt", 2), ("ledgers", 3), ("decisions", 1),
                     ("timeline", 4), ("commands", 6), ("scalars", 1)):
            getattr(L, "ref_sim_" + f).argtypes = [_p] + [_p] * k
        L.ref_sim_run_many.argtypes = [C.POINTER(Profile), C.POINTER(Policy), _p, _i64,
                                       C.POINTER(Slo), C.POINTER(SimCfg), _i64, _p, _p, _p,
                                       C.c_int, _p, _p]

    def default_profile(self) -> Profile:
        p = Profile()
        self.lib.ref_default_profile(C.byref(p))
        return p

    def validate(self, prof) -> bool:
        return self.lib.ref_profile_validate(C.byref(prof)) == 0

    def active_power(self, prof, f):
        return self.lib.ref_active_power_w(C.byref(prof), f)

    def t_ref(self, prof, prompts, wf=None):
        p = np.ascontiguousarray(prompts, np.int32)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        return self.lib.ref_t_ref_total_ms(C.byref(prof), len(p), ptr(p), ptr(w))

    def energy_total(self, prof, prompts, f, window, wf=None):
        p = np.ascontiguousarray(prompts, np.int32)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        a, i, t, fe = _d(), _d(), _d(), C.c_int()
        rc = self.lib.ref_energy_total(C.byref(prof), len(p), ptr(p), ptr(w), f, window,
                                       C.byref(a), C.byref(i), C.byref(t), C.byref(fe))
        if rc != 0:
            raise ValueError("ModelError")
        return a.value, i.value, t.value, bool(fe.value)

    def closed_form(self, prof, prompts, f, window, wf=None):
        p = np.ascontiguousarray(prompts, np.int32)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        return self.lib.ref_energy_closed_form(C.byref(prof), len(p), ptr(p), ptr(w), f, window)

    def select_frequency(self, prof, prompts, window, wf=None):
        """-> (f_mhz, energy_j) or None."""
        p = np.ascontiguousarray(prompts, np.int32)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        f, e = _d(), _d()
        ok = self.lib.ref_select_frequency(C.byref(prof), len(p), ptr(p), ptr(w), window,
                                           C.byref(f), C.byref(e))
        return (f.value, e.value) if ok else None

    def select_many(self, prof, off, prompts, windows, wf=None, threads=1):
        off = np.ascontiguousarray(off, np.int64)
        prompts = np.ascontiguousarray(prompts, np.int32)
        windows = np.ascontiguousarray(windows, np.float64)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        nb = len(off) - 1
        f = np.zeros(nb)
        e = np.zeros(nb)
        found = np.zeros(nb, np.uint8)
        self.lib.ref_select_frequency_many(C.byref(prof), nb, ptr(off), ptr(prompts), ptr(w),
                                           ptr(windows), threads, ptr(f), ptr(e), ptr(found))
        return f, e, found.astype(bool)

    def freq_timeline_csv(self, applied, pool, worker, f) -> bytes:
        a = [np.ascontiguousarray(applied, np.float64), np.ascontiguousarray(pool, np.uint8),
             np.ascontiguousarray(worker, np.int32), np.ascontiguousarray(f, np.float64)]
        n = len(a[0])
        cap = 64 * n + 64
        buf = C.create_string_buffer(cap)
        k = self.lib.ref_freq_timeline_csv(n, *(ptr(x) for x in a), buf, cap)
        return buf.raw[:k]

    def prefill_commands_csv(self, tick, cls, worker, f, window, infeasible) -> bytes:
        a = [np.ascontiguousarray(tick, np.float64), np.ascontiguousarray(cls, np.int32),
             np.ascontiguousarray(worker, np.int32), np.ascontiguousarray(f, np.float64),
             np.ascontiguousarray(window, np.float64), np.ascontiguousarray(infeasible, np.uint8)]
        n = len(a[0])
        cap = 96 * n + 64
        buf = C.create_string_buffer(cap)
        k = self.lib.ref_prefill_commands_csv(n, *(ptr(x) for x in a), buf, cap)
        return buf.raw[:k]

    def decision_log_csv(self, records) -> bytes:
        """greensim::decision_log_csv over records in the gsb_decision layout (a structured or
        raw uint8 array of 64-byte records, action as its index), run by
        oracle/_ref/ref_save_trace --decisions in its own process."""
        import subprocess
        import tempfile
        raw = np.ascontiguousarray(records).view(np.uint8).reshape(-1)
        n = raw.size // 64
        with tempfile.TemporaryDirectory() as d:
            src, dst = os.path.join(d, "rec.bin"), os.path.join(d, "log.csv")
            with open(src, "wb") as f:
                f.write(np.int64(n).tobytes() + raw.tobytes())
            subprocess.run([os.path.join(os.path.dirname(REF_SO), "ref_save_trace"),
                            "--decisions", src, dst], check=True)
            with open(dst, "rb") as f:
                return f.read()

    def prefill_pass(self, profs, thresholds, arrival, prompt, window_ms, w0, n_windows, D,
                     threads=1, outputs=True, enabled=True):
        """ref_prefill_pass: Dispatcher routing + select_frequency for every (window, class,
        profile) of the trace (the reference's CPU path). Returns (f_idx [P, cells] or None,
        energy [P, cells] or None, evaluated (cell, profile) pairs)."""
        t = np.ascontiguousarray(thresholds, np.int32)
        a = np.ascontiguousarray(arrival, np.int64)
        p = np.ascontiguousarray(prompt, np.int32)
        P = len(profs)
        arr = (Profile * P)(*profs)
        C_ = len(t) + 1 if enabled else 1
        cells = n_windows * C_
        fi = np.empty((P, cells), np.int16) if outputs else None
        en = np.empty((P, cells), np.float64) if outputs else None
        n = self.lib.ref_prefill_pass(P, C.cast(arr, _p), 1 if enabled else 0, len(t), ptr(t), len(a), ptr(a),
                                      ptr(p), int(window_ms), int(w0), int(n_windows), float(D),
                                      int(threads), ptr(fi), ptr(en))
        return fi, en, int(n)

    def prefill_pass_deadline(self, profs, thresholds, arrival, prompt, window_ms, w0, n_windows,
                              qopt=None, ttft_sm=400.0, ttft_l=2000.0, threads=1):
        """ref_prefill_pass_ex mode 1: queue_optimizer_tick per window at now = window start.
        Returns (f_idx [P, cells] (-1 infeasible, -2 no command), window [cells] (profile 0),
        number of commands)."""
        t = np.ascontiguousarray(thresholds, np.int32)
        a = np.ascontiguousarray(arrival, np.int64)
        p = np.ascontiguousarray(prompt, np.int32)
        P = len(profs)
        arr = (Profile * P)(*profs)
        cells = n_windows * (len(t) + 1)
        fi = np.empty((P, cells), np.int16)
        win = np.zeros(cells, np.float64)
        q = qopt if qopt is not None else default_qopt_cfg()
        n = self.lib.ref_prefill_pass_ex(1, P, C.cast(arr, _p), 1, len(t), ptr(t), len(a), ptr(a),
                                         ptr(p), int(window_ms), int(w0), int(n_windows), 0.0,
                                         C.byref(q), float(ttft_sm), float(ttft_l), int(threads),
                                         ptr(fi), None, ptr(win))
        return fi, win, int(n)

    def queue_optimizer_tick(self, prof, cfg, class_ids, off, prompts, deadlines, now, wf=None):
        class_ids = np.ascontiguousarray(class_ids, np.int32)
        off = np.ascontiguousarray(off, np.int64)
        prompts = np.ascontiguousarray(prompts, np.int32)
        deadlines = np.ascontiguousarray(deadlines, np.float64)
        w = None if wf is None else np.ascontiguousarray(wf, np.float64)
        nq = len(class_ids)
        cc = np.zeros(nq, np.int32)
        cf = np.zeros(nq)
        cw = np.zeros(nq)
        ci = np.zeros(nq, np.uint8)
        n = self.lib.ref_queue_optimizer_tick(C.byref(prof), C.byref(cfg), nq, ptr(class_ids),
                                              ptr(off), ptr(prompts), ptr(deadlines), ptr(w), now,
                                              ptr(cc), ptr(cf), ptr(cw), ptr(ci))
        return [(int(cc[i]), cf[i], cw[i], bool(ci[i])) for i in range(n)]

    def classify(self, thresholds, prompt):
        t = np.ascontiguousarray(thresholds, np.int32)
        return self.lib.ref_classify(len(t), ptr(t), int(prompt))

    def dispatch(self, thresholds, prompts, ids=None, enabled=True):
        t = np.ascontiguousarray(thresholds, np.int32)
        prompts = np.ascontiguousarray(prompts, np.int32)
        n = len(prompts)
        ids = np.arange(n, dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        q = np.zeros(n, np.int32)
        fifo = np.zeros(n, np.int64)
        sizes = np.zeros(len(t) + 1, np.int64)
        rc = self.lib.ref_dispatch(1 if enabled else 0, len(t), ptr(t), n, ptr(ids), ptr(prompts),
                                   ptr(q), ptr(fifo), ptr(sizes))
        if rc != 0:
            raise ValueError("RouterError")
        return q, fifo, sizes

    def quantile(self, xs, q):
        x = np.ascontiguousarray(xs, np.float64)
        return self.lib.ref_quantile(len(x), ptr(x), q)

    def steady_state(self, prof, tps, f, max_batch=64):
        b, t = _d(), _d()
        s = self.lib.ref_decode_steady_state(C.byref(prof), tps, f, max_batch, C.byref(b), C.byref(t))
        return bool(s), b.value, t.value

    def band_table(self, prof, levels, t_slo, workers=4, max_batch=64):
        lv = np.ascontiguousarray(levels, np.float64)
        n = len(lv)
        lo, hi, fo = np.zeros(n), np.zeros(n), np.zeros(n)
        fe = np.zeros(n, np.uint8)
        rc = self.lib.ref_build_band_table(C.byref(prof), n, ptr(lv), t_slo, workers, max_batch,
                                           ptr(lo), ptr(hi), ptr(fo), ptr(fe))
        if rc != 0:
            raise ValueError("ModelError")
        return lo, hi, fo, fe.astype(bool)

    def tps_window(self, window_ms, t, tokens, now):
        t = np.ascontiguousarray(t, np.float64)
        k = np.ascontiguousarray(tokens, np.int32)
        return self.lib.ref_tps_window(window_ms, len(t), ptr(t), ptr(k), now)

    def tbt_p95(self, capacity, gaps):
        g = np.ascontiguousarray(gaps, np.float64)
        return self.lib.ref_tbt_window_p95(capacity, len(g), ptr(g))

    def replay_telemetry(self, cfg, table: _TableHolder, prof: Profile, worker, tel, t_end):
        ct = tel.c()
        cap = 1 << 14
        while True:
            out = np.zeros(cap, DECISION_DTYPE)
            n = self.lib.ref_replay_telemetry(C.byref(cfg), C.byref(table.c), prof.f_min_mhz,
                                              prof.f_max_mhz, prof.step_mhz, prof.f_ref_mhz,
                                              worker, C.byref(ct), t_end, ptr(out), cap)
            if n < 0:
                raise ValueError("ModelError")
            if n <= cap:
                return out[:n]
            cap = n

    def decode_script(self, cfg, table: _TableHolder, prof: Profile, worker, kind, t, value, has):
        """DecodeController on an explicit call script -> (records, command, bucket, f_opt)."""
        kind = np.ascontiguousarray(kind, np.int8)
        t = np.ascontiguousarray(t, np.float64)
        value = np.ascontiguousarray(value, np.float64)
        has = np.ascontiguousarray(has, np.uint8)
        out = np.zeros(max(1, len(kind)), DECISION_DTYPE)
        cmd = C.c_double()
        bucket = C.c_int32()
        f_opt = np.zeros(table.c.n, np.float64)
        n = self.lib.ref_decode_script(C.byref(cfg), C.byref(table.c), prof.f_min_mhz,
                                       prof.f_max_mhz, prof.step_mhz, prof.f_ref_mhz, worker,
                                       len(kind), ptr(kind), ptr(t), ptr(value), ptr(has),
                                       ptr(out), len(out), C.byref(cmd), C.byref(bucket),
                                       ptr(f_opt))
        if n < 0:
            raise ValueError("ModelError")
        return out[:n], cmd.value, bucket.value, f_opt

    def replay_many(self, cfgs, tables, table_of, tels, tel_of, worker_of, prof, t_end, threads=1):
        n = len(cfgs)
        carr = (CtlCfg * n)(*cfgs)
        tarr = (BandTable * len(tables))(*[t.c for t in tables])
        tl = (Telemetry * len(tels))(*[t.c() for t in tels])
        table_of = np.ascontiguousarray(table_of, np.int32)
        tel_of = np.ascontiguousarray(tel_of, np.int32)
        worker_of = np.ascontiguousarray(worker_of, np.int32)
        nrec = np.zeros(n, np.int64)
        dig = np.zeros(n, np.uint64)
        self.lib.ref_replay_many(n, C.cast(carr, _p), C.cast(tarr, _p), ptr(table_of),
                                 C.cast(tl, _p), ptr(tel_of), ptr(worker_of), prof.f_min_mhz,
                                 prof.f_max_mhz, prof.step_mhz, prof.f_ref_mhz, t_end, threads,
                                 ptr(nrec), ptr(dig))
        return nrec, dig

    def load_trace(self, path: str, class_threshold: int = 1024):
        """greensim::load_trace itself: same return convention as Restatement.trace_parse
        (without has_class)."""
        L = self.lib
        L.ref_load_trace.argtypes = [C.c_char_p, _i32, _i64, _p, _p, _p, _p, _p, C.c_char_p, _i64]
        L.ref_load_trace.restype = _i64
        cap = max(1, os.path.getsize(path) // 2 + 2)
        a = np.zeros(cap, np.int64)
        p = np.zeros(cap, np.int32)
        o = np.zeros(cap, np.int32)
        c = np.zeros(cap, np.uint8)
        kind = np.zeros(1, np.int32)
        msg = C.create_string_buffer(16384)
        n = L.ref_load_trace(path.encode(), class_threshold, cap, ptr(a), ptr(p), ptr(o), ptr(c),
                             ptr(kind), msg, 16384)
        if n < 0:
            m = msg.value.decode(errors="replace")
            row = None
            if m.startswith("row "):
                row = int(m[4:m.index(":")])
            elif TRACE_KINDS[kind[0]] == "BadHeader":
                row = 1
            return ("error", TRACE_KINDS[kind[0]], row, m)
        return a[:n], p[:n], o[:n], c[:n]

    def save_trace_csv(self, path: str, a, p, o, cls=None) -> bytes:
        """greensim::save_trace_csv, run by oracle/_ref/ref_save_trace in its own process."""
        import subprocess
        a = np.ascontiguousarray(a, np.int64)
        n = len(a)
        blob = (np.int64(n).tobytes() + a.tobytes() + np.ascontiguousarray(p, np.int32).tobytes()
                + np.ascontiguousarray(o, np.int32).tobytes()
                + bytes([0 if cls is None else 1])
                + (np.zeros(n, np.uint8) if cls is None
                   else np.ascontiguousarray(cls, np.uint8)).tobytes())
        with open(path + ".soa", "wb") as f:
            f.write(blob)
        subprocess.run([os.path.join(os.path.dirname(REF_SO), "ref_save_trace"), path + ".soa",
                        path], check=True)
        os.remove(path + ".soa")
        with open(path, "rb") as f:
            return f.read()

    def digest(self, recs):
        recs = np.ascontiguousarray(recs, DECISION_DTYPE)
        return int(self.lib.ref_digest_records(ptr(recs), len(recs)))

    def gen_poisson_trace(self, qps, duration_ms, short=512.0, long=4096.0, long_fraction=0.1,
                          output=128.0, seed=7):
        cap = int(qps * duration_ms / 1000.0 * 1.2 + 1000)
        a = np.zeros(cap, np.int64)
        p = np.zeros(cap, np.int32)
        o = np.zeros(cap, np.int32)
        n = self.lib.ref_gen_poisson_trace(qps, duration_ms, short, long, long_fraction, output,
                                           seed, cap, ptr(a), ptr(p), ptr(o))
        assert n <= cap
        return a[:n], p[:n], o[:n]

    def gen_sinusoid_decode_trace(self, mean, amp, period, duration_ms, seed):
        cap = int(duration_ms / 1000.0 * mean / 64 * 1.5 + 100)
        a = np.zeros(cap, np.int64)
        p = np.zeros(cap, np.int32)
        o = np.zeros(cap, np.int32)
        n = self.lib.ref_gen_sinusoid_decode_trace(mean, amp, period, duration_ms, seed, cap,
                                                   ptr(a), ptr(p), ptr(o))
        assert n <= cap
        return a[:n], p[:n], o[:n]

    def run_capture(self, arrival, prompt, output, prof, policy="greenllm", fixed_f=0.0,
                    thresholds=(1024,), worker_map=(0, 1), qcfg=None, ccfg=None):
        """Reference run() with the capture hooks; returns a dict of numpy arrays."""
        pol = {"defaultnv": 0, "fixed": 1, "greenllm": 2, "prefillsplit": 3}[policy]
        arrival = np.ascontiguousarray(arrival, np.int64)
        prompt = np.ascontiguousarray(prompt, np.int32)
        output = np.ascontiguousarray(output, np.int32)
        thr = np.ascontiguousarray(thresholds, np.int32)
        wm = np.ascontiguousarray(worker_map, np.int32)
        h = self.lib.ref_run_capture(len(arrival), ptr(arrival), ptr(prompt), ptr(output),
                                     C.byref(prof), pol, fixed_f, len(thr), ptr(thr), len(wm),
                                     ptr(wm), C.byref(qcfg) if qcfg else None,
                                     C.byref(ccfg) if ccfg else None)
        if not h:
            raise RuntimeError("reference run() threw")
        try:
            s = np.zeros(9, np.int64)
            self.lib.ref_run_sizes(h, ptr(s))
            ns, nj, nc, nf, nco, na, nd, nr = (int(x) for x in s[:8])
            out = {}
            out["snap_now"] = np.zeros(ns)
            out["snap_class"] = np.zeros(ns, np.int32)
            out["snap_off"] = np.zeros(ns + 1, np.int64)
            out["job_id"] = np.zeros(nj, np.int64)
            out["job_prompt"] = np.zeros(nj, np.int32)
            out["job_deadline"] = np.zeros(nj)
            out["job_wf"] = np.zeros(nj)
            self.lib.ref_run_snapshots(h, *(ptr(out[k]) for k in (
                "snap_now", "snap_class", "snap_off", "job_id", "job_prompt", "job_deadline",
                "job_wf")))
            out["cmd_now"] = np.zeros(nc)
            out["cmd_class"] = np.zeros(nc, np.int32)
            out["cmd_f"] = np.zeros(nc)
            out["cmd_window"] = np.zeros(nc)
            out["cmd_infeasible"] = np.zeros(nc, np.uint8)
            self.lib.ref_run_commands(h, *(ptr(out[k]) for k in (
                "cmd_now", "cmd_class", "cmd_f", "cmd_window", "cmd_infeasible")))
            out["fine_worker"] = np.zeros(nf, np.int32)
            out["fine_t"] = np.zeros(nf)
            out["fine_has"] = np.zeros(nf, np.uint8)
            out["fine_p95"] = np.zeros(nf)
            out["coarse_worker"] = np.zeros(nco, np.int32)
            out["coarse_t"] = np.zeros(nco)
            out["coarse_tps"] = np.zeros(nco)
            out["adapt_worker"] = np.zeros(na, np.int32)
            out["adapt_t"] = np.zeros(na)
            self.lib.ref_run_controller_inputs(h, *(ptr(out[k]) for k in (
                "fine_worker", "fine_t", "fine_has", "fine_p95", "coarse_worker", "coarse_t",
                "coarse_tps", "adapt_worker", "adapt_t")))
            out["decisions"] = np.zeros(nd, DECISION_DTYPE)
            self.lib.ref_run_decisions(h, ptr(out["decisions"]))
            out["decode_worker"] = np.zeros(nr, np.int32)
            out["prefill_start"] = np.zeros(nr)
            out["prefill_end"] = np.zeros(nr)
            out["first_token"] = np.zeros(nr)
            out["finish"] = np.zeros(nr)
            out["class_queue"] = np.zeros(nr, np.int32)
            out["completed"] = np.zeros(nr, np.uint8)
            out["energy"] = np.zeros(2)
            self.lib.ref_run_requests(h, *(ptr(out[k]) for k in (
                "decode_worker", "prefill_start", "prefill_end", "first_token", "finish",
                "class_queue", "completed", "energy")))
            return out
        finally:
            self.lib.ref_run_free(h)

    def sim_run(self, prof, policy: "PolicyHolder", slo, cfg, arrival, prompt, output, cls=None,
                scripted=None) -> dict:
        """The reference's own run() (simkernel.cpp) behind the gso_sim_* getters' layout."""
        arrival = np.ascontiguousarray(arrival, np.int64)
        prompt = np.ascontiguousarray(prompt, np.int32)
        output = np.ascontiguousarray(output, np.int32)
        cls = None if cls is None else np.ascontiguousarray(cls, np.int8)
        sc = None
        if scripted:
            sc = (Scripted * len(scripted))(*[Scripted(*x) for x in scripted])
        err = C.create_string_buffer(256)
        h = self.lib.ref_sim_run(C.byref(prof), C.byref(policy.c), C.byref(slo), C.byref(cfg),
                                 len(arrival), ptr(arrival), ptr(prompt), ptr(output), ptr(cls),
                                 len(scripted or ()), sc, err, 256)
        if not h:
            raise RuntimeError(err.value.decode())
        try:
            return _read_sim(self.lib, "ref_sim_", h)
        finally:
            self.lib.ref_sim_free(h)

    def sim_run_many(self, prof, policy: "PolicyHolder", cfgs, slo, sim_cfg, arrival, prompt,
                     output, threads=1):
        """One reference run() per controller config (CPU baseline of K5)."""
        arrival = np.ascontiguousarray(arrival, np.int64)
        prompt = np.ascontiguousarray(prompt, np.int32)
        output = np.ascontiguousarray(output, np.int32)
        arr = (CtlCfg * len(cfgs))(*cfgs)
        ej = np.zeros(len(cfgs))
        nd = np.zeros(len(cfgs), np.int64)
        self.lib.ref_sim_run_many(C.byref(prof), C.byref(policy.c), arr, len(cfgs), C.byref(slo),
                                  C.byref(sim_cfg), len(arrival), ptr(arrival), ptr(prompt),
                                  ptr(output), threads, ptr(ej), ptr(nd))
        return ej, nd


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def restatement_available() -> bool:
    return os.path.exists(RESTATE_SO)
