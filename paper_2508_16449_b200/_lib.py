"""ctypes binding of libgsb.so (include/gsb.h). Fails loudly when the library is missing:
there is no CPU fallback anywhere in this package."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# GSB_LIB: another build of the same library (tools/ A/B timing of two kernel variants)
LIB_PATH = os.environ.get("GSB_LIB") or os.path.join(HERE, "lib", "libgsb.so")

_d, _i32, _i64, _u64, _p = C.c_double, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p

GSB_MAX_PROFILES = 4
GSB_MAX_GRID = 256
GSB_MAX_CLASSES = 8
GSB_MAX_BUCKETS = 32
GSB_MAX_TBT_WINDOW = 256

OK, MODEL_ERROR, ROUTER_ERROR, TRACE_ERROR, CUDA_ERROR, INVALID_ARGUMENT = range(6)
FIXED_WINDOW, DEADLINE_SLACK, PER_CELL_WINDOW = range(3)


TRACE_KINDS = ("EmptyTrace", "NonMonotoneArrivals", "MalformedRow", "BadHeader",
               "ClassMismatch", "BadShape")  # greensim::TraceError::Kind order


class CTraceResult(C.Structure):
    _fields_ = [("status", _i32), ("kind", _i32), ("detail", _i32), ("has_class", _i32),
                ("n_cols", _i32), ("line_len", _i32), ("line_truncated", _i32), ("pad_", _i32),
                ("row", _i64), ("n_rows", _i64), ("max_arrival_ms", _i64),
                ("line", C.c_char * 1024)]


class CCellList(C.Structure):
    """gsb_cell_list (include/gsb.h)."""
    _fields_ = [("d_cells", _p), ("d_n", _p), ("d_t_ref", _p), ("d_min_deadline", _p),
                ("capacity", _i64)]


class CRunningJobs(C.Structure):
    """gsb_running_jobs (include/gsb.h)."""
    _fields_ = [("d_running", _p), ("d_remaining_ref_ms", _p), ("d_updated_ms", _p),
                ("d_freq_mhz", _p), ("d_t_ref_ms", _p)]


class CProfile(C.Structure):
    _fields_ = [(n, _d) for n in (
        "f_min_mhz", "f_max_mhz", "step_mhz", "f_ref_mhz",
        "lat_a", "lat_b", "lat_c", "lat_f_ref_mhz",
        "dec_alpha0_ms", "dec_alpha1_ms", "dec_beta0_ms", "dec_beta1_ms", "dec_f_ref_mhz",
        "k3", "k2", "k1", "k0", "p_idle_w")]


class CQoptCfg(C.Structure):
    _fields_ = [("resolve_period_ms", _d), ("margin_prefill", _d), ("min_budget_ms", _d),
                ("first_token_allowance_ms", _d)]


class CCtlCfg(C.Structure):
    _fields_ = [("tslo_ms", _d), ("margin_decode", _d), ("fine_period_ms", _d),
                ("coarse_period_ms", _d), ("adapt_period_s", _d), ("step_mhz", _d),
                ("max_step_mhz", _d), ("hysteresis_count", _i32), ("tbt_window_tokens", _i32),
                ("bias_threshold", _d), ("tps_scale", _d), ("upper_margin", _d),
                ("lower_margin", _d)]


class CRouteCfg(C.Structure):
    _fields_ = [("n_thresholds", _i32), ("thresholds", _i32 * (GSB_MAX_CLASSES - 1)),
                ("enabled", _i32), ("slo_boundary_tokens", _i32), ("window_ms", _i64),
                ("w0", _i64), ("n_windows", _i64), ("ttft_sm_ms", _d), ("ttft_l_ms", _d),
                ("first_token_allowance_ms", _d)]


class CSelectCfg(C.Structure):
    _fields_ = [("mode", _i32), ("n_classes", _i32), ("fixed_window_ms", _d), ("w0", _i64),
                ("window_ms", _i64), ("qopt", CQoptCfg)]


class CClassSummary(C.Structure):
    _fields_ = [("n_cmd", _i64), ("n_infeasible", _i64), ("n_empty", _i64),
                ("sum_energy_j", _d), ("min_energy_j", _d), ("argmin_cell", _i64)]


class CTelemetry(C.Structure):
    _fields_ = [("n_streams", _i64), ("d_ev_off", _p), ("d_t_ms", _p), ("d_tokens", _p),
                ("d_gap_off", _p), ("d_gaps", _p)]


class CReplayArgs(C.Structure):
    _fields_ = [("n_traj", _i64), ("d_cfg", _p), ("d_table_of", _p), ("d_stream_of", _p),
                ("d_worker", _p), ("n_buckets", _i32), ("d_tps_hi", _p), ("d_f_opt", _p),
                ("f_min_mhz", _d), ("f_max_mhz", _d), ("fine_period_ms", _d),
                ("coarse_period_ms", _d), ("t_end_ms", _d), ("d_fine_has", _p),
                ("d_fine_p95", _p), ("d_coarse_tps", _p), ("d_digest", _p), ("d_n_rec", _p),
                ("d_counts", _p), ("d_mean_cmd", _p), ("d_records", _p), ("rec_cap", _i64)]


class CCtlState(C.Structure):
    _fields_ = [("band_lo", _d), ("band_hi", _d), ("set_point", _d), ("last_tps", _d),
                ("last_p95", _d), ("current_bucket", _i32), ("pending_bucket", _i32),
                ("consecutive", _i32), ("adj_total", _i32), ("adj_up", _i32), ("adj_down", _i32),
                ("initialized", _i32), ("pad_", _i32), ("f_opt", _d * 32)]


class CPoolCfg(C.Structure):
    _fields_ = [("n_decode_workers", _i32), ("max_batch", _i32), ("max_queue", _i32),
                ("tbt_cap", _i32), ("tps_cap", _i32), ("pending_cap", _i32),
                ("actuation_delay_ms", _d), ("tbt_p95_ms", _d)]


class CPoolStream(C.Structure):
    _fields_ = [("n_streams", _i64), ("d_off", _p), ("d_t_ms", _p), ("d_req", _p),
                ("d_end_floor_ms", _p), ("n_requests", _i64), ("d_output_tokens", _p),
                ("d_arrival_ms", _p), ("d_ttft_slo_ms", _p)]


class CPoolSummary(C.Structure):
    _fields_ = [("decode_pool_j", _d), ("active_decode_j", _d), ("idle_j", _d),
                ("sim_end_ms", _d), ("n_completed", _i64), ("n_rejected", _i64),
                ("n_ttft_ok", _i64), ("n_tbt_ok", _i64), ("tbt_samples", _i64),
                ("tbt_samples_ok", _i64), ("n_decisions", _i64), ("n_freq_changes", _i64),
                ("n_steps", _i64), ("decision_digest", _u64), ("freq_digest", _u64),
                ("request_digest", _u64), ("status", _i32), ("pad_", _i32)]


class CPoolArgs(C.Structure):
    _fields_ = [("n_scen", _i64), ("d_cfg", _p), ("d_fixed_mhz", _p), ("d_table_of", _p),
                ("d_stream_of", _p), ("n_buckets", _i32), ("d_tps_hi", _p), ("d_f_opt", _p),
                ("d_out", _p), ("d_ledger", _p), ("d_records", _p), ("rec_cap", _i64),
                ("d_freq", _p), ("freq_cap", _i64), ("d_req_worker", _p), ("d_req_first", _p),
                ("d_req_finish", _p)]


# every symbol include/gsb.h declares (checked by tests/test_boundary.py)
EXPORTS = (
    "gsb_version", "gsb_status_string", "gsb_ctx_create", "gsb_ctx_destroy", "gsb_last_error",
    "gsb_ctx_stream", "gsb_synchronize", "gsb_profile_validate", "gsb_ctl_cfg_validate",
    "gsb_set_profiles", "gsb_routing_validate", "gsb_window_bounds", "gsb_route_bin",
    "gsb_fifo_order", "gsb_prefill_select", "gsb_select_batches", "gsb_energy_batches",
    "gsb_prefill_summary", "gsb_n_ticks", "gsb_window_series", "gsb_build_band_tables",
    "gsb_decode_replay", "gsb_replay_validate", "gsb_fp64_probe", "gsb_selftest_division",
    "gsb_decode_script", "gsb_quantile_batch", "gsb_tps_window_batch", "gsb_steady_state_batch",
    "gsb_set_profiles_ex", "gsb_malloc", "gsb_free", "gsb_host_alloc", "gsb_host_free",
    "gsb_memcpy", "gsb_classify",
    "gsb_t_ref_batches", "gsb_energy_closed_form_batches",
    "gsb_decode_pool", "gsb_decode_pool_tps_cap", "gsb_prefill_select_summary",
    "gsb_trace_parse", "gsb_trace_format", "gsb_route_bin_list", "gsb_prefill_select_list",
    "gsb_prefill_pass", "gsb_prefill_pass_host", "gsb_select_batches_running", "gsb_freq_timeline_csv",
    "gsb_prefill_commands_csv", "gsb_format_g10", "gsb_mg1_side_output",
    "gsb_decision_log_csv", "gsb_format_g",
    "gsb_combine_summaries", "gsb_reduce_summaries", "gsb_tally_pool", "gsb_combine_tallies",
    "gsb_reduce_tallies",
)

# gsb_allgather_fn: int (*)(const void* d_send, void* d_recv, size_t bytes, void* stream, void* user)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libgsb.so once and declare every prototype. Raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build the sm_100a library first "
                          f"(python -c 'import __graft_entry__ as g; g.build()')")
    L = C.CDLL(path)
    P = C.POINTER
    L.gsb_version.restype = C.c_char_p
    L.gsb_status_string.argtypes = [C.c_int]
    L.gsb_status_string.restype = C.c_char_p
    L.gsb_ctx_create.argtypes = [C.c_int, P(_p)]
    L.gsb_ctx_destroy.argtypes = [_p]
    L.gsb_ctx_destroy.restype = None
    L.gsb_last_error.argtypes = [_p]
    L.gsb_last_error.restype = C.c_char_p
    L.gsb_ctx_stream.argtypes = [_p]
    L.gsb_ctx_stream.restype = _p
    L.gsb_synchronize.argtypes = [_p]
    L.gsb_profile_validate.argtypes = [P(CProfile), C.c_char_p, C.c_size_t]
    L.gsb_ctl_cfg_validate.argtypes = [P(CCtlCfg), C.c_char_p, C.c_size_t]
    L.gsb_set_profiles.argtypes = [_p, C.c_int, _p]
    L.gsb_routing_validate.argtypes = [P(CRouteCfg), C.c_int, _p, C.c_char_p, C.c_size_t]
    L.gsb_window_bounds.argtypes = [_p, P(CRouteCfg), _i64, _p, _p, _p]
    L.gsb_route_bin.argtypes = [_p, P(CRouteCfg), _i64, _p, _p, _p, _p, _p, _p, _p, _p]
    L.gsb_fifo_order.argtypes = [_p, P(CRouteCfg), _i64, _p, _p, _p, _p, _p, _p]
    L.gsb_prefill_select.argtypes = [_p, P(CSelectCfg), _i64, _p, _p, _p, _p, _p, _p, _p]
    L.gsb_select_batches.argtypes = [_p, P(CSelectCfg), C.c_int, _i64, _p, _p, _p, _p, _p, _p,
                                     _p, _p, _p, _p]
    L.gsb_energy_batches.argtypes = [_p, C.c_int, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]
    L.gsb_prefill_summary.argtypes = [_p, C.c_int, C.c_int, _i64, _p, _p, _p, _p]
    L.gsb_prefill_select_summary.argtypes = [_p, P(CSelectCfg), _i64, _p, _p, _p, _p, _p, _p,
                                             _p, _p]
    L.gsb_route_bin_list.argtypes = [_p, P(CRouteCfg), _i64, _p, _p, _p, _p, _p, _p, _p,
                                     P(CCellList), _p]
    L.gsb_prefill_select_list.argtypes = [_p, P(CSelectCfg), _i64, _p, _p, P(CCellList), _p, _p,
                                          _p, _p, _p, _p]
    L.gsb_select_batches_running.argtypes = [_p, P(CSelectCfg), C.c_int, _i64, _p, _p, _p,
                                             P(CRunningJobs), _p, _p, _p, _p, _p, _p, _p]
    L.gsb_freq_timeline_csv.argtypes = [_p, _i64, _p, _p, _p, _p, _p, _i64, P(_i64), _p]
    L.gsb_prefill_commands_csv.argtypes = [_p, _i64, _p, _p, _p, _p, _p, _p, _p, _i64, P(_i64),
                                           _p]
    L.gsb_format_g10.argtypes = [_p, _i64, _p, _p, _p, _p]
    L.gsb_format_g.argtypes = [_p, _i32, _i64, _p, _p, _p, _p]
    L.gsb_decision_log_csv.argtypes = [_p, _i64, _p, _p, _i64, P(_i64), _p]
    L.gsb_combine_summaries.argtypes = [C.c_int, C.c_int, _p, _p, _p]
    L.gsb_reduce_summaries.argtypes = [_p, C.c_int, C.c_int, C.c_int, _p, _p, ALLGATHER_FN, _p,
                                       _p, _p]
    L.gsb_tally_pool.argtypes = [_i64, _p, _i64, _p]
    L.gsb_combine_tallies.argtypes = [C.c_int, _p, _p]
    L.gsb_reduce_tallies.argtypes = [_p, C.c_int, C.c_int, _p, ALLGATHER_FN, _p, _p, _p]
    L.gsb_mg1_side_output.argtypes = [_p, C.c_int, _i64, _d, _p, _p, _p, _p, _p, _p, _p, _p, _p]
    L.gsb_prefill_pass.argtypes = [_p, P(CRouteCfg), _i64, _p, _p, _p, _p, _p, _p, _p,
                                   P(CCellList), P(CSelectCfg), _p, _p, _p, _p, _p]
    L.gsb_prefill_pass_host.argtypes = [_p, P(CRouteCfg), _i64, _p, _p, P(CSelectCfg), C.c_int,
                                        _p, _p, _p, _p]
    L.gsb_n_ticks.argtypes = [_d, _d]
    L.gsb_n_ticks.restype = _i64
    L.gsb_window_series.argtypes = [_p, P(CTelemetry), C.c_int, _d, _d, _d, _p, _p, _p, _p]
    L.gsb_build_band_tables.argtypes = [_p, _i64, _p, _p, _p, _p, _p, C.c_int, _p, _p, _p, _p,
                                        _p, _p]
    L.gsb_decode_replay.argtypes = [_p, P(CReplayArgs), _p]
    L.gsb_replay_validate.argtypes = [_p, _i64, _i32, _p, _p, _i64, C.c_char_p, C.c_size_t]
    L.gsb_fp64_probe.argtypes = [_p, _i64, C.c_int, _p, _p]
    L.gsb_selftest_division.argtypes = [_p, _i64, _u64, _p, _p]
    L.gsb_decode_script.argtypes = [_p, P(CReplayArgs), _p, _p, _p, _p, _p, _p, _p]
    L.gsb_quantile_batch.argtypes = [_p, _d, _i64, _p, _p, _p, _p]
    L.gsb_tps_window_batch.argtypes = [_p, _i64, _p, _p, _p, _p, _p, _p, _p]
    L.gsb_steady_state_batch.argtypes = [_p, _i64, _p, _p, _p, _p, _p, _p, _p, _p]
    L.gsb_set_profiles_ex.argtypes = [_p, C.c_int, _p, C.c_int]
    L.gsb_malloc.argtypes = [_p, C.c_size_t, P(_p)]
    L.gsb_free.argtypes = [_p, _p]
    L.gsb_host_alloc.argtypes = [_p, C.c_size_t, P(_p)]
    L.gsb_host_free.argtypes = [_p, _p]
    L.gsb_memcpy.argtypes = [_p, _p, _p, C.c_size_t, C.c_int, _p]
    L.gsb_classify.argtypes = [_p, C.c_int, _p, _i64, _p, _p, _p]
    L.gsb_t_ref_batches.argtypes = [_p, P(_d), _i64, _p, _p, _p, _p, _p]
    L.gsb_energy_closed_form_batches.argtypes = [_p, C.c_int, _i64, _p, _p, _p, _p, _p, _p, _p]
    L.gsb_decode_pool_tps_cap.argtypes = [P(CProfile), _i32, _d]
    L.gsb_trace_parse.argtypes = [_p, _p, _i64, _i32, _i64, _p, _p, _p, _p, P(CTraceResult), _p]
    L.gsb_trace_format.argtypes = [_p, _i64, _p, _p, _p, _p, _p, _i64, P(_i64), _p]
    L.gsb_decode_pool.argtypes = [_p, P(CProfile), P(CPoolCfg), P(CPoolStream), P(CPoolArgs), _p]
    _lib = L
    return L
