"""Multi-GPU plumbing for the decision engine.

The path shards without any data-path exchange: windows (and their requests) and decode
scenarios are split into contiguous per-rank ranges. The only collective is the end-of-step
all-gather of the per-(profile, class) summaries produced by `gsb_prefill_summary`; every
rank then combines the gathered records in RANK ORDER, so the global result is bitwise
identical on every rank (an fp64 all-reduce would depend on the reduction tree).
"""
from __future__ import annotations

import numpy as np

SUMMARY_DTYPE = np.dtype([("n_cmd", "<i8"), ("n_infeasible", "<i8"), ("n_empty", "<i8"),
                          ("sum_energy_j", "<f8"), ("min_energy_j", "<f8"),
                          ("argmin_cell", "<i8")])


def window_shard(total_windows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous window range (w0, n) of `rank` for strong scaling (balanced to +-1)."""
    base, extra = divmod(total_windows, world)
    n = base + (1 if rank < extra else 0)
    w0 = rank * base + min(rank, extra)
    return w0, n


def trace_slice(arrival: np.ndarray, window_ms: int, w0: int, n_windows: int) -> tuple[int, int]:
    """Request index range of windows [w0, w0+n) in a non-decreasing arrival array."""
    lo = int(np.searchsorted(arrival, w0 * window_ms, side="left"))
    hi = int(np.searchsorted(arrival, (w0 + n_windows) * window_ms, side="left"))
    return lo, hi


def scenario_shard(total: int, world: int, rank: int) -> tuple[int, int]:
    return window_shard(total, world, rank)


def gather_summaries(summary_bytes, group=None):
    """All-gather the [P*C, 48] byte summaries of every rank (NCCL on GPU tensors, gloo on
    CPU tensors). Returns a [world, P*C, 48] tensor on the input's device."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(summary_bytes.shape), dtype=summary_bytes.dtype,
                      device=summary_bytes.device)
    try:
        dist.all_gather_into_tensor(out, summary_bytes.contiguous(), group=group)
    except (RuntimeError, NotImplementedError):  # backends without the fused collective
        parts = [torch.empty_like(summary_bytes) for _ in range(world)]
        dist.all_gather(parts, summary_bytes.contiguous(), group=group)
        out = torch.stack(parts)
    return out


def combine_summaries(per_rank: np.ndarray, cell_offsets) -> np.ndarray:
    """Combine per-rank summaries [R, P, C] (SUMMARY_DTYPE) in rank order.

    Counts add exactly; energies are folded left to right over ranks (deterministic); the
    argmin is the lexicographic minimum of (energy, global cell) where global cell =
    cell_offsets[r] + local cell (ties -> lowest global cell, i.e. the earliest window)."""
    per_rank = np.asarray(per_rank)
    R = per_rank.shape[0]
    out = np.zeros(per_rank.shape[1:], SUMMARY_DTYPE)
    out["min_energy_j"] = np.inf
    out["argmin_cell"] = -1
    for r in range(R):
        s = per_rank[r]
        out["n_cmd"] += s["n_cmd"]
        out["n_infeasible"] += s["n_infeasible"]
        out["n_empty"] += s["n_empty"]
        out["sum_energy_j"] = out["sum_energy_j"] + s["sum_energy_j"]
        has = s["argmin_cell"] >= 0
        g_cell = np.where(has, s["argmin_cell"] + int(cell_offsets[r]), -1)
        better = has & ((out["argmin_cell"] < 0) | (s["min_energy_j"] < out["min_energy_j"])
                        | ((s["min_energy_j"] == out["min_energy_j"]) & (g_cell < out["argmin_cell"])))
        out["min_energy_j"] = np.where(better, s["min_energy_j"], out["min_energy_j"])
        out["argmin_cell"] = np.where(better, g_cell, out["argmin_cell"])
    return out


# ------------------------------------------------------------------ decode pool (K5) tallies
# The end-of-run decode reductions of SURVEY.md 8(e) item 4: per rank, the per-scenario
# gsb_pool_summary records (energy, SLO counts, trajectory digests) are folded in scenario
# order into one DECODE_TALLY record; the records of all ranks are all-gathered (NCCL) and
# combined in rank order, so every rank holds the same bytes.
DECODE_TALLY_DTYPE = np.dtype([
    ("n_scenarios", "<i8"), ("decode_pool_j", "<f8"), ("min_decode_pool_j", "<f8"),
    ("argmin_scenario", "<i8"), ("n_completed", "<i8"), ("n_rejected", "<i8"),
    ("n_ttft_ok", "<i8"), ("n_tbt_ok", "<i8"), ("tbt_samples", "<i8"),
    ("tbt_samples_ok", "<i8"), ("n_decisions", "<i8"), ("n_freq_changes", "<i8"),
    ("digest", "<u8")])
_COUNTS = ("n_completed", "n_rejected", "n_ttft_ok", "n_tbt_ok", "tbt_samples",
           "tbt_samples_ok", "n_decisions", "n_freq_changes")
_M64 = (1 << 64) - 1


def _mix64(x: int) -> int:  # splitmix64 finaliser
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def tally_pool(summary: np.ndarray, scen0: int) -> np.ndarray:
    """Fold the per-scenario pool summaries of global scenarios [scen0, scen0 + N) in order.
    digest = sum over scenarios of mix(decision ^ freq ^ request digest ^ global index)
    (mod 2^64): independent of how the scenarios are split over ranks."""
    out = np.zeros(1, DECODE_TALLY_DTYPE)[0]
    out["n_scenarios"] = len(summary)
    out["min_decode_pool_j"] = np.inf
    out["argmin_scenario"] = -1
    e = 0.0
    dig = 0
    for i, s in enumerate(summary):
        x = float(s["decode_pool_j"])
        e = e + x
        if x < out["min_decode_pool_j"]:
            out["min_decode_pool_j"] = x
            out["argmin_scenario"] = scen0 + i
        d = int(s["decision_digest"]) ^ int(s["freq_digest"]) ^ int(s["request_digest"])
        dig = (dig + _mix64(d ^ (scen0 + i))) & _M64
    out["decode_pool_j"] = e
    for k in _COUNTS:
        out[k] = int(summary[k].sum())
    out["digest"] = dig
    return out


def combine_tallies(per_rank: np.ndarray) -> np.ndarray:
    """Rank-order combine of [R] DECODE_TALLY records (ranks hold consecutive scenario ranges):
    counts and digests add exactly, energies fold left to right, the argmin keeps the lowest
    energy, then the lowest global scenario."""
    per_rank = np.asarray(per_rank, DECODE_TALLY_DTYPE)
    out = np.zeros(1, DECODE_TALLY_DTYPE)[0]
    out["min_decode_pool_j"] = np.inf
    out["argmin_scenario"] = -1
    e = 0.0
    dig = 0
    for s in per_rank:
        out["n_scenarios"] += s["n_scenarios"]
        e = e + float(s["decode_pool_j"])
        if s["argmin_scenario"] >= 0 and (
                out["argmin_scenario"] < 0 or s["min_decode_pool_j"] < out["min_decode_pool_j"]):
            out["min_decode_pool_j"] = s["min_decode_pool_j"]
            out["argmin_scenario"] = s["argmin_scenario"]
        dig = (dig + int(s["digest"])) & _M64
        for k in _COUNTS:
            out[k] += s[k]
    out["decode_pool_j"] = e
    out["digest"] = dig
    return out


def gather_records(rec: np.ndarray, device, group=None) -> np.ndarray:
    """All-gather one numpy record per rank (as bytes) and return the [world] records."""
    import torch
    t = torch.from_numpy(np.frombuffer(rec.tobytes(), np.uint8).copy()).to(device)
    g = gather_summaries(t, group)
    return g.cpu().numpy().reshape(g.shape[0], -1).view(rec.dtype).reshape(-1)


# ------------------------------------------------------------------ the C-ABI reductions
# gsb_combine_summaries / gsb_tally_pool / gsb_combine_tallies (host C, no device needed) and
# gsb_reduce_summaries / gsb_reduce_tallies with a torch.distributed all-gather as the
# transport callback (NCCL on GPU tensors, gloo otherwise): the same rank-order combine a C++
# host runs with ncclAllGather.
def _lib():
    from . import _lib as L
    return L.load()


def combine_summaries_c(per_rank: np.ndarray, cell_offsets) -> np.ndarray:
    """gsb_combine_summaries over [R, N] SUMMARY_DTYPE records."""
    import ctypes as C
    pr = np.ascontiguousarray(per_rank, SUMMARY_DTYPE).reshape(per_rank.shape[0], -1)
    off = np.ascontiguousarray(cell_offsets, np.int64)
    out = np.zeros(pr.shape[1], SUMMARY_DTYPE)
    rc = _lib().gsb_combine_summaries(pr.shape[0], pr.shape[1], pr.ctypes.data_as(C.c_void_p),
                                      off.ctypes.data_as(C.c_void_p),
                                      out.ctypes.data_as(C.c_void_p))
    assert rc == 0, rc
    return out.reshape(per_rank.shape[1:])


def tally_pool_c(summary: np.ndarray, scen0: int) -> np.ndarray:
    """gsb_tally_pool over POOL_SUMMARY_DTYPE records."""
    import ctypes as C
    sm = np.ascontiguousarray(summary)
    out = np.zeros(1, DECODE_TALLY_DTYPE)
    rc = _lib().gsb_tally_pool(len(sm), sm.ctypes.data_as(C.c_void_p), int(scen0),
                               out.ctypes.data_as(C.c_void_p))
    assert rc == 0, rc
    return out[0]


def combine_tallies_c(per_rank: np.ndarray) -> np.ndarray:
    import ctypes as C
    pr = np.ascontiguousarray(per_rank, DECODE_TALLY_DTYPE)
    out = np.zeros(1, DECODE_TALLY_DTYPE)
    rc = _lib().gsb_combine_tallies(len(pr), pr.ctypes.data_as(C.c_void_p),
                                    out.ctypes.data_as(C.c_void_p))
    assert rc == 0, rc
    return out[0]


def torch_allgather_callback(engine, group=None):
    """A gsb_allgather_fn that moves the bytes through torch.distributed (device staging via
    gsb_memcpy, all_gather on tensors of the group's backend). Keep the returned object alive
    while the library may call it."""
    import ctypes as C
    import torch
    import torch.distributed as dist
    from . import _lib as L

    lib = engine.lib
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

    def cb(d_send, d_recv, nbytes, stream, user):
        try:
            world = dist.get_world_size(group)
            lib.gsb_synchronize(engine.ctx)
            torch.cuda.synchronize()
            mine = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            host = torch.empty(nbytes, dtype=torch.uint8)
            if lib.gsb_memcpy(engine.ctx, host.data_ptr(), d_send, nbytes, 1, None) != 0:
                return 1
            lib.gsb_synchronize(engine.ctx)
            mine.copy_(host)
            out = torch.empty(world * nbytes, dtype=torch.uint8, device=dev)
            dist.all_gather_into_tensor(out, mine, group=group)
            outh = out.cpu()
            if lib.gsb_memcpy(engine.ctx, d_recv, outh.data_ptr(), world * nbytes, 0, None) != 0:
                return 1
            lib.gsb_synchronize(engine.ctx)
            return 0
        except Exception:  # noqa: BLE001 - reported to the library as a failed transport
            return 1

    return L.ALLGATHER_FN(cb)


def reduce_summaries(engine, summary_dev, n_records: int, cell_offsets, group=None) -> np.ndarray:
    """gsb_reduce_summaries: this rank's device summaries -> the global records (host)."""
    import ctypes as C
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    off = np.ascontiguousarray(cell_offsets, np.int64)
    out = np.zeros(n_records, SUMMARY_DTYPE)
    cb = torch_allgather_callback(engine, group)
    engine._check(engine.lib.gsb_reduce_summaries(
        engine.ctx, world, rank, n_records, summary_dev.data_ptr(), off.ctypes.data_as(C.c_void_p),
        cb, None, out.ctypes.data_as(C.c_void_p), None))
    return out
