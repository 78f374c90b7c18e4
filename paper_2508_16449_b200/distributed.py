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
