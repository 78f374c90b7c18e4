"""N > 1 with the REAL kernels: two processes share the GPU, each runs K1 + K2 (+ the summary)
on its window shard of ONE global trace (strong split, distributed.window_shard / trace_slice),
and the per-class summaries go through gsb_reduce_summaries with a torch.distributed (gloo)
all-gather as the transport callback. Both ranks must hold identical bytes, equal to the
single-process computation of the same shards combined by gsb_combine_summaries, and (counts,
argmin exact; energy within 1e-12) to one pass over the whole trace."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C_CLASSES, WMS, TOTAL_W = 8, 60_000, 3_001


def _trace():
    from paper_2508_16449_b200 import workloads as wl
    return wl.poisson_trace(5.0, TOTAL_W * WMS, "alibaba_chat", seed=21)


def _shard_summary(eng, a, p, w0, n):
    import torch
    from paper_2508_16449_b200 import api, distributed as D, workloads as wl
    lo, hi = D.trace_slice(a, WMS, w0, n)
    routing = api.RoutingConfig(True, wl.THRESHOLDS[C_CLASSES], list(range(C_CLASSES)))
    rr = eng.route_bin(torch.as_tensor(a[lo:hi], device="cuda"),
                       torch.as_tensor(p[lo:hi], device="cuda"), routing, WMS, w0, n)
    summ = eng.summary_buffer(C_CLASSES)
    eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=0.95 * WMS, summary_out=summ)
    torch.cuda.synchronize()
    return summ


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2508_16449_b200 import api, distributed as D, workloads as wl
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    eng = api.Engine(0, wl.synth_profiles(4))
    a, p, _ = _trace()
    w0, n = D.window_shard(TOTAL_W, world, rank)
    summ = _shard_summary(eng, a, p, w0, n)
    offsets = [D.window_shard(TOTAL_W, world, r)[0] * C_CLASSES for r in range(world)]
    glob = D.reduce_summaries(eng, summ, 4 * C_CLASSES, offsets)
    np.save(os.path.join(out_dir, f"glob{rank}.npy"), glob)
    eng.close()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_processes_real_kernels_reduce_summaries(gsb, tmp_path):
    import torch.multiprocessing as mp
    from paper_2508_16449_b200 import api, distributed as D, workloads as wl
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    g0, g1 = np.load(tmp_path / "glob0.npy"), np.load(tmp_path / "glob1.npy")
    assert g0.tobytes() == g1.tobytes()
    # the same shards in this process, combined by the C ABI: identical bytes
    gsb.set_profiles(wl.synth_profiles(4))
    a, p, _ = _trace()
    parts, offsets = [], []
    for r in range(world):
        w0, n = D.window_shard(TOTAL_W, world, r)
        s = _shard_summary(gsb, a, p, w0, n)
        parts.append(s.cpu().numpy().reshape(-1).view(D.SUMMARY_DTYPE))
        offsets.append(w0 * C_CLASSES)
    local = D.combine_summaries_c(np.stack(parts), offsets)
    assert local.tobytes() == g0.tobytes()
    # one pass over the whole trace: counts and argmin exact, energy within 1e-12
    whole = _shard_summary(gsb, a, p, 0, TOTAL_W).cpu().numpy().reshape(-1).view(D.SUMMARY_DTYPE)
    for k in ("n_cmd", "n_infeasible", "n_empty", "argmin_cell", "min_energy_j"):
        np.testing.assert_array_equal(g0[k], whole[k])
    np.testing.assert_allclose(g0["sum_energy_j"], whole["sum_energy_j"], rtol=1e-12)
    assert g0["n_cmd"].sum() > 10_000
