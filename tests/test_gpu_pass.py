"""The fused prefill pass (gsb_prefill_pass: K1b and K2 in one persistent kernel) against the
two-call path (gsb_route_bin_list + gsb_prefill_select_list) and, at the C4 shape, against the
unmodified reference: every output bit for bit, over shapes that exercise the tile / chunk
hand-off (partial last chunk, empty windows, one profile, eight classes, routing off, deadline
mode), repeated passes (the counters and epochs) and a captured CUDA graph replay."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _cmp_pass(gsb, a, p, routing, wms, nW, mode, **kw):
    from paper_2508_16449_b200 import api
    da, dp = torch.as_tensor(a, device="cuda"), torch.as_tensor(p, device="cuda")
    C = routing.n_classes() if routing.enabled else 1
    want_dl = mode == api.L.DEADLINE_SLACK
    rr1 = gsb.route_bin(da, dp, routing, wms, 0, nW, want_deadline=want_dl)
    s1 = gsb.summary_buffer(C)
    sel1 = gsb.prefill_select(rr1, mode, summary_out=s1, **kw)
    s2 = gsb.summary_buffer(C)
    rr2, sel2 = gsb.prefill_pass(da, dp, routing, wms, 0, nW, mode, summary_out=s2, **kw)
    torch.cuda.synchronize()
    for f in ("bounds", "cls", "count", "t_ref"):
        assert torch.equal(getattr(rr1, f), getattr(rr2, f)), f
    if want_dl:
        assert torch.equal(rr1.min_deadline.view(torch.int64), rr2.min_deadline.view(torch.int64))
    n1, n2 = int(rr1.n_nonempty.item()), int(rr2.n_nonempty.item())
    assert n1 == n2
    assert torch.equal(rr1.nonempty[:n1], rr2.nonempty[:n2])
    assert torch.equal(sel1.f_idx, sel2.f_idx)
    assert torch.equal(sel1.energy_j.view(torch.int64), sel2.energy_j.view(torch.int64))
    live = rr1.count.view(torch.int32) != 0
    assert torch.equal(sel1.window_ms[live].view(torch.int64), sel2.window_ms[live].view(torch.int64))
    assert torch.equal(s1, s2)
    return rr2, sel2


@pytest.mark.parametrize("C,P,qps,minutes", [
    (8, 4, 5.0, 2000),      # C4 shape, 2000 windows
    (3, 1, 5.0, 600),       # one profile (8-window tiles)
    (5, 2, 0.05, 3000),     # sparse: most windows empty, partial last chunk
    (8, 3, 40.0, 120),      # dense windows: tiles span several staging chunks
    (2, 4, 1.0, 7),         # fewer windows than one tile, a single partial chunk
])
def test_pass_equals_two_call_path(gsb, C, P, qps, minutes):
    from paper_2508_16449_b200 import api, workloads as wl
    gsb.set_profiles(wl.synth_profiles(P))
    a, p, _ = wl.poisson_trace(qps, minutes * 60_000, "alibaba_chat", seed=C * 10 + P)
    thr = wl.THRESHOLDS.get(C, [512] if C == 2 else wl.THRESHOLDS[3])
    routing = api.RoutingConfig(True, thr, list(range(len(thr) + 1)))
    for _ in range(3):  # repeated passes: tickets, readiness counters and look-back epochs
        _cmp_pass(gsb, a, p, routing, 60_000, minutes, api.L.FIXED_WINDOW,
                  fixed_window_ms=0.95 * 60_000)


def test_pass_deadline_mode_and_routing_off(gsb):
    from paper_2508_16449_b200 import api, workloads as wl
    gsb.set_profiles(wl.synth_profiles(4))
    a, p, _ = wl.poisson_trace(5.0, 500 * 60_000, "alibaba_chat", seed=3)
    routing = api.RoutingConfig(True, wl.THRESHOLDS[8], list(range(8)))
    _cmp_pass(gsb, a, p, routing, 60_000, 500, api.L.DEADLINE_SLACK,
              qopt=api.QueueOptimizerConfig())
    off = api.RoutingConfig(False, [1024], [0])
    _cmp_pass(gsb, a, p, off, 60_000, 500, api.L.FIXED_WINDOW, fixed_window_ms=57_000.0)


def test_pass_c4_matches_reference_and_replays_in_a_graph(gsb, ref):
    """The bench's C4 step through the fused pass: every cell and profile equals the unmodified
    reference (Dispatcher + select_frequency), and a captured graph replays to the same bytes."""
    from paper_2508_16449_b200 import api, workloads as wl
    from oracle import oracle as O
    profs = wl.synth_profiles(4)
    gsb.set_profiles(profs)
    C, nW, wms = 8, 10_000, 60_000
    a, p, _ = wl.poisson_trace(5.0, nW * wms, "alibaba_chat", seed=1000, t0_ms=0)
    routing = api.RoutingConfig(True, wl.THRESHOLDS[C], list(range(C)))
    da, dp = torch.as_tensor(a, device="cuda"), torch.as_tensor(p, device="cuda")
    summ = gsb.summary_buffer(C)
    rr, sel = gsb.prefill_pass(da, dp, routing, wms, 0, nW, api.L.FIXED_WINDOW,
                               fixed_window_ms=0.95 * wms, summary_out=summ)
    torch.cuda.synchronize()
    fi_r, en_r, _ = ref.prefill_pass([O.Profile(*x.key()) for x in profs], wl.THRESHOLDS[C], a, p,
                                     wms, 0, nW, 0.95 * wms, threads=os.cpu_count() or 1)
    np.testing.assert_array_equal(sel.f_idx.cpu().numpy(), fi_r)
    np.testing.assert_array_equal(u64(sel.energy_j.cpu().numpy()), u64(en_r))
    f0, e0, s0 = sel.f_idx.clone(), sel.energy_j.clone(), summ.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        gsb.prefill_pass(da, dp, routing, wms, 0, nW, api.L.FIXED_WINDOW,
                         fixed_window_ms=0.95 * wms, rr=rr, sel=sel, summary_out=summ)
    for _ in range(3):
        sel.f_idx.fill_(7)
        summ.fill_(0)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(sel.f_idx, f0)
        assert torch.equal(sel.energy_j.view(torch.int64), e0.view(torch.int64))
        assert torch.equal(summ, s0)


def _cmp_host_pass(gsb, a, p, routing, wms, w0, nW, mode, chunks, **kw):
    """prefill_pass_host (pinned host in, host out, chunked pipeline) against the device pass:
    f_idx / energy bit for bit; the combined chunk summaries: counts and argmin exact, the
    energy sum (folded chunk by chunk instead of one tree) to 1e-12."""
    from paper_2508_16449_b200 import api
    C = routing.n_classes() if routing.enabled else 1
    da, dp = torch.as_tensor(a, device="cuda"), torch.as_tensor(p, device="cuda")
    s1 = gsb.summary_buffer(C)
    _, sel = gsb.prefill_pass(da, dp, routing, wms, w0, nW, mode, summary_out=s1, **kw)
    ha, hp = torch.as_tensor(a).pin_memory(), torch.as_tensor(p).pin_memory()
    res = gsb.prefill_pass_host(ha, hp, routing, wms, w0, nW, mode, chunks=chunks, **kw)
    torch.cuda.synchronize()
    assert torch.equal(sel.f_idx.cpu(), res.f_idx)
    assert torch.equal(sel.energy_j.cpu().view(torch.int64), res.energy_j.view(torch.int64))
    want = np.frombuffer(s1.cpu().numpy().tobytes(), gsb.SUMMARY_DTYPE)
    got = res.summary().reshape(-1)
    for f in ("n_cmd", "n_infeasible", "n_empty", "argmin_cell"):
        assert np.array_equal(want[f], got[f]), f
    assert np.array_equal(u64(want["min_energy_j"]), u64(got["min_energy_j"]))
    np.testing.assert_allclose(got["sum_energy_j"], want["sum_energy_j"], rtol=1e-12, atol=0)
    return res


@pytest.mark.parametrize("chunks", [1, 3, 4, 7])
def test_host_pass_equals_device_pass(gsb, chunks):
    from paper_2508_16449_b200 import api, workloads as wl
    gsb.set_profiles(wl.synth_profiles(4))
    a, p, _ = wl.poisson_trace(5.0, 1000 * 60_000, "alibaba_chat", seed=21)
    routing = api.RoutingConfig(True, wl.THRESHOLDS[8], list(range(8)))
    for _ in range(2):  # repeated calls reuse the context's buffers, streams and events
        _cmp_host_pass(gsb, a, p, routing, 60_000, 0, 1000, api.L.FIXED_WINDOW, chunks,
                       fixed_window_ms=0.95 * 60_000)


def test_host_pass_deadline_offset_windows_and_sparse(gsb):
    from paper_2508_16449_b200 import api, workloads as wl
    gsb.set_profiles(wl.synth_profiles(3))
    a, p, _ = wl.poisson_trace(5.0, 700 * 60_000, "alibaba_chat", seed=22)
    routing = api.RoutingConfig(True, wl.THRESHOLDS[5], list(range(5)))
    # requests before window 0 (w0 = 100) and after the last window (n_windows = 450)
    _cmp_host_pass(gsb, a, p, routing, 60_000, 100, 450, api.L.DEADLINE_SLACK, 4,
                   qopt=api.QueueOptimizerConfig())
    # sparse (most windows empty; the sampled K1a path), chunks with no requests
    b, q, _ = wl.poisson_trace(0.02, 3000 * 60_000, "alibaba_chat", seed=23)
    _cmp_host_pass(gsb, b, q, routing, 60_000, 0, 3000, api.L.FIXED_WINDOW, 16,
                   fixed_window_ms=0.95 * 60_000)
