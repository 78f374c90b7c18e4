"""K1a window bounds: the interpolation search (dense traces) and the sampled pass against a host
lower_bound, bounds[k] = #{i : arrival[i] < (w0 + k) * W} — the first request of window k in
the Dispatcher's binning (router.cpp:33-43, trace order trace.cpp:109-111). Both kernels are
forced in turn with GSB_BOUNDS; the default choice is checked too. Integer output: bit-exact."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _bounds(eng, arrival, window_ms, w0, n_windows, kernel=None, pinned=False):
    from paper_2508_16449_b200 import api
    routing = api.RoutingConfig(True, [512, 1024], [0, 1, 2])
    cfg = api._route_cfg(routing, window_ms, w0, n_windows, api.SloConfig(), 100.0)
    a = torch.as_tensor(np.asarray(arrival, np.int64))
    a = a.pin_memory() if pinned else a.cuda()
    out = torch.full((n_windows + 1,), -7, dtype=torch.int64, device="cuda")
    old = os.environ.get("GSB_BOUNDS")
    try:
        if kernel is None:
            os.environ.pop("GSB_BOUNDS", None)
        else:
            os.environ["GSB_BOUNDS"] = kernel
        eng._check(eng.lib.gsb_window_bounds(eng.ctx, C.byref(cfg), a.numel(),
                                             C.c_void_p(a.data_ptr()), C.c_void_p(out.data_ptr()),
                                             eng.stream()))
    finally:
        if old is None:
            os.environ.pop("GSB_BOUNDS", None)
        else:
            os.environ["GSB_BOUNDS"] = old
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _host(arrival, window_ms, w0, n_windows):
    t = (w0 + np.arange(n_windows + 1, dtype=np.int64)) * window_ms
    return np.searchsorted(np.asarray(arrival, np.int64), t, side="left").astype(np.int64)


def _poisson(rng, qps, dur_ms, t0=0):
    n = rng.poisson(qps * dur_ms / 1000.0)
    return np.sort(t0 + np.floor(rng.uniform(0, dur_ms, n))).astype(np.int64)


def _cases():
    rng = np.random.default_rng(7)
    W = 60_000
    out = []
    out.append(("c4-like", _poisson(rng, 5.0, 2000 * W), W, 0, 2000))
    segs = [_poisson(rng, 20.0, 50 * W, t0=s * W) for s in (0, 400, 401, 2000)]
    out.append(("gaps", np.sort(np.concatenate(segs)), W, 0, 2100))
    out.append(("duplicates", np.sort(rng.integers(0, 300 * W, 400_000) // 977 * 977), W, 0, 300))
    a = _poisson(rng, 8.0, 600 * W, t0=100 * W)
    out.append(("w0-and-cut", a, W, 150, 300))  # requests before window 0 and after the last
    out.append(("on-edges", np.repeat(np.arange(0, 200) * W, 400), W, 0, 200))
    out.append(("w1", np.sort(rng.integers(0, 5000, 300_000)), 1, 0, 5000))
    out.append(("tail-windows", _poisson(rng, 30.0, 100 * W), W, 0, 400))
    out.append(("empty", np.zeros(0, np.int64), W, 0, 10))
    out.append(("tiny", np.array([5, 5, 70_000], np.int64), W, 0, 3))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_bounds_kernels_equal_host_lower_bound(gsb, case):
    name, arr, W, w0, nW = case
    want = _host(arr, W, w0, nW)
    for kernel in ("search", "sampled", None):
        got = _bounds(gsb, arr, W, w0, nW, kernel)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (name, kernel, bad[:5], got[bad[:5]], want[bad[:5]])


def test_bounds_search_reads_pinned_host_arrivals(gsb):
    rng = np.random.default_rng(11)
    W, nW = 60_000, 3000
    arr = _poisson(rng, 5.0, nW * W)
    want = _host(arr, W, 0, nW)
    got = _bounds(gsb, arr, W, 0, nW, "search", pinned=True)
    assert np.array_equal(got, want)


def test_bounds_pinned_arrivals_in_a_cuda_graph(gsb):
    # the default launch from pinned host arrivals (the search) captured and replayed in a graph
    from paper_2508_16449_b200 import api, workloads as wl
    a, p, _ = wl.poisson_trace(5.0, 800 * 60_000, "alibaba_chat", seed=5)
    h_arr = torch.as_tensor(a).pin_memory()
    d_prm = torch.as_tensor(p, device="cuda")
    routing = api.RoutingConfig(True, wl.THRESHOLDS[8], list(range(8)))
    rr = gsb.route_bin(h_arr, d_prm, routing, 60_000, 0, 800)
    torch.cuda.synchronize()
    rr.bounds.fill_(-1)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        gsb.route_bin(h_arr, d_prm, routing, 60_000, 0, 800, out=rr)
    rr.bounds.fill_(-1)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(rr.bounds.cpu().numpy(), _host(a, 60_000, 0, 800))
    dev = gsb.route_bin(torch.as_tensor(a, device="cuda"), d_prm, routing, 60_000, 0, 800)
    assert torch.equal(dev.count, rr.count) and torch.equal(dev.t_ref, rr.t_ref)


def test_bounds_default_picks_search_for_dense_traces(gsb):
    # from pinned host memory the C4 shape (~300 requests per window) takes the search and a
    # sparse trace the sampled pass (kSearchDense = 64 requests per window); device arrivals
    # always take the sampled pass. Both exact.
    from paper_2508_16449_b200 import api  # noqa: F401
    rng = np.random.default_rng(3)
    dense = _poisson(rng, 5.0, 500 * 60_000)
    sparse = _poisson(rng, 0.5, 500 * 60_000)
    assert len(dense) >= 64 * 501 and len(sparse) < 64 * 501
    for arr in (dense, sparse):
        for pinned in (False, True):
            got = _bounds(gsb, arr, 60_000, 0, 500, pinned=pinned)
            assert np.array_equal(got, _host(arr, 60_000, 0, 500))


def test_route_bin_zero_copy_inputs_equal_device_inputs(gsb):
    # K1a and K1b reading pinned host arrivals and prompts in place (plain loads instead of the
    # TMA stage) give the device-input results bit for bit, list and T_ref in list order too
    from paper_2508_16449_b200 import api, workloads as wl
    a, p, _ = wl.poisson_trace(5.0, 700 * 60_000, "alibaba_chat", seed=9)
    routing = api.RoutingConfig(True, wl.THRESHOLDS[8], list(range(8)))
    for want_deadline in (False, True):
        dev = gsb.route_bin(torch.as_tensor(a, device="cuda"), torch.as_tensor(p, device="cuda"),
                            routing, 60_000, 0, 700, want_deadline=want_deadline)
        zc = gsb.route_bin(torch.as_tensor(a).pin_memory(), torch.as_tensor(p).pin_memory(),
                           routing, 60_000, 0, 700, want_deadline=want_deadline)
        torch.cuda.synchronize()
        for f in ("bounds", "cls", "count", "t_ref", "n_nonempty"):
            assert torch.equal(getattr(dev, f), getattr(zc, f)), (f, want_deadline)
        n = int(dev.n_nonempty.item())  # the list's capacity past n is scratch
        assert torch.equal(dev.nonempty[:n], zc.nonempty[:n])
        assert torch.equal(dev.t_ref_list[:, :n], zc.t_ref_list[:, :n])
        if want_deadline:
            assert torch.equal(dev.min_deadline.view(torch.int64), zc.min_deadline.view(torch.int64))
            assert torch.equal(dev.min_deadline_list[:n].view(torch.int64),
                               zc.min_deadline_list[:n].view(torch.int64))
