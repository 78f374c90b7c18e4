"""Device time of K1 / K2 / the two-call step at the C4 shape, by CUDA-graph differencing over
many replays (one event pair around N replays of [L2 flush, op] minus N replays of [L2 flush]),
which resolves sub-microsecond differences that single-replay event timing quantizes away.
python tools/k_ab.py   (set GSB_LIB to time another build of libgsb.so)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_16449_b200 import api, workloads as wl  # noqa: E402

N = 40


def graph_of(fn, flush):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        flush.zero_()
        if fn is not None:
            fn()
    return g


def per_replay(g):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(N):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / N


def main():
    C, P, nW, wms = 8, 4, 10_000, 60_000
    eng = api.Engine(0, wl.synth_profiles(P))
    a, p, _ = wl.poisson_trace(5.0, nW * wms, "alibaba_chat", seed=1000)
    da, dp = torch.as_tensor(a, device="cuda"), torch.as_tensor(p, device="cuda")
    routing = api.RoutingConfig(True, wl.THRESHOLDS[C], list(range(C)))
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    rr = eng.route_bin(da, dp, routing, wms, 0, nW)
    summ = eng.summary_buffer(C)
    D = 0.95 * wms
    sel = eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, summary_out=summ)
    rn = eng.route_bin(da, dp, routing, wms, 0, nW)
    rn.nonempty = rn.n_nonempty = rn.t_ref_list = None
    ops = {
        "K1nolist": lambda: eng.route_bin(da, dp, routing, wms, 0, nW, out=rn),
        "K1a": lambda: eng.window_bounds(da, routing, wms, 0, nW),
        "K1": lambda: eng.route_bin(da, dp, routing, wms, 0, nW, out=rr),
        "K1+K2k": lambda: (eng.route_bin(da, dp, routing, wms, 0, nW, out=rr),
                           eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel)),
        "K1+K2": lambda: (eng.route_bin(da, dp, routing, wms, 0, nW, out=rr),
                          eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel,
                                             summary_out=summ)),
    }
    g0 = graph_of(lambda: None, flush)
    gs = {k: graph_of(f, flush) for k, f in ops.items()}
    res = {k: [] for k in ops}
    for _ in range(5):
        t0 = per_replay(g0)
        for k, g in gs.items():
            res[k].append(per_replay(g) - t0)
    for k, v in res.items():
        v.sort()
        print(f"{k:8s} median {v[len(v) // 2]:7.2f} us  min {v[0]:7.2f}  max {v[-1]:7.2f}")


if __name__ == "__main__":
    main()
