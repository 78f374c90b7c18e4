"""Per-entry-point device times at the C4 shape (tools only): K1 with / without the non-empty
list, K2 over K1b's list / over a k_compact list / without list, with / without the summary.
python tools/k_probe.py  (one GPU)"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_16449_b200 import api, workloads as wl  # noqa: E402


def timed(fn, reps=20, flush=None):
    """median device time of fn captured in a CUDA graph (no host launch gaps)"""
    if NCU:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        return 0.0
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return timed_eager(g.replay, reps, flush)


def timed_eager(fn, reps=20, flush=None):
    ts = []
    for i in range(reps + 3):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


NCU = "--ncu" in sys.argv  # run each variant 3x eagerly (for an ncu launch list), no timing


def main():
    C, P, nW, wms = 8, 4, 10_000, 60_000
    profs = wl.synth_profiles(P)
    eng = api.Engine(0, profs)
    a, p, _ = wl.poisson_trace(5.0, nW * wms, "alibaba_chat", seed=1000)
    da, dp = torch.as_tensor(a, device="cuda"), torch.as_tensor(p, device="cuda")
    routing = api.RoutingConfig(True, wl.THRESHOLDS[C], list(range(C)))
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    rr = eng.route_bin(da, dp, routing, wms, 0, nW)
    rr_nolist = eng.route_bin(da, dp, routing, wms, 0, nW)
    rr_nolist.nonempty = None
    rr_nolist.n_nonempty = None
    summ = eng.summary_buffer(C)
    sel = eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=0.95 * wms, summary_out=summ)
    D = 0.95 * wms
    out = {}
    out["K1 (bounds + route_bin + list)"] = timed(lambda: eng.route_bin(da, dp, routing, wms, 0, nW, out=rr), flush=flush)
    out["K1 (bounds + route_bin, no list)"] = timed(lambda: eng.route_bin(da, dp, routing, wms, 0, nW, out=rr_nolist), flush=flush)
    out["window_bounds only"] = timed(lambda: eng.window_bounds(da, routing, wms, 0, nW), flush=flush)
    out["K2 list + summary"] = timed(lambda: eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ), flush=flush)
    out["K2 list, no summary"] = timed(lambda: eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel), flush=flush)
    out["K2 compact + list + summary"] = timed(lambda: eng.prefill_select(rr_nolist, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ), flush=flush)
    out["K2 compact + list, no summary"] = timed(lambda: eng.prefill_select(rr_nolist, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel), flush=flush)
    out["summary standalone"] = timed(lambda: eng.prefill_summary_dev(sel, C), flush=flush)
    prr, psel = eng.prefill_pass(da, dp, routing, wms, 0, nW, api.L.FIXED_WINDOW,
                                 fixed_window_ms=D, summary_out=summ)
    out["fused pass (K1a + K1b/K2 + finish + summary)"] = timed(
        lambda: eng.prefill_pass(da, dp, routing, wms, 0, nW, api.L.FIXED_WINDOW, fixed_window_ms=D,
                                 rr=prr, sel=psel, summary_out=summ), flush=flush)
    out["two-call path (K1 + K2 + finish + summary)"] = timed(
        lambda: (eng.route_bin(da, dp, routing, wms, 0, nW, out=rr),
                 eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel,
                                    summary_out=summ)), flush=flush)
    if NCU:
        return
    for k, v in out.items():
        print(f"{k:40s} {v:8.1f} us")


if __name__ == "__main__":
    main()
