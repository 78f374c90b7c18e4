"""Where the end-to-end prefill step's time goes at the C4 shape (tools only): each piece of
bench.py's e2e step captured alone in a CUDA graph and timed by events over replays, with L2
flushed before each.  python tools/e2e_probe.py  (one GPU)"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_16449_b200 import api, workloads as wl  # noqa: E402


def graph(fn):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def timed(g, flush, reps=30):
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def gpu_local_cpus(dev=0):
    """CPUs on the GPU's own NUMA node (sysfs local_cpulist of its PCI function), or None"""
    pr = torch.cuda.get_device_properties(dev)
    dom, bus, d = (getattr(pr, k, None) for k in ("pci_domain_id", "pci_bus_id", "pci_device_id"))
    if bus is None:
        return None
    path = f"/sys/bus/pci/devices/{dom or 0:04x}:{bus:02x}:{d or 0:02x}.0/local_cpulist"
    try:
        spec = open(path).read().strip()
    except OSError:
        return None
    cpus = set()
    for part in spec.split(","):
        lo, _, hi = part.partition("-")
        cpus.update(range(int(lo), int(hi or lo) + 1))
    return cpus or None


def main():
    if "--numa" in sys.argv:
        cpus = gpu_local_cpus(0)
        print("gpu-local cpus:", sorted(cpus) if cpus else None, "of", os.cpu_count())
        if cpus:
            os.sched_setaffinity(0, cpus)
    C, P, nW, wms = 8, 4, 10_000, 60_000
    D = 0.95 * wms
    profs = wl.synth_profiles(P)
    eng = api.Engine(0, profs)
    a, p, _ = wl.poisson_trace(5.0, nW * wms, "alibaba_chat", seed=1000)
    da, dp = torch.as_tensor(a, device="cuda"), torch.as_tensor(p, device="cuda")
    h_arr, h_prm = torch.as_tensor(a).pin_memory(), torch.as_tensor(p).pin_memory()
    routing = api.RoutingConfig(True, wl.THRESHOLDS[C], list(range(C)))
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    rr = eng.route_bin(da, dp, routing, wms, 0, nW)
    summ = eng.summary_buffer(C)
    sel = eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, summary_out=summ)
    h_fidx = torch.empty(sel.f_idx.shape, dtype=sel.f_idx.dtype).pin_memory()
    h_en = torch.empty(sel.energy_j.shape, dtype=sel.energy_j.dtype).pin_memory()
    d_prm = torch.empty_like(dp)
    up = torch.cuda.Stream()
    fork, ready = torch.cuda.Event(), torch.cuda.Event()
    cfg = api._route_cfg(routing, wms, 0, nW, api.SloConfig(), 100.0)
    import ctypes as Cc

    def k1a(arr):
        def f():
            eng._check(eng.lib.gsb_window_bounds(eng.ctx, Cc.byref(cfg), arr.numel(), api._ptr(arr),
                                                 api._ptr(rr.bounds), eng.stream()))
        return f

    def upload():
        d_prm.copy_(h_prm, non_blocking=True)

    def d2h():
        h_fidx.copy_(sel.f_idx, non_blocking=True)
        h_en.copy_(sel.energy_j, non_blocking=True)

    def compute(arr):
        def f():
            eng.route_bin(arr, d_prm, routing, wms, 0, nW, out=rr)
            eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ)
        return f

    def full():
        fork.record()
        with torch.cuda.stream(up):
            up.wait_event(fork)
            d_prm.copy_(h_prm, non_blocking=True)
            ready.record()
        eng.route_bin(h_arr, d_prm, routing, wms, 0, nW, out=rr, prompt_ready=ready)
        eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ)
        d2h()

    def full_no_d2h():
        fork.record()
        with torch.cuda.stream(up):
            up.wait_event(fork)
            d_prm.copy_(h_prm, non_blocking=True)
            ready.record()
        eng.route_bin(h_arr, d_prm, routing, wms, 0, nW, out=rr, prompt_ready=ready)
        eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ)

    def full_dev_prompts():
        eng.route_bin(h_arr, dp, routing, wms, 0, nW, out=rr)
        eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ)
        d2h()

    def full_zero_copy():  # K1a and K1b read both inputs from pinned host memory in place
        eng.route_bin(h_arr, h_prm, routing, wms, 0, nW, out=rr)
        eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ)
        d2h()

    ups = [torch.cuda.Stream() for _ in range(4)]
    evs = [(torch.cuda.Event(), torch.cuda.Event()) for _ in range(4)]
    q = (d_prm.numel() + 3) // 4

    def full_split_upload():  # the upload as 4 copies on 4 streams (several copy engines)
        for k in range(4):
            evs[k][0].record()
            with torch.cuda.stream(ups[k]):
                ups[k].wait_event(evs[k][0])
                d_prm[k * q:(k + 1) * q].copy_(h_prm[k * q:(k + 1) * q], non_blocking=True)
                evs[k][1].record()
        for k in range(4):
            torch.cuda.current_stream().wait_event(evs[k][1])
        eng.route_bin(h_arr, d_prm, routing, wms, 0, nW, out=rr)
        eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ)
        d2h()

    def full_serial():  # the upload first, then K1a's PCIe reads (no contention between them)
        d_prm.copy_(h_prm, non_blocking=True)
        eng.route_bin(h_arr, d_prm, routing, wms, 0, nW, out=rr)
        eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ)
        d2h()

    dstream = torch.cuda.Stream()
    dfork, djoin = torch.cuda.Event(), torch.cuda.Event()

    def d2h_two():  # f_idx and energy read back on two streams
        dfork.record()
        with torch.cuda.stream(dstream):
            dstream.wait_event(dfork)
            h_fidx.copy_(sel.f_idx, non_blocking=True)
            djoin.record()
        h_en.copy_(sel.energy_j, non_blocking=True)
        torch.cuda.current_stream().wait_event(djoin)

    def up_and_k1a():
        fork.record()
        with torch.cuda.stream(up):
            up.wait_event(fork)
            d_prm.copy_(h_prm, non_blocking=True)
            ready.record()
        k1a(h_arr)()
        torch.cuda.current_stream().wait_event(ready)

    rows = [
        ("flush only", lambda: None),
        ("K1a device arrivals", k1a(da)),
        ("K1a pinned host arrivals", k1a(h_arr)),
        ("prompt upload 12 MB", upload),
        ("upload || K1a pinned", up_and_k1a),
        ("compute (device inputs)", compute(da)),
        ("compute (pinned arrivals)", compute(h_arr)),
        ("D2H f_idx + energy", d2h),
        ("full e2e step", full),
        ("full without D2H", full_no_d2h),
        ("full, prompts on device", full_dev_prompts),
        ("full, zero-copy prompts", full_zero_copy),
        ("full, serial upload then K1", full_serial),
        ("D2H on two streams", d2h_two),
        ("full, 4-stream upload", full_split_upload),
    ]
    gs = [(name, graph(fn) if name != "flush only" else graph(lambda: flush.zero_()))
          for name, fn in rows]
    res = {name: [] for name, _ in rows}
    for _ in range(5):  # interleaved rounds: PCIe rates drift between processes and over time
        for name, g in gs:
            res[name].append(timed(g, flush, reps=10))
    base = statistics.median(res["flush only"])
    for name, _ in rows:
        t = statistics.median(res[name])
        print(f"{name:32s} {t:9.1f} us  (minus flush-only graph: {t - base:8.1f})  "
              f"[{min(res[name]):.1f} .. {max(res[name]):.1f}]", flush=True)
    # the pipelined host-buffer pass (eager: its chunk split reads the arrivals on the host)
    for chunks in (1, 2, 3, 4, 8, 16):
        res = eng.prefill_pass_host(h_arr, h_prm, routing, wms, 0, nW, api.L.FIXED_WINDOW,
                                    fixed_window_ms=D, chunks=chunks)
        torch.cuda.synchronize()
        ts, hs = [], []
        for i in range(23):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            h0 = time.perf_counter()
            eng.prefill_pass_host(h_arr, h_prm, routing, wms, 0, nW, api.L.FIXED_WINDOW,
                                  fixed_window_ms=D, chunks=chunks, out=res)
            h1 = time.perf_counter()
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
                hs.append((h1 - h0) * 1e6)
        ok = torch.equal(res.f_idx, sel.f_idx.cpu())
        print(f"prefill_pass_host chunks={chunks:2d}     {statistics.median(ts):9.1f} us  "
              f"[{min(ts):.1f} .. {max(ts):.1f}]  host enqueue {statistics.median(hs):.1f} us  "
              f"equal={ok}", flush=True)
    print("bytes: prompts", h_prm.numel() * 4, "arrivals", h_arr.numel() * 8,
          "d2h", h_fidx.numel() * 2 + h_en.numel() * 8)


if __name__ == "__main__":
    main()
