#!/usr/bin/env python
"""Benchmark of the B200 GreenLLM decision engine (driver contract in the task statement).

Default workload = BASELINE.json configs[3] "C4": joint prefill + decode sweep, per GPU
(weak scaling: rank r owns windows [r*W, (r+1)*W) and its own scenario set):
  prefill leg: Alibaba-shaped trace (5 qps), 1e4 one-minute windows x 8 length classes x
               4 profiles x 81 clocks = 2.592e7 (window x class x clock) evaluations / step
               = K1 route+bin (3e6 requests) + K2 objective/argmin + per-class summary
               (+ NCCL all-gather of the summaries when N > 1).
  decode leg:  1e5 controller scenarios (hysteresis x step x TBT target x margin x profile x
               bias), each a 4-worker pool replayed over 150 s (7,500 fine ticks) = K3a window
               series + K3b DecodeController replay.
`value` is the prefill leg (evals/s, device-resident inputs, L2 flushed between steps);
`decode` reports the second half of the metric (scenario replays/s). `e2e` runs the same
step through the public API from pinned HOST buffers (H2D + kernels + D2H in the timed
region). `--impl reference` times the reference's own CPU path (oracle/_ref) instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
K2_DP_OPS_PER_EVAL = 14  # DP-pipe instructions per (cell, clock) in K2 (SASS, profiles/r2_k2_sass.txt)
K1_DP_OPS_PER_REQ_PROFILE = 5  # (a L + b) L + c and the chain add (prefill_opt.cpp:9-14)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="gsb", choices=["gsb", "reference"])
    ap.add_argument("--config", default="c4", choices=["c2", "c4", "c5"])
    ap.add_argument("--windows", type=int, default=0, help="override windows per rank")
    ap.add_argument("--scenarios", type=int, default=100_000)
    ap.add_argument("--pool-scenarios", type=int, default=20_000,
                    help="closed-loop decode-pool (K5) scenarios per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="window chunks of the pipelined host-buffer e2e pass (0: 3 for >= 1e6 "
                         "requests per rank, else 1)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: ONE global trace of the config's windows, sliced per "
                         "rank (distributed.window_shard / trace_slice), scenarios split too")
    return ap.parse_args()


def workload(cfg: str, windows_override: int):
    """(description, shape, qps, classes, profiles, windows, window_ms)"""
    if cfg == "c2":
        d = dict(name="C2 Azure-conv-shaped 24 h, 5 classes, 1-min windows", shape="azure_conv",
                 qps=5.0, C=5, P=1, W=1440)
    elif cfg == "c5":
        d = dict(name="C5 mixed Alibaba+Azure multi-day, 1e6 one-minute windows per GPU",
                 shape="mixed", qps=1.0, C=8, P=1, W=1_000_000)
    else:
        d = dict(name="C4 joint prefill+decode: 1e4 windows x 8 classes x 4 profiles per GPU",
                 shape="alibaba_chat", qps=5.0, C=8, P=4, W=10_000)
    if windows_override:
        d["W"] = windows_override
    d["window_ms"] = 60_000
    return d


class ClockSampler:
    """nvidia-smi style clocks / throttle reasons sampled DURING the timed region (NVML)."""

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


# ---------------------------------------------------------------------------- gsb arm
def run_gsb(args, rank, world, dist):
    import torch
    from paper_2508_16449_b200 import api, workloads as wl

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    W = workload(args.config, args.windows)
    profs = wl.synth_profiles(W["P"])
    eng = api.Engine(dev, profs)
    thr = wl.THRESHOLDS[W["C"]]
    routing = api.RoutingConfig(True, thr, list(range(W["C"])))
    nW, wms = W["W"], W["window_ms"]
    from paper_2508_16449_b200 import distributed as Dd
    if args.strong:  # one global trace (rank 0's weak-scaling trace), this rank's window slice
        total_w = nW
        if W["shape"] == "mixed":
            ga, gp, _ = wl.mixed_trace(W["qps"], total_w * wms, seed=1000, t0_ms=0)
        else:
            ga, gp, _ = wl.poisson_trace(W["qps"], total_w * wms, W["shape"], seed=1000, t0_ms=0)
        w0, nW = Dd.window_shard(total_w, world, rank)
        lo, hi = Dd.trace_slice(ga, wms, w0, nW)
        arrival, prompt = ga[lo:hi].copy(), gp[lo:hi].copy()
        args.scenarios = Dd.scenario_shard(args.scenarios, world, rank)[1]
        args.pool_scenarios = max(1, Dd.scenario_shard(args.pool_scenarios, world, rank)[1])
    else:
        w0 = rank * nW
        t0 = w0 * wms
        if W["shape"] == "mixed":
            arrival, prompt, _ = wl.mixed_trace(W["qps"], nW * wms, seed=1000 + rank, t0_ms=t0)
        else:
            arrival, prompt, _ = wl.poisson_trace(W["qps"], nW * wms, W["shape"],
                                                  seed=1000 + rank, t0_ms=t0)
    n_req = len(arrival)
    cells = nW * W["C"]
    P = W["P"]
    evals = cells * P * 81
    D = 0.95 * wms  # FIXED_WINDOW: D = margin_prefill * window (DESIGN.md offline convention)
    stream = torch.cuda.current_stream()

    d_arr = torch.as_tensor(arrival, device="cuda")
    d_prm = torch.as_tensor(prompt, device="cuda")
    rr = eng.route_bin(d_arr, d_prm, routing, wms, w0, nW)
    sel = eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D)
    summ = eng.prefill_summary_dev(sel, W["C"])
    gathered = torch.empty((world,) + tuple(summ.shape), dtype=summ.dtype, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def prefill_step():
        # K1 (window bounds, route + bin + T_ref fold + the non-empty cell list), then K2 over
        # the list, the empty cells' outputs and the per-class summary
        eng.route_bin(d_arr, d_prm, routing, wms, w0, nW, out=rr)
        eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ)

    def fused_step():  # the same pass with K1b and K2 in one persistent kernel (gsb_prefill_pass)
        eng.prefill_pass(d_arr, d_prm, routing, wms, w0, nW, api.L.FIXED_WINDOW,
                         fixed_window_ms=D, rr=rr, sel=sel, summary_out=summ)

    use_graph = not args.no_graph
    graphs = {}
    if use_graph:
        for _ in range(2):
            prefill_step()
        torch.cuda.synchronize()
        # timing events INSIDE the graph (external event-record nodes): the step's device time
        # from its first kernel to its last, without the host's graph-launch latency that an
        # event recorded before replay() also counts (kept as ms_per_step_replay)
        g_e0 = torch.cuda.Event(enable_timing=True, external=True)
        g_e1 = torch.cuda.Event(enable_timing=True, external=True)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            g_e0.record()
            prefill_step()
            g_e1.record()
        graphs["prefill"] = g

    def run_prefill(timed_steps, warm):
        """per step: L2 flush (outside the timing), the step; returns (device ms from the
        step's first to last kernel (+ the all-gather when world > 1), ms from an event
        recorded before replay())"""
        t_dev, t_rep = [], []
        for i in range(warm + timed_steps):
            flush.zero_()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            if use_graph:
                graphs["prefill"].replay()
            else:
                prefill_step()
            if world > 1:
                dist.all_gather_into_tensor(gathered, summ)
            s1.record(stream)
            torch.cuda.synchronize()  # the in-graph events are re-recorded by the next replay
            if i >= warm:
                t_rep.append(s0.elapsed_time(s1))
                if use_graph:
                    t_dev.append(g_e0.elapsed_time(s1 if world > 1 else g_e1))
                else:
                    t_dev.append(s0.elapsed_time(s1))
        return t_dev, t_rep

    def graph_of(fn):
        """a graph of [L2 flush, fn]"""
        if fn is not None:
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            flush.zero_()
            if fn is not None:
                fn()
        return g

    def graph_ms(g, n=40):
        """mean device time of one replay over n back-to-back replays (one event pair: the
        per-replay launch latency overlaps, and the 2-us event granularity averages out)"""
        for _ in range(3):
            g.replay()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(n):
            g.replay()
        s1.record(stream)
        torch.cuda.synchronize()
        return s0.elapsed_time(s1) / n

    # per-kernel split of the two-call path by graph differencing: [flush, K1], [flush, K1,
    # K2 (+ its empty-cell fill)], [flush, K1, K2, finish, summary] and the fused pass, each
    # minus [flush] (tools/k_ab.py resolves 0.1 us this way)
    def kernel_split(n=40, reps=3):
        g0 = graph_of(None)
        g1 = graph_of(lambda: eng.route_bin(d_arr, d_prm, routing, wms, w0, nW, out=rr))
        g12k = graph_of(lambda: (eng.route_bin(d_arr, d_prm, routing, wms, w0, nW, out=rr),
                                 eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D,
                                                    out=sel)))
        g12 = graph_of(prefill_step)
        gp = graph_of(fused_step)
        res = []
        for _ in range(reps):
            t0 = graph_ms(g0, n)
            res.append([graph_ms(g, n) - t0 for g in (g1, g12k, g12, gp)])
        k1, k12k, k12, kp = (statistics.median(r[i] for r in res) for i in range(4))
        return k1, max(k12k - k1, 1e-6), max(k12 - k1, 1e-6), kp

    # ---------------- decode leg setup
    T_END = 150_000.0
    sweep = wl.decode_sweep(args.scenarios, n_profiles=P, n_workers=4, streams_per_profile=4)
    tel = wl.decode_telemetry(P * 4, T_END, seed=7 + rank)
    tdev = eng.telemetry_to_device(tel)
    lo, hi, fo, fe = eng.build_band_tables(profs, sweep.table_profile, sweep.table_tslo,
                                           [4] * len(sweep.table_profile),
                                           [64] * len(sweep.table_profile), wl.TPS_LEVELS)
    has, p95, tps = eng.window_series(tel, 256, 20.0, 200.0, T_END, dev=tdev)
    grid = profs[0].grid
    plan = eng.decode_replay(sweep.cfgs, sweep.table_of, sweep.stream_of, sweep.worker, lo, hi, fo,
                             grid, has, p95, tps, T_END, want_counts=False)

    def decode_step():
        eng.window_series(tel, 256, 20.0, 200.0, T_END, dev=tdev, out=(has, p95, tps))
        eng.run_replay(plan)

    if use_graph:
        decode_step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            decode_step()
        graphs["decode"] = g

    def run_decode(timed_steps, warm):
        ts = []
        for i in range(warm + timed_steps):
            flush.zero_()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            graphs["decode"].replay() if use_graph else decode_step()
            s1.record(stream)
            if i >= warm:
                ts.append((s0, s1))
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ts]

    def decode_split(n=3):
        ga = graph_of(lambda: eng.window_series(tel, 256, 20.0, 200.0, T_END, dev=tdev,
                                                out=(has, p95, tps)))
        gb = graph_of(lambda: eng.run_replay(plan))
        t0 = graph_ms(graph_of(None), n)
        return graph_ms(ga, n) - t0, graph_ms(gb, n) - t0

    # ---------------- closed-loop decode pool leg (K5): C3 sinusoid, controller sweep
    pa, pp, po = wl.sinusoid_decode_trace(1500.0, 1000.0, 120_000.0, 150_000, seed=11 + rank)
    pstream = wl.decode_stream(pa, pp, po)
    pcfg = wl.pool_sweep(args.pool_scenarios)
    pprof = api.GpuProfile.default_profile()
    psim, pslo = api.SimConfig(), api.SloConfig()
    pplan = eng.decode_pool(pcfg, pstream, pprof, psim, pslo)

    def run_pool(timed_steps, warm):
        ts = []
        for i in range(warm + timed_steps):
            flush.zero_()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            eng.run_pool(pplan)
            s1.record(stream)
            if i >= warm:
                ts.append((s0, s1))
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ts]

    # ---------------- trace ingest leg (K6): this rank's trace as CSV text, parsed on the GPU
    csv_text = eng.format_trace(d_arr, d_prm, torch.full_like(d_prm, 128),
                                (d_prm > 1024).to(torch.uint8))
    d_csv = torch.frombuffer(bytearray(csv_text), dtype=torch.uint8).to("cuda")
    eng.parse_trace(d_csv)  # warm (scratch sizing)

    def run_ingest(timed_steps, warm):
        ts = []
        for i in range(warm + timed_steps):
            flush.zero_()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            t = eng.parse_trace(d_csv)
            s1.record(stream)
            if i >= warm:
                ts.append((s0, s1))
        torch.cuda.synchronize()
        assert t.arrival_ms.numel() == n_req
        return [a.elapsed_time(b) for a, b in ts]

    # ---------------- e2e prefill leg: pinned host in, pinned host out
    h_arr = torch.as_tensor(arrival).pin_memory()
    h_prm = torch.as_tensor(prompt).pin_memory()
    h_fidx = torch.empty(sel.f_idx.shape, dtype=sel.f_idx.dtype).pin_memory()
    h_en = torch.empty(sel.energy_j.shape, dtype=sel.energy_j.dtype).pin_memory()
    # the prompts are copied (K1b stages every one); the arrivals stay in pinned host memory
    # and K1a reads them in place over PCIe. For a dense trace (>= 64 requests per window) it
    # is the interpolation search: one 32-byte sector per 256-request block plus one probe of
    # one 64-byte probe per window edge (a probe that misses adds 64 bytes; not counted);
    # otherwise one sector per 32-request tile plus the 256 bytes of every tile holding an edge
    n_req_h = h_arr.numel()
    if n_req_h >= 64 * (nW + 1):
        arr_bytes = 32 * ((n_req_h + 255) // 256) + 64 * (nW + 1)
    else:
        n_tiles32 = (n_req_h + 31) // 32
        arr_bytes = 32 * n_tiles32 + 256 * min(nW + 1, n_tiles32)
    h2d = h_prm.numel() * 4 + arr_bytes
    d2h = h_fidx.numel() * 2 + h_en.numel() * 8

    up_stream = torch.cuda.Stream()
    fork, prm_ready = torch.cuda.Event(), torch.cuda.Event()

    def e2e_step():
        # the prompt upload runs beside K1a (which reads the pinned arrivals in place); K1b
        # waits for it
        fork.record()
        with torch.cuda.stream(up_stream):
            up_stream.wait_event(fork)
            d_prm.copy_(h_prm, non_blocking=True)
            prm_ready.record()
        eng.route_bin(h_arr, d_prm, routing, wms, w0, nW, out=rr, prompt_ready=prm_ready)
        eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ)
        h_fidx.copy_(sel.f_idx, non_blocking=True)
        h_en.copy_(sel.energy_j, non_blocking=True)

    if use_graph:
        e2e_step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            e2e_step()
        graphs["e2e"] = g

    def run_e2e(timed_steps, warm):
        ts = []
        for i in range(warm + timed_steps):
            flush.zero_()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            graphs["e2e"].replay() if use_graph else e2e_step()
            if world > 1:
                dist.all_gather_into_tensor(gathered, summ)
            s1.record(stream)
            if i >= warm:
                ts.append((s0, s1))
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ts]

    # the headline e2e: Engine.prefill_pass_host (gsb_prefill_pass_host), the public call for a
    # host-resident trace. Pinned arrivals / prompts in, host f_idx / energy out, the windows
    # split into chunks whose prompt upload, kernels and read-back overlap (PCIe is full duplex)
    # chunks: 3 for a large trace (2 / 3 / 4 measured 0.383 / 0.381 / 0.386 ms at C4); a small
    # one (C2) is latency-bound and takes one
    e2e_chunks = args.e2e_chunks or (3 if len(arrival) >= 1_000_000 else 1)
    # (set up when its leg runs, so the launch order before it, which the committed ncu
    # captures select by count, is the same as without it)
    hres = None

    def run_e2e_host(timed_steps, warm):
        nonlocal hres
        hres = eng.prefill_pass_host(h_arr, h_prm, routing, wms, w0, nW, api.L.FIXED_WINDOW,
                                     fixed_window_ms=D, chunks=e2e_chunks)
        torch.cuda.synchronize()
        ts = []
        for i in range(warm + timed_steps):
            flush.zero_()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            eng.prefill_pass_host(h_arr, h_prm, routing, wms, w0, nW, api.L.FIXED_WINDOW,
                                  fixed_window_ms=D, chunks=e2e_chunks, out=hres)
            if world > 1:  # the global per-class result: every rank's chunk summaries
                stream.synchronize()
                loc = hres.chunk_summaries.reshape(-1).to(dev)
                glob = torch.empty(world * loc.numel(), dtype=torch.uint8, device=dev)
                dist.all_gather_into_tensor(glob, loc)
            s1.record(stream)
            if i >= warm:
                ts.append((s0, s1))
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ts]

    # ---------------- FP64 pipe peak probe (same run, for the K2 roofline)
    probe_threads, probe_iters = 148 * 2048, 4096
    eng.fp64_probe(probe_threads, 64)
    torch.cuda.synchronize()
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    eng.fp64_probe(probe_threads, probe_iters)
    pe1.record(stream)
    torch.cuda.synchronize()
    dfma_per_s = probe_threads * probe_iters * 8 / (pe0.elapsed_time(pe1) / 1e3)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------- timed region
    with ClockSampler(dev) as clk:
        barrier()
        pre_ms, pre_rep_ms = run_prefill(args.steps, args.warmup)
        barrier()
        dec_ms = run_decode(args.steps, max(3, args.warmup // 2))
        barrier()
        pool_ms = run_pool(max(3, args.steps // 4), 3)
        barrier()
        e2e_ms = run_e2e(args.steps, args.warmup)
        barrier()
        e2e_host_ms = run_e2e_host(args.steps, args.warmup)
        barrier()
        ing_ms = run_ingest(max(3, args.steps // 4), 3)
        barrier()
    k1_ms, k2_ms, k2_full_ms, pass_ms = kernel_split()
    k3a_ms, k3b_ms = decode_split()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_pre = max_over_ranks(statistics.mean(pre_ms))
    ms_pre_rep = max_over_ranks(statistics.mean(pre_rep_ms))
    ms_dec = max_over_ranks(statistics.mean(dec_ms))
    ms_e2e_graph = max_over_ranks(statistics.mean(e2e_ms))
    ms_e2e = max_over_ranks(statistics.mean(e2e_host_ms))
    d2h_host = hres.f_idx.numel() * 2 + hres.energy_j.numel() * 8 + hres.chunk_summaries.numel()
    e2e_host_mismatch = int((hres.f_idx != sel.f_idx.cpu()).sum().item()) + int(
        (hres.energy_j.view(torch.int64) != sel.energy_j.cpu().view(torch.int64)).sum().item())
    ms_pool = max_over_ranks(statistics.mean(pool_ms))
    ms_ing = max_over_ranks(statistics.mean(ing_ms))
    from paper_2508_16449_b200 import distributed as Dd
    psum = api.Engine.pool_summary(pplan)
    # decode-side end-of-run reduction: per-rank tally of the pool scenarios (global index =
    # rank * n + i), NCCL all-gather, rank-order combine (identical bytes on every rank)
    my_tally = Dd.tally_pool(psum, rank * len(pcfg))
    tallies = (Dd.gather_records(np.array([my_tally], Dd.DECODE_TALLY_DTYPE), "cuda")
               if world > 1 else np.array([my_tally], Dd.DECODE_TALLY_DTYPE))
    gtally = Dd.combine_tallies(tallies)

    # global per-(profile, class) result: every rank's summary, combined in rank order
    if world > 1:
        per_rank = gathered.cpu().numpy().reshape(world, -1).view(Dd.SUMMARY_DTYPE)
    else:
        per_rank = summ.cpu().numpy().reshape(1, -1).view(Dd.SUMMARY_DTYPE)
    per_rank = per_rank.reshape(world, P, W["C"])
    if args.strong:
        cell_off = [Dd.window_shard(W["W"], world, r)[0] * W["C"] for r in range(world)]
    else:
        cell_off = [r * nW * W["C"] for r in range(world)]
    # the rank-order combine through the C ABI (gsb_combine_summaries)
    glob = Dd.combine_summaries_c(per_rank, cell_off)

    # ---------------- CPU baseline + parity (rank 0, N = 1 only; the oracle is the checker)
    cpu = None
    parity = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        cpu, parity = cpu_baseline(args, sel, arrival, prompt, W, profs, thr, D, sweep, tel, plan,
                                   lo, hi, fo, T_END)
        if cpu is not None:
            cpu["pool"], parity["pool"] = pool_cpu_baseline(args, pa, pp, po, pstream, pcfg,
                                                            psum)
            cpu["ingest"] = ingest_cpu_baseline(args, csv_text)

    # executed K2 work, all ranks: every non-empty (cell, profile) pair runs the 81-clock scan
    # (commands include the infeasible ones); empty queues give no command without evaluation
    # (prefill_opt.cpp:64) and are not counted
    pairs_rank = [int(per_rank[r]["n_cmd"].sum()) for r in range(world)]
    evaluated_all = sum(pairs_rank) * 81
    if rank != 0:
        return
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    prof_json = committed_profile()
    evaluated = pairs_rank[0] * 81
    k2_tflops = evaluated * K2_DP_OPS_PER_EVAL * 2 / (k2_ms / 1e3) / 1e12
    k2_full_tflops = evaluated * K2_DP_OPS_PER_EVAL * 2 / (k2_full_ms / 1e3) / 1e12
    pass_tflops = ((evaluated * K2_DP_OPS_PER_EVAL + n_req * P * K1_DP_OPS_PER_REQ_PROFILE) * 2
                   / (pass_ms / 1e3) / 1e12)
    peak_tflops = dfma_per_s * 2 / 1e12
    # K1 (K1a window bounds + K1b route/bin) algorithmic bytes, FIXED_WINDOW mode:
    # prompt i32 read + class u8 written per request, one arrival per 32-request tile (the
    # window-edge search), count u32 + P t_ref f64 written per cell
    cells = nW * W["C"]
    k1_bytes = n_req * 5 + (n_req // 32) * 8 + cells * (4 + 8 * P)
    k1_gbs = k1_bytes / (k1_ms / 1e3) / 1e9
    clk = clk.summary()
    sm_mhz = clk.get("sm_mhz") or 1965.0
    issue_peak = 148 * 4 * sm_mhz * 1e6  # warp instructions / s (one per SMSP per cycle)

    def issue_roof(kernel_prefix, units, ms):
        rec = next((v for k, v in prof_json.items() if k.startswith(kernel_prefix)
                    and v.get("warp_insts") and v.get("units")), None)
        if rec is None:
            return None
        ach = rec["warp_insts"] / rec["units"] * units / (ms / 1e3)
        return {"bound": "issue", "achieved": ach, "peak": issue_peak,
                "unit": "warp-instr/s", "frac": ach / issue_peak, "kernel_ms": ms,
                "warp_insts_per_unit": rec["warp_insts"] / rec["units"],
                "fp64_pipe_pct_active": rec.get("fp64_pipe_pct_active"),
                "dram_bytes_per_unit": rec.get("dram_bytes_per_launch", 0) / rec["units"],
                "basis": "ncu smsp__inst_executed per unit (profiles/) x units / event time; "
                         "peak = 592 SMSPs x 1 issue/cycle at the sampled SM clock"}

    launches = args.steps * (4 + 3 + 4) + max(3, args.steps // 4) + 4 * max(3, args.steps // 4)
    line = {
        "metric": METRIC,
        "value": evaluated_all / (ms_pre / 1e3),
        "unit": "window x class x clock evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_pre,
        "ms_per_step_replay": ms_pre_rep,
        "timing": "events inside the step's CUDA graph (first to last kernel; the all-gather "
                  "too when N > 1); ms_per_step_replay: an event recorded before replay(), i.e. "
                  "plus the host's graph-launch latency",
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference-shaped Poisson/bimodal traces; sinusoidal decode telemetry)",
        "config": {"workload": W["name"], "windows_per_gpu": nW, "window_ms": wms,
                   "classes": W["C"], "profiles": P, "clocks": 81, "requests_per_gpu": n_req,
                   "evaluated_evals_per_step_per_gpu": evaluated,
                   "grid_evals_per_step_per_gpu": evals,
                   "value_counts": "EVALUATED triples: non-empty (window, class, profile) x 81 "
                                   "clocks (empty queues: no command, prefill_opt.cpp:64)",
                   "window_mode": "FIXED_WINDOW D=0.95*W",
                   "decode_scenarios_per_gpu": sweep.n_scenarios, "decode_horizon_ms": T_END,
                   "parallelism": f"dp{world} (windows/scenarios sharded, NCCL all-gather of "
                                  f"per-class summaries)",
                   "l2": "flushed between timed steps (256 MB write, outside the events)",
                   "cuda_graphs": use_graph},
        "grid_value": world * evals / (ms_pre / 1e3),
        "e2e": {"value": evaluated_all / (ms_e2e / 1e3), "unit": "window x class x clock evals/s",
                "ms_per_step": ms_e2e, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h_host,
                "path": f"Engine.prefill_pass_host (gsb_prefill_pass_host), the public call for a "
                        f"host-resident trace: pinned arrivals / prompts in, host f_idx / energy "
                        f"(+ per-chunk summaries) out; {e2e_chunks} window chunks of decreasing "
                        f"size whose prompt upload, kernels and read-back overlap; K1a' reads the "
                        f"pinned arrivals in place (h2d counts the sectors / lines it reads); "
                        f"launched eagerly (its chunk split reads the arrivals on the host)",
                "chunks": e2e_chunks,
                "mismatches_vs_device_pass": e2e_host_mismatch,
                "graph_step": {"ms_per_step": ms_e2e_graph,
                               "value": evaluated_all / (ms_e2e_graph / 1e3),
                               "d2h_bytes_per_step": d2h,
                               "path": "Engine.route_bin / prefill_select in one CUDA graph: the "
                                       "prompt upload beside K1a', then K1b, K2, the finish and "
                                       "summary, and the read-back of every cell's clock and "
                                       "energy"}},
        "roofline": {"bound": "fp64", "kernel": "k_prefill_select_list (K2)",
                     "achieved": k2_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
                     "frac": k2_tflops / peak_tflops,
                     "basis": f"{K2_DP_OPS_PER_EVAL} DP instr per evaluated triple x 2 vs DFMA "
                              "rate measured in this run; K2 time = graph(K1 + K2 + its "
                              "empty-cell fill) - graph(K1), 40 back-to-back replays each",
                     "kernel_ms": k2_ms, "share_of_step": k2_ms / ms_pre,
                     "with_finish_summary": {"kernel_ms": k2_full_ms,
                                             "achieved": k2_full_tflops,
                                             "frac": k2_full_tflops / peak_tflops},
                     "traffic": prof_json.get("_k2_dram"),
                     "fp64_warp_insts_ncu": prof_json.get("_k2_fp64_insts")},
        "roofline_pass": {"bound": "fp64", "kernel": "gsb_prefill_pass: K1a, k_prefill_pass "
                                                     "(K1b + K2 in one persistent kernel), "
                                                     "finish, summary",
                          "achieved": pass_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
                          "frac": pass_tflops / peak_tflops, "kernel_ms": pass_ms,
                          "basis": f"{K2_DP_OPS_PER_EVAL} DP instr/evaluated triple + "
                                   f"{K1_DP_OPS_PER_REQ_PROFILE}/(request, profile) of K1b's "
                                   "ordered T_ref fold, x 2, vs the measured DFMA rate"},
        "roofline_k1": {"bound": "hbm", "kernel": "k_window_bounds + k_route_bin (K1)",
                        "achieved": k1_gbs, "peak": hbm, "unit": "GB/s", "frac": k1_gbs / hbm,
                        "kernel_ms": k1_ms, "algorithmic_bytes": k1_bytes,
                        "basis": "5 B/request (prompt i32 in, class u8 out) + 8 B per 32-request "
                                 "tile + (4 + 8P) B/cell",
                        "traffic": prof_json.get("_k1_dram")},
        "ingest": {"value": world * len(csv_text) / (ms_ing / 1e3) / 1e9,
                   "unit": "GB/s of trace CSV parsed (load_trace semantics)",
                   "rows_per_s": world * n_req / (ms_ing / 1e3), "ms_per_step": ms_ing,
                   "roofline": {"bound": "hbm", "achieved": (len(csv_text) * 2 + n_req * 21)
                                / (ms_ing / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                                "frac": (len(csv_text) * 2 + n_req * 21) / (ms_ing / 1e3) / 1e9
                                / hbm}},
        "fp64_peak_measured_dfma_per_s": dfma_per_s,
        "result": {"commands": int(glob["n_cmd"].sum()),
                   "infeasible": int(glob["n_infeasible"].sum()),
                   "empty_cells": int(glob["n_empty"].sum()),
                   "sum_energy_j_per_profile": [float(x) for x in glob["sum_energy_j"].sum(axis=1)]},
        "clocks": clk,
        "gpu_launches": launches,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if parity:
        line["parity_sample"] = parity
    # the decode half of the metric last: the driver keeps the tail of stdout
    line["pool"] = {"value": world * len(pcfg) / (ms_pool / 1e3),
                    "unit": "closed-loop decode-pool scenario replays/s",
                    "ms_per_step": ms_pool, "scenarios_per_step": len(pcfg),
                    "workload": "C3 sinusoid, 150 s, 4 decode workers x max_batch 64; K5 "
                                "k_decode_pool, one warp per scenario",
                    "roofline": issue_roof("k_decode_pool", len(pcfg), ms_pool),
                    "global_digest": int(gtally["digest"]),
                    "reduction": "per-rank scenario tallies, NCCL all-gather, rank-order combine"}
    line["decode"] = {"value": world * sweep.n_scenarios / (ms_dec / 1e3),
                      "unit": "decode-controller scenario replays/s",
                      "kind": "open-loop DecodeController replay (4 workers per scenario) over "
                              f"{tel.n_streams} shared telemetry streams: a controller "
                              "state-machine rate",
                      "ms_per_step": ms_dec, "k3a_ms": k3a_ms, "k3b_ms": k3b_ms,
                      "trajectories_per_step": len(sweep.cfgs),
                      "roofline": issue_roof("k_decode_replay", len(sweep.cfgs), k3b_ms)}
    print(json.dumps(line), flush=True)


def committed_profile():
    """Per-kernel ncu numbers committed under profiles/ (latest round): dram bytes and warp
    instructions per launch with the launch's work units (tools/summarize_profiles.py)."""
    import glob as _glob
    out = {}
    try:
        tj = sorted(_glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))[-1]
        out = json.load(open(tj))
    except (IndexError, OSError, ValueError):
        return out
    k2 = [v for k, v in out.items() if k.startswith("k_prefill_select")]
    if k2:
        out["_k2_dram"] = k2[0].get("dram_bytes_per_launch")
        out["_k2_fp64_insts"] = k2[0].get("fp64_insts")
    k1 = [v.get("dram_bytes_per_launch", 0) for k, v in out.items()
          if k.startswith("k_route_bin") or k.startswith("k_window_bounds")]
    out["_k1_dram"] = sum(k1) or None
    return out


def lscpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(args, sel, arrival, prompt, W, profs, thr, D, sweep, tel, plan, lo, hi, fo,
                 T_END):
    """The reference's CPU path (oracle/_ref, the unmodified reference sources) on this host:
    Dispatcher routing + select_frequency for every (window, class, profile) of THIS rank's
    whole trace with all host threads (the same config as the GPU arm), plus a 1-thread rate
    on a prefix of the windows. Its outputs are compared with the GPU's for EVERY cell and
    profile (grid index and energy bits)."""
    from oracle import oracle as O

    if not O.reference_available():
        return None, None
    ref = O.Reference()
    threads = os.cpu_count() or 1
    C, nW, wms = W["C"], W["W"], W["window_ms"]
    rp = [O.Profile(*p.key()) for p in profs]
    budget = args.cpu_seconds
    w0 = 0  # rank 0's windows (cpu_baseline runs at N = 1 only)
    # one untimed pass (first-touch page faults, thread start-up), then the timed passes
    fi_r, en_r, pairs = ref.prefill_pass(rp, thr, arrival, prompt, wms, w0, nW, D,
                                         threads=threads)
    reps, t_tot = 0, 0.0
    while reps < 2 or (t_tot < budget / 4 and reps < 8):
        t0 = time.perf_counter()
        ref.prefill_pass(rp, thr, arrival, prompt, wms, w0, nW, D, threads=threads, outputs=False)
        t_tot += time.perf_counter() - t0
        reps += 1
    dt_n = t_tot / reps
    # 1-thread rate on the first windows (about a second of work)
    n1 = max(1, min(nW, int(nW * min(1.0, 1.0 / max(dt_n * threads, 1e-3)))))
    s_end = int(np.searchsorted(arrival, (w0 + n1) * wms))
    t0 = time.perf_counter()
    _, _, pairs1 = ref.prefill_pass(rp, thr, arrival[:s_end], prompt[:s_end], wms, w0, n1, D,
                                    threads=1, outputs=False)
    dt_1 = time.perf_counter() - t0
    fi_g = sel.f_idx.cpu().numpy()
    en_g = sel.energy_j.cpu().numpy()
    per_prof = []
    for p in range(len(profs)):
        bad = (fi_g[p] != fi_r[p]) | (en_g[p].view(np.uint64) != en_r[p].view(np.uint64))
        per_prof.append({"profile": p, "cells": int(fi_g.shape[1]),
                         "commands": int((fi_r[p] != -2).sum()),
                         "infeasible": int((fi_r[p] == -1).sum()),
                         "mismatches": int(bad.sum())})
    pre = {"value": pairs * 81 / dt_n, "unit": "window x class x clock evals/s",
           "cores": threads, "kind": "reference", "seconds": dt_n,
           "value_1thread": pairs1 * 81 / dt_1, "seconds_1thread": dt_1,
           "cpu_model": lscpu_model(),
           "sample": f"the whole GPU workload ({nW} windows x {C} classes x {len(profs)} "
                     f"profiles, {len(arrival)} requests), mean of {reps} passes after one "
                     f"untimed: Dispatcher::dispatch/pop + select_frequency, one Dispatcher per "
                     f"std::thread over contiguous windows; 1-thread rate on the first {n1} "
                     f"windows"}
    # decode sample: full reference composition (windows + controller) per trajectory
    tels = []
    for s in range(tel.n_streams):
        e0, e1 = tel.ev_off[s], tel.ev_off[s + 1]
        go = tel.gap_off[e0:e1 + 1]
        tels.append(O.TelemetryArrays(tel.t_ms[e0:e1].copy(), tel.tokens[e0:e1].copy(),
                                      (go - go[0]).astype(np.int64), tel.gaps[go[0]:go[-1]].copy()))
    lo_h, hi_h, fo_h = lo.cpu().numpy(), hi.cpu().numpy(), fo.cpu().numpy()
    n_s = 8
    while True:
        idx = np.arange(min(len(sweep.cfgs), n_s * 4))
        cfgs = [O.CtlCfg(*[sweep.cfgs[i][n] for n in sweep.cfgs.dtype.names]) for i in idx]
        tabs_used = np.unique(sweep.table_of[idx])
        remap = {t: k for k, t in enumerate(tabs_used)}
        tables = [O.band_table(lo_h[t], hi_h[t], fo_h[t]) for t in tabs_used]
        t0 = time.perf_counter()
        nrec, dig = ref.replay_many(cfgs, tables, [remap[t] for t in sweep.table_of[idx]], tels,
                                    sweep.stream_of[idx], sweep.worker[idx], O.default_profile(),
                                    T_END, threads=threads)
        ddt = time.perf_counter() - t0
        if ddt > budget / 4 or len(idx) >= len(sweep.cfgs):
            break
        n_s = int(n_s * max(2.0, min(16.0, budget / 2 / max(ddt, 1e-4))))
    gd = plan["digest"].cpu().numpy().view(np.uint64)[idx]
    gn = plan["n_rec"].cpu().numpy()[idx]
    dmism = int(((gd != dig) | (gn != nrec)).sum())
    scen = len(idx) / 4
    pre["decode"] = {"value": scen / ddt, "unit": "decode-controller scenario replays/s",
                     "cores": threads, "kind": "reference", "seconds": ddt,
                     "sample": f"{int(scen)} scenarios x 4 workers x 150 s: DecodeController + "
                               f"TbtWindow + TpsWindow composed as Sim, {threads} std::threads"}
    parity = {"prefill": per_prof,
              "prefill_mismatches": int(sum(x["mismatches"] for x in per_prof)),
              "decode_trajectories_checked": int(len(idx)), "decode_digest_mismatches": dmism}
    return pre, parity


def ingest_cpu_baseline(args, csv_text: bytes):
    """greensim::load_trace (oracle/_ref, the unmodified reference) on a bounded prefix of the
    same CSV: one thread (the reference loader is a single sequential getline loop)."""
    import tempfile
    from oracle import oracle as O
    if not O.reference_available():
        return None
    ref = O.Reference()
    n = min(len(csv_text), 8 << 20)
    cut = csv_text.rfind(b"\n", 0, n) + 1
    with tempfile.NamedTemporaryFile(suffix=".csv", delete=False) as f:
        f.write(csv_text[:cut])
        path = f.name
    try:
        reps, t_tot = 0, 0.0
        while t_tot < args.cpu_seconds / 4 and reps < 20:
            t0 = time.perf_counter()
            r = ref.load_trace(path, 1024)
            t_tot += time.perf_counter() - t0
            reps += 1
    finally:
        os.remove(path)
    rows = len(r[0])
    return {"value": cut / (t_tot / reps) / 1e9, "unit": "GB/s of trace CSV parsed",
            "rows_per_s": rows / (t_tot / reps), "cores": 1, "kind": "reference",
            "sample": f"greensim::load_trace on the first {cut} bytes ({rows} rows) of the same "
                      f"CSV, {reps} reps"}


def pool_cpu_baseline(args, pa, pp, po, pstream, pcfg, psum):
    """K5's CPU reference: greensim::run() (oracle/_ref) per scenario on the same trace, all
    host threads, bounded sample; plus the restated decode pool (oracle, checker only) on the
    GPU's exact input stream for a few scenarios, compared field by field."""
    from oracle import oracle as O

    ref = O.Reference()
    restate = O.Restatement()
    threads = os.cpu_count() or 1
    prof, slo, scfg = O.default_profile(), O.default_slo(), O.default_sim_cfg()
    pol = O.PolicyHolder()
    names = pcfg.dtype.names
    n = max(threads, 8)
    budget = args.cpu_seconds
    while True:
        cfgs = [O.CtlCfg(*[pcfg[i][k] for k in names]) for i in range(min(n, len(pcfg)))]
        t0 = time.perf_counter()
        ref.sim_run_many(prof, pol, cfgs, slo, scfg, pa, pp, po, threads=threads)
        dt = time.perf_counter() - t0
        if dt > budget / 4 or n >= len(pcfg):
            break
        n = int(n * max(2.0, min(8.0, budget / 2 / max(dt, 1e-3))))
    cpu = {"value": len(cfgs) / dt, "unit": "closed-loop decode-pool scenario replays/s",
           "cores": threads, "kind": "reference", "seconds": dt,
           "sample": f"{len(cfgs)} scenarios of the C3 sweep: one greensim::run() each (150 s "
                     f"sinusoid, 4 decode workers), {threads} std::threads"}
    idx = np.linspace(0, len(pcfg) - 1, 6).astype(int)
    mism = 0
    for i in idx:
        c = O.CtlCfg(*[pcfg[i][k] for k in names])
        q = restate.pool_run(prof, O.PolicyHolder(ccfg=c), slo, scfg, pa, pp, po, pstream.t_ms,
                             pstream.req.astype(np.int64), pstream.end_floor_ms)
        mism += int(any(psum[k][i].item() != v for k, v in q["summary"].items()))
    return cpu, {"scenarios_checked": len(idx), "mismatches": mism}


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The reference's own CPU implementation of the path (oracle/_ref, the unmodified reference
    sources) on the SAME config as the gsb arm: rank 0's trace (same generator and seed), every
    window x class x profile: Dispatcher::dispatch/pop routing + select_frequency per non-empty
    (cell, profile), all host threads (one Dispatcher per thread over contiguous windows). The
    metric counts evaluated triples exactly as the gsb arm does."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2508_16449_b200 import workloads as wl
    if not O.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    ref = O.Reference()
    W = workload(args.config, args.windows)
    thr = wl.THRESHOLDS[W["C"]]
    threads = os.cpu_count() or 1
    nW, wms = W["W"], W["window_ms"]
    if W["shape"] == "mixed":
        arrival, prompt, _ = wl.mixed_trace(W["qps"], nW * wms, seed=1000, t0_ms=0)
    else:
        arrival, prompt, _ = wl.poisson_trace(W["qps"], nW * wms, W["shape"], seed=1000, t0_ms=0)
    profs = [O.Profile(*p.key()) for p in wl.synth_profiles(W["P"])]
    D = 0.95 * wms
    times, pairs = [], 0
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _, _, pairs = ref.prefill_pass(profs, thr, arrival, prompt, wms, 0, nW, D,
                                       threads=threads, outputs=False)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    dt = statistics.mean(times)
    v = pairs * 81 / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "window x class x clock evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (same generator, seed and config as the gsb arm's rank 0)",
        "config": {"workload": W["name"], "windows": nW, "classes": W["C"],
                   "profiles": W["P"], "clocks": 81, "requests": int(len(arrival)),
                   "evaluated_evals_per_step": pairs * 81, "same_config": True},
        "cpu_baseline": {"value": v, "unit": "window x class x clock evals/s", "cores": threads,
                         "kind": "reference", "cpu_model": lscpu_model(),
                         "sample": "the whole workload per step: Dispatcher::dispatch/pop + "
                                   "select_frequency per non-empty (window, class, profile), "
                                   f"{threads} std::threads"},
        "e2e": {"value": v, "unit": "window x class x clock evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if torch.cuda.is_available():  # the reference arm is host-only
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl" if args.impl == "gsb" else "gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_gsb(args, rank, world, dist)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
