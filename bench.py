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
K2_DP_OPS_PER_EVAL = 15  # DP-pipe instructions per (cell, clock) in k_prefill_select (SASS)
K1_BYTES_PER_REQ = 8 + 4 + 1  # arrival i64 + prompt i32 read, class u8 written


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
    w0 = rank * nW
    t0 = w0 * wms
    if W["shape"] == "mixed":
        arrival, prompt, _ = wl.mixed_trace(W["qps"], nW * wms, seed=1000 + rank, t0_ms=t0)
    else:
        arrival, prompt, _ = wl.poisson_trace(W["qps"], nW * wms, W["shape"], seed=1000 + rank,
                                              t0_ms=t0)
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

    def prefill_step(mark=False):
        if mark:
            ev[0].record(stream)
        eng.route_bin(d_arr, d_prm, routing, wms, w0, nW, out=rr)
        if mark:
            ev[1].record(stream)
        # K2 + the per-class summary: one launch (objective, argmin, reduction)
        eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=D, out=sel, summary_out=summ)
        if mark:
            ev[2].record(stream)

    use_graph = not args.no_graph
    graphs = {}
    if use_graph:
        for _ in range(2):
            prefill_step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            prefill_step()
        graphs["prefill"] = g

    def run_prefill(timed_steps, warm):
        t_step, t_k1, t_k2 = [], [], []
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
            if i >= warm:
                t_step.append((s0, s1))
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in t_step]

    # per-kernel split (separate, eager, with events between the kernels)
    def kernel_split(n=5):
        k1, k2 = [], []
        for _ in range(n):
            flush.zero_()
            prefill_step(mark=True)
            ev[3].record(stream)
            torch.cuda.synchronize()
            k1.append(ev[0].elapsed_time(ev[1]))
            k2.append(ev[1].elapsed_time(ev[2]))
        return statistics.median(k1), statistics.median(k2)

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
    h2d = h_arr.numel() * 8 + h_prm.numel() * 4
    d2h = h_fidx.numel() * 2 + h_en.numel() * 8

    def e2e_step():
        d_arr.copy_(h_arr, non_blocking=True)
        d_prm.copy_(h_prm, non_blocking=True)
        prefill_step()
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
        pre_ms = run_prefill(args.steps, args.warmup)
        barrier()
        dec_ms = run_decode(args.steps, max(3, args.warmup // 2))
        barrier()
        pool_ms = run_pool(max(3, args.steps // 4), 3)
        barrier()
        e2e_ms = run_e2e(args.steps, args.warmup)
        barrier()
        ing_ms = run_ingest(max(3, args.steps // 4), 3)
        barrier()
    k1_ms, k2_ms = kernel_split()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_pre = max_over_ranks(statistics.mean(pre_ms))
    ms_dec = max_over_ranks(statistics.mean(dec_ms))
    ms_e2e = max_over_ranks(statistics.mean(e2e_ms))
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
    glob = Dd.combine_summaries(per_rank, [r * nW * W["C"] for r in range(world)])

    # ---------------- parity spot check + CPU baseline (rank 0, checker only)
    cpu = None
    parity = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        cpu, parity = cpu_baseline(args, eng, rr, sel, arrival, prompt, W, profs, thr, D, sweep,
                                   tel, plan, lo, hi, fo, T_END)
        if cpu is not None:
            cpu["pool"], parity["pool"] = pool_cpu_baseline(args, pa, pp, po, pstream, pcfg,
                                                            psum)
            cpu["ingest"] = ingest_cpu_baseline(args, csv_text)

    if rank != 0:
        return
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    traffic_k2 = traffic_k1 = None  # dram bytes per launch from the committed ncu capture
    try:
        import glob as _glob
        tj = sorted(_glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))[-1]
        tr = json.load(open(tj))
        traffic_k2 = next((v["dram_bytes_per_launch"] for k, v in tr.items()
                           if k.startswith("k_prefill_select")), None)
        traffic_k1 = sum(v["dram_bytes_per_launch"] for k, v in tr.items()
                         if k.startswith("k_route_bin") or k.startswith("k_window_bounds")) or None
    except (IndexError, OSError, ValueError, KeyError):
        pass
    # executed K2 work: only non-empty (cell, profile) pairs run the 81-clock loop (empty
    # queues give no command, prefill_opt.cpp:64, and are compacted away inside K2)
    evaluated = int(per_rank[rank]["n_cmd"].sum()) * 81
    k2_tflops = evaluated * K2_DP_OPS_PER_EVAL * 2 / (k2_ms / 1e3) / 1e12
    peak_tflops = dfma_per_s * 2 / 1e12
    k1_gbs = n_req * K1_BYTES_PER_REQ / (k1_ms / 1e3) / 1e9
    # timed launches of our kernels: prefill step = window_bounds + route_bin + prefill_select
    # with the fused summary partials + summary final (4); decode step = tbt_p95 + tps +
    # decode_replay (3); e2e = 4
    # + pool (1 per step) + ingest (K6: count, header end, parse, monotone per call; the CUB
    # scan is library code)
    launches = args.steps * (4 + 3 + 4) + max(3, args.steps // 4) + 4 * max(3, args.steps // 4)
    line = {
        "metric": METRIC,
        "value": world * evals / (ms_pre / 1e3),
        "unit": "window x class x clock evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_pre,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference-shaped Poisson/bimodal traces; sinusoidal decode telemetry)",
        "config": {"workload": W["name"], "windows_per_gpu": nW, "window_ms": wms,
                   "classes": W["C"], "profiles": P, "clocks": 81, "requests_per_gpu": n_req,
                   "evals_per_step_per_gpu": evals,
                   "evaluated_evals_per_step_per_gpu": evaluated,
                   "value_counts": "every (window, class, profile, clock) triple of the grid is "
                                   "decided each step; empty cells are decided as 'no command' "
                                   "without evaluation (prefill_opt.cpp:64); the roofline counts "
                                   "only the evaluated triples",
                   "window_mode": "FIXED_WINDOW D=0.95*W",
                   "decode_scenarios_per_gpu": sweep.n_scenarios, "decode_horizon_ms": T_END,
                   "parallelism": f"dp{world} (windows/scenarios sharded, NCCL all-gather of "
                                  f"per-class summaries)",
                   "l2": "flushed between timed steps (256 MB write, outside the events)",
                   "cuda_graphs": use_graph},
        "e2e": {"value": world * evals / (ms_e2e / 1e3), "unit": "window x class x clock evals/s",
                "ms_per_step": ms_e2e, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "public API (Engine.route_bin/prefill_select) from pinned host buffers"},
        "decode": {"value": world * sweep.n_scenarios / (ms_dec / 1e3),
                   "unit": "decode-controller scenario replays/s",
                   "fine_ticks_per_s": world * sweep.n_scenarios * 4 * 7500 / (ms_dec / 1e3),
                   "ms_per_step": ms_dec, "trajectories_per_step": len(sweep.cfgs)},
        "pool": {"value": world * len(pcfg) / (ms_pool / 1e3),
                 "unit": "closed-loop decode-pool scenario replays/s",
                 "decode_steps_per_s": world * float(psum["n_steps"].sum()) / (ms_pool / 1e3),
                 "events_per_scenario": float((psum["n_steps"] + psum["n_decisions"]
                                               + psum["n_freq_changes"]).mean() + len(pstream.t_ms)),
                 "ms_per_step": ms_pool, "scenarios_per_step": len(pcfg),
                 "workload": "C3 sinusoid 1500+-1000 tps, 150 s, 4 decode workers x max_batch 64; "
                             "sweep hysteresis x step x TBT target x margin x bias; K5 "
                             "k_decode_pool, one warp per scenario",
                 "mean_decode_pool_j": float(psum["decode_pool_j"].mean()),
                 "global_tally": {k: (int(gtally[k]) if gtally.dtype[k].kind in "iu"
                                      else float(gtally[k])) for k in gtally.dtype.names},
                 "reduction": "per-rank scenario tallies, NCCL all-gather, rank-order combine"},
        "roofline": {"bound": "fp64", "kernel": "k_prefill_select (K2)",
                     "achieved": k2_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
                     "frac": k2_tflops / peak_tflops,
                     "basis": f"{K2_DP_OPS_PER_EVAL} DP-pipe instr per EVALUATED (non-empty "
                              "cell, profile, clock) x 2 (DFMA-equivalent) vs DFMA throughput "
                              "measured in this run (gsb_fp64_probe); kernel time includes the "
                              "fused per-class summary and its final combine",
                     "kernel_ms": k2_ms, "share_of_step": k2_ms / ms_pre, "traffic": traffic_k2,
                     "traffic_note": "dram__bytes_read+write per launch, profiles/ ncu capture"},
        "ingest": {"value": world * len(csv_text) / (ms_ing / 1e3) / 1e9,
                   "unit": "GB/s of trace CSV parsed (load_trace semantics)",
                   "rows_per_s": world * n_req / (ms_ing / 1e3), "ms_per_step": ms_ing,
                   "csv_bytes_per_step": len(csv_text), "rows_per_step": n_req,
                   "workload": "this rank's trace rendered by save_trace_csv (4 columns), "
                               "device-resident bytes -> SoA via gsb_trace_parse (K6: count, scan, "
                               "parse, monotone check; two host syncs per call)",
                   "roofline": {"bound": "hbm", "achieved": (len(csv_text) * 2 + n_req * 21)
                                / (ms_ing / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                                "frac": (len(csv_text) * 2 + n_req * 21) / (ms_ing / 1e3) / 1e9
                                / hbm,
                                "basis": "CSV bytes read twice (count + parse passes) + 17 B/row "
                                         "written + 4 B/row line index"}},
        "roofline_k1": {"bound": "hbm", "kernel": "k_route_bin (K1)", "achieved": k1_gbs,
                        "peak": hbm, "unit": "GB/s", "frac": k1_gbs / hbm, "kernel_ms": k1_ms,
                        "bytes_per_request": K1_BYTES_PER_REQ,
                        "traffic": traffic_k1},
        "fp64_peak_measured_dfma_per_s": dfma_per_s,
        "result": {"commands": int(glob["n_cmd"].sum()),
                   "infeasible": int(glob["n_infeasible"].sum()),
                   "empty_cells": int(glob["n_empty"].sum()),
                   "sum_energy_j_per_profile": [float(x) for x in glob["sum_energy_j"].sum(axis=1)]},
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if parity:
        line["parity_sample"] = parity
    print(json.dumps(line), flush=True)


def cpu_baseline(args, eng, rr, sel, arrival, prompt, W, profs, thr, D, sweep, tel, plan, lo, hi,
                 fo, T_END):
    """Reference CPU path (oracle/_ref, the unmodified reference sources) on a bounded sample
    of the same workload, all host threads; also bit-checks the GPU outputs on that sample."""
    import torch
    from oracle import oracle as O

    if not O.reference_available():
        return None, None
    ref = O.Reference()
    threads = os.cpu_count() or 1
    C = W["C"]
    # prefill sample: the FIFO job lists of the first windows (Dispatcher order)
    cls = rr.cls.cpu().numpy()
    cnt = rr.count.cpu().numpy().view(np.uint32)
    bounds = rr.bounds.cpu().numpy()
    n_w = 1
    t_rate = None
    res = {}
    budget = args.cpu_seconds
    while True:
        s_end = bounds[n_w]
        key = (arrival[:s_end] // W["window_ms"] - rr.w0) * C + cls[:s_end]
        order = np.argsort(key, kind="stable")
        ncell = n_w * C
        off = np.concatenate([[0], np.cumsum(cnt[:ncell])]).astype(np.int64)
        prompts = prompt[order].astype(np.int32)
        nonempty = np.nonzero(cnt[:ncell])[0]
        t0 = time.perf_counter()
        f, e, found = ref.select_many(O.Profile(*profs[0].key()), off, prompts,
                                      np.full(ncell, D), threads=threads)
        dt = time.perf_counter() - t0
        if dt > budget / 4 or n_w >= rr.n_windows:
            break
        n_w = min(rr.n_windows, int(n_w * max(2.0, min(16.0, budget / 2 / max(dt, 1e-4)))))
    # repeat the sample until the time budget is used (bounded CPU work, stable rate)
    reps, t_tot = 1, dt
    while t_tot < budget / 2:
        t0 = time.perf_counter()
        ref.select_many(O.Profile(*profs[0].key()), off, prompts, np.full(ncell, D),
                        threads=threads)
        t_tot += time.perf_counter() - t0
        reps += 1
    dt = t_tot / reps
    evals = ncell * 81
    fi = sel.f_idx.cpu().numpy()[0, :ncell]
    en = sel.energy_j.cpu().numpy()[0, :ncell]
    gf = np.where(fi >= 0, 210.0 + 15.0 * fi, 0.0)
    mism = int(((fi[nonempty] >= 0) != found[nonempty]).sum()
               + (found[nonempty] & ((gf[nonempty] != f[nonempty])
                                     | (en[nonempty] != e[nonempty]))).sum())
    pre = {"value": evals / dt, "unit": "window x class x clock evals/s", "cores": threads,
           "kind": "reference", "seconds": dt,
           "sample": f"{n_w} windows x {C} classes (profile 0) of this rank's trace through "
                     f"greensim::select_frequency on the FIFO job lists, {threads} std::threads"}
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
    dec = {"value": scen / ddt, "unit": "decode-controller scenario replays/s", "cores": threads,
           "kind": "reference", "seconds": ddt,
           "sample": f"{int(scen)} scenarios x 4 workers x 150 s: DecodeController + TbtWindow + "
                     f"TpsWindow composed as Sim, {threads} std::threads"}
    pre["decode"] = dec
    parity = {"prefill_cells_checked": int(len(nonempty)), "prefill_mismatches": mism,
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
    """The reference's own CPU implementation of the path (oracle/_ref) on the same config,
    all host threads, each step a bounded sample."""
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
    n_w = min(W["W"], 600)
    if W["shape"] == "mixed":
        arrival, prompt, _ = wl.mixed_trace(W["qps"], n_w * W["window_ms"], seed=1000)
    else:
        arrival, prompt, _ = wl.poisson_trace(W["qps"], n_w * W["window_ms"], W["shape"], seed=1000)
    C = W["C"]
    t_route0 = time.perf_counter()
    q, _, _ = ref.dispatch(thr, prompt)
    t_route = time.perf_counter() - t_route0
    key = (arrival // W["window_ms"]) * C + q
    order = np.argsort(key, kind="stable")
    cnt = np.bincount(key, minlength=n_w * C)[: n_w * C]
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    prof = O.default_profile()
    D = 0.95 * W["window_ms"]
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ref.select_many(prof, off, prompt[order], np.full(n_w * C, D), threads=threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0 + t_route)
    dt = statistics.mean(times)
    evals = n_w * C * 81
    v = evals / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "window x class x clock evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (same generator and config as the gsb arm)",
        "config": {"workload": W["name"], "sample_windows": n_w, "classes": C, "profiles": 1},
        "cpu_baseline": {"value": v, "unit": "window x class x clock evals/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"{n_w} one-minute windows x {C} classes per step: Dispatcher "
                                   f"routing + select_frequency per cell, {threads} threads"},
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
