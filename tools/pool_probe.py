"""Focused K5 (k_decode_pool) launcher for ncu / quick timing on one GPU:
python tools/pool_probe.py [n_scenarios] [launches]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_16449_b200 import api, workloads as wl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eng = api.Engine(0)
a, p, o = wl.sinusoid_decode_trace(1500.0, 1000.0, 120_000.0, 150_000, seed=11)
st = wl.decode_stream(a, p, o)
cfg = wl.pool_sweep(n)
plan = eng.decode_pool(cfg, st, api.GpuProfile.default_profile(), api.SimConfig(), api.SloConfig())
torch.cuda.synchronize()
s = torch.cuda.current_stream()
for r in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    eng.run_pool(plan)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"K5 {n} scenarios: {ms:.2f} ms -> {n / ms * 1e3:.4g} scenarios/s", flush=True)
sm = api.Engine.pool_summary(plan)
print("mean steps", sm["n_steps"].mean(), "decisions", sm["n_decisions"].mean(),
      "freq", sm["n_freq_changes"].mean(), "E", sm["decode_pool_j"].mean())
