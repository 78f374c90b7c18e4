"""K6 launch list (run under ncu --metrics gpu__time_duration.sum) and end-to-end parse time of
the bench's C4 CSV: python tools/k6_probe.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_16449_b200 import api, workloads as wl  # noqa: E402

eng = api.Engine(0, wl.synth_profiles(4))
a, p, _ = wl.poisson_trace(5.0, 10_000 * 60_000, "alibaba_chat", seed=1000)
d_arr, d_prm = torch.as_tensor(a, device="cuda"), torch.as_tensor(p, device="cuda")
csv = eng.format_trace(d_arr, d_prm, torch.full_like(d_prm, 128), (d_prm > 1024).to(torch.uint8))
d_csv = torch.frombuffer(bytearray(csv), dtype=torch.uint8).to("cuda")
for _ in range(3):
    eng.parse_trace(d_csv)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    eng.parse_trace(d_csv)
torch.cuda.synchronize()
print(f"{len(csv) / 1e6:.1f} MB, {(time.perf_counter() - t0) / 10 * 1e6:.1f} us per parse (wall)")
