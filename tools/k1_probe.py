"""K1b with and without the non-empty list, 8 eager launches each (run under ncu for per-launch
device times): python tools/k1_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_16449_b200 import api, workloads as wl  # noqa: E402

C, P, nW, wms = 8, 4, 10_000, 60_000
eng = api.Engine(0, wl.synth_profiles(P))
a, p, _ = wl.poisson_trace(5.0, nW * wms, "alibaba_chat", seed=1000)
da, dp = torch.as_tensor(a, device="cuda"), torch.as_tensor(p, device="cuda")
routing = api.RoutingConfig(True, wl.THRESHOLDS[C], list(range(C)))
rr = eng.route_bin(da, dp, routing, wms, 0, nW)
rn = eng.route_bin(da, dp, routing, wms, 0, nW)
rn.nonempty = rn.n_nonempty = rn.t_ref_list = None
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for r in [rr] * 8 + [rn] * 8:
    flush.zero_()
    eng.route_bin(da, dp, routing, wms, 0, nW, out=r)
torch.cuda.synchronize()
