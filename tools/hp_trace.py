import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2508_16449_b200 import api, workloads as wl
eng = api.Engine(0, wl.synth_profiles(4))
a, p, _ = wl.poisson_trace(5.0, 10000 * 60000, "alibaba_chat", seed=1000)
ha, hp = torch.as_tensor(a).pin_memory(), torch.as_tensor(p).pin_memory()
routing = api.RoutingConfig(True, wl.THRESHOLDS[8], list(range(8)))
for ch in (1, 4):
    r = eng.prefill_pass_host(ha, hp, routing, 60000, 0, 10000, api.L.FIXED_WINDOW, fixed_window_ms=57000.0, chunks=ch)
    torch.cuda.synchronize()
    for i in range(3):
        if i == 2: os.environ["GSB_HP_TRACE"] = "1"; print("== chunks", ch, file=sys.stderr, flush=True)
        eng.prefill_pass_host(ha, hp, routing, 60000, 0, 10000, api.L.FIXED_WINDOW, fixed_window_ms=57000.0, chunks=ch, out=r)
        torch.cuda.synchronize()
    os.environ.pop("GSB_HP_TRACE")
