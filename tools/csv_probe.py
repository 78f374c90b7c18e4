import sys; sys.path.insert(0, ".")
from paper_2508_16449_b200 import api
import torch
from oracle.oracle import Restatement
R = Restatement(); a, p, o = R.gen_poisson_trace(5.0, 600_000_000, seed=3)
e = api.Engine(0); txt = e.format_trace(a, p, o, (p > 1024).astype("uint8"))
d = torch.frombuffer(bytearray(txt), dtype=torch.uint8).cuda()
for _ in range(2): e.parse_trace(d)
