"""Kernel-time breakdown of one config-5 network step (dev tool, torch.profiler)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_08002_b200 import conv as cv  # noqa: E402
from paper_2104_08002_b200.network import ResidualNet, train_step  # noqa: E402

per = int(sys.argv[1]) if len(sys.argv) > 1 else 64
net = ResidualNet(precision=cv.Precision.Bf16, seed=1)
pad = net.pad()
x = torch.poisson(torch.full((per, 1, 60000 + 2 * pad), 2.0, device="cuda"))
t = torch.poisson(torch.full((per, 1, 60000), 2.0, device="cuda"))
lab = (torch.rand((per, 1, 60000), device="cuda") < 0.1).float()
for _ in range(3):
    train_step(net, x, t, lab)
    net.sgd_step(1e-3)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    train_step(net, x, t, lab)
    net.sgd_step(1e-3)
    torch.cuda.synchronize()
tot = 0.0
rows = []
for e in prof.key_averages():
    t = getattr(e, "self_device_time_total", 0) or getattr(e, "self_cuda_time_total", 0)
    if t > 0:
        rows.append((t, e.count, e.key))
        tot += t
rows.sort(reverse=True)
for t, c, k in rows[:25]:
    print(f"{t / 1e3:8.3f} ms {t / tot * 100:5.1f}% n={c:4d}  {k[:90]}")
print(f"total {tot / 1e3:.3f} ms")
