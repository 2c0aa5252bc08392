"""Time one pass on an ad-hoc d=8 BF16 shape (dev tool).

usage: python tools/time_shape.py N C K S Q [pass ...]     pass in {fwd,bwd_d,bwd_w}
(env D = dilation, default 8)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_08002_b200 import conv as cv  # noqa: E402

n, c, k, s, q = (int(a) for a in sys.argv[1:6])
passes = sys.argv[6:] or ["fwd", "bwd_d", "bwd_w"]
dil = int(os.environ.get("D", "8"))
w_in = q + dil * (s - 1)
p = cv.ConvParams(c, k, s, dil, cv.Precision.Bf16)
x = torch.randn((n, c, w_in), device="cuda").bfloat16()
dy = torch.randn((n, k, q), device="cuda").bfloat16()
w = torch.randn((k, c, s), device="cuda") * 0.05
y = torch.empty((n, k, q), device="cuda")
dx = torch.empty((n, c, w_in), device="cuda")
dw = torch.empty((k, c, s), device="cuda")
wb = cv.pack_weights_backward(w)
wf = w if os.environ.get("KCS") else cv.pack_weights_forward(w)  # KCS=1: pack inside every call
flush = torch.empty(64 * 1024 * 1024, device="cuda")
fn = {"fwd": lambda: cv.conv1d_forward(x, wf, p, out=y), "bwd_d": lambda: cv.conv1d_backward_data(dy, wb, p, out=dx),
      "bwd_w": lambda: cv.conv1d_backward_weight(dy, x, p, out=dw)}
flops = cv.conv_flops(p, n, q)
for name in passes:
    f = fn[name]
    for _ in range(3):
        f()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(f"N={n} C={c} K={k} S={s} d={dil} Q={q} {name:6s} median {ts[5]:8.1f} us  {flops / ts[5] / 1e6:7.1f} TFLOP/s")
