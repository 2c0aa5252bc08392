"""Run one pass of one BASELINE config a few times (dev tool, for ncu captures).

usage: python tools/run_pass.py CFG PASS [REPS]     PASS in {fwd,bwd_d,bwd_w}
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.time_passes import CFGS  # noqa: E402
from paper_2104_08002_b200 import conv as cv  # noqa: E402

ci, pname = int(sys.argv[1]), sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
c = CFGS[ci]
w_in = c["q"] + c["d"] * (c["s"] - 1)
p = cv.ConvParams(c["c"], c["k"], c["s"], c["d"], c["prec"])
dt = torch.bfloat16 if c["prec"] == cv.Precision.Bf16 else torch.float32
x = torch.randn((c["n"], c["c"], w_in), device="cuda").to(dt)
dy = torch.randn((c["n"], c["k"], c["q"]), device="cuda").to(dt)
w = torch.randn((c["k"], c["c"], c["s"]), device="cuda") * 0.05
for _ in range(reps):
    if pname == "fwd":
        cv.conv1d_forward(x, w, p)
    elif pname == "bwd_d":
        cv.conv1d_backward_data(dy, cv.pack_weights_backward(w), p)
    else:
        cv.conv1d_backward_weight(dy, x, p)
torch.cuda.synchronize()
print("ok")
