import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2104_08002_b200 import conv as cv
# FP32 config-4 points on the FFMA kernels: (C, S, d, pass)
cases = [(16, 9, 1, "bwd_w"), (64, 3, 1, "fwd"), (16, 3, 1, "fwd")]
for c, s, d, ps in cases:
    n, q = 16, 20000
    p = cv.ConvParams(c, c, s, d, cv.Precision.Fp32)
    x = torch.randn(n, c, q + d * (s - 1), device="cuda")
    dy = torch.randn(n, c, q, device="cuda")
    w = torch.randn(c, c, s, device="cuda") * 0.1
    for _ in range(3):
        if ps == "fwd":
            cv.conv1d_forward(x, w, p)
        else:
            cv.conv1d_backward_weight(dy, x, p)
    torch.cuda.synchronize()
