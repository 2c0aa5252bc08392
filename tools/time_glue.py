"""Per-launch times of the glued conv passes vs the plain ones at the config-5 body-layer shape
(dev tool): python tools/time_glue.py [N] [Q]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_08002_b200 import conv as cv  # noqa: E402
from paper_2104_08002_b200.network import conv_backward_data_glued, conv_forward_glued, mask_shape  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
q = int(sys.argv[2]) if len(sys.argv) > 2 else 60000
c = k = 15
s, d = 51, 8
pad = d * (s - 1) // 2
p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
dev = "cuda"
x = cv.round_bf16(torch.randn((n, c, q + 2 * pad), device=dev))
w = torch.randn((k, c, s), device=dev) * 0.05
b = torch.randn(k, device=dev) * 0.1
y = torch.empty((n, k, q), device=dev)
skip = torch.randn((n, k, q), device=dev)
act = torch.empty((n, k, q), device=dev)
act_b = torch.zeros((n, k, q + 2 * pad), dtype=torch.bfloat16, device=dev)
mask = torch.zeros(mask_shape(n, k, q), dtype=torch.int32, device=dev)
dy = cv.round_bf16(torch.randn((n, k, q), device=dev))
dx = torch.empty((n, c, q + 2 * pad), device=dev)
gadd = torch.randn((n, c, q), device=dev)
gsum = torch.empty((n, c, q), device=dev)
gp = torch.empty((n, c, q), dtype=torch.bfloat16, device=dev)
db = torch.empty(c, device=dev)


def timeit(name, fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:42s} {e0.elapsed_time(e1) / reps * 1e3:9.1f} us")


timeit("forward plain", lambda: cv.conv1d_forward(x, w, p, out=y))
timeit("forward glued (act_bf16 + mask)", lambda: conv_forward_glued(x, w, p, bias=b, act_bf16=act_b, act_pad=pad,
                                                                     mask=mask))
timeit("forward glued (+skip, act, act_bf16, mask)",
       lambda: conv_forward_glued(x, w, p, bias=b, skip=skip, act=act, act_bf16=act_b, act_pad=pad, mask=mask))
timeit("backward-data plain", lambda: cv.conv1d_backward_data(dy, w, p, out=dx))
timeit("backward-data glued (mask, gp_bf16, db)",
       lambda: conv_backward_data_glued(dy, w, p, pad, q, mask=mask, grad_pre_bf16=gp, bias_grad=db))
timeit("backward-data glued (+gadd, gsum)",
       lambda: conv_backward_data_glued(dy, w, p, pad, q, gadd=gadd, mask=mask, gsum=gsum, grad_pre_bf16=gp,
                                        bias_grad=db))
