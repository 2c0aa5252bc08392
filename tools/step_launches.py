"""Run the bench's device step (config-3 layer: forward, backward-data, backward-weight through
the C ABI) a few times and nothing else, for an ncu launch list of one step (dev tool).

usage: python tools/step_launches.py [steps]
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_08002_b200 import _lib as L  # noqa: E402
from paper_2104_08002_b200 import conv as cv  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n, c, k, s, d, q = 32, 64, 64, 51, 8, 60000
w_in = q + d * (s - 1)
p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn((n, c, w_in), device="cuda", generator=g).bfloat16()
dy = torch.randn((n, k, q), device="cuda", generator=g).bfloat16()
w = torch.randn((k, c, s), device="cuda", generator=g) * 0.0429
y = torch.empty((n, k, q), device="cuda")
dx = torch.empty((n, c, w_in), device="cuda")
dw = torch.empty((k, c, s), device="cuda")
lib = L.lib()
desc = cv.make_desc(p, n, w_in, L.DTYPE_BF16)
sp = torch.cuda.current_stream().cuda_stream
torch.cuda.synchronize()
for _ in range(steps):
    assert lib.c1d_forward(C.byref(desc), x.data_ptr(), w.data_ptr(), y.data_ptr(), None, 0, sp) == 0
    assert lib.c1d_backward_data(C.byref(desc), dy.data_ptr(), w.data_ptr(), dx.data_ptr(), None, 0, sp) == 0
    assert lib.c1d_backward_weight(C.byref(desc), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), None, 0, sp) == 0
torch.cuda.synchronize()
print("ok", lib.c1d_launch_count())
