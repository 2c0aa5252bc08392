"""Run backward-weight once on a small d=8 shape and compare with the oracle (dev tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2104_08002_b200 import conv as cv  # noqa: E402

n, c, k, s, q = (int(a) for a in (sys.argv[1:6] if len(sys.argv) > 5 else (1, 16, 16, 51, 256)))
rng = oracle.Rng(7)
w_in = q + 8 * (s - 1)
x, dy = rng.fill_uniform((n, c, w_in)), rng.fill_uniform((n, k, q))
p = cv.ConvParams(c, k, s, 8, cv.Precision.Bf16)
print("algo", cv.selected_algo(p, n, w_in, 2, in_dtype=0))
dw = cv.conv1d_backward_weight(torch.from_numpy(dy).cuda(), torch.from_numpy(x).cuda(), p)
torch.cuda.synchronize()
want = oracle.naive_backward_weight(oracle.round_bf16(dy), oracle.round_bf16(x), s, 8)
print("err", oracle.norm_rel_error(dw.cpu().numpy(), want))
