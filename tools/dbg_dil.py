import sys, os
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import oracle
from paper_2104_08002_b200 import conv as cv
n, c, k, s, d, q = (int(a) for a in sys.argv[1:7])
which = sys.argv[7]
w_in = q + d * (s - 1)
rng = oracle.Rng(5)
x, w, dy = rng.fill_uniform((n, c, w_in)), rng.fill_uniform((k, c, s)), rng.fill_uniform((n, k, q))
p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
xt, wt, gt = (torch.from_numpy(a).cuda() for a in (x, w, dy))
print('algo', [cv.selected_algo(p, n, w_in, i, in_dtype=0) for i in range(3)], flush=True)
if which == 'fwd':
    r = cv.conv1d_forward(xt, wt, p); want = oracle.naive_forward(oracle.round_bf16(x), oracle.round_bf16(w), d)
elif which == 'bwd_d':
    r = cv.conv1d_backward_data(gt, cv.pack_weights_backward(wt), p); want = oracle.naive_backward_data(oracle.round_bf16(dy), oracle.round_bf16(w), d)
else:
    r = cv.conv1d_backward_weight(gt, xt, p); want = oracle.naive_backward_weight(oracle.round_bf16(dy), oracle.round_bf16(x), s, d)
torch.cuda.synchronize()
print(which, 'err', oracle.norm_rel_error(r.cpu().numpy(), want), flush=True)
