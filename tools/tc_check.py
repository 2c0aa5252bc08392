"""Quick tcgen05-path check on the GPU (dev tool): run the three passes on a few d=8 shapes with
algo=auto (tensor-core where supported) and report the algorithm and error vs the oracle."""
import sys
import os
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2104_08002_b200 import conv as cv  # noqa: E402

shapes = [(1, 16, 16, 51, 8, 256), (2, 15, 15, 51, 8, 1000), (1, 64, 64, 51, 8, 512), (2, 64, 64, 51, 8, 1024),
          (1, 32, 32, 9, 8, 640), (3, 4, 15, 5, 8, 384), (1, 100, 70, 51, 8, 256)]
if len(sys.argv) > 1:
    shapes = shapes[: int(sys.argv[1])]
ok = True
for (n, c, k, s, d, q) in shapes:
    rng = oracle.Rng(7)
    w_in = q + d * (s - 1)
    x, w, dy = rng.fill_uniform((n, c, w_in)), rng.fill_uniform((k, c, s)), rng.fill_uniform((n, k, q))
    xr, wr, dyr = oracle.round_bf16(x), oracle.round_bf16(w), oracle.round_bf16(dy)
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    algos = [cv.selected_algo(p, n, w_in, i, in_dtype=0) for i in range(3)]
    t0 = time.time()
    y = cv.conv1d_forward(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), p)
    dx = cv.conv1d_backward_data(torch.from_numpy(dy).cuda(), cv.pack_weights_backward(torch.from_numpy(w).cuda()), p)
    dw = cv.conv1d_backward_weight(torch.from_numpy(dy).cuda(), torch.from_numpy(x).cuda(), p)
    torch.cuda.synchronize()
    e = [oracle.norm_rel_error(y.cpu().numpy(), oracle.naive_forward(xr, wr, d)),
         oracle.norm_rel_error(dx.cpu().numpy(), oracle.naive_backward_data(dyr, wr, d)),
         oracle.norm_rel_error(dw.cpu().numpy(), oracle.naive_backward_weight(dyr, xr, s, d))]
    good = all(np.isfinite(v) and v <= 1e-5 for v in e)
    ok &= good
    print(f"{(n, c, k, s, d, q)} algos={algos} err={['%.2e' % v for v in e]} {'OK' if good else 'FAIL'} "
          f"({time.time() - t0:.2f}s)", flush=True)
print("ALL OK" if ok else "FAILURES")
