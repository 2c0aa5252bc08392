"""Replay acceptance criterion 1's draws (acceptance.cpp:66-135, Rng(101), 220 combos) through the
Python API and report the worst-error combos per pass and algorithm (dev tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2104_08002_b200 import conv as cv  # noqa: E402

rng = oracle.Rng(101)
widths, chans = [1000, 2000], [1, 4, 8, 10, 15, 16, 32, 64]
taps, dils = [1, 5, 9, 15, 21, 25, 31, 49, 51], [1, 2, 4, 8, 16]
rows = []
done = 0
while done < 220:
    c, k = chans[rng.next_below(8)], chans[rng.next_below(8)]
    s, d = taps[rng.next_below(9)], dils[rng.next_below(5)]
    q = widths[rng.next_below(2)]
    n = 1 + rng.next_below(4)
    w_in = q + d * (s - 1)
    if n * c * k * s * w_in > 100_000_000:
        continue
    x, w, dy = rng.fill_uniform((n, c, w_in)), rng.fill_uniform((k, c, s)), rng.fill_uniform((n, k, q))
    done += 1
    if d != 8:
        continue  # only the tensor-core paths are of interest here
    p = cv.ConvParams(c, k, s, d)
    xt, wt, gt = (torch.from_numpy(a).cuda() for a in (x, w, dy))
    res = [cv.conv1d_forward(xt, wt, p), cv.conv1d_backward_data(gt, cv.pack_weights_backward(wt), p),
           cv.conv1d_backward_weight(gt, xt, p)]
    want = [oracle.naive_forward(x, w, d), oracle.naive_backward_data(dy, w, d), oracle.naive_backward_weight(dy, x, s, d)]
    for j in range(3):
        err = oracle.norm_rel_error(res[j].cpu().numpy(), want[j])
        rows.append((err, ("fwd", "bwd_d", "bwd_w")[j], cv.selected_algo(p, n, w_in, j, in_dtype=0), (n, c, k, s, d, q)))
rows.sort(reverse=True)
for r in rows[:15]:
    print(f"{r[0]:.3e} {r[1]:6s} {r[2]:7s} {r[3]}")
