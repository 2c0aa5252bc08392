"""Isolate the tail-tap path of tc_conv (dev tool): zero either the tail taps or the main taps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2104_08002_b200 import conv as cv  # noqa: E402

n, c, k, s, q = 1, 64, 64, 51, 512
w_in = q + 8 * (s - 1)
rng = oracle.Rng(7)
x, w = rng.fill_uniform((n, c, w_in)), rng.fill_uniform((k, c, s))
p = cv.ConvParams(c, k, s, 8, cv.Precision.Bf16)
for name, sl in (("tail only", slice(0, 48)), ("main only", slice(48, 51)), ("full", slice(0, 0))):
    ww = w.copy()
    ww[:, :, sl] = 0
    y = cv.conv1d_forward(torch.from_numpy(x).cuda(), torch.from_numpy(ww).cuda(), p).cpu().numpy()
    want = oracle.naive_forward(oracle.round_bf16(x), oracle.round_bf16(ww), 8)
    err = oracle.norm_rel_error(y, want)
    bad = np.abs(y - want) > 1e-3 * np.abs(want).max()
    cols = np.nonzero(bad.any(axis=(0, 1)))[0]
    chans = np.nonzero(bad.any(axis=(0, 2)))[0]
    print(f"{name}: err {err:.3e} bad cols {cols[:8]}..{cols[-4:] if len(cols) else ''} ({len(cols)}) chans {chans[:8]} ({len(chans)})")
    if name == "tail only" and len(cols):
        j, o = cols[0], chans[0]
        print("  y", y[0, o, j:j + 4], "want", want[0, o, j:j + 4])
