"""The performance switches (DESIGN.md §5 "Developer switches") change how data moves, not what is
computed: with programmatic dependent launch off, resident weights off or the one-box-per-stage
TMA view off, every pass gives bit-identical results. The switches are read once per process, so
each setting runs in a subprocess (same seeded inputs) and the outputs are compared bitwise."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (C, K, S, d, Q, N): the narrow body layer (resident weights, one-box stages, split carry), an
# odd width whose last super-tile takes the per-channel boxes, a wide layer (streamed weights, tail
# taps) and an expanded-row dilation
SHAPES = [(15, 15, 51, 8, 6000, 3), (15, 15, 51, 8, 3001, 2), (64, 64, 51, 8, 4000, 2), (16, 16, 33, 2, 3000, 2)]

_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2104_08002_b200 import conv as cv
out = {}
for i, (c, k, s, d, q, n) in enumerate(eval(sys.argv[3])):
    g = torch.Generator(device="cuda").manual_seed(100 + i)
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    x = cv.round_bf16(torch.randn((n, c, q + d * (s - 1)), device="cuda", generator=g))
    dy = cv.round_bf16(torch.randn((n, k, q), device="cuda", generator=g))
    w = torch.randn((k, c, s), device="cuda", generator=g) * 0.05
    out[f"y{i}"] = cv.conv1d_forward(x, w, p).cpu().numpy()
    out[f"dx{i}"] = cv.conv1d_backward_data(dy, cv.pack_weights_backward(w), p).cpu().numpy()
    out[f"dw{i}"] = cv.conv1d_backward_weight(dy, x, p).cpu().numpy()
np.savez(sys.argv[2], **out)
"""


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(tmp_path, name, env_extra):
    path = str(tmp_path / f"{name}.npz")
    env = dict(os.environ)
    for k in ("C1D_NO_PDL", "C1D_NO_WRES", "C1D_NO_BOX3"):
        env.pop(k, None)
    env.update(env_extra)
    subprocess.run([sys.executable, "-c", _CHILD, ROOT, path, repr(SHAPES)], env=env, check=True, timeout=300)
    return dict(np.load(path))


@pytest.mark.parametrize("switch", ["C1D_NO_PDL", "C1D_NO_WRES", "C1D_NO_BOX3"])
def test_switch_is_bit_identical(tmp_path, switch):
    base = _run(tmp_path, "base", {})
    alt = _run(tmp_path, switch, {switch: "1"})
    assert base.keys() == alt.keys()
    for key in base:
        assert np.isfinite(base[key]).all(), key
        assert np.array_equal(base[key].view(np.uint32), alt[key].view(np.uint32)), f"{switch}: {key} differs"
