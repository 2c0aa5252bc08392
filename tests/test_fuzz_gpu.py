"""Seeded shape fuzz over the kernel plans added for wide channels and other dilations: the
expanded-row modes (d = 1, 2, 4; inline and row-tensor), the d = 8 direct mode (K > 64), the FP32
split's channel halves (C_in*S > 3300) and block backward-weight, odd widths and both storages.
Every pass vs the oracle at the reference's bounds (FP32 1e-5; BF16 1e-5 against the oracle on
BF16-rounded operands)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2104_08002_b200 import conv as cv

from test_parity_gpu import BF16_TOL_ROUNDED, FP32_TOL, assert_close, oracle_passes, run_passes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cases(count=60, budget=5e8):
    rng = oracle.Rng(777)
    chans, taps, dils, widths = [15, 48, 96, 128], [3, 17, 33, 51], [1, 2, 4, 8, 16], [300, 777, 1024]
    out = []
    while len(out) < count:
        c, k = chans[rng.next_below(4)], chans[rng.next_below(4)]
        s, d, q = taps[rng.next_below(4)], dils[rng.next_below(5)], widths[rng.next_below(3)]
        n = 1 + rng.next_below(2)
        if n * c * k * s * q > budget:
            continue
        prec = [cv.Precision.Bf16, cv.Precision.Bf16, cv.Precision.Fp32][rng.next_below(3)]
        bf16_storage = prec == cv.Precision.Bf16 and rng.next_below(2) == 1
        out.append((c, k, s, d, q, n, prec, bf16_storage))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda t: "c{}k{}s{}d{}q{}n{}{}{}".format(
    *t[:6], "bf16" if t[6] == cv.Precision.Bf16 else "fp32", "s" if t[7] else ""))
def test_fuzz_passes_vs_oracle(case):
    c, k, s, d, q, n, prec, bf16_storage = case
    rng = oracle.Rng(9000 + c * 7 + k * 3 + s + d + q)
    w_in = q + d * (s - 1)
    x, w, dy = rng.fill_uniform((n, c, w_in)), rng.fill_uniform((k, c, s)), rng.fill_uniform((n, k, q))
    got = run_passes(x, w, dy, d, prec, bf16_storage=bf16_storage)
    if prec == cv.Precision.Fp32:
        want, tol = oracle_passes(x, w, dy, d), FP32_TOL
    else:
        want = oracle_passes(oracle.round_bf16(x), oracle.round_bf16(w), oracle.round_bf16(dy), d)
        tol = BF16_TOL_ROUNDED
    for g, wv, name in zip(got, want, ("fwd", "bwd_d", "bwd_w")):
        assert np.all(np.isfinite(g)), name
        assert_close(g, wv, tol, f"{case} {name}")
