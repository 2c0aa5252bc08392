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


# Wide channel counts at d = 8 (128 < K or C <= 320): the carry-free direct mode and the carry mode
# need different workspaces; every pass runs once with the internal workspace and once with a
# caller buffer of exactly c1d_workspace_size bytes (the advisor's sizing case C=128 K=160 S=51).
WIDE = [(128, 160, 51), (160, 128, 51), (144, 192, 9), (192, 144, 17), (300, 64, 3), (64, 300, 3)]


def _run_with_workspace(x, w, dy, d, prec, exact=False):
    import ctypes as C

    from paper_2104_08002_b200 import _lib as L

    k, c, s = w.shape
    n, _, w_in = x.shape
    p = cv.ConvParams(c, k, s, d, prec)
    desc = cv.make_desc(p, n, w_in, L.DTYPE_F32, exact=exact)
    lib = L.lib()
    xt, wt, gt = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (x, w, dy))
    q = w_in - d * (s - 1)
    outs = [torch.empty((n, k, q), device="cuda"), torch.empty((n, c, w_in), device="cuda"),
            torch.empty((k, c, s), device="cuda")]
    sp = torch.cuda.current_stream().cuda_stream
    calls = [(lib.c1d_forward, xt, wt), (lib.c1d_backward_data, gt, wt), (lib.c1d_backward_weight, xt, gt)]
    for pass_, ((fn, a, b), out) in enumerate(zip(calls, outs)):
        nbytes = cv.workspace_size(p, n, w_in, pass_, L.DTYPE_F32, exact=exact)
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
        cv._check(fn(C.byref(desc), a.data_ptr(), b.data_ptr(), out.data_ptr(), ws.data_ptr(), nbytes, sp))
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs]


@pytest.mark.parametrize("shape", WIDE, ids=lambda t: "c{}k{}s{}".format(*t))
def test_wide_channels_d8_workspace(shape):
    c, k, s = shape
    d, q, n = 8, 520, 1
    rng = oracle.Rng(4242 + c + k + s)
    w_in = q + d * (s - 1)
    x, w, dy = rng.fill_uniform((n, c, w_in)), rng.fill_uniform((k, c, s)), rng.fill_uniform((n, k, q))
    want = oracle_passes(oracle.round_bf16(x), oracle.round_bf16(w), oracle.round_bf16(dy), d)
    # default accumulation: one TMEM chain of C_in*S products (up to 15300 here: ~2e-5 drift);
    # exact (C1D_FLAG_EXACT_ACCUM): chains capped at ~4096 products, the reference's 1e-5
    for exact, tol in ((False, 1e-4), (True, BF16_TOL_ROUNDED)):
        for got in (run_passes(x, w, dy, d, cv.Precision.Bf16, exact=exact),
                    _run_with_workspace(x, w, dy, d, cv.Precision.Bf16, exact=exact)):
            for g, wv, name in zip(got, want, ("fwd", "bwd_d", "bwd_w")):
                assert_close(g, wv, tol, f"{shape} exact={exact} {name}")


def test_workspace_too_small_is_an_error():
    """A caller buffer one byte short of c1d_workspace_size fails with C1D_ERR_WORKSPACE before any
    launch (no device fault)."""
    import ctypes as C

    from paper_2104_08002_b200 import _lib as L

    c, k, s, d, q, n = 128, 160, 51, 8, 520, 1
    w_in = q + d * (s - 1)
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    desc = cv.make_desc(p, n, w_in, L.DTYPE_F32)
    nbytes = cv.workspace_size(p, n, w_in, 0, L.DTYPE_F32)
    assert nbytes > 0
    x = torch.zeros((n, c, w_in), device="cuda")
    w = torch.zeros((k, c, s), device="cuda")
    y = torch.empty((n, k, q), device="cuda")
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    st = L.lib().c1d_forward(C.byref(desc), x.data_ptr(), w.data_ptr(), y.data_ptr(), ws.data_ptr(), nbytes - 1,
                             torch.cuda.current_stream().cuda_stream)
    assert st == L.ERR_WORKSPACE
    torch.cuda.synchronize()
