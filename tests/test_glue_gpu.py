"""Layer-glued conv passes (c1d_forward_glued / c1d_backward_data_glued) vs the plain conv passes
plus the ConvLayer glue restated in torch (train.cpp:176-192, 205-221). The glue itself is FP32
elementwise work on the conv output, so everything but the bias-gradient sum is compared
bit-exactly; the conv passes are pinned to the oracle in test_parity_gpu.py."""
import pytest
import torch

from paper_2104_08002_b200 import _lib as L
from paper_2104_08002_b200 import conv as cv
from paper_2104_08002_b200.network import conv_backward_data_glued, conv_forward_glued, glue_is_fused, mask_shape

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def unpack_mask(words: torch.Tensor, channels: int) -> torch.Tensor:
    """(N, ceil(C/16), Q) channel-block words -> (N, C, Q) bools."""
    n, nb, q = words.shape
    assert not (words >> 16).any()  # bits 16-31 stay zero
    bits = (words.unsqueeze(2) >> torch.arange(16, device=words.device, dtype=torch.int32).view(1, 1, 16, 1)) & 1
    return bits.reshape(n, nb * 16, q)[:, :channels].bool()


def pack_mask(keep: torch.Tensor) -> torch.Tensor:
    n, c, q = keep.shape
    nb = (c + 15) // 16
    full = torch.zeros((n, nb * 16, q), dtype=torch.int32, device=keep.device)
    full[:, :c] = keep.int()
    shifts = torch.arange(16, device=keep.device, dtype=torch.int32).view(1, 1, 16, 1)
    return (full.view(n, nb, 16, q) << shifts).sum(2, dtype=torch.int32)


# (C, K, S, d, precision, in bf16, expect fused)
CASES = [
    (15, 15, 51, 8, cv.Precision.Bf16, True, True),     # config-5 body layer
    (1, 15, 51, 8, cv.Precision.Bf16, True, None),      # config-5 input layer
    (64, 64, 33, 8, cv.Precision.Bf16, True, True),     # KP = 64, tail taps
    (24, 80, 9, 8, cv.Precision.Bf16, True, True),      # two filter groups (forward)
    (16, 16, 17, 2, cv.Precision.Bf16, True, None),     # phase rewrite or FFMA
    (6, 6, 5, 8, cv.Precision.Fp32, False, False),      # FP32: conv + separate glue pass
    (8, 8, 7, 3, cv.Precision.Bf16, True, False),       # FFMA path
    (96, 40, 17, 4, cv.Precision.Bf16, False, None),    # expanded rows (fused forward, 96-wide backward)
    (40, 100, 9, 8, cv.Precision.Bf16, True, None),     # carry mode, two filter groups under glue
    (128, 128, 9, 1, cv.Precision.Bf16, True, None),    # 128-wide expanded rows: conv + glue pass
    (15, 2, 1, 1, cv.Precision.Fp32, False, False),     # config-5 heads: 1-tap FP32 (backward glue computes dx)
]


@pytest.mark.parametrize("c,k,s,d,prec,bf16_in,fused", CASES)
@pytest.mark.parametrize("q", [1000, 1027])
def test_forward_glued(c, k, s, d, prec, bf16_in, fused, q):
    g = torch.Generator(device="cuda").manual_seed(c * 131 + k + q)
    n, pad = 3, 12
    p = cv.ConvParams(c, k, s, d, prec)
    w_in = q + d * (s - 1)
    x = torch.randn((n, c, w_in), device="cuda", generator=g)
    x = cv.round_bf16(x) if bf16_in else x
    w = torch.randn((k, c, s), device="cuda", generator=g) * (1.0 / (c * s) ** 0.5)
    bias = torch.randn(k, device="cuda", generator=g) * 0.1
    skip = torch.randn((n, k, q), device="cuda", generator=g)
    if fused is not None:
        assert glue_is_fused(p, n, w_in, L.PASS_FORWARD, L.DTYPE_BF16 if bf16_in else L.DTYPE_F32) == fused
    y = cv.conv1d_forward(x, w, p)
    v = y + bias.view(1, -1, 1)
    want_act = torch.relu(v) + skip
    pre = torch.empty_like(y)
    act = torch.empty_like(y)
    act_b = torch.zeros((n, k, q + 2 * pad), dtype=torch.bfloat16, device="cuda")
    mask = torch.empty(mask_shape(n, k, q), dtype=torch.int32, device="cuda")
    conv_forward_glued(x, w, p, bias=bias, skip=skip, relu=True, pre=pre, act=act, act_bf16=act_b, act_pad=pad,
                       mask=mask)
    assert torch.equal(pre, v)
    assert torch.equal(act, want_act)
    assert torch.equal(act_b[:, :, pad:pad + q], cv.round_bf16(want_act))
    assert not act_b[:, :, :pad].any() and not act_b[:, :, pad + q:].any()
    assert torch.equal(unpack_mask(mask, k), v > 0)
    # only the bf16 activation (what a body layer writes), no ReLU
    act_b2 = torch.zeros_like(act_b)
    conv_forward_glued(x, w, p, bias=bias, relu=False, act_bf16=act_b2, act_pad=pad)
    assert torch.equal(act_b2[:, :, pad:pad + q], cv.round_bf16(v))


@pytest.mark.parametrize("c,k,s,d,prec,bf16_in,fused", CASES)
@pytest.mark.parametrize("q", [1000, 1027])
def test_backward_data_glued(c, k, s, d, prec, bf16_in, fused, q):
    g = torch.Generator(device="cuda").manual_seed(c * 17 + k + q)
    n = 3
    p = cv.ConvParams(c, k, s, d, prec)
    halo = d * (s - 1)
    w_in = q + halo
    dy = torch.randn((n, k, q), device="cuda", generator=g)
    dy = cv.round_bf16(dy) if bf16_in else dy
    w = torch.randn((k, c, s), device="cuda", generator=g) * (1.0 / (k * s) ** 0.5)
    if fused is not None:
        assert glue_is_fused(p, n, w_in, L.PASS_BACKWARD_DATA, L.DTYPE_BF16 if bf16_in else L.DTYPE_F32) == fused
    dx = cv.conv1d_backward_data(dy, w, p)
    # the glued layer owns an interior window of dx (a same-padded layer: off = pad)
    off = halo // 2
    gq = w_in - 2 * off
    gadd = torch.randn((n, c, gq), device="cuda", generator=g)
    keep = torch.rand((n, c, gq), device="cuda", generator=g) < 0.6
    mask = pack_mask(keep)
    assert torch.equal(unpack_mask(mask, c), keep)
    want_g = dx[:, :, off:off + gq] + gadd
    want_gp = torch.where(keep, want_g, torch.zeros_like(want_g))
    gsum = torch.empty_like(want_g)
    gp32 = torch.empty_like(want_g)
    gpb = torch.empty((n, c, gq), dtype=torch.bfloat16, device="cuda")
    db = torch.empty(c, device="cuda")
    conv_backward_data_glued(dy, w, p, off, gq, gadd=gadd, mask=mask, gsum=gsum, grad_pre=gp32, grad_pre_bf16=gpb,
                             bias_grad=db)
    assert torch.equal(gsum, want_g)
    assert torch.equal(gp32, want_gp)
    assert torch.equal(gpb, cv.round_bf16(want_gp))
    want_db = want_gp.double().sum(dim=(0, 2))
    assert torch.allclose(db.double(), want_db, rtol=1e-5, atol=1e-4 * (1 + want_gp.abs().sum().item() / c) ** 0.5)
    db2 = torch.empty(c, device="cuda")
    conv_backward_data_glued(dy, w, p, off, gq, gadd=gadd, mask=mask, grad_pre_bf16=gpb, bias_grad=db2)
    assert torch.equal(db, db2)  # deterministic, independent of which outputs are requested
    # no mask (no ReLU), no skip, whole width
    gp_all = torch.empty_like(dx)
    conv_backward_data_glued(dy, w, p, 0, w_in, grad_pre=gp_all)
    assert torch.equal(gp_all, dx)


def test_glued_edge_cases():
    p = cv.ConvParams(15, 15, 51, 8, cv.Precision.Bf16)
    x = torch.zeros((0, 15, 1400), dtype=torch.bfloat16, device="cuda")
    w = torch.zeros((15, 15, 51), device="cuda")
    conv_forward_glued(x, w, p, relu=True)  # empty batch: nothing to do
    db = torch.full((15,), 7.0, device="cuda")
    conv_backward_data_glued(torch.zeros((0, 15, 1000), dtype=torch.bfloat16, device="cuda"), w, p, 200, 1000,
                             bias_grad=db)
    assert not db.any()  # empty batch: zero bias gradient
    with pytest.raises(cv.Error):  # window outside the input gradient
        conv_backward_data_glued(torch.zeros((1, 15, 1000), dtype=torch.bfloat16, device="cuda"), w, p, 300, 1200)
