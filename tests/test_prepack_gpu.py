"""C1D_FLAG_PREPACKED_WEIGHTS: weight images made by c1d_pack_weights (one launch for many layers)
give the same glued passes, bit for bit, as the calls that pack their own weights; plans that pack
their own weights refuse images; the network step is unchanged by them."""
import os

import pytest
import torch

from paper_2104_08002_b200 import _lib as L
from paper_2104_08002_b200 import conv as cv
from paper_2104_08002_b200.network import (ResidualNet, conv_backward_data_glued, conv_forward_glued, mask_shape,
                                           pack_weights, packed_weights_bytes, train_step)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("n,c,k,q", [(2, 15, 15, 1000), (3, 1, 15, 777), (2, 15, 1, 512), (1, 32, 24, 640)])
def test_prepacked_glued_passes_match(n, c, k, q):
    s, d = 51, 8
    pad = d * (s - 1) // 2
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    g = torch.Generator(device="cuda").manual_seed(11 + c + k)
    x = cv.round_bf16(torch.randn((n, c, q + 2 * pad), device="cuda", generator=g))
    w = torch.randn((k, c, s), device="cuda", generator=g) * 0.05
    b = torch.randn(k, device="cuda", generator=g) * 0.1
    dy = cv.round_bf16(torch.randn((n, k, q), device="cuda", generator=g))
    w_in = q + 2 * pad
    nb_f = packed_weights_bytes(p, n, w_in, L.PASS_FORWARD)
    nb_b = packed_weights_bytes(p, n, w_in, L.PASS_BACKWARD_DATA)
    assert nb_f > 0 and nb_b > 0
    img_f = torch.full((nb_f,), 0x5A, dtype=torch.uint8, device="cuda")  # garbage first: packing overwrites all
    img_b = torch.full((nb_b,), 0x5A, dtype=torch.uint8, device="cuda")
    pack_weights([(p, n, w_in, L.PASS_FORWARD, w, img_f), (p, n, w_in, L.PASS_BACKWARD_DATA, w, img_b)])

    outs = []
    for image_f, image_b in ((None, None), (img_f, img_b)):
        act_b = torch.zeros((n, k, q + 2 * pad), dtype=torch.bfloat16, device="cuda")
        mask = torch.zeros(mask_shape(n, k, q), dtype=torch.int32, device="cuda")
        conv_forward_glued(x, w, p, bias=b, act_bf16=act_b, act_pad=pad, mask=mask, image=image_f)
        gpb = torch.zeros((n, c, q), dtype=torch.bfloat16, device="cuda")
        conv_backward_data_glued(dy, w, p, pad, q, grad_pre_bf16=gpb, image=image_b)
        torch.cuda.synchronize()
        outs.append((act_b, mask, gpb))
    for a, bb in zip(*outs):
        assert torch.equal(a, bb)


def test_plans_with_their_own_packing_refuse_images():
    # 64 filters per group (tail-tap plan): no image; the flag on such a call is an error
    p = cv.ConvParams(64, 64, 51, 8, cv.Precision.Bf16)
    assert packed_weights_bytes(p, 2, 1400, L.PASS_FORWARD) == 0
    x = torch.zeros((2, 64, 1400), dtype=torch.bfloat16, device="cuda")
    img = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    with pytest.raises(Exception):
        conv_forward_glued(x, torch.zeros((64, 64, 51), device="cuda"), p, act_bf16=None, image=img)
    # FP32 precision packs its own (split) operands
    pf = cv.ConvParams(15, 15, 51, 8, cv.Precision.Fp32)
    assert packed_weights_bytes(pf, 2, 1400, L.PASS_FORWARD) == 0


def test_network_step_unchanged_by_prepacked_images():
    n, width = 2, 2048
    losses, grads = [], []
    for no_prepack in (True, False):
        if no_prepack:
            os.environ["C1D_NET_NO_PREPACK"] = "1"
        else:
            os.environ.pop("C1D_NET_NO_PREPACK", None)
        net = ResidualNet(precision=cv.Precision.Bf16, seed=3)
        pad = net.pad()
        g = torch.Generator(device="cuda").manual_seed(4)
        x = torch.poisson(torch.full((n, 1, width + 2 * pad), 2.0, device="cuda"), generator=g)
        t = torch.poisson(torch.full((n, 1, width), 2.0, device="cuda"), generator=g)
        lab = (torch.rand((n, 1, width), device="cuda", generator=g) < 0.1).float()
        out = []
        for _ in range(2):
            out.append(float(train_step(net, x, t, lab)))
            net.sgd_step(1e-3)
        torch.cuda.synchronize()
        losses.append(out)
        grads.append(net.grad_bucket.clone())
        if not no_prepack:
            assert any(layer.img for layer in net.layers())
    os.environ.pop("C1D_NET_NO_PREPACK", None)
    assert losses[0] == losses[1]
    assert torch.equal(grads[0], grads[1])
