"""Config-5 network step on the B200 kernels vs a float64 torch autograd restatement of the same
network (only as a checker for the floating-point glue; the conv passes themselves are pinned to
the oracle in test_parity_gpu.py). Mirrors the reference's end-to-end gradient check of a small
net (proj/tests/test_train.cpp:316-349)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2104_08002_b200 import conv as cv
from paper_2104_08002_b200.network import ResidualNet, train_step

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def torch_reference(net, x_padded, target, labels):
    """float64 autograd version of ResidualNet.forward + loss; returns (loss, grads per layer)."""
    params = []
    for layer in net.layers():
        w = layer.w.double().clone().requires_grad_(True)
        b = layer.b.double().clone().requires_grad_(True)
        params.append((layer, w, b))
    it = iter(params)

    def apply(layer, w, b, x, skip=None):
        xp = F.pad(x, (layer.pad, layer.pad)) if layer.pad else x
        pre = F.conv1d(xp, w, b, dilation=layer.p.dilation)
        out = torch.relu(pre) if layer.relu else pre
        return out + skip if skip is not None else out

    layer, w, b = next(it)
    h = apply(layer, w, b, x_padded.double())
    for blk in net.blocks:
        skip = h
        for i in range(len(blk)):
            layer, w, b = next(it)
            h = apply(layer, w, b, h, skip if i == len(blk) - 1 else None)
    layer, w, b = next(it)
    pred = apply(layer, w, b, h)
    layer, w, b = next(it)
    logits = apply(layer, w, b, h)
    mse = ((pred - target.double()) ** 2).mean()
    bce = (F.softplus(logits) - labels.double() * logits).mean()
    loss = mse + bce
    loss.backward()
    return loss.item(), [(w.grad, b.grad) for _, w, b in params]


@pytest.mark.parametrize("precision", [cv.Precision.Fp32, cv.Precision.Bf16])
def test_network_step_matches_autograd(precision):
    torch.manual_seed(0)
    net = ResidualNet(blocks=2, convs_per_block=3, hidden=6, taps=5, dilation=8, precision=precision, seed=3)
    n, width = 3, 512
    pad = net.pad()
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.poisson(torch.full((n, 1, width + 2 * pad), 2.0, device="cuda"), generator=g)
    target = torch.poisson(torch.full((n, 1, width), 2.0, device="cuda"), generator=g)
    labels = (torch.rand((n, 1, width), device="cuda", generator=g) < 0.1).float()
    if precision == cv.Precision.Bf16:
        # the reference BF16 path rounds conv operands; compare against a net whose weights and
        # input are already BF16-representable and only check the glue loosely
        for layer in net.layers():
            layer.w.copy_(layer.w.bfloat16().float())
    loss_ref, grads_ref = torch_reference(net, x, target, labels)
    loss = train_step(net, x, target, labels).item()
    tol = 1e-5 if precision == cv.Precision.Fp32 else 2e-2
    assert abs(loss - loss_ref) <= tol * max(1.0, abs(loss_ref))
    for layer, (gw, gb) in zip(net.layers(), grads_ref):
        for got, want in ((layer.grad_w, gw), (layer.grad_b, gb)):
            want = want.float().cpu().numpy()
            err = np.abs(got.cpu().numpy() - want).max() / max(1.0, np.abs(want).max())
            assert err <= tol, (err, layer.p)


def test_grad_bucket_is_one_flat_buffer():
    net = ResidualNet(blocks=5, convs_per_block=3, hidden=15, seed=1)
    # BASELINE config 5: 173,162 gradient floats in a single all-reduce bucket
    assert net.grad_bucket.numel() == net.num_parameters() == 1 * 15 * 51 + 15 + 15 * (15 * 15 * 51 + 15) + 2 * (15 + 1)
    assert net.layers()[3].grad_w.data_ptr() > net.layers()[0].grad_w.data_ptr()


def test_fused_glue_matches_torch():
    """c1d_layer_forward_epilogue / c1d_layer_backward_prologue vs the same glue in torch."""
    from paper_2104_08002_b200.network import layer_backward_prologue, layer_forward_epilogue

    g = torch.Generator(device="cuda").manual_seed(3)
    n, k, q, pad = 3, 5, 1000, 12
    pre = torch.randn((n, k, q), device="cuda", generator=g)
    bias = torch.randn(k, device="cuda", generator=g)
    skip = torch.randn((n, k, q), device="cuda", generator=g)
    want_pre = pre + bias.view(1, -1, 1)
    want_act = torch.relu(want_pre) + skip
    act = torch.empty_like(pre)
    act_b = torch.zeros((n, k, q + 2 * pad), dtype=torch.bfloat16, device="cuda")
    p2 = pre.clone()
    layer_forward_epilogue(p2, bias, skip, True, act, act_b, pad)
    assert torch.equal(p2, pre)  # pre untouched unless store_pre
    layer_forward_epilogue(p2, bias, skip, True, act, act_b, pad, store_pre=True)
    assert torch.equal(p2, want_pre)
    assert torch.equal(act, want_act)
    assert torch.equal(act_b[:, :, pad:pad + q], cv.round_bf16(want_act))
    assert not act_b[:, :, :pad].any() and not act_b[:, :, pad + q:].any()
    # backward: gradient from the interior of a padded buffer + skip gradient, ReLU mask
    gin = torch.randn((n, k, q + 2 * pad), device="cuda", generator=g)
    gadd = torch.randn((n, k, q), device="cuda", generator=g)
    gsum = torch.empty_like(pre)
    gp32 = torch.empty_like(pre)
    gpb = torch.empty((n, k, q), dtype=torch.bfloat16, device="cuda")
    db = torch.empty(k, device="cuda")
    layer_backward_prologue(gin, pad, want_pre, n, k, q, relu=True, gadd=gadd, gsum=gsum, grad_pre=gp32,
                            grad_pre_bf16=gpb, bias_grad=db)
    want_g = gin[:, :, pad:pad + q] + gadd
    want_gp = want_g * (want_pre > 0)
    assert torch.equal(gsum, want_g)
    assert torch.equal(gp32, want_gp)
    assert torch.equal(gpb, cv.round_bf16(want_gp))
    assert torch.allclose(db, want_gp.sum(dim=(0, 2)), rtol=1e-5, atol=1e-4)
    db2 = torch.empty(k, device="cuda")
    layer_backward_prologue(gin, pad, want_pre, n, k, q, relu=True, gadd=gadd, bias_grad=db2)
    assert torch.equal(db, db2)  # deterministic
    # mask from the unbiased conv output + the bias (what the network does)
    gpb2 = torch.empty_like(gpb)
    layer_backward_prologue(gin, pad, pre, n, k, q, relu=True, gadd=gadd, grad_pre_bf16=gpb2, pre_bias=bias)
    assert torch.equal(gpb2, gpb)


def test_network_step_under_cuda_graph():
    """The whole training step (C-ABI passes + torch losses) captured in one CUDA graph replays to
    the eager step's results bit for bit (bench.py --workload network replays it)."""
    net = ResidualNet(blocks=2, convs_per_block=3, hidden=15, taps=51, dilation=8, seed=5)
    n, width = 2, 2048
    pad = net.pad()
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.poisson(torch.full((n, 1, width + 2 * pad), 2.0, device="cuda"), generator=g)
    target = torch.poisson(torch.full((n, 1, width), 2.0, device="cuda"), generator=g)
    labels = (torch.rand((n, 1, width), device="cuda", generator=g) < 0.1).float()
    loss_eager = train_step(net, x, target, labels).item()
    grads_eager = net.grad_bucket.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        train_step(net, x, target, labels)  # warm this stream's internal workspace
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        loss_g = train_step(net, x, target, labels)
    net.grad_bucket.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert loss_g.item() == loss_eager
    assert torch.equal(net.grad_bucket, grads_eager)
