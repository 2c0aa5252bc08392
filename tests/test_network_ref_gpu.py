"""The GPU network step pinned to the reference's own network (proj/src/train.cpp:173-353).

`ResidualNet(convs_per_block=1, precision_rule="reference")` has the layer list, precisions and
glue of the reference's DemoNet (an input conv 1 -> hidden, `blocks` residual convs whose ReLU
output is added to their input, two 1-tap FP32 heads). With the reference's own initial
parameters loaded (gather_params order) and the reference's synthetic dataset
(generate_synthetic_dataset, train.cpp:62-98) as input, one train_step must give the reference's
loss and every weight and bias gradient:

* FP32 (hidden 15): norm-relative error <= 1e-5 per layer tensor (the reference's FP32 bound);
* BF16 (hidden 16, the reference's BF16 width; its 1-channel input layer and heads stay FP32 by
  make_layer's even-dims rule): <= 1e-2 (acceptance.cpp:526).

Then the acceptance criterion-8 bar (acceptance.cpp:534-564: validation loss halves over the
documented 25-epoch run and the best validation AUROC exceeds 0.9), run by the reference's own
train() linked against the B200 conv backend, and by the device network itself.
"""
import os
import subprocess

import numpy as np
import pytest
import torch

import oracle
from paper_2104_08002_b200 import conv as cv
from paper_2104_08002_b200.network import ResidualNet, forward_backward

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _dataset(count, width, pad, seed=1):
    noisy, clean, mask = oracle.ref_synthetic_dataset(oracle.Ref(), seed, count, width)
    return oracle.zero_pad_width(noisy, pad, pad), clean, mask


def _layer_slices(net: ResidualNet):
    out, off = [], 0
    for i, layer in enumerate(net.layers()):
        for name, t in (("w", layer.w), ("b", layer.b)):
            out.append((f"layer{i}.{name}", off, off + t.numel()))
            off += t.numel()
    return out


def float64_truth(net: ResidualNet, x, clean, mask):
    """Loss and flat gradient (gather_grads order) of the same network in float64 autograd on the
    BF16-rounded operands the layers actually use (a checker, not the product path)."""
    import torch.nn.functional as F

    params = []
    for layer in net.layers():
        w = layer.w.double().clone()
        if layer.bf16:
            w = w.to(torch.bfloat16).double()
        params.append((layer, w.requires_grad_(True), layer.b.double().clone().requires_grad_(True)))

    def apply(layer, w, b, h, skip=None):
        xin = F.pad(h, (layer.pad, layer.pad)) if layer.pad else h
        if layer.bf16:  # the reference rounds a BF16 layer's input (conv.cpp:182-183)
            xin = xin.to(torch.bfloat16).double() + (xin - xin.detach())  # rounded value, identity gradient
        pre = F.conv1d(xin, w, b, dilation=layer.p.dilation)
        out = torch.relu(pre) if layer.relu else pre
        return out + skip if skip is not None else out

    it = iter(params)
    layer, w, b = next(it)
    h = apply(layer, w, b, torch.from_numpy(x).double().cuda())
    for blk in net.blocks:
        for layer_ in blk:
            layer, w, b = next(it)
            h = apply(layer, w, b, h, h)
    layer, w, b = next(it)
    pred = apply(layer, w, b, h)
    layer, w, b = next(it)
    logits = apply(layer, w, b, h)
    yt, mt = torch.from_numpy(clean).double().cuda(), torch.from_numpy(mask).double().cuda()
    loss = ((pred - yt) ** 2).mean() + (F.softplus(logits) - mt * logits).mean()
    loss.backward()
    flat = torch.cat([t.grad.reshape(-1) for _, w, b in params for t in (w, b)])
    return float(loss), flat.cpu().numpy()


@pytest.mark.parametrize("precision,hidden,tol", [(0, 15, 1e-5), (1, 16, 1e-2)], ids=["fp32", "bf16"])
def test_train_step_matches_demonet(precision, hidden, tol):
    """One train_step from the reference's own parameters and data: loss and every layer's weight
    and bias gradient against the reference's DemoNet, and both against a float64 evaluation of
    the same network (which tells whose rounding a difference is). FP32: ours within 1e-5 of the
    float64 truth, and of the reference up to the reference's own deviation from that truth."""
    blocks, width, count = 3, 4096, 4
    ref = oracle.RefNet(blocks, hidden, 51, 8, precision, seed=1)
    prec = cv.Precision.Bf16 if precision else cv.Precision.Fp32
    net = ResidualNet(blocks=blocks, convs_per_block=1, hidden=hidden, taps=51, dilation=8, precision=prec,
                      device="cuda", precision_rule="reference")
    want_prec = ref.layer_precisions()
    got_prec = [int(layer.p.precision) for layer in net.layers()]
    assert got_prec == want_prec, (got_prec, want_prec)
    params = ref.params()
    net.load_params(params)
    x, clean, mask = _dataset(count, width, ref.pad())
    ref_loss = ref.train_step(x, clean, mask, 1.0)
    ref_grads = ref.grads()
    loss = forward_backward(net, torch.from_numpy(x).cuda(), torch.from_numpy(clean).cuda(),
                            torch.from_numpy(mask).cuda(), 1.0)
    torch.cuda.synchronize()
    got = net.grad_bucket.cpu().numpy()
    tag = "bf16" if precision else "fp32"
    true_loss, truth = float64_truth(net, x, clean, mask)
    lrel = abs(float(loss) - ref_loss) / abs(ref_loss)
    print(f"[demonet pin {tag}] loss {float(loss):.9g} vs reference {ref_loss:.9g} (rel {lrel:.2e}), "
          f"float64 {true_loss:.9g}")
    assert lrel <= tol

    def rel(a, b):
        return oracle.norm_rel_error(a, b) if np.any(b) else float(np.abs(a).max())

    worst = 0.0
    for name, a, b in _layer_slices(net):
        e_ref = rel(got[a:b], ref_grads[a:b])
        e_true = rel(got[a:b], truth[a:b].astype(np.float32))
        r_true = rel(ref_grads[a:b], truth[a:b].astype(np.float32))
        worst = max(worst, e_ref)
        print(f"[demonet pin {tag}] grad {name}: vs reference {e_ref:.3e}; vs float64: ours {e_true:.3e}, "
              f"reference {r_true:.3e}")
        if precision == 0:
            assert e_true <= tol, f"{name}: {e_true:.3e} from float64 > {tol}"
            assert e_ref <= tol + r_true, f"{name}: {e_ref:.3e} from the reference"
        else:
            assert e_ref <= tol, f"{name}: {e_ref:.3e} > {tol}"
    print(f"[demonet pin {tag}] worst gradient difference from the reference {worst:.3e}")
    # the SGD update over the flat buckets equals the reference's per-layer sgd_step
    ref.step(0.05)
    net.sgd_step(0.05)
    torch.cuda.synchronize()
    pe = oracle.norm_rel_error(net.param_bucket.cpu().numpy(), ref.params())
    print(f"[demonet pin {tag}] params after sgd_step(0.05): norm_rel_error {pe:.3e}")
    assert pe <= tol


def test_reference_training_run_on_gpu_backend():
    """Acceptance criterion 8 (acceptance.cpp:534-564) by the reference's own train() with its conv
    passes on the B200 backend (oracle/_ref/acceptance_gpu)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "acceptance_gpu")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/acceptance_gpu not built (needs /root/reference at build time)")
    out = subprocess.run([exe, "8"], capture_output=True, text=True, timeout=1200)
    print(out.stdout)
    assert out.returncode == 0 and "criterion 8 PASS" in out.stdout, out.stdout + out.stderr


def test_device_network_trains_like_criterion8():
    """The same bar on the device network itself: TrainConfig's defaults (train.hpp: 25 epochs,
    batch 16, lr 0.05, width 4096, 256 segments, 4 blocks, FP32, seed 1) with the reference's
    dataset, its 10% validation split and its initial parameters; validation loss must halve and
    the best validation AUROC (the reference's rank statistic, train.cpp:143-171) exceed 0.9."""
    from paper_2104_08002_b200 import network as nw

    blocks, hidden, width, segments, batch, lr, epochs = 4, 15, 4096, 256, 16, 0.05, 25
    ref = oracle.RefNet(blocks, hidden, 51, 8, 0, seed=1)
    net = ResidualNet(blocks=blocks, convs_per_block=1, hidden=hidden, precision=cv.Precision.Fp32, device="cuda",
                      precision_rule="reference")
    net.load_params(ref.params())
    x, clean, mask = _dataset(segments, width, ref.pad())
    val = max(1, segments // 10)
    tr = segments - val
    X, Y, M = (torch.from_numpy(a).cuda() for a in (x, clean, mask))
    stats = []
    for _ in range(epochs):
        for b in range(0, tr, batch):
            e = min(tr, b + batch)
            forward_backward(net, X[b:e], Y[b:e], M[b:e], 1.0)
            net.sgd_step(lr)
        pred, logits = net.forward(X[tr:])
        mse, _ = nw.mse_loss(pred, Y[tr:])
        bce, _ = nw.bce_with_logits(logits, M[tr:])
        stats.append((float(mse + bce), nw.auroc(logits, M[tr:])))
    first, last = stats[0][0], stats[-1][0]
    best = max(a for _, a in stats)
    print(f"[criterion 8, device net] val loss {first:.4f} -> {last:.4f} (ratio {last / first:.2f}), "
          f"best val AUROC {best:.4f}")
    # the device AUROC equals the reference's rank statistic on the same scores
    pred, logits = net.forward(X[tr:])
    a_dev = nw.auroc(logits, M[tr:])
    a_ref = oracle.ref_auroc(oracle.Ref(), logits.cpu().numpy(), mask[tr:])
    assert abs(a_dev - a_ref) <= 1e-12, (a_dev, a_ref)
    assert last <= 0.5 * first and best > 0.9
