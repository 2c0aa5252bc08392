"""Config-5 residual 1D CNN training step on the B200 conv kernels.

Mirrors the reference's layer/network code (proj/src/train.cpp) on device tensors:

* `ConvLayer`      ConvLayer::forward/backward (train.cpp:173-221): pad -> conv -> +bias -> ReLU
                   -> (+skip); backward: ReLU mask -> bias grad (row sums) -> backward-weight ->
                   backward-data -> strip pad -> (+skip grad). Conv passes run through the C ABI.
* `ResidualNet`    DemoNet (train.cpp:257-305) extended to BASELINE config 5: a valid input layer
                   1 -> hidden (S=51, d=8, ReLU) consuming the 200-column pad, `blocks` residual
                   blocks of `convs_per_block` same-padded hidden -> hidden convs, and two 1-tap
                   heads (regression, peak logits). The reference's block is one conv whose ReLU
                   output is added to its input (train.cpp:187-192); a 3-conv block here is
                   conv-ReLU, conv-ReLU, conv-ReLU with the block input added after the last ReLU
                   (the reference does not specify the 3-conv arrangement; this is the natural
                   generalisation of its one-conv block).
* losses           mse_loss / bce_with_logits (train.cpp:106-135), means over the local batch.
* `train_step`     forward, combined loss, backward; with a process group the gradients of every
                   layer (one flat bucket) are all-reduced and divided by the world size (the
                   local losses are means over local items).
* `sgd_step`       p <- p - lr*g (train.cpp:137-141).

Weights are Kaiming-uniform with the reference's damping (input 1.0, body 0.3, heads 0.1;
train.cpp:247-248, 263-268), seeded. Activations stay FP32 in HBM; BF16 layers round their
inputs inside the conv call exactly as the reference's BF16 path does.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import conv as cv


def _uniform(shape, limit, gen, device):
    return (torch.rand(shape, generator=gen, device=device, dtype=torch.float32) * 2 - 1) * limit


class ConvLayer:
    """One conv with bias, optional ReLU and optional skip input (train.hpp ConvLayer)."""

    def __init__(self, in_ch, out_ch, taps, dilation, precision, relu, same_pad, weight_scale, gen, device):
        self.p = cv.ConvParams(in_ch, out_ch, taps, dilation, precision)
        self.pad = cv.same_pad_width(taps, dilation) if same_pad else 0
        self.relu = relu
        limit = weight_scale * math.sqrt(6.0 / (in_ch * taps))
        self.w = _uniform((out_ch, in_ch, taps), limit, gen, device)
        self.b = torch.zeros(out_ch, device=device)
        self.grad_w = torch.zeros_like(self.w)
        self.grad_b = torch.zeros_like(self.b)
        self.x_padded = None
        self.pre = None

    def forward(self, x: torch.Tensor, skip: torch.Tensor | None = None) -> torch.Tensor:
        xp = torch.nn.functional.pad(x, (self.pad, self.pad)) if self.pad else x
        if self.p.precision == cv.Precision.Bf16:
            # round once (reference RNE, bf16.hpp:29-40) and reuse it for backward-weight
            xp = cv.round_bf16(xp)
        self.x_padded = xp
        pre = cv.conv1d_forward(self.x_padded, self.w, self.p)
        pre.add_(self.b.view(1, -1, 1))
        self.pre = pre
        out = torch.relu(pre) if self.relu else pre.clone()
        if skip is not None:
            out.add_(skip)
        return out

    def backward(self, grad_out: torch.Tensor) -> torch.Tensor:
        grad_pre = grad_out * (self.pre > 0) if self.relu else grad_out
        grad_pre = grad_pre.contiguous()
        self.grad_b.copy_(grad_pre.sum(dim=(0, 2)))
        g = cv.round_bf16(grad_pre) if self.p.precision == cv.Precision.Bf16 else grad_pre
        cv.conv1d_backward_weight(g, self.x_padded, self.p, out=self.grad_w)
        grad_x = cv.conv1d_backward_data(g, cv.pack_weights_backward(self.w), self.p)
        if self.pad:
            grad_x = grad_x[:, :, self.pad:grad_x.shape[2] - self.pad]
        return grad_x

    def parameters(self):
        return [self.w, self.b]

    def gradients(self):
        return [self.grad_w, self.grad_b]


class ResidualNet:
    """BASELINE config 5: input layer, `blocks` residual blocks of `convs_per_block` convs, 2 heads."""

    def __init__(self, blocks=5, convs_per_block=3, hidden=15, taps=51, dilation=8,
                 precision=cv.Precision.Bf16, seed=1, device="cuda"):
        gen = torch.Generator(device=device).manual_seed(seed)
        self.input = ConvLayer(1, hidden, taps, dilation, precision, True, False, 1.0, gen, device)
        self.blocks = [[ConvLayer(hidden, hidden, taps, dilation, precision, True, True, 0.3, gen, device)
                        for _ in range(convs_per_block)] for _ in range(blocks)]
        self.reg_head = ConvLayer(hidden, 1, 1, 1, cv.Precision.Fp32, False, False, 0.1, gen, device)
        self.peak_head = ConvLayer(hidden, 1, 1, 1, cv.Precision.Fp32, False, False, 0.1, gen, device)
        # one flat gradient bucket (all dW and bias grads) for a single all-reduce per step
        layers = self.layers()
        n = sum(t.numel() for layer in layers for t in layer.gradients())
        self.grad_bucket = torch.zeros(n, device=device)
        off = 0
        for layer in layers:
            views = []
            for g in layer.gradients():
                views.append(self.grad_bucket[off:off + g.numel()].view_as(g))
                off += g.numel()
            layer.grad_w, layer.grad_b = views

    def pad(self) -> int:
        return self.input.p.dilation * (self.input.p.taps - 1) // 2

    def layers(self):
        out = [self.input]
        for blk in self.blocks:
            out.extend(blk)
        return out + [self.reg_head, self.peak_head]

    def num_parameters(self) -> int:
        return sum(t.numel() for layer in self.layers() for t in layer.parameters())

    def conv_flops(self, batch: int, width: int) -> int:
        """2*N*K*C*S*Q per conv pass, three passes per layer (backward-data of the input layer
        included, as the reference's DemoNet::backward computes it)."""
        total = 0
        for layer in self.layers():
            p = layer.p
            total += 3 * cv.conv_flops(p, batch, width)
        return total

    def forward(self, x_padded: torch.Tensor):
        h = self.input.forward(x_padded)
        for blk in self.blocks:
            skip = h
            for i, layer in enumerate(blk):
                h = layer.forward(h, skip if i == len(blk) - 1 else None)
        return self.reg_head.forward(h), self.peak_head.forward(h)

    def backward(self, grad_pred: torch.Tensor, grad_logits: torch.Tensor) -> None:
        grad_h = self.reg_head.backward(grad_pred) + self.peak_head.backward(grad_logits)
        for blk in reversed(self.blocks):
            grad_skip = grad_h
            for layer in reversed(blk):
                grad_h = layer.backward(grad_h)
            grad_h = grad_h + grad_skip
        self.input.backward(grad_h)  # gradient w.r.t. the padded input is discarded

    def sgd_step(self, lr: float) -> None:
        if not lr > 0:
            raise ValueError("sgd_step needs a positive learning rate")
        for layer in self.layers():
            for p, g in zip(layer.parameters(), layer.gradients()):
                p.sub_(lr * g)


def mse_loss(pred: torch.Tensor, target: torch.Tensor):
    """mean((pred-target)^2), grad 2*(pred-target)/count (train.cpp:106-118)."""
    diff = pred.double() - target.double()
    n = diff.numel()
    return (diff * diff).sum() / n, (2.0 * diff / n).float()


def bce_with_logits(logits: torch.Tensor, mask: torch.Tensor):
    """mean(softplus(l) - m*l) in the stable form, grad (sigmoid(l)-m)/count (train.cpp:120-135)."""
    l, m = logits.double(), mask.double()
    n = l.numel()
    value = (torch.nn.functional.softplus(l) - m * l).sum() / n
    return value, ((torch.sigmoid(l) - m) / n).float()


def train_step(net: ResidualNet, x_padded, target, labels, bce_weight: float = 1.0, group=None):
    """One data-parallel training step on this rank's shard; returns the local loss (a tensor)."""
    pred, logits = net.forward(x_padded)
    mse, g_pred = mse_loss(pred, target)
    bce, g_log = bce_with_logits(logits, labels)
    loss = mse + bce_weight * bce
    net.backward(g_pred, bce_weight * g_log)
    if group is not None or (dist.is_available() and dist.is_initialized()):
        world = dist.get_world_size(group)
        if world > 1:
            dist.all_reduce(net.grad_bucket, group=group)
            net.grad_bucket.div_(world)
    return loss
