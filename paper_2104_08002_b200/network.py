"""Config-5 residual 1D CNN training step on the B200 conv kernels.

Mirrors the reference's layer/network code (proj/src/train.cpp) on device tensors:

* `ConvLayer`      ConvLayer::forward/backward (train.cpp:173-221): pad -> conv -> +bias -> ReLU
                   -> (+skip); backward: ReLU mask -> bias grad (row sums) -> backward-weight ->
                   backward-data -> strip pad -> (+skip grad).
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

Fused glue (csrc/layer.cu through the C ABI): every layer's forward is the
conv plus ONE epilogue pass (bias in place, ReLU, skip, and the activation written straight into
the next layer's zero-padded BF16 input buffer), and every backward is ONE prologue pass (the
incoming gradient read from the interior of the padded backward-data output, plus the skip
gradient, ReLU mask, BF16 rounding for the next passes, deterministic bias-gradient sums) plus
the two conv passes. BF16 layers therefore never see an FP32 copy of their input: the activation
is rounded once, exactly where the reference's conv would round it (conv.cpp:182-183).

Weights are Kaiming-uniform with the reference's damping (input 1.0, body 0.3, heads 0.1;
train.cpp:247-248, 263-268), seeded.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import _lib as L
from . import conv as cv


def _uniform(shape, limit, gen, device):
    return (torch.rand(shape, generator=gen, device=device, dtype=torch.float32) * 2 - 1) * limit


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def layer_forward_epilogue(pre, bias=None, skip=None, relu=True, act=None, act_bf16=None, pad=0, store_pre=False):
    """C-ABI fused forward glue (c1d_layer_forward_epilogue) on pre (N, K, Q); with store_pre the
    biased pre-activation is written back in place."""
    n, k, q = pre.shape
    cv._check(L.lib().c1d_layer_forward_epilogue(pre.data_ptr(), _ptr(bias), _ptr(skip), n, k, q, int(relu),
                                                 int(store_pre), _ptr(act), _ptr(act_bf16), pad, _stream()))


def layer_backward_prologue(gin, gin_off, pre, n, k, q, relu=True, gadd=None, gsum=None, grad_pre=None,
                            grad_pre_bf16=None, bias_grad=None, pre_bias=None):
    """C-ABI fused backward glue (c1d_layer_backward_prologue). gin is (N, K, W) with the layer's
    gradient at columns [gin_off, gin_off + q); the ReLU mask is pre + pre_bias > 0."""
    cv._check(L.lib().c1d_layer_backward_prologue(gin.data_ptr(), gin.shape[-1], gin_off, _ptr(gadd), _ptr(pre),
                                                  _ptr(pre_bias), n, k, q, int(relu), _ptr(gsum), _ptr(grad_pre),
                                                  _ptr(grad_pre_bf16), _ptr(bias_grad), None, 0, _stream()))


class ConvLayer:
    """One conv with bias, optional ReLU and optional skip input (train.hpp ConvLayer).

    Forward reads its input from `self.x_in` (N, C, W_in) — bf16 for BF16 layers (zero-padded, as
    written by the previous layer's epilogue), fp32 otherwise — and leaves `self.pre`
    (N, K, Q) = conv + bias for the backward's ReLU mask."""

    def __init__(self, in_ch, out_ch, taps, dilation, precision, relu, same_pad, weight_scale, gen, device):
        self.p = cv.ConvParams(in_ch, out_ch, taps, dilation, precision)
        self.pad = cv.same_pad_width(taps, dilation) if same_pad else 0
        self.relu = relu
        limit = weight_scale * math.sqrt(6.0 / (in_ch * taps))
        self.w = _uniform((out_ch, in_ch, taps), limit, gen, device)
        self.b = torch.zeros(out_ch, device=device)
        self.grad_w = torch.zeros_like(self.w)
        self.grad_b = torch.zeros_like(self.b)
        self.x_in = None
        self.pre = None

    @property
    def bf16(self) -> bool:
        return self.p.precision == cv.Precision.Bf16

    def conv(self, x_in: torch.Tensor) -> torch.Tensor:
        self.x_in = x_in
        self.pre = cv.conv1d_forward(x_in, self.w, self.p, out=self.pre if self._pre_fits(x_in) else None)
        return self.pre

    def _pre_fits(self, x_in) -> bool:
        if self.pre is None:
            return False
        q = x_in.shape[2] - self.p.dilation * (self.p.taps - 1)
        return tuple(self.pre.shape) == (x_in.shape[0], self.p.filters, q)

    def backward_convs(self, grad_pre: torch.Tensor, dx: torch.Tensor | None = None) -> torch.Tensor:
        """backward-weight into grad_w and backward-data (gradient w.r.t. the padded input)."""
        cv.conv1d_backward_weight(grad_pre, self.x_in, self.p, out=self.grad_w)
        return cv.conv1d_backward_data(grad_pre, cv.pack_weights_backward(self.w), self.p, out=dx)

    def parameters(self):
        return [self.w, self.b]

    def gradients(self):
        return [self.grad_w, self.grad_b]


class ResidualNet:
    """BASELINE config 5: input layer, `blocks` residual blocks of `convs_per_block` convs, 2 heads."""

    def __init__(self, blocks=5, convs_per_block=3, hidden=15, taps=51, dilation=8,
                 precision=cv.Precision.Bf16, seed=1, device="cuda"):
        gen = torch.Generator(device=device).manual_seed(seed)
        self.device = device
        self.input = ConvLayer(1, hidden, taps, dilation, precision, True, False, 1.0, gen, device)
        self.blocks = [[ConvLayer(hidden, hidden, taps, dilation, precision, True, True, 0.3, gen, device)
                        for _ in range(convs_per_block)] for _ in range(blocks)]
        self.reg_head = ConvLayer(hidden, 1, 1, 1, cv.Precision.Fp32, False, False, 0.1, gen, device)
        self.peak_head = ConvLayer(hidden, 1, 1, 1, cv.Precision.Fp32, False, False, 0.1, gen, device)
        # both 1-tap heads run as ONE 2-filter FP32 conv (each output channel is accumulated on its
        # own, so the values are the separate heads'): h is read once per pass
        self.heads = ConvLayer(hidden, 2, 1, 1, cv.Precision.Fp32, False, False, 0.1, gen, device)
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
        self._bufs = {}

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

    # ---------------------------------------------------------------- activation buffers
    def _buf(self, name, shape, dtype, zero=False):
        """Persistent per-shape buffers (the zero borders of padded inputs are written once)."""
        key = (name, tuple(shape), dtype)
        t = self._bufs.get(key)
        if t is None:
            t = (torch.zeros if zero else torch.empty)(shape, dtype=dtype, device=self.device)
            self._bufs[key] = t
        return t

    def _padded_input(self, name, layer: ConvLayer, n: int, width: int):
        """Zero-bordered input buffer of a same-padded layer: bf16 for BF16 layers, fp32 otherwise."""
        dt = torch.bfloat16 if layer.bf16 else torch.float32
        return self._buf(name, (n, layer.p.channels, width + 2 * layer.pad), dt, zero=True)

    def _epilogue_into(self, layer: ConvLayer, nxt: ConvLayer, nxt_name: str, skip=None, act=None):
        """Fused glue after `layer`'s conv; writes the activation into `nxt`'s padded input."""
        n, k, q = layer.pre.shape
        nin = self._padded_input(nxt_name, nxt, n, q)
        if nxt.bf16:
            layer_forward_epilogue(layer.pre, layer.b, skip, layer.relu, act, nin, nxt.pad)
            return nin
        a = act if act is not None else self._buf(nxt_name + ".act", (n, k, q), torch.float32)
        layer_forward_epilogue(layer.pre, layer.b, skip, layer.relu, a, None, 0)
        nin[:, :, nxt.pad:nxt.pad + q].copy_(a)  # FP32 layers (tests / FP32 nets): plain padded copy
        return nin

    # ---------------------------------------------------------------- forward / backward
    def forward(self, x_padded: torch.Tensor):
        n = x_padded.shape[0]
        first = self.input
        x0 = cv.round_bf16(x_padded) if first.bf16 else x_padded.float().contiguous()
        first.conv(x0)
        width = first.pre.shape[2]
        h = self._buf("h.in", (n, first.p.filters, width), torch.float32)  # block input (skip source)
        nxt = self.blocks[0][0] if self.blocks else None
        if nxt is not None:
            x_next = self._epilogue_into(first, nxt, "x.b0.0", act=h)
        else:
            layer_forward_epilogue(first.pre, first.b, None, first.relu, h)
        for bi, blk in enumerate(self.blocks):
            skip = h
            for li, layer in enumerate(blk):
                layer.conv(x_next)
                last = li == len(blk) - 1
                if not last:
                    x_next = self._epilogue_into(layer, blk[li + 1], f"x.b{bi}.{li + 1}")
                    continue
                h = self._buf(f"h.b{bi}", (n, layer.p.filters, width), torch.float32)
                if bi + 1 < len(self.blocks):
                    x_next = self._epilogue_into(layer, self.blocks[bi + 1][0], f"x.b{bi + 1}.0", skip=skip, act=h)
                else:
                    layer_forward_epilogue(layer.pre, layer.b, skip, layer.relu, h)
        self.h_last = h
        heads = self.heads
        torch.cat([self.reg_head.w, self.peak_head.w], out=heads.w)
        torch.cat([self.reg_head.b, self.peak_head.b], out=heads.b)
        heads.conv(h)
        layer_forward_epilogue(heads.pre, heads.b, None, False, store_pre=True)
        return heads.pre[:, 0:1], heads.pre[:, 1:2]

    def backward(self, grad_pred: torch.Tensor, grad_logits: torch.Tensor) -> None:
        h = self.h_last
        n, hidden, width = h.shape
        # heads (one 2-filter conv): bias grads, dW, and the gradient w.r.t. the last block output
        # (backward-data of the 2-filter conv = the sum of both heads' backward-data)
        heads = self.heads
        g2 = self._buf("g.heads", (n, 2, width), torch.float32)
        torch.cat([grad_pred, grad_logits], dim=1, out=g2)
        layer_backward_prologue(g2, 0, None, n, 2, width, relu=False, bias_grad=heads.grad_b)
        gin = heads.backward_convs(g2, self._buf("dx.heads", (n, hidden, width), torch.float32))
        self.reg_head.grad_w.copy_(heads.grad_w[0:1])
        self.peak_head.grad_w.copy_(heads.grad_w[1:2])
        self.reg_head.grad_b.copy_(heads.grad_b[0:1])
        self.peak_head.grad_b.copy_(heads.grad_b[1:2])
        gin_off, gadd = 0, None
        for bi in reversed(range(len(self.blocks))):
            blk = self.blocks[bi]
            g_out = self._buf(f"g.b{bi}", (n, hidden, width), torch.float32)  # grad w.r.t. block output
            for li in reversed(range(len(blk))):
                layer = blk[li]
                gp = self._buf(f"gp.{li}", (n, hidden, width), torch.bfloat16 if layer.bf16 else torch.float32)
                last = li == len(blk) - 1
                layer_backward_prologue(gin, gin_off, layer.pre, n, hidden, width, relu=layer.relu,
                                        gadd=gadd if last else None, gsum=g_out if last else None,
                                        grad_pre=None if layer.bf16 else gp, grad_pre_bf16=gp if layer.bf16 else None,
                                        bias_grad=layer.grad_b, pre_bias=layer.b)
                dx = self._buf(f"dx.b.{li}", (n, hidden, width + 2 * layer.pad), torch.float32)
                layer.backward_convs(gp, dx)
                gin, gin_off, gadd = dx, layer.pad, None
            gadd = g_out  # the skip: block input gradient = conv path + block output gradient
        first = self.input
        gp = self._buf("gp.in", (n, hidden, width), torch.bfloat16 if first.bf16 else torch.float32)
        layer_backward_prologue(gin, gin_off, first.pre, n, hidden, width, relu=first.relu, gadd=gadd,
                                grad_pre=None if first.bf16 else gp, grad_pre_bf16=gp if first.bf16 else None,
                                bias_grad=first.grad_b, pre_bias=first.b)
        # gradient w.r.t. the padded network input: computed as the reference does, then discarded
        first.backward_convs(gp, self._buf("dx.in", (n, 1, first.x_in.shape[2]), torch.float32))

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
