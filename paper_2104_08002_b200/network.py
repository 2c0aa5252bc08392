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

Fused glue (through the C ABI's glued passes): every layer's forward is ONE
call, c1d_forward_glued, whose tcgen05 epilogue adds the bias, applies ReLU and the skip, writes
the ReLU-mask bits and the activation straight into the next layer's zero-padded BF16 input
buffer (the FP32 conv output never reaches HBM). Every backward-data pass is ONE call,
c1d_backward_data_glued, whose epilogue applies the glue of the layer below: the interior of the
input gradient plus the skip gradient, the ReLU mask, BF16 rounding for that layer's own backward
passes and deterministic bias-gradient partial sums. BF16 layers never see an FP32 copy of their
input: the activation is rounded once, where the reference's conv would round it
(conv.cpp:182-183). Shapes off the tensor-core path run the same calls as conv + one glue pass.

Weights are Kaiming-uniform with the reference's damping (input 1.0, body 0.3, heads 0.1;
train.cpp:247-248, 263-268), seeded.
"""
from __future__ import annotations

import ctypes as C
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


def mask_shape(n: int, channels: int, q: int) -> tuple:
    """ReLU-mask tensor (int32): word (n, b, x) holds channels 16b..16b+15 of column x (c1d.h)."""
    return (n, (channels + 15) // 16, q)


def _desc_for(x: torch.Tensor, p: cv.ConvParams, w_in: int):
    dt = L.DTYPE_BF16 if x.dtype == torch.bfloat16 else L.DTYPE_F32
    return cv.make_desc(p, x.shape[0], w_in, dt)


def conv_forward_glued(x, w_kcs, p: cv.ConvParams, *, bias=None, skip=None, relu=True, pre=None, act=None,
                       act_bf16=None, act_pad=0, mask=None):
    """c1d_forward_glued: conv + bias + ReLU (+ skip) in one call; the glue runs in the tcgen05 conv
    epilogue where the shape allows it. mask: int32 mask_shape(N, K, Q) ReLU-mask words."""
    desc = _desc_for(x, p, x.shape[2])
    glue = L.FwdGlue(_ptr(bias), _ptr(skip), _ptr(pre), _ptr(act), _ptr(act_bf16), _ptr(mask), act_pad, int(relu), 0)
    cv._check(L.lib().c1d_forward_glued(C.byref(desc), x.data_ptr(), w_kcs.data_ptr(), C.byref(glue), None, 0,
                                        _stream()))


def conv_backward_data_glued(dy, w_kcs, p: cv.ConvParams, off: int, q: int, *, gadd=None, mask=None, gsum=None,
                             grad_pre=None, grad_pre_bf16=None, bias_grad=None):
    """c1d_backward_data_glued: backward-data, then the glue of the layer that owns columns
    [off, off + q) of the input gradient (skip gradient, ReLU mask bits, BF16 rounding, bias grad)."""
    w_in = dy.shape[2] + p.dilation * (p.taps - 1)
    desc = _desc_for(dy, p, w_in)
    glue = L.BwdGlue(off, q, _ptr(gadd), _ptr(mask), _ptr(gsum), _ptr(grad_pre), _ptr(grad_pre_bf16),
                     _ptr(bias_grad))
    cv._check(L.lib().c1d_backward_data_glued(C.byref(desc), dy.data_ptr(), w_kcs.data_ptr(), C.byref(glue), None,
                                              0, _stream()))


def glue_is_fused(p: cv.ConvParams, n: int, w_in: int, pass_: int, in_dtype: int = L.DTYPE_BF16) -> bool:
    """Whether the glued pass runs its glue inside the tcgen05 conv epilogue."""
    b, f = C.c_size_t(0), C.c_int(0)
    cv._check(L.lib().c1d_glued_workspace_size(C.byref(cv.make_desc(p, n, w_in, in_dtype)), pass_, 1, C.byref(b),
                                               C.byref(f)))
    return bool(f.value)


class ConvLayer:
    """One conv with bias, optional ReLU and optional skip input (train.hpp ConvLayer).

    The forward reads `self.x_in` (N, C, W_in) — bf16 for BF16 layers (zero-padded, as written by
    the previous layer's glued epilogue), fp32 otherwise — and leaves `self.mask`, the ReLU-mask
    bits of conv + bias > 0 that the backward glue reads (no FP32 pre-activation is kept)."""

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
        self.mask = None

    @property
    def bf16(self) -> bool:
        return self.p.precision == cv.Precision.Bf16

    def out_width(self, x_in: torch.Tensor) -> int:
        return x_in.shape[2] - self.p.dilation * (self.p.taps - 1)

    def forward(self, x_in: torch.Tensor, *, skip=None, act=None, act_bf16=None, act_pad=0, pre=None):
        """Glued forward (c1d_forward_glued): conv, bias, ReLU, skip, activation outputs."""
        self.x_in = x_in
        n, q = x_in.shape[0], self.out_width(x_in)
        mask = None
        if self.relu:
            shape = mask_shape(n, self.p.filters, q)
            if self.mask is None or tuple(self.mask.shape) != shape:
                self.mask = torch.empty(shape, dtype=torch.int32, device=x_in.device)
            mask = self.mask
        conv_forward_glued(x_in, self.w, self.p, bias=self.b, skip=skip, relu=self.relu, pre=pre, act=act,
                           act_bf16=act_bf16, act_pad=act_pad, mask=mask)

    def backward_weight(self, grad_pre: torch.Tensor) -> None:
        cv.conv1d_backward_weight(grad_pre, self.x_in, self.p, out=self.grad_w)

    def backward_data_into(self, dy: torch.Tensor, target: "ConvLayer | None", q: int, **glue) -> None:
        """backward-data of this layer (dy = its pre-activation gradient) glued to `target`'s
        backward (the layer whose activation is this layer's input, at columns [pad, pad + q) of
        the padded input gradient)."""
        conv_backward_data_glued(dy, self.w, self.p, self.pad, q,
                                 mask=target.mask if target is not None and target.relu else None,
                                 bias_grad=target.grad_b if target is not None else None, **glue)

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

    def _run_into(self, layer: ConvLayer, x_in, nxt: ConvLayer | None, nxt_name: str, skip=None, act=None):
        """Glued forward of `layer`; its activation goes straight into `nxt`'s padded input (BF16) or
        through `act` (FP32 consumers). Returns nxt's input (or None)."""
        n, q = x_in.shape[0], layer.out_width(x_in)
        if nxt is None:
            layer.forward(x_in, skip=skip, act=act)
            return None
        nin = self._padded_input(nxt_name, nxt, n, q)
        if nxt.bf16:
            layer.forward(x_in, skip=skip, act=act, act_bf16=nin, act_pad=nxt.pad)
            return nin
        a = act if act is not None else self._buf(nxt_name + ".act", (n, layer.p.filters, q), torch.float32)
        layer.forward(x_in, skip=skip, act=a)
        nin[:, :, nxt.pad:nxt.pad + q].copy_(a)  # FP32 layers (tests / FP32 nets): plain padded copy
        return nin

    # ---------------------------------------------------------------- forward / backward
    def forward(self, x_padded: torch.Tensor):
        n = x_padded.shape[0]
        first = self.input
        x0 = cv.round_bf16(x_padded) if first.bf16 else x_padded.float().contiguous()
        width = first.out_width(x0)
        h = self._buf("h.in", (n, first.p.filters, width), torch.float32)  # block input (skip source)
        x_next = self._run_into(first, x0, self.blocks[0][0] if self.blocks else None, "x.b0.0", act=h)
        for bi, blk in enumerate(self.blocks):
            skip = h
            for li, layer in enumerate(blk):
                if li < len(blk) - 1:
                    x_next = self._run_into(layer, x_next, blk[li + 1], f"x.b{bi}.{li + 1}")
                    continue
                h = self._buf(f"h.b{bi}", (n, layer.p.filters, width), torch.float32)
                nxt = self.blocks[bi + 1][0] if bi + 1 < len(self.blocks) else None
                x_next = self._run_into(layer, x_next, nxt, f"x.b{bi + 1}.0", skip=skip, act=h)
        self.h_last = h
        heads = self.heads
        torch.cat([self.reg_head.w, self.peak_head.w], out=heads.w)
        torch.cat([self.reg_head.b, self.peak_head.b], out=heads.b)
        pre = self._buf("heads.pre", (n, 2, width), torch.float32)
        heads.forward(h, pre=pre)
        return pre[:, 0:1], pre[:, 1:2]

    def backward(self, grad_pred: torch.Tensor, grad_logits: torch.Tensor) -> None:
        """Each backward-data pass carries the glue of the layer below it (c1d_backward_data_glued):
        skip gradient, ReLU mask, BF16 rounding and bias gradient happen in the conv epilogue."""
        h = self.h_last
        n, hidden, width = h.shape
        heads = self.heads
        g2 = self._buf("g.heads", (n, 2, width), torch.float32)
        torch.cat([grad_pred, grad_logits], dim=1, out=g2)
        layer_backward_prologue(g2, 0, None, n, 2, width, relu=False, bias_grad=heads.grad_b)
        heads.backward_weight(g2)
        chain = [self.input] + [layer for blk in self.blocks for layer in blk]  # forward order

        def gp_buf(layer, slot):
            return self._buf(f"gp.{slot}", (n, hidden, width), torch.bfloat16 if layer.bf16 else torch.float32)

        def glue_out(layer, slot):
            gp = gp_buf(layer, slot)
            return gp, ({"grad_pre_bf16": gp} if layer.bf16 else {"grad_pre": gp})

        # chain index of each block's first conv: its backward-data feeds the block input, which
        # also receives the block output's gradient through the skip
        first_of_block = {}
        idx = 1
        for bi, blk in enumerate(self.blocks):
            first_of_block[idx] = bi
            idx += len(blk)

        # heads' backward-data -> glue of the last chain layer (the last block's output layer)
        top = chain[-1]
        slot = 0
        gp, kw = glue_out(top, slot)
        g_out = None
        if self.blocks:
            g_out = self._buf(f"g.b{len(self.blocks) - 1}", (n, hidden, width), torch.float32)
            kw["gsum"] = g_out
        heads.backward_data_into(g2, top, width, **kw)
        self.reg_head.grad_w.copy_(heads.grad_w[0:1])
        self.peak_head.grad_w.copy_(heads.grad_w[1:2])
        self.reg_head.grad_b.copy_(heads.grad_b[0:1])
        self.peak_head.grad_b.copy_(heads.grad_b[1:2])
        g_outs = {len(self.blocks) - 1: g_out} if self.blocks else {}
        for li in range(len(chain) - 1, 0, -1):
            layer, below = chain[li], chain[li - 1]
            layer.backward_weight(gp)
            slot ^= 1
            gp_next, kw = glue_out(below, slot)
            if li in first_of_block:
                # below = the previous block's output (or the input layer): + the skip gradient
                bi = first_of_block[li]
                kw["gadd"] = g_outs[bi]
                if bi > 0:
                    g_outs[bi - 1] = self._buf(f"g.b{bi - 1}", (n, hidden, width), torch.float32)
                    kw["gsum"] = g_outs[bi - 1]
            layer.backward_data_into(gp, below, width, **kw)
            gp = gp_next
        first = self.input
        first.backward_weight(gp)
        # gradient w.r.t. the padded network input: computed as the reference does, then discarded
        cv.conv1d_backward_data(gp, first.w, first.p, out=self._buf("dx.in", (n, 1, first.x_in.shape[2]),
                                                                     torch.float32))

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
