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
* losses           mse_loss + bce_with_logits (train.cpp:106-135), means over the local batch, in one
                   device pass (c1d_mse_bce_loss) that writes both heads' gradients; torch
                   float64 restatements (mse_loss, bce_with_logits) stay for checks.
* `train_step`     forward, combined loss, backward; with a process group the gradients of every
                   layer (one flat bucket) are all-reduced and divided by the world size (the
                   local losses are means over local items).
* `sgd_step`       p <- p - lr*g (train.cpp:137-141) over the flat parameter / gradient buckets
                   (c1d_sgd_update, one launch).
* samplers         Poisson(2) inputs / targets and Bernoulli(0.1) labels (c1d_fill_poisson /
                   c1d_fill_bernoulli) for BASELINE config 5; `auroc` (train.cpp:143-171).

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
import os

import torch

from . import _lib as L
from . import conv as cv
from . import parallel


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
                       act_bf16=None, act_pad=0, mask=None, image=None):
    """c1d_forward_glued: conv + bias + ReLU (+ skip) in one call; the glue runs in the tcgen05 conv
    epilogue where the shape allows it. mask: int32 mask_shape(N, K, Q) ReLU-mask words. image: a
    weight image from pack_weights (C1D_FLAG_PREPACKED_WEIGHTS) used instead of w_kcs."""
    desc = _desc_for(x, p, x.shape[2])
    if image is not None:
        desc.flags |= L.FLAG_PREPACKED_WEIGHTS
    glue = L.FwdGlue(_ptr(bias), _ptr(skip), _ptr(pre), _ptr(act), _ptr(act_bf16), _ptr(mask), act_pad, int(relu), 0)
    w = image if image is not None else w_kcs
    cv._check(L.lib().c1d_forward_glued(C.byref(desc), x.data_ptr(), w.data_ptr(), C.byref(glue), None, 0,
                                        _stream()))


def conv_backward_data_glued(dy, w_kcs, p: cv.ConvParams, off: int, q: int, *, gadd=None, mask=None, gsum=None,
                             grad_pre=None, grad_pre_bf16=None, bias_grad=None, image=None):
    """c1d_backward_data_glued: backward-data, then the glue of the layer that owns columns
    [off, off + q) of the input gradient (skip gradient, ReLU mask bits, BF16 rounding, bias grad).
    image: a backward-data weight image from pack_weights, used instead of w_kcs."""
    w_in = dy.shape[2] + p.dilation * (p.taps - 1)
    desc = _desc_for(dy, p, w_in)
    if image is not None:
        desc.flags |= L.FLAG_PREPACKED_WEIGHTS
    glue = L.BwdGlue(off, q, _ptr(gadd), _ptr(mask), _ptr(gsum), _ptr(grad_pre), _ptr(grad_pre_bf16),
                     _ptr(bias_grad))
    w = image if image is not None else w_kcs
    cv._check(L.lib().c1d_backward_data_glued(C.byref(desc), dy.data_ptr(), w.data_ptr(), C.byref(glue), None,
                                              0, _stream()))


def packed_weights_bytes(p: cv.ConvParams, n: int, w_in: int, pass_: int) -> int:
    """Bytes of the pass's weight image (c1d_packed_weights_size), 0 when its plan packs its own."""
    b = C.c_size_t(0)
    st = L.lib().c1d_packed_weights_size(C.byref(cv.make_desc(p, n, w_in, L.DTYPE_BF16)), pass_, C.byref(b))
    return int(b.value) if st == 0 else 0


def pack_weights(jobs) -> None:
    """c1d_pack_weights: jobs = [(params, n, w_in, pass, w_kcs, image)], one launch per 32 images."""
    if not jobs:
        return
    cnt = len(jobs)
    descs = (L.Desc * cnt)(*[cv.make_desc(p, n, w_in, L.DTYPE_BF16) for p, n, w_in, _, _, _ in jobs])
    passes = (C.c_int32 * cnt)(*[j[3] for j in jobs])
    ws = (C.c_void_p * cnt)(*[j[4].data_ptr() for j in jobs])
    imgs = (C.c_void_p * cnt)(*[j[5].data_ptr() for j in jobs])
    cv._check(L.lib().c1d_pack_weights(cnt, descs, passes, ws, imgs, _stream()))


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
        self.img = {}  # pass -> weight image (C1D_FLAG_PREPACKED_WEIGHTS), refreshed by ResidualNet.forward

    @property
    def bf16(self) -> bool:
        return self.p.precision == cv.Precision.Bf16

    def out_width(self, x_in: torch.Tensor) -> int:
        return self.out_width_of(x_in.shape[2])

    def out_width_of(self, w_in: int) -> int:
        return w_in - self.p.dilation * (self.p.taps - 1)

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
                           act_bf16=act_bf16, act_pad=act_pad, mask=mask, image=self.img.get(L.PASS_FORWARD))

    def backward_weight(self, grad_pre: torch.Tensor) -> None:
        cv.conv1d_backward_weight(grad_pre, self.x_in, self.p, out=self.grad_w)

    def backward_data_into(self, dy: torch.Tensor, target: "ConvLayer | None", q: int, **glue) -> None:
        """backward-data of this layer (dy = its pre-activation gradient) glued to `target`'s
        backward (the layer whose activation is this layer's input, at columns [pad, pad + q) of
        the padded input gradient)."""
        conv_backward_data_glued(dy, self.w, self.p, self.pad, q,
                                 mask=target.mask if target is not None and target.relu else None,
                                 bias_grad=target.grad_b if target is not None else None,
                                 image=self.img.get(L.PASS_BACKWARD_DATA), **glue)

    def parameters(self):
        return [self.w, self.b]

    def gradients(self):
        return [self.grad_w, self.grad_b]


class ResidualNet:
    """BASELINE config 5: input layer, `blocks` residual blocks of `convs_per_block` convs, 2 heads."""

    def __init__(self, blocks=5, convs_per_block=3, hidden=15, taps=51, dilation=8,
                 precision=cv.Precision.Bf16, seed=1, device="cuda", precision_rule="all"):
        """precision_rule "all": every conv but the 1-tap heads runs in `precision` (BASELINE config
        5: BF16 with 15 channels, which the C ABI accepts). "reference": make_layer's rule
        (train.cpp:233-239), BF16 only where the channel and filter counts are both even, so the
        1-channel input layer stays FP32 (the layout the reference's DemoNet uses)."""
        if precision_rule not in ("all", "reference"):
            raise ValueError("precision_rule is 'all' or 'reference'")
        gen = torch.Generator(device=device).manual_seed(seed)
        self.device = device

        def prec(cin, cout):
            if precision_rule == "reference" and (cin % 2 or cout % 2):
                return cv.Precision.Fp32
            return precision

        self.input = ConvLayer(1, hidden, taps, dilation, prec(1, hidden), True, False, 1.0, gen, device)
        self.blocks = [[ConvLayer(hidden, hidden, taps, dilation, prec(hidden, hidden), True, True, 0.3, gen, device)
                        for _ in range(convs_per_block)] for _ in range(blocks)]
        self.reg_head = ConvLayer(hidden, 1, 1, 1, cv.Precision.Fp32, False, False, 0.1, gen, device)
        self.peak_head = ConvLayer(hidden, 1, 1, 1, cv.Precision.Fp32, False, False, 0.1, gen, device)
        # both 1-tap heads run as ONE 2-filter FP32 conv (each output channel is accumulated on its
        # own, so the values are the separate heads'): h is read once per pass
        self.heads = ConvLayer(hidden, 2, 1, 1, cv.Precision.Fp32, False, False, 0.1, gen, device)
        # one flat gradient bucket (all dW and bias grads) for a single all-reduce per step, and a
        # parameter bucket in the same order (w then bias per layer, the reference's gather_params
        # order, train.cpp:318-325) so the SGD update is one pass over two flat vectors
        layers = self.layers()
        n = sum(t.numel() for layer in layers for t in layer.gradients())
        self.grad_bucket = torch.zeros(n, device=device)
        self.param_bucket = torch.zeros(n, device=device)
        off = 0
        for layer in layers:
            gviews, pviews = [], []
            for g, prm in zip(layer.gradients(), layer.parameters()):
                gviews.append(self.grad_bucket[off:off + g.numel()].view_as(g))
                pv = self.param_bucket[off:off + prm.numel()].view_as(prm)
                pv.copy_(prm)
                pviews.append(pv)
                off += g.numel()
            layer.grad_w, layer.grad_b = gviews
            layer.w, layer.b = pviews
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
    def _pack_images(self, n: int, w_first: int) -> None:
        """One c1d_pack_weights launch for the step: every BF16 conv's forward image and every body
        conv's backward-data image (the weights changed at the last SGD step). The glued passes then
        skip their own pack launches and load their images while the previous kernel runs."""
        if os.environ.get("C1D_NET_NO_PREPACK"):  # dev A/B switch
            for layer in self.layers():
                layer.img = {}
            return
        jobs = []
        width = self.input.out_width_of(w_first)
        chain = [(self.input, w_first, False)] + [(layer, width + 2 * layer.pad, True)
                                                  for blk in self.blocks for layer in blk]
        for layer, w_in, bwd in chain:
            if not layer.bf16:
                continue
            for pass_ in ((L.PASS_FORWARD, L.PASS_BACKWARD_DATA) if bwd else (L.PASS_FORWARD,)):
                img = layer.img.get(pass_)
                if img is None:
                    nb = packed_weights_bytes(layer.p, n, w_in, pass_)
                    if nb == 0:
                        continue
                    img = torch.empty(nb, dtype=torch.uint8, device=layer.w.device)
                    layer.img[pass_] = img
                jobs.append((layer.p, n, w_in, pass_, layer.w, img))
        pack_weights(jobs)

    def forward(self, x_padded: torch.Tensor):
        n = x_padded.shape[0]
        first = self.input
        self._pack_images(n, x_padded.shape[2])
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
        g2 = self.head_grad_buffer(n, width)
        torch.cat([grad_pred, grad_logits], dim=1, out=g2)
        self.backward_heads(g2)

    def head_grad_buffer(self, n: int, width: int) -> torch.Tensor:
        """(N, 2, width) gradient of the two heads' outputs (channel 0 regression, 1 peak logits)."""
        return self._buf("g.heads", (n, 2, width), torch.float32)

    def _wgrad_stream(self, dev):
        """Side stream for the backward-weight passes (None: run them in order on the current
        stream; C1D_NET_SERIAL=1, a dev A/B switch)."""
        if os.environ.get("C1D_NET_SERIAL"):
            return None
        if getattr(self, "_side", None) is None or self._side.device != dev:
            self._side = torch.cuda.Stream(dev)
        return self._side

    def backward_heads(self, g2: torch.Tensor) -> None:
        """The backward pass from the heads' output gradient g2 = head_grad_buffer(...).

        Each layer's backward-weight (reads its pre-activation gradient gp and its forward input)
        runs on a side stream, concurrently with that layer's glued backward-data (which writes the
        other gp slot); the next backward-data, which overwrites this gp slot, waits for it. The
        kernels and their inputs are the same as in order, so the results are bit-identical; the
        overlap fills each pass's fill / drain tails and takes the wgrad reduce off the critical
        path (it matters most at the small per-rank batches of data-parallel strong scaling)."""
        h = self.h_last
        n, hidden, width = h.shape
        heads = self.heads
        main = torch.cuda.current_stream(g2.device)
        side = self._wgrad_stream(g2.device)

        def wgrad_async(layer, grad):
            if side is None:
                layer.backward_weight(grad)
                return None
            side.wait_stream(main)  # grad is ready
            with torch.cuda.stream(side):
                layer.backward_weight(grad)
            ev = torch.cuda.Event()
            ev.record(side)
            return ev

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
            wg_done = wgrad_async(layer, gp)
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
            if wg_done is not None:
                main.wait_event(wg_done)  # the next backward-data overwrites the gp slot it reads
            gp = gp_next
        first = self.input
        wg_done = wgrad_async(first, gp)
        # gradient w.r.t. the padded network input: computed as the reference does, then discarded
        cv.conv1d_backward_data(gp, first.w, first.p, out=self._buf("dx.in", (n, 1, first.x_in.shape[2]),
                                                                     torch.float32))
        if wg_done is not None:
            main.wait_event(wg_done)

    def load_params(self, flat) -> None:
        """Set every weight and bias from a flat vector in the reference's gather_params order
        (train.cpp:318-325; layers() order, w then bias)."""
        flat = torch.as_tensor(flat, dtype=torch.float32).reshape(-1)
        if flat.numel() != self.param_bucket.numel():
            raise cv.ShapeMismatch(f"flat parameter vector has {flat.numel()} values, the net {self.param_bucket.numel()}")
        self.param_bucket.copy_(flat.to(self.param_bucket.device))

    def sgd_step(self, lr: float) -> None:
        """p <- p - lr*g over the flat buckets (sgd_step, train.cpp:137-141): one fused launch."""
        if not lr > 0:
            raise ValueError("sgd_step needs a positive learning rate")
        sgd_update_(self.param_bucket, self.grad_bucket, lr)


def sgd_update_(params: torch.Tensor, grads: torch.Tensor, lr: float) -> None:
    """params <- params - lr*grads in place: c1d_sgd_update, one launch over the flat buckets with
    the reference's float rounding (a multiply, then a subtract; train.cpp:137-141)."""
    if params.shape != grads.shape or params.dtype != torch.float32 or not params.is_contiguous() \
            or not grads.is_contiguous():
        raise cv.ShapeMismatch("sgd_update_ needs two contiguous float32 tensors of one shape")
    cv._check(L.lib().c1d_sgd_update(params.data_ptr(), grads.data_ptr(), params.numel(), lr,
                                     torch.cuda.current_stream(params.device).cuda_stream))


def fill_poisson(shape, lam: float, seed: int, device) -> torch.Tensor:
    """Poisson(lam) counts as float32 (c1d_fill_poisson: Knuth's product of uniforms on a
    per-element splitmix64 stream; the reference's Rng has no Poisson sampler)."""
    out = torch.empty(shape, dtype=torch.float32, device=device)
    cv._check(L.lib().c1d_fill_poisson(out.data_ptr(), out.numel(), lam, seed,
                                       torch.cuda.current_stream(out.device).cuda_stream))
    return out


def fill_bernoulli(shape, p: float, seed: int, device) -> torch.Tensor:
    """Bernoulli(p) 0/1 labels as float32 (c1d_fill_bernoulli, same per-element streams)."""
    out = torch.empty(shape, dtype=torch.float32, device=device)
    cv._check(L.lib().c1d_fill_bernoulli(out.data_ptr(), out.numel(), p, seed,
                                         torch.cuda.current_stream(out.device).cuda_stream))
    return out


def sample_inputs(n: int, width: int, pad: int, seed: int, device):
    """BASELINE config 5's synthetic batch: inputs ~ Poisson(2) zero-padded by `pad` columns per
    side, regression targets ~ Poisson(2), peak labels ~ Bernoulli(0.1); three seeded streams."""
    x = torch.zeros((n, 1, width + 2 * pad), dtype=torch.float32, device=device)
    x[:, :, pad:pad + width] = fill_poisson((n, 1, width), 2.0, 3 * seed, device)
    return x, fill_poisson((n, 1, width), 2.0, 3 * seed + 1, device), fill_bernoulli((n, 1, width), 0.1, 3 * seed + 2,
                                                                                    device)


_LOSS_WS = {}


def mse_bce(pred: torch.Tensor, logits: torch.Tensor, target: torch.Tensor, labels: torch.Tensor,
            bce_weight: float = 1.0, grad: torch.Tensor | None = None) -> torch.Tensor:
    """mse_loss + bce_weight * bce_with_logits on the device (c1d_mse_bce_loss, one pass;
    train.cpp:106-135). pred / logits are (N, 1, W) views sharing one item stride (e.g. channels 0
    and 1 of the heads' (N, 2, W) output); grad, if given, is an (N, 2, W) buffer that receives
    the regression gradient in channel 0 and bce_weight * the logit gradient in channel 1.
    Returns a float64 device tensor [mse, bce, total]."""
    n, _, width = pred.shape
    stride = pred.stride(0)
    if logits.stride(0) != stride or pred.stride(2) != 1 or logits.stride(2) != 1:
        raise cv.ShapeMismatch("pred and logits must be unit-stride rows with one item stride")
    tgt, lab = target.contiguous(), labels.contiguous()
    if tgt.numel() != n * width or lab.numel() != n * width:
        raise cv.ShapeMismatch("targets and labels must be (N, 1, W)")
    dev = pred.device
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    ws = _LOSS_WS.get(key)
    if ws is None:
        ws = torch.zeros(L.lib().c1d_loss_workspace_size(), dtype=torch.uint8, device=dev)
        _LOSS_WS[key] = ws
    out = torch.empty(3, dtype=torch.float64, device=dev)
    gp = gl = None
    gstride = 0
    if grad is not None:
        if tuple(grad.shape) != (n, 2, width) or not grad.is_contiguous():
            raise cv.ShapeMismatch("grad must be a contiguous (N, 2, W) buffer")
        gp, gl, gstride = grad.data_ptr(), grad.data_ptr() + 4 * width, 2 * width
    cv._check(L.lib().c1d_mse_bce_loss(pred.data_ptr(), logits.data_ptr(), stride, tgt.data_ptr(), lab.data_ptr(), n,
                                       width, bce_weight, gp, gl, gstride, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                       torch.cuda.current_stream(dev).cuda_stream))
    return out


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


def auroc(scores: torch.Tensor, labels: torch.Tensor) -> float:
    """Area under the ROC curve by the rank statistic with ties averaged (auroc, train.cpp:143-171),
    on the device: stable sort, tie groups as runs of equal scores, 1-based ranks i+1..j averaged
    per group, U = sum of positive ranks - P(P+1)/2, AUROC = U / (P*N). NaN with one class."""
    s = scores.reshape(-1).float()
    pos_mask = labels.reshape(-1) > 0.5
    n = s.numel()
    order = torch.argsort(s, stable=True)
    ss, ll = s[order], pos_mask[order].double()
    _, counts = torch.unique_consecutive(ss, return_counts=True)
    ends = torch.cumsum(counts, 0).double()
    rank = 0.5 * (ends - counts.double() + 1 + ends)
    group = torch.repeat_interleave(torch.arange(counts.numel(), device=s.device), counts)
    pos_per_group = torch.zeros(counts.numel(), dtype=torch.float64, device=s.device).index_add_(0, group, ll)
    pos = float(ll.sum())
    neg = n - pos
    if pos == 0.0 or neg == 0.0:
        return float("nan")
    u = float((rank * pos_per_group).sum()) - pos * (pos + 1.0) / 2.0
    return u / (pos * neg)


def forward_backward(net: ResidualNet, x_padded, target, labels, bce_weight: float = 1.0):
    """The local part of a training step (train_step, train.cpp:327-353): forward, combined loss
    mse + bce_weight*bce, full backward into net.grad_bucket. No collective, so it can be captured
    in a CUDA graph. Returns the local loss (a device tensor)."""
    pred, logits = net.forward(x_padded)
    n, _, width = pred.shape
    g2 = net.head_grad_buffer(n, width)
    loss3 = mse_bce(pred, logits, target, labels, bce_weight, grad=g2)  # losses + both head gradients
    net.backward_heads(g2)
    return loss3[2]


def train_step(net: ResidualNet, x_padded, target, labels, bce_weight: float = 1.0, group=None):
    """One data-parallel training step on this rank's shard: forward_backward, then the bucket
    all-reduce divided by the world size (parallel.allreduce_mean_). Returns the local loss."""
    loss = forward_backward(net, x_padded, target, labels, bce_weight)
    parallel.allreduce_mean_(net.grad_bucket, group)
    return loss
