"""Host-buffer layer step with the PCIe transfers overlapped with the conv kernels.

The reference operator API takes host arrays (conv.hpp:42-57, std::vector storage) and returns
host arrays. Through the device C ABI that means H2D of the inputs, the pass, and D2H of the
outputs. Run naively these serialise, and at config 3 the 1.5 GB of transfers take ~14x longer than
the three passes. ``HostLayerStep`` splits the batch into item chunks and runs three streams:

    copy-in  : x[i], dy[i]  host -> device                  (waits for chunk i's previous use)
    compute  : forward(x[i]) -> y[i], backward_data(dy[i]) -> dx[i],
               backward_weight(x[i], dy[i]) -> dW_part[i]   (waits for copy-in i)
    copy-out : y[i], dx[i]  device -> host                  (waits for compute i)

so chunk i+1's upload and chunk i-1's download run while chunk i computes, in both PCIe
directions at once. Items are independent in forward and backward-data (conv.cpp:24-25), so y
and dx are bitwise the single-call results. dW is the fixed-order sum of the per-chunk partials
(chunk 0 + 1 + ...), the multi-chunk analogue of the reference's ascending-item sum
(conv.cpp:308-314).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L
from . import conv as cv


class HostLayerStep:
    """fwd + bwd-d + bwd-w of one conv layer from pinned host buffers, transfers pipelined."""

    def __init__(self, p: cv.ConvParams, n: int, w_in: int, chunks: int = 4, device=None,
                 in_dtype: torch.dtype = torch.bfloat16):
        if n % chunks:
            raise ValueError(f"batch {n} is not a multiple of chunks={chunks}")
        if in_dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("inputs are bfloat16 or float32")
        self.p, self.n, self.w_in, self.chunks = p, n, w_in, chunks
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.q = w_in - p.dilation * (p.taps - 1)
        if self.q <= 0:
            raise cv.TooNarrow("input narrower than the receptive field")
        dt = L.DTYPE_BF16 if in_dtype == torch.bfloat16 else L.DTYPE_F32
        self.desc = cv.make_desc(p, n // chunks, w_in, dt)
        k, c, m = p.filters, p.channels, n // chunks
        self.x = torch.empty((chunks, m, c, w_in), dtype=in_dtype, device=self.dev)
        self.dy = torch.empty((chunks, m, k, self.q), dtype=in_dtype, device=self.dev)
        self.y = torch.empty((chunks, m, k, self.q), dtype=torch.float32, device=self.dev)
        self.dx = torch.empty((chunks, m, c, w_in), dtype=torch.float32, device=self.dev)
        self.dw_parts = torch.empty((chunks, k, c, p.taps), dtype=torch.float32, device=self.dev)
        self.dw = torch.empty((k, c, p.taps), dtype=torch.float32, device=self.dev)
        self.s_in = torch.cuda.Stream(device=self.dev)
        self.s_out = torch.cuda.Stream(device=self.dev)
        self.ev_in = [torch.cuda.Event() for _ in range(chunks)]
        self.ev_comp = [torch.cuda.Event() for _ in range(chunks)]
        self.ev_out = [torch.cuda.Event() for _ in range(chunks)]
        self.ev_dw = torch.cuda.Event()
        self.ev_dw_out = torch.cuda.Event()
        self._ran = False

    def h2d_bytes(self) -> int:
        return self.x.numel() * self.x.element_size() + self.dy.numel() * self.dy.element_size()

    def d2h_bytes(self) -> int:
        return (self.y.numel() + self.dx.numel() + self.dw.numel()) * 4

    def run(self, hx: torch.Tensor, hdy: torch.Tensor, w: torch.Tensor, hy: torch.Tensor, hdx: torch.Tensor,
            hdw: torch.Tensor, compute: torch.cuda.Stream | None = None, reduce_dw=None) -> None:
        """Enqueue one step. hx (N,C,W_in), hdy (N,K,Q): pinned host inputs in the step's dtype;
        w (K,C,S) fp32 on the device; hy (N,K,Q), hdx (N,C,W_in), hdw (K,C,S): pinned fp32 host
        outputs. ``reduce_dw(t)``, if given, runs on the compute stream on the summed dW before its
        download (the data-parallel all-reduce). Returns without synchronising; the outputs are
        complete once ``s_out`` drains."""
        for t in (hx, hdy, hy, hdx, hdw):
            if t.is_cuda or not t.is_pinned():
                raise cv.ShapeMismatch("host buffers must be pinned CPU tensors")
        comp = compute if compute is not None else torch.cuda.current_stream(self.dev)
        lib = L.lib()
        sp = comp.cuda_stream
        cx, cdy = hx.view(self.x.shape), hdy.view(self.dy.shape)
        cy, cdx = hy.view(self.y.shape), hdx.view(self.dx.shape)
        wp = w.data_ptr()
        for i in range(self.chunks):
            with torch.cuda.stream(self.s_in):
                if self._ran:  # chunk i's inputs of the previous step are consumed
                    self.s_in.wait_event(self.ev_comp[i])
                self.x[i].copy_(cx[i], non_blocking=True)
                self.dy[i].copy_(cdy[i], non_blocking=True)
                self.ev_in[i].record(self.s_in)
            comp.wait_event(self.ev_in[i])
            if self._ran:  # chunk i's outputs of the previous step are downloaded
                comp.wait_event(self.ev_out[i])
            cv._check(lib.c1d_forward(C.byref(self.desc), self.x[i].data_ptr(), wp, self.y[i].data_ptr(), None, 0, sp))
            cv._check(lib.c1d_backward_data(C.byref(self.desc), self.dy[i].data_ptr(), wp, self.dx[i].data_ptr(),
                                            None, 0, sp))
            cv._check(lib.c1d_backward_weight(C.byref(self.desc), self.x[i].data_ptr(), self.dy[i].data_ptr(),
                                              self.dw_parts[i].data_ptr(), None, 0, sp))
            self.ev_comp[i].record(comp)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.ev_comp[i])
                cy[i].copy_(self.y[i], non_blocking=True)
                cdx[i].copy_(self.dx[i], non_blocking=True)
                self.ev_out[i].record(self.s_out)
        with torch.cuda.stream(comp):
            if self._ran:
                comp.wait_event(self.ev_dw_out)
            acc = self.dw_parts[0].clone() if self.chunks > 1 else self.dw_parts[0]
            for i in range(1, self.chunks):  # fixed order: chunk 0 + 1 + ...
                acc.add_(self.dw_parts[i])
            self.dw.copy_(acc)
            if reduce_dw is not None:
                reduce_dw(self.dw)
            self.ev_dw.record(comp)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_dw)
            hdw.copy_(self.dw, non_blocking=True)
            self.ev_dw_out.record(self.s_out)
        self._ran = True
