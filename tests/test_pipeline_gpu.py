"""Pipelined host-buffer layer step (pipeline.HostLayerStep) vs the single-call device passes:
forward / backward-data bitwise (items are independent), dW within FP32 summation-order error."""
import pytest
import torch

from paper_2104_08002_b200 import conv as cv
from paper_2104_08002_b200.pipeline import HostLayerStep

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("chunks", [1, 2, 4])
def test_pipeline_matches_single_calls(chunks):
    n, c, k, s, q = 4, 16, 16, 51, 1024
    w_in = q + 8 * (s - 1)
    p = cv.ConvParams(c, k, s, 8, cv.Precision.Bf16)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((n, c, w_in), device="cuda", generator=g).bfloat16()
    dy = torch.randn((n, k, q), device="cuda", generator=g).bfloat16()
    w = torch.randn((k, c, s), device="cuda", generator=g) * 0.05
    y_ref = cv.conv1d_forward(x, w, p)
    dx_ref = cv.conv1d_backward_data(dy, cv.pack_weights_backward(w), p)
    dw_ref = cv.conv1d_backward_weight(dy, x, p)
    pipe = HostLayerStep(p, n, w_in, chunks=chunks)
    hx, hdy = x.cpu().pin_memory(), dy.cpu().pin_memory()
    hy = torch.empty(y_ref.shape, pin_memory=True)
    hdx = torch.empty(dx_ref.shape, pin_memory=True)
    hdw = torch.empty(dw_ref.shape, pin_memory=True)
    for _ in range(2):  # the second run exercises the cross-step buffer hazards
        pipe.run(hx, hdy, w, hy, hdx, hdw)
    torch.cuda.synchronize()
    assert torch.equal(hy, y_ref.cpu())
    assert torch.equal(hdx, dx_ref.cpu())
    err = (hdw - dw_ref.cpu()).abs().max() / dw_ref.abs().max().cpu()
    assert err <= 1e-6
