"""conv.py caches the natural KCS copy of a PackedWeights object (the reference API passes packed
weights on every call); the cache must follow in-place updates of the packed data and
replacement of the data tensor, e.g. an optimizer step between two calls."""
import pytest
import torch

from paper_2104_08002_b200 import conv as cv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("layout", ["forward", "backward"])
def test_packed_weight_cache_follows_updates(layout):
    g = torch.Generator(device="cuda").manual_seed(3)
    c, k, s, d, q, n = 15, 15, 51, 8, 2000, 2
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    w = torch.randn((k, c, s), device="cuda", generator=g) * 0.05
    if layout == "forward":
        x = cv.round_bf16(torch.randn((n, c, q + d * (s - 1)), device="cuda", generator=g))
        pack, run = cv.pack_weights_forward, lambda pw: cv.conv1d_forward(x, pw, p)
    else:
        dy = cv.round_bf16(torch.randn((n, k, q), device="cuda", generator=g))
        pack, run = cv.pack_weights_backward, lambda pw: cv.conv1d_backward_data(dy, pw, p)
    pw = pack(w)
    first = run(pw)
    assert torch.equal(run(pw), first)  # cached copy, same result
    pw.data.mul_(2.0)  # in-place update of the packed data (exact in FP32 and BF16)
    assert torch.equal(run(pw), 2.0 * first)
    pw.data = pack(3.0 * w).data  # replaced tensor
    assert torch.allclose(run(pw), run(pack(3.0 * w)), rtol=0, atol=0)
