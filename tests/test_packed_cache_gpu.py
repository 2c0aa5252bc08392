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


@pytest.mark.parametrize("layout", ["forward", "backward"])
@pytest.mark.parametrize("shape", [(15, 15, 51, 8), (16, 16, 3, 8), (64, 64, 51, 8), (16, 16, 9, 1)])
def test_packed_weights_carry_the_device_image(layout, shape):
    """PackedWeights build the pass's device weight image once (packing is setup work, bench.cpp:184-203)
    where the plan takes one; the result is bit-identical to the call with KCS weights, which packs
    inside the call. Plans without images (wide filter groups, other dilations) keep the KCS copy."""
    from paper_2104_08002_b200 import _lib as L
    from paper_2104_08002_b200.network import packed_weights_bytes

    c, k, s, d = shape
    g = torch.Generator(device="cuda").manual_seed(5)
    q, n = 3000, 3
    w_in = q + d * (s - 1)
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    w = torch.randn((k, c, s), device="cuda", generator=g) * 0.05
    if layout == "forward":
        x = cv.round_bf16(torch.randn((n, c, w_in), device="cuda", generator=g))
        pw, pi = cv.pack_weights_forward(w), L.PASS_FORWARD
        run = lambda wt: cv.conv1d_forward(x, wt, p)  # noqa: E731
    else:
        dy = cv.round_bf16(torch.randn((n, k, q), device="cuda", generator=g))
        pw, pi = cv.pack_weights_backward(w), L.PASS_BACKWARD_DATA
        run = lambda wt: cv.conv1d_backward_data(dy, wt, p)  # noqa: E731
    packed_out = run(pw)
    images = [v for v in pw.__dict__["_images"].values()]
    assert len(images) == 1
    assert (images[0] is not None) == (packed_weights_bytes(p, n, w_in, pi) > 0)
    assert torch.equal(packed_out, run(w))
    assert torch.equal(run(pw), packed_out) and len(pw.__dict__["_images"]) == 1


def test_packed_weight_cache_survives_recycled_memory():
    """Replacing the data tensor by a new one that lands on the freed tensor's address (same pointer,
    same version counter) must still rebuild the cached copy and image."""
    g = torch.Generator(device="cuda").manual_seed(9)
    c, k, s, d, q, n = 15, 15, 51, 8, 1000, 1
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    x = cv.round_bf16(torch.randn((n, c, q + d * (s - 1)), device="cuda", generator=g))
    w = torch.randn((k, c, s), device="cuda", generator=g) * 0.05
    pw = cv.pack_weights_forward(w)
    first = cv.conv1d_forward(x, pw, p)
    for scale in (2.0, 4.0, 8.0):
        pw.data = (scale * w).permute(2, 0, 1).contiguous()  # the previous tensor is freed here
        assert torch.equal(cv.conv1d_forward(x, pw, p), scale * first)
