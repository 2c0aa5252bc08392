"""Calls on different CUDA streams with the library's internal workspace (workspace = NULL) run
concurrently without sharing scratch memory: results equal the same calls made one after another
(c1d.h: the internal buffer is per (device, stream))."""
import pytest
import torch

from paper_2104_08002_b200 import conv as cv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _problem(seed, c, k, s, d, q, n=3):
    g = torch.Generator(device="cuda").manual_seed(seed)
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    x = cv.round_bf16(torch.randn((n, c, q + d * (s - 1)), device="cuda", generator=g))
    dy = cv.round_bf16(torch.randn((n, k, q), device="cuda", generator=g))
    w = torch.randn((k, c, s), device="cuda", generator=g) * 0.05
    return p, x, dy, w


def _passes(p, x, dy, w):
    return (cv.conv1d_forward(x, w, p), cv.conv1d_backward_data(dy, w, p), cv.conv1d_backward_weight(dy, x, p))


def test_concurrent_streams_internal_workspace():
    # two shapes with different workspace needs (FP32-stored inputs force bf16 copies in scratch)
    probs = [_problem(1, 64, 64, 51, 8, 4000), _problem(2, 32, 48, 25, 2, 3000)]
    probs = [(p, x.float(), dy.float(), w) for p, x, dy, w in probs]
    want = [_passes(*pr) for pr in probs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    got = [None, None]
    for _ in range(3):
        for i, (st, pr) in enumerate(zip(streams, probs)):
            with torch.cuda.stream(st):
                got[i] = _passes(*pr)
        torch.cuda.synchronize()
        for g, wv in zip(got, want):
            for a, b in zip(g, wv):
                assert torch.equal(a, b)  # bitwise deterministic, no cross-stream scratch sharing
