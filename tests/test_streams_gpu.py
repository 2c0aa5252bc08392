"""Calls on different CUDA streams with the library's internal workspace (workspace = NULL) run
concurrently without sharing scratch memory: results equal the same calls made one after another
(c1d.h: the internal buffer is per (device, stream))."""
import pytest
import torch

import oracle
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


def test_graph_survives_workspace_growth():
    """A graph captured on a stream keeps the stream's internal workspace address; a later, larger
    call on that stream grows the workspace without freeing the old buffer, so replays stay
    correct (c1d.h: retired buffers live until c1d_release_workspace)."""
    rng = oracle.Rng(31)
    c = k = 16
    s, d = 51, 8
    small_q, big_q = 256, 4096
    x_s = torch.from_numpy(rng.fill_uniform((1, c, small_q + d * (s - 1)))).cuda()
    x_b = torch.from_numpy(rng.fill_uniform((4, c, big_q + d * (s - 1)))).cuda()
    w = torch.from_numpy(rng.fill_uniform((k, c, s))).cuda()
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        y_ref = cv.conv1d_forward(x_s, w, p)
        y = torch.empty_like(y_ref)
        cv.conv1d_forward(x_s, w, p, out=y)  # warm the stream's workspace at the small size
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        cv.conv1d_forward(x_s, w, p, out=y)
    with torch.cuda.stream(st):
        cv.conv1d_forward(x_b, w, p)  # grows the internal workspace of `st`
    st.synchronize()
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
    del g
    cv.release_workspace(st)


def test_out_argument_is_validated():
    c = k = 16
    s, d, q = 3, 8, 64
    x = torch.zeros((1, c, q + d * (s - 1)), device="cuda")
    w = torch.zeros((k, c, s), device="cuda")
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    for bad in (torch.empty((1, k, q - 1), device="cuda"), torch.empty((1, k, q), device="cuda", dtype=torch.bfloat16),
                torch.empty((1, k, 2 * q), device="cuda")[:, :, ::2]):
        with pytest.raises(cv.ShapeMismatch):
            cv.conv1d_forward(x, w, p, out=bad)
    with pytest.raises(cv.ShapeMismatch):
        cv.conv1d_backward_weight(torch.zeros((1, k, q), device="cuda"), x, p, out=torch.empty((k, c, s + 1),
                                                                                                device="cuda"))
