"""The training-step kernels around the conv layers (csrc/train.cu):

* c1d_fill_poisson / c1d_fill_bernoulli vs their C restatement in the oracle: bit-exact (integer
  counts and 0/1 labels), and independent of how a batch is split;
* c1d_mse_bce_loss vs the reference's own mse_loss / bce_with_logits (train.cpp:106-135, through
  oracle/_ref): the MSE gradient bit-exact, the BCE gradient within 1 float ulp (device exp/log1p
  vs the host's), the loss values to 1e-12 (summation order);
* c1d_sgd_update vs the reference's sgd_step: bit-exact;
* network.auroc (device) vs the reference's auroc (train.cpp:143-171), ties included."""
import numpy as np
import pytest
import torch

import oracle
from paper_2104_08002_b200 import network as nw

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("count,seed", [(1, 0), (1000003, 20260822), (64 * 60000, 7)])
def test_samplers_match_oracle_bit_exact(count, seed):
    p = nw.fill_poisson((count,), 2.0, seed, "cuda").cpu().numpy()
    b = nw.fill_bernoulli((count,), 0.1, seed + 1, "cuda").cpu().numpy()
    np.testing.assert_array_equal(p, oracle.sample_poisson(count, 2.0, seed))
    np.testing.assert_array_equal(b, oracle.sample_bernoulli(count, 0.1, seed + 1))
    if count > 100000:
        assert abs(p.mean() - 2.0) < 0.01 and abs(p.var() - 2.0) < 0.02
        assert abs(b.mean() - 0.1) < 0.002


def test_sample_inputs_shapes_and_padding():
    x, t, lab = nw.sample_inputs(3, 1000, 200, seed=5, device="cuda")
    assert x.shape == (3, 1, 1400) and t.shape == (3, 1, 1000) and lab.shape == (3, 1, 1000)
    assert not x[:, :, :200].any() and not x[:, :, 1200:].any()
    np.testing.assert_array_equal(x[:, :, 200:1200].reshape(-1).cpu().numpy(), oracle.sample_poisson(3000, 2.0, 15))


@pytest.mark.parametrize("n,width", [(1, 5), (4, 4096), (16, 60000)])
def test_mse_bce_matches_reference(n, width):
    g = torch.Generator(device="cuda").manual_seed(n + width)
    heads = torch.randn((n, 2, width), device="cuda", generator=g) * 3
    target = nw.fill_poisson((n, 1, width), 2.0, 3, "cuda")
    labels = nw.fill_bernoulli((n, 1, width), 0.1, 4, "cuda")
    grad = torch.empty((n, 2, width), device="cuda")
    bw = 0.7
    loss = nw.mse_bce(heads[:, 0:1], heads[:, 1:2], target, labels, bw, grad=grad).cpu().numpy()
    h = heads.cpu().numpy()
    mse, gm, bce, gb = oracle.ref_losses(oracle.Ref(), h[:, 0:1], target.cpu().numpy(), h[:, 1:2], labels.cpu().numpy())
    assert abs(loss[0] - mse) <= 1e-12 * abs(mse) and abs(loss[1] - bce) <= 1e-12 * abs(bce)
    bw32 = float(np.float32(bw))  # the C ABI's bce_weight is a float, as the reference's (train.cpp:336)
    assert abs(loss[2] - (mse + bw32 * bce)) <= 1e-12 * abs(mse + bw32 * bce)
    gr = grad.cpu().numpy()
    np.testing.assert_array_equal(gr[:, 0].reshape(-1), gm)
    want_b = (np.float32(bw) * gb).astype(np.float32)
    np.testing.assert_allclose(gr[:, 1].reshape(-1), want_b, rtol=2e-7, atol=0)
    # deterministic: a second call gives the identical bits
    loss2 = nw.mse_bce(heads[:, 0:1], heads[:, 1:2], target, labels, bw).cpu().numpy()
    np.testing.assert_array_equal(loss, loss2)


def test_sgd_update_matches_reference_bit_exact():
    g = torch.Generator(device="cuda").manual_seed(9)
    ref = oracle.Ref()
    ref.lib.ref_sgd_step.argtypes = [oracle._f32p, oracle._f32p, oracle.I64, oracle.C.c_float]
    for count in (1, 3, 173162, 1000001):
        p = torch.randn(count, device="cuda", generator=g)
        gr = torch.randn(count, device="cuda", generator=g)
        want = p.cpu().numpy().copy()
        ref.lib.ref_sgd_step(want, gr.cpu().numpy(), count, 0.05)
        nw.sgd_update_(p, gr, 0.05)
        np.testing.assert_array_equal(p.cpu().numpy(), want)
    with pytest.raises(Exception):
        nw.sgd_update_(p, gr, 0.0)  # train.cpp:139: lr must be positive


@pytest.mark.parametrize("case", ["random", "ties", "one_class"])
def test_auroc_matches_reference(case):
    rng = np.random.default_rng(3)
    n = 20000
    if case == "ties":
        scores = rng.integers(0, 7, n).astype(np.float32)
    else:
        scores = rng.standard_normal(n).astype(np.float32)
    labels = (rng.random(n) < (0.0 if case == "one_class" else 0.1)).astype(np.float32)
    got = nw.auroc(torch.from_numpy(scores).cuda(), torch.from_numpy(labels).cuda())
    want = oracle.ref_auroc(oracle.Ref(), scores, labels)
    if case == "one_class":
        assert np.isnan(got) and np.isnan(want)
    else:
        assert abs(got - want) <= 1e-12, (got, want)
