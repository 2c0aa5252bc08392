"""The product's data-parallel network step on two ranks: `network.train_step` on
each rank's half of the batch, with the bucket all-reduce and division by the world size
(`parallel.allreduce_mean_`), equals the single-process full-batch step.

Two processes share the one visible GPU and talk over gloo (host-staged CUDA tensors): the
collective is a host-side exchange between two complete local steps, so no kernel of one rank
waits on the other rank's kernels. NCCL carries the same call on a multi-GPU box (bench.py).
FP32 network, so the bound is the reference's FP32 1e-5 (the two halves' sum is a different
summation order than the full batch)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WIDTH, N, BLOCKS, CPB, HIDDEN = 2048, 4, 2, 3, 15


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _batch(device):
    g = torch.Generator(device="cpu").manual_seed(3)
    pad = 200
    x = torch.zeros((N, 1, WIDTH + 2 * pad))
    x[:, :, pad:pad + WIDTH] = torch.poisson(torch.full((N, 1, WIDTH), 2.0), generator=g)
    target = torch.poisson(torch.full((N, 1, WIDTH), 2.0), generator=g)
    labels = (torch.rand((N, 1, WIDTH), generator=g) < 0.1).float()
    return x.to(device), target.to(device), labels.to(device)


def _net(device):
    from paper_2104_08002_b200 import conv as cv
    from paper_2104_08002_b200.network import ResidualNet

    return ResidualNet(blocks=BLOCKS, convs_per_block=CPB, hidden=HIDDEN, precision=cv.Precision.Fp32, seed=11,
                       device=device)


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2104_08002_b200.network import train_step
    from paper_2104_08002_b200.parallel import shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    net = _net(dev)
    x, t, l = _batch(dev)
    b, e = shard_range(N, rank, world)
    loss = train_step(net, x[b:e], t[b:e], l[b:e])
    torch.cuda.synchronize()
    out[rank] = (net.grad_bucket.cpu().numpy().copy(), float(loss))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_train_step_equals_full_batch():
    from paper_2104_08002_b200.network import forward_backward

    import oracle

    dev = torch.device("cuda", 0)
    net = _net(dev)
    x, t, l = _batch(dev)
    full_loss = float(forward_backward(net, x, t, l))
    full = net.grad_bucket.cpu().numpy().copy()
    world = 2
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    out = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(timeout=300)
        assert p_.exitcode == 0
    g0, l0 = out[0]
    g1, l1 = out[1]
    np.testing.assert_array_equal(g0, g1)  # every rank holds the identical reduced bucket
    err = oracle.norm_rel_error(g0, full)
    print(f"[dp 2 ranks] reduced gradient bucket vs full batch: norm_rel_error {err:.3e}; "
          f"mean local loss {(l0 + l1) / 2:.9g} vs full {full_loss:.9g}")
    assert err <= 1e-5
    assert abs((l0 + l1) / 2 - full_loss) <= 1e-6 * abs(full_loss)
