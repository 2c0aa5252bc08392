"""Multi-process (gloo, world_size 2) checks of the data-parallel path on CPU: batch sharding as
in the reference's parallel_for_items (conv.cpp:15-31) and the dW all-reduce reproduce the
single-process full-batch gradient. Local partials come from the oracle (no GPU here)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_08002_b200.parallel import allreduce_mean_, allreduce_sum_, data_parallel_backward_weight, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_matches_reference_partition():
    for n in (1, 2, 5, 16, 64):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and a <= b
            # conv.cpp:24-25: begin = count*t/workers
            assert all(r == (n * i // world, n * (i + 1) // world) for i, r in enumerate(ranges))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _worker(rank, world, port, x, dy, s, d, out):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = shard_range(x.shape[0], rank, world)

    def oracle_wgrad(g, xx, p):
        return torch.from_numpy(oracle.naive_backward_weight(g.numpy(), xx.numpy(), s, d))

    dw = data_parallel_backward_weight(torch.from_numpy(dy[b:e]), torch.from_numpy(x[b:e]), None,
                                       wgrad=oracle_wgrad)
    out[rank] = dw.numpy().copy()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_data_parallel_wgrad_equals_full_batch(world):
    import oracle

    rng = oracle.Rng(77)
    n, c, k, s, d, q = 5, 4, 3, 5, 8, 96
    x = rng.fill_uniform((n, c, q + d * (s - 1)))
    dy = rng.fill_uniform((n, k, q))
    full = oracle.naive_backward_weight(dy, x, s, d)
    manager = mp.Manager()
    out = manager.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, dy, s, d, out)) for r in range(world)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    for r in range(world):
        # the all-reduced partial sums equal the full-batch gradient (fp32 sum of 2 partials)
        assert oracle.norm_rel_error(out[r], full) <= 1e-6
    np.testing.assert_array_equal(out[0], out[1])  # every rank holds the identical dW


def _bucket_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(100 + rank)
    local = torch.randn(173162, generator=g)  # the config-5 bucket length
    mean = allreduce_mean_(local.clone())
    summed = allreduce_sum_(local.clone())
    out[rank] = (local.numpy().copy(), mean.numpy().copy(), summed.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_bucket_mean_and_sum():
    """network.train_step's exchange (parallel.allreduce_mean_: sum over ranks / world) and the
    layer bench's dW exchange (allreduce_sum_) on two gloo ranks."""
    world = 2
    manager = mp.Manager()
    out = manager.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_bucket_worker, args=(r, world, port, out)) for r in range(world)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    l0, l1 = out[0][0], out[1][0]
    for r in range(world):
        np.testing.assert_allclose(out[r][2], l0 + l1, rtol=0, atol=1e-6)
        np.testing.assert_allclose(out[r][1], (l0 + l1) / 2, rtol=0, atol=1e-6)
    np.testing.assert_array_equal(out[0][1], out[1][1])


def test_single_process_collectives_are_noops():
    t = torch.arange(5.0)
    assert torch.equal(allreduce_mean_(t.clone()), t)
    assert torch.equal(allreduce_sum_(t.clone()), t)
