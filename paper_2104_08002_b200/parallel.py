"""Data-parallel plumbing; the product's only collective code.

The batch shards exactly like the reference's `parallel_for_items` (proj/src/conv.cpp:15-31):
contiguous item ranges, rank r owning items [n*r/world, n*(r+1)/world). Forward and
backward-data need no communication. Backward-weight produces a per-rank partial dW that one
all-reduce sums: the multi-GPU form of the reference's ascending per-item reduction
(conv.cpp:308-314). NCCL carries it on B200; the CPU tests run the same functions over gloo.

Callers:
* `bench.py` (layer workload, weak scaling): `allreduce_sum_(dW)` once per step.
* `network.train_step` (config 5, strong scaling): `allreduce_mean_(grad_bucket)` once per step
  over the flat bucket of every layer's dW and bias gradient; the losses are means over the local
  items (train.cpp:110,125), so the global gradient is the sum over ranks divided by the world size.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) of items owned by `rank` (conv.cpp:24-25 partition)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n_items * rank // world, n_items * (rank + 1) // world


def world_size(group=None) -> int:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group)
    return 1


def allreduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-rank partials in place (one collective); no-op on one process."""
    if world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def allreduce_mean_(t: torch.Tensor, group=None) -> torch.Tensor:
    """Sum over ranks, then divide by the world size, in place: the global-batch gradient from
    per-rank gradients of local-mean losses."""
    w = world_size(group)
    if w > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        t.div_(w)
    return t


def data_parallel_backward_weight(grad_out: torch.Tensor, inp: torch.Tensor, params, group=None,
                                  wgrad=None) -> torch.Tensor:
    """dW over the global batch from this rank's shard: local wgrad, then all-reduce.

    `grad_out`/`inp` hold only this rank's items. `wgrad(grad_out, inp, params)` computes the
    local partial (defaults to the B200 kernel through the C ABI)."""
    if wgrad is None:
        from .conv import conv1d_backward_weight as wgrad
    return allreduce_sum_(wgrad(grad_out, inp, params), group)
