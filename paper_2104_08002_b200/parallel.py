"""Data-parallel plumbing for the conv layer.

The batch shards exactly like the reference's `parallel_for_items` (proj/src/conv.cpp:15-31):
contiguous item ranges, rank r owning items [n*r/world, n*(r+1)/world). Forward and
backward-data need no communication; backward-weight produces a per-rank partial dW that one
all-reduce (NCCL on B200, gloo in the CPU tests) sums — the multi-GPU form of the reference's
ascending per-item reduction (conv.cpp:308-314).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) of items owned by `rank` (conv.cpp:24-25 partition)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n_items * rank // world, n_items * (rank + 1) // world


def allreduce_dw(dw: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-rank partial weight gradients in place (one collective per step)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(dw, op=dist.ReduceOp.SUM, group=group)
    return dw


def data_parallel_backward_weight(grad_out: torch.Tensor, inp: torch.Tensor, params, group=None,
                                  wgrad=None) -> torch.Tensor:
    """dW over the global batch from this rank's shard: local wgrad, then all-reduce.

    `grad_out`/`inp` hold only this rank's items. `wgrad(grad_out, inp, params)` computes the
    local partial (defaults to the B200 kernel through the C ABI)."""
    if wgrad is None:
        from .conv import conv1d_backward_weight as wgrad
    dw = wgrad(grad_out, inp, params)
    return allreduce_dw(dw, group)
