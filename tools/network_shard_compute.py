"""Per-rank compute of the config-5 network step at the batch sizes N-way data parallelism gives each
rank (dev tool): global batch 64 -> 64/N items per rank, timed on ONE GPU without the gradient
all-reduce (which needs N GPUs). The ratio (t(64) / N) / t(64 / N) bounds the strong-scaling
efficiency the compute alone allows.

usage: python tools/network_shard_compute.py [steps]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_08002_b200 import conv as cv  # noqa: E402
from paper_2104_08002_b200.network import ResidualNet, forward_backward, sample_inputs  # noqa: E402


def per_rank_ms(per: int, steps: int) -> float:
    dev = torch.device("cuda", 0)
    net = ResidualNet(blocks=5, convs_per_block=3, hidden=15, taps=51, dilation=8, precision=cv.Precision.Bf16,
                      seed=1, device=dev)
    x, target, labels = sample_inputs(per, 60000, net.pad(), seed=20260822, device=dev)
    for _ in range(3):
        forward_backward(net, x, target, labels)
        net.sgd_step(1e-3)
    torch.cuda.synchronize()
    gstream = torch.cuda.Stream(dev)
    gstream.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(gstream):
        for _ in range(2):
            forward_backward(net, x, target, labels)
    gstream.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=gstream):
        forward_backward(net, x, target, labels)
    for _ in range(3):
        graph.replay()
        net.sgd_step(1e-3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        graph.replay()
        net.sgd_step(1e-3)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    res = {}
    for n in (1, 2, 4, 8):
        res[n] = per_rank_ms(64 // n, steps)
    t1 = res[1]
    out = {"what": "config-5 step per rank (graph replay + SGD, no all-reduce), one B200",
           "per_rank_ms": {f"{n} ranks ({64 // n} items)": round(t, 4) for n, t in res.items()},
           "compute_scaling_bound": {f"{n}": round((t1 / n) / t, 3) for n, t in res.items()}}
    print(json.dumps(out, indent=1))
