"""bench.py — B200 1D dilated conv layer benchmark (BASELINE.json metric).

One step = forward + backward-data + backward-weight of the BASELINE config-3 layer
(N=32, C=K=64, S=51, d=8, W_in=60400, BF16 storage, FP32 accumulation; the compute-bound
roofline case the north_star target is quoted on). Inputs (bf16 X 247 MB, dY 246 MB) are larger
than the 126 MB L2, so no flush is needed between steps.

  value   device-resident throughput (TFLOP/s, 3 x 2*N*K*C*S*Q per step), CUDA events, max over ranks
  e2e     the same metric through the C ABI (c1d_forward/backward_data/backward_weight, the call a
          reference host would make) with pinned HOST buffers: H2D of x and dy and D2H of y, dx
          and dW inside every timed step, pipelined over item chunks so both PCIe directions run
          under the passes (pipeline.HostLayerStep); the 987 MB fp32 download bounds it
  roofline  the dominant kernel's achieved TFLOP/s vs the measured B200 bf16 peak
  cpu_baseline  the unmodified reference CPU path (oracle/_ref, built from /root/reference) on a
          bounded sample of the same layer, timed on this host's cores

Multi-GPU (torchrun, one rank per GPU): every rank runs the full per-GPU batch (weak scaling)
and the dW of all ranks is summed with one NCCL all-reduce per step (the data-parallel exchange).

`--impl reference` runs only the reference CPU path (rank 0) and prints its line.

`--workload network` measures BASELINE config 5 instead: the residual 1D CNN training step
(input layer 1->15, 5 residual blocks x 3 convs C=K=15 S=51 d=8, two 1-tap heads, MSE+BCE loss,
SGD) at global batch 64 split across the ranks (64/N items per GPU, one NCCL all-reduce of the
173,162-float gradient bucket per step). value = conv FLOP/s of the whole job (3 passes per layer).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(n=32, c=64, k=64, s=51, d=8, q=60000)
METRIC = "1D dilated conv TFLOP/s (fwd/bwd-d/bwd-w) and % of B200 tensor peak"


def flops_per_pass(c=CFG) -> int:
    return 2 * c["n"] * c["k"] * c["c"] * c["s"] * c["q"]


def config_block(extra=None):
    cfg = {
        "workload": "BASELINE config 3: conv1d layer fwd+bwd_data+bwd_weight, N=32 C=K=64 S=51 d=8 "
                    "W_in=60400 (Q=60000), bf16 storage / fp32 accumulation",
        "n": CFG["n"], "c": CFG["c"], "k": CFG["k"], "s": CFG["s"], "d": CFG["d"],
        "w_in": CFG["q"] + CFG["d"] * (CFG["s"] - 1), "q": CFG["q"],
        "l2": "inputs larger than L2 (x 247 MB, dy 246 MB bf16), no flush",
        "flops_per_pass": flops_per_pass(),
    }
    if extra:
        cfg.update(extra)
    return cfg


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md recipe)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None
        self._thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None
            return

        def reader():
            for line in self._proc.stdout:
                self.samples.append([x.strip() for x in line.split(",")])

        self._thread = threading.Thread(target=reader, daemon=True)
        self._thread.start()

    def stop(self) -> dict:
        if self._proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self._proc.terminate()
        try:
            self._proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self._proc.kill()
        if self._thread:
            self._thread.join(timeout=2)
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for row in self.samples:
            try:
                sms.append(float(row[0]))
                maxes.append(float(row[1]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, row[3:7]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        sms.sort()
        return {"sm_mhz": sms[len(sms) // 2] if sms else None, "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms)}


# ----------------------------------------------------------------------------- reference arm
def run_reference_sample(items: int, threads: int, iterations: int = 1, warmup: int = 0):
    """Reference CPU path (measure_kernel semantics, proj/src/bench.cpp:172-234) on `items` items of
    the config-3 layer in BF16 mode (the reference's software BF16 path). Returns
    (seconds per pass list, flops per pass)."""
    import oracle

    ref = oracle.Ref()
    secs = []
    for pass_ in (0, 1, 2):
        t = ref.measure_kernel(items, CFG["c"], CFG["k"], CFG["s"], CFG["d"], CFG["q"], 1, pass_, iterations,
                               warmup, threads)
        if t < 0:
            raise RuntimeError(f"reference measure_kernel failed ({t})")
        secs.append(t)
    f = 2 * items * CFG["k"] * CFG["c"] * CFG["s"] * CFG["q"]
    return secs, f, ref.path


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ncores = os.cpu_count() or 1
    items = max(1, min(ncores, 32))  # reference threads fan out over items only (conv.cpp:15-31)
    threads = ncores
    step_times = []
    for _ in range(args.warmup):
        run_reference_sample(items, threads)
    for _ in range(args.steps):
        secs, f, path = run_reference_sample(items, threads)
        step_times.append(sum(secs))
    t = sum(step_times) / len(step_times)
    value = 3 * f / t / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (reference Rng(20260822) buffers)",
        "impl": "reference",
        "config": config_block({"sample": f"{items} of 32 items per step (bounded sample)",
                                "parallelism": f"reference std::thread fan-out, {min(items, threads)} effective"}),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": min(items, threads), "kind": "reference",
                         "sample": f"config-3 layer, {items} items, 3 passes, measure_kernel, BF16 mode",
                         "library": os.path.relpath(path, ROOT)},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def main_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2104_08002_b200 import _lib as L
    from paper_2104_08002_b200 import conv as cv

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    n, c, k, s, d, q = (CFG[x] for x in ("n", "c", "k", "s", "d", "q"))
    w_in = q + d * (s - 1)
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    g = torch.Generator(device=dev).manual_seed(20260822 + rank)
    x = torch.randn((n, c, w_in), device=dev, generator=g).to(torch.bfloat16)
    dy = torch.randn((n, k, q), device=dev, generator=g).to(torch.bfloat16)
    lim = (6.0 / (c * s)) ** 0.5  # Kaiming-uniform, fan_in = C*S
    w = (torch.rand((k, c, s), device=dev, generator=g) * 2 - 1) * lim
    y = torch.empty((n, k, q), device=dev)
    dx = torch.empty((n, c, w_in), device=dev)
    dw = torch.empty((k, c, s), device=dev)
    lib = L.lib()
    desc = cv.make_desc(p, n, w_in, L.DTYPE_BF16)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def chk(st):
        if st != 0:
            raise RuntimeError(f"c1d error {st}: {lib.c1d_last_error_message().decode()}")

    def step_device(mark=None):
        # mark: (pass name, event pair) bracketing that pass inside the timed region
        for name, fn in pass_fns.items():
            if mark is not None and mark[0] == name:
                mark[1].record(stream)
                fn()
                mark[2].record(stream)
            else:
                fn()
        if world > 1:
            dist.all_reduce(dw)

    # ---- per-pass kernel timing (roofline of the dominant kernel), events on our stream
    pass_fns = {
        "forward": lambda: chk(lib.c1d_forward(C.byref(desc), x.data_ptr(), w.data_ptr(), y.data_ptr(), None, 0, sp)),
        "backward_data": lambda: chk(lib.c1d_backward_data(C.byref(desc), dy.data_ptr(), w.data_ptr(), dx.data_ptr(),
                                                           None, 0, sp)),
        "backward_weight": lambda: chk(lib.c1d_backward_weight(C.byref(desc), x.data_ptr(), dy.data_ptr(),
                                                               dw.data_ptr(), None, 0, sp)),
    }
    for _ in range(max(args.warmup, 3)):
        step_device()
    torch.cuda.synchronize()
    per_pass = {}  # each pass timed alone (3 launches, median): burst-clock numbers
    for name, fn in pass_fns.items():
        evs = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in evs)[1]
        per_pass[name] = {"ms": ms, "tflops": flops_per_pass() / (ms * 1e-3) / 1e12,
                          "algo": cv.selected_algo(p, n, w_in, list(pass_fns).index(name))}

    # ---- timed region: K steps, device-resident inputs
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.c1d_launch_count()
    # the dominant pass (longest alone) is bracketed by events in every timed step: its average
    # duration inside the long run is the roofline's achieved rate (sustained-clock conditions)
    dom = max(per_pass, key=lambda kname: per_pass[kname]["ms"])
    marks = [(dom, torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        step_device(marks[i])
    e1.record(stream)
    torch.cuda.synchronize()
    launches = lib.c1d_launch_count() - launches0
    dom_ms = sum(m[1].elapsed_time(m[2]) for m in marks) / len(marks)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_total = e0.elapsed_time(e1)
    t_max = torch.tensor([ms_total], device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_step = t_max.item() / args.steps
    step_flops = 3 * flops_per_pass()
    value = world * step_flops / (ms_step * 1e-3) / 1e12

    # ---- e2e through the C ABI with host buffers (H2D inputs, D2H outputs every step), the
    # transfers pipelined against the passes over item chunks (paper_2104_08002_b200/pipeline.py)
    from paper_2104_08002_b200.pipeline import HostLayerStep

    pipe = HostLayerStep(p, n, w_in, chunks=args.e2e_chunks, device=dev, in_dtype=torch.bfloat16)
    hx = torch.empty(x.shape, dtype=torch.bfloat16, pin_memory=True)
    hdy = torch.empty(dy.shape, dtype=torch.bfloat16, pin_memory=True)
    hx.copy_(x)
    hdy.copy_(dy)
    hy = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
    hdx = torch.empty(dx.shape, dtype=torch.float32, pin_memory=True)
    hdw = torch.empty(dw.shape, dtype=torch.float32, pin_memory=True)
    h2d = pipe.h2d_bytes()
    d2h = pipe.d2h_bytes()
    e2e_steps = max(2, min(args.steps, 5))
    reduce_dw = (lambda t: dist.all_reduce(t)) if world > 1 else None  # the DP exchange, every step
    pipe.run(hx, hdy, w, hy, hdx, hdw, compute=stream, reduce_dw=reduce_dw)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(pipe.s_in)
    for _ in range(e2e_steps):
        pipe.run(hx, hdy, w, hy, hdx, hdw, compute=stream, reduce_dw=reduce_dw)
    f1.record(pipe.s_out)
    torch.cuda.synchronize()
    te = torch.tensor([f0.elapsed_time(f1) / e2e_steps], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * step_flops / (te.item() * 1e-3) / 1e12

    # ---- roofline of the dominant kernel (longest pass)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    # a kernel timed inside a long step: the sustained bf16 peak is the denominator
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0))
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    dom_tflops = flops_per_pass() / (dom_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(dom)
    except (OSError, ValueError):
        pass
    roofline = {"bound": "tensor", "kernel": dom, "achieved": dom_tflops, "peak": peak,
                "unit": "TFLOP/s", "frac": dom_tflops / peak, "traffic": traffic,
                "avg_launch_ms": dom_ms, "launches_timed": len(marks),
                "alone": {"achieved": per_pass[dom]["tflops"], "peak_burst": peak_burst,
                          "frac": per_pass[dom]["tflops"] / peak_burst},
                "peak_source": ("MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside the long timed "
                                "region); 'alone' = the same kernel timed alone vs the burst peak") if peaks
                else "fallback 1590 TFLOP/s (B200_PROFILING.md)"}

    # ---- CPU baseline (rank 0, N=1 only): reference on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            ncores = os.cpu_count() or 1
            items = max(1, min(ncores, 32))
            secs, f, path = run_reference_sample(items, ncores)
            cpu = {"value": 3 * f / sum(secs) / 1e12, "unit": "TFLOP/s", "cores": min(items, ncores),
                   "kind": "reference",
                   "sample": f"config-3 layer, {items} of 32 items, fwd+bwd_d+bwd_w once each (measure_kernel, "
                             f"BF16 mode), {sum(secs):.1f} s",
                   "library": os.path.relpath(path, ROOT)}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) x/dy, Kaiming-uniform w)",
            "config": config_block({"parallelism": f"dp{world}" + (" (NCCL all-reduce of dW)" if world > 1 else "")}),
            "passes": per_pass,
            "frac_of_peak_step": value / world / peak,  # vs the sustained peak
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": te.item(),
                    "path": f"c1d_* C ABI from pinned host buffers, {args.e2e_chunks} item chunks with H2D/D2H "
                            "overlapped with the passes (pipeline.HostLayerStep)"},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def network_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2104_08002_b200 import conv as cv
    from paper_2104_08002_b200.network import ResidualNet, train_step

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    global_batch, width = 64, 60000
    if global_batch % world:
        raise SystemExit("global batch 64 must divide by the GPU count")
    per = global_batch // world
    net = ResidualNet(blocks=5, convs_per_block=3, hidden=15, taps=51, dilation=8,
                      precision=cv.Precision.Bf16, seed=1, device=dev)
    pad = net.pad()
    g = torch.Generator(device=dev).manual_seed(20260822 + rank)
    x = torch.poisson(torch.full((per, 1, width + 2 * pad), 2.0, device=dev), generator=g)
    target = torch.poisson(torch.full((per, 1, width), 2.0, device=dev), generator=g)
    labels = (torch.rand((per, 1, width), device=dev, generator=g) < 0.1).float()
    stream = torch.cuda.current_stream(dev)
    from paper_2104_08002_b200 import _lib as L

    lib = L.lib()

    def step_eager():
        loss = train_step(net, x, target, labels)
        net.sgd_step(1e-3)
        return loss

    for _ in range(max(args.warmup, 3)):
        step_eager()
    torch.cuda.synchronize()
    step, launches_per_replay = step_eager, None
    if world == 1 and not args.no_graph:
        # One CUDA graph for the whole step (~120 launches): the C-ABI passes launch on the capture
        # stream, whose internal workspace is warmed first (no allocation under capture)
        gstream = torch.cuda.Stream(dev)
        gstream.wait_stream(stream)
        with torch.cuda.stream(gstream):
            for _ in range(2):
                step_eager()
        gstream.synchronize()
        graph = torch.cuda.CUDAGraph()
        lc0 = lib.c1d_launch_count()
        with torch.cuda.graph(graph, stream=gstream):
            loss_g = step_eager()
        launches_per_replay = lib.c1d_launch_count() - lc0

        def step():
            graph.replay()
            return loss_g

        for _ in range(2):
            step()
        torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = lib.c1d_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        loss = step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = lib.c1d_launch_count() - l0
    if launches_per_replay is not None:  # graph replays launch without the host counter
        launches = launches_per_replay * args.steps
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    flops_job = net.conv_flops(global_batch, width)
    value = flops_job / (ms * 1e-3) / 1e12
    # e2e: H2D of this rank's batch (pinned) + D2H of the loss each step
    hx, ht, hl = (torch.empty(a.shape, pin_memory=True) for a in (x, target, labels))
    hx.copy_(x)
    ht.copy_(target)
    hl.copy_(labels)
    hloss = torch.empty((), dtype=torch.float64, pin_memory=True)

    def step_e2e():
        x.copy_(hx, non_blocking=True)
        target.copy_(ht, non_blocking=True)
        labels.copy_(hl, non_blocking=True)
        hloss.copy_(step(), non_blocking=True)

    step_e2e()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_e2e = max(1, min(args.steps, 5))
    f0.record(stream)
    for _ in range(n_e2e):
        step_e2e()
    f1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([f0.elapsed_time(f1) / n_e2e], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    if rank == 0:
        line = {
            "metric": METRIC + " (config-5 network step)", "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic Poisson(2) inputs/targets, Bernoulli(0.1) labels, seeded init",
            "config": {"workload": "BASELINE config 5: residual 1D CNN training step (input 1->15, 5 blocks x 3 "
                                   "convs C=K=15 S=51 d=8 same-pad ReLU skip, 2 heads S=1), global batch 64, "
                                   "width 60000 (+200 pad/side), MSE+BCE, SGD",
                       "global_batch": global_batch, "per_gpu_batch": per, "width": width,
                       "parallelism": f"dp{world} (NCCL all-reduce of one 173,162-float gradient bucket)",
                       "flops_per_step": flops_job, "params": net.num_parameters()},
            "steps_per_s": 1e3 / ms, "loss": float(loss),
            "e2e": {"value": flops_job / (te.item() * 1e-3) / 1e12, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": (hx.numel() + ht.numel() + hl.numel()) * 4, "d2h_bytes_per_step": 8,
                    "ms_per_step": te.item()},
            "gpu_launches": int(launches), "clocks": clk,
            "cuda_graph": launches_per_replay is not None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="layer", choices=["layer", "network"])
    ap.add_argument("--e2e-chunks", type=int, default=8, help="item chunks of the pipelined host-buffer e2e step")
    ap.add_argument("--no-graph", action="store_true", help="network workload: launch eagerly (no CUDA graph)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    if args.workload == "network":
        return network_arm(args)
    return main_arm(args)


if __name__ == "__main__":
    sys.exit(main())
