"""bench.py — B200 1D dilated conv layer benchmark (BASELINE.json metric).

One step = forward + backward-data + backward-weight of the BASELINE config-3 layer
(N=32, C=K=64, S=51, d=8, W_in=60400, BF16 storage, FP32 accumulation; the compute-bound
roofline case the north_star target is quoted on). Inputs (bf16 X 247 MB, dY 246 MB) are larger
than the 126 MB L2, so no flush is needed between steps.

  value     device-resident throughput (TFLOP/s, 3 x 2*N*K*C*S*Q per step), CUDA events, max over ranks
  parity    the last timed step's y and dx on items {0, N-1} and dW on 256 sampled entries against a
            float64 recomputation on the device (norm-relative on BF16-rounded operands; 1e-5, and
            1e-4 for the default-mode bwd-w, whose 1.92M-product sums drift ~6e-5 in the tensor core's
            FP32 accumulation); `backward_weight_exact` times the C1D_FLAG_EXACT_ACCUM bwd-w (1e-5)
  e2e       the same metric through the C ABI (c1d_forward/backward_data/backward_weight, the call a
            reference host would make) with pinned HOST buffers: H2D of x and dy and D2H of y, dx
            and dW inside every timed step, pipelined over item chunks (pipeline.HostLayerStep)
  roofline  the dominant kernel's achieved TFLOP/s vs the measured B200 bf16 peak: the burst peak,
            unless the timed region lasted >= 1 s AND the clock sampler saw sw_power_cap (then the
            sustained peak); `peak_kind` says which
  roofline_narrow  config 2 (N=16, C=K=15, BF16), each pass timed alone over rotating buffers (> L2):
            achieved HBM GB/s of the algorithmic bytes and the fraction of max(HBM, tensor) time
  network   BASELINE config 5 (residual 1D CNN training step, global batch 64 split over the ranks:
            strong scaling), the north_star's multi-GPU figure
  cpu_baseline  the unmodified reference CPU path (oracle/_ref, built from /root/reference) on the
            whole config-3 layer (32 items), timed on this host's cores

Multi-GPU: `--gpus N` (N > 1) starts N ranks itself through torch.distributed.run unless it is
already running under torchrun. Every rank runs the full per-GPU layer batch (weak scaling) and
the dW of all ranks is summed with one NCCL all-reduce per step (parallel.allreduce_sum_); the
network step shards its global batch of 64 (parallel.allreduce_mean_ of the gradient bucket).

`--impl reference` runs only the reference CPU path (rank 0) and prints its line.
`--workload network` prints the config-5 network line as the headline instead.
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
CFG2 = dict(n=16, c=15, k=15, s=51, d=8, q=60000)
METRIC = "1D dilated conv TFLOP/s (fwd/bwd-d/bwd-w) and % of B200 tensor peak"
PASSES = ("forward", "backward_data", "backward_weight")


def flops_per_pass(c=CFG) -> int:
    return 2 * c["n"] * c["k"] * c["c"] * c["s"] * c["q"]


def w_in_of(c=CFG) -> int:
    return c["q"] + c["d"] * (c["s"] - 1)


def config_block(extra=None):
    cfg = {
        "workload": "BASELINE config 3: conv1d layer fwd+bwd_data+bwd_weight, N=32 C=K=64 S=51 d=8 "
                    "W_in=60400 (Q=60000), bf16 storage / fp32 accumulation",
        "n": CFG["n"], "c": CFG["c"], "k": CFG["k"], "s": CFG["s"], "d": CFG["d"],
        "w_in": w_in_of(), "q": CFG["q"],
        "l2": "inputs larger than L2 (x 247 MB, dy 246 MB bf16), no flush",
        "flops_per_pass": flops_per_pass(),
    }
    if extra:
        cfg.update(extra)
    return cfg


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def load_traffic() -> dict:
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md recipe)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
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


# ----------------------------------------------------------------------------- reference (CPU) path
REF_MODE = ("FP32 mode on the whole layer: the reference computes BF16 precision as its FP32 path on BF16-rounded "
            "operands (test_conv.cpp:274-295; identical results) and its FP32 path is the faster of the two "
            "(SURVEY §0: 6.27 vs 8.70 s per pass), so this is the reference's best time for this computation")


def run_reference_sample(items: int, threads: int, iterations: int = 1, warmup: int = 0):
    """Reference CPU path (measure_kernel semantics, proj/src/bench.cpp:172-234) on `items` items of
    the config-3 layer. Returns (seconds per pass list, flops per pass, library path)."""
    import oracle

    ref = oracle.Ref()
    secs = []
    for pass_ in (0, 1, 2):
        t = ref.measure_kernel(items, CFG["c"], CFG["k"], CFG["s"], CFG["d"], CFG["q"], 0, pass_, iterations,
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
    items = CFG["n"]  # the whole layer: same config as our arm
    step_times = []
    for _ in range(min(args.warmup, 1)):  # the CPU path needs no more than one warm-up pass
        run_reference_sample(items, ncores)
    path = None
    for _ in range(args.steps):
        secs, f, path = run_reference_sample(items, ncores)
        step_times.append(sum(secs))
    t = sum(step_times) / len(step_times)
    value = 3 * f / t / 1e12
    cores = min(items, ncores)  # the reference fans out over items only (conv.cpp:15-31)
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": min(args.warmup, 1), "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (bf16-representable operands)",
        "data": "synthetic (reference Rng(20260822) buffers)", "impl": "reference",
        "config": config_block({"sample": "all 32 items per step (the whole layer)",
                                "parallelism": f"reference std::thread fan-out over items, {cores} threads"}),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "reference",
                         "sample": f"config-3 layer, all {items} items, 3 passes per step, measure_kernel; {REF_MODE}",
                         "library": os.path.relpath(path, ROOT) if path else None},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_line():
    ncores = os.cpu_count() or 1
    items = CFG["n"]
    try:
        secs, f, path = run_reference_sample(items, ncores)
        return {"value": 3 * f / sum(secs) / 1e12, "unit": "TFLOP/s", "cores": min(items, ncores), "kind": "reference",
                "sample": f"config-3 layer, all {items} items, fwd+bwd_d+bwd_w once each (measure_kernel), "
                          f"{sum(secs):.1f} s; {REF_MODE}",
                "library": os.path.relpath(path, ROOT)}
    except Exception as exc:  # noqa: BLE001
        return {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference", "sample": f"failed: {exc}"}


# ----------------------------------------------------------------------------- helpers (device)
def dist_setup():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    return world, rank, local, dev


def max_over_ranks(v: float, dev, world: int) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def barrier(world: int):
    import torch.distributed as dist

    if world > 1:
        dist.barrier()


def parity_check(x, w, dy, y, dx, dw, d: int):
    """The last step's outputs vs a float64 recomputation on the device: y and dx on items {0, N-1}
    (torch fp64 conv1d / conv_transpose1d on the BF16-rounded operands), dW on 256 sampled
    (k, c, s) entries (fp64 dot products over the whole batch). Checker only: nothing here feeds
    the timed path."""
    import torch
    import torch.nn.functional as F

    n, k, q = dy.shape
    c, s = w.shape[1], w.shape[2]
    w64 = w.to(torch.bfloat16).double()  # the kernels round w with RNE, as torch does
    items = [0, n - 1]

    def rel(a, b):
        return float((a.double() - b).norm() / b.norm())

    y_ref = F.conv1d(x[items].double(), w64, dilation=d)
    dx_ref = F.conv_transpose1d(dy[items].double(), w64, dilation=d)
    g = torch.Generator(device="cpu").manual_seed(5)
    idx = torch.stack([torch.randint(0, k, (256,), generator=g), torch.randint(0, c, (256,), generator=g),
                       torch.randint(0, s, (256,), generator=g)], 1).tolist()
    got, want = [], []
    for kk, cc, ss in idx:
        want.append(torch.dot(x[:, cc, ss * d:ss * d + q].double().reshape(-1), dy[:, kk, :].double().reshape(-1)))
        got.append(dw[kk, cc, ss])
    want_t, got_t = torch.stack(want), torch.stack(got)
    out = {"forward": rel(y[items], y_ref), "backward_data": rel(dx[items], dx_ref),
           "backward_weight": rel(got_t, want_t),
           # bwd-w sums 1.92M products per entry; the default accumulation mode (one tensor-core
           # chain per CTA) drifts ~6e-5, inside the reference's BF16 bound (1e-2, acceptance.cpp:526)
           "tol": {"forward": 1e-5, "backward_data": 1e-5, "backward_weight": 1e-4},
           "how": "items {0, N-1} of y and dx, 256 sampled dW entries, vs float64 on the BF16-rounded operands"}
    out["ok"] = all(out[p] <= out["tol"][p] for p in PASSES)
    return out


def exact_wgrad(lib, desc_exact, x, dy, w, d, stream):
    """Backward-weight in the exact-accumulation mode (C1D_FLAG_EXACT_ACCUM: chains capped at ~4096
    products): its time alone and its parity on the same 256 sampled entries (bound 1e-5)."""
    import torch

    k, c, s = w.shape
    q = dy.shape[2]
    dw = torch.empty((k, c, s), device=x.device)
    sp = stream.cuda_stream

    def run():
        st = lib.c1d_backward_weight(C.byref(desc_exact), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), None, 0, sp)
        if st != 0:
            raise RuntimeError(lib.c1d_last_error_message().decode())

    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[1]
    g = torch.Generator(device="cpu").manual_seed(5)
    idx = torch.stack([torch.randint(0, k, (256,), generator=g), torch.randint(0, c, (256,), generator=g),
                       torch.randint(0, s, (256,), generator=g)], 1).tolist()
    want = torch.stack([torch.dot(x[:, cc, ss * d:ss * d + q].double().reshape(-1), dy[:, kk, :].double().reshape(-1))
                        for kk, cc, ss in idx])
    got = torch.stack([dw[kk, cc, ss] for kk, cc, ss in idx]).double()
    err = float((got - want).norm() / want.norm())
    return {"ms": ms, "tflops": flops_per_pass() / (ms * 1e-3) / 1e12, "parity_backward_weight": err, "tol": 1e-5,
            "ok": err <= 1e-5, "flag": "C1D_FLAG_EXACT_ACCUM"}


def narrow_roofline(lib, dev, stream, peaks, traffic):
    """Config 2 (N=16, C=K=15, BF16): each pass timed alone, 20 launches over 4 rotating buffer sets
    (4 x 174 MB > L2). Achieved HBM GB/s of the algorithmic bytes and the fraction
    of max(bytes / HBM peak, FLOPs / tensor burst peak)."""
    import torch

    from paper_2104_08002_b200 import _lib as L
    from paper_2104_08002_b200 import conv as cv

    n, c, k, s, d, q = (CFG2[x] for x in ("n", "c", "k", "s", "d", "q"))
    w_in = w_in_of(CFG2)
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16)
    desc = cv.make_desc(p, n, w_in, L.DTYPE_BF16)
    g = torch.Generator(device=dev).manual_seed(2)
    sets = []
    for _ in range(4):
        sets.append(dict(x=torch.randn((n, c, w_in), device=dev, generator=g).to(torch.bfloat16),
                         dy=torch.randn((n, k, q), device=dev, generator=g).to(torch.bfloat16),
                         y=torch.empty((n, k, q), device=dev), dx=torch.empty((n, c, w_in), device=dev),
                         dw=torch.empty((k, c, s), device=dev)))
    w = (torch.rand((k, c, s), device=dev, generator=g) * 2 - 1) * (6.0 / (c * s)) ** 0.5
    sp = stream.cuda_stream
    # weight images packed before the clock, as the reference's measure_kernel packs (bench.cpp:184-203)
    wd, wp, images = {}, {}, []
    for name, pi in (("forward", L.PASS_FORWARD), ("backward_data", L.PASS_BACKWARD_DATA)):
        wd[name], wp[name] = cv.make_desc(p, n, w_in, L.DTYPE_BF16), w.data_ptr()
        nbytes = C.c_size_t(0)
        if lib.c1d_packed_weights_size(C.byref(wd[name]), pi, C.byref(nbytes)) == 0 and nbytes.value:
            img = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
            if lib.c1d_pack_weights(1, C.byref(wd[name]), (C.c_int32 * 1)(pi), (C.c_void_p * 1)(w.data_ptr()),
                                    (C.c_void_p * 1)(img.data_ptr()), sp) != 0:
                raise RuntimeError(lib.c1d_last_error_message().decode())
            wd[name].flags |= L.FLAG_PREPACKED_WEIGHTS
            wp[name] = img.data_ptr()
            images.append(img)

    def call(name, b):
        if name == "forward":
            st = lib.c1d_forward(C.byref(wd[name]), b["x"].data_ptr(), wp[name], b["y"].data_ptr(), None, 0, sp)
        elif name == "backward_data":
            st = lib.c1d_backward_data(C.byref(wd[name]), b["dy"].data_ptr(), wp[name], b["dx"].data_ptr(), None, 0, sp)
        else:
            st = lib.c1d_backward_weight(C.byref(desc), b["x"].data_ptr(), b["dy"].data_ptr(), b["dw"].data_ptr(),
                                         None, 0, sp)
        if st != 0:
            raise RuntimeError(lib.c1d_last_error_message().decode())

    flops = flops_per_pass(CFG2)
    algo_bytes = {
        "forward": n * c * w_in * 2 + k * c * s * 4 + n * k * q * 4,
        "backward_data": n * k * q * 2 + k * c * s * 4 + n * c * w_in * 4,
        "backward_weight": n * c * w_in * 2 + n * k * q * 2 + k * c * s * 4,
    }
    hbm = peaks.get("hbm_gbs", 6441.3)
    tensor = peaks.get("bf16_tflops", 1689.5)
    out = {}
    for name in PASSES:
        for i in range(4):
            call(name, sets[i])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record(stream)
        for i in range(reps):
            call(name, sets[i % 4])
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps * 1e-3
        b = algo_bytes[name]
        t_hbm, t_tc = b / (hbm * 1e9), flops / (tensor * 1e12)
        out[name] = {"us": t * 1e6, "tflops": flops / t / 1e12, "algo_bytes": b, "hbm_gbs": b / t / 1e9,
                     "bound": "hbm" if t_hbm >= t_tc else "tensor", "bound_us": max(t_hbm, t_tc) * 1e6,
                     "frac": max(t_hbm, t_tc) / t, "traffic": traffic.get(f"cfg2_{name}")}
    out["peaks"] = {"hbm_gbs": hbm, "bf16_tflops": tensor, "source": "MEASURED_PEAKS.json (burst)"}
    out["config"] = "BASELINE config 2: N=16 C=K=15 S=51 d=8 W_in=60400, bf16 storage; 4 rotating buffer sets > L2"
    out["weights"] = ("prepacked images (c1d_pack_weights before the clock, like the reference's measure_kernel)"
                      if images else "KCS, packed inside every call")
    return out


# ----------------------------------------------------------------------------- config-5 network step
def measure_network(world, rank, local, dev, steps, warmup, use_graph=True):
    """Config 5 at `world` ranks: global batch 64, 64/world items per rank (strong scaling). One
    step = forward + loss + backward (one CUDA graph), the gradient-bucket all-reduce
    (parallel.allreduce_mean_, NCCL) and the SGD update over the flat parameter bucket."""
    import torch

    from paper_2104_08002_b200 import _lib as L
    from paper_2104_08002_b200 import conv as cv
    from paper_2104_08002_b200 import parallel
    from paper_2104_08002_b200.network import ResidualNet, forward_backward, sample_inputs

    global_batch, width = 64, 60000
    if global_batch % world:
        raise SystemExit("global batch 64 must divide by the GPU count")
    per = global_batch // world
    net = ResidualNet(blocks=5, convs_per_block=3, hidden=15, taps=51, dilation=8,
                      precision=cv.Precision.Bf16, seed=1, device=dev)
    pad = net.pad()
    x, target, labels = sample_inputs(per, width, pad, seed=20260822 + rank, device=dev)
    lib = L.lib()
    stream = torch.cuda.current_stream(dev)
    lr = 1e-3

    def local_eager():
        return forward_backward(net, x, target, labels)

    for _ in range(max(warmup, 3)):
        local_eager()
        parallel.allreduce_mean_(net.grad_bucket)
        net.sgd_step(lr)
    torch.cuda.synchronize()
    local_step, launches_per_local = local_eager, None
    if use_graph:
        # the local step (~120 launches) as one CUDA graph; the C-ABI passes launch on the capture
        # stream, whose internal workspace is warmed first
        gstream = torch.cuda.Stream(dev)
        gstream.wait_stream(stream)
        with torch.cuda.stream(gstream):
            for _ in range(2):
                local_eager()
        gstream.synchronize()
        graph = torch.cuda.CUDAGraph()
        lc0 = lib.c1d_launch_count()
        with torch.cuda.graph(graph, stream=gstream):
            loss_g = local_eager()
        launches_per_local = lib.c1d_launch_count() - lc0

        def local_step():
            graph.replay()
            return loss_g

    def step():
        loss = local_step()
        parallel.allreduce_mean_(net.grad_bucket)
        net.sgd_step(lr)
        return loss

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(world)
    torch.cuda.synchronize()
    l0 = lib.c1d_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        loss = step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = lib.c1d_launch_count() - l0
    loss_timed = float(loss)  # the graph's loss buffer is overwritten by the e2e replays below
    if launches_per_local is not None:  # graph replays launch without the host counter
        launches = launches_per_local * steps
    barrier(world)
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, dev, world)
    flops_job = net.conv_flops(global_batch, width)
    # e2e: H2D of this rank's batch (pinned) + D2H of the loss, every step. The batch of step i+2
    # crosses PCIe on a copy stream into one of two device staging sets while steps i and i+1
    # compute (a training input pipeline); step i copies its staged batch into the graph's input
    # buffers (device to device, ~15 us) before its replay.
    hx, ht, hl = (torch.empty(a.shape, pin_memory=True) for a in (x, target, labels))
    hx.copy_(x)
    ht.copy_(target)
    hl.copy_(labels)
    hloss = torch.empty((), dtype=torch.float64, pin_memory=True)
    cstream = torch.cuda.Stream(dev)
    staged = [tuple(torch.empty_like(a) for a in (x, target, labels)) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]

    def h2d(slot):
        cstream.wait_event(ev_free[slot])  # the step that used this staging set has copied it out
        with torch.cuda.stream(cstream):
            for dst, src in zip(staged[slot], (hx, ht, hl)):
                dst.copy_(src, non_blocking=True)
        ev_in[slot].record(cstream)

    def step_e2e(i):
        slot = i % 2
        stream.wait_event(ev_in[slot])
        for dst, src in zip((x, target, labels), staged[slot]):
            dst.copy_(src, non_blocking=True)
        ev_free[slot].record(stream)
        h2d(slot)  # the batch of step i + 2
        hloss.copy_(step(), non_blocking=True)

    h2d(0)
    h2d(1)
    step_e2e(0)
    step_e2e(1)
    torch.cuda.synchronize()
    barrier(world)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_e2e = max(2, min(steps, 10))
    f0.record(stream)
    for i in range(n_e2e):
        step_e2e(i)
    f1.record(stream)
    torch.cuda.synchronize()
    te = max_over_ranks(f0.elapsed_time(f1) / n_e2e, dev, world)
    return {
        "metric": METRIC + " (config-5 network step)", "value": flops_job / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
        "n_gpus": world, "steps": steps, "ms_per_step": ms, "steps_per_s": 1e3 / ms, "scaling": "strong",
        "dtype": "bf16", "data": "synthetic Poisson(2) inputs/targets, Bernoulli(0.1) labels (device samplers), "
                                 "seeded init",
        "config": {"workload": "BASELINE config 5: residual 1D CNN training step (input 1->15, 5 blocks x 3 convs "
                               "C=K=15 S=51 d=8 same-pad ReLU skip, 2 heads S=1), global batch 64, width 60000 "
                               "(+200 pad/side), MSE+BCE, SGD",
                   "global_batch": global_batch, "per_gpu_batch": per, "width": width,
                   "parallelism": f"dp{world} (one all-reduce of the 173,162-float gradient bucket per step)",
                   "flops_per_step": flops_job, "params": net.num_parameters()},
        "loss": loss_timed,
        "e2e": {"value": flops_job / (te * 1e-3) / 1e12, "unit": "TFLOP/s",
                "h2d_bytes_per_step": (hx.numel() + ht.numel() + hl.numel()) * 4, "d2h_bytes_per_step": 8,
                "ms_per_step": te,
                "path": "pinned host batch -> device every step on a copy stream (two staging sets, two steps "
                        "ahead), device-to-device into the graph's inputs, graph replay, loss to the host"},
        "gpu_launches": int(launches), "clocks": clk, "cuda_graph": launches_per_local is not None,
    }


# ----------------------------------------------------------------------------- our arm (layer)
def main_arm(args):
    import torch

    from paper_2104_08002_b200 import _lib as L
    from paper_2104_08002_b200 import conv as cv
    from paper_2104_08002_b200 import parallel

    world, rank, local, dev = dist_setup()
    n, c, k, s, d, q = (CFG[x] for x in ("n", "c", "k", "s", "d", "q"))
    w_in = w_in_of()
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

    pass_fns = {
        "forward": lambda: chk(lib.c1d_forward(C.byref(desc), x.data_ptr(), w.data_ptr(), y.data_ptr(), None, 0, sp)),
        "backward_data": lambda: chk(lib.c1d_backward_data(C.byref(desc), dy.data_ptr(), w.data_ptr(), dx.data_ptr(),
                                                           None, 0, sp)),
        "backward_weight": lambda: chk(lib.c1d_backward_weight(C.byref(desc), x.data_ptr(), dy.data_ptr(),
                                                               dw.data_ptr(), None, 0, sp)),
    }

    def step_device(mark=None):
        # mark: (pass name, event pair) bracketing that pass inside the timed region
        for name, fn in pass_fns.items():
            if mark is not None and mark[0] == name:
                mark[1].record(stream)
                fn()
                mark[2].record(stream)
            else:
                fn()
        parallel.allreduce_sum_(dw)

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
    barrier(world)
    torch.cuda.synchronize()
    launches0 = lib.c1d_launch_count()
    # the dominant pass (longest alone) is bracketed by events in every timed step: its average
    # duration inside the timed region is the roofline's achieved rate
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
    barrier(world)
    clk = clocks.stop()
    ms_total = max_over_ranks(e0.elapsed_time(e1), dev, world)
    ms_step = ms_total / args.steps
    step_flops = 3 * flops_per_pass()
    value = world * step_flops / (ms_step * 1e-3) / 1e12

    # ---- parity of the last timed step (rank 0's outputs; dW is the all-reduced sum when world > 1)
    parity = exact = None
    if world == 1 and not args.no_parity:
        parity = parity_check(x, w, dy, y, dx, dw, d)
        exact = exact_wgrad(lib, cv.make_desc(p, n, w_in, L.DTYPE_BF16, exact=True), x, dy, w, d, stream)

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
    reduce_dw = parallel.allreduce_sum_ if world > 1 else None  # the DP exchange, every step
    pipe.run(hx, hdy, w, hy, hdx, hdw, compute=stream, reduce_dw=reduce_dw)
    torch.cuda.synchronize()
    barrier(world)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(pipe.s_in)
    for _ in range(e2e_steps):
        pipe.run(hx, hdy, w, hy, hdx, hdw, compute=stream, reduce_dw=reduce_dw)
    f1.record(pipe.s_out)
    torch.cuda.synchronize()
    te = max_over_ranks(f0.elapsed_time(f1) / e2e_steps, dev, world)
    e2e_value = world * step_flops / (te * 1e-3) / 1e12
    del pipe, hx, hdy, hy, hdx, hdw

    # ---- roofline of the dominant kernel (longest pass)
    peaks = load_peaks()
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    peak_sust = peaks.get("bf16_tflops_sustained", peak_burst)
    long_capped = ms_total >= 1000.0 and "sw_power_cap" in (clk.get("reasons") or [])
    peak, peak_kind = (peak_sust, "sustained") if long_capped else (peak_burst, "burst")
    dom_tflops = flops_per_pass() / (dom_ms * 1e-3) / 1e12
    traffic = load_traffic()
    roofline = {"bound": "tensor", "kernel": dom, "achieved": dom_tflops, "peak": peak,
                "unit": "TFLOP/s", "frac": dom_tflops / peak, "traffic": traffic.get(dom),
                "avg_launch_ms": dom_ms, "launches_timed": len(marks), "peak_kind": peak_kind,
                "alone": {"achieved": per_pass[dom]["tflops"], "peak_burst": peak_burst,
                          "frac": per_pass[dom]["tflops"] / peak_burst},
                "peak_source": ("MEASURED_PEAKS.json bf16_tflops (burst): the timed region was "
                                f"{ms_total / 1e3:.2f} s" + (" with sw_power_cap, so bf16_tflops_sustained"
                                                             if long_capped else ""))
                if peaks else "fallback 1590 TFLOP/s (B200_PROFILING.md)"}

    narrow = None
    if not args.no_narrow:
        narrow = narrow_roofline(lib, dev, stream, peaks, traffic)

    network = None
    if not args.no_network:
        network = measure_network(world, rank, local, dev, args.network_steps, args.warmup, use_graph=not args.no_graph)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) x/dy, Kaiming-uniform w)",
            "config": config_block({"parallelism": f"dp{world}" + (" (NCCL all-reduce of dW)" if world > 1 else "")}),
            "passes": per_pass,
            "frac_of_peak_step": value / world / peak,
            "roofline": roofline,
            "roofline_narrow": narrow,
            "parity": parity,
            "backward_weight_exact": exact,
            "network": network,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": te,
                    "path": f"c1d_* C ABI from pinned host buffers, {args.e2e_chunks} item chunks with H2D/D2H "
                            "overlapped with the passes (pipeline.HostLayerStep)"},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def network_arm(args):
    world, rank, local, dev = dist_setup()
    line = measure_network(world, rank, local, dev, args.steps, args.warmup, use_graph=not args.no_graph)
    if rank == 0:
        line.update({"warmup": args.warmup, "higher_is_better": True, "vs_baseline": None})
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def spawn_ranks(n: int) -> int:
    """--gpus N outside torchrun: start N ranks (one per GPU) with torch.distributed.run."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)  # the reference measure_kernel's 20 iterations (bench.hpp:31)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-narrow", action="store_true")
    ap.add_argument("--no-network", action="store_true")
    ap.add_argument("--network-steps", type=int, default=20)
    ap.add_argument("--workload", default="layer", choices=["layer", "network"])
    ap.add_argument("--e2e-chunks", type=int, default=8, help="item chunks of the pipelined host-buffer e2e step")
    ap.add_argument("--no-graph", action="store_true", help="network: launch the local step eagerly (no CUDA graph)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.workload == "network":
        return network_arm(args)
    return main_arm(args)


if __name__ == "__main__":
    sys.exit(main())
