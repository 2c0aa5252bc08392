"""Small problems through every kernel mode, for compute-sanitizer (memcheck / racecheck / synccheck)
runs. PDL stays on. Usage:

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Each case runs its three passes once and checks them against the oracle (so a sanitizer-clean run is
also a correct one); the last line is "sanitize cases OK (<n> cases)".
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2104_08002_b200 import conv as cv  # noqa: E402
from paper_2104_08002_b200 import network as nw  # noqa: E402

# (C, K, S, d, Q, N, precision, exact, note)
CASES = [
    (16, 16, 51, 8, 512, 2, "bf16", False, "carry mode, double-buffered TMEM, resident weights (narrow)"),
    (64, 64, 51, 8, 1024, 1, "bf16", False, "carry mode KP=64 with the tail-tap MMA; wgrad v3 (T=2, P=4)"),
    (128, 128, 9, 8, 512, 1, "bf16", False, "carry-free direct mode (K > 64)"),
    (160, 128, 51, 8, 256, 1, "bf16", True, "exact: two TMEM regions; segmented wgrad chains"),
    (64, 64, 17, 1, 520, 1, "bf16", False, "expanded rows d=1 (row tensor / inline); wgrad xin"),
    (48, 48, 33, 2, 500, 1, "bf16", False, "expanded rows d=2, unaligned width"),
    (32, 32, 33, 4, 512, 1, "bf16", False, "expanded rows d=4 inline"),
    (24, 40, 11, 16, 512, 1, "bf16", False, "chunk planes d=16"),
    (8, 8, 7, 3, 300, 2, "bf16", False, "FFMA direct kernels (d=3)"),
    (15, 15, 51, 8, 512, 2, "fp32", False, "FP32 six-block split (carry mode, two regions); 3-level wgrad"),
    (72, 72, 9, 8, 256, 1, "fp32", False, "FP32 wgrad block passes (2C > 128)"),
    (16, 16, 9, 2, 256, 1, "fp32", False, "FP32 split on expanded rows"),
    (16, 160, 5, 8, 256, 1, "bf16", False, "wgrad v1 (K > 128)"),
]


def run_case(c, k, s, d, q, n, prec, exact):
    rng = oracle.Rng(100 + c + k + s + d)
    w_in = q + d * (s - 1)
    x, w, dy = rng.fill_uniform((n, c, w_in)), rng.fill_uniform((k, c, s)), rng.fill_uniform((n, k, q))
    p = cv.ConvParams(c, k, s, d, cv.Precision.Bf16 if prec == "bf16" else cv.Precision.Fp32)
    t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    y = cv.conv1d_forward(t(x), t(w), p, exact=exact)
    dx = cv.conv1d_backward_data(t(dy), t(w), p, exact=exact)
    dw = cv.conv1d_backward_weight(t(dy), t(x), p, exact=exact)
    torch.cuda.synchronize()
    if prec == "bf16":
        x, w, dy = oracle.round_bf16(x), oracle.round_bf16(w), oracle.round_bf16(dy)
    errs = [oracle.norm_rel_error(y.cpu().numpy(), oracle.naive_forward(x, w, d)),
            oracle.norm_rel_error(dx.cpu().numpy(), oracle.naive_backward_data(dy, w, d)),
            oracle.norm_rel_error(dw.cpu().numpy(), oracle.naive_backward_weight(dy, x, s, d))]
    assert all(e <= 1e-4 for e in errs), errs
    return errs


def run_glue():
    """Glued forward (mode 1, skip, two epilogue groups) and glued backward-data (mode 2, bias grad)."""
    n, c, q, pad = 2, 15, 512, 200
    g = torch.Generator(device="cuda").manual_seed(3)
    p = cv.ConvParams(c, c, 51, 8, cv.Precision.Bf16)
    x = torch.zeros((n, c, q + 2 * pad), device="cuda", dtype=torch.bfloat16)
    x[:, :, pad:pad + q] = torch.randn((n, c, q), device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn((c, c, 51), device="cuda", generator=g) * 0.05
    bias = torch.randn(c, device="cuda", generator=g)
    skip = torch.randn((n, c, q), device="cuda", generator=g)
    act = torch.empty((n, c, q), device="cuda")
    act_b = torch.zeros((n, c, q + 2 * pad), device="cuda", dtype=torch.bfloat16)
    mask = torch.empty(nw.mask_shape(n, c, q), dtype=torch.int32, device="cuda")
    nw.conv_forward_glued(x, w, p, bias=bias, skip=skip, act=act, act_bf16=act_b, act_pad=pad, mask=mask)
    gy = torch.randn((n, c, q), device="cuda", generator=g).to(torch.bfloat16)
    gsum = torch.empty((n, c, q), device="cuda")
    gp = torch.empty((n, c, q), device="cuda", dtype=torch.bfloat16)
    bg = torch.empty(c, device="cuda")
    nw.conv_backward_data_glued(gy, w, p, pad, q, gadd=skip, mask=mask, gsum=gsum, grad_pre_bf16=gp, bias_grad=bg)
    torch.cuda.synchronize()
    assert torch.isfinite(act).all() and torch.isfinite(gsum).all() and torch.isfinite(bg).all()


def run_train():
    """Samplers, fused loss, SGD update and a small network step."""
    x, t, lab = nw.sample_inputs(2, 1024, 200, seed=1, device="cuda")
    net = nw.ResidualNet(blocks=1, convs_per_block=2, hidden=15, device="cuda")
    nw.forward_backward(net, x, t, lab)
    net.sgd_step(1e-3)
    torch.cuda.synchronize()
    assert torch.isfinite(net.grad_bucket).all()


def main():
    only = set(sys.argv[1:])
    done = 0
    for i, case in enumerate(CASES):
        if only and str(i) not in only:
            continue
        errs = run_case(*case[:8])
        print(f"case {i} ({case[8]}): errs {['%.1e' % e for e in errs]}", flush=True)
        done += 1
    if not only or "glue" in only:
        run_glue()
        print("glue OK", flush=True)
        done += 1
    if not only or "train" in only:
        run_train()
        print("train OK", flush=True)
        done += 1
    print(f"sanitize cases OK ({done} cases)")


if __name__ == "__main__":
    main()
