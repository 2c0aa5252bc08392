"""Dev timing tool: CUDA-event time of each pass at a BASELINE config (inputs resident in HBM).

usage: python tools/time_passes.py [cfg ...]   cfg in {1,2,3,33}  (33: config 3 in FP32)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_08002_b200 import conv as cv  # noqa: E402

CFGS = {
    1: dict(n=4, c=15, k=15, s=51, d=8, q=60000, prec=cv.Precision.Fp32),
    2: dict(n=16, c=15, k=15, s=51, d=8, q=60000, prec=cv.Precision.Bf16),
    3: dict(n=32, c=64, k=64, s=51, d=8, q=60000, prec=cv.Precision.Bf16),
    33: dict(n=32, c=64, k=64, s=51, d=8, q=60000, prec=cv.Precision.Fp32),
}


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for ci in cfgs:
        c = CFGS[ci]
        w_in = c["q"] + c["d"] * (c["s"] - 1)
        p = cv.ConvParams(c["c"], c["k"], c["s"], c["d"], c["prec"])
        dt = torch.bfloat16 if c["prec"] == cv.Precision.Bf16 else torch.float32
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.randn((c["n"], c["c"], w_in), device="cuda", generator=g).to(dt)
        dy = torch.randn((c["n"], c["k"], c["q"]), device="cuda", generator=g).to(dt)
        w = torch.randn((c["k"], c["c"], c["s"]), device="cuda", generator=g) * 0.05
        y = torch.empty((c["n"], c["k"], c["q"]), device="cuda")
        dx = torch.empty((c["n"], c["c"], w_in), device="cuda")
        dw = torch.empty((c["k"], c["c"], c["s"]), device="cuda")
        wb = cv.pack_weights_backward(w)
        flops = cv.conv_flops(p, c["n"], c["q"])
        passes = {
            "fwd": lambda: cv.conv1d_forward(x, w, p, out=y),
            "bwd_d": lambda: cv.conv1d_backward_data(dy, wb, p, out=dx),
            "bwd_w": lambda: cv.conv1d_backward_weight(dy, x, p, out=dw),
        }
        for name, fn in passes.items():
            algo = cv.selected_algo(p, c["n"], w_in, ["fwd", "bwd_d", "bwd_w"].index(name),
                                    in_dtype=1 if dt == torch.bfloat16 else 0)
            for _ in range(3):
                fn()
            times = []
            for _ in range(10):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            times.sort()
            t = times[len(times) // 2]
            print(f"cfg{ci} {name:6s} {algo:8s} median {t * 1e3:9.1f} us  {flops / (t * 1e-3) / 1e12:8.1f} TFLOP/s")
    print("done")


if __name__ == "__main__":
    main()
