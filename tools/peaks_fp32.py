"""Measured FP32 peaks of this GPU for the FP32 rooflines:
FFMA (tools/probe_fp32, all SMs, independent FMA chains) and TF32 / FP32 matmul through cuBLAS
(torch.matmul 8192^3, best of 10). Writes one JSON object (argv[1], default stdout)."""
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def mm_tflops(tf32: bool, n: int = 8192) -> float:
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn((n, n), device="cuda")
    b = torch.randn((n, n), device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2 * n ** 3 / (best * 1e-3) / 1e12


def main():
    ffma = json.loads(subprocess.run([os.path.join(ROOT, "tools", "probe_fp32")], capture_output=True, text=True,
                                     check=True).stdout)
    out = {"ffma_fp32_tflops": ffma["ffma_fp32_tflops"], "ffma_nominal_tflops": ffma["nominal_tflops"],
           "tf32_matmul_tflops": mm_tflops(True), "fp32_matmul_tflops": mm_tflops(False),
           "gpu": torch.cuda.get_device_name(), "how": "tools/probe_fp32 (FFMA, best of 5) and torch.matmul 8192^3 "
                                                      "fp32 with / without TF32 (cuBLAS, best of 10)"}
    text = json.dumps(out, indent=1)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
