"""Generate tests/golden/*.npz from the UNMODIFIED reference library (oracle/_ref).

Run here (where /root/reference exists and `make -C oracle` built oracle/_ref):

    python tests/golden/make_golden.py

The fixtures pin both the C restatement in oracle/ and the CUDA kernels to the reference's own
outputs. Every array below is produced by calling the reference (proj/src/conv.cpp,
proj/src/reference.cpp, proj/include/conv1d/{rng,bf16}.hpp) through oracle/ref_capi.cpp.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Ref  # noqa: E402

BENCH_SEED = 20260822  # proj/include/conv1d/bench.hpp:37


def rng_fixtures(ref: Ref) -> dict:
    out = {}
    for seed in (0, 1, 50, BENCH_SEED):
        out[f"rng_u64_{seed}"] = np.array(ref.rng_stream(seed, 32, "u64"), dtype=np.uint64)
        out[f"rng_double_{seed}"] = np.array(ref.rng_stream(seed, 32, "double"), dtype=np.float64)
        out[f"rng_normal_{seed}"] = np.array(ref.rng_stream(seed, 32, "normal"), dtype=np.float64)
        out[f"rng_uniform_{seed}"] = ref.rng_stream(seed, 64, "uniform")
    return out


def bf16_fixtures(ref: Ref) -> dict:
    vals = np.array(
        [1.0, 1.00390625, 1.0078125, 1.01171875, 3.141592, -2.5, 0.0, -0.0, 1e-40, -1e-40, 3.4e38,
         -3.4e38, 65504.0, 1.0 / 3.0, 2.0 / 3.0, 1e-8, 0.1, 0.2, 123456.789, float("inf"), float("-inf")],
        dtype=np.float32)
    nan_bits = np.array([0x7FC00000, 0x7F800001, 0xFF800001, 0x7FBFFFFF], dtype=np.uint32)
    vals = np.concatenate([vals, nan_bits.view(np.float32)])
    # values straddling rounding ties
    rs = np.random.default_rng(7)
    rnd = rs.standard_normal(200).astype(np.float32)
    tie = (np.arange(64, dtype=np.uint32) << 16 | 0x8000).view(np.float32) + 0  # exact ties
    vals = np.concatenate([vals, rnd, tie.astype(np.float32)])
    bits = np.array([ref.lib.ref_fp32_to_bf16(float(v)) for v in vals], dtype=np.uint16)
    return {"bf16_in": vals, "bf16_bits": bits}


def conv_cases(ref: Ref) -> dict:
    """Small seeded conv problems: inputs, reference blocked outputs (FP32 and, for even dims,
    BF16) and naive double-accumulation outputs."""
    shapes = [
        # (n, c, k, s, d, q)
        (1, 1, 1, 1, 1, 3),
        (1, 1, 1, 2, 2, 3),
        (2, 5, 4, 3, 3, 17),
        (3, 4, 6, 5, 2, 40),
        (2, 3, 4, 5, 1, 12),
        (1, 15, 15, 51, 8, 64),
        (2, 16, 16, 9, 1, 100),
        (1, 8, 4, 51, 2, 64),
        (2, 4, 15, 5, 8, 100),
        (1, 64, 64, 9, 8, 128),
        (1, 32, 32, 51, 8, 64),
        (2, 16, 16, 51, 8, 200),
        (1, 7, 5, 9, 3, 150),
        (1, 1, 16, 5, 16, 64),
        (3, 2, 1, 1, 1, 1000),
    ]
    out = {"conv_shapes": np.array(shapes, dtype=np.int64)}
    for i, (n, c, k, s, d, q) in enumerate(shapes):
        rr = ref.lib.ref_rng_new(1000 + i)
        w_in = q + d * (s - 1)
        x = np.empty((n, c, w_in), np.float32)
        w = np.empty((k, c, s), np.float32)
        dy = np.empty((n, k, q), np.float32)
        # draw order w, x, dy as in measure_kernel (proj/src/bench.cpp:188-201)
        ref.lib.ref_rng_fill_uniform(rr, w.reshape(-1), w.size, -1.0, 1.0)
        ref.lib.ref_rng_fill_uniform(rr, x.reshape(-1), x.size, -1.0, 1.0)
        ref.lib.ref_rng_fill_uniform(rr, dy.reshape(-1), dy.size, -1.0, 1.0)
        ref.lib.ref_rng_free(rr)
        rc0, y = ref.forward(x, w, d)
        rc1, dx = ref.backward_data(dy, w, d)
        rc2, dw = ref.backward_weight(dy, x, s, d)
        assert rc0 == rc1 == rc2 == 0
        out[f"c{i}_x"], out[f"c{i}_w"], out[f"c{i}_dy"] = x, w, dy
        out[f"c{i}_y"], out[f"c{i}_dx"], out[f"c{i}_dw"] = y, dx, dw
        out[f"c{i}_y_naive"] = ref.naive_forward(x, w, d)
        out[f"c{i}_dx_naive"] = ref.naive_backward_data(dy, w, d)
        out[f"c{i}_dw_naive"] = ref.naive_backward_weight(dy, x, s, d)
        if c % 2 == 0 and k % 2 == 0 and w_in % 2 == 0 and q % 2 == 0:
            _, yb = ref.forward(x, w, d, precision=1)
            _, dxb = ref.backward_data(dy, w, d, precision=1)
            _, dwb = ref.backward_weight(dy, x, s, d, precision=1)
            out[f"c{i}_y_bf16"], out[f"c{i}_dx_bf16"], out[f"c{i}_dw_bf16"] = yb, dxb, dwb
    return out


def pack_fixtures(ref: Ref) -> dict:
    w = np.arange(3 * 2 * 4, dtype=np.float32).reshape(3, 2, 4)  # K=3, C=2, S=4
    f = np.empty(w.size, np.float32)
    b = np.empty(w.size, np.float32)
    ref.lib.ref_pack_forward(w.reshape(-1), 3, 2, 4, f)
    ref.lib.ref_pack_backward(w.reshape(-1), 3, 2, 4, b)
    return {"pack_w": w, "pack_fwd": f.reshape(4, 3, 2), "pack_bwd": b.reshape(4, 2, 3)}


def main() -> None:
    ref = Ref()
    data = {}
    data.update(rng_fixtures(ref))
    data.update(bf16_fixtures(ref))
    data.update(pack_fixtures(ref))
    data.update(conv_cases(ref))
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {path}: {len(data)} arrays, {os.path.getsize(path)} bytes (reference lib {ref.path})")


if __name__ == "__main__":
    main()
