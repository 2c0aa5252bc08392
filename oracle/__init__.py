"""oracle — CPU parity checkers for the B200 conv1d kernels.

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of bench.py, never by the product package.

Two checkers live here:

* :mod:`oracle` itself binds ``liboracle.so``, a plain-C restatement of the reference
  algorithm (``oracle/conv1d_oracle.c``; every function cites the reference file:line it
  follows).
* :class:`Ref` binds ``oracle/_ref/libconv1d_ref_v{3,4}.so``: the unmodified reference
  library compiled from ``/root/reference/proj/src`` by ``oracle/Makefile`` (the reference's
  own blocked CPU path, naive oracles, ``measure_kernel`` and ``Rng``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
I64 = C.c_int64


def build() -> None:
    """Build liboracle.so (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load_oracle() -> C.CDLL:
    path = os.path.join(HERE, "liboracle.so")
    if not os.path.exists(path):
        build()
    lib = C.CDLL(path)
    lib.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
    lib.orc_rng_next_u64.restype = C.c_uint64
    lib.orc_rng_next_u64.argtypes = [C.c_void_p]
    lib.orc_rng_next_double.restype = C.c_double
    lib.orc_rng_next_double.argtypes = [C.c_void_p]
    lib.orc_rng_next_float.restype = C.c_float
    lib.orc_rng_next_float.argtypes = [C.c_void_p, C.c_float, C.c_float]
    lib.orc_rng_next_below.restype = C.c_uint64
    lib.orc_rng_next_below.argtypes = [C.c_void_p, C.c_uint64]
    lib.orc_rng_next_normal.restype = C.c_double
    lib.orc_rng_next_normal.argtypes = [C.c_void_p]
    lib.orc_fill_uniform.argtypes = [C.c_void_p, _f32p, I64, C.c_float, C.c_float]
    lib.orc_fill_normal.argtypes = [C.c_void_p, _f32p, I64]
    lib.orc_fill_poisson.argtypes = [C.c_void_p, _f32p, I64, C.c_double]
    lib.orc_fill_bernoulli.argtypes = [C.c_void_p, _f32p, I64, C.c_double]
    lib.orc_fp32_to_bf16.restype = C.c_uint16
    lib.orc_fp32_to_bf16.argtypes = [C.c_float]
    lib.orc_to_bf16_bits.argtypes = [_f32p, _u16p, I64]
    lib.orc_round_bf16.argtypes = [_f32p, _f32p, I64]
    lib.orc_validate_params.argtypes = [I64, I64, I64, I64, C.c_int, I64]
    lib.orc_output_width.argtypes = [I64, I64, I64, I64, I64, C.POINTER(I64)]
    lib.orc_conv_flops.restype = I64
    lib.orc_conv_flops.argtypes = [I64] * 5
    lib.orc_same_pad_width.restype = I64
    lib.orc_same_pad_width.argtypes = [I64, I64]
    lib.orc_pack_forward.argtypes = [_f32p, I64, I64, I64, _f32p]
    lib.orc_pack_backward.argtypes = [_f32p, I64, I64, I64, _f32p]
    lib.orc_unpack.argtypes = [_f32p, C.c_int, I64, I64, I64, _f32p]
    lib.orc_zero_pad_width.argtypes = [_f32p, I64, I64, I64, I64, I64, _f32p]
    lib.orc_naive_forward.argtypes = [_f32p, I64, I64, I64, _f32p, I64, I64, I64, _f32p]
    lib.orc_naive_backward_data.argtypes = [_f32p, I64, I64, I64, _f32p, I64, I64, I64, _f32p]
    lib.orc_naive_backward_weight.argtypes = [_f32p, _f32p, I64, I64, I64, I64, I64, I64, _f32p]
    lib.orc_norm_rel_error.restype = C.c_double
    lib.orc_norm_rel_error.argtypes = [_f32p, _f32p, I64]
    return lib


_lib = _load_oracle()


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ----------------------------------------------------------------------------- rng
class Rng:
    """xoshiro256** seeded by splitmix64 (restates rng.hpp:12-64)."""

    def __init__(self, seed: int):
        self._state = (C.c_uint64 * 4)()
        _lib.orc_rng_seed(self._state, C.c_uint64(seed))

    def next_u64(self) -> int:
        return _lib.orc_rng_next_u64(self._state)

    def next_double(self) -> float:
        return _lib.orc_rng_next_double(self._state)

    def next_float(self, lo: float, hi: float) -> float:
        return _lib.orc_rng_next_float(self._state, lo, hi)

    def next_below(self, bound: int) -> int:
        return _lib.orc_rng_next_below(self._state, bound)

    def next_normal(self) -> float:
        return _lib.orc_rng_next_normal(self._state)

    def fill_uniform(self, shape, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        out = np.empty(shape, dtype=np.float32)
        _lib.orc_fill_uniform(self._state, out.reshape(-1), out.size, lo, hi)
        return out

    def fill_normal(self, shape) -> np.ndarray:
        out = np.empty(shape, dtype=np.float32)
        _lib.orc_fill_normal(self._state, out.reshape(-1), out.size)
        return out

    def fill_poisson(self, shape, lam: float = 2.0) -> np.ndarray:
        out = np.empty(shape, dtype=np.float32)
        _lib.orc_fill_poisson(self._state, out.reshape(-1), out.size, lam)
        return out

    def fill_bernoulli(self, shape, p: float = 0.1) -> np.ndarray:
        out = np.empty(shape, dtype=np.float32)
        _lib.orc_fill_bernoulli(self._state, out.reshape(-1), out.size, p)
        return out


# ----------------------------------------------------------------------------- bf16
def fp32_to_bf16_bits(a) -> np.ndarray:
    a = _f32(a)
    out = np.empty(a.shape, dtype=np.uint16)
    _lib.orc_to_bf16_bits(a.reshape(-1), out.reshape(-1), a.size)
    return out


def round_bf16(a) -> np.ndarray:
    a = _f32(a)
    out = np.empty_like(a)
    _lib.orc_round_bf16(a.reshape(-1), out.reshape(-1), a.size)
    return out


# ----------------------------------------------------------------------------- geometry / packing
def validate_params(c, k, s, d, precision=0, block_w=64) -> int:
    return _lib.orc_validate_params(c, k, s, d, precision, block_w)


def output_width(c, k, s, d, w_padded):
    q = I64(0)
    rc = _lib.orc_output_width(c, k, s, d, w_padded, C.byref(q))
    return rc, q.value


def conv_flops(n, c, k, s, q) -> int:
    return _lib.orc_conv_flops(n, c, k, s, q)


def same_pad_width(s, d) -> int:
    return _lib.orc_same_pad_width(s, d)


def pack_forward(w_kcs) -> np.ndarray:
    w = _f32(w_kcs)
    k, c, s = w.shape
    out = np.empty((s, k, c), dtype=np.float32)
    _lib.orc_pack_forward(w.reshape(-1), k, c, s, out.reshape(-1))
    return out


def pack_backward(w_kcs) -> np.ndarray:
    w = _f32(w_kcs)
    k, c, s = w.shape
    out = np.empty((s, c, k), dtype=np.float32)
    _lib.orc_pack_backward(w.reshape(-1), k, c, s, out.reshape(-1))
    return out


def unpack(packed, layout: int, k: int, c: int, s: int) -> np.ndarray:
    out = np.empty((k, c, s), dtype=np.float32)
    _lib.orc_unpack(_f32(packed).reshape(-1), layout, k, c, s, out.reshape(-1))
    return out


def zero_pad_width(t, left: int, right: int) -> np.ndarray:
    t = _f32(t)
    n, c, w = t.shape
    out = np.empty((n, c, w + left + right), dtype=np.float32)
    _lib.orc_zero_pad_width(t.reshape(-1), n, c, w, left, right, out.reshape(-1))
    return out


# ----------------------------------------------------------------------------- naive passes
def naive_forward(x, w_kcs, d: int) -> np.ndarray:
    x, w = _f32(x), _f32(w_kcs)
    n, c, w_in = x.shape
    k, c2, s = w.shape
    assert c == c2
    q = w_in - d * (s - 1)
    out = np.empty((n, k, q), dtype=np.float32)
    _lib.orc_naive_forward(x.reshape(-1), n, c, w_in, w.reshape(-1), k, s, d, out.reshape(-1))
    return out


def naive_backward_data(dy, w_kcs, d: int) -> np.ndarray:
    dy, w = _f32(dy), _f32(w_kcs)
    n, k, q = dy.shape
    k2, c, s = w.shape
    assert k == k2
    out = np.empty((n, c, q + d * (s - 1)), dtype=np.float32)
    _lib.orc_naive_backward_data(dy.reshape(-1), n, k, q, w.reshape(-1), c, s, d, out.reshape(-1))
    return out


def naive_backward_weight(dy, x, s: int, d: int) -> np.ndarray:
    dy, x = _f32(dy), _f32(x)
    n, k, q = dy.shape
    n2, c, w_in = x.shape
    assert n == n2 and w_in == q + d * (s - 1)
    out = np.empty((k, c, s), dtype=np.float32)
    _lib.orc_naive_backward_weight(dy.reshape(-1), x.reshape(-1), n, c, k, s, d, q, out.reshape(-1))
    return out


def norm_rel_error(got, want) -> float:
    got, want = _f32(got).reshape(-1), _f32(want).reshape(-1)
    assert got.size == want.size
    return _lib.orc_norm_rel_error(got, want, got.size)


# ----------------------------------------------------------------------------- the reference itself
def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
        return all(f" {x}" in flags for x in ("avx512f", "avx512bw", "avx512dq", "avx512vl"))
    except OSError:
        return False


def ref_library_path() -> str | None:
    for variant in (("v4", "v3") if _cpu_has_avx512() else ("v3",)):
        p = os.path.join(HERE, "_ref", f"libconv1d_ref_{variant}.so")
        if os.path.exists(p):
            return p
    return None


class Ref:
    """ctypes view of the unmodified reference library (oracle/_ref)."""

    def __init__(self, path: str | None = None):
        path = path or ref_library_path()
        if path is None:
            raise FileNotFoundError("oracle/_ref/libconv1d_ref_*.so not built (make -C oracle)")
        self.path = path
        lib = self.lib = C.CDLL(path)
        lib.ref_forward.argtypes = [_f32p, I64, I64, I64, _f32p, I64, I64, I64, C.c_int, I64, C.c_int, _f32p]
        lib.ref_backward_data.argtypes = [_f32p, I64, I64, I64, _f32p, I64, I64, I64, C.c_int, I64, C.c_int,
                                          _f32p]
        lib.ref_backward_weight.argtypes = [_f32p, _f32p, I64, I64, I64, I64, I64, I64, C.c_int, I64, C.c_int,
                                            _f32p]
        lib.ref_output_width.argtypes = [I64, I64, I64, I64, C.c_int, I64, C.POINTER(I64)]
        lib.ref_conv_flops.restype = I64
        lib.ref_conv_flops.argtypes = [I64] * 5
        lib.ref_pack_forward.argtypes = [_f32p, I64, I64, I64, _f32p]
        lib.ref_pack_backward.argtypes = [_f32p, I64, I64, I64, _f32p]
        lib.ref_naive_forward.argtypes = [_f32p, I64, I64, I64, _f32p, I64, I64, I64, _f32p]
        lib.ref_naive_backward_data.argtypes = [_f32p, I64, I64, I64, _f32p, I64, I64, I64, _f32p]
        lib.ref_naive_backward_weight.argtypes = [_f32p, _f32p, I64, I64, I64, I64, I64, I64, _f32p]
        lib.ref_norm_rel_error.restype = C.c_double
        lib.ref_norm_rel_error.argtypes = [_f32p, _f32p, I64]
        lib.ref_fp32_to_bf16.restype = C.c_uint16
        lib.ref_fp32_to_bf16.argtypes = [C.c_float]
        lib.ref_rng_new.restype = C.c_void_p
        lib.ref_rng_new.argtypes = [C.c_uint64]
        lib.ref_rng_free.argtypes = [C.c_void_p]
        lib.ref_rng_next_u64.restype = C.c_uint64
        lib.ref_rng_next_u64.argtypes = [C.c_void_p]
        lib.ref_rng_next_double.restype = C.c_double
        lib.ref_rng_next_double.argtypes = [C.c_void_p]
        lib.ref_rng_next_normal.restype = C.c_double
        lib.ref_rng_next_normal.argtypes = [C.c_void_p]
        lib.ref_rng_next_below.restype = C.c_uint64
        lib.ref_rng_next_below.argtypes = [C.c_void_p, C.c_uint64]
        lib.ref_rng_fill_uniform.argtypes = [C.c_void_p, _f32p, I64, C.c_float, C.c_float]
        lib.ref_measure_kernel.restype = C.c_double
        lib.ref_measure_kernel.argtypes = [I64, I64, I64, I64, I64, I64, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_uint64]

    # reference fast (blocked) passes; return (status, array)
    def forward(self, x, w_kcs, d, precision=0, threads=1, block_w=64):
        x, w = _f32(x), _f32(w_kcs)
        n, c, w_in = x.shape
        k, _, s = w.shape
        q = max(w_in - d * (s - 1), 0)
        out = np.zeros((n, k, q), dtype=np.float32)
        rc = self.lib.ref_forward(x.reshape(-1), n, c, w_in, w.reshape(-1), k, s, d, precision, block_w,
                                  threads, out.reshape(-1))
        return rc, out

    def backward_data(self, dy, w_kcs, d, precision=0, threads=1, block_w=64):
        dy, w = _f32(dy), _f32(w_kcs)
        n, k, q = dy.shape
        _, c, s = w.shape
        out = np.zeros((n, c, q + d * (s - 1)), dtype=np.float32)
        rc = self.lib.ref_backward_data(dy.reshape(-1), n, k, q, w.reshape(-1), c, s, d, precision, block_w,
                                        threads, out.reshape(-1))
        return rc, out

    def backward_weight(self, dy, x, s, d, precision=0, threads=1, block_w=64):
        dy, x = _f32(dy), _f32(x)
        n, k, q = dy.shape
        c = x.shape[1]
        out = np.zeros((k, c, s), dtype=np.float32)
        rc = self.lib.ref_backward_weight(dy.reshape(-1), x.reshape(-1), n, c, k, s, d, q, precision, block_w,
                                          threads, out.reshape(-1))
        return rc, out

    def naive_forward(self, x, w_kcs, d):
        x, w = _f32(x), _f32(w_kcs)
        n, c, w_in = x.shape
        k, _, s = w.shape
        out = np.zeros((n, k, w_in - d * (s - 1)), dtype=np.float32)
        self.lib.ref_naive_forward(x.reshape(-1), n, c, w_in, w.reshape(-1), k, s, d, out.reshape(-1))
        return out

    def naive_backward_data(self, dy, w_kcs, d):
        dy, w = _f32(dy), _f32(w_kcs)
        n, k, q = dy.shape
        _, c, s = w.shape
        out = np.zeros((n, c, q + d * (s - 1)), dtype=np.float32)
        self.lib.ref_naive_backward_data(dy.reshape(-1), n, k, q, w.reshape(-1), c, s, d, out.reshape(-1))
        return out

    def naive_backward_weight(self, dy, x, s, d):
        dy, x = _f32(dy), _f32(x)
        n, k, q = dy.shape
        c = x.shape[1]
        out = np.zeros((k, c, s), dtype=np.float32)
        self.lib.ref_naive_backward_weight(dy.reshape(-1), x.reshape(-1), n, c, k, s, d, q, out.reshape(-1))
        return out

    def norm_rel_error(self, got, want):
        got, want = _f32(got).reshape(-1), _f32(want).reshape(-1)
        return self.lib.ref_norm_rel_error(got, want, got.size)

    def measure_kernel(self, n, c, k, s, d, q, precision, pass_, iterations, warmup, threads,
                       seed=20260822) -> float:
        return self.lib.ref_measure_kernel(n, c, k, s, d, q, precision, pass_, iterations, warmup, threads,
                                           seed)

    def rng_stream(self, seed: int, count: int, kind: str = "u64"):
        r = self.lib.ref_rng_new(seed)
        try:
            if kind == "u64":
                return [self.lib.ref_rng_next_u64(r) for _ in range(count)]
            if kind == "double":
                return [self.lib.ref_rng_next_double(r) for _ in range(count)]
            if kind == "normal":
                return [self.lib.ref_rng_next_normal(r) for _ in range(count)]
            if kind == "uniform":
                out = np.empty(count, dtype=np.float32)
                self.lib.ref_rng_fill_uniform(r, out, count, -1.0, 1.0)
                return out
            raise ValueError(kind)
        finally:
            self.lib.ref_rng_free(r)


class RefNet:
    """The reference's DemoNet (proj/src/train.cpp:257-353) through oracle/_ref: the network the
    GPU ResidualNet(convs_per_block=1) is pinned to. TEST INFRASTRUCTURE ONLY."""

    def __init__(self, blocks: int, hidden: int, taps: int = 51, dilation: int = 8, precision: int = 0,
                 seed: int = 1, ref: "Ref | None" = None):
        self.ref = ref or Ref()
        L = self.ref.lib
        L.ref_demonet_new.restype = C.c_void_p
        L.ref_demonet_new.argtypes = [C.c_int, I64, I64, I64, C.c_int, C.c_uint64]
        L.ref_demonet_free.argtypes = [C.c_void_p]
        L.ref_demonet_layer_precision.argtypes = [C.c_void_p, C.c_int]
        L.ref_demonet_param_count.restype = I64
        L.ref_demonet_param_count.argtypes = [C.c_void_p]
        L.ref_demonet_gather_params.argtypes = [C.c_void_p, _f32p]
        L.ref_demonet_scatter_params.argtypes = [C.c_void_p, _f32p, I64]
        L.ref_demonet_gather_grads.argtypes = [C.c_void_p, _f32p]
        L.ref_demonet_forward.argtypes = [C.c_void_p, _f32p, I64, I64, C.c_int, _f32p, _f32p]
        L.ref_demonet_train_step.argtypes = [C.c_void_p, _f32p, _f32p, _f32p, I64, I64, I64, C.c_float, C.c_int,
                                             C.POINTER(C.c_double)]
        L.ref_demonet_step.argtypes = [C.c_void_p, C.c_float]
        self.L = L
        self.blocks, self.taps, self.dilation = blocks, taps, dilation
        self.h = L.ref_demonet_new(blocks, hidden, taps, dilation, precision, seed)
        if not self.h:
            raise RuntimeError("DemoNet construction failed")

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_demonet_free(self.h)
            self.h = None

    def pad(self) -> int:
        return self.dilation * (self.taps - 1) // 2

    def layer_precisions(self) -> list[int]:
        return [self.L.ref_demonet_layer_precision(self.h, i) for i in range(self.blocks + 3)]

    def params(self) -> np.ndarray:
        out = np.empty(self.L.ref_demonet_param_count(self.h), dtype=np.float32)
        self.L.ref_demonet_gather_params(self.h, out)
        return out

    def set_params(self, flat) -> None:
        flat = _f32(flat).reshape(-1)
        if self.L.ref_demonet_scatter_params(self.h, flat, flat.size) != 0:
            raise ValueError("scatter_params rejected the vector")

    def grads(self) -> np.ndarray:
        out = np.empty(self.L.ref_demonet_param_count(self.h), dtype=np.float32)
        self.L.ref_demonet_gather_grads(self.h, out)
        return out

    def forward(self, x_padded, threads: int = 1):
        x = _f32(x_padded)
        n, _, wp = x.shape
        width = wp - 2 * self.pad()
        pred = np.empty((n, 1, width), dtype=np.float32)
        logits = np.empty((n, 1, width), dtype=np.float32)
        rc = self.L.ref_demonet_forward(self.h, x.reshape(-1), n, wp, threads, pred.reshape(-1), logits.reshape(-1))
        if rc:
            raise RuntimeError(f"DemoNet forward failed ({rc})")
        return pred, logits

    def train_step(self, x_padded, clean, mask, bce_weight: float = 1.0, threads: int = 1) -> float:
        x, y, m = _f32(x_padded), _f32(clean), _f32(mask)
        n, _, wp = x.shape
        loss = C.c_double(0.0)
        rc = self.L.ref_demonet_train_step(self.h, x.reshape(-1), y.reshape(-1), m.reshape(-1), n, wp, y.shape[2],
                                           bce_weight, threads, C.byref(loss))
        if rc:
            raise RuntimeError(f"DemoNet train_step failed ({rc})")
        return loss.value

    def step(self, lr: float) -> None:
        self.L.ref_demonet_step(self.h, lr)


def ref_losses(ref: "Ref", pred, target, logits, labels):
    """mse_loss / bce_with_logits of the reference (train.cpp:106-135): (mse, g_mse, bce, g_bce)."""
    L = ref.lib
    for name in ("ref_mse_loss", "ref_bce_with_logits"):
        fn = getattr(L, name)
        fn.restype = C.c_double
        fn.argtypes = [_f32p, _f32p, I64, _f32p]
    a, b, c, d = (_f32(v).reshape(-1) for v in (pred, target, logits, labels))
    ga, gc = np.empty_like(a), np.empty_like(c)
    mse = L.ref_mse_loss(a, b, a.size, ga)
    bce = L.ref_bce_with_logits(c, d, c.size, gc)
    return mse, ga, bce, gc


def ref_auroc(ref: "Ref", scores, labels) -> float:
    """auroc of the reference (train.cpp:143-171): rank statistic, ties averaged."""
    L = ref.lib
    L.ref_auroc.restype = C.c_double
    L.ref_auroc.argtypes = [_f32p, _f32p, I64]
    a, b = _f32(scores).reshape(-1), _f32(labels).reshape(-1)
    return L.ref_auroc(a, b, a.size)


def ref_synthetic_dataset(ref: "Ref", seed: int, count: int, width: int):
    """generate_synthetic_dataset of the reference (train.cpp:62-98): (noisy, clean, mask)."""
    L = ref.lib
    L.ref_synthetic_dataset.argtypes = [C.c_uint64, I64, I64, _f32p, _f32p, _f32p]
    out = [np.empty((count, 1, width), dtype=np.float32) for _ in range(3)]
    rc = L.ref_synthetic_dataset(seed, count, width, *(o.reshape(-1) for o in out))
    if rc:
        raise RuntimeError(f"generate_synthetic_dataset failed ({rc})")
    return tuple(out)


def sample_poisson(count: int, lam: float, seed: int) -> np.ndarray:
    """The device sampler's per-element splitmix64 Poisson draw (c1d_fill_poisson), restated."""
    out = np.empty(count, dtype=np.float32)
    _lib.orc_sample_poisson.argtypes = [_f32p, I64, C.c_double, C.c_uint64]
    _lib.orc_sample_poisson(out, count, lam, seed)
    return out


def sample_bernoulli(count: int, p: float, seed: int) -> np.ndarray:
    """The device sampler's Bernoulli draw (c1d_fill_bernoulli), restated."""
    out = np.empty(count, dtype=np.float32)
    _lib.orc_sample_bernoulli.argtypes = [_f32p, I64, C.c_double, C.c_uint64]
    _lib.orc_sample_bernoulli(out, count, p, seed)
    return out

