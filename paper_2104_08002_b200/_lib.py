"""ctypes binding of libc1d.so (include/c1d.h). Fails loudly when the CUDA library is missing:
there is no CPU fallback on the product path."""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("C1D_LIB_PATH") or os.path.join(HERE, "libc1d.so")  # override: dev A/B only
HEADER_PATH = os.path.join(ROOT, "include", "c1d.h")

# status codes (c1d_status)
OK, ERR_SHAPE_MISMATCH, ERR_ODD_DIMS, ERR_TOO_NARROW, ERR_INVALID_ARGUMENT, ERR_WORKSPACE, ERR_UNSUPPORTED, \
    ERR_CUDA, ERR_NO_DEVICE = range(9)
PASS_FORWARD, PASS_BACKWARD_DATA, PASS_BACKWARD_WEIGHT = 0, 1, 2
ALGO_AUTO, ALGO_DIRECT, ALGO_TCGEN05, ALGO_BF16X3 = 0, 1, 2, 3
DTYPE_F32, DTYPE_BF16 = 0, 1
FLAG_STRICT_BF16_DIMS = 0x1
FLAG_EXACT_ACCUM = 0x2
FLAG_PREPACKED_WEIGHTS = 0x4


class Desc(C.Structure):
    """Mirror of c1d_desc."""

    _fields_ = [
        ("n", C.c_int64),
        ("c", C.c_int64),
        ("k", C.c_int64),
        ("s", C.c_int64),
        ("d", C.c_int64),
        ("w_in", C.c_int64),
        ("precision", C.c_int32),
        ("in_dtype", C.c_int32),
        ("algo", C.c_int32),
        ("flags", C.c_uint32),
        ("block_w", C.c_int64),
    ]


class FwdGlue(C.Structure):
    """Mirror of c1d_fwd_glue."""

    _fields_ = [
        ("bias", C.c_void_p),
        ("skip", C.c_void_p),
        ("pre", C.c_void_p),
        ("act", C.c_void_p),
        ("act_bf16", C.c_void_p),
        ("mask", C.c_void_p),
        ("act_pad", C.c_int64),
        ("relu", C.c_int32),
        ("reserved", C.c_int32),
    ]


class BwdGlue(C.Structure):
    """Mirror of c1d_bwd_glue."""

    _fields_ = [
        ("off", C.c_int64),
        ("q", C.c_int64),
        ("gadd", C.c_void_p),
        ("mask", C.c_void_p),
        ("gsum", C.c_void_p),
        ("grad_pre", C.c_void_p),
        ("grad_pre_bf16", C.c_void_p),
        ("bias_grad", C.c_void_p),
    ]


def exported_symbols() -> list[str]:
    """Function names declared C1D_EXPORT in include/c1d.h."""
    with open(HEADER_PATH) as f:
        text = f.read()
    return re.findall(r"C1D_EXPORT\s+[\w\s\*]+?\b(c1d_\w+)\s*\(", text)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2104_08002_b200)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    L.c1d_api_version.restype = C.c_int
    L.c1d_strerror.restype = C.c_char_p
    L.c1d_strerror.argtypes = [C.c_int]
    L.c1d_last_error_message.restype = C.c_char_p
    L.c1d_output_width.argtypes = [P(Desc), P(C.c_int64)]
    L.c1d_output_width.restype = C.c_int
    L.c1d_conv_flops.argtypes = [P(Desc)]
    L.c1d_conv_flops.restype = C.c_int64
    L.c1d_workspace_size.argtypes = [P(Desc), C.c_int, P(C.c_size_t)]
    L.c1d_workspace_size.restype = C.c_int
    L.c1d_selected_algo.argtypes = [P(Desc), C.c_int, P(C.c_int)]
    L.c1d_selected_algo.restype = C.c_int
    for name in ("c1d_forward", "c1d_backward_data"):
        fn = getattr(L, name)
        fn.argtypes = [P(Desc), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        fn.restype = C.c_int
    L.c1d_backward_weight.argtypes = [P(Desc), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                      C.c_void_p]
    L.c1d_backward_weight.restype = C.c_int
    L.c1d_packed_weights_size.argtypes = [P(Desc), C.c_int, P(C.c_size_t)]
    L.c1d_packed_weights_size.restype = C.c_int
    L.c1d_pack_weights.argtypes = [C.c_int, P(Desc), P(C.c_int32), P(C.c_void_p), P(C.c_void_p), C.c_void_p]
    L.c1d_pack_weights.restype = C.c_int
    L.c1d_round_bf16.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    L.c1d_round_bf16.restype = C.c_int
    L.c1d_launch_count.restype = C.c_uint64
    L.c1d_release_workspace.argtypes = [C.c_void_p]
    L.c1d_release_workspace.restype = C.c_int
    i64, vp = C.c_int64, C.c_void_p
    L.c1d_layer_forward_epilogue.argtypes = [vp, vp, vp, i64, i64, i64, C.c_int, C.c_int, vp, vp, i64, vp]
    L.c1d_layer_forward_epilogue.restype = C.c_int
    L.c1d_layer_backward_workspace.argtypes = [i64, i64, i64]
    L.c1d_layer_backward_workspace.restype = C.c_size_t
    L.c1d_layer_backward_prologue.argtypes = [vp, i64, i64, vp, vp, vp, i64, i64, i64, C.c_int, vp, vp, vp, vp,
                                              vp, C.c_size_t, vp]
    L.c1d_layer_backward_prologue.restype = C.c_int
    L.c1d_glued_workspace_size.argtypes = [P(Desc), C.c_int, i64, P(C.c_size_t), P(C.c_int)]
    L.c1d_glued_workspace_size.restype = C.c_int
    L.c1d_forward_glued.argtypes = [P(Desc), vp, vp, P(FwdGlue), vp, C.c_size_t, vp]
    L.c1d_forward_glued.restype = C.c_int
    L.c1d_backward_data_glued.argtypes = [P(Desc), vp, vp, P(BwdGlue), vp, C.c_size_t, vp]
    L.c1d_backward_data_glued.restype = C.c_int
    L.c1d_fill_poisson.argtypes = [vp, i64, C.c_double, C.c_uint64, vp]
    L.c1d_fill_poisson.restype = C.c_int
    L.c1d_fill_bernoulli.argtypes = [vp, i64, C.c_double, C.c_uint64, vp]
    L.c1d_fill_bernoulli.restype = C.c_int
    L.c1d_loss_workspace_size.restype = C.c_size_t
    L.c1d_mse_bce_loss.argtypes = [vp, vp, i64, vp, vp, i64, i64, C.c_float, vp, vp, i64, vp, vp, C.c_size_t, vp]
    L.c1d_mse_bce_loss.restype = C.c_int
    L.c1d_sgd_update.argtypes = [vp, vp, i64, C.c_float, vp]
    L.c1d_sgd_update.restype = C.c_int
    _lib = L
    return L
