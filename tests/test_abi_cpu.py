"""CPU-side checks of the C ABI: the library loads, exports every symbol include/c1d.h declares,
and host-side validation mirrors the reference's error classes (no GPU needed)."""
import ctypes as C
import subprocess

import pytest

from paper_2104_08002_b200 import _lib as L
from paper_2104_08002_b200 import conv as cv


def test_library_exports_every_declared_symbol():
    names = L.exported_symbols()
    assert len(names) >= 12
    lib = L.lib()
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert f" T {n}" in out, n


def test_api_version():
    assert L.lib().c1d_api_version() == 1


def _desc(**kw):
    base = dict(n=1, c=5, k=4, s=3, d=3, w_in=23, precision=0, in_dtype=0, algo=0, flags=0, block_w=64)
    base.update(kw)
    return L.Desc(**base)


def test_output_width_and_too_narrow():
    q = C.c_int64()
    assert L.lib().c1d_output_width(C.byref(_desc()), C.byref(q)) == L.OK and q.value == 17
    assert L.lib().c1d_output_width(C.byref(_desc(c=1, k=1, s=5, d=4, w_in=16)), C.byref(q)) == L.ERR_TOO_NARROW
    assert L.lib().c1d_output_width(C.byref(_desc(c=1, k=1, s=5, d=4, w_in=100)), C.byref(q)) == L.OK
    assert q.value == 84
    # geometry through the Python mirror (test_conv.cpp:53-62)
    assert cv.output_width(cv.ConvParams(5, 4, 3, 3), 23) == 17
    assert cv.output_width(cv.ConvParams(1, 1, 1, 7), 10) == 10
    with pytest.raises(cv.TooNarrow):
        cv.output_width(cv.ConvParams(1, 1, 5, 4), 16)
    s = cv.conv_shapes(cv.ConvParams(5, 4, 3, 3), 23)
    assert (s.q, s.receptive, s.w_padded) == (17, 6, 23)


def test_conv_flops():
    assert L.lib().c1d_conv_flops(C.byref(_desc(n=1, c=15, k=15, s=51, d=8, w_in=60400))) == 1377000000
    assert cv.conv_flops(cv.ConvParams(64, 64, 9, 1), 64, 20000) == 94371840000


def test_shape_mismatch_on_nonpositive_params():
    q = C.c_int64()
    for bad in (dict(c=0), dict(k=0), dict(s=0), dict(d=0)):
        assert L.lib().c1d_output_width(C.byref(_desc(**bad)), C.byref(q)) == L.ERR_SHAPE_MISMATCH
    assert b"positive" in L.lib().c1d_last_error_message()


def test_strict_bf16_odd_dims_mirror_reference():
    q = C.c_int64()
    strict = dict(precision=1, flags=L.FLAG_STRICT_BF16_DIMS)
    # odd channels / odd filters / odd widths (test_conv.cpp:297-315, acceptance.cpp:499-526)
    assert L.lib().c1d_output_width(C.byref(_desc(c=3, k=4, s=5, d=2, w_in=16, **strict)), C.byref(q)) == L.ERR_ODD_DIMS
    assert L.lib().c1d_output_width(C.byref(_desc(c=4, k=3, s=5, d=2, w_in=16, **strict)), C.byref(q)) == L.ERR_ODD_DIMS
    assert L.lib().c1d_output_width(C.byref(_desc(c=4, k=4, s=5, d=1, w_in=15, **strict)), C.byref(q)) == L.ERR_ODD_DIMS
    assert L.lib().c1d_output_width(C.byref(_desc(c=4, k=4, s=5, d=1, w_in=20, block_w=33, **strict)),
                                    C.byref(q)) == L.ERR_ODD_DIMS
    # default (non-strict) accepts odd dims in BF16: the documented deviation
    assert L.lib().c1d_output_width(C.byref(_desc(c=15, k=15, s=51, d=8, w_in=60400, precision=1)),
                                    C.byref(q)) == L.OK


def test_algo_selection_host_side():
    a = C.c_int()
    # FP32 precision at d=8 runs the split-BF16 tensor path, elsewhere the direct kernels
    assert L.lib().c1d_selected_algo(C.byref(_desc(c=15, k=15, s=51, d=8, w_in=60400)), 0, C.byref(a)) == L.OK
    assert a.value == L.ALGO_BF16X3
    assert L.lib().c1d_selected_algo(C.byref(_desc(c=15, k=15, s=51, d=3, w_in=60150)), 0, C.byref(a)) == L.OK
    assert a.value == L.ALGO_DIRECT
    # BF16 precision at d=8 runs tcgen05
    assert L.lib().c1d_selected_algo(C.byref(_desc(c=64, k=64, s=51, d=8, w_in=60400, precision=1)), 2,
                                     C.byref(a)) == L.OK
    assert a.value == L.ALGO_TCGEN05
    # forced direct is always allowed
    assert L.lib().c1d_selected_algo(C.byref(_desc(precision=1, algo=L.ALGO_DIRECT)), 2, C.byref(a)) == L.OK
    assert a.value == L.ALGO_DIRECT


def test_workspace_query():
    b = C.c_size_t()
    d = _desc(n=4, c=15, k=15, s=51, d=8, w_in=60400)
    for p in (0, 1, 2):
        assert L.lib().c1d_workspace_size(C.byref(d), p, C.byref(b)) == L.OK
        assert b.value > 0


def test_packed_weight_layout_checks():
    import torch

    w = torch.arange(3 * 2 * 4, dtype=torch.float32).reshape(3, 2, 4)
    pf = cv.pack_weights_forward(w)
    pb = cv.pack_weights_backward(w)
    assert tuple(pf.data.shape) == (4, 3, 2) and tuple(pb.data.shape) == (4, 2, 3)
    assert torch.equal(cv.unpack_weights(pf), w) and torch.equal(cv.unpack_weights(pb), w)
    # slot t of the backward layout holds original tap S-1-t transposed (tensor.hpp:63-66)
    assert torch.equal(pb.data[0], w[:, :, 3].t())
    with pytest.raises(cv.ShapeMismatch):
        cv._weights_kcs(pb, cv.ConvParams(2, 3, 4, 1), cv.WeightLayout.ForwardSKC)


def test_ctypes_structs_match_the_header(tmp_path):
    """The ctypes mirrors (_lib.Desc / FwdGlue / BwdGlue) have the C structs' size and field offsets
    (compiled against include/c1d.h with the host compiler)."""
    structs = {"c1d_desc": L.Desc, "c1d_fwd_glue": L.FwdGlue, "c1d_bwd_glue": L.BwdGlue}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{L.HEADER_PATH}"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(src)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        cname, field, val = line.split()
        got[(cname, field)] = int(val)
    for cname, py in structs.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)
