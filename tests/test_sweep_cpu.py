"""Sweep driver host logic (paper_2104_08002_b200/sweep.py) against the reference's sweep code
(proj/src/bench.cpp:236-405): CSV schema read back by the reference's own parse_csv, the loop
helpers, roofline arithmetic. No GPU needed."""
import ctypes as C
import os

import pytest

import oracle
from paper_2104_08002_b200 import conv as cv
from paper_2104_08002_b200 import sweep as sw


def _records():
    recs = []
    for i, ps in enumerate(sw.PASSES):
        flops = cv.conv_flops(cv.ConvParams(64, 64, 51, 8), 16, 20000)
        secs = 1.234567e-4 * (i + 1)
        recs.append(sw.SweepRecord(16, 64, 64, 51, 8, 20000, ps, secs, flops, flops / secs / 1e9,
                                   sw.efficiency(flops, secs, 1.6e15), sw.meets_condition(51, 20000, 64, 64), 1,
                                   precision="bf16", algo="tcgen05",
                                   bytes=sw.algorithmic_bytes(ps, 16, 64, 64, 51, 8, 20000, 2)))
    return recs


def test_csv_roundtrip_and_header(tmp_path):
    path = str(tmp_path / "s.csv")
    recs = _records()
    sw.write_csv(recs, path)
    with open(path) as f:
        assert f.readline().strip() == "N,C,K,S,d,Q,pass,seconds,flops,gflops,efficiency,meets_condition,threads"
    back = sw.parse_csv(path)
    assert [(r.pass_, r.seconds, r.flops, r.gflops, r.efficiency) for r in back] == \
           [(r.pass_, r.seconds, r.flops, r.gflops, r.efficiency) for r in recs]


def test_reference_parse_csv_accepts_our_file(tmp_path):
    path_lib = oracle.ref_library_path()
    if path_lib is None:
        pytest.skip("oracle/_ref not built")
    lib = C.CDLL(path_lib)
    lib.ref_parse_csv_count.restype = C.c_int64
    lib.ref_parse_csv_count.argtypes = [C.c_char_p]
    path = str(tmp_path / "s.csv")
    sw.write_csv(_records(), path)
    assert lib.ref_parse_csv_count(path.encode()) == 3
    bad = str(tmp_path / "bad.csv")
    with open(bad, "w") as f:
        f.write("N,C\n1,2\n")
    assert lib.ref_parse_csv_count(bad.encode()) == -1


def test_loop_helpers_match_reference():
    # bench.cpp:242-244, 97-105, 236-240
    assert sw.meets_condition(5, 1000, 2, 2) and not sw.meets_condition(3, 20000, 64, 64)
    assert not sw.meets_condition(51, 999, 64, 64) and not sw.meets_condition(51, 20000, 1, 64)
    assert sw.skip_reason(1, 15, 16, 3, 1, 100, cv.Precision.Bf16) == "bf16 needs even channels"
    assert sw.skip_reason(1, 16, 15, 3, 1, 100, cv.Precision.Bf16) == "bf16 needs even filters"
    assert sw.skip_reason(1, 16, 16, 3, 1, 101, cv.Precision.Bf16) == "bf16 needs an even output width"
    assert sw.skip_reason(1, 16, 16, 2, 1, 100, cv.Precision.Bf16) == "bf16 needs an even input width"
    assert sw.skip_reason(1, 15, 15, 3, 1, 101, cv.Precision.Fp32) == ""
    with pytest.raises(ValueError):
        sw.efficiency(1, 0.0, 1.0)
    cfg = sw.config4(cv.Precision.Bf16)
    shapes = list(sw._iter_shapes(cfg))
    assert len(shapes) == 4 * 4 * 5 and all(c == k for _, c, k, _, _ in shapes)
    assert shapes[0] == (20000, 16, 16, 3, 1) and shapes[-1] == (20000, 128, 128, 51, 16)


def test_roofline_columns(tmp_path):
    peaks = {"bf16_tflops": 1600.0, "hbm_gbs": 6500.0}
    r = _records()[0]
    bound, t, frac = sw.roofline(r, peaks)
    assert bound == "compute" and t == pytest.approx(r.flops / 1.6e15) and frac == pytest.approx(t / r.seconds)
    small = sw.SweepRecord(16, 16, 16, 3, 1, 20000, "forward", 1e-4, cv.conv_flops(cv.ConvParams(16, 16, 3, 1), 16,
                                                                                      20000), 0, 0, False, 1,
                           precision="bf16", algo="tcgen05",
                           bytes=sw.algorithmic_bytes("forward", 16, 16, 16, 3, 1, 20000, 2))
    assert sw.roofline(small, peaks)[0] == "hbm"
    path = str(tmp_path / "r.csv")
    sw.write_roofline_csv([r, small], path, peaks)
    rows = open(path).read().strip().split("\n")
    assert rows[0] == sw.ROOFLINE_HEADER and len(rows) == 3
    assert len(rows[1].split(",")) == len(sw.ROOFLINE_HEADER.split(","))
    assert "Summary" not in sw.summarize(sw.SweepResult(records=[r]))
    assert os.path.exists(path)
