"""GPU sweep driver: the reference's parameter sweep (proj/src/bench.cpp:242-334,
bench.hpp:24-58) measured through the B200 C ABI, plus roofline columns.

* ``SweepConfig``      bench.hpp:24-38 (widths, channels, filters, filter_sizes, dilations, batch,
                       iterations=20, warmup=3, precision, peak_flops, passes, seed); ``pairs`` adds
                       the BASELINE config-4 form (C = K on the diagonal instead of the C x K grid).
* ``run_sweep``        bench.cpp:246-303: the same loop nest (widths > channels > filters > filter
                       sizes > dilations > passes), ``skip_reason`` (bench.cpp:97-105) only in strict
                       mode because the GPU path accepts odd BF16 dims, ``meets_condition``
                       (bench.cpp:242-244), efficiency = flops / seconds / peak (bench.cpp:236-240).
                       seconds = mean of ``iterations`` CUDA-event-timed calls after ``warmup``, the
                       measure_kernel convention (bench.cpp:172-234).
* ``write_csv``        bench.cpp:305-334 byte-for-byte header and column order (13 fields), so the
                       reference's own ``parse_csv`` reads it; ``write_roofline_csv`` writes the
                       extra per-point roofline columns to a second file.
* ``summarize``        bench.cpp:372-405 (best / worst efficiency per pass, anomaly count).

Inputs are seeded on the device: BASELINE config 4 asks for i.i.d. N(0,1) data (x, dy) with
Kaiming-uniform weights; BF16 precision runs with BF16 storage, FP32 with FP32 storage.

CLI: ``python -m paper_2104_08002_b200.sweep --config4 --out sweep.csv`` (see ``--help``).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field

from . import conv as cv

CSV_HEADER = "N,C,K,S,d,Q,pass,seconds,flops,gflops,efficiency,meets_condition,threads"
ROOFLINE_HEADER = ("N,C,K,S,d,Q,precision,pass,algo,seconds,tflops,bytes,arith_intensity,bound,"
                   "roofline_seconds,roofline_frac,algo_roofline_frac")
PASSES = ("forward", "backward_data", "backward_weight")


@dataclass
class SweepConfig:
    widths: list = field(default_factory=list)
    channels: list = field(default_factory=list)
    filters: list = field(default_factory=list)
    filter_sizes: list = field(default_factory=list)
    dilations: list = field(default_factory=list)
    batch: int = 1
    iterations: int = 20
    warmup: int = 3
    precision: cv.Precision = cv.Precision.Fp32
    peak_flops: float = 0.0
    passes: tuple = PASSES
    threads: int = 1
    seed: int = 20260822
    pairs: bool = False      # C = K (BASELINE config 4) instead of the C x K grid
    strict: bool = False     # reference skip_reason for odd BF16 dims
    algo: str = "auto"       # "auto" or a forced c1d_algo ("direct", "tcgen05", "bf16x3")


@dataclass
class SweepRecord:
    n: int
    c: int
    k: int
    s: int
    d: int
    q: int
    pass_: str
    seconds: float
    flops: int
    gflops: float
    efficiency: float
    meets_condition: bool
    threads: int = 1
    # GPU extras (roofline file only)
    precision: str = ""
    algo: str = ""
    bytes: int = 0


@dataclass
class SweepResult:
    records: list = field(default_factory=list)
    skips: list = field(default_factory=list)


def meets_condition(s: int, q: int, c: int, k: int) -> bool:
    """bench.cpp:242-244."""
    return s >= 5 and q >= 1000 and c > 1 and k > 1


def skip_reason(n, c, k, s, d, q, precision) -> str:
    """bench.cpp:97-105 (only applied in strict mode)."""
    if precision != cv.Precision.Bf16:
        return ""
    width = q + d * (s - 1)
    if c % 2:
        return "bf16 needs even channels"
    if k % 2:
        return "bf16 needs even filters"
    if q % 2:
        return "bf16 needs an even output width"
    if width % 2:
        return "bf16 needs an even input width"
    return ""


def efficiency(flops: int, seconds: float, peak_flops: float) -> float:
    """bench.cpp:236-240."""
    if not seconds > 0:
        raise ValueError("seconds must be positive")
    if not peak_flops > 0:
        raise ValueError("peak_flops must be positive")
    return flops / seconds / peak_flops


def algorithmic_bytes(pass_: str, n, c, k, s, d, q, in_bytes: int) -> int:
    """Compulsory traffic per pass: inputs in their storage type, weights and
    outputs FP32."""
    w_in = q + d * (s - 1)
    if pass_ == "forward":
        return n * c * w_in * in_bytes + k * c * s * 4 + n * k * q * 4
    if pass_ == "backward_data":
        return n * k * q * in_bytes + k * c * s * 4 + n * c * w_in * 4
    return n * c * w_in * in_bytes + n * k * q * in_bytes + k * c * s * 4


def load_peaks(root: str | None = None) -> dict:
    """MEASURED_PEAKS.json (driver-written: HBM, BF16) plus profiles/fp32_peaks.json (measured here by
    tools/peaks_fp32.py: FFMA, TF32/FP32 cuBLAS)."""
    root = root or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        peaks = {"bf16_tflops": 1590.0, "hbm_gbs": 7000.0}
    try:
        with open(os.path.join(root, "profiles", "fp32_peaks.json")) as f:
            peaks.update(json.load(f))
    except (OSError, ValueError):
        pass
    return peaks


# BF16 products per credited FP32 product of the split paths (split.cu): six channel blocks for the
# conv-shaped passes, two launches of four blocks for backward-weight
SPLIT_PRODUCTS = {"forward": 6, "backward_data": 6, "backward_weight": 8}


def ffma_peak_flops(peaks: dict) -> float:
    """Measured FFMA roof (profiles/fp32_peaks.json), else the nominal 148 x 128 x 2 x 1.965 GHz."""
    v = peaks.get("ffma_fp32_tflops")
    return v * 1e12 if v else 148 * 128 * 2 * 1.965e9


def fp32_peak_flops(peaks: dict) -> float:
    """One fixed FP32 roof for every FP32 point, whatever algorithm ran it: the fastest FP32-exact
    method this GPU offers, max(measured FFMA, BF16 peak / 6 for the six-product split)."""
    return max(ffma_peak_flops(peaks), peaks.get("bf16_tflops", 1590.0) * 1e12 / 6.0)


def compute_peak_flops(algo: str, peaks: dict, pass_: str = "forward") -> float:
    """Roof of the kernel family a point ran on (FLOP/s of the credited 2NKCSQ work): BF16 tensor
    cores at the measured dense peak; the FP32 split over its BF16 products per FP32 product; the
    FFMA direct kernels at the measured FFMA peak. Reported beside the fixed roof as
    algo_roofline_frac."""
    tc = peaks.get("bf16_tflops", 1590.0) * 1e12
    if algo == "tcgen05":
        return tc
    if algo == "bf16x3":
        return tc / SPLIT_PRODUCTS.get(pass_, 6)
    return ffma_peak_flops(peaks)


def _iter_shapes(cfg: SweepConfig):
    for q in cfg.widths:
        for c in cfg.channels:
            ks = [c] if cfg.pairs else cfg.filters
            for k in ks:
                for s in cfg.filter_sizes:
                    for d in cfg.dilations:
                        yield q, c, k, s, d


def run_sweep(cfg: SweepConfig, progress=None, device="cuda") -> SweepResult:
    """bench.cpp:246-303 on the GPU."""
    import torch

    from . import _lib as L

    if not cfg.widths or not cfg.channels or not cfg.filter_sizes or not cfg.dilations:
        raise ValueError("sweep lists must be non-empty")
    if not cfg.pairs and not cfg.filters:
        raise ValueError("filters must be non-empty")
    if cfg.iterations < 1 or cfg.warmup < 0 or cfg.batch < 1:
        raise ValueError("bad iteration / batch counts")
    peaks = load_peaks()
    peak = cfg.peak_flops or peaks.get("bf16_tflops", 1590.0) * 1e12
    lib = L.lib()
    res = SweepResult()
    bf16 = cfg.precision == cv.Precision.Bf16
    dt = torch.bfloat16 if bf16 else torch.float32
    for q, c, k, s, d in _iter_shapes(cfg):
        n = cfg.batch
        reason = skip_reason(n, c, k, s, d, q, cfg.precision) if cfg.strict else ""
        if reason:
            res.skips.extend((n, c, k, s, d, q, ps, reason) for ps in cfg.passes)
            continue
        w_in = q + d * (s - 1)
        p = cv.ConvParams(c, k, s, d, cfg.precision)
        g = torch.Generator(device=device).manual_seed(cfg.seed)
        lim = math.sqrt(6.0 / (c * s))
        w = (torch.rand((k, c, s), device=device, generator=g) * 2 - 1) * lim
        x = torch.randn((n, c, w_in), device=device, generator=g).to(dt)
        dy = torch.randn((n, k, q), device=device, generator=g).to(dt)
        desc = cv.make_desc(p, n, w_in, L.DTYPE_BF16 if bf16 else L.DTYPE_F32, algo=cfg.algo)
        sp = torch.cuda.current_stream().cuda_stream
        outs = {"forward": torch.empty((n, k, q), device=device),
                "backward_data": torch.empty((n, c, w_in), device=device),
                "backward_weight": torch.empty((k, c, s), device=device)}
        # Weight packing is setup work, done before the clock starts as in the reference's
        # measure_kernel (bench.cpp:184-203): plans that take a prepacked image get one here.
        wdesc, wptr, keep = {}, {}, []
        for ps, pi in (("forward", L.PASS_FORWARD), ("backward_data", L.PASS_BACKWARD_DATA)):
            dsc = cv.make_desc(p, n, w_in, L.DTYPE_BF16 if bf16 else L.DTYPE_F32, algo=cfg.algo)
            nbytes = C.c_size_t(0)
            wdesc[ps], wptr[ps] = dsc, w.data_ptr()
            if ps in cfg.passes and lib.c1d_packed_weights_size(C.byref(dsc), pi, C.byref(nbytes)) == 0 and nbytes.value:
                img = torch.empty(nbytes.value, dtype=torch.uint8, device=device)
                cv._check(lib.c1d_pack_weights(1, C.byref(dsc), (C.c_int32 * 1)(pi), (C.c_void_p * 1)(w.data_ptr()),
                                               (C.c_void_p * 1)(img.data_ptr()), sp))
                dsc.flags |= L.FLAG_PREPACKED_WEIGHTS
                wptr[ps] = img.data_ptr()
                keep.append(img)
        calls = {
            "forward": lambda: lib.c1d_forward(C.byref(wdesc["forward"]), x.data_ptr(), wptr["forward"],
                                               outs["forward"].data_ptr(), None, 0, sp),
            "backward_data": lambda: lib.c1d_backward_data(C.byref(wdesc["backward_data"]), dy.data_ptr(),
                                                           wptr["backward_data"],
                                                           outs["backward_data"].data_ptr(), None, 0, sp),
            "backward_weight": lambda: lib.c1d_backward_weight(C.byref(desc), x.data_ptr(), dy.data_ptr(),
                                                               outs["backward_weight"].data_ptr(), None, 0, sp),
        }
        for ps in cfg.passes:
            fn = calls[ps]
            if cfg.algo != "auto" and fn() != 0:  # the forced algorithm does not support this shape
                res.skips.append((n, c, k, s, d, q, ps, f"algo {cfg.algo} unsupported"))
                continue
            for _ in range(cfg.warmup):
                cv._check(fn())
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * cfg.iterations)]
            for i in range(cfg.iterations):
                ev[2 * i].record()
                cv._check(fn())
                ev[2 * i + 1].record()
            torch.cuda.synchronize()
            secs = sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(cfg.iterations)) / cfg.iterations / 1e3
            flops = cv.conv_flops(p, n, q)
            rec = SweepRecord(n, c, k, s, d, q, ps, secs, flops, flops / secs / 1e9, efficiency(flops, secs, peak),
                              meets_condition(s, q, c, k), cfg.threads,
                              precision="bf16" if bf16 else "fp32",
                              algo=cfg.algo if cfg.algo != "auto" else cv.selected_algo(
                                  p, n, w_in, PASSES.index(ps), in_dtype=L.DTYPE_BF16 if bf16 else L.DTYPE_F32),
                              bytes=algorithmic_bytes(ps, n, c, k, s, d, q, 2 if bf16 else 4))
            res.records.append(rec)
            if progress:
                progress(rec)
        del x, dy, w, outs, keep
    return res


def _num(v) -> str:
    """std::to_chars-like shortest round-trip text for ints and doubles."""
    if isinstance(v, bool):
        return "1" if v else "0"
    if isinstance(v, int):
        return str(v)
    r = repr(float(v))
    return r[:-2] if r.endswith(".0") else r


def write_csv(records, path: str) -> None:
    """bench.cpp:305-334: the reference's 13-column schema (its parse_csv reads this file)."""
    lines = [CSV_HEADER]
    for r in records:
        lines.append(",".join([_num(r.n), _num(r.c), _num(r.k), _num(r.s), _num(r.d), _num(r.q), r.pass_,
                               _num(r.seconds), _num(r.flops), _num(r.gflops), _num(r.efficiency),
                               "1" if r.meets_condition else "0", _num(r.threads)]))
    with open(path, "w", newline="\n") as f:
        f.write("\n".join(lines) + "\n")


def parse_csv(path: str) -> list:
    """bench.cpp:336-370 (same header / field-count / value checks)."""
    with open(path) as f:
        rows = [ln.strip() for ln in f]
    if not rows or rows[0] != CSV_HEADER:
        raise ValueError(f"unexpected CSV header in {path}")
    out = []
    for ln in rows[1:]:
        if not ln:
            continue
        f = ln.split(",")
        if len(f) != 13:
            raise ValueError(f"CSV row with {len(f)} fields in {path}")
        if f[6] not in PASSES:
            raise ValueError(f"unknown pass {f[6]}")
        if f[11] not in ("0", "1"):
            raise ValueError("meets_condition must be 0 or 1")
        out.append(SweepRecord(int(f[0]), int(f[1]), int(f[2]), int(f[3]), int(f[4]), int(f[5]), f[6],
                               float(f[7]), int(f[8]), float(f[9]), float(f[10]), f[11] == "1", int(f[12])))
    return out


def roofline(rec: SweepRecord, peaks: dict) -> tuple[str, float, float]:
    """(bound, roofline seconds, fraction achieved) for one record against the fixed roof of its
    precision: the BF16 tensor peak, or fp32_peak_flops for every FP32 point."""
    roof = peaks.get("bf16_tflops", 1590.0) * 1e12 if rec.precision.lower().startswith("bf16") else fp32_peak_flops(peaks)
    t_c = rec.flops / roof
    t_m = rec.bytes / (peaks.get("hbm_gbs", 7000.0) * 1e9)
    bound = "compute" if t_c >= t_m else "hbm"
    t = max(t_c, t_m)
    return bound, t, t / rec.seconds


def algo_roofline_frac(rec: SweepRecord, peaks: dict) -> float:
    """The same fraction against the roof of the algorithm that actually ran (compute_peak_flops)."""
    t_c = rec.flops / compute_peak_flops(rec.algo, peaks, rec.pass_)
    t_m = rec.bytes / (peaks.get("hbm_gbs", 7000.0) * 1e9)
    return max(t_c, t_m) / rec.seconds


def write_roofline_csv(records, path: str, peaks: dict | None = None) -> None:
    peaks = peaks or load_peaks()
    lines = [ROOFLINE_HEADER]
    for r in records:
        bound, t, frac = roofline(r, peaks)
        lines.append(",".join([_num(r.n), _num(r.c), _num(r.k), _num(r.s), _num(r.d), _num(r.q), r.precision,
                               r.pass_, r.algo, _num(r.seconds), _num(r.flops / r.seconds / 1e12), _num(r.bytes),
                               _num(r.flops / max(r.bytes, 1)), bound, _num(t), _num(frac),
                               _num(algo_roofline_frac(r, peaks))]))
    with open(path, "w", newline="\n") as f:
        f.write("\n".join(lines) + "\n")


def summarize(result: SweepResult) -> str:
    """bench.cpp:372-405."""
    out = [f"{len(result.records)} measurements, {len(result.skips)} skipped"]
    for ps in PASSES:
        rs = [r for r in result.records if r.pass_ == ps]
        if not rs:
            continue
        best = max(rs, key=lambda r: r.efficiency)
        worst = min(rs, key=lambda r: r.efficiency)

        def shape(r):
            return f"N={r.n} C={r.c} K={r.k} S={r.s} d={r.d} Q={r.q}"

        out.append(f"{ps}: best efficiency {best.efficiency:g} ({shape(best)}, {best.gflops:g} GFLOP/s), "
                   f"worst {worst.efficiency:g} ({shape(worst)})")
    anomalies = sum(1 for r in result.records if r.efficiency > 1.0)
    if anomalies:
        out.append(f"{anomalies} rows exceed the declared peak (timing anomaly or wrong peak)")
    return "\n".join(out) + "\n"


def config4(precision: cv.Precision, iterations: int = 20, warmup: int = 3) -> SweepConfig:
    """BASELINE config 4: N=16, Q=20000, C=K in {16,32,64,128}, S in {3,9,25,51}, d in {1,2,4,8,16}."""
    return SweepConfig(widths=[20000], channels=[16, 32, 64, 128], filters=[], filter_sizes=[3, 9, 25, 51],
                       dilations=[1, 2, 4, 8, 16], batch=16, iterations=iterations, warmup=warmup,
                       precision=precision, pairs=True)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--config4", action="store_true", help="BASELINE config 4 (BF16 and FP32)")
    ap.add_argument("--precision", choices=["bf16", "fp32", "both"], default="both")
    ap.add_argument("--iterations", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--algo", choices=["auto", "direct", "tcgen05", "bf16x3"], default="auto",
                    help="force one algorithm (shapes it does not support are skipped)")
    ap.add_argument("--out", default="sweep.csv", help="reference-schema CSV; <out>.roofline.csv has the extras")
    args = ap.parse_args(argv)
    precs = {"bf16": [cv.Precision.Bf16], "fp32": [cv.Precision.Fp32],
             "both": [cv.Precision.Bf16, cv.Precision.Fp32]}[args.precision]
    allrec = SweepResult()
    for prec in precs:
        cfg = config4(prec, args.iterations, args.warmup)
        cfg.algo = args.algo
        r = run_sweep(cfg, progress=lambda rec: print(
            f"{rec.precision} C={rec.c} S={rec.s} d={rec.d} {rec.pass_:15s} {rec.algo:8s} "
            f"{rec.seconds * 1e6:10.1f} us {rec.gflops / 1e3:8.2f} TFLOP/s", flush=True))
        allrec.records.extend(r.records)
        allrec.skips.extend(r.skips)
    write_csv(allrec.records, args.out)
    root, _ = os.path.splitext(args.out)
    write_roofline_csv(allrec.records, root + ".roofline.csv")
    print(summarize(allrec), end="")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
