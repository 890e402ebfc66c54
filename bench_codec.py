"""Codec-only roofline (the paper's "Store" and "MatMul" tasks): 512M 16-bit
fixed-point numbers (256M 32-bit records of two 16-bit fields) encoded from fp32
by the standalone codec (qmpm_encode), round-to-nearest and dithered, and decoded back
(qmpm_decode).  HBM-bound: bytes moved per record = 8 (two fp32 in) + 4 (record out)
[+ 4 (dither key in)].  One JSON line with GB/s and the fraction of the measured copy
bandwidth (MEASURED_PEAKS.json).

    python bench_codec.py [--records 268435456] [--reps 10]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    from paper_2207_04658_b200 import qmpm, schemes

    torch.cuda.set_device(0)
    n = args.records
    R = 1.0
    sch = dict(dim=3, material="elastic", rounding="dither", seed=schemes.DITHER_SEED,
               fields=[dict(attr="x", comp=c, kind="fixed", frac_bits=15, range=R, offset=0.0) for c in range(2)])
    g = torch.Generator(device="cuda").manual_seed(0)
    vals = (torch.rand((n, 2), device="cuda", generator=g) * 2 - 1) * (R * 0.999)
    keys = torch.arange(n, device="cuda", dtype=torch.int32)
    words = torch.empty((n, 1), device="cuda", dtype=torch.int32)
    back = torch.empty_like(vals)
    peaks = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak = json.load(open(peaks))["hbm_gbs"] if os.path.exists(peaks) else 6650.0
    stream = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.reps):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / args.reps

    out = {"task": "Store (P:796, P:807): 2 x 16-bit fixed-point per 32-bit record", "records": n, "values": 2 * n,
           "peak_gbs": peak, "results": {}}
    for name, k, sch_r in [("encode_rne", None, schemes.with_rounding(sch, "rne")),
                           ("encode_dither", keys, sch)]:
        ms = timed(lambda: qmpm.encode(sch_r, vals, words, keys=k, step=1, stream=stream))
        b = n * (8 + 4 + (4 if k is not None else 0))
        out["results"][name] = {"ms": ms, "GBps": b / ms / 1e6, "frac": b / ms / 1e6 / peak, "bytes_per_record": b / n}
    ms = timed(lambda: qmpm.decode(sch, words, back, stream=stream))
    b = n * 12
    out["results"]["decode"] = {"ms": ms, "GBps": b / ms / 1e6, "frac": b / ms / 1e6 / peak, "bytes_per_record": 12}
    err = float((back - vals).abs().max())
    out["max_abs_error_over_delta"] = err / (R * 2.0 ** -15)
    del vals, back, words, keys
    torch.cuda.empty_cache()
    # MatMul: 3x3 matrices of 16-bit fixed point (144 bits -> 5-word records),
    # each multiplied by a constant 3x3 and re-encoded, RNE and dithered
    nm = args.records
    msch = dict(dim=3, material="elastic", rounding="dither", seed=schemes.DITHER_SEED,
                fields=[dict(attr="F", comp=c, kind="fixed", frac_bits=15, range=2.0, offset=0.0) for c in range(9)])
    _, Wm, _ = qmpm.layout(msch)
    mv = (torch.rand((nm, 9), device="cuda", generator=g) * 2 - 1) * 0.9
    win = torch.empty((nm, Wm), device="cuda", dtype=torch.int32)
    wout = torch.empty_like(win)
    qmpm.encode(schemes.with_rounding(msch, "rne"), mv, win, stream=stream)
    del mv
    torch.cuda.empty_cache()
    mkeys = torch.arange(nm, device="cuda", dtype=torch.int32)
    A = [[0.6, -0.8, 0.0], [0.8, 0.6, 0.0], [0.0, 0.0, 1.0]]  # a rotation: values stay in range
    for name, k, s in [("matmul_rne", None, schemes.with_rounding(msch, "rne")), ("matmul_dither", mkeys, msch)]:
        ms = timed(lambda: qmpm.codec_matmul3(s, win, A, wout, keys=k, step=1, stream=stream))
        b = nm * (2 * 4 * Wm + (4 if k is not None else 0))
        out["results"][name] = {"ms": ms, "GBps": b / ms / 1e6, "frac": b / ms / 1e6 / peak,
                                "bytes_per_record": b / nm, "matrices": nm}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
