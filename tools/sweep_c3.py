"""BASELINE.json configs[2] (C3): 3D Poisson SIPG k = 1..7 at ~130M dofs on one
B200 -- operator vmult and one multiplicative smoother step, fp64 and fp32,
GDoF/s and the fraction of the roofline that bounds each,
plus one mixed-precision GMG-CG solve per degree.

  python tools/sweep_c3.py [--out gpurun_out/c3.jsonl] [--degrees 1,2,...]

Sizes: power-of-two boxes closest to 2^27 dofs.
Timing: CUDA events on the handle's stream, 3 warm-up + 10 timed calls; all
vectors are larger than L2.  Peaks: HBM from MEASURED_PEAKS.json; FP32/FP64
CUDA-core peaks measured live (ipmg_alu_peak: FFMA2 / DFMA), as in bench.py.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2405_18982_b200 import ipmg  # noqa: E402

# k -> (coarse cells, levels): finest = coarse * 2^(levels-1) cells per direction
SIZES = {1: ((2, 2, 2), 8), 2: ((2, 1, 1), 8), 3: ((2, 2, 2), 7), 4: ((2, 2, 1), 7),
         5: ((2, 1, 1), 7), 6: ((2, 2, 2), 6), 7: ((2, 2, 2), 6)}


def vmult_flops_per_dof(k):
    """sum-factorised 3D SIPG operator, 14(k+1) + 48 flops/dof."""
    return 14 * (k + 1) + 48


def timeit(stream, fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ALU = {}   # measured CUDA-core peaks (TF/s) per precision, filled in main()


def roof(bytes_, flops, ms, prec, peaks):
    hbm = peaks["hbm_gbs"]
    alu = ALU[prec]
    t_b, t_f = bytes_ / (hbm * 1e9), flops / (alu * 1e12)
    if t_b >= t_f:
        return {"bound": "hbm", "achieved": bytes_ / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": t_b / (ms * 1e-3)}
    return {"bound": "alu", "achieved": flops / (ms * 1e-3) / 1e12, "peak": alu, "unit": "TFLOP/s",
            "frac": t_f / (ms * 1e-3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c3.jsonl"))
    ap.add_argument("--degrees", default="1,2,3,4,5,6,7")
    a = ap.parse_args()
    peaks, src = bench.measured_peaks()
    ALU["fp32"] = ipmg.alu_peak(0, "ffma2")
    ALU["fp64"] = ipmg.alu_peak(0, "dfma")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    out = open(a.out, "w")
    for k in [int(v) for v in a.degrees.split(",")]:
        cc, nl = SIZES[k]
        h = ipmg.Handle(3, k, nl, coarse_cells=cc, vcycle_precision=ipmg.FP32)
        s = h.stream
        L = nl - 1
        n, cells, _ = h.level_info(L)
        res = {"k": k, "cells": cells, "ndofs": n, "peak_source": src}
        x64 = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
        y64 = torch.empty_like(x64)
        b64 = torch.empty_like(x64)
        h.rhs(L, b64)
        for prec, x, y, b in (("fp64", x64, y64, b64), ("fp32", x64.float(), y64.float(), b64.float())):
            es = 8 if prec == "fp64" else 4
            ms = timeit(s, lambda: h.vmult(L, x, y))
            res["vmult_" + prec] = {"ms": ms, "gdofs": n / (ms * 1e-3) / 1e9,
                                    "roofline": roof(2 * es * n, vmult_flops_per_dof(k) * n, ms, prec, peaks)}
            xs = x.clone()
            ms = timeit(s, lambda: h.smooth(L, xs, b))
            nb = 2 ** 3 * 3 * es * n
            res["smooth_" + prec] = {"ms": ms, "gdofs": n / (ms * 1e-3) / 1e9,
                                     "roofline": roof(nb, 2 ** 3 * bench.smoother_flops_per_dof(3, k) * n, ms, prec,
                                                      peaks)}
            del xs
        sol = torch.empty_like(b64)
        info = {}

        def solve():
            info.update(h.cg_solve(b64, sol))
        ms = timeit(s, solve, reps=3, warm=1)
        res["solve_mixed"] = {"ms": ms, "gdofs": n / (ms * 1e-3) / 1e9, "iterations": info["iterations"],
                              "nu": info["nu"]}
        out.write(json.dumps(res) + "\n")
        out.flush()
        print(json.dumps(res), flush=True)
        h.close()
        del x64, y64, b64, sol
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
