"""Profiling driver: one warm-up GMG-CG solve of the bench workload, then one
solve inside an NVTX range "timed" (for ncu --nvtx --nvtx-include timed/).

  python profiles/solve_once.py [--dim 3 --degree 4 --levels 8 --coarse 2,2,1] [--fp64-vcycle]

Defaults: the bench headline workload C4 (BASELINE.json configs[3]); C2 is
--dim 2 --degree 7 --levels 10 --coarse 2,2.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2405_18982_b200 import ipmg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--degree", type=int, default=4)
    ap.add_argument("--levels", type=int, default=8)
    ap.add_argument("--coarse", default="2,2,1")
    ap.add_argument("--fp64-vcycle", action="store_true")
    a = ap.parse_args()
    coarse = tuple(int(c) for c in a.coarse.split(","))[:a.dim]
    h = ipmg.Handle(a.dim, a.degree, a.levels, coarse_cells=coarse, vcycle_precision=ipmg.FP64 if a.fp64_vcycle else ipmg.FP32)
    L = a.levels - 1
    n = h.ndofs(L)
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    h.rhs(L, b)
    x = torch.empty_like(b)
    r = h.cg_solve(b, x)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("timed")
    r = h.cg_solve(b, x)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("dofs", n, "iterations", r["iterations"], "launches", h.launch_count())


if __name__ == "__main__":
    main()
