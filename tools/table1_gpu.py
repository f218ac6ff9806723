"""The paper's Table 1 / Table 2 (Dirichlet column) fractional iteration counts on the GPU
(PAPER.md:284-300): 3D, full kernel, GMRES to 1e-8 preconditioned by the GMG
V-cycle, f == 1, unit cube, reading A5 (row L = 2^L cells per direction).

  python tools/table1_gpu.py [--levels 2,3,4,5] [--degrees 3,4,5,6,7] [--fp64]
Prints one JSON line per (L, k) with nu (GPU), the paper's value and the
iteration count.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_18982_b200 import ipmg  # noqa: E402

TABLE1 = {}   # tests/golden/table1_full_kernel.txt
for line in open(os.path.join(ROOT, "tests", "golden", "table1_full_kernel.txt")):
    line = line.split("#", 1)[0].split()
    if line:
        for j, v in enumerate(line[1:]):
            if v != "---":
                TABLE1[(int(line[0]), 3 + j)] = float(v)


TABLE2D, TABLE2C = {}, {}   # tests/golden/table2_dirichlet_clamped.txt
for line in open(os.path.join(ROOT, "tests", "golden", "table2_dirichlet_clamped.txt")):
    line = line.split("#", 1)[0].split()
    if line:
        for j, v in enumerate(line[1:6]):
            if v != "---":
                TABLE2D[(int(line[0]), 3 + j)] = float(v)
        for j, v in enumerate(line[6:11]):
            if v != "---":
                TABLE2C[(int(line[0]), 3 + j)] = float(v)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", default="2,3,4,5")
    ap.add_argument("--degrees", default="3,4,5,6,7")
    ap.add_argument("--fp64", action="store_true")
    ap.add_argument("--forward-post", action="store_true", help="post-smoothing in forward colour order")
    ap.add_argument("--penalty", type=float, default=1.0, help="penalty_scale (reading A2 probe)")
    ap.add_argument("--kernel", choices=["full", "dirichlet", "clamped"], default="full")
    a = ap.parse_args()
    for L in [int(v) for v in a.levels.split(",")]:
        for k in [int(v) for v in a.degrees.split(",")]:
            h = ipmg.Handle(3, k, L, vcycle_precision=ipmg.FP64 if a.fp64 else ipmg.FP32,
                            post_smooth_reverse=0 if a.forward_post else 1, penalty_scale=a.penalty,
                            kernel={"full": ipmg.KERNEL_FULL, "dirichlet": ipmg.KERNEL_DIRICHLET,
                                    "clamped": ipmg.KERNEL_CLAMPED}[a.kernel])
            n = h.ndofs(L - 1)
            b = torch.empty(n, dtype=torch.float64, device="cuda")
            h.rhs(L - 1, b)
            x = torch.empty_like(b)
            r = h.gmres_solve(b, x, rtol=1e-8, max_it=100)
            paper = {"full": TABLE1, "dirichlet": TABLE2D, "clamped": TABLE2C}[a.kernel].get((L, k))
            print(json.dumps({"L": L, "k": k, "dofs": n, "nu": r["nu"], "paper": paper, "kernel": a.kernel,
                              "iterations": r["iterations"], "converged": r["converged"],
                              "vcycle": "fp64" if a.fp64 else "fp32", "post": "forward" if a.forward_post else "reverse",
                              "penalty_scale": a.penalty}),
                  flush=True)
            h.close()
            del b, x
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
