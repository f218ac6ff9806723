"""BASELINE.json configs other than the bench line, on one B200:

  C1  2D SIPG k=2, 8x8 cells, 3-level GMG-CG, fp64 V-cycle (the oracle-sized case)
  C4  3D SIPG k=4, (0,1)^2 x (0,1/2), T_0 = 2x2x1, 8 levels = 256x256x128 cells,
      1,048,576,000 dofs -- the multi-GPU configuration, here its 1-GPU point
  C5  3D SIPG k=3, unit cube, 4..8 levels: additive vs multiplicative smoother,
      fp32 vs fp64 V-cycle -- CG iterations, nu and time to solution
  T   throughput vs problem size (the paper's Fig. 12/13 analogue, NEXT-4):
      operator vmult (fp64) and smoother step (fp32) GDoF/s for 3D k=4, 4..8 levels

  python tools/configs.py [--only C1,C4,C5,T] [--out gpurun_out/configs.jsonl]

Every solve: f == 1, x0 = 0, ||r|| <= 1e-8 ||b||; times are CUDA
events around complete solves after one warm-up solve (setup excluded).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_18982_b200 import ipmg  # noqa: E402


def ev_time(fn, reps, warm=1):
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def solve_case(dim, k, nl, coarse=None, h0=0.5, solver="cg", reps=3, **kw):
    h = ipmg.Handle(dim, k, nl, coarse_cells=coarse, h0=h0, **kw)
    L = nl - 1
    n = h.ndofs(L)
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    h.rhs(L, b)
    x = torch.empty_like(b)
    info = {}
    fn = h.cg_solve if solver == "cg" else h.gmres_solve

    def go():
        info.update(fn(b, x, rtol=1e-8, max_it=200))
    ms = ev_time(go, reps)
    res = {"dim": dim, "k": k, "levels": nl, "dofs": n, "solver": solver, "ms": ms, "gdofs": n / (ms * 1e-3) / 1e9,
           "iterations": info["iterations"], "nu": info["nu"], "converged": info["converged"]}
    h.close()
    del b, x
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C4,C5,T")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.jsonl"))
    a = ap.parse_args()
    only = set(a.only.split(","))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    out = open(a.out, "w")

    def emit(d):
        out.write(json.dumps(d) + "\n")
        out.flush()
        print(json.dumps(d), flush=True)

    if "C1" in only:
        emit(dict(config="C1", **solve_case(2, 2, 3, vcycle_precision=ipmg.FP64, reps=20)))
    if "C4" in only:
        emit(dict(config="C4 (1 GPU)", **solve_case(3, 4, 8, coarse=(2, 2, 1), h0=0.5, vcycle_precision=ipmg.FP32,
                                                    reps=2)))
    if "C5" in only:
        for nl in (4, 5, 6, 7, 8):
            for sm, smn in ((ipmg.MULTIPLICATIVE, "multiplicative"), (ipmg.ADDITIVE, "additive")):
                for vp, vpn in ((ipmg.FP32, "fp32"), (ipmg.FP64, "fp64")):
                    r = solve_case(3, 3, nl, smoother=sm, vcycle_precision=vp, reps=2 if nl >= 7 else 3)
                    emit(dict(config="C5", smoother=smn, vcycle=vpn, **r))
    if "T" in only:
        for nl in (3, 4, 5, 6, 7, 8):
            h = ipmg.Handle(3, 4, nl, vcycle_precision=ipmg.FP32)
            L = nl - 1
            n = h.ndofs(L)
            x = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
            y = torch.empty_like(x)
            reps = max(3, min(200, int(2e9 // n)))
            t_v = ev_time(lambda: h.vmult(L, x, y), reps, warm=3)
            xf, bf = x.float(), x.float()
            t_s = ev_time(lambda: h.smooth(L, xf, bf), max(3, reps // 8), warm=2)
            emit({"config": "T", "dim": 3, "k": 4, "levels": nl, "dofs": n,
                  "vmult_fp64_gdofs": n / (t_v * 1e-3) / 1e9, "smooth_fp32_gdofs": n / (t_s * 1e-3) / 1e9,
                  "vmult_ms": t_v, "smooth_ms": t_s})
            h.close()
            del x, y, xf, bf
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
