"""A/B timing of the hot kernels for one library build (IPMG_LIB selects it):
smoother colour pass (fp32), operator apply (fp64), residual+restrict (fp32),
prolongation (fp32) on the finest level, and a full GMG-CG solve.

  IPMG_LIB=paper_2405_18982_b200/libipmg_x.so python tools/ab_kernels.py [dim k levels]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_18982_b200 import ipmg  # noqa: E402


def timeit(fn, reps=20, warm=3):
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


def main():
    dim, k, nl = (int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (2, 7, 10)
    coarse = tuple(int(c) for c in os.environ["AB_COARSE"].split(",")) if os.environ.get("AB_COARSE") else None
    h = ipmg.Handle(dim, k, nl, coarse_cells=coarse, vcycle_precision=ipmg.FP32)
    L = nl - 1
    n = h.ndofs(L)
    nc = h.ndofs(L - 1)
    x64 = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    y64 = torch.empty_like(x64)
    x32, b32, o32 = x64.float(), x64.float() * 0.5, torch.empty(n, device="cuda")
    rc = torch.empty(nc, device="cuda")
    res = {"lib": os.path.basename(ipmg.LIB_PATH), "dim": dim, "k": k, "ndofs": n}
    res["smooth_c0_ms"] = timeit(lambda: h.smooth_colour(L, None, b32, o32, 0))
    res["smooth_c1_ms"] = timeit(lambda: h.smooth_colour(L, x32, b32, o32, 1))
    res["smooth_c3_ms"] = timeit(lambda: h.smooth_colour(L, x32, b32, o32, (1 << dim) - 1))
    res["vmult64_ms"] = timeit(lambda: h.vmult(L, x64, y64))
    res["vmult32_ms"] = timeit(lambda: h.vmult(L, x32, o32))
    res["restrict32_ms"] = timeit(lambda: h.residual_restrict(L, x32, b32, rc))
    h64 = ipmg.Handle(dim, k, nl, coarse_cells=coarse, vcycle_precision=ipmg.FP64)
    rc64 = torch.empty(nc, dtype=torch.float64, device="cuda")
    b64 = x64 * 0.5
    res["restrict64_ms"] = timeit(lambda: h64.residual_restrict(L, x64, b64, rc64))
    h64.close()
    res["prolong32_ms"] = timeit(lambda: h.prolongate_add(L, rc, o32))
    hd = ipmg.Handle(dim, k, nl, coarse_cells=coarse, vcycle_precision=ipmg.FP32, kernel=ipmg.KERNEL_DIRICHLET)
    res["smooth_dir_c1_ms"] = timeit(lambda: hd.smooth_colour(L, x32, b32, o32, 1))
    xs = x32.clone()
    res["smooth_step_ms"] = timeit(lambda: h.smooth(L, xs, b32))
    res["smooth_dir_step_ms"] = timeit(lambda: hd.smooth(L, xs, b32))
    if os.environ.get("AB_QUICK"):   # kernels only (timing experiments with invalid numerics)
        print(json.dumps(res), flush=True)
        return
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    h.rhs(L, b)
    sol = torch.empty_like(b)
    info = {}

    def solve():
        info.update(h.cg_solve(b, sol))
    res["solve_ms"] = timeit(solve, reps=5, warm=2)
    res["iterations"] = info["iterations"]

    def gsolve(hh):
        info.update(hh.gmres_solve(b, sol))
    res["gmres_full_ms"] = timeit(lambda: gsolve(h), reps=3, warm=1)
    res["gmres_full_its"] = info["iterations"]
    res["gmres_dir_ms"] = timeit(lambda: gsolve(hd), reps=3, warm=1)
    res["gmres_dir_its"] = info["iterations"]
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
