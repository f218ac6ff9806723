"""Exercise every kernel of libipmg.so on small meshes (2D and 3D, k = 1..7, both
precisions): operator, every smoother colour (with x and from zero), additive and
Dirichlet/clamped smoothers, residual+restriction, prolongation, coarse solve, V-cycle,
CG and GMRES -- the driver for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck):

  compute-sanitizer --tool racecheck python tools/sanitize.py [--quick]
IPMG_PAIR3=1 forces the 3D patch-pair smoother for every degree."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_18982_b200 import ipmg  # noqa: E402


def run(dim, k, nl, kernel=ipmg.KERNEL_FULL, smoother=0):
    for vp in (ipmg.FP64, ipmg.FP32):
        h = ipmg.Handle(dim, k, nl, vcycle_precision=vp, kernel=kernel, smoother=smoother)
        L = nl - 1
        n = h.ndofs(L)
        nc = h.ndofs(L - 1)
        for dt in (torch.float64, torch.float32):
            x = torch.rand(n, dtype=dt, device="cuda")
            b = torch.rand(n, dtype=dt, device="cuda")
            o = torch.empty_like(x)
            if kernel == ipmg.KERNEL_FULL:
                h.vmult(L, x, o)
            for c in range(2 ** dim):
                h.smooth_colour(L, x, b, o, c)
            h.smooth_colour(L, None, b, o, 0)
            rc = torch.empty(nc, dtype=dt, device="cuda")
            if kernel == ipmg.KERNEL_FULL:
                h.residual_restrict(L, x, b, rc)
                h.prolongate_add(L, rc, o)
        r = torch.rand(n, dtype=torch.float64, device="cuda")
        z = torch.empty_like(r)
        h.vcycle(r, z)
        bb = torch.empty_like(r)
        h.rhs(L, bb)
        h.cg_solve(bb, z, rtol=1e-6, max_it=20)
        if kernel == ipmg.KERNEL_FULL and smoother == 0:
            h.gmres_solve(bb, z, rtol=1e-6, max_it=20)
        torch.cuda.synchronize()
        h.close()


def main():
    quick = "--quick" in sys.argv
    degs = (1, 4, 7) if quick else range(1, 8)
    for k in degs:
        run(2, k, 3)
        run(3, k, 3 if k <= 4 else 2)
        print("k=%d full ok" % k, flush=True)
    run(2, 3, 3, smoother=1)
    run(3, 3, 2, smoother=1)
    for kern in (ipmg.KERNEL_DIRICHLET,):
        run(2, 3, 3, kernel=kern)
        run(3, 4, 2, kernel=kern)
    print("sanitize driver done", flush=True)


if __name__ == "__main__":
    main()
