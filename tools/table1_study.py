"""Table 1 readings study on the GPU.

The paper's Table 1: 3D, full kernel, GMRES to 1e-8 preconditioned by
one GMG V-cycle, f == 1, nu = -8 n / log10(||r_n|| / ||r_0||).  The printed counts FALL with
the level L; ours (reading A2/A5/A7, right-preconditioned GMRES) rise.  This tool runs the
full kernel under combinations of the readings the paper leaves open:

  post    : post-smoothing colour order, reverse (symmetric V) | forward       (reading A7)
  pen     : interior penalty scale x boundary penalty scale:
              "1x1"   gamma = 2k(k+1)/h on every face                         (reading A2)
              "1x0.5" one-sided boundary penalty k(k+1)/h
              "0.5x2" interior k(k+1)/h (average of the two one-sided values), boundary 2k(k+1)/h
  solver  : "right" right-preconditioned GMRES, true residual (library ipmg_gmres_solve)
            "left"  left-preconditioned GMRES, preconditioned residual norm (reading A22 probe;
                    Arnoldi on P^{-1}A over the library's vmult / V-cycle, vector algebra in
                    torch fp64 -- a study harness, not the product path)
            "cg"    the library's PCG (the north star's solver; needs post = reverse)

Rows are written for n_levels = L (reading A5, 2^L cells per direction); the SPEC reading
2^{L+1} is the same data shifted by one row (tools/render_table1_study.py does both).

  python tools/table1_study.py --out profiles/tables/r02_study.jsonl [--levels 2,..] [--degrees ..]
"""
import argparse
import itertools
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_18982_b200 import ipmg  # noqa: E402

PENALTIES = {"1x1": (1.0, 1.0), "1x0.5": (1.0, 0.5), "0.5x2": (0.5, 2.0)}


def left_gmres(h, L, b, rtol=1e-8, max_it=60):
    """Left-preconditioned GMRES (MGS, no restart) on P^{-1} A x = P^{-1} b, x0 = 0,
    history of the preconditioned residual estimates."""
    r0 = torch.empty_like(b)
    h.vcycle(b, r0)
    beta0 = float(torch.linalg.vector_norm(r0))
    V = [r0 / beta0]
    H = [[0.0] * (max_it + 1) for _ in range(max_it)]   # H[j][i]
    cs, sn = [0.0] * max_it, [0.0] * max_it
    g = [0.0] * (max_it + 1)
    g[0] = beta0
    hist = [beta0]
    t = torch.empty_like(b)
    w = torch.empty_like(b)
    for j in range(max_it):
        h.vmult(L, V[j], t)
        h.vcycle(t, w)
        for i in range(j + 1):
            H[j][i] = float(torch.dot(w, V[i]))
            w.sub_(V[i], alpha=H[j][i])
        H[j][j + 1] = float(torch.linalg.vector_norm(w))
        V.append(w / H[j][j + 1])
        for i in range(j):
            a = cs[i] * H[j][i] + sn[i] * H[j][i + 1]
            H[j][i + 1] = -sn[i] * H[j][i] + cs[i] * H[j][i + 1]
            H[j][i] = a
        den = math.hypot(H[j][j], H[j][j + 1])
        cs[j], sn[j] = H[j][j] / den, H[j][j + 1] / den
        H[j][j] = den
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        hist.append(abs(g[j + 1]))
        if abs(g[j + 1]) <= rtol * beta0:
            break
    n = len(hist) - 1
    return {"iterations": n, "nu": -8.0 * n / math.log10(hist[-1] / hist[0]), "history": hist}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", default="2,3,4,5,6")
    ap.add_argument("--degrees", default="3,4,5,6,7")
    ap.add_argument("--posts", default="reverse,forward")
    ap.add_argument("--pens", default="1x1,1x0.5,0.5x2")
    ap.add_argument("--solvers", default="right,left,cg")
    ap.add_argument("--fp64", action="store_true")
    ap.add_argument("--max-dofs", type=float, default=3e8)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = open(a.out, "a") if a.out else None
    for L, k in itertools.product([int(v) for v in a.levels.split(",")], [int(v) for v in a.degrees.split(",")]):
        if (2 ** L) ** 3 * (k + 1) ** 3 > a.max_dofs:
            continue
        for post, pen in itertools.product(a.posts.split(","), a.pens.split(",")):
            ps, bs = PENALTIES[pen]
            h = ipmg.Handle(3, k, L, vcycle_precision=ipmg.FP64 if a.fp64 else ipmg.FP32,
                            post_smooth_reverse=1 if post == "reverse" else 0, penalty_scale=ps,
                            boundary_penalty_scale=bs)
            n = h.ndofs(L - 1)
            b = torch.empty(n, dtype=torch.float64, device="cuda")
            h.rhs(L - 1, b)
            x = torch.empty_like(b)
            for solver in a.solvers.split(","):
                if solver == "cg" and post != "reverse":
                    continue
                if solver == "right":
                    r = h.gmres_solve(b, x, rtol=1e-8, max_it=100)
                elif solver == "cg":
                    r = h.cg_solve(b, x, rtol=1e-8, max_it=100)
                else:
                    r = left_gmres(h, L - 1, b)
                rec = {"L": L, "k": k, "dofs": n, "post": post, "pen": pen, "solver": solver,
                       "vcycle": "fp64" if a.fp64 else "fp32", "nu": r["nu"], "iterations": r["iterations"]}
                line = json.dumps(rec)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
                    out.flush()
            h.close()
            del b, x
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
