"""The oracle's fractional iteration counts for Table 1 on the oracle-
reachable block, under the readings DESIGN.md adopts for the table (A2 penalty, A5 level index,
A7 reverse post-smoothing, A22 left-preconditioned GMRES reporting the preconditioned residual),
fp64 V-cycle.  Calls only oracle/ (test infrastructure; the stored values are the oracle's,
never the CUDA path's).  Writes tests/golden/table1_oracle.txt:

  python tools/oracle_table1.py [--cells 2:3,2:4,...] > tests/golden/table1_oracle.txt
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import assemble, krylov, multigrid  # noqa: E402

BLOCK = [(2, 3), (2, 4), (2, 5), (2, 6), (2, 7), (3, 3), (3, 4), (3, 5), (4, 3)]


def nu_cell(L, k, solver="left"):
    V = multigrid.VCycle(3, k, L)           # row L: 2^L cells per direction (reading A5)
    A = V.A64[L - 1]
    b = assemble.rhs(V.levels[L - 1], k)
    fn = krylov.gmres_left if solver == "left" else krylov.gmres
    x, hist, conv = fn(A, b, V, rtol=1e-8)
    assert conv
    return krylov.nu(hist), len(hist) - 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", default=",".join("%d:%d" % c for c in BLOCK))
    a = ap.parse_args()
    print("# Table 1 cells computed by the ORACLE (tools/oracle_table1.py): 3D full kernel, f == 1,")
    print("# left-preconditioned GMRES to 1e-8 on the preconditioned residual (reading A22),")
    print("# symmetric V-cycle (A7), fp64, row L = 2^L cells per direction (A5).")
    print("# columns: L k nu_left n_left nu_right(true residual) n_right seconds")
    for c in a.cells.split(","):
        L, k = map(int, c.split(":"))
        t0 = time.time()
        nl, il = nu_cell(L, k, "left")
        nr, ir = nu_cell(L, k, "right")
        print("%d %d %.6f %d %.6f %d %.1f" % (L, k, nl, il, nr, ir, time.time() - t0), flush=True)


if __name__ == "__main__":
    main()
