"""Additive smoother damping study (oracle, CPU): PCG iterations and nu over levels for
omega = 1/2^d (the default, reading A17), 1/lambda_max(QA) and 2/(lambda_max + 1), with
lambda_max by power iteration.  python tools/additive_damping_study.py"""
import sys, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import multigrid, krylov, assemble
from synth_inputs import uniform
def lam_max(S, n, it=30):
    v = uniform(n, seed=5); v/=np.linalg.norm(v)
    lam=0
    for _ in range(it):
        w = S.smooth_additive(np.zeros(n), S.A @ v, omega=1.0)   # Q A v
        lam = float(v @ w); v = w/np.linalg.norm(w)
    return lam
dim, k = 2, 2
for nl in (3,4,5,6):
    V = multigrid.VCycle(dim, k, nl, smoother="additive")
    L=nl-1; A=V.A64[L]; b=assemble.rhs(V.levels[L],k)
    lm = lam_max(V.S[L], A.shape[0])
    res=[]
    for om in (None, 1.0/lm, 2.0/(lm+1.0)):
        V.omega = om
        x,h,c = krylov.pcg(A,b,V,rtol=1e-8,max_it=300)
        n=len(h)-1; nu = -8*n/np.log10(h[-1]/h[0])
        res.append((om, n, round(nu,2)))
    print(nl, 'lam_max %.3f'%lm, res, flush=True)
