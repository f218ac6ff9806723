"""Kernel-variant equivalence on the GPU: the staged kernels the library picks by degree
(op3 fp64 operator; patch-pair smoother incl. its zero-start instantiation,
4.8; the r.z fused into the V-cycle's last colour pass, §6) against the kernels they
replace (vmult_kernel, smooth_kernel, the separate dot pass).  Each arm runs in its own
process because the switches (IPMG_OP3, IPMG_PAIR3, IPMG_RZ_FUSE) are read once per
process; both arms use the same seeded inputs (synth_inputs-style uniform vectors).

Bars (largest element difference over the largest magnitude): the operator is the same
arithmetic in another order (fp64, 1e-13); the fp32 colour passes and
V-cycle 1e-5 (the north star's fp32 bar); CG iterations +-1 and solutions 1e-6 (the
mixed-precision bar of the oracle parity tests: the arms' fp32 V-cycles round differently).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import json, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2405_18982_b200 import ipmg
dim, k, nl = 3, int(sys.argv[2]), int(sys.argv[3])
out = sys.argv[4]
h = ipmg.Handle(dim, k, nl, coarse_cells=(2, 2, 1), vcycle_precision=ipmg.FP32)
L = nl - 1
n = h.ndofs(L)
g = torch.Generator().manual_seed(7)
x64 = (torch.rand(n, dtype=torch.float64, generator=g) * 2 - 1).cuda()
b64 = (torch.rand(n, dtype=torch.float64, generator=g) * 2 - 1).cuda()
res = {}
y = torch.empty_like(x64)
h.vmult(L, x64, y)
res["vmult"] = y.cpu().numpy()
x32, b32 = x64.float(), b64.float()
o = torch.empty_like(x32)
for c in (0, 1, 3, 7):
    h.smooth_colour(L, x32, b32, o, c)
    res["smooth%d" % c] = o.cpu().numpy()
h.smooth_colour(L, None, b32, o, 0)
res["smooth_zero"] = o.cpu().numpy()
z = torch.empty_like(x64)
h.vcycle(b64, z)
res["vcycle"] = z.cpu().numpy()
rhs = torch.empty_like(x64)
h.rhs(L, rhs)
sol = torch.empty_like(x64)
info = h.cg_solve(rhs, sol, rtol=1e-8, max_it=50)
res["cg"] = sol.cpu().numpy()
res["its"] = np.array([info["iterations"]])
np.savez(out, **res)
'''


def _run(tmp_path, env_extra, k, nl, tag):
    script = tmp_path / "arm.py"
    script.write_text(SCRIPT)
    out = str(tmp_path / ("%s.npz" % tag))
    env = dict(os.environ)
    env.update(env_extra)
    p = subprocess.run([sys.executable, str(script), ROOT, str(k), str(nl), out], env=env,
                       stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:]
    return dict(np.load(out))


def _rel_max(a, b):
    scale = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) / scale


@pytest.mark.parametrize("k,nl", [(4, 4), (2, 4), (6, 3)], ids=["k4", "k2", "k6"])
def test_staged_kernels_match_legacy(tmp_path, k, nl):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    new = _run(tmp_path, {"IPMG_OP3": "1", "IPMG_PAIR3": "1", "IPMG_RZ_FUSE": "1"}, k, nl, "new")
    old = _run(tmp_path, {"IPMG_OP3": "0", "IPMG_PAIR3": "0", "IPMG_RZ_FUSE": "0"}, k, nl, "old")
    assert _rel_max(new["vmult"], old["vmult"]) <= 1e-13
    for key in ("smooth0", "smooth1", "smooth3", "smooth7", "smooth_zero", "vcycle"):
        assert _rel_max(new[key], old[key]) <= 1e-5, key
    assert abs(int(new["its"][0]) - int(old["its"][0])) <= 1
    assert _rel_max(new["cg"], old["cg"]) <= 1e-6
