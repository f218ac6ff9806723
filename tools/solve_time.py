"""Time-to-solution of the mixed GMG-CG solve (CUDA events, one warm-up solve, then
`reps` timed solves) on the bench headline workload C4 or a smaller level count:

  python tools/solve_time.py [levels] [reps]     (levels 8 = C4, 1.05 B dofs)

Used for A/B runs of environment switches (IPMG_RZ_FUSE, IPMG_OP3, IPMG_PAIR3)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_18982_b200 import ipmg  # noqa: E402

nl = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
h = ipmg.Handle(3, 4, nl, coarse_cells=(2, 2, 1), vcycle_precision=ipmg.FP32)
L = nl - 1
n = h.ndofs(L)
b = torch.empty(n, dtype=torch.float64, device="cuda")
h.rhs(L, b)
x = torch.empty_like(b)
info = h.cg_solve(b, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    info = h.cg_solve(b, x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(json.dumps({"levels": nl, "dofs": n, "ms": round(ms, 3), "gdofs": round(n / ms / 1e6, 4),
                  "iterations": info["iterations"], "env": {k: v for k, v in os.environ.items() if k.startswith("IPMG_")}}))
