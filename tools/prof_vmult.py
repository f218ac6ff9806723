"""ncu driver: three warm-up fp64 operator applications on the finest level, then one more.
  ncu -k regex:vmult_kernel -s 2 -c 1 python tools/prof_vmult.py [dim k levels]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_18982_b200 import ipmg  # noqa: E402

dim, k, nl = (int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (3, 4, 7)
h = ipmg.Handle(dim, k, nl, vcycle_precision=ipmg.FP32)
L = nl - 1
n = h.ndofs(L)
x = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
y = torch.empty_like(x)
for _ in range(4):
    h.vmult(L, x, y)
torch.cuda.synchronize()
