"""ncu driver: two warm-up calls, then one finest-level smoother colour pass
with x = 0 (colour 0, no face traces) and one with x (colour 1).
  ncu -k regex:smooth_kernel -s 4 -c 2 python tools/prof_smooth.py [dim k levels]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_18982_b200 import ipmg  # noqa: E402

dim, k, nl = (int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (2, 7, 10)
coarse = tuple(int(c) for c in os.environ["AB_COARSE"].split(",")) if os.environ.get("AB_COARSE") else None
h = ipmg.Handle(dim, k, nl, coarse_cells=coarse, vcycle_precision=ipmg.FP32)
L = nl - 1
n = h.ndofs(L)
x = torch.empty(n, device="cuda").uniform_(-1, 1)
b = torch.empty_like(x).uniform_(-1, 1)
o = torch.empty_like(x)
for _ in range(3):
    h.smooth_colour(L, None, b, o, 0)
    h.smooth_colour(L, x, b, o, 1)
torch.cuda.synchronize()
