"""paper_2405_18982_b200 -- B200-native (sm_100a) hot path of arXiv 2405.18982
(Cui & Kanschat, *Multilevel Interior Penalty Methods on GPUs*): matrix-free
patch-wise SIPG operator, vertex-patch Schwarz smoother with fast-diagonalised
local solves, transfers, V-cycle and GMG-preconditioned CG, behind the C ABI of
include/ipmg.h (libipmg.so).  ``ipmg`` is the thin ctypes binding.
"""
from . import ipmg  # noqa: F401
from .ipmg import ADDITIVE, FP32, FP64, MULTIPLICATIVE, Handle, IpmgError, load, tables_1d  # noqa: F401
