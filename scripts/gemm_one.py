"""One tg_gemm call (for ncu captures).  Usage: gemm_one.py M N K a_kmaj b_nmaj [engine]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2503_13795_b200 import _lib  # noqa: E402

M, N, K, ak, bn = (int(v) for v in sys.argv[1:6])
eng = int(sys.argv[6]) if len(sys.argv) > 6 else 1
A = torch.randn(M * K, device="cuda")
B = torch.randn(K * N, device="cuda")
Cm = torch.empty(M * N, device="cuda")
for _ in range(2):
    assert _lib.lib.tg_gemm(1, eng, M, N, K, C.c_void_p(A.data_ptr()), K if ak else M, ak, C.c_void_p(B.data_ptr()),
                            N if bn else K, bn, C.c_void_p(Cm.data_ptr()), N, 0, None) == 0
torch.cuda.synchronize()
print("ok")
