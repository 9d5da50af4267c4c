"""tcgen05 GEMM time for M=1024, N=65536, K=1024 under each operand layout."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2503_13795_b200 import _lib  # noqa: E402

M, N, K = 1024, 65536, 1024
A = torch.randn(M * K, device="cuda")
B = torch.randn(K * N, device="cuda")
Cm = torch.empty(M * N, device="cuda")
for ak, bn in [(1, 1), (1, 0), (0, 1), (0, 0)]:
    f = lambda: _lib.lib.tg_gemm(1, 1, M, N, K, C.c_void_p(A.data_ptr()), K if ak else M, ak, C.c_void_p(B.data_ptr()),
                                 N if bn else K, bn, C.c_void_p(Cm.data_ptr()), N, 0, None)
    f(); f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"a_kmaj={ak} b_nmaj={bn}  {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.1f} TF/s", flush=True)
