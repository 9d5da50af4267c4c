"""Normwise error of tg_gemm (dW shape, K-major x K-major) vs K: SIMT vs tcgen05."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2503_13795_b200 import _lib  # noqa: E402

M, N = 256, 256
for K in (512, 2048, 8192, 32768, 131072):
    torch.manual_seed(0)
    A = torch.randn(M * K, device="cuda")
    B = torch.randn(N * K, device="cuda")
    ref = A.view(M, K).double() @ B.view(N, K).double().t()
    row = []
    for eng in (0, 1):
        Cm = torch.empty(M * N, device="cuda")
        assert _lib.lib.tg_gemm(1, eng, M, N, K, C.c_void_p(A.data_ptr()), K, 1, C.c_void_p(B.data_ptr()), K, 0,
                                C.c_void_p(Cm.data_ptr()), N, 0, None) == 0
        torch.cuda.synchronize()
        row.append(float((Cm.view(M, N).double() - ref).norm() / ref.norm()))
    # positive data (no cancellation): exposes a biased accumulation
    Ap, Bp = A.abs(), B.abs()
    refp = Ap.view(M, K).double() @ Bp.view(N, K).double().t()
    for eng in (0, 1):
        Cm = torch.empty(M * N, device="cuda")
        _lib.lib.tg_gemm(1, eng, M, N, K, C.c_void_p(Ap.data_ptr()), K, 1, C.c_void_p(Bp.data_ptr()), K, 0,
                         C.c_void_p(Cm.data_ptr()), N, 0, None)
        torch.cuda.synchronize()
        row.append(float(((Cm.view(M, N).double() - refp) / refp).mean()))
    print(f"K={K:7d}  randn err simt {row[0]:.1e} umma {row[1]:.1e} | positive mean rel bias simt {row[2]:+.1e} umma {row[3]:+.1e}",
          flush=True)
