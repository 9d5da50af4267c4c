"""tcgen05 GEMM time vs K at fixed M, N: intercept = per-CTA fixed cost, slope = per-k-tile cost."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2503_13795_b200 import _lib  # noqa: E402

M, N = 1024, 65536
for K in (32, 128, 512, 1024, 2048):
    A = torch.randn(M * K, device="cuda")
    B = torch.randn(K * N, device="cuda")
    Cm = torch.empty(M * N, device="cuda")
    f = lambda: _lib.lib.tg_gemm(1, 1, M, N, K, C.c_void_p(A.data_ptr()), K, 1, C.c_void_p(B.data_ptr()), N, 1,
                                 C.c_void_p(Cm.data_ptr()), N, 0, None)
    f(); f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    ctas = (M // 128) * (N // 128)
    print(f"K={K:5d} ms={ms:.3f}  per-CTA-wave us={ms * 1e3 / (ctas / 148):.2f}  k-tiles={K // 32}", flush=True)
