"""tg_gemm (tcgen05 3xTF32) normwise error vs fp64 over odd shapes / majors /
value distributions.  Usage: python scripts/gemm_shapes_err.py"""
import ctypes as C
import itertools
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2503_13795_b200 import _lib  # noqa: E402

torch.manual_seed(0)
worst = 0
for (M, N, K), ak, bn, dist in itertools.product(
        [(65, 1024, 64), (64, 1024, 64), (192, 1024, 64), (64, 1024, 256), (256, 1024, 64), (64, 64, 16384),
         (65, 64, 1024), (200, 4096, 30), (1024, 512, 784), (96, 333, 70)],
        [True, False], [True, False], ["randn", "unif", "big", "mixed"]):
    def gen(n):
        if dist == "randn": return torch.randn(n, device="cuda")
        if dist == "unif": return torch.rand(n, device="cuda")
        if dist == "big": return torch.randn(n, device="cuda") * 1e4
        return torch.randn(n, device="cuda") * torch.exp(torch.randn(n, device="cuda") * 3)
    A, B = gen(M * K), gen(K * N)
    lda = K if ak else M
    ldb = N if bn else K
    Cm = torch.zeros(M * N, device="cuda")
    st = _lib.lib.tg_gemm(1, 1, M, N, K, C.c_void_p(A.data_ptr()), lda, int(ak), C.c_void_p(B.data_ptr()), ldb, int(bn),
                          C.c_void_p(Cm.data_ptr()), N, 0, None)
    torch.cuda.synchronize()
    Am = A.view(M, K) if ak else A.view(K, M).t()
    Bm = B.view(K, N) if bn else B.view(N, K).t()
    ref = Am.double() @ Bm.double()
    err = float((Cm.view(M, N).double() - ref).norm() / ref.norm())
    worst = max(worst, err)
    flag = "  <-- BAD" if err > 2e-6 else ""
    print(f"M{M} N{N} K{K} a_kmaj={ak} b_nmaj={bn} {dist:6s} status={st} err={err:.2e}{flag}", flush=True)
print("worst", worst)
