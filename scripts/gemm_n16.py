import ctypes as C, os, sys, itertools
import torch
sys.path.insert(0, os.getcwd())
from paper_2503_13795_b200 import _lib
torch.manual_seed(0)
for M, N, K, ldb, ak in itertools.product([256, 192, 64], [16, 64, 200], [64, 256], [None, 128, 1024], [True, False]):
    ldb_ = ldb or N
    if ldb_ < N: continue
    A = torch.randn(M * K, device="cuda")
    B = torch.randn(K * ldb_, device="cuda") * 3
    lda = K if ak else M
    Cm = torch.zeros(M * N, device="cuda")
    st = _lib.lib.tg_gemm(1, 1, M, N, K, C.c_void_p(A.data_ptr()), lda, int(ak), C.c_void_p(B.data_ptr()), ldb_, 1,
                          C.c_void_p(Cm.data_ptr()), N, 0, None)
    torch.cuda.synchronize()
    Am = A.view(M, K) if ak else A.view(K, M).t()
    Bm = B.view(K, ldb_)[:, :N]
    ref = Am.double() @ Bm.double()
    err = float((Cm.view(M, N).double() - ref).norm() / ref.norm())
    print(f"M{M} N{N} K{K} ldb{ldb_} akmaj{ak} st{st} err {err:.2e}" + ("  <-- BAD" if err > 2e-6 else ""), flush=True)
