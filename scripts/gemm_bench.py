"""tg_gemm throughput on cfg5's dense-layer shapes: SIMT (engine 0) vs
tcgen05 3xTF32 (engine 1; TG_UMMA_TMA=0 selects the register-staged kernel),
plus the max normwise error vs an fp64 product."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2503_13795_b200 import _lib  # noqa: E402

S = int(os.environ.get("GB_S", "65536"))
# (name, M, N, K, a_kmaj, b_nmaj): forward Z = W X, input adjoint dX = W^T dZ, weight grad dW = dZ X^T
SHAPES_CFG4 = [("c4_m64_k64", 64, S, 64, True, True), ("c4_m64_k256", 64, S, 256, True, True),
               ("c4_m192_k64", 192, S, 64, True, True), ("c4_m256_k64", 256, S, 64, True, True)]
SHAPES = [("fwd_l1", 1024, S, 784, True, True), ("fwd_l2", 1024, S, 1024, True, True),
          ("dx_l2", 1024, S, 1024, False, True), ("dw_l2", 1024, 1024, S, True, False),
          ("dw_l1", 1024, 784, S, True, False)]


def mat(M, N, K, a_kmaj, b_nmaj):
    A = torch.randn(M * K, device="cuda")
    B = torch.randn(K * N, device="cuda")
    return A, B


def run(engine, M, N, K, a_kmaj, b_nmaj, A, B, Cm, reps):
    lda = K if a_kmaj else M
    ldb = N if b_nmaj else K
    f = lambda: _lib.lib.tg_gemm(1, engine, M, N, K, C.c_void_p(A.data_ptr()), lda, int(a_kmaj), C.c_void_p(B.data_ptr()),
                                 ldb, int(b_nmaj), C.c_void_p(Cm.data_ptr()), N, 0, None)
    for _ in range(2):
        assert f() == 0, _lib.lib.tg_last_error()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


SHAPES_SHORTK = [("c3_l1_k30", 200, 262144, 30, True, True), ("c5_dx3_k10", 1024, 1048576, 10, False, True),
                 ("c5_fwd3_m10", 10, 1048576, 1024, True, True), ("c5_dw3_m10", 10, 1024, 1048576, True, False),
                 ("c4_m64_k64", 64, 524288, 64, True, True), ("c4_m64_k256", 64, 524288, 256, True, True)]
out = {}
if os.environ.get("GB_SET") == "cfg4":
    SHAPES = SHAPES_CFG4
if os.environ.get("GB_SET") == "shortk":
    SHAPES = SHAPES_SHORTK
for name, M, N, K, ak, bn in SHAPES:
    A, B = mat(M, N, K, ak, bn)
    Am = A.view(M, K) if ak else A.view(K, M).t()
    Bm = B.view(K, N) if bn else B.view(N, K).t()
    ref = (Am.double() @ Bm.double())
    Cm = torch.empty(M * N, device="cuda")
    row = {}
    for eng in tuple(int(e) for e in os.environ.get("GB_ENGINES", "0,1").split(",")):
        ms = run(eng, M, N, K, ak, bn, A, B, Cm, 5)
        err = float((Cm.view(M, N).double() - ref).norm() / ref.norm())
        row[f"e{eng}"] = {"ms": round(ms, 3), "tflops": round(2 * M * N * K / ms / 1e9, 1), "err": f"{err:.1e}"}
    out[name] = row
    print(name, json.dumps(row), flush=True)
    del A, B, Cm, ref
    torch.cuda.empty_cache()
