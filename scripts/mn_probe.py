"""Probe of the TMA-fed tcgen05 GEMM on one 128x128x32 tile per operand-major
combination; each case in a fresh process so a device fault stays isolated."""
import ctypes as C
import os
import subprocess
import sys

CHILD = r'''
import ctypes as C, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2503_13795_b200 import _lib
M, N, K = 128, 128, 32
ak, bn = bool(int(sys.argv[1])), bool(int(sys.argv[2]))
torch.manual_seed(0)
A = torch.randn(M * K, device="cuda"); B = torch.randn(K * N, device="cuda")
Am = A.view(M, K) if ak else A.view(K, M).t()
Bm = B.view(K, N) if bn else B.view(N, K).t()
ref = Am.double() @ Bm.double()
Cm = torch.zeros(M * N, device="cuda")
st = _lib.lib.tg_gemm(1, 1, M, N, K, C.c_void_p(A.data_ptr()), K if ak else M, int(ak), C.c_void_p(B.data_ptr()),
                      N if bn else K, int(bn), C.c_void_p(Cm.data_ptr()), N, 0, None)
try:
    torch.cuda.synchronize()
    err = float((Cm.view(M, N).double() - ref).norm() / ref.norm())
    print("status", st, f"err {err:.2e}", "zeros" if float(Cm.abs().max()) == 0 else "")
except Exception as e:
    print("status", st, "CUDA:", str(e).splitlines()[0])
'''
for ak, bn in [(1, 0), (1, 1), (0, 0), (0, 1)]:
    r = subprocess.run([sys.executable, "-c", CHILD, str(ak), str(bn)], capture_output=True, text=True, timeout=120)
    print(os.environ.get("TG_MN_VARIANT", "0"), "a_kmaj", ak, "b_nmaj", bn, (r.stdout + r.stderr).strip().splitlines()[-1:])
