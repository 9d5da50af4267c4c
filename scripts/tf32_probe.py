"""How tcgen05 kind::tf32 reads fp32 operand bits (TG_UMMA_EXP=4: one MMA on the
raw tiles).  A = 1 + 2^-11 + 2^-12 (between tf32 neighbours 1 and 1 + 2^-10),
B = 1, K = 32: C = 32 * tf32(A) -> 32 (truncation) or 32 * (1 + 2^-10) (rounding).
Also a value just below a tie and negative values."""
import ctypes as C
import os
import sys

os.environ["TG_UMMA_EXP"] = "4"
import torch  # noqa: E402

sys.path.insert(0, os.getcwd())
from paper_2503_13795_b200 import _lib  # noqa: E402

M, N, K = 128, 128, 32
for a in [1 + 2**-11 + 2**-12, 1 + 2**-11, 1 + 2**-12, -(1 + 2**-11 + 2**-12), 1 + 2**-10 + 2**-11]:
    A = torch.full((M * K,), a, device="cuda")
    B = torch.ones(K * N, device="cuda")
    Cm = torch.zeros(M * N, device="cuda")
    assert _lib.lib.tg_gemm(1, 1, M, N, K, C.c_void_p(A.data_ptr()), K, 1, C.c_void_p(B.data_ptr()), N, 1,
                            C.c_void_p(Cm.data_ptr()), N, 0, None) == 0
    torch.cuda.synchronize()
    v = Cm[0].item() / K
    print(f"a = {a!r}: tf32(a) as used = {v!r}  trunc={abs(v) == 1 or abs(v) == 1 + 2**-10 and abs(a) > 1 + 2**-10}"
          f"  (trunc -> {1.0 if abs(a) < 1 + 2**-10 else 1 + 2**-10}, diff from a {v - a:+.3e})")
