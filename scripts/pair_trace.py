"""k-tile timeline of one CTA pair of k_umma_pair under full load (profiling build only:
`make prof` -> build_prof/libtg_prof.so; the product library has no trace code).

Runs tg_gemm on one of cfg5's shapes so that every SM pair is busy, then reads the SM-clock
stamps the leader CTA of the middle N tile left for its first 96 k-tiles:
  0 TMA issue, 1 `full` seen by converter warp 2, 2 that warp's conv arrive,
  3 `conv` (all 32 arrivals) seen by the MMA warp, 4 MMAs issued + committed,
  5 drain of the accumulation group two back finished.
Prints per-k-tile deltas in ns (cycles / the SM clock nvidia-smi reports).
Usage: python scripts/pair_trace.py [fwd|dw]"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import torch

lib = C.CDLL(os.path.join(os.getcwd(), "build_prof", "libtg_prof.so"))
lib.tg_gemm.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p,
                        C.c_size_t, C.c_int, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
lib.tg_last_error.restype = C.c_char_p
lib.tg_debug_pair_trace.argtypes = [C.c_void_p]

which = sys.argv[1] if len(sys.argv) > 1 else "fwd"
S = 262144
if which == "fwd":      # Z = W X: A K-major weights, B MN-major activations
    M, N, K, ak, bn = 1024, S, 1024, 1, 1
else:                   # dW = dZ X^T: both operands K-major streams (one tile per cluster, 16 clusters)
    M, N, K, ak, bn = 1024, 1024, S, 1, 0
A = torch.randn(M * K, device="cuda")
B = torch.randn(K * N, device="cuda")
Cm = torch.empty(M * N, device="cuda")
lda = K if ak else M
ldb = N if bn else K
for _ in range(3):
    st = lib.tg_gemm(1, 1, M, N, K, A.data_ptr(), lda, ak, B.data_ptr(), ldb, bn, Cm.data_ptr(), N, 0, None)
    assert st == 0, lib.tg_last_error()
torch.cuda.synchronize()
mhz = float(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True).stdout.split()[0])
tr = np.zeros((7, 96), dtype=np.int64)
assert lib.tg_debug_pair_trace(tr.ctypes.data) == 0
T = min(96, (K + 31) // 32)
ns = lambda c: c * 1e3 / mhz
print(f"shape {which}: M {M} N {N} K {K}; SM clock {mhz:.0f} MHz (read after the run); {T} k-tiles traced")
print("  t  issue->full  full->conv  conv(w2)->all32  all32->issued  issued(t)->issue(t+3)  period  [drain]")
rows = []
for t in range(T):
    e = tr[:6, t]
    nxt = tr[0, t + 3] if t + 3 < T else 0
    per = tr[4, t] - tr[4, t - 1] if t else 0
    row = (ns(e[1] - e[0]), ns(e[2] - e[1]), ns(e[3] - e[2]), ns(e[4] - e[3]), ns(nxt - e[4]) if nxt else float("nan"), ns(per))
    rows.append(row)
    dr = f"  drain end +{ns(e[5] - e[2]):.0f}" if e[5] else ""
    print(f"{t:3d}  {row[0]:9.0f}  {row[1]:9.0f}  {row[2]:13.0f}  {row[3]:12.0f}  {row[4]:18.0f}  {row[5]:7.0f}{dr}")
r = np.array(rows[8:T - 4])
print("mean over k-tiles 8..T-5 (ns): issue->full %.0f, full->conv(w2) %.0f, conv(w2)->all32 seen %.0f, all32->MMAs issued %.0f, "
      "issued(t)->TMA issue(t+3) %.0f, period %.0f" % tuple(np.nanmean(r, axis=0)))
m = tr[6]
print("tile (ns from kernel entry): set-up done %.0f, first TMA issue %.0f, first MMAs issued %.0f, last MMAs issued %.0f, "
      "last drain done %.0f, tile staged %.0f, stores issued %.0f, exit %.0f"
      % (ns(m[1] - m[0]), ns(tr[0, 0] - m[0]), ns(tr[4, 0] - m[0]), ns(tr[4, T - 1] - m[0]), ns(m[2] - m[0]), ns(m[3] - m[0]),
         ns(m[4] - m[0]), ns(m[5] - m[0])))
