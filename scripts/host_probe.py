"""Host cost of one tg_pipeline_step call (small batch, so the host is the bottleneck)."""
import ctypes as C
import os
import time
import torch
import paper_2503_13795_b200 as tg
from paper_2503_13795_b200._lib import lib

desc = tg.build_model("moons").describe()
prog = tg.Program(desc)
b = 1024
x, _ = tg.synth_batch("moons", batch=b, seed=1, n_inputs=desc.n_inputs)
for graph in ("0", "1"):
    os.environ["TG_PIPE_GRAPH"] = graph
    os.environ["TG_PIPE_TRACE"] = "1"
    P = torch.tensor(desc.param_values(), device="cuda")
    xh = torch.from_numpy(x).pin_memory()
    lh = torch.empty(b, dtype=torch.float64).pin_memory()
    pl = prog.pipeline(b, P)
    n = 2000
    for _ in range(50):
        pl.step(xh, None, lh, 0.01)
    pl.sync()
    t = time.perf_counter()
    for _ in range(n):
        pl.step(xh, None, lh, 0.01)
    wrap = (time.perf_counter() - t) / n * 1e6
    pl.sync()
    a = (pl._h, C.c_void_p(xh.data_ptr()), None, C.c_void_p(lh.data_ptr()), C.c_double(0.01))
    t = time.perf_counter()
    for _ in range(n):
        lib.tg_pipeline_step(*a)
    direct = (time.perf_counter() - t) / n * 1e6
    pl.sync()
    print(f"graph={graph}: python wrapper {wrap:.1f} us/call, direct ctypes {direct:.1f} us/call", flush=True)
    del pl
    torch.cuda.synchronize()
