"""Where does the e2e step time go?  cfg2 pipeline variants, event timed,
plus the host cost of one pipeline call (small batch: host-bound)."""
import json
import os
import time
import torch
import paper_2503_13795_b200 as tg

desc = tg.build_model("moons").describe()
prog = tg.Program(desc)
st = torch.cuda.current_stream()
out = {}


def run(b, n, depth):
    os.environ["TG_PIPE_DEPTH"] = str(depth)
    x, _ = tg.synth_batch("moons", batch=b, seed=1, n_inputs=desc.n_inputs)
    P = torch.tensor(desc.param_values(), device="cuda")
    xh = torch.from_numpy(x).pin_memory()
    lh = torch.empty(b, dtype=torch.float64).pin_memory()
    pl = prog.pipeline(b, P, st)
    for _ in range(20):
        pl.step(xh, None, lh, 0.01)
    pl.sync()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    e0.record(st)
    for _ in range(n):
        t = time.perf_counter()
        pl.step(xh, None, lh, 0.01)
        ts.append((time.perf_counter() - t) * 1e6)
    pl.join(st)
    e1.record(st)
    torch.cuda.synchronize()
    ts.sort()
    return {"gpu_us_per_step": e0.elapsed_time(e1) / n * 1e3, "call_us_p50": ts[n // 2], "call_us_p99": ts[int(n * .99)],
            "call_us_max": ts[-1]}


for graph in ("0", "1"):
    os.environ["TG_PIPE_GRAPH"] = graph
    for depth in (2, 4):
        out[f"g{graph}_b65536_d{depth}_n1000"] = run(65536, 1000, depth)
    out[f"g{graph}_b1024_d4_n1000"] = run(1024, 1000, 4)
for k, v in out.items():
    print(k, {a: round(b, 1) for a, b in v.items()})
