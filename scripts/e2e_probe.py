"""e2e (tg_pipeline_step) vs device-only train_step for cfg2, under env variants."""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, time, torch, paper_2503_13795_b200 as tg
b = 65536
desc = tg.build_model("moons").describe()
prog = tg.Program(desc)
x, _ = tg.synth_batch("moons", batch=b, seed=1, n_inputs=desc.n_inputs)
st = torch.cuda.current_stream()
P = torch.tensor(desc.param_values(), device="cuda")
xh = torch.from_numpy(x).pin_memory()
lh = torch.empty(b, dtype=torch.float64).pin_memory()
pl = prog.pipeline(b, P, st)
def timeit(fn, n=400):
    for _ in range(20): fn()
    pl.sync(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n): fn()
    pl.join(st); e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
out = {"pipeline_us": timeit(lambda: pl.step(xh, None, lh, 0.01))}
W = prog.alloc_workspace(b); X = torch.tensor(x, device="cuda")
L = torch.zeros(b, device="cuda", dtype=torch.float64); G = torch.zeros(desc.n_params, device="cuda", dtype=torch.float64)
out["train_step_us"] = timeit(lambda: prog.train_step(X, None, b, P, L, G, 0.01, W, st))
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
'''

for env in [{"TG_JIT_FUSE": "1"}, {"TG_JIT_FUSE": "0"}, {"TG_JIT_FUSE": "1", "TG_PDL": "0"},
            {"TG_JIT_FUSE": "1", "TG_PIPE_GRAPH": "0"}]:
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", CHILD], env=e, capture_output=True, text=True)
    print(env, r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
