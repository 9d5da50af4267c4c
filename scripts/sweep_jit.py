"""Times the tape kernel of a bench config under JIT tuning overrides.

Each setting runs in a fresh process (the overrides are read when the
program is first uploaded).  Usage: python scripts/sweep_jit.py cfg2
"""
import itertools
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, bench, paper_2503_13795_b200 as tg
cfg = bench.CONFIGS[sys.argv[1]]
desc = tg.build_model(cfg["model"], cfg["dims"], cfg["dtype"], seed=0).describe()
prog = tg.Program(desc)
b = cfg["batch"]
x, k = tg.synth_batch(cfg["model"], cfg["dims"], cfg["dtype"], seed=1000, batch=b, n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
tdt = torch.float64 if cfg["dtype"] == "f64" else torch.float32
X = torch.tensor(x, device="cuda") if x.size else None
K = torch.tensor(k, device="cuda") if k.size else None
P = torch.tensor(desc.param_values(), device="cuda", dtype=tdt)
L = torch.zeros(b, device="cuda", dtype=tdt); G = torch.zeros(max(desc.n_params,1), device="cuda", dtype=tdt)
W = prog.alloc_workspace(b)
for _ in range(5): prog.forward_backward(X, K, b, P, L, None, G, W)
torch.cuda.synchronize()
prog.profile(True)
for _ in range(50): prog.forward_backward(X, K, b, P, L, None, G, W)
ms, n = prog.profile_read()
print(json.dumps({"kernel_us": 1e3 * ms / n, "storage": prog.info["storage"]}))
'''


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    grid = {"TG_JIT_BLOCK": ["64", "128", "256"], "TG_JIT_SPT": ["1", "2"], "TG_JIT_MINB": ["0", "2", "4"]}
    if len(sys.argv) > 2:
        grid = json.loads(sys.argv[2])
    keys = list(grid)
    for vals in itertools.product(*[grid[k] for k in keys]):
        env = dict(os.environ)
        env.update(dict(zip(keys, vals)))
        r = subprocess.run([sys.executable, "-c", CHILD, cfg], env=env, capture_output=True, text=True, timeout=300)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip().splitlines()[-1:]
        print(dict(zip(keys, vals)), line, flush=True)


if __name__ == "__main__":
    main()
