"""One forward_backward + train_step of a bench config at a small batch, for
compute-sanitizer (memcheck / racecheck / synccheck) runs.
Usage: python scripts/sanitize_run.py cfgN BATCH"""
import os
import sys
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2503_13795_b200 as tg

cfg = bench.CONFIGS[sys.argv[1]]
b = int(sys.argv[2])
desc = tg.build_model(cfg["model"], cfg["dims"], cfg["dtype"], seed=0).describe()
prog = tg.Program(desc)
x, k = tg.synth_batch(cfg["model"], cfg["dims"], cfg["dtype"], seed=1000, batch=b, n_inputs=desc.n_inputs,
                      n_index=desc.n_index_inputs)
tdt = torch.float64 if cfg["dtype"] == "f64" else torch.float32
X = torch.tensor(x, device="cuda") if x.size else None
K = torch.tensor(k, device="cuda") if k.size else None
P = torch.tensor(desc.param_values(), device="cuda", dtype=tdt)
L = torch.zeros(b, device="cuda", dtype=tdt)
G = torch.zeros(max(desc.n_params, 1), device="cuda", dtype=tdt)
W = prog.alloc_workspace(b)
prog.forward_backward(X, K, b, P, L, None, G, W)
if desc.n_params:
    prog.train_step(X, K, b, P, L, G, cfg["gamma"], W)
torch.cuda.synchronize()
prog.check_device_error()
print("ok", sys.argv[1], b, "tier", prog.info["storage"], "launches", prog.launches)
