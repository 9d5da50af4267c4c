"""GPT b=16 grad_sum through the package found first on sys.path (argv[1]),
saved to argv[2]; with argv[3] == 'ref' also the reference fp64 grad."""
import os
import sys
sys.path.insert(0, sys.argv[1])
sys.path.insert(1, os.getcwd())
import numpy as np
import torch
import paper_2503_13795_b200 as tg
import oracle
from paper_2503_13795_b200.tape import model_id
print("lib", tg._lib.LIB_PATH)
desc = oracle.ref_describe(model_id("gpt"), None, "f32", seed=3)
x, k = tg.synth_batch("gpt", None, "f32", seed=41, batch=16, n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
b = 16
prog = tg.Program(desc)
P = torch.tensor(desc.param_values(), device="cuda")
X = torch.tensor(x, device="cuda") if desc.n_inputs else None
K = torch.tensor(k, device="cuda")
L = torch.zeros(b, device="cuda")
G = torch.zeros(desc.n_params, device="cuda")
W = prog.alloc_workspace(b)
prog.forward_backward(X, K, b, P, L, None, G, W)
torch.cuda.synchronize()
np.save(sys.argv[2], G.cpu().double().numpy())
if len(sys.argv) > 3:
    r = oracle.ref_run(model_id("gpt"), None, "f64", desc.param_values().astype(np.float64), x.astype(np.float64), k, threads=16)
    np.save(sys.argv[2].replace(".npy", "_ref.npy"), r["grad_sum"])
