import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import oracle
import paper_2503_13795_b200 as tg
from paper_2503_13795_b200.tape import model_id
from test_gpu import run
desc = oracle.ref_describe(model_id("gpt"), None, "f32", seed=3)
b = int(sys.argv[2]) if len(sys.argv) > 2 else 16
x, k = tg.synth_batch("gpt", None, "f32", seed=41, batch=b, n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
prog = tg.Program(desc)
L, _, G = run(prog, desc, x, k, desc.param_values(), b, want_igrad=False)
np.save(sys.argv[1], G)
r = oracle.ref_run(model_id("gpt"), None, "f64", desc.param_values().astype(np.float64), x.astype(np.float64), k, threads=16)
np.save(sys.argv[1].replace(".npy", "_ref.npy"), r["grad_sum"])
rel = lambda a, c: np.linalg.norm(a - c) / np.linalg.norm(c)
print("rel", rel(G, r["grad_sum"]))
for lo in range(0, len(G), 2048):
    hi = min(len(G), lo + 2048)
    e = rel(G[lo:hi], r["grad_sum"][lo:hi])
    if e > 2e-6: print(lo, hi, f"{e:.2e}", f"norm {np.linalg.norm(r['grad_sum'][lo:hi]):.3e}")
