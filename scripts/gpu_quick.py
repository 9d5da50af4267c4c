"""Quick GPU parity probe: GPU program vs oracle for each workload."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2503_13795_b200 as tg
import oracle

def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

cases = [("fig1", None, "f64", 1000), ("listing1", None, "f64", 1000), ("moons", None, "f64", 4096),
         ("char_mlp", None, "f32", 512), ("wide_mlp", [64, 48, 32, 10], "f32", 256), ("gpt", [11, 6, 8, 2, 2, 16], "f32", 64)]
for m, dims, dt, b in cases:
    t0 = time.time()
    tape = tg.build_model(m, dims, dt, seed=1)
    d = tape.describe()
    prog = tg.Program(d)
    x, k = tg.synth_batch(m, dims, dt, seed=7, batch=b, n_inputs=d.n_inputs, n_index=d.n_index_inputs)
    p = d.param_values()
    ref = oracle.run(d, x, k, p, threads=8)
    tdt = torch.float64 if dt == "f64" else torch.float32
    X = torch.tensor(x, device="cuda", dtype=tdt) if x.size else None
    K = torch.tensor(k, device="cuda") if k.size else None
    P = torch.tensor(p, device="cuda", dtype=tdt)
    L = torch.zeros(b, device="cuda", dtype=tdt)
    IG = torch.zeros((max(d.n_inputs,1), b), device="cuda", dtype=tdt)
    GS = torch.zeros(max(d.n_params,1), device="cuda", dtype=tdt)
    prog.forward_backward(X, K, b, P, L, IG if d.n_inputs else None, GS)
    torch.cuda.synchronize()
    prog.check_device_error()
    out = {"loss": rel(L.cpu().numpy(), ref["loss"])}
    if d.n_inputs: out["igrad"] = rel(IG.cpu().numpy()[:d.n_inputs], ref["input_grad"])
    if d.n_params: out["grad"] = rel(GS.cpu().numpy()[:d.n_params], ref["grad_sum"])
    print(m, dt, b, prog.info["storage"], prog.info["tile_samples"], out, f"{time.time()-t0:.2f}s", flush=True)
