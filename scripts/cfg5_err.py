import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2503_13795_b200 as tg, oracle
desc = tg.build_model("wide_mlp", None, "f32", seed=3).describe()
b = 512
x, k = tg.synth_batch("wide_mlp", None, "f32", seed=17, batch=b, n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
r = oracle.run(desc, x.astype(np.float64), k, desc.param_values(), threads=os.cpu_count())
# fp64 oracle of the same graph (tape re-recorded in fp64) for a precision reference
d64 = tg.build_model("wide_mlp", None, "f64", seed=3).describe()
r64 = oracle.run(d64, x.astype(np.float64), k, desc.param_values().astype(np.float32).astype(np.float64), threads=os.cpu_count())
for umma in ("1", "0"):
    os.environ["TG_UMMA"] = umma
    p = tg.Program(desc)
    X = torch.tensor(x, device="cuda"); K = torch.tensor(k, device="cuda"); P = torch.tensor(desc.param_values(), device="cuda", dtype=torch.float32)
    L = torch.zeros(b, device="cuda"); G = torch.zeros(desc.n_params, device="cuda")
    p.forward_backward(X, K, b, P, L, None, G); torch.cuda.synchronize()
    L = L.double().cpu().numpy(); G = G.double().cpu().numpy()
    print("umma", umma, "loss max rel vs fp32 oracle", np.max(np.abs(L - r["loss"]) / np.abs(r["loss"])),
          "vs fp64", np.max(np.abs(L - r64["loss"]) / np.abs(r64["loss"])),
          "grad rel vs fp32", np.linalg.norm(G - r["grad_sum"]) / np.linalg.norm(r["grad_sum"]),
          "vs fp64", np.linalg.norm(G - r64["grad_sum"]) / np.linalg.norm(r64["grad_sum"]))
print("fp32 oracle vs fp64: loss", np.max(np.abs(r["loss"] - r64["loss"]) / np.abs(r64["loss"])), "grad", np.linalg.norm(r["grad_sum"] - r64["grad_sum"]) / np.linalg.norm(r64["grad_sum"]))
