"""Generates tests/golden/golden.npz from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libtgref.so, built from
/root/reference/proj/include).  The fixture pins:
  * the Fig. 1 / Listing-1 known answers,
  * reference outputs on replayable random graphs from the reference's own
    fuzzer (testsupport::random_recipe, testing_support.hpp:206-302),
    per sample, for both backward variants and fp64 / fp32,
  * reference per-sample losses and batch gradient sums of the workloads at
    small batch sizes, and the sha256 of their recorded topology.

Usage:  python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2503_13795_b200 as tg  # noqa: E402
from paper_2503_13795_b200.tape import model_id  # noqa: E402

N_RECIPES = 120
RECIPE_BATCH = 6

# small instances of each workload: (name, dims, dtype, batch)
WORKLOADS = [
    ("fig1", None, "f64", 64),
    ("listing1", None, "f64", 64),
    ("moons", None, "f64", 64),
    ("char_mlp", None, "f32", 32),
    ("wide_mlp", [24, 16, 12, 10], "f32", 16),
    ("gpt", [11, 6, 8, 2, 2, 16], "f32", 4),
]


def recipe_leaf_batch(rec, rng, b):
    """Sample 0 = the recipe's own leaves; others redrawn in the same ranges
    (general leaves in [-2, 2] away from 0, the last 4 positive in [0.5, 2.5])."""
    n = len(rec["leaves"])
    lv = np.zeros((n, b))
    lv[:, 0] = rec["leaves"]
    for s in range(1, b):
        for i in range(n):
            if i >= n - 4:
                lv[i, s] = rng.uniform(0.5, 2.5)
            else:
                v = rng.uniform(-2, 2)
                if abs(v) < 1e-2:
                    v += 0.05 if v >= 0 else -0.05
                lv[i, s] = v
    return lv


def topo_hash(t):
    h = hashlib.sha256()
    for k in ("op", "child_offset", "child", "constant"):
        h.update(np.ascontiguousarray(t[k]).tobytes())
    return h.hexdigest()


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle)"
    out = {}
    # --- known answers through the reference ---
    for name, x in (("fig1", [[-41.0], [2.0]]), ("listing1", [[-4.0], [2.0]])):
        r = oracle.ref_run(model_id(name), None, "f64", np.zeros(0), np.array(x), np.zeros((0, 1), np.int32))
        out[f"{name}_value"] = r["loss"]
        out[f"{name}_grad"] = r["input_grad"][:, 0]
    # --- reference fuzzer recipes ---
    rng = np.random.default_rng(2503)
    rec_seeds, rec_max = [], []
    offs = {"leaves": [0], "ops": [0], "args": [0]}
    cat = {"leaves": [], "ops": [], "arg_off": [], "args": [], "consts": [], "lv": [], "root64": [], "grad64": [],
           "root32": [], "grad32": [], "eval": [], "rootR": [], "gradR": []}
    for i in range(N_RECIPES):
        seed = 1000 + i
        max_nodes = [8, 20, 60, 200][i % 4]
        rec = oracle.ref_recipe(seed, max_nodes)
        lv = recipe_leaf_batch(rec, rng, RECIPE_BATCH)
        r64, g64, ev, nn, ne = oracle.ref_recipe_eval(rec, lv, "f64", 1)
        rR, gR, _, _, _ = oracle.ref_recipe_eval(rec, lv, "f64", 0)
        r32, g32, _, _, _ = oracle.ref_recipe_eval(rec, lv, "f32", 1)
        rec_seeds.append(seed)
        rec_max.append(max_nodes)
        cat["leaves"].append(rec["leaves"])
        cat["ops"].append(rec["ops"])
        cat["arg_off"].append(rec["arg_off"])
        cat["args"].append(rec["args"])
        cat["consts"].append(rec["consts"])
        cat["lv"].append(lv.ravel())
        cat["root64"].append(r64)
        cat["grad64"].append(g64.ravel())
        cat["root32"].append(r32)
        cat["grad32"].append(g32.ravel())
        cat["eval"].append(ev)
        cat["rootR"].append(rR)
        cat["gradR"].append(gR.ravel())
    out["recipe_seed"] = np.array(rec_seeds)
    out["recipe_max_nodes"] = np.array(rec_max)
    out["recipe_n_leaves"] = np.array([len(x) for x in cat["leaves"]])
    out["recipe_n_steps"] = np.array([len(x) for x in cat["ops"]])
    out["recipe_n_args"] = np.array([len(x) for x in cat["args"]])
    for k, v in cat.items():
        out[f"recipe_{k}"] = np.concatenate(v)
    out["recipe_batch"] = np.array(RECIPE_BATCH)
    # --- workloads at small batch ---
    for name, dims, dt, b in WORKLOADS:
        m = model_id(name)
        desc = tg.build_model(name, dims, dt, seed=5).describe()
        x, k = tg.synth_batch(name, dims, dt, seed=77, batch=b, n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
        p = desc.param_values()
        r = oracle.ref_run(m, dims, dt, p, x.astype(np.float64), k)
        out[f"w_{name}_loss"] = r["loss"]
        out[f"w_{name}_input_grad"] = r["input_grad"]
        out[f"w_{name}_grad_sum"] = r["grad_sum"]
        x1, k1 = tg.synth_batch(name, dims, "f64", seed=6, batch=1, n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
        t = oracle.ref_build(m, dims, 5, dt, x1[:, 0] if x1.size else np.zeros(1), k1[:, 0] if k1.size else np.zeros(1, np.int32))
        out[f"w_{name}_topo_sha256"] = np.array(topo_hash(t))
        out[f"w_{name}_n_nodes"] = np.array(len(t["op"]))
        out[f"w_{name}_n_edges"] = np.array(len(t["child"]))
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), sum(v.nbytes for v in out.values()), "bytes raw")


if __name__ == "__main__":
    main()
