"""Shared test helpers: golden fixture access, recipe replay, tolerances."""
import os

import numpy as np

import paper_2503_13795_b200 as tg
from paper_2503_13795_b200.tape import OpKind

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = np.load(os.path.join(HERE, "golden", "golden.npz"))

# north_star tolerances: relative 1e-12 (fp64) / 1e-5 (fp32), normwise for
# batch gradients; elementwise with the reference's abs floor (close_rel,
# testing_support.hpp:41-45) for per-sample values.
TOL = {"f64": 1e-12, "f32": 1e-5}


def rel(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = max(float(np.linalg.norm(want)), 1e-300)
    return float(np.linalg.norm(got - want)) / den


def close_rel(got, want, rel_tol, abs_tol=1e-8):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    same = (got == want) | (np.isnan(got) & np.isnan(want))   # equal infinities / both NaN
    with np.errstate(invalid="ignore"):
        diff = np.abs(got - want)
        ok = (diff <= abs_tol) | (diff <= rel_tol * np.maximum(np.abs(got), np.abs(want)))
    return bool(np.all(same | ok))


def recipes():
    """Yield dict(recipe arrays + reference outputs) from the golden fixture."""
    g = GOLDEN
    b = int(g["recipe_batch"])
    ol = os_ = oa = ob = 0
    for i in range(len(g["recipe_seed"])):
        nl, ns, na = int(g["recipe_n_leaves"][i]), int(g["recipe_n_steps"][i]), int(g["recipe_n_args"][i])
        r = {
            "seed": int(g["recipe_seed"][i]),
            "leaves": g["recipe_leaves"][ol:ol + nl],
            "ops": g["recipe_ops"][os_:os_ + ns],
            "arg_off": g["recipe_arg_off"][os_ + i:os_ + i + ns + 1],
            "args": g["recipe_args"][oa:oa + na],
            "consts": g["recipe_consts"][os_:os_ + ns],
            "lv": g["recipe_lv"][ob:ob + nl * b].reshape(nl, b),
            "root64": g["recipe_root64"][i * b:(i + 1) * b],
            "grad64": g["recipe_grad64"][ob:ob + nl * b].reshape(nl, b),
            "root32": g["recipe_root32"][i * b:(i + 1) * b],
            "grad32": g["recipe_grad32"][ob:ob + nl * b].reshape(nl, b),
            "eval": g["recipe_eval"][i * b:(i + 1) * b],
            "rootR": g["recipe_rootR"][i * b:(i + 1) * b],
            "gradR": g["recipe_gradR"][ob:ob + nl * b].reshape(nl, b),
            "batch": b,
        }
        ol += nl
        os_ += ns
        oa += na
        ob += nl * b
        yield r


def replay(rec, dtype="f64", n_params=1):
    """Replays a reference fuzzer recipe on the GPU recorder.

    Leaves 0..n_params-1 become trainable params (batch-summed gradient), the
    rest per-sample inputs; GraphRecipe::build order (testing_support.hpp:
    152-199) so node numbering equals the reference tape's.
    """
    t = tg.Tape(capacity=256, dtype=dtype)
    refs = []
    nl = len(rec["leaves"])
    n_params = min(n_params, nl)
    for i in range(nl):
        v = float(rec["leaves"][i])
        refs.append(t.param(v) if i < n_params else t.input(i - n_params, v))
    ops, off, args, cs = rec["ops"], rec["arg_off"], rec["args"], rec["consts"]
    for k in range(len(ops)):
        a = [refs[j] for j in args[off[k]:off[k + 1]]]
        op = int(ops[k])
        if op == OpKind.MulByConst:
            r = t.mul_by_constant(a[0], float(cs[k]))
        else:
            r = t.op(op, a)
        refs.append(r)
    t.set_root(refs[-1])
    return t, n_params


def tdtype(dt):
    import torch
    return torch.float64 if dt == "f64" else torch.float32
