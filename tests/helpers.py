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
    """Normwise relative error over the finite entries; entries where both
    sides are the same non-finite value (both NaN, equal infinities: the
    reference itself overflowed) are equal, any other non-finite mismatch is
    an infinite error."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    fin = np.isfinite(got) & np.isfinite(want)
    if not fin.all():
        same = (got == want) | (np.isnan(got) & np.isnan(want))
        if not np.all(fin | same):
            return float("inf")
        got, want = np.where(fin, got, 0.0), np.where(fin, want, 0.0)
    den = max(float(np.linalg.norm(want)), 1e-300)
    return float(np.linalg.norm(got - want)) / den


def rel_sum(got, want, terms):
    """Normwise error of a batch sum relative to the sum of its terms'
    magnitudes: ||got - want|| / || sum_i |terms[:, i]| || (terms: [n][batch]).
    Equals rel() when the terms do not cancel."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    t = np.abs(np.asarray(terms, np.float64)).sum(axis=1)
    fin = np.isfinite(got) & np.isfinite(want) & np.isfinite(t)
    if not fin.all():
        same = (got == want) | (np.isnan(got) & np.isnan(want))
        if not np.all(fin | same):
            return float("inf")
    den = max(float(np.linalg.norm(t[fin])), 1e-300)
    return float(np.linalg.norm(got[fin] - want[fin])) / den


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


# ---- independent restatement of the counter-based generator (tg_synth.cuh) ----
M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85


def philox4x32_10(ctr, key):
    """Philox4x32-10 over numpy uint32 arrays: ctr (4, n), key (2, n) -> (4, n)."""
    c = [np.asarray(v, np.uint64) for v in ctr]
    k0, k1 = (np.asarray(v, np.uint64) for v in key)
    m32 = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = np.uint64(M0) * c[0]
        p1 = np.uint64(M1) * c[2]
        h0, l0 = p0 >> np.uint64(32), p0 & m32
        h1, l1 = p1 >> np.uint64(32), p1 & m32
        c = [h1 ^ c[1] ^ k0, l1, h0 ^ c[3] ^ k1, l0]
        k0 = (k0 + np.uint64(W0)) & m32
        k1 = (k1 + np.uint64(W1)) & m32
    return [v.astype(np.uint32) for v in c]


def ctr_draws(seed, samples, n_draws):
    """u64 draws [n_draws][len(samples)]: draw j of sample s = word j % 2 of
    Philox(key = seed, counter = (s, j / 2))."""
    s = np.asarray(samples, np.uint64)
    key = (np.full_like(s, seed & 0xFFFFFFFF), np.full_like(s, seed >> 32))
    out = []
    for p in range((n_draws + 1) // 2):
        ctr = (s & np.uint64(0xFFFFFFFF), s >> np.uint64(32), np.full_like(s, p & 0xFFFFFFFF), np.full_like(s, p >> 32))
        w = [v.astype(np.uint64) for v in philox4x32_10(ctr, key)]
        out.append(w[0] | (w[1] << np.uint64(32)))
        out.append(w[2] | (w[3] << np.uint64(32)))
    return out[:n_draws]


def unit53(u):
    return (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def below(u, n):
    return np.array([(int(v) * n) >> 64 for v in u], np.int64)
