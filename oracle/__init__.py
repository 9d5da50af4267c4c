"""Checkers for the gradient-oracle path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
`--impl reference` arm) may import this package.  The product package never
does.

* `run` / `sgd` / `order`: liboracle.so, the CPU restatement of the
  reference per-sample algorithm (tg_oracle.cpp).
* `ref_*`: oracle/_ref/libtgref.so, the UNMODIFIED reference headers
  (/root/reference/proj/include) compiled in the build container, driving
  the same model compositions and the reference's own random-graph fuzzer.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "build", "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libtgref.so")

_DT = {"f64": 0, "f32": 1}


def _d(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _Oracle:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        lib = C.CDLL(ORACLE_SO)
        P, sz = C.c_void_p, C.c_size_t
        lib.oracle_run.restype = C.c_int
        lib.oracle_run.argtypes = [P, P, P, sz, P, P, P, P, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_uint32)]
        lib.oracle_sgd.restype = None
        lib.oracle_sgd.argtypes = [C.c_int, P, P, sz, C.c_double, sz]
        lib.oracle_order.restype = C.c_int
        lib.oracle_order.argtypes = [P, P, sz, sz, P, C.POINTER(C.c_uint32)]
        lib.oracle_last_error.restype = C.c_char_p
        self.lib = lib


_oracle = None


def _lib():
    global _oracle
    if _oracle is None:
        _oracle = _Oracle()
    return _oracle.lib


class OracleError(RuntimeError):
    def __init__(self, status, msg, sample=-1, node=0):
        super().__init__(msg)
        self.status, self.sample, self.node = status, sample, node


def run(desc, x, idx, params, threads: int = 1, want_loss=True, want_input_grad=True):
    """Reference algorithm per sample over `desc` (a tape.TapeDesc).

    x: [n_inputs][b] float, idx: [n_index][b] int32, params: [n_params].
    Returns dict(loss [b], input_grad [n_inputs][b], grad_sum [n_params]) in float64.
    """
    b = x.shape[1] if x.size else idx.shape[1]
    x64 = np.ascontiguousarray(x, np.float64)
    k32 = np.ascontiguousarray(idx, np.int32)
    p64 = np.ascontiguousarray(params, np.float64)
    loss = np.zeros(b) if want_loss else None
    ig = np.zeros((desc.n_inputs, b)) if want_input_grad and desc.n_inputs else None
    gs = np.zeros(max(desc.n_params, 1))
    cd = desc.to_c()
    s, n = C.c_int64(-1), C.c_uint32(0)
    st = _lib().oracle_run(C.byref(cd), _d(x64), _d(k32), b, _d(p64), _d(loss), _d(ig), _d(gs), threads,
                           C.byref(s), C.byref(n))
    if st != 0:
        raise OracleError(st, _lib().oracle_last_error().decode(), s.value, n.value)
    return {"loss": loss, "input_grad": ig, "grad_sum": gs[:desc.n_params]}


def sgd(dtype: str, params, grad_sum, gamma: float, batch: int):
    """sgd_step in the tape's scalar type (in place on a float64 array)."""
    _lib().oracle_sgd(_DT[dtype], _d(params), _d(np.ascontiguousarray(grad_sum, np.float64)),
                      params.shape[0], float(gamma), int(batch))


def order(desc, idx=None, sample: int = 0):
    """Processing order of backward_with_scratch for one sample."""
    out = np.zeros(desc.n_nodes, np.uint32)
    n = C.c_uint32()
    k32 = np.ascontiguousarray(idx if idx is not None else np.zeros((1, 1)), np.int32)
    ld = k32.shape[1]
    cd = desc.to_c()
    st = _lib().oracle_order(C.byref(cd), _d(k32), ld, sample, _d(out), C.byref(n))
    if st != 0:
        raise OracleError(st, _lib().oracle_last_error().decode())
    return out[:n.value]


# ---------------------------------------------------------------------------
# the reference itself (oracle/_ref)
# ---------------------------------------------------------------------------

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _reflib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise ImportError(f"{REF_SO} missing (built only where /root/reference exists)")
        lib = C.CDLL(REF_SO)
        P, sz = C.c_void_p, C.c_size_t
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_build.restype = C.c_int
        lib.ref_build.argtypes = [C.c_int, P, C.c_uint64, C.c_int, P, P, C.POINTER(C.c_uint32),
                                  C.POINTER(C.c_uint64), P, P, P, P, P, C.POINTER(C.c_uint32)]
        lib.ref_run.restype = C.c_int
        lib.ref_run.argtypes = [C.c_int, P, C.c_int, P, P, P, sz, P, P, P, C.c_int]
        lib.ref_params.restype = C.c_int
        lib.ref_params.argtypes = [C.c_int, P, C.c_uint64, C.c_int, P, C.POINTER(C.c_uint32)]
        lib.ref_synth.restype = C.c_int
        lib.ref_synth.argtypes = [C.c_int, P, C.c_int, C.c_uint64, sz, P, P, C.POINTER(C.c_uint32),
                                  C.POINTER(C.c_uint32)]
        lib.ref_describe.restype = C.c_int
        lib.ref_describe.argtypes = [C.c_int, P, C.c_uint64, C.c_int, P, P]
        lib.ref_recipe.restype = C.c_int
        lib.ref_recipe.argtypes = [C.c_uint64, sz, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        lib.ref_recipe_fetch.restype = None
        lib.ref_recipe_fetch.argtypes = [P, P, P, P, P]
        lib.ref_recipe_eval.restype = C.c_int
        lib.ref_recipe_eval.argtypes = [C.c_uint32, C.c_uint32, P, P, P, P, C.c_int, C.c_int, P, sz, P, P, P,
                                        C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)]
        _ref = lib
    return _ref


def _dims(dims):
    a = np.zeros(8, np.uint32)
    for i, v in enumerate(dims or []):
        a[i] = v
    return a


def ref_build(model: int, dims, seed: int, dtype: str, x1, idx1):
    """Topology of params + one sample recorded on the reference tape."""
    lib = _reflib()
    dm = _dims(dims)
    x1 = np.ascontiguousarray(x1, np.float64)
    k1 = np.ascontiguousarray(idx1, np.int32)
    n, e, root = C.c_uint32(), C.c_uint64(), C.c_uint32()
    st = lib.ref_build(model, _d(dm), seed, _DT[dtype], _d(x1), _d(k1), C.byref(n), C.byref(e),
                       None, None, None, None, None, C.byref(root))
    if st:
        raise OracleError(st, lib.ref_last_error().decode())
    ops = np.zeros(n.value, np.uint8)
    off = np.zeros(n.value + 1, np.uint64)
    ch = np.zeros(max(e.value, 1), np.uint32)
    cs = np.zeros(n.value)
    vals = np.zeros(n.value)
    st = lib.ref_build(model, _d(dm), seed, _DT[dtype], _d(x1), _d(k1), C.byref(n), C.byref(e),
                       _d(ops), _d(off), _d(ch), _d(cs), _d(vals), C.byref(root))
    if st:
        raise OracleError(st, lib.ref_last_error().decode())
    return {"op": ops, "child_offset": off, "child": ch[:e.value], "constant": cs, "value": vals,
            "root": root.value}


def ref_params(model: int, dims, dtype: str, seed: int = 0):
    """Initial parameters of `model` recorded on the reference tape (make_params)."""
    lib = _reflib()
    n = C.c_uint32()
    dm = _dims(dims)
    st = lib.ref_params(model, _d(dm), seed, _DT[dtype], None, C.byref(n))
    if st:
        raise OracleError(st, lib.ref_last_error().decode())
    out = np.zeros(max(n.value, 1))
    st = lib.ref_params(model, _d(dm), seed, _DT[dtype], _d(out), C.byref(n))
    if st:
        raise OracleError(st, lib.ref_last_error().decode())
    return out[:n.value]


def ref_synth(model: int, dims, dtype: str, seed: int, batch: int):
    """Synthetic batch (x [n_inputs][batch] float64, idx [n_index][batch] int32),
    the same bits as the product's tg_synth_batch for the same seed."""
    lib = _reflib()
    dm = _dims(dims)
    ni, nk = C.c_uint32(), C.c_uint32()
    st = lib.ref_synth(model, _d(dm), _DT[dtype], seed, batch, None, None, C.byref(ni), C.byref(nk))
    if st:
        raise OracleError(st, lib.ref_last_error().decode())
    x = np.zeros((max(ni.value, 1), batch))
    k = np.zeros((max(nk.value, 1), batch), np.int32)
    st = lib.ref_synth(model, _d(dm), _DT[dtype], seed, batch, _d(x), _d(k), C.byref(ni), C.byref(nk))
    if st:
        raise OracleError(st, lib.ref_last_error().decode())
    return x[:ni.value], k[:nk.value]


def ref_describe(model: int, dims, dtype: str, seed: int = 0, x1=None):
    """A template sample recorded on the UNMODIFIED reference tape with the
    drop-in adapter (include/tg_from_tapegrad.hpp: tgadapt::Recording +
    describe): a tape.TapeDesc the product compiles like its own recordings."""
    from paper_2503_13795_b200 import _lib as plib
    from paper_2503_13795_b200.tape import _desc_from_c
    lib = _reflib()
    d = plib.tg_tape_desc()
    x = None if x1 is None else np.ascontiguousarray(x1, np.float64)
    st = lib.ref_describe(model, _d(_dims(dims)), seed, _DT[dtype], _d(x), C.byref(d))
    if st:
        raise OracleError(st, lib.ref_last_error().decode())
    return _desc_from_c(d)


def ref_run(model: int, dims, dtype: str, params, x, idx, threads: int = 1):
    """The reference's own per-sample train_step path (rewind/build/backward)."""
    lib = _reflib()
    b = x.shape[1] if x.size else idx.shape[1]
    ni = x.shape[0]
    loss = np.zeros(b)
    ig = np.zeros((max(ni, 1), b))
    gs = np.zeros(max(len(params), 1))
    st = lib.ref_run(model, _d(_dims(dims)), _DT[dtype], _d(np.ascontiguousarray(params, np.float64)),
                     _d(np.ascontiguousarray(x, np.float64)), _d(np.ascontiguousarray(idx, np.int32)), b,
                     _d(loss), _d(ig), _d(gs), threads)
    if st:
        raise OracleError(st, lib.ref_last_error().decode())
    return {"loss": loss, "input_grad": ig[:ni], "grad_sum": gs[:len(params)]}


def ref_recipe(seed: int, max_nodes: int):
    """testsupport::random_recipe serialised: dict of numpy arrays."""
    lib = _reflib()
    nl, ns, na = C.c_uint32(), C.c_uint32(), C.c_uint32()
    lib.ref_recipe(seed, max_nodes, C.byref(nl), C.byref(ns), C.byref(na))
    leaves = np.zeros(nl.value)
    ops = np.zeros(ns.value, np.uint8)
    off = np.zeros(ns.value + 1, np.uint32)
    args = np.zeros(max(na.value, 1), np.uint32)
    cs = np.zeros(ns.value)
    lib.ref_recipe_fetch(_d(leaves), _d(ops), _d(off), _d(args), _d(cs))
    return {"leaves": leaves, "ops": ops, "arg_off": off, "args": args[:na.value], "consts": cs}


def ref_recipe_eval(rec, leaf_values, dtype: str = "f64", variant: int = 1):
    """Per-sample GraphRecipe::build + backward on reference tapes.

    leaf_values: [n_leaves][b].  Returns (root [b], leaf_grad [n_leaves][b],
    eval [b] from the independent interpreter, n_nodes, n_edges).
    """
    lib = _reflib()
    lv = np.ascontiguousarray(leaf_values, np.float64)
    nl, b = lv.shape
    root = np.zeros(b)
    lg = np.zeros((nl, b))
    ev = np.zeros(b)
    nn, ne = C.c_uint32(), C.c_uint64()
    args = np.ascontiguousarray(rec["args"], np.uint32)
    if args.size == 0:
        args = np.zeros(1, np.uint32)
    st = lib.ref_recipe_eval(nl, len(rec["ops"]), _d(np.ascontiguousarray(rec["ops"], np.uint8)),
                             _d(np.ascontiguousarray(rec["arg_off"], np.uint32)), _d(args),
                             _d(np.ascontiguousarray(rec["consts"], np.float64)), _DT[dtype], variant,
                             _d(lv), b, _d(root), _d(lg), _d(ev), C.byref(nn), C.byref(ne))
    if st:
        raise OracleError(st, lib.ref_last_error().decode())
    return root, lg, ev, nn.value, ne.value
