"""CPU: the oracle restatement pinned against the reference and its known answers."""
import math

import numpy as np
import pytest

import oracle
import paper_2503_13795_b200 as tg
from paper_2503_13795_b200.tape import OpKind, model_id
from helpers import GOLDEN, TOL, close_rel, recipes, rel, replay

NOIDX = np.zeros((0, 1), np.int32)


def run1(name, x):
    d = tg.build_model(name).describe()
    return oracle.run(d, np.array(x, float).reshape(-1, 1), NOIDX, d.param_values())


def test_fig1_known_answer():
    # g = 612.5, dg/da = -35, dg/db = 1050 at a=-41, b=2
    r = run1("fig1", [-41.0, 2.0])
    assert r["loss"][0] == 612.5
    assert list(r["input_grad"][:, 0]) == [-35.0, 1050.0]
    assert r["loss"][0] == GOLDEN["fig1_value"][0]


def test_listing1_known_answer_and_structure():
    # PAPER.md:1296 Listing 1; 32 nodes / 44 edges
    d = tg.build_model("listing1").describe()
    assert d.n_nodes == 32 and d.n_edges == 44
    r = run1("listing1", [-4.0, 2.0])
    assert r["loss"][0] == GOLDEN["listing1_value"][0] == 24.704081632653061
    assert list(r["input_grad"][:, 0]) == list(GOLDEN["listing1_grad"])
    assert GOLDEN["listing1_grad"][0] == 138.83381924198252
    assert GOLDEN["listing1_grad"][1] == 645.57725947521863


def test_listing1_finite_differences():
    # central differences h=1e-6, rel 1e-6
    d = tg.build_model("listing1").describe()
    x0 = np.array([-4.0, 2.0])
    g = run1("listing1", x0)["input_grad"][:, 0]
    for i in range(2):
        xp, xm = x0.copy(), x0.copy()
        xp[i] += 1e-6
        xm[i] -= 1e-6
        fd = (run1("listing1", xp)["loss"][0] - run1("listing1", xm)["loss"][0]) / 2e-6
        assert close_rel(g[i], fd, 1e-6)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_recipes_match_reference_bitwise(dtype):
    """Restatement == reference backward_with_scratch on the reference fuzzer
    graphs, bit for bit (same op order, -ffp-contract=off both sides)."""
    n = 0
    for rec in recipes():
        t, npar = replay(rec, dtype, n_params=0)
        d = t.describe()
        lv = rec["lv"]
        r = oracle.run(d, lv, NOIDX[:, :0].reshape(0, lv.shape[1]), np.zeros(0))
        want_root = rec["root64"] if dtype == "f64" else rec["root32"]
        want_grad = rec["grad64"] if dtype == "f64" else rec["grad32"]
        np.testing.assert_array_equal(r["loss"], want_root)
        np.testing.assert_array_equal(r["input_grad"], want_grad)
        n += 1
    assert n == len(GOLDEN["recipe_seed"])


def test_reference_variants_agree():
    # backward == backward_with_scratch bit-exactly
    for rec in recipes():
        np.testing.assert_array_equal(rec["root64"], rec["rootR"])
        np.testing.assert_array_equal(rec["grad64"], rec["gradR"])


def test_recipe_eval_interpreter_agrees():
    # GraphRecipe::eval, the independent interpreter, vs the tape value
    for rec in recipes():
        assert close_rel(rec["root64"], rec["eval"], 1e-12)


def test_recipe_finite_differences_small_graphs():
    # FD oracle on graphs <= 20 nodes, rel 1e-5 (abs 1e-8)
    checked = 0
    for rec in recipes():
        if rec["ops"].shape[0] > 12:
            continue
        t, _ = replay(rec, "f64", n_params=0)
        d = t.describe()
        x = rec["lv"][:, :1].copy()
        g = oracle.run(d, x, np.zeros((0, 1), np.int32), np.zeros(0))["input_grad"][:, 0]
        for i in range(x.shape[0]):
            xp, xm = x.copy(), x.copy()
            xp[i] += 1e-6
            xm[i] -= 1e-6
            try:
                fp = oracle.run(d, xp, np.zeros((0, 1), np.int32), np.zeros(0))["loss"][0]
                fm = oracle.run(d, xm, np.zeros((0, 1), np.int32), np.zeros(0))["loss"][0]
            except oracle.OracleError:
                continue
            fd = (fp - fm) / 2e-6
            if abs(fd) > 1e3 or not math.isfinite(fd):
                continue
            assert close_rel(g[i], fd, 1e-4, 1e-5), (rec["seed"], i, g[i], fd)
            checked += 1
    assert checked > 50


@pytest.mark.parametrize("name,dims,dtype,b", [
    ("fig1", None, "f64", 64), ("listing1", None, "f64", 64), ("moons", None, "f64", 64),
    ("char_mlp", None, "f32", 32), ("wide_mlp", [24, 16, 12, 10], "f32", 16), ("gpt", [11, 6, 8, 2, 2, 16], "f32", 4)])
def test_workloads_match_reference(name, dims, dtype, b):
    """Restatement over the compiled-tape description == the reference
    re-recording every sample with its own token ids (golden fixture)."""
    desc = tg.build_model(name, dims, dtype, seed=5).describe()
    x, k = tg.synth_batch(name, dims, dtype, seed=77, batch=b, n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
    r = oracle.run(desc, x.astype(np.float64), k, desc.param_values())
    np.testing.assert_array_equal(r["loss"], GOLDEN[f"w_{name}_loss"])
    np.testing.assert_array_equal(r["grad_sum"], GOLDEN[f"w_{name}_grad_sum"])
    if desc.n_inputs:
        np.testing.assert_array_equal(r["input_grad"], GOLDEN[f"w_{name}_input_grad"][:desc.n_inputs])


def test_linearity_of_estimator():
    # batch accumulator = sum of independent per-sample grads (1e-12)
    desc = tg.build_model("moons").describe()
    x, k = tg.synth_batch("moons", batch=40, seed=3)
    p = desc.param_values()
    full = oracle.run(desc, x, k, p)["grad_sum"]
    acc = np.zeros_like(full)
    for s in range(40):
        acc += oracle.run(desc, x[:, s:s + 1], k[:, s:s + 1], p)["grad_sum"]
    assert rel(full, acc) <= 1e-12


def test_threads_do_not_change_result_beyond_order():
    desc = tg.build_model("moons").describe()
    x, k = tg.synth_batch("moons", batch=256, seed=3)
    p = desc.param_values()
    a = oracle.run(desc, x, k, p, threads=1)
    b = oracle.run(desc, x, k, p, threads=7)
    np.testing.assert_array_equal(a["loss"], b["loss"])
    assert rel(b["grad_sum"], a["grad_sum"]) <= 1e-13


def test_processing_order_matches_compiler():
    """The compiler's single DFS equals backward_with_scratch's order."""
    for name, dims, dt in [("fig1", None, "f64"), ("listing1", None, "f64"), ("moons", None, "f64"),
                           ("char_mlp", None, "f32")]:
        desc = tg.build_model(name, dims, dt).describe()
        prog = tg.Program(desc)
        k = np.zeros((max(desc.n_index_inputs, 1), 1), np.int32)
        want = oracle.order(desc, k)
        got = prog.order()
        np.testing.assert_array_equal(got, want)


def test_domain_error_message_matches_reference():
    t = tg.Tape(dtype="f64")
    a = t.input(0, 1.0)
    lg = t.log(a)
    t.set_root(lg)
    d = t.describe()
    with pytest.raises(oracle.OracleError) as e:
        oracle.run(d, np.array([[2.0, 1.0, -1.0, 3.0]]), np.zeros((0, 4), np.int32), np.zeros(0))
    assert str(e.value) == "logarithm: input -1.000000 is outside the operator domain"
    assert e.value.sample == 2


def test_sgd_step_formula():
    # SPEC.md:424-430 examples
    p = np.array([1.0])
    oracle.sgd("f64", p, np.array([2.0]), 0.1, 1)
    assert p[0] == 0.8
    p = np.array([1.0])
    oracle.sgd("f64", p, np.array([4.0]), 0.5, 2)  # mean 2
    assert p[0] == 0.0


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name,dims,dt", [("char_mlp", None, "f32"), ("gpt", [13, 8, 16, 2, 2, 32], "f32"),
                                         ("wide_mlp", [24, 16, 12, 10], "f32"), ("moons", None, "f64")])
def test_reference_recording_drop_in_describes_like_tg_tape(name, dims, dt):
    """A model recorded with the UNMODIFIED tapegrad::Tape plus the drop-in
    adapter's side record (include/tg_from_tapegrad.hpp: per-sample row
    selections become gathers, the softmax max-shift leaf becomes the
    per-sample stop-gradient max) describes to exactly the arrays this
    package's own recorder produces: ops, children with gather references,
    gather table, leaf roles, parameter values."""
    from paper_2503_13795_b200.tape import model_id
    a = oracle.ref_describe(model_id(name), dims, dt, seed=3)
    b = tg.build_model(name, dims, dt, seed=3).describe()
    for f in ("op", "child_offset", "child", "constant", "leaf_class", "leaf_index", "gathers"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
    assert (a.root, a.n_params, a.n_inputs, a.n_index_inputs) == (b.root, b.n_params, b.n_inputs, b.n_index_inputs)
    np.testing.assert_array_equal(a.param_values(), b.param_values())


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_reference_recording_rejects_ambiguous_selection():
    """Two columns selecting the same row of one table in the template sample
    cannot be told apart on a reference tape: describe refuses."""
    import ctypes as C
    lib = oracle._reflib()
    from paper_2503_13795_b200 import _lib as plib
    d = plib.tg_tape_desc()
    # gpt with a vocabulary of 3 over 8 positions: the template's idx[c] = c % 3 repeats rows
    st = lib.ref_describe(5, oracle._d(oracle._dims([3, 8, 16, 2, 1, 32])), 0, 1, None, C.byref(d))
    assert st != 0 and b"selected twice" in lib.ref_last_error()


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name,dims,dt", [("char_mlp", None, "f32"), ("wide_mlp", [24, 16, 12, 10], "f32"),
                                         ("moons", None, "f64"), ("gpt", None, "f32"), ("fig1", None, "f64")])
def test_reference_side_inputs_equal_product_generators(name, dims, dt):
    """The bench's reference arm takes its parameters and samples from
    oracle/_ref (ref_params / ref_synth), never from the product library;
    they are the same bits as the product's for the same seeds."""
    from paper_2503_13795_b200.tape import model_id
    d = tg.build_model(name, dims, dt, seed=0).describe()
    np.testing.assert_array_equal(oracle.ref_params(model_id(name), dims, dt, seed=0), d.param_values())
    x, k = tg.synth_batch(name, dims, dt, seed=1234, batch=300, n_inputs=d.n_inputs, n_index=d.n_index_inputs)
    xr, kr = oracle.ref_synth(model_id(name), dims, dt, 1234, 300)
    np.testing.assert_array_equal(xr, x.astype(np.float64))
    np.testing.assert_array_equal(kr, k)
