"""CPU: the C-ABI boundary, the recorder's reference-compatible behaviour and
the compiler's lowering decisions (no device needed)."""
import ctypes
import hashlib
import os

import numpy as np
import pytest

import oracle
import paper_2503_13795_b200 as tg
from paper_2503_13795_b200 import _lib
from paper_2503_13795_b200.tape import OpKind, model_id
from helpers import GOLDEN


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = _lib.header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_oracle_libraries_load():
    assert os.path.exists(oracle.ORACLE_SO)
    oracle._lib()


def test_status_and_op_names():
    assert _lib.lib.tg_status_name(5).decode() == "TG_DOMAIN"
    # op_kind.hpp:89-123 mnemonics
    assert tg.op_name(OpKind.Cub) == "pow3"
    assert tg.op_name(OpKind.Log) == "logarithm"
    assert tg.op_name(OpKind.InnerProductWithBias) == "innerProductWithBias"
    assert tg.op_name(OpKind.StopGradMax) == "stopGradMax"


def test_recorder_eager_values_and_indices():
    # SPEC.md leaf / raw index examples
    t = tg.Tape(capacity=16)
    a = t.leaf(-41.0)
    b = t.leaf(2.0)
    assert (a, b) == (0, 1)
    assert t.value_of(t.add_squares(t.leaf(3.0), t.leaf(4.0))) == 25.0
    assert t.value_of(t.mean(t.leaf(1.0), t.leaf(3.0))) == 2.0
    x = [t.leaf(1.0), t.leaf(2.0)]
    y = [t.leaf(3.0), t.leaf(4.0)]
    assert t.value_of(t.inner_product_with_bias(x, y, t.leaf(5.0))) == 16.0
    assert t.value_of(t.reduce_mul([t.leaf(2.0), t.leaf(3.0), t.leaf(0.0)])) == 0.0
    assert t.value_of(t.tanh(t.leaf(0.0))) == 0.0
    assert t.value_of(t.relu(t.leaf(-3.0))) == 0.0


@pytest.mark.parametrize("op,val,msg", [
    (OpKind.Log, -1.0, "logarithm: input -1.000000 is outside the operator domain"),
    (OpKind.Sqrt, 0.0, "sqrt: input 0.000000 is outside the operator domain"),
    (OpKind.NegLog, 0.0, "negativeLog: input 0.000000 is outside the operator domain"),
    (OpKind.Inv, 0.0, "inv: input 0.000000 is outside the operator domain"),
    (OpKind.InvSqrt, -2.0, "invSqrt: input -2.000000 is outside the operator domain"),
])
def test_recorder_domain_errors_match_reference(op, val, msg):
    # ops.hpp:16-32 throw std::domain_error with this exact text
    t = tg.Tape()
    x = t.leaf(val)
    with pytest.raises(tg.DomainError) as e:
        t.op(op, [x])
    assert str(e.value).endswith(msg)


def test_recorder_div_by_zero_and_arity_errors():
    t = tg.Tape()
    one, zero = t.leaf(1.0), t.leaf(0.0)
    with pytest.raises(tg.DomainError, match="div: input 0.000000 is outside the operator domain"):
        t.div(one, zero)
    with pytest.raises(tg.InvalidArgument, match="reduceSum: empty input sequence"):
        t.reduce_sum([])
    with pytest.raises(tg.InvalidArgument, match=r"innerProduct: sequence lengths differ \(2 vs 1\)"):
        t.inner_product([one, one], [one])
    with pytest.raises(tg.TgError, match="TG_INVALID_HANDLE"):
        t.add(one, 9999)


def test_recorder_topology_matches_reference_tape():
    """Same composition recorded on tg::Tape and on the reference tapegrad::Tape:
    opcodes, child lists (gathers resolved with the template sample) and
    constants identical."""
    for name, dims, dt, _ in [("fig1", None, "f64", 0), ("listing1", None, "f64", 0), ("moons", None, "f64", 0),
                              ("char_mlp", None, "f32", 0), ("wide_mlp", [24, 16, 12, 10], "f32", 0),
                              ("gpt", [11, 6, 8, 2, 2, 16], "f32", 0)]:
        d = tg.build_model(name, dims, dt, seed=5).describe()
        x1, k1 = tg.synth_batch(name, dims, "f64", seed=6, batch=1, n_inputs=d.n_inputs, n_index=d.n_index_inputs)
        # resolve my tape to the reference's form: gathers -> template rows, stop-gradient max -> Leaf
        ops = d.op.copy()
        ops[ops == OpKind.StopGradMax] = OpKind.Leaf
        child, off = [], [0]
        for i in range(d.n_nodes):
            if d.op[i] != OpKind.StopGradMax:
                for c in d.children(i):
                    if c & _lib.TG_GATHER_FLAG:
                        first, stride, n_rows, col, o = (int(v) for v in d.gathers[int(c) & 0x7FFFFFFF])
                        c = first + stride * int(k1[col, 0]) + o
                    child.append(c)
            off.append(len(child))
        h = hashlib.sha256()
        h.update(ops.tobytes())
        h.update(np.array(off, np.uint64).tobytes())
        h.update(np.array(child, np.uint32).tobytes())
        h.update(np.where(d.op == OpKind.StopGradMax, 0.0, d.constant).astype(np.float64).tobytes())
        assert h.hexdigest() == str(GOLDEN[f"w_{name}_topo_sha256"]), name
        assert d.n_nodes == int(GOLDEN[f"w_{name}_n_nodes"])


def test_param_counts():
    # BASELINE.json: cfg2 d=337, cfg3 ~11.9k, cfg5 1,863,690, cfg4 ~0.21M
    assert tg.build_model("moons").describe().n_params == 337
    assert tg.build_model("char_mlp").describe().n_params == 11897
    d5 = tg.build_model("wide_mlp", dims=[784, 64, 64, 10]).describe()
    assert d5.n_params == 784 * 64 + 64 + 64 * 64 + 64 + 64 * 10 + 10


def test_compiler_hoists_sample_invariant_nodes():
    # the 1e-4 * sum p^2 regulariser of cfg2 depends on parameters only
    p = tg.Program(tg.build_model("moons"))
    i = p.info
    assert i["n_uniform_nodes"] == 2
    assert i["n_params"] == 337 and i["n_inputs"] == 3


def test_compiler_rejects_malformed_tapes():
    d = tg.build_model("fig1").describe()
    bad = tg.TapeDesc(**{k: getattr(d, k) for k in ("op", "child_offset", "child", "constant", "leaf_class",
                                                     "leaf_index", "leaf_value", "gathers", "root", "n_params",
                                                     "n_inputs", "n_index_inputs", "dtype")})
    bad.child = bad.child.copy()
    bad.child[0] = 50  # forward reference: not a topological order
    with pytest.raises(tg.InvalidArgument, match="topological"):
        tg.Program(bad)
    bad2 = tg.TapeDesc(**{**bad.__dict__, "child": d.child.copy(), "root": 999})
    with pytest.raises(tg.InvalidArgument, match="stale root"):
        tg.Program(bad2)


def test_workspace_size_is_bounded_and_monotone():
    p = tg.Program(tg.build_model("moons"))
    a, b = p.workspace_size(1024), p.workspace_size(65536)
    assert 0 < a <= b < 64 << 20


@pytest.mark.parametrize("form,marker", [("dmma", "mma.sync.aligned.m8n8k4.row.col.f64"),
                                         ("group", "lane & 15u"),
                                         ("classic", "dense weight gradient 16x16")])
def test_jit_source_compiles_with_nvrtc(form, marker, monkeypatch):
    """The specialised kernels are generated and compiled (NVRTC, sm_100a)
    without a device; only loading needs the GPU.  cfg2's dense chain takes the
    FP64 tensor-core form by default; the fused module carries the uniform
    prologue in tg_jit_tape and the generated epilogue kernel tg_jit_epi."""
    monkeypatch.setenv("TG_JIT_FORM", form)
    p = tg.Program(tg.build_model("moons"))
    src, log, ms = ctypes.c_char_p(), ctypes.c_char_p(), ctypes.c_double()
    st = _lib.lib.tg_program_jit(p._h, ctypes.byref(src), ctypes.byref(log), ctypes.byref(ms))
    text = src.value.decode()
    assert "tg_jit_tape" in text and marker in text
    # the dense-layer forms carry the fused prologue + generated epilogue; the
    # one-thread-per-sample form keeps constant-bank weights (fuses dense-free tapes only)
    assert ("tg_jit_epi" in text and "griddepcontrol.wait" in text) == (form != "classic")
    assert "compiled" in log.value.decode() or st == 0, log.value


def test_synthetic_generators_are_prefix_stable():
    x1, _ = tg.synth_batch("moons", batch=10, seed=9)
    x2, _ = tg.synth_batch("moons", batch=100, seed=9)
    np.testing.assert_array_equal(x1, x2[:, :10])
    _, k = tg.synth_batch("char_mlp", batch=2000, seed=1)
    assert k.min() >= 0 and k.max() < 27
    counts = np.bincount(k.ravel(), minlength=27)
    assert counts[0] > counts[5] > counts[20]   # Zipf: rank 1 most frequent


@pytest.mark.parametrize("form", ["dmma", "group", "classic"])
@pytest.mark.parametrize("fuse", ["1", "0"])
def test_every_jit_program_compiles(form, fuse, monkeypatch):
    """Every JIT-eligible workload and a sample of the reference's fuzzer
    graphs generate NVRTC-clean sources in every form, fused and unfused (a
    generator bug would otherwise surface on the GPU only as a silent
    interpreter fallback)."""
    from helpers import recipes, replay
    monkeypatch.setenv("TG_JIT_FORM", form)
    monkeypatch.setenv("TG_JIT_FUSE", fuse)
    descs = [tg.build_model(m).describe() for m in ("fig1", "listing1", "moons")]
    descs.append(tg.build_model("moons", None, "f32").describe())
    for rec in list(recipes())[:12]:
        for dt in ("f64", "f32"):
            t, _ = replay(rec, dt, n_params=1)
            descs.append(t.describe())
    for d in descs:
        p = tg.Program(d)
        src, log, ms = ctypes.c_char_p(), ctypes.c_char_p(), ctypes.c_double()
        _lib.lib.tg_program_jit(p._h, ctypes.byref(src), ctypes.byref(log), ctypes.byref(ms))
        text = (log.value or b"").decode()
        assert "compiled" in text or "not eligible" in text, text[-2000:]


@pytest.mark.parametrize("name,dims", [("char_mlp", None), ("wide_mlp", None), ("gpt", None)])
def test_memory_budget_bounds_staged_workspace(name, dims):
    """Sequential-accumulation mode: with a memory
    budget the staged workspace stops growing with the batch (peak device
    memory independent of b), chunks are multiples of 128 samples, and 0
    restores the one-chunk default."""
    p = tg.Program(tg.build_model(name, dims, "f32"))
    assert p.info["storage"] == 3
    big = p.workspace_size(1 << 20)
    p.set_memory_budget(64 << 20)
    cb = p.chunk_samples(1 << 20)
    assert cb % 128 == 0 and 128 <= cb < (1 << 20)
    sizes = [p.workspace_size(b) for b in (cb, 4 * cb, 1 << 20, 1 << 22)]
    assert len(set(sizes)) == 1 and sizes[0] < big
    assert p.chunk_samples(100) == 100
    p.set_memory_budget(0)
    assert p.workspace_size(1 << 20) == big


def test_philox_known_answers():
    """The test-side Philox4x32-10 against the Random123 known-answer vectors."""
    from helpers import philox4x32_10
    cases = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
             ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
             ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
              (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in cases:
        got = philox4x32_10([np.array([v]) for v in ctr], [np.array([v]) for v in key])
        assert [int(g[0]) for g in got] == list(want)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_counter_synth_matches_restatement_and_is_split_invariant(dt):
    """tg_synth_ctr: every integer draw (Zipf ids, labels)
    and every uniform equals the independent numpy restatement bit for bit;
    any split of the sample range gives the same bits."""
    from helpers import below, ctr_draws, unit53
    seed, first, b = 0x1234_5678_9ABC, 1000, 700
    # uniforms: Fig. 1 leaves U[-4, 4] (one fma), wide-MLP pixels U[0, 1) and labels
    x, _ = tg.synth_ctr("fig1", dtype="f64", seed=seed, first=first, batch=b)
    d = ctr_draws(seed, np.arange(first, first + b), 2)
    want = [np.array([np.float64(8.0) * u + np.float64(-4.0) for u in unit53(d[j])]) for j in range(2)]
    # fma(8, u, -4) is exact for 53-bit u (8u is exact), so the plain numpy expression matches it
    assert np.array_equal(x[0], want[0]) and np.array_equal(x[1], want[1])
    dims = [20, 8, 8, 7]
    x, k = tg.synth_ctr("wide_mlp", dims, dt, seed=seed, first=first, batch=b)
    d = ctr_draws(seed, np.arange(first, first + b), 21)
    for c in range(20):
        assert np.array_equal(x[c], unit53(d[c]).astype(x.dtype))
    assert np.array_equal(k[0], below(d[20], 7))
    # Zipf ids: inverse CDF over p_k ∝ k^-s (s = 1.1, V = 27)
    _, k = tg.synth_ctr("char_mlp", dtype="f32", seed=seed, first=first, batch=b)
    p = np.arange(1, 28, dtype=np.float64) ** -1.1
    cdf = np.cumsum(p) / p.sum()
    d = ctr_draws(seed, np.arange(first, first + b), 4)
    for c in range(4):
        assert np.array_equal(k[c], np.searchsorted(cdf, unit53(d[c]), side="right"))
    # split invariance for every model
    for m, dm in [("fig1", None), ("moons", None), ("char_mlp", None), ("gpt", [17, 8, 16, 2, 2, 32]), ("wide_mlp", dims)]:
        xa, ka = tg.synth_ctr(m, dm, dt, seed=9, first=0, batch=1000)
        xb, kb = tg.synth_ctr(m, dm, dt, seed=9, first=333, batch=401)
        assert np.array_equal(xa[:, 333:734], xb) and np.array_equal(ka[:, 333:734], kb)


def test_counter_synth_math_accuracy():
    """Moons: the generator's own cos/sin/log polynomials (tg_synth.cuh) against
    libm through the restated draws: x = arc(theta) + N(0, 0.1) noise agrees to
    a few ulp of 1, labels exactly."""
    from helpers import below, ctr_draws, unit53
    b = 20000
    x, _ = tg.synth_ctr("moons", dtype="f64", seed=77, first=5, batch=b)
    d = ctr_draws(77, np.arange(5, 5 + b), 6)
    second = below(d[0], 2) == 1
    th = np.pi * unit53(d[1])
    a, c = np.cos(th), np.sin(th)
    a = np.where(second, 1.0 - a, a)
    c = np.where(second, 0.5 - c, c)

    def noise(u1, u2):
        return 0.1 * np.sqrt(-2.0 * np.log(1.0 - unit53(u1))) * np.cos(2 * np.pi * unit53(u2))
    assert np.max(np.abs(x[0] - (a + noise(d[2], d[3])))) < 2e-15
    assert np.max(np.abs(x[1] - (c + noise(d[4], d[5])))) < 2e-15
    assert np.array_equal(x[2], np.where(second, 1.0, -1.0))


def test_null_program_handle_is_invalid_handle_everywhere():
    """Every entry point that takes a program handle returns TG_INVALID_HANDLE
    for NULL instead of dereferencing it (reference InvalidHandle,
    tape.hpp:268-273)."""
    L = _lib.lib
    P = None
    i = _lib.tg_program_info()
    pu32 = ctypes.POINTER(ctypes.c_uint32)()
    n32, sz, i64 = ctypes.c_uint32(), ctypes.c_size_t(), ctypes.c_int64()
    d, u64 = ctypes.c_double(), ctypes.c_uint64()
    s = ctypes.c_char_p()
    calls = {
        "tg_program_info_get": lambda: L.tg_program_info_get(P, ctypes.byref(i)),
        "tg_program_order": lambda: L.tg_program_order(P, ctypes.byref(pu32), ctypes.byref(n32)),
        "tg_workspace_size": lambda: L.tg_workspace_size(P, 10, ctypes.byref(sz)),
        "tg_set_memory_budget": lambda: L.tg_set_memory_budget(P, 10),
        "tg_forward_backward": lambda: L.tg_forward_backward(P, None, None, 1, None, None, None, None, None, 0, None),
        "tg_gd_update": lambda: L.tg_gd_update(P, None, None, 0.1, 1, None),
        "tg_allreduce_gd_step": lambda: L.tg_allreduce_gd_step(P, None, None, 0.1, 1, None, None),
        "tg_train_step": lambda: L.tg_train_step(P, None, None, 1, None, None, None, 0.1, None, 0, None),
        "tg_check_device_error": lambda: L.tg_check_device_error(P, None, ctypes.byref(i64), ctypes.byref(n32)),
        "tg_profile_enable": lambda: L.tg_profile_enable(P, 1),
        "tg_profile_read": lambda: L.tg_profile_read(P, ctypes.byref(d), ctypes.byref(u64)),
        "tg_program_jit": lambda: L.tg_program_jit(P, ctypes.byref(s), ctypes.byref(s), ctypes.byref(d)),
        "tg_pipeline_new": lambda: L.tg_pipeline_new(P, 1, None, None, ctypes.byref(ctypes.c_void_p())),
    }
    for name, f in calls.items():
        assert f() == 3, name
    assert L.tg_launch_count(P) == 0


def test_nccl_binding_and_argument_checks():
    """The NCCL exchange is bound at run time (tg_comm.cpp): the library
    reports the bound version, and bad communicator arguments are rejected
    before NCCL is called."""
    L = _lib.lib
    v = L.tg_nccl_version()
    assert v == 0 or v >= 21000
    h = ctypes.c_void_p()
    uid = (ctypes.c_char * 128)()
    assert L.tg_nccl_comm_init(2, uid, 2, ctypes.byref(h)) == 1
    assert L.tg_nccl_comm_init(0, uid, 0, ctypes.byref(h)) == 1
    assert L.tg_nccl_comm_init(1, None, 0, ctypes.byref(h)) == 1
    assert L.tg_nccl_get_unique_id(None) == 1
    assert L.tg_nccl_comm_destroy(None) == 0
    assert _lib.lib.tg_status_name(10).decode() == "TG_NCCL"


def test_fused_mlp_recogniser_accepts_the_composition_only(monkeypatch):
    """tg_fused.cu's pattern (gathers -> dense(act) -> dense -> softmax CE) is
    recognised exactly in the compiled graph (opt-in TG_FUSED_MLP=1): char-MLP
    variants are, the other workloads and a CE with an extra node are not."""
    monkeypatch.setenv("TG_FUSED_MLP", "1")
    monkeypatch.setenv("TG_STAGED", "1")
    for dims in (None, [27, 5, 6, 96], [40, 2, 16, 192]):
        d = tg.build_model("char_mlp", dims, "f32", seed=0).describe()
        assert tg.Program(d).info["fused_mlp"] == 1, dims
    assert tg.Program(tg.build_model("char_mlp", [40, 2, 16, 256], "f32", seed=0).describe()).info["fused_mlp"] == 0  # smem
    assert tg.Program(tg.build_model("char_mlp", None, "f64", seed=0).describe()).info["fused_mlp"] == 0
    for name, dims in (("wide_mlp", [24, 16, 12, 10]), ("gpt", [11, 6, 8, 2, 2, 16])):
        assert tg.Program(tg.build_model(name, dims, "f32", seed=0).describe()).info["fused_mlp"] == 0
    # the composition as tg_models.hpp records it (all inner products, then the
    # activations); with one extra node on the loss (x 1.0) it is not the pattern
    t = tg.Tape(4096, "f32")
    V, C, E, H = 5, 2, 3, 8
    emb = [t.param(0.01 * i) for i in range(V * E)]
    x = [t.gather(emb[0], E, V, c, e, 1) for c in range(C) for e in range(E)]
    w1 = [[t.param(0.02 * (j + k)) for k in range(C * E)] for j in range(H)]
    b1 = [t.param(0.0) for _ in range(H)]
    h = [t.unary(OpKind.Tanh, zj) for zj in [t.inner_product_with_bias(x, w1[j], b1[j]) for j in range(H)]]
    w2 = [[t.param(0.03 * (c - j)) for j in range(H)] for c in range(V)]
    b2 = [t.param(0.0) for _ in range(V)]
    z = [t.inner_product_with_bias(h, w2[c], b2[c]) for c in range(V)]
    m = t.op(OpKind.StopGradMax, z)
    sh = [t.sub(zc, m) for zc in z]
    lse = t.unary(OpKind.Log, t.reduce_sum([t.unary(OpKind.Exp, s) for s in sh]))
    zt = t.gather(sh[0], 1, V, C, 0, 2)
    loss = t.sub(lse, zt)
    t.set_root(loss)
    assert tg.Program(t.describe()).info["fused_mlp"] == 1
    t.set_root(t.mul_by_constant(loss, 1.0))
    assert tg.Program(t.describe()).info["fused_mlp"] == 0
