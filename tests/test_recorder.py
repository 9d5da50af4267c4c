"""Recorder invariants of the reference Tape through the C-ABI (CPU only):
rewind discipline (acceptance 7; tape.hpp:228-242), peak_nodes
examples, fixed-capacity errors (tape.hpp:79-81, :278-295),
and the memory-invariance identity of the per-sample loop (SPEC.md:645,
acceptance 5; the peak node count of a train step equals the
single-sample peak for every b)."""
import numpy as np
import pytest

import paper_2503_13795_b200 as tg
from paper_2503_13795_b200.tape import OpKind


def build_block(t, xs, width):
    """A tanh layer of `width` inner products over xs (children + bias)."""
    out = []
    for j in range(width):
        ws = [t.constant(0.1 * (j + 1) + 0.01 * i) for i in range(len(xs))]
        out.append(t.unary(OpKind.Tanh, t.inner_product_with_bias(ws, xs, t.constant(0.05 * j))))
    return out


def values(t, refs):
    return np.array([t.value_of(r) for r in refs])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_rewind_round_trip_restores_state_exactly(dtype):
    t = tg.Tape(4096, dtype)
    a, b = t.leaf(0.25), t.leaf(-1.5)
    prefix = [a, b] + build_block(t, [a, b], 4)
    before = t.stats()
    vals = values(t, range(before["size"]))
    cp = t.checkpoint()
    assert cp.mark == before["size"] and cp.child_mark == before["child_pool_size"]
    suffix = build_block(t, prefix[2:], 6)
    assert t.size() > cp.mark
    t.rewind(cp)
    after = t.stats()
    assert after["size"] == before["size"]
    assert after["child_pool_size"] == before["child_pool_size"]
    # surviving values byte-identical
    assert values(t, range(after["size"])).tobytes() == vals.tobytes()
    # handles into the discarded range are stale
    with pytest.raises(tg.TgError, match="TG_INVALID_HANDLE"):
        t.value_of(suffix[0])
    # the next node reuses raw index mark
    n = t.add(a, b)
    assert n == cp.mark
    assert t.value_of(n) == pytest.approx(-1.25)


def test_rewind_ahead_is_invalid_checkpoint():
    t = tg.Tape(64)
    t.leaf(1.0)
    cp = t.checkpoint()
    cp.mark = 7
    with pytest.raises(tg.TgError, match="TG_INVALID_CHECKPOINT.*rewind: checkpoint mark 7 is ahead of tape size 1"):
        t.rewind(cp)
    assert t.size() == 1


def test_peak_nodes_examples():
    # SPEC.md:84-87
    assert tg.Tape(16).peak_nodes() == 0
    t = tg.Tape(16)
    cp0 = t.checkpoint()
    for i in range(5):
        t.leaf(float(i))
    t.rewind(cp0)
    assert t.size() == 0 and t.peak_nodes() == 5
    t = tg.Tape(16)
    t.leaf(1.0), t.leaf(2.0)
    base = t.checkpoint()
    for _ in range(10):
        x = t.leaf(3.0)
        y = t.add(x, 0)
        t.mul(y, 1)
        t.rewind(base)
    assert t.peak_nodes() == 5
    st = t.stats()
    assert st["peak_children"] == 4 and st["size"] == 2 and st["child_pool_size"] == 0


def test_fixed_capacity_errors_leave_tape_unchanged():
    with pytest.raises(tg.InvalidArgument, match="Tape: capacity must be >= 1"):
        tg.Tape(0, fixed_capacity=True)
    t = tg.Tape(4, fixed_capacity=True)
    xs = [t.leaf(float(i)) for i in range(4)]
    with pytest.raises(tg.TgError, match="TG_CAPACITY.*tape capacity exceeded: 4 nodes"):
        t.add(xs[0], xs[1])
    assert t.size() == 4 and t.stats()["child_pool_size"] == 0
    t = tg.Tape(16, fixed_capacity=True, child_capacity=3)
    xs = [t.leaf(float(i)) for i in range(4)]
    with pytest.raises(tg.TgError, match="TG_CAPACITY.*tape child pool capacity exceeded: 3 entries"):
        t.reduce_sum(xs)
    assert t.size() == 4 and t.stats()["child_pool_size"] == 0
    s = t.reduce_sum(xs[:3])       # still fits exactly
    assert t.value_of(s) == 3.0


@pytest.mark.parametrize("b", [1, 8, 64])
def test_peak_nodes_of_a_train_step_is_independent_of_batch(b):
    """per sample, rewind to the post-parameter checkpoint and
    re-record; the step's peak node count equals the single-sample peak."""
    rng = np.random.default_rng(5)
    t = tg.Tape(1 << 14)
    w = [[t.param(float(v)) for v in rng.normal(0, 0.3, 2)] for _ in range(8)]
    bias = [t.param(0.0) for _ in range(8)]
    w2 = [t.param(float(v)) for v in rng.normal(0, 0.3, 8)]
    after_params = t.checkpoint()
    peaks = []
    for i in range(b):
        t.rewind(after_params)
        x = [t.input(0, float(rng.uniform(-1, 1))), t.input(1, float(rng.uniform(-1, 1)))]
        h = [t.unary(OpKind.Tanh, t.inner_product_with_bias(w[j], x, bias[j])) for j in range(8)]
        t.set_root(t.inner_product(w2, h))
        peaks.append(t.stats()["size"])
    single = peaks[0]
    assert t.peak_nodes() == single == max(peaks)
    assert t.stats()["peak_arena_bytes"] > 0
