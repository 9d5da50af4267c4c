"""Pins the fp64 PyTorch restatement (tests/torch_ref.py) against the oracle
(the reference per-sample algorithm over the recorded fp64 tape) before the
GPU tests use it as the checker at the BASELINE batch sizes the oracle cannot
run in seconds (cfg4 b = 8,192; cfg5 b = 32,768 / 1,048,576)."""
import os

import numpy as np
import pytest

import oracle
import paper_2503_13795_b200 as tg
import torch_ref
from helpers import rel


@pytest.mark.parametrize("name,dims,b", [("moons", None, 300), ("char_mlp", None, 257), ("wide_mlp", None, 64),
                                         ("wide_mlp", [40, 30, 20, 10], 500), ("gpt", [13, 8, 32, 2, 2, 64], 20),
                                         ("gpt", None, 2)])
def test_torch_restatement_equals_oracle_f64(name, dims, b):
    desc = tg.build_model(name, dims, "f64", seed=9).describe()
    x, k = tg.synth_batch(name, dims, "f64", seed=31, batch=b, n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
    p = desc.param_values()
    r = oracle.run(desc, x, k, p, threads=os.cpu_count() or 8)
    t = torch_ref.run(name, dims, p, x if desc.n_inputs else None, k if desc.n_index_inputs else None)
    assert len(t["grad_sum"]) == desc.n_params
    assert rel(t["loss"], r["loss"]) <= 1e-12
    assert np.max(np.abs(t["loss"] - r["loss"]) / np.maximum(1e-12, np.abs(r["loss"]))) <= 1e-11
    assert rel(t["grad_sum"], r["grad_sum"]) <= 1e-12
