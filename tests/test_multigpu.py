"""CPU: the data-parallel path with world_size 2 over gloo.

Each rank owns a contiguous shard, computes its local gradient sum (the
oracle stands in for the device program here — no GPU on the build box),
all-reduces it and applies the GD update with the global batch size.  The
result must equal the single-process full-batch step, and both ranks must
hold identical parameters."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2503_13795_b200 as tg
from paper_2503_13795_b200.dp import DataParallelStep, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out, ctr=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    desc = tg.build_model("moons").describe()
    b = 1000
    lo, hi = shard(b, rank, world)
    if ctr:   # each rank generates only its own shard (counter-based generator, §8f row 2)
        xs, ks = tg.synth_ctr("moons", seed=4, first=lo, batch=hi - lo)
        x = np.zeros((xs.shape[0], b)); x[:, lo:hi] = xs
        k = np.zeros((0, b), np.int32)
    else:
        x, k = tg.synth_batch("moons", batch=b, seed=4)
    params = torch.tensor(desc.param_values(), dtype=torch.float64)
    grad = torch.zeros(desc.n_params, dtype=torch.float64)

    def local_grad(p):
        r = oracle.run(desc, x[:, lo:hi], k[:, lo:hi], p.numpy())
        grad.copy_(torch.from_numpy(r["grad_sum"]))

    dp = DataParallelStep()
    for _ in range(3):
        dp.step(params, grad, 0.05, b, local_grad)
    gathered = [torch.zeros_like(params) for _ in range(world)]
    dist.all_gather(gathered, params)
    if rank == 0:
        out.put([g.numpy() for g in gathered])
    dist.destroy_process_group()


def test_shard_covers_batch():
    for b in (1, 7, 1000, 65536):
        for w in (1, 2, 3, 8):
            parts = [shard(b, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == b
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1
    with pytest.raises(ValueError):
        shard(10, 2, 2)


@pytest.mark.parametrize("ctr", [False, True])
def test_world_size_2_gloo_equals_full_batch(ctr):
    """ctr: every rank generates its own shard with the counter-based
    generator (no data exchange); the full-batch reference generates samples
    [0, b) in one call."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, ctr)) for r in range(2)]
    for p in ps:
        p.start()
    res = q.get(timeout=180)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(res[0], res[1])          # replicas stay identical
    # single-process reference: three full-batch steps
    desc = tg.build_model("moons").describe()
    x, k = tg.synth_ctr("moons", seed=4, first=0, batch=1000) if ctr else tg.synth_batch("moons", batch=1000, seed=4)
    p = desc.param_values().copy()
    for _ in range(3):
        g = oracle.run(desc, x, k, p)["grad_sum"]
        oracle.sgd("f64", p, g, 0.05, 1000)
    assert np.linalg.norm(res[0] - p) / np.linalg.norm(p) <= 1e-13
