"""GPU: the data-parallel step around the real device Program (north_star
(d)) with single-rank NCCL communicators — libtg's own
(tg_nccl_comm_init + tg_allreduce_gd_step, the C-ABI path) and
torch.distributed's (DataParallelStep on the caller's stream).  With one rank
the all-reduce is the identity, so the step must equal the fused train_step
bit for bit and the oracle's per-sample loop + sgd_step to the dtype's bar;
the multi-rank reduction identity is covered by test_shard_invariance and the
gloo test (tests/test_multigpu.py)."""
import os
import socket

import numpy as np
import pytest

import oracle
import paper_2503_13795_b200 as tg
from helpers import TOL, rel, tdtype
from paper_2503_13795_b200.dp import DataParallelStep, NcclComm, nccl_unique_id

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _setup(name, dt, b):
    desc = tg.build_model(name, None, dt, seed=2).describe()
    x, k = tg.synth_batch(name, None, dt, seed=8, batch=b, n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
    prog = tg.Program(desc)
    T = tdtype(dt)
    X = torch.tensor(x, device="cuda") if desc.n_inputs else None
    K = torch.tensor(k, device="cuda") if desc.n_index_inputs else None
    return desc, x, k, prog, T, X, K


@pytest.mark.parametrize("name,dt,b", [("moons", "f64", 4096), ("char_mlp", "f32", 4096)])
@pytest.mark.parametrize("path", ["tg_nccl", "torch_nccl"])
def test_dp_step_single_rank_nccl_equals_train_step(name, dt, b, path):
    desc, x, k, prog, T, X, K = _setup(name, dt, b)
    W = prog.alloc_workspace(b)
    P1 = torch.tensor(desc.param_values(), device="cuda", dtype=T)
    P2 = P1.clone()
    L = torch.zeros(b, device="cuda", dtype=T)
    G1 = torch.zeros(desc.n_params, device="cuda", dtype=T)
    G2 = torch.zeros_like(G1)
    side = torch.cuda.Stream()          # not torch's current stream: ordering must follow it
    prog.train_step(X, K, b, P1, L, G1, 0.05, W)
    torch.cuda.synchronize()
    if path == "tg_nccl":
        assert tg._lib.lib.tg_nccl_version() >= 22000
        comm = NcclComm(0, 1, uid=nccl_unique_id())
        dp = DataParallelStep(prog, comm=comm)
    else:
        import torch.distributed as dist
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        dp = DataParallelStep(prog)
    try:
        for _ in range(3):
            side.wait_stream(torch.cuda.current_stream())
            prog.forward_backward(X, K, b, P2, L, None, G2, W, stream=side)
            dp.step(P2, G2, 0.05, b, stream=side)
            torch.cuda.current_stream().wait_stream(side)
            if _ == 0:
                torch.cuda.synchronize()
                assert torch.equal(P1, P2) and torch.equal(G1, G2)
        torch.cuda.synchronize()
    finally:
        if path == "tg_nccl":
            comm.close()
        else:
            import torch.distributed as dist
            dist.destroy_process_group()
    p = desc.param_values().copy()
    for _ in range(3):
        r = oracle.run(desc, x.astype(np.float64), k, p, threads=os.cpu_count() or 8, want_input_grad=False)
        oracle.sgd(dt, p, r["grad_sum"], 0.05, b)
    assert rel(P2.cpu().double().numpy(), p) <= TOL[dt]


def test_allreduce_gd_step_without_comm_is_gd_update():
    desc, x, k, prog, T, X, K = _setup("moons", "f64", 1000)
    P1 = torch.tensor(desc.param_values(), device="cuda", dtype=T)
    P2 = P1.clone()
    G = torch.randn(desc.n_params, device="cuda", dtype=T)
    prog.gd_update(P1, G, 0.1, 1000)
    prog.allreduce_gd_step(P2, G, 0.1, 1000, comm=None)
    torch.cuda.synchronize()
    assert torch.equal(P1, P2)


@pytest.mark.parametrize("name,dt,b", [("moons", "f64", 4096), ("char_mlp", "f32", 4096), ("wide_mlp", "f32", 512)])
def test_fused_window_exchange_equals_nccl_path(name, dt, b):
    """§8f row 4: the fused exchange + GD kernel over NCCL symmetric memory
    (tg_window_allreduce_gd) against the NCCL path (tg_allreduce_gd_step) on a
    single-rank communicator: identical parameters and global gradient sums,
    bit for bit, over several steps (the window's barrier epochs advance)."""
    from paper_2503_13795_b200.dp import SymmetricWindow
    desc, x, k, prog, T, X, K = _setup(name, dt, b)
    W = prog.alloc_workspace(b)
    comm = NcclComm(0, 1, uid=nccl_unique_id())
    try:
        win = SymmetricWindow(comm, dt, desc.n_params)
    except tg.TgError as e:
        comm.close()
        pytest.skip(f"no NCCL symmetric-memory device API here: {e}")
    try:
        P1 = torch.tensor(desc.param_values(), device="cuda", dtype=T)
        P2 = P1.clone()
        L = torch.zeros(b, device="cuda", dtype=T)
        G1 = torch.zeros(desc.n_params, device="cuda", dtype=T)
        dp = DataParallelStep(prog, window=win)
        side = torch.cuda.Stream()
        for _ in range(4):
            prog.forward_backward(X, K, b, P1, L, None, G1, W)
            prog.allreduce_gd_step(P1, G1, 0.05, b, comm)
            side.wait_stream(torch.cuda.current_stream())
            prog.forward_backward(X, K, b, P2, L, None, win.grad, W, stream=side)
            dp.step(P2, win.grad, 0.05, b, stream=side)
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            assert torch.equal(G1, win.grad), "global gradient sums differ"
            assert torch.equal(P1, P2), "parameters differ"
        assert not bool(torch.isnan(P2).any())
    finally:
        win.close()
        comm.close()


def test_fused_window_exchange_in_cuda_graph():
    """The fused exchange's barrier epochs live on the device, so a captured
    CUDA graph (forward_backward + tg_window_allreduce_gd) replays correctly:
    five replays equal five eager NCCL-path steps bit for bit."""
    from paper_2503_13795_b200.dp import SymmetricWindow
    desc, x, k, prog, T, X, K = _setup("char_mlp", "f32", 2048)
    b = 2048
    W = prog.alloc_workspace(b)
    comm = NcclComm(0, 1, uid=nccl_unique_id())
    try:
        win = SymmetricWindow(comm, "f32", desc.n_params)
    except tg.TgError as e:
        comm.close()
        pytest.skip(f"no NCCL symmetric-memory device API here: {e}")
    try:
        P1 = torch.tensor(desc.param_values(), device="cuda", dtype=T)
        P2 = P1.clone()
        L1 = torch.zeros(b, device="cuda", dtype=T)
        L2 = torch.zeros(b, device="cuda", dtype=T)
        G1 = torch.zeros(desc.n_params, device="cuda", dtype=T)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):     # warm-up call outside the capture (first-use allocations)
            prog.forward_backward(X, K, b, P2, L2, None, win.grad, W, stream=s)
            win.allreduce_gd(P2, 0.0, b, s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            prog.forward_backward(X, K, b, P2, L2, None, win.grad, W, stream=s)
            win.allreduce_gd(P2, 0.05, b, s)
        torch.cuda.synchronize()
        for _ in range(5):
            prog.forward_backward(X, K, b, P1, L1, None, G1, W)
            prog.allreduce_gd_step(P1, G1, 0.05, b, comm)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(G1, win.grad) and torch.equal(P1, P2) and torch.equal(L1, L2)
    finally:
        del g
        win.close()
        comm.close()
