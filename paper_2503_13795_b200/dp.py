"""Data-parallel gradient oracle across GPUs (north_star (d)).

One process per GPU.  The batch is sharded into contiguous per-rank slices,
parameters are replicated, every rank computes its local sum of per-sample
gradients with the device program, one all-reduce (sum) of the d-length
gradient runs over NCCL / NVLink, and every rank applies the same GD update
x -= gamma * g / b_global (sgd_step) — identical parameters
on all ranks without a broadcast.

The reference has no parallelism (PAPER.md:748 single core); this is the
B200 build's scaling axis.  The path has exactly one exchange per step.  The
exchange runs either through libtg's own NCCL communicator
(tg_allreduce_gd_step, the C-ABI a C++ caller uses; `NcclComm`) or through
torch.distributed's all-reduce; both are enqueued on the caller's stream, so
the GD update that follows never races the reduction.
"""
from __future__ import annotations

import ctypes as C

from ._lib import check, lib


def shard(global_batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of the batch owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    return global_batch * rank // world, global_batch * (rank + 1) // world


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through libtg (rank 0 creates it, every rank receives it)."""
    buf = (C.c_char * 128)()
    check(lib.tg_nccl_get_unique_id(buf))
    return bytes(buf)


class NcclComm:
    """An NCCL communicator created by libtg (tg_nccl_comm_init) on the current
    CUDA device.  `uid` is rank 0's nccl_unique_id(); when it is None the id is
    broadcast from rank 0 over the initialised torch.distributed group (any
    backend)."""

    def __init__(self, rank: int, world: int, uid: bytes | None = None, group=None):
        if uid is None:
            import torch.distributed as dist
            obj = [nccl_unique_id() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(obj, src=0, group=group)
            uid = obj[0]
        h = C.c_void_p()
        check(lib.tg_nccl_comm_init(int(world), C.c_char_p(uid), int(rank), C.byref(h)))
        self.handle = h.value
        self.rank, self.world = rank, world

    def close(self):
        if getattr(self, "handle", None):
            check(lib.tg_nccl_comm_destroy(C.c_void_p(self.handle)))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _CudaArray:
    """__cuda_array_interface__ view of a raw device buffer (torch.as_tensor wraps it without a copy)."""

    def __init__(self, ptr: int, n: int, dtype: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8" if dtype == "f64" else "<f4",
                                         "data": (ptr, False), "version": 3, "strides": None}


class SymmetricWindow:
    """The gradient buffer of the fused exchange: NCCL
    symmetric memory on every rank of `comm` (tg_window_create).  `grad` is
    this rank's buffer as a torch tensor (zero-copy): pass it as grad_sum to
    forward_backward, then allreduce_gd() sums it over the ranks and applies
    the GD update in one kernel (multicast / NVLS when `multimem`, NVLink peer
    loads summed in rank order otherwise).  Collective on all ranks."""

    def __init__(self, comm: NcclComm, dtype: str, count: int, multimem: bool = True):
        import torch
        h = C.c_void_p()
        check(lib.tg_window_create(C.c_void_p(comm.handle), 0 if dtype == "f64" else 1, int(count),
                                   1 if multimem else 0, C.byref(h)))
        self.handle = h.value
        self.dtype, self.count = dtype, count
        self.multimem = bool(lib.tg_window_multimem(h))
        ptr = lib.tg_window_buffer(h)
        self.grad = torch.as_tensor(_CudaArray(ptr, count, dtype), device="cuda")

    def allreduce_gd(self, params, gamma: float, global_batch: int, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        check(lib.tg_window_allreduce_gd(C.c_void_p(self.handle), C.c_void_p(params.data_ptr()), float(gamma),
                                         int(global_batch), C.c_void_p(s.cuda_stream)))
        return params

    def close(self):
        if getattr(self, "handle", None):
            self.grad = None
            check(lib.tg_window_destroy(C.c_void_p(self.handle)))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DataParallelStep:
    """One DP training step over a compiled Program.

    comm: an NcclComm (the exchange and the update go through
    tg_allreduce_gd_step on `stream`), or None to use torch.distributed's
    all-reduce (enqueued on `stream` too).  local_grad(params) must fill the
    local gradient sum tensor when given.
    """

    def __init__(self, program=None, group=None, comm: NcclComm | None = None, window: SymmetricWindow | None = None):
        self.program = program
        self.group = group
        self.comm = comm
        self.window = window   # fused exchange + GD (grad must be window.grad)

    def step(self, params, grad, gamma: float, global_batch: int, local_grad=None, stream=None):
        if local_grad is not None:
            local_grad(params)
        if self.window is not None:
            if grad is not None and grad.data_ptr() != self.window.grad.data_ptr():
                raise ValueError("DataParallelStep: with a window the gradient buffer is window.grad")
            return self.window.allreduce_gd(params, gamma, global_batch, stream)
        if self.comm is not None and self.program is not None:
            self.program.allreduce_gd_step(params, grad, gamma, global_batch, self.comm, stream)
            return params
        import torch.distributed as dist
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1
        if self.program is not None:
            import torch
            s = stream if stream is not None else torch.cuda.current_stream()
            with torch.cuda.stream(s):          # the all-reduce is ordered on the caller's stream
                if multi:
                    dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=self.group)
                self.program.gd_update(params, grad, gamma, global_batch, s)
        else:  # host-side update for CPU process groups (tests): same formula as k_gd
            if multi:
                dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=self.group)
            params.sub_(gamma * grad / global_batch)
        return params
