"""Data-parallel gradient oracle across GPUs (north_star (d)).

One process per GPU.  The batch is sharded into contiguous per-rank slices,
parameters are replicated, every rank computes its local sum of per-sample
gradients with the device program, one all-reduce (sum) of the d-length
gradient runs over NCCL / NVLink, and every rank applies the same GD update
x -= gamma * g / b_global (sgd_step) — identical parameters
on all ranks without a broadcast.

The reference has no parallelism (PAPER.md:748 single core); this is the
B200 build's scaling axis.  The path has exactly one exchange per step, so
the collective is torch.distributed's NCCL all-reduce (NVLS in-switch
reduction when NCCL selects it).
"""
from __future__ import annotations


def shard(global_batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of the batch owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    return global_batch * rank // world, global_batch * (rank + 1) // world


class DataParallelStep:
    """One DP training step over a compiled Program.

    local_grad(params) must fill and return the local gradient sum tensor
    (by default Program.forward_backward on this rank's shard).
    """

    def __init__(self, program=None, group=None):
        self.program = program
        self.group = group

    def step(self, params, grad, gamma: float, global_batch: int, local_grad=None, stream=None):
        import torch.distributed as dist

        if local_grad is not None:
            local_grad(params)
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=self.group)
        if self.program is not None:
            self.program.gd_update(params, grad, gamma, global_batch, stream)
        else:  # host-side update for CPU process groups (tests): same formula as k_gd
            params.sub_(gamma * grad / global_batch)
        return params
