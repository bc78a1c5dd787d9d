"""Multi-GPU modes of the superposed gradient.

shot-parallel: one process per GPU (torchrun, NCCL).  Rank r evaluates shots
r, r+P, r+2P, ... into its own device accumulator; the unscaled accumulators
and the costs are summed with one all-reduce per evaluation, then every rank
applies acc /= T(2k).  Summation order differs from the reference's serial
shared accumulator, so this mode is NOT bitwise (the reference itself notes
shot concurrency); it is the throughput mode for multi-shot
problems that fit one GPU.  ``shot_partition`` and ``reduce_plan`` hold the
host logic and are exercised with gloo on CPU in tests/test_distributed_cpu.py.
"""

from __future__ import annotations

import numpy as np


def shot_partition(n_shots, rank, world):
    """Round-robin shot indices owned by rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return list(range(rank, n_shots, world))


def accumulator_tensor(ctx):
    """Zero-copy torch view of a DeviceGrid's accumulator (CUDA array interface)."""
    import torch

    ptr = ctx.L.wo_accumulator_ptr(ctx.h)
    typestr = "<f4" if ctx.dtype.itemsize == 4 else "<f8"

    class _View:
        __cuda_array_interface__ = {"shape": tuple(ctx.grid.shape), "typestr": typestr,
                                    "data": (int(ptr), False), "version": 3, "strides": None}

    return torch.as_tensor(_View(), device=f"cuda:{ctx.device}")


def reduce_plan(acc, cost, group=None):
    """Sum accumulators (in place) and costs over the process group."""
    import torch
    import torch.distributed as dist

    dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    c = torch.tensor([cost], dtype=torch.float64, device=acc.device)
    dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
    return float(c.item())


class ShotParallelGradient:
    """gradient_superposed split over ranks by shots (device-resident)."""

    def __init__(self, problem, material, config, rank, world, group=None):
        from .gradients import SuperposedPlan, _shot_list

        n_shots = len(_shot_list(problem))
        self.plan = SuperposedPlan(problem, material, config,
                                   shot_indices=shot_partition(n_shots, rank, world))
        self.group = group
        self.acc = None

    def upload(self):
        self.plan.upload()
        self.acc = accumulator_tensor(self.plan.ctx)
        return self

    def run(self):
        import torch

        cost = self.plan.run(finish=False)          # synchronous on the library stream
        cost = reduce_plan(self.acc, cost, self.group)
        torch.cuda.current_stream().synchronize()   # NCCL done before the library reuses acc
        self.plan.finish()
        return cost

    def download(self):
        return self.plan.download()
