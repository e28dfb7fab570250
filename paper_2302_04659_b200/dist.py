"""Multi-GPU plumbing: one process per GPU, environments sharded across ranks,
one collective per env step for the step statistics.

Environments are independent worlds (shell.hpp:392-397): no halo,
no particle migration, so the data path has no collective. The only exchange
is the per-env-step stats vector (particle-substeps, CFL cycles, lost
particles, max penetration, max force-balance error), all-reduced with NCCL
over NVLink on GPU ranks (gloo on CPU for the tests)."""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def shard(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous env range [lo, hi) of a rank (strong scaling of a fixed batch)."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def weak_first_env(n_per_rank: int, rank: int) -> int:
    """First global env id of a rank when every rank owns n_per_rank envs (weak scaling)."""
    return rank * n_per_rank


def rank_envs(n_envs: int, rank: int, world: int, weak: bool = False) -> tuple[int, int]:
    """(first global env id, env count) of a rank: the contiguous shard of a fixed
    batch of n_envs (strong scaling, bench.py's default), or n_envs of its own
    (weak). Seeds follow the global env id, so any world size steps the same
    per-env worlds."""
    if weak:
        return weak_first_env(n_envs, rank), n_envs
    lo, hi = shard(n_envs, rank, world)
    return lo, hi - lo


class LibStats:
    """The library's own statistics exchange (msim_gpu_comm_init / msim_gpu_step_stats):
    device-side reduction + NCCL all-reduce on the context stream. The NCCL id is
    made by rank 0 and broadcast over the torch process group (host plumbing)."""

    def __init__(self, lib, ctx, rank: int, world: int):
        import ctypes as C

        import numpy as np

        self.lib, self.ctx, self.C, self.np = lib, ctx, C, np
        uid = np.zeros(128, dtype=np.uint8)
        if rank == 0 and lib.msim_gpu_nccl_unique_id(uid.ctypes.data_as(C.POINTER(C.c_uint8))) != 0:
            raise RuntimeError(lib.msim_gpu_create_error().decode())
        if world > 1:
            box = [uid.tobytes()]
            dist.broadcast_object_list(box, src=0)
            uid = np.frombuffer(box[0], dtype=np.uint8).copy()
        if lib.msim_gpu_comm_init(ctx, rank, world, uid.ctypes.data_as(C.POINTER(C.c_uint8))) != 0:
            raise RuntimeError(lib.msim_gpu_last_error(ctx).decode())

    def step(self) -> StepStats:
        sums, maxs = self.np.zeros(4), self.np.zeros(2)
        dp = self.C.POINTER(self.C.c_double)
        if self.lib.msim_gpu_step_stats(self.ctx, 1, sums.ctypes.data_as(dp), maxs.ctypes.data_as(dp)) != 0:
            raise RuntimeError(self.lib.msim_gpu_last_error(self.ctx).decode())
        return StepStats(*sums.tolist(), *maxs.tolist())


@dataclass
class StepStats:
    particle_substeps: float = 0.0
    env_steps: float = 0.0
    cfl_cycles: float = 0.0
    lost_particles: float = 0.0
    max_penetration: float = 0.0
    max_force_balance_error: float = 0.0

    @classmethod
    def from_reports(cls, reports, particles_per_env, substeps):
        s = cls()
        for r, n in zip(reports, particles_per_env):
            s.particle_substeps += n * substeps
            s.env_steps += 1
            s.cfl_cycles += r.cfl_cycles
            s.lost_particles += r.lost_particles
            s.max_penetration = max(s.max_penetration, r.max_penetration)
            s.max_force_balance_error = max(s.max_force_balance_error, r.max_force_balance_error)
        return s


def allreduce_stats(s: StepStats, device=None) -> StepStats:
    """Sum the counters and max the diagnostics over all ranks (2 tiny collectives)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return s
    dev = device if device is not None else ("cuda" if dist.get_backend() == "nccl" else "cpu")
    sums = torch.tensor([s.particle_substeps, s.env_steps, s.cfl_cycles, s.lost_particles], dtype=torch.float64,
                        device=dev)
    maxs = torch.tensor([s.max_penetration, s.max_force_balance_error], dtype=torch.float64, device=dev)
    dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    dist.all_reduce(maxs, op=dist.ReduceOp.MAX)
    a, b = sums.tolist(), maxs.tolist()
    return StepStats(a[0], a[1], a[2], a[3], b[0], b[1])
