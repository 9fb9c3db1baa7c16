"""Multi-GPU sharding: one process per GPU, contiguous env shards.

Environments are independent (the result at env e depends only on inputs at
e — batching.py:1-9), so the batch shards across GPUs with no collective in
the step.  Rank r of N holds the global env range shard_range(r, N, Bg) and
keeps the reference's GLOBAL random-stream layout (Env(env_offset=...,
global_batch=...)), so an N-GPU run is bitwise the 1-GPU run of Bg envs.

The two real exchange steps, both over torch.distributed (NCCL on NVLink for
GPUs, gloo for the CPU tests), both outside the step:
  * episode statistics: one all_reduce(SUM) of a small float64 vector;
  * a sharded masked reset: every rank needs the number of selected envs on
    lower ranks (its offset in the global draw order) and the global total
    (how far the shared stream advances) — one all_gather of an int64.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(rank: int, world_size: int, global_batch: int) -> tuple[int, int]:
    """(env_offset, batch) of `rank`: contiguous, remainder to the first ranks."""
    if not 0 <= rank < world_size:
        raise ValueError(f"rank {rank} outside world of {world_size}")
    base, rem = divmod(global_batch, world_size)
    count = base + (1 if rank < rem else 0)
    offset = rank * base + min(rank, rem)
    return offset, count


def make_sharded_env(scenario, global_batch: int, rank: int | None = None, world_size: int | None = None,
                     seed: int = 0, device=None, **kwargs):
    """Env holding this rank's shard of a global_batch-env run."""
    from .env import Env

    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if world_size is None:
        world_size = dist.get_world_size() if dist.is_initialized() else 1
    off, count = shard_range(rank, world_size, global_batch)
    return Env(scenario, count, seed=seed, device=device, env_offset=off, global_batch=global_batch, **kwargs)


def global_mask_offsets(local_count: torch.Tensor, group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """(#selected on lower ranks, #selected overall) for a sharded masked reset.

    local_count: int64 tensor of shape (1,) on this rank's device.  Returns two
    (1,) int64 tensors on the same device; no host synchronisation.
    """
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return torch.zeros_like(local_count), local_count.clone()
    ws = dist.get_world_size(group)
    gathered = [torch.empty_like(local_count) for _ in range(ws)]
    dist.all_gather(gathered, local_count, group=group)
    counts = torch.cat(gathered)
    rank = dist.get_rank(group)
    base = counts[:rank].sum().reshape(1)
    total = counts.sum().reshape(1)
    return base, total


def reset_at_sharded(env, mask, group=None):
    """Env.reset_at for one shard of a sharded run (global stream order)."""
    import ctypes

    from . import _native as N
    from .env import _as_mask

    m = _as_mask(mask, env.batch_size, env.device)
    sc, world = env.scenario, env.world
    if not env.fused:
        raise NotImplementedError("sharded reset_at is provided for the built-in scenarios")
    h = sc.native_handle(world)
    count = torch.zeros(1, dtype=torch.int64, device=env.device)
    m8 = m.to(torch.uint8).contiguous()
    N.check(N.lib().ss_mask_count(h.handle, N.ptr(m8), N.ptr(count), N.stream_handle(env.device)))
    base, total = global_mask_offsets(count, group)
    sc.reset_world_masked(world, m8, base, total)
    return env.observations()


class EpisodeStats:
    """Per-shard episode accounting on the device, reduced across ranks.

    update() follows run_episode's rule (rollout.py:46-69): the mean reward
    over non-scripted agents counts until (and including) each env's first
    done.  reduce() is one all_reduce(SUM) of [return_sum, finished, env_steps].
    """

    def __init__(self, batch_size: int, device):
        self.returns = torch.zeros(batch_size, dtype=torch.float64, device=device)
        self.alive = torch.ones(batch_size, dtype=torch.bool, device=device)
        self.env_steps = torch.zeros((), dtype=torch.float64, device=device)

    def update(self, rewards, dones) -> None:
        r = torch.stack(list(rewards)).to(torch.float64).mean(dim=0)
        self.returns += torch.where(self.alive, r, torch.zeros_like(r))
        self.alive &= ~dones
        self.env_steps += self.alive.numel()

    def reduce(self, group=None) -> dict:
        v = torch.stack([self.returns.sum(), (~self.alive).sum().to(torch.float64),
                         torch.tensor(float(self.returns.numel()), dtype=torch.float64, device=self.returns.device),
                         self.env_steps])
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
        s = v.tolist()
        return {"mean_return": s[0] / max(s[2], 1.0), "finished": s[1], "envs": s[2], "env_steps": s[3]}
