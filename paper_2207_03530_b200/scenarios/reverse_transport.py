"""reverse_transport (swarmsim/scenarios/reverse_transport.py), fused.

Agents trapped inside a hollow crate drive it to a goal.  The world is
transport's (agents, a movable non-rotatable box, a goal marker; pairs
agent-agent then (agent, crate) per agent; sphere-box contacts on the box
perimeter), so the step is k_transport<n, 1> (csrc/ss_small.cu): the same
physics and reward (-|crate - goal|, float32; done when < success_dist) with
the reverse observation [x, y, vx, vy, crate - self, crate vel, goal - crate].
Resets place the agents relative to the freshly drawn crate; they run the
reference's host program (catalog.ReverseTransport.reset_world_at) on the
Env's Philox stream, one env at a time for masked resets.
"""
from __future__ import annotations

import torch

from ..core import World
from ..errors import ContractViolation
from . import register
from .catalog import ReverseTransport as _Reference
from .transport import Transport


@register("reverse_transport")
class ReverseTransport(Transport):
    max_steps = 250

    def __init__(self, n_agents: int = 4, crate_size: float = 0.6, crate_mass: float = 3.0,
                 success_dist: float = 0.1):
        super().__init__(n_agents=n_agents, package_mass=crate_mass, package_size=crate_size,
                         success_dist=success_dist)
        self.crate_size, self.crate_mass = crate_size, crate_mass

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def reset_ops(self, world):
        return []            # resets run on the host (reset_world_at)

    def obs_dim(self, world):
        return 10

    def fill_constants(self, world, d):
        super().fill_constants(world, d)
        d.si[1] = 1          # reverse observation layout

    def reset_world_at(self, world: World, env_index: int | None = None) -> None:
        _Reference.reset_world_at(self, world, env_index)

    def reset_world_masked(self, world: World, mask: torch.Tensor, mask_base=None, mask_total=None) -> None:
        if mask_base is not None:
            raise ContractViolation("reverse_transport resets on the host: no sharded masked reset")
        for i in torch.nonzero(mask).flatten().tolist():
            self.reset_world_at(world, i)
            world.step_count[i] = 0

    def heuristic_action(self, agent_index: int, obs):
        return _Reference.heuristic_action(self, agent_index, obs)
