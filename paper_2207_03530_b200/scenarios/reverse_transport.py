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

from ..core import World
from . import register
from ._fused import HostReset
from .catalog import ReverseTransport as _Reference
from .transport import Transport


@register("reverse_transport")
class ReverseTransport(HostReset, Transport):
    max_steps = 250
    _reference = _Reference

    def __init__(self, n_agents: int = 4, crate_size: float = 0.6, crate_mass: float = 3.0,
                 success_dist: float = 0.1):
        super().__init__(n_agents=n_agents, package_mass=crate_mass, package_size=crate_size,
                         success_dist=success_dist)
        self.crate_size, self.crate_mass = crate_size, crate_mass

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def obs_dim(self, world):
        return 10

    def fill_constants(self, world, d):
        super().fill_constants(world, d)
        d.si[1] = 1          # reverse observation layout
