"""waterfall (swarmsim/scenarios/waterfall.py), fused reward / observation.

Agents drift down under gravity through staggered baffles to a basin.
Physics (gravity, sphere-box contacts) is world_step's generic kernel,
launched first; the rest of the step — count, reward -gap - penalty *
(touching teammates + block bumps via closest points, float64), done when
every agent is in the basin, observation — is k_waterfall<n>
(csrc/ss_small.cu).  Resets are a device reset program (ResetProgram).
"""
from __future__ import annotations

from .. import _native as N
from ..core import World
from ..shapes import min_contact_distance
from . import register
from ._fused import FusedScenario, RefHeuristic, ResetProgram, f32
from .catalog import BLOCKS, Waterfall as _Reference


@register("waterfall")
class Waterfall(RefHeuristic, FusedScenario):
    native_id = N.SCN_WATERFALL
    max_steps = 200
    _reference = _Reference

    def __init__(self, n_agents: int = 4, gravity: float = -0.2, collision_penalty: float = 0.3):
        _Reference.__init__(self, n_agents, gravity, collision_penalty)

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def obs_dim(self, world):
        return 6 + 2 * len(BLOCKS)

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def fill_constants(self, world, d):
        a = world.agents[0].shape
        d.sc[0] = f32(min_contact_distance(a, a) + 0.0)     # common.touching
        d.sc[1] = f32(a.radius)                             # _block_bumps: <= r
        d.sc[2] = f32(0.2)
        d.sd[0] = float(self.collision_penalty)
        d.si[2] = len(BLOCKS)

    def reset_program(self, world):
        """waterfall.py:52-62: agents drawn (x then y) along the top; the basin
        and the baffles placed."""
        from .catalog import BASIN

        p, idx = ResetProgram(), world.index_of
        for agent in world.agents:
            p.scatter(idx(agent), (-0.6, 0.75), (0.6, 0.95))
        p.place(idx(world.entity("basin")), *BASIN)
        for k, (bx, by) in enumerate(BLOCKS):
            p.place(idx(world.entity(f"block_{k}")), bx, by)
        return p
