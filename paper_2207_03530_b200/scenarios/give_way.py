"""give_way (swarmsim/scenarios/give_way.py), fused reward / observation.

Two wide agents swap ends of a corridor with one recess.  Physics (the walls
are line segments) is world_step's generic kernel, launched first; the rest
of the step — count, reward -gap + 5 * (gap < 0.15) in float64 cast to
float32, done when both agents are home, observation with the float64 alcove
offsets — is k_give_way (csrc/ss_small.cu).  Resets run the reference's host
program.
"""
from __future__ import annotations

import numpy as np

from .. import _native as N
from ..core import World
from . import register
from ._fused import FusedScenario, RefHeuristic, ResetProgram, f32
from .catalog import GiveWay as _Reference


@register("give_way")
class GiveWay(RefHeuristic, FusedScenario):
    native_id = N.SCN_GIVE_WAY
    max_steps = 300
    _reference = _Reference

    def __init__(self, agent_radius: float = 0.12, corridor_half_width: float = 0.2):
        self.agent_radius, self.half_width = agent_radius, corridor_half_width
        self.alcove = (0.0, 0.35)

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def obs_dim(self, world):
        return 12

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def fill_constants(self, world, d):
        d.sc[0] = f32(0.15)
        d.sd[0], d.sd[1] = float(self.alcove[0]), float(self.alcove[1])

    def reset_program(self, world):
        """give_way.py:48-72: each agent drawn (x then y) at its corridor end,
        goals, walls and the alcove (its side walls turned upright)."""
        p, idx, hw = ResetProgram(), world.index_of, self.half_width
        a0, a1 = world.agents
        for agent, lo, hi in ((a0, -1.6, -1.4), (a1, 1.4, 1.6)):
            p.scatter(idx(agent), (lo, -0.04), (hi, 0.04))     # x block, then y block
        p.place(idx(world.entity("goal_0")), 1.5, 0.0)
        p.place(idx(world.entity("goal_1")), -1.5, 0.0)
        p.place(idx(world.entity("wall_bottom")), 0.0, -hw)
        p.place(idx(world.entity("wall_top_left")), -1.15, hw)
        p.place(idx(world.entity("wall_top_right")), 1.15, hw)
        for name, x in (("alcove_left", -0.3), ("alcove_right", 0.3)):
            k = idx(world.entity(name))
            p.place(k, x, hw + 0.15)
            p.setrot(k, p.const(np.pi / 2))
        p.place(idx(world.entity("alcove_top")), 0.0, hw + 0.3)
        return p
