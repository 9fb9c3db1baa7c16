"""give_way (swarmsim/scenarios/give_way.py), fused reward / observation.

Two wide agents swap ends of a corridor with one recess.  Physics (the walls
are line segments) is world_step's generic kernel, launched first; the rest
of the step — count, reward -gap + 5 * (gap < 0.15) in float64 cast to
float32, done when both agents are home, observation with the float64 alcove
offsets — is k_give_way (csrc/ss_small.cu).  Resets run the reference's host
program.
"""
from __future__ import annotations

from .. import _native as N
from ..core import World
from . import register
from ._fused import FusedScenario, HostReset, f32
from .catalog import GiveWay as _Reference


@register("give_way")
class GiveWay(HostReset, FusedScenario):
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

    def physics_fused(self, world) -> bool:
        return False         # world_step's generic kernel, then k_give_way

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def fill_constants(self, world, d):
        d.sc[0] = f32(0.15)
        d.sd[0], d.sd[1] = float(self.alcove[0]), float(self.alcove[1])
