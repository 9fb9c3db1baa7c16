"""passage (swarmsim/scenarios/passage.py), fused reward / observation.

A cross formation squeezes through two wall gaps and reforms.  Physics (the
walls are line segments) is world_step's generic kernel, launched first; the
rest of the step — count, reward -gap - penalty * #touching teammates
(float32), done when every agent sits within 0.05 of its slot, observation
with the float64 gap offsets — is k_passage<n> (csrc/ss_small.cu).  Resets
run the reference's host program (formation drawn around one centre).
"""
from __future__ import annotations

from .. import _native as N
from ..core import World
from ..shapes import min_contact_distance
from . import register
from ._fused import FusedScenario, HostReset, f32
from .catalog import GAPS, Passage as _Reference


@register("passage")
class Passage(HostReset, FusedScenario):
    native_id = N.SCN_PASSAGE
    max_steps = 250
    _reference = _Reference

    def __init__(self, collision_penalty: float = 0.5):
        _Reference.__init__(self, collision_penalty)

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def obs_dim(self, world):
        return 10 + 2 * (len(world.agents) - 1)

    def physics_fused(self, world) -> bool:
        return False         # world_step's generic kernel, then k_passage

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def fill_constants(self, world, d):
        a = world.agents[0].shape
        d.sc[0] = f32(min_contact_distance(a, a) + 0.0)     # common.touching
        d.sc[1] = f32(self.collision_penalty)
        d.sc[2] = f32(0.05)
        d.sd[0], d.sd[1] = float(GAPS[0]), float(GAPS[1])
