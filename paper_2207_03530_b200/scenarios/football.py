"""football (swarmsim/scenarios/football.py), fused reward / observation.

Two-a-side: the controlled blue team attacks against scripted reds.  The
reds' chase script runs on the device before the step (Env's host-decode
path), physics (ball, fences and nets as line segments) is world_step's
generic kernel, and the rest of the step — count, goal test, reward
10 * right - 10 * left - 0.1 * gap for blues (0 for scripted reds), done,
observation — is k_football<n> (csrc/ss_small.cu).  Resets run the
reference's host program.
"""
from __future__ import annotations

from .. import _native as N
from ..core import World
from . import register
from ._fused import FusedScenario, HostReset, f32
from .catalog import FIELD_HX, Football as _Reference


@register("football")
class Football(HostReset, FusedScenario):
    native_id = N.SCN_FOOTBALL
    max_steps = 400
    _reference = _Reference

    def __init__(self, n_per_team: int = 2, ball_mass: float = 0.25):
        _Reference.__init__(self, n_per_team, ball_mass)

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def obs_dim(self, world):
        return 8 + 2 * (len(world.agents) - 1) + 2

    def physics_fused(self, world) -> bool:
        return False         # world_step's generic kernel, then k_football

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def fill_constants(self, world, d):
        d.sc[0] = f32(FIELD_HX + 0.04)     # _scored thresholds (python double)
        d.sc[1] = f32(0.1)
        d.sc[2] = f32(FIELD_HX)            # Vec2.full(B, FIELD_HX, 0.0): float32
        d.sd[0] = float(FIELD_HX)
